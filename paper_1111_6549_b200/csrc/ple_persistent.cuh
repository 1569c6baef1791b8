// ple_persistent.cuh -- persistent cooperative driver of the B200 PLE.
//
// One launch factors the whole matrix. CTA 0 is the panel CTA: it runs
// panel_factor_body for step w+1 as soon as every worker has finished the
// look-ahead tile (the 64-byte tile holding word w+1) of step w, i.e. while
// the workers are still streaming the rest of step w's trailing update.
// CTAs 1..G-1 are workers: per step they
//   claim   pre-work chunks (apply a chunk of rows -- multipliers, d,
//           compressed words -- then sweep them over the look-ahead tiles;
//           the panel CTA waits on their completion count), so the workers
//           idle at the step barrier do it and the last one finds none left,
//   wait    until every worker finished step w-1 (the pivot rows' raw tails
//           are then final; tables read them in place, and the pivot rows'
//           own swept tails go to ubuf, so no staging copy is needed) and all
//           pre-work of step w is done,
//   update  their linear share of the remaining tiles.
// Cross-CTA ordering uses release/acquire counters in SyncState; every wait
// has a watchdog so a bug turns into an error code, not a hung GPU. The grid
// is launched cooperatively, so all CTAs are co-resident.
#pragma once

#include "ple_kernels.cuh"

namespace gf2cu {

__device__ __forceinline__ bool cta_wait(SyncState* sy, const u32* ctr, u32 target, u32& s_ok) {
    if (threadIdx.x == 0) s_ok = spin_geq(ctr, target, &sy->error) ? 1u : 0u;
    __syncthreads();
    return s_ok != 0;
}

// CTA arrival on a device-scope counter. The barrier orders every thread's
// prior writes before thread 0's red.release.gpu, and a release is cumulative
// over what is ordered before it (PTX memory model: bar.sync synchronizes the
// CTA, causality order is transitive), so no separate fence is needed -- the
// same pattern as CUTLASS's GenericBarrier::arrive_inc. (An explicit
// __threadfence() before it cost 0.1-0.6 %, paired A/B.)
__device__ __forceinline__ void cta_arrive(u32* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        red_release_add(ctr, 1u);
    }
}

// Panel CTA of the persistent drivers: the last warp only signals. After each
// panel the body threads sync among themselves and thread 0 publishes the step
// in shared memory (release, CTA scope); one signal thread acquires it, fences
// the panel's global outputs and publishes the step to the workers
// (panel_done), and polls the error word -- so the fence latency is off the
// panels' critical path. Spins have the watchdog; a step index of
// 0x80000000 | (w + 1) means "last step".
__device__ __forceinline__ void signal_step(PanelShared& sh, int nbody, u32 w, bool last) {
    named_bar(kBodyBar, nbody);
    if (threadIdx.x == 0) st_release_cta(&sh.sig_step, (int)((w + 1u) | (last ? 0x80000000u : 0u)));
}

__device__ __noinline__ void signal_loop(PanelShared& sh, SyncState* sy, u32 nsteps, u32 first = 0u) {
    for (u32 w = first; w < nsteps; ++w) {
        const u64 t0 = globaltimer();
        u32 st;
        for (u32 spin = 0;; ++spin) {
            st = (u32)ld_acquire_cta(&sh.sig_step);
            if ((st & 0x7fffffffu) >= w + 1u) break;
            if ((spin & 255u) == 255u) {
                if (*(volatile u32*)&sy->error) {
                    *(volatile int*)&sh.sig_err = 1;
                    return;
                }
                if (globaltimer() - t0 > g_watchdog_ns) {
                    atomicExch(&sy->error, 1u);
                    *(volatile int*)&sh.sig_err = 1;
                    return;
                }
            }
        }
        red_release_add(&sy->panel_done, 1u);  // (cumulative over the body's writes, see cta_arrive)
        if (*(volatile u32*)&sy->error) *(volatile int*)&sh.sig_err = 1;
        if (st & 0x80000000u) return;
    }
}

__device__ __forceinline__ void stamp(const Params& p, u32 w, u32 k) {
    if (p.phase_ns && threadIdx.x == 0) p.phase_ns[(size_t)w * 8 + k] = globaltimer();
}

__global__ void __launch_bounds__(kTrailThreads, 1) ple_persistent_kernel(Params p, u32 nsteps) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ PanelShared psh;
    __shared__ ApplyShared ash;
    __shared__ u32 s_ok;
    __shared__ u32 s_piv[64];  // physical rows of the step's pivots
    SyncState* sy = p.sync;
    const u32 nworkers = gridDim.x - 1;

    if (blockIdx.x == 0) {
        // ------------------------------------------------------ panel CTA
        // Look-ahead: step w+1's window words are computed at the end of step
        // w, so the next factorization starts at once; only its scans and its
        // writeback wait for the workers' look-ahead capture of step w.
        // The last warp only signals: after each panel it fences the panel's
        // global outputs and publishes the step (and polls the error word),
        // while the other warps go on with the next panel.
        const int nbody = (int)blockDim.x - 32;
        if (threadIdx.x == 0) {
            psh.sig_step = 0;
            psh.sig_err = 0;
        }
        __syncthreads();
        if ((int)threadIdx.x >= nbody) {
            if (threadIdx.x == (u32)nbody) signal_loop(psh, sy, nsteps);
            return;
        }
        LookAhead la{0u, false, p.ap_done, 0u, &sy->error};
        u32 prev_r = 0u;
        for (u32 w = 0; w < nsteps; ++w) {
            // step w-1's look-ahead capture = all of its pre-work chunks
            la.cap_ctr = p.ap_done + (w > 0 ? w - 1 : 0);
            la.cap_target = w > 0 ? pw_chunks(p.m - prev_r, p.pw_div) : 0u;
            prev_r = la.r;
            stamp(p, w, 0);
            const u32 rb = panel_factor_body<true>(p, w, psh, nbody, &la);
            stamp(p, w, 1);
            // (an aborted panel returns 0: then check the error word itself)
            if (rb == 0u && *(volatile u32*)&sy->error) {
                if (threadIdx.x == 0) st_release_cta(&psh.sig_step, (int)(0x80000000u | (w + 1u)));
                return;
            }
            const bool done = la.r >= p.m;
            signal_step(psh, nbody, w, done);
            if (done || *(volatile int*)&psh.sig_err) return;
            la.r += rb;
            la.have_window = true;
        }
        return;
    }

    // ---------------------------------------------------------- workers
    const u32 wk = blockIdx.x - 1;
    for (u32 w = 0; w < nsteps; ++w) {
        if (!cta_wait(sy, &sy->panel_done, w + 1, s_ok)) return;
        // this step's r / rb (the shared state word may already belong to the
        // next step: the panel CTA runs ahead)
        const u32 r = *(volatile u32*)&p.rhist[w], rb = *(volatile u32*)&p.rbhist[w];
        if (r >= p.m) return;
        Params q = p;
        q.info = p.info + (size_t)(w & 1u) * p.m;
        const u32 nrows = p.m - r;
        const bool sweep = w + 1 < p.W;
        const u32 tile0 = (w + 1) >> 3, tcap = cap_last_tile(w, p.W);
        const u32 crow = pw_rows(nrows, p.pw_div), nch = pw_chunks(nrows, p.pw_div);
        for (u32 k = threadIdx.x; k < rb; k += blockDim.x) s_piv[k] = ldcg(p.perm + r + k);
        __syncthreads();
        if (wk == 0) stamp(p, w, 2);

        // Pre-work chunks of step w (apply + look-ahead tiles of crow rows),
        // claimed from a per-step counter: the workers waiting for the last
        // one of step w-1 do (nearly) all of it. Its tiles were finished by
        // step w-1's look-ahead sweep, unless a new tile joins this step.
        if (sweep && !early_cap(w, p.W) && w > 0 &&
            !cta_wait(sy, &sy->t_count, nworkers * w, s_ok))
            return;
        u32 mine = 0;
        bool loaded = false;
        for (;;) {
            if (threadIdx.x == 0) s_ok = atomicAdd(&p.ap_claim[w], 1u);
            __syncthreads();
            const u32 c = s_ok;
            __syncthreads();
            if (c >= nch) break;
            if (!loaded) {  // pout is step w's while any chunk of it is open
                apply_load(q, ash, rb);
                __syncthreads();
                loaded = true;
            }
            const u32 a0 = r + c * crow, a1 = min(p.m, a0 + crow);
            apply_rows(q, ash, w, r, rb, a0, a1, threadIdx.x, blockDim.x);
            if (sweep) {
                for (u32 tt = tile0; tt <= tcap; ++tt) {
                    __syncthreads();
                    if (rb > 0) {
                        build_tables(q, smem, tt, w, rb, s_piv);
                        __syncthreads();
                    }
                    trail_rows(q, smem, w, r, tt, a0 - r, a1 - a0, rb);
                }
            }
            ++mine;
        }
        if (mine) {
            __syncthreads();
            if (threadIdx.x == 0) red_release_add(&p.ap_done[w], mine);  // (see cta_arrive)
        }
        // the rest: after step w-1 everywhere (the pivot rows' raw tails are
        // final; tables read them in place, their swept tails go to ubuf) and
        // all pre-work of step w (every row's info and compressed words)
        if (threadIdx.x == 0)
            s_ok = spin_geq2(&sy->t_count, nworkers * w, &p.ap_done[w], nch, &sy->error) ? 1u : 0u;
        __syncthreads();
        if (!s_ok) return;
        if (wk == 0) stamp(p, w, 3);
        if (sweep) {
            if (p.worker_ns && threadIdx.x == 0)
                p.worker_ns[((size_t)w * nworkers + wk) * 2] = globaltimer();
            const u32 nt = (p.Wpad8 >> 3) - tcap - 1;
            const u64 total = (u64)nt * nrows;
            trail_share(q, smem, w, r, rb, tcap + 1, total * wk / nworkers,
                        total * (wk + 1) / nworkers, s_piv);
        }
        if (p.worker_ns && threadIdx.x == 0) {
            p.worker_ns[((size_t)w * nworkers + wk) * 2 + 1] = globaltimer();
            if (w == 0) {
                u32 smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                p.worker_ns[((size_t)nsteps * nworkers + wk) * 2] = smid;
            }
        }
        cta_arrive(&sy->t_count);
        if (wk == 0) stamp(p, w, 5);
    }
}

}  // namespace gf2cu
