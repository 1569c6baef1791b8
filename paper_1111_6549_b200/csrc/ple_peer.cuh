// ple_peer.cuh -- row-sharded block_iterative_ple driven entirely on the
// device, ranks exchanging through peer memory.
//
// Rows are distributed block-cyclically (row g on rank (g / B) % G, local
// index (g / (B G)) B + g % B, as in ple_shard.cuh) and never move. Every
// rank runs one persistent kernel: CTA 0 is its panel CTA, the others are
// workers, exactly as in the single-GPU persistent driver
// (ple_persistent.cuh), and every rank keeps its own replica of the position
// state (perm, inv, r, the panel outputs), updated by its own panel CTA with
// the same deterministic factorization. What the single-GPU driver reads from
// one HBM, a rank receives through stores its peers make into its memory:
//
//   pb[w&1], pb2[w&1]  position-indexed panel words (word w and, for the
//                      look-ahead window, word w+1 before step w): every
//                      rank's look-ahead sweep of step w-1 stores its own
//                      rows' words into EVERY rank's buffers; the last of its
//                      pre-work chunks then signals kCtrCap on every rank.
//   stage[w&1]         step w's pivot-row tails (the Gray-table sources):
//                      the owner of each pivot row stores it into every
//                      rank's stage, in two parts -- the look-ahead tiles as
//                      soon as the panel is known (kCtrLa), the remaining
//                      tiles once its own step w-1 sweep is done (kCtrSt).
//
// All counters are cumulative over the launch (targets G*(w+1)), signalled
// with system-scope release reductions and waited on with system-scope
// acquire loads, so the same kernel runs one rank per GPU over NVLink peer
// mappings, or G ranks in ONE cooperative launch on one GPU (the emulation
// the tests use: the ranks' CTAs are co-resident, so their waits on one
// another cannot deadlock). Double-buffering by step parity is safe because
// every rank's step w+1 traffic into buffer (w+1)&1 is ordered after every
// rank's step w-1 reads of it by the counters above.
#pragma once

#include "ple_kernels.cuh"
#include "ple_shard.cuh"

namespace gf2cu {

constexpr int kMaxRanks = 8;

// The buffers of one rank that its peers write into.
struct PeerBufs {
    u64* pb[2];
    u64* pb2[2];
    u64* stage[2];
    u32* ctr;  // kCtr* words
};
constexpr int kCtrCap = 0;  // +1 per rank per step: its look-ahead captures landed
constexpr int kCtrLa = 1;   // +1 per rank per step: its pivots' look-ahead tiles staged
constexpr int kCtrSt = 2;   // +1 per rank per step: its pivots' remaining tiles staged
constexpr int kCtrErr = 3;  // watchdog tripped somewhere (set on every rank)
constexpr int kCtrPing = 8; // [8, 16): gf2cu_peer_ping markers, one word per sender rank
constexpr int kCtrWords = 16;

struct SuperOut;

struct PeerParams {
    Params p;             // this rank's replicated state (p.m = global rows); p.sync, p.ap_* local
    u64* mat;             // this rank's rows, tile-major (m_loc rows per tile)
    ulonglong2* info[2];  // per local row {d, (position << 32) | local row}, by step parity
                          // (super-step form: {d~_a, d_b}, positions in ipos)
    u32* ipos[2];         // super-step form: position of each local row, by parity
    PanelOut* pout_b;     // super-step form: panel b's outputs and the panel-side extras
    SuperOut* so;
    u32* lo;              // [W+1]: first local row still active at step w (lo[0] unused)
    u32 m_loc, rank, nranks, block;
    PeerBufs peer[kMaxRanks];  // every rank's buffers, this rank's included
};

__device__ __forceinline__ void peer_signal(const PeerParams& s, int which) {
    __threadfence_system();
    for (u32 j = 0; j < s.nranks; ++j) red_release_add_sys(s.peer[j].ctr + which, 1u);
}

__device__ __forceinline__ void peer_fail(const PeerParams& s) {
    for (u32 j = 0; j < s.nranks; ++j) atomicExch(s.peer[j].ctr + kCtrErr, 1u);
}

// One thread waits (local counter, gpu scope), the CTA learns the outcome.
__device__ __forceinline__ bool peer_wait(const PeerParams& s, const u32* ctr, u32 target, bool sys,
                                          u32& s_ok) {
    if (threadIdx.x == 0) {
        u32* err = s.peer[s.rank].ctr + kCtrErr;
        const bool ok = sys ? spin_geq_sys(ctr, target, err) : spin_geq(ctr, target, err);
        if (!ok) peer_fail(s);
        s_ok = ok ? 1u : 0u;
    }
    __syncthreads();
    return s_ok != 0;
}

// Local rows [l0, l1) of step w: multipliers, the combination d of raw pivot
// rows, the compressed write (apply_rows with rows addressed locally and
// positions looked up in inv). Rows already retired get d = 0; the smallest
// row still active at step w+1 goes to lo[w+1].
template <bool Check>
__device__ __forceinline__ void peer_apply_rows_t(const PeerParams& s, const ApplyShared& a, u32 w,
                                                  u32 r, u32 rb, const u64* pbw, ulonglong2* info,
                                                  u32 l0, u32 l1) {
    const u32 w0 = r >> 6, b0 = r & 63;
    u32 lomin = 0xffffffffu;
    for (u32 l = l0 + threadIdx.x; l < l1; l += blockDim.x) {
        const u32 g = shard_global(l, s.rank, s.nranks, s.block);
        const u32 pos = ldcg(s.p.inv + g);
        if (pos < r) {
            info[l] = make_ulonglong2(0ull, ((u64)pos << 32) | l);
            continue;
        }
        if (pos >= r + rb) lomin = min(lomin, l);
        u64 v = ldcg(pbw + pos), acc = 0, c = 0;
        const u32 off = pos - r;
        const u32 tl = off < rb ? off : rb;
#pragma unroll 8
        for (u32 k = 0; k < 64; ++k) {
            if (k >= tl) break;
            const u64 bit = (v >> a.q[k]) & 1ull;
            const u64 msk = 0ull - bit;
            v ^= a.E[k] & msk;
            acc ^= a.D[k] & msk;
            c |= bit << k;
        }
        u64 epart = 0;
        if constexpr (Check) check_panel_word(s.p.check, w, v, tl, off < rb, a.q);
        if (off < rb) {
            c |= 1ull << off;
            epart = v & ~low_mask64((int)a.q[off] + 1);
        }
        info[l] = make_ulonglong2(acc, ((u64)pos << 32) | l);
        const u64 clo = c << b0;
        const u64 chi = b0 ? (c >> (64 - b0)) : 0ull;
        if (w0 == w) {
            *tword(s.mat, s.m_loc, l, w) = clo | epart;
        } else {
            u64* x0 = tword(s.mat, s.m_loc, l, w0);
            *x0 = ldcg(x0) | clo;
            if (w0 + 1 == w) {
                *tword(s.mat, s.m_loc, l, w) = chi | epart;
            } else {
                if (chi) {
                    u64* x1 = tword(s.mat, s.m_loc, l, w0 + 1);
                    *x1 = ldcg(x1) | chi;
                }
                *tword(s.mat, s.m_loc, l, w) = epart;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lomin = min(lomin, __shfl_xor_sync(0xffffffffu, lomin, o));
    if ((threadIdx.x & 31) == 0 && lomin != 0xffffffffu) atomicMin(s.lo + w + 1, lomin);
}

// This rank's pivot rows of step w (piv = global rows of pivots 0..rb-1),
// tiles [t0, t1], into every rank's stage[w & 1]; 16-byte units split as
// part `part` of `nparts`.
__device__ __forceinline__ void peer_ship(const PeerParams& s, const u32* piv, u32 rb, u32 w,
                                          u32 t0, u32 t1, u32 part, u32 nparts) {
    if (t1 < t0 || rb == 0) return;
    const u32 per = (t1 - t0 + 1) * 4u;
    const u32 units = rb * per;
    for (u32 e = part * blockDim.x + threadIdx.x; e < units; e += nparts * blockDim.x) {
        const u32 k = e / per, rem = e - k * per;
        const u32 tt = t0 + (rem >> 2), q = rem & 3u;
        const u32 g = piv[k];
        if (shard_owner(g, s.nranks, s.block) != s.rank) continue;
        const u32 l = shard_local(g, s.nranks, s.block);
        const ulonglong2 v = ldcg(reinterpret_cast<const ulonglong2*>(
            s.mat + (((size_t)tt * s.m_loc + l) << 3) + 2u * q));
        const size_t off = (((size_t)tt * 64u + k) << 3) + 2u * q;
        for (u32 j = 0; j < s.nranks; ++j)
            *reinterpret_cast<ulonglong2*>(s.peer[j].stage[w & 1u] + off) = v;
    }
}

// The part of step w's remaining-tile shipment that this worker's own step
// w-1 sweep share finalized: the share is units [beg, end) of (tile, local
// row) pairs over tiles from tlo and rows [lo, lo + nrows), tile-major, so
// for one pivot row the tiles inside it are a contiguous range. Tiles below
// t_first (step w's look-ahead tiles, shipped separately) are skipped.
__device__ __forceinline__ void peer_ship_share(const PeerParams& s, const u32* piv, u32 rb, u32 w,
                                                u32 t_first, u32 ntiles, u32 tlo, u32 lo,
                                                u32 nrows, u64 beg, u64 end) {
    if (nrows == 0 || beg >= end) return;
    // the share runs from (tile bt, row br) to (tile et, row er), inclusive
    const u32 bt = (u32)(beg / nrows), br = (u32)(beg - (u64)bt * nrows);
    const u32 et = (u32)((end - 1) / nrows), er = (u32)(end - 1 - (u64)et * nrows);
    // all (pivot, tile, 16-byte chunk) units at once, so the loads overlap
    const u32 span = (et - bt + 1u) * 4u;
    for (u32 e = threadIdx.x; e < rb * span; e += blockDim.x) {
        const u32 k = e / span, rem = e - k * span;
        const u32 g = piv[k];
        if (shard_owner(g, s.nranks, s.block) != s.rank) continue;
        const u32 l = shard_local(g, s.nranks, s.block);
        if (l < lo || l >= lo + nrows) continue;
        const u32 off = l - lo;
        const u32 t = bt + (rem >> 2), q = rem & 3u;  // share-relative tile
        if ((t == bt && off < br) || (t == et && off > er)) continue;
        const u32 tt = tlo + t;
        if (tt < t_first || tt >= ntiles) continue;
        const ulonglong2 v = ldcg(reinterpret_cast<const ulonglong2*>(
            s.mat + (((size_t)tt * s.m_loc + l) << 3) + 2u * q));
        const size_t o = (((size_t)tt * 64u + k) << 3) + 2u * q;
        for (u32 j2 = 0; j2 < s.nranks; ++j2)
            *reinterpret_cast<ulonglong2*>(s.peer[j2].stage[w & 1u] + o) = v;
    }
}

// Local rows [row0, row0 + cnt) of tile `tile` (trail_rows with rows indexed
// locally): tail ^= sum_g T_g[byte_g(d)]; the tile holding word w+1 (w+2)
// stores each active row's new word into every rank's pb (pb2) at the row's
// position. Tables must be built.
__device__ __forceinline__ void peer_trail_rows(const PeerParams& s, const unsigned char* smem,
                                                u32 w, u32 r, u32 tile, u32 row0, u32 cnt,
                                                const ulonglong2* info) {
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3u, par = rg & 1u;
    const u32 cap_word = w + 1;
    const bool capture1 = (cap_word >> 3) == tile;
    const bool cap_lane = capture1 && ((cap_word & 7u) >> 1) == ch;
    const bool cap_hi = (cap_word & 1u) != 0;
    const u32 cap2_word = w + 2;
    const bool capture2 = cap2_word < s.p.W && (cap2_word >> 3) == tile;
    const bool cap2_lane = capture2 && ((cap2_word & 7u) >> 1) == ch;
    const bool cap2_hi = (cap2_word & 1u) != 0;
    const bool capture = capture1 || capture2;
    const u32 nxt = (w + 1u) & 1u;
    const u32 lane_row = wid * 8u + rg;
    u32 lsel[4], lkoff[4];
    lookup8_consts(par, ch, lsel, lkoff);
    u64* tbase = s.mat + (((size_t)tile * s.m_loc) << 3) + 2u * ch;
    const u32 rend = row0 + cnt;
    const u32 nit = (cnt + kRowsPerIter - 1) / kRowsPerIter;

    ulonglong2 infC[kUnroll], infN[kUnroll], valC[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 4);
        infC[k] = ld_info(info, ri, ri < rend);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
        infN[k] = ld_info(info, ri, ri < rend);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 4);
        const bool act = (u32)(infC[k].y >> 32) >= r;
        valC[k] = make_ulonglong2(0ull, 0ull);
        if (ri < rend && (infC[k].x != 0ull || (capture && act)))
            valC[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((infC[k].y & 0xffffffffull) << 3)));
    }
    for (u32 it = 0; it < nit; ++it) {
        const u32 base = row0 + it * kRowsPerIter;
        ulonglong2 valN[kUnroll], infNN[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
            const bool act = (u32)(infN[k].y >> 32) >= r;
            valN[k] = make_ulonglong2(0ull, 0ull);
            if (ri < rend && (infN[k].x != 0ull || (capture && act)))
                valN[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((infN[k].y & 0xffffffffull) << 3)));
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + 2 * kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
            infNN[k] = ld_info(info, ri, ri < rend);
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + lane_row + (u32)k * (kTrailThreads / 4);
            const u64 d = infC[k].x;
            if (d != 0ull && ri < rend) {
                lookup8(valC[k], smem, d, lsel, lkoff);
                *reinterpret_cast<ulonglong2*>(tbase + ((infC[k].y & 0xffffffffull) << 3)) = valC[k];
            }
            const u32 pos = (u32)(infC[k].y >> 32);
            if (ri < rend && pos >= r) {
                if (cap_lane) {
                    const u64 v1 = cap_hi ? valC[k].y : valC[k].x;
                    for (u32 j = 0; j < s.nranks; ++j) s.peer[j].pb[nxt][pos] = v1;
                }
                if (cap2_lane) {
                    const u64 v2 = cap2_hi ? valC[k].y : valC[k].x;
                    for (u32 j = 0; j < s.nranks; ++j) s.peer[j].pb2[nxt][pos] = v2;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            infC[k] = infN[k];
            infN[k] = infNN[k];
            valC[k] = valN[k];
        }
    }
}

// Share [beg, end) of the (tile, local row) work over tiles from tile_lo and
// local rows [lo, m_loc); tables from stage[w & 1], rebuilt per tile segment.
__device__ __forceinline__ void peer_trail_share(const PeerParams& s, const Params& q,
                                                 unsigned char* smem, u32 w, u32 r, u32 rb,
                                                 u32 lo, u32 tile_lo, u64 beg, u64 end,
                                                 const ulonglong2* info) {
    const u32 nrows = s.m_loc - lo;
    u64 u = beg;
    while (u < end) {
        const u32 tile = tile_lo + (u32)(u / nrows);
        const u32 row0 = (u32)(u % nrows);
        const u32 cnt = (u32)min((u64)(nrows - row0), end - u);
        if (rb > 0) {
            __syncthreads();
            build_tables(q, smem, tile, w, rb);
            __syncthreads();
            peer_trail_rows(s, smem, w, r, tile, lo + row0, cnt, info);
        }
        u += cnt;
    }
}

// One launch = the whole factorization of every rank in `ranks` (one per GPU,
// or all of them in the one-GPU emulation); cpr CTAs per rank.
__global__ void __launch_bounds__(kTrailThreads, 1)
    ple_peer_kernel(const PeerParams* __restrict__ ranks, u32 cpr, u32 nsteps) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ PeerParams s;
    __shared__ PanelShared psh;
    __shared__ ApplyShared ash;
    __shared__ u32 s_ok;
    __shared__ u32 s_piv[64];
    {
        const u32* src = reinterpret_cast<const u32*>(ranks + blockIdx.x / cpr);
        u32* dst = reinterpret_cast<u32*>(&s);
        for (u32 i = threadIdx.x; i < sizeof(PeerParams) / 4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const Params& p = s.p;
    SyncState* sy = p.sync;
    u32* ctr = s.peer[s.rank].ctr;
    u32* err = ctr + kCtrErr;
    const u32 G = s.nranks, cta = blockIdx.x % cpr, nworkers = cpr - 1;

    if (cta == 0) {
        // ---------------------------------------------------- panel CTA
        if (!peer_wait(s, ctr + kCtrCap, G, true, s_ok)) return;  // every rank's init
        LookAhead la{0u, false, ctr + kCtrCap, 0u, err};
        la.sys = true;
        for (u32 w = 0; w < nsteps; ++w) {
            la.cap_target = G * (w + 1u);  // every rank's step w-1 captures
            Params q = p;
            q.pb = s.peer[s.rank].pb[w & 1u];
            q.pb2 = s.peer[s.rank].pb2[w & 1u];
            const u32 rb = panel_factor_body<true>(q, w, psh, blockDim.x, &la);
            if (*(volatile u32*)err) {
                if (threadIdx.x == 0) peer_fail(s);
                return;
            }
            const bool done = la.r >= p.m;
            cta_arrive(&sy->panel_done);
            if (done) return;
            la.r += rb;
            la.have_window = true;
        }
        return;
    }

    // -------------------------------------------------------------- workers
    const u32 wk = cta - 1;
    {
        // init (step -1): identity position state, and every rank's pb[0] /
        // pb2[0] get this rank's rows' words 0 and 1 (position = global row)
        const u32 gt = wk * blockDim.x + threadIdx.x, gs = nworkers * blockDim.x;
        for (u32 i = gt; i < p.m; i += gs) {
            p.perm[i] = i;
            p.inv[i] = i;
        }
        for (u32 l = gt; l < s.m_loc; l += gs) {
            const u32 g = shard_global(l, s.rank, s.nranks, s.block);
            const u64 v0 = *tword(s.mat, s.m_loc, l, 0);
            const u64 v1 = p.W > 1 ? *tword(s.mat, s.m_loc, l, 1) : 0ull;
            for (u32 j = 0; j < G; ++j) {
                s.peer[j].pb[0][g] = v0;
                s.peer[j].pb2[0][g] = v1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&sy->cap_count, 1u) == nworkers - 1u) peer_signal(s, kCtrCap);
        }
    }
    // this worker's sweep share of the previous step (tile-major units
    // [pbeg, pend) over tiles from ptlo and local rows [plo, plo + pnrows))
    u32 ptlo = 0, plo = 0, pnrows = 0;
    u64 pbeg = 0, pend = 0;
    const u32 ntiles = p.Wpad8 >> 3;
    for (u32 w = 0; w < nsteps; ++w) {
        if (!peer_wait(s, &sy->panel_done, w + 1u, false, s_ok)) return;
        const u32 r = *(volatile u32*)&p.rhist[w], rb = *(volatile u32*)&p.rbhist[w];
        if (r >= p.m) return;
        const u32 lo = w ? min(ldcg(s.lo + w), s.m_loc) : 0u;
        const u32 nrows = s.m_loc - lo;
        Params q = p;
        q.stage = s.peer[s.rank].stage[w & 1u];
        ulonglong2* info = s.info[w & 1u];
        const u64* pbw = s.peer[s.rank].pb[w & 1u];
        const bool sweep = w + 1 < p.W;
        const u32 tile0 = (w + 1) >> 3, tcap = cap_last_tile(w, p.W);
        const u32 crow = pw_rows(max(nrows, 1u), p.pw_div);
        const u32 nch = nrows ? (nrows + crow - 1u) / crow : 0u;
        for (u32 k = threadIdx.x; k < rb; k += blockDim.x) s_piv[k] = ldcg(p.perm + r + k);
        __syncthreads();

        // close step w-1: stage on every rank the tiles of step w's pivot
        // rows that this worker's step w-1 share finished, then arrive; the
        // last arrival of the rank tells every rank (kCtrSt). One barrier per
        // step, as in the single-GPU driver.
        if (sweep && rb > 0 && tcap + 1u < ntiles) {
            if (w == 0)
                peer_ship(s, s_piv, rb, w, tcap + 1u, ntiles - 1u, wk, nworkers);
            else
                peer_ship_share(s, s_piv, rb, w, tcap + 1u, ntiles, ptlo, plo, pnrows, pbeg, pend);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&sy->t_count, 1u) == nworkers * (w + 1u) - 1u) peer_signal(s, kCtrSt);
        }

        // pre-work: job 0 stages this rank's pivots' look-ahead tiles on
        // every rank; jobs 1.. apply a chunk of local rows and sweep them
        // over the look-ahead tiles (capturing words w+1, w+2 everywhere)
        u32 mine = 0;
        bool loaded = false, la_ready = false;
        for (;;) {
            if (threadIdx.x == 0) s_ok = atomicAdd(&p.ap_claim[w], 1u);
            __syncthreads();
            const u32 job = s_ok;
            __syncthreads();
            if (job == 0) {
                if (sweep) {
                    if (!early_cap(w, p.W) && w > 0 &&
                        !peer_wait(s, &sy->t_count, nworkers * (w + 1u), false, s_ok))
                        return;
                    peer_ship(s, s_piv, rb, w, tile0, tcap, 0, 1);
                }
                __syncthreads();
                if (threadIdx.x == 0) peer_signal(s, kCtrLa);
                continue;
            }
            const u32 c = job - 1u;
            if (c >= nch) break;
            if (!loaded) {
                apply_load(p, ash, rb);
                __syncthreads();
                loaded = true;
            }
            const u32 l0 = lo + c * crow, l1 = min(s.m_loc, l0 + crow);
            if (s.p.check)
                peer_apply_rows_t<true>(s, ash, w, r, rb, pbw, info, l0, l1);
            else
                peer_apply_rows_t<false>(s, ash, w, r, rb, pbw, info, l0, l1);
            if (sweep) {
                __syncthreads();
                if (!la_ready) {
                    if (!peer_wait(s, ctr + kCtrLa, G * (w + 1u), true, s_ok)) return;
                    la_ready = true;
                }
                for (u32 tt = tile0; tt <= tcap; ++tt) {
                    __syncthreads();
                    if (rb > 0) {
                        build_tables(q, smem, tt, w, rb);
                        __syncthreads();
                    }
                    peer_trail_rows(s, smem, w, r, tt, l0, l1 - l0, info);
                }
            }
            ++mine;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // the chunk that completes the step's pre-work tells every rank
            // that this rank's captures landed
            if (mine) {
                // (gpu scope suffices here: the signalling thread's system-
                // scope fence and release are cumulative over what it saw)
                __threadfence();
                if (atomicAdd(&p.ap_done[w], mine) + mine == nch) peer_signal(s, kCtrCap);
            } else if (nch == 0 && wk == 0) {
                peer_signal(s, kCtrCap);
            }
        }

        // rest: after every local worker closed step w-1 (t_count) and all of
        // this step's pre-work (every row's info); then, for the sweep, after
        // every rank staged its pivots' remaining tiles (kCtrSt)
        if (threadIdx.x == 0) {
            s_ok = spin_geq2(&sy->t_count, nworkers * (w + 1u), &p.ap_done[w], nch, err) ? 1u : 0u;
            if (!s_ok) peer_fail(s);
        }
        __syncthreads();
        if (!s_ok) return;
        ptlo = tcap + 1u;
        plo = lo;
        pnrows = nrows;
        pbeg = pend = 0;
        if (sweep && tcap + 1u < ntiles && nrows > 0) {
            const u64 total = (u64)(ntiles - tcap - 1u) * nrows;
            pbeg = total * wk / nworkers;
            pend = total * (wk + 1u) / nworkers;
        }
        if (sweep && tcap + 1u < ntiles) {
            // (waited even without work: a rank's step w+2 stores into
            // stage[w & 1] must follow every rank's step w reads of it)
            if (!peer_wait(s, ctr + kCtrSt, G * (w + 1u), true, s_ok)) return;
            if (rb > 0 && pend > pbeg)
                peer_trail_share(s, q, smem, w, r, rb, lo, tcap + 1u, pbeg, pend, info);
        }
    }
}

// Diagnostic of the peer mappings: store `value` into word kCtrPing + rank of
// every rank's counter block (one thread; nothing waits on anything).
__global__ void peer_ping_kernel(const PeerParams* __restrict__ me, u32 value) {
    const PeerParams& s = *me;
    for (u32 j = 0; j < s.nranks; ++j) s.peer[j].ctr[kCtrPing + s.rank] = value;
    __threadfence_system();
}

// Global row-major -> every rank's tile-major local rows (blockIdx.y = rank;
// the one-GPU emulation's upload).
__global__ void peer_tile_kernel(const PeerParams* __restrict__ ranks, const u64* __restrict__ src,
                                 u32 Wp) {
    const PeerParams& s = ranks[blockIdx.y];
    const u32 per_row = s.p.Wpad8 >> 1;
    const u64 total = (u64)s.m_loc * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        const u32 l = (u32)(e / per_row), x = 2u * (u32)(e - (u64)l * per_row);
        const u32 g = shard_global(l, s.rank, s.nranks, s.block);
        *reinterpret_cast<ulonglong2*>(tword(s.mat, s.m_loc, l, x)) =
            *reinterpret_cast<const ulonglong2*>(src + (size_t)g * Wp + x);
    }
}

// Every rank's local rows -> global row-major at their final positions.
__global__ void peer_untile_kernel(const PeerParams* __restrict__ ranks, u64* __restrict__ dst, u32 Wp) {
    const PeerParams& s = ranks[blockIdx.y];
    const u32 per_row = s.p.Wpad8 >> 1;
    const u64 total = (u64)s.m_loc * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        const u32 l = (u32)(e / per_row), x = 2u * (u32)(e - (u64)l * per_row);
        const u32 pos = s.p.inv[shard_global(l, s.rank, s.nranks, s.block)];
        *reinterpret_cast<ulonglong2*>(dst + (size_t)pos * Wp + x) =
            *reinterpret_cast<const ulonglong2*>(tword(s.mat, s.m_loc, l, x));
    }
}

}  // namespace gf2cu
