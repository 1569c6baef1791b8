// ple_peer_super.cuh -- the row-sharded peer-memory driver (ple_peer.cuh)
// with two 64-column panels per trailing sweep, as in the single-GPU
// super-step driver (ple_super.cuh): 32-byte tiles, 16 Gray tables, every
// row's update new_tail = d~_a . R_a ^ d_b . R_b over the 128 raw pivot rows
// of the super-step. The exchange is that of ple_peer.cuh with the
// super-step S in place of the step w:
//   pb[S&1] / pb2[S&1]  words 2S / 2S+1 of every active position before
//                       super-step S, captured by every rank's look-ahead
//                       sweep of S-1 (the 32-byte tile holding them) into
//                       every rank's buffers (kCtrCap);
//   stage[S&1]          the 128 pivot rows' tails before S, 32-byte tiles:
//                       slot k < 64 = panel a's pivot k, 64 + k = panel b's;
//                       the look-ahead tile first (kCtrLa), the remaining
//                       tiles from each worker's previous sweep share at the
//                       step boundary (kCtrSt).
#pragma once

#include "ple_peer.cuh"
#include "ple_super.cuh"

namespace gf2cu {

constexpr u32 kSuperSlots = 128;  // stage rows per super-step (panel a, panel b)

__device__ __forceinline__ u64* stage4(u64* stage, u32 tile, u32 slot) {
    return stage + (((size_t)tile * kSuperSlots + slot) << 2);
}

// apply2_rows (ple_super.cuh) on local rows [l0, l1): positions from inv,
// records info[l] = {d~_a, d_b}, ipos[l] = position; lo[S+1] = the smallest
// local row still active after the super-step.
template <bool Check>
__device__ __forceinline__ void peer_apply2_rows_t(const PeerParams& s, const ApplyShared2& a, u32 S,
                                                 u32 r, u32 rba, u32 rbb, bool has_b,
                                                 const u64* pbw, const u64* pb2w, ulonglong2* info,
                                                 u32* ipos, u32 l0, u32 l1) {
    const u32 w = 2u * S, rb0 = r + rba;
    u32 lomin = 0xffffffffu;
    for (u32 l = l0 + threadIdx.x; l < l1; l += blockDim.x) {
        const u32 pos = ldcg(s.p.inv + shard_global(l, s.rank, s.nranks, s.block));
        ipos[l] = pos;
        if (pos < r) {
            info[l] = make_ulonglong2(0ull, 0ull);
            continue;
        }
        if (pos >= rb0 + rbb) lomin = min(lomin, l);
        u64 v = ldcg(pbw + pos);
        const u64 x1 = has_b ? ldcg(pb2w + pos) : 0ull;
        const u32 off = pos - r;
        const u32 tla = off < rba ? off : rba;
        u64 c = 0ull, da = 0ull, epa = 0ull;
#pragma unroll 8
        for (u32 k = 0; k < 64; ++k) {
            if (k >= tla) break;
            const u64 bit = (v >> a.qa[k]) & 1ull;
            const u64 msk = 0ull - bit;
            v ^= a.Ea[k] & msk;
            da ^= a.Da[k] & msk;
            c |= bit << k;
        }
        if constexpr (Check) check_panel_word(s.p.check, w, v, tla, off < rba, a.qa);
        if (off < rba) {
            c |= 1ull << off;
            epa = v & ~low_mask64((int)a.qa[off] + 1);
        }
        compress_write(s.mat, s.m_loc, l, r, w, c, epa);
        u64 db = 0ull, dta = da;
        if (has_b) {
            u64 v1 = x1;  // word w+1 after panel a
#pragma unroll 8
            for (u32 k = 0; k < 64; ++k) {
                if (k >= rba) break;
                v1 ^= a.piv2[k] & (0ull - ((da >> k) & 1ull));
            }
            if (pos < rb0) {
                *tw4(s.mat, s.m_loc, l, w + 1u) = v1;  // a pivot row of panel a: its U word w+1
            } else {
                const u32 offb = pos - rb0;
                const u32 tlb = offb < rbb ? offb : rbb;
                u64 cb = 0ull, epb = 0ull;
#pragma unroll 8
                for (u32 k = 0; k < 64; ++k) {
                    if (k >= tlb) break;
                    const u64 bit = (v1 >> a.qb[k]) & 1ull;
                    const u64 msk = 0ull - bit;
                    v1 ^= a.Eb[k] & msk;
                    db ^= a.Db[k] & msk;
                    cb |= bit << k;
                }
                if constexpr (Check) check_panel_word(s.p.check, w + 1u, v1, tlb, offb < rbb, a.qb);
                if (offb < rbb) {
                    cb |= 1ull << offb;
                    epb = v1 & ~low_mask64((int)a.qb[offb] + 1);
                }
                compress_write(s.mat, s.m_loc, l, rb0, w + 1u, cb, epb);
#pragma unroll 8
                for (u32 k = 0; k < 64; ++k) {
                    if (k >= rbb) break;
                    dta ^= a.C[k] & (0ull - ((db >> k) & 1ull));
                }
            }
        }
        info[l] = make_ulonglong2(dta, db);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lomin = min(lomin, __shfl_xor_sync(0xffffffffu, lomin, o));
    if ((threadIdx.x & 31) == 0 && lomin != 0xffffffffu) atomicMin(s.lo + S + 1u, lomin);
}

// build16 (ple_super.cuh) with the 128 pivot rows read from the stage.
__device__ __forceinline__ void peer_build16(unsigned char* smem, const u64* stage, u32 tile, u32 w,
                                             u32 rba, u32 rbb) {
    const u32 tid = threadIdx.x;
    const u32 h = tid & 1u;
    const u32 t = (((tid >> 5) & 3u) << 2) | ((tid >> 1) & 3u);
    const u32 sg = (((tid >> 7) & 3u) << 2) | ((tid >> 3) & 3u);
    const u32 x0 = tile * 4u;
    const u32 zlim = w + 2u > x0 ? min(w + 2u - x0, 4u) : 0u;  // words <= w+1
    const u32 nsrc = t < 8u ? rba : rbb;
    const u32 base = 8u * (t & 7u);
    const u32 slot0 = (t < 8u ? 0u : 64u) + base;
    ulonglong2 R[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        ulonglong2 v = make_ulonglong2(0ull, 0ull);
        if (base + b < nsrc)
            v = ldcg(reinterpret_cast<const ulonglong2*>(stage4(const_cast<u64*>(stage), tile, slot0 + b) + 2u * h));
        if (2u * h < zlim) v.x = 0ull;
        if (2u * h + 1u < zlim) v.y = 0ull;
        R[b] = v;
    }
    const u32 i0 = 16u * sg;
    const u32 e0 = i0 ^ (i0 >> 1);
    ulonglong2 acc = make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int b = 3; b < 8; ++b)
        if ((e0 >> b) & 1u) xor2(acc, R[b]);
    *reinterpret_cast<ulonglong2*>(smem + tab16_off(t, e0, h)) = acc;
#pragma unroll
    for (u32 k = 1; k < 16; ++k) {
        const int b = (k & 1u) ? 0 : (k & 2u) ? 1 : (k & 4u) ? 2 : 3;
        xor2(acc, R[b]);
        const u32 i = i0 + k;
        *reinterpret_cast<ulonglong2*>(smem + tab16_off(t, i ^ (i >> 1), h)) = acc;
    }
}

// trail16_rows (ple_super.cuh) over local rows [row0, row0 + cnt), in place;
// the tile holding words w+2, w+3 stores every active row's new words into
// every rank's pb / pb2 for super-step S+1.
__device__ __forceinline__ void peer_trail16_rows(const PeerParams& s, const unsigned char* smem,
                                                  u32 S, u32 r, u32 tile, u32 row0, u32 cnt,
                                                  const ulonglong2* info, const u32* ipos) {
    const u32 w = 2u * S;
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const u32 rw = lane >> 1, h = lane & 1u, rq = rw & 3u;
    const bool capture = (w + 2u < s.p.W) && ((w + 2u) >> 2) == tile;
    const bool cap_lane = capture && (((w + 2u) & 3u) >> 1) == h;
    const bool cap2 = cap_lane && (w + 3u < s.p.W);
    const u32 nxt = (S + 1u) & 1u;
    const u32 lane_row = wid * 16u + rw;
    u32 lsel[4], lkoff[4];
    lookup16_consts(rq, h, lsel, lkoff);
    u64* tbase = s.mat + (((size_t)tile * s.m_loc) << 2) + 2u * h;
    const u32 rend = row0 + cnt;
    const u32 nit = (cnt + kRows16 - 1) / kRows16;
    ulonglong2 dC[kUnroll], dN[kUnroll], valC[kUnroll];
    u32 pC[kUnroll], pN[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 2);
        const bool v = ri < rend;
        dC[k] = v ? ldcg(info + ri) : make_ulonglong2(0ull, 0ull);
        pC[k] = v ? ldcg(ipos + ri) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + kRows16 + lane_row + (u32)k * (kTrailThreads / 2);
        const bool v = ri < rend;
        dN[k] = v ? ldcg(info + ri) : make_ulonglong2(0ull, 0ull);
        pN[k] = v ? ldcg(ipos + ri) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 2);
        valC[k] = make_ulonglong2(0ull, 0ull);
        if (ri < rend && ((dC[k].x | dC[k].y) != 0ull || (capture && pC[k] >= r)))
            valC[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)ri << 2)));
    }
    for (u32 it = 0; it < nit; ++it) {
        const u32 base = row0 + it * kRows16;
        ulonglong2 valN[kUnroll], dNN[kUnroll];
        u32 pNN[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + kRows16 + lane_row + (u32)k * (kTrailThreads / 2);
            valN[k] = make_ulonglong2(0ull, 0ull);
            if (ri < rend && ((dN[k].x | dN[k].y) != 0ull || (capture && pN[k] >= r)))
                valN[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)ri << 2)));
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + 2u * kRows16 + lane_row + (u32)k * (kTrailThreads / 2);
            const bool v = ri < rend;
            dNN[k] = v ? ldcg(info + ri) : make_ulonglong2(0ull, 0ull);
            pNN[k] = v ? ldcg(ipos + ri) : 0u;
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + lane_row + (u32)k * (kTrailThreads / 2);
            const ulonglong2 d = dC[k];
            if ((d.x | d.y) != 0ull && ri < rend) {
                lookup16(valC[k], smem, d, lsel, lkoff);
                *reinterpret_cast<ulonglong2*>(tbase + ((size_t)ri << 2)) = valC[k];
            }
            const u32 pos = pC[k];
            if (cap_lane && ri < rend && pos >= r) {
                for (u32 j = 0; j < s.nranks; ++j) s.peer[j].pb[nxt][pos] = valC[k].x;
                if (cap2)
                    for (u32 j = 0; j < s.nranks; ++j) s.peer[j].pb2[nxt][pos] = valC[k].y;
            }
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            dC[k] = dN[k];
            pC[k] = pN[k];
            dN[k] = dNN[k];
            pN[k] = pNN[k];
            valC[k] = valN[k];
        }
    }
}

__device__ __forceinline__ bool slot_valid(u32 k, u32 rba, u32 rbb) {
    return k < 64u ? k < rba : k - 64u < rbb;
}

// This rank's pivot rows of super-step S (piv = 128 slots of global rows),
// tiles [t0, t1], into every rank's stage[S & 1]; part `part` of `nparts`.
__device__ __forceinline__ void peer_ship4(const PeerParams& s, const u32* piv, u32 rba, u32 rbb,
                                           u32 S, u32 t0, u32 t1, u32 part, u32 nparts) {
    if (t1 < t0 || rba + rbb == 0) return;
    const u32 per = (t1 - t0 + 1u) * 2u;  // 16-byte units per row
    const u32 units = kSuperSlots * per;
    for (u32 e = part * blockDim.x + threadIdx.x; e < units; e += nparts * blockDim.x) {
        const u32 k = e / per, rem = e - k * per;
        if (!slot_valid(k, rba, rbb)) continue;
        const u32 g = piv[k];
        if (shard_owner(g, s.nranks, s.block) != s.rank) continue;
        const u32 tt = t0 + (rem >> 1), q = rem & 1u;
        const u32 l = shard_local(g, s.nranks, s.block);
        const ulonglong2 v = ldcg(reinterpret_cast<const ulonglong2*>(tw4(s.mat, s.m_loc, l, 4u * tt) + 2u * q));
        for (u32 j = 0; j < s.nranks; ++j)
            *reinterpret_cast<ulonglong2*>(stage4(s.peer[j].stage[S & 1u], tt, k) + 2u * q) = v;
    }
}

// The part of super-step S's remaining-tile shipment that this worker's own
// S-1 sweep share (units [beg, end) over tiles from tlo and local rows
// [lo, lo + nrows), tile-major) finished; tiles below t_first skipped.
__device__ __forceinline__ void peer_ship4_share(const PeerParams& s, const u32* piv, u32 rba, u32 rbb,
                                                 u32 S, u32 t_first, u32 ntiles, u32 tlo, u32 lo,
                                                 u32 nrows, u64 beg, u64 end) {
    if (nrows == 0 || beg >= end) return;
    const u32 bt = (u32)(beg / nrows), br = (u32)(beg - (u64)bt * nrows);
    const u32 et = (u32)((end - 1) / nrows), er = (u32)(end - 1 - (u64)et * nrows);
    const u32 span = (et - bt + 1u) * 2u;
    for (u32 e = threadIdx.x; e < kSuperSlots * span; e += blockDim.x) {
        const u32 k = e / span, rem = e - k * span;
        if (!slot_valid(k, rba, rbb)) continue;
        const u32 g = piv[k];
        if (shard_owner(g, s.nranks, s.block) != s.rank) continue;
        const u32 l = shard_local(g, s.nranks, s.block);
        if (l < lo || l >= lo + nrows) continue;
        const u32 off = l - lo;
        const u32 t = bt + (rem >> 1), q = rem & 1u;
        if ((t == bt && off < br) || (t == et && off > er)) continue;
        const u32 tt = tlo + t;
        if (tt < t_first || tt >= ntiles) continue;
        const ulonglong2 v = ldcg(reinterpret_cast<const ulonglong2*>(tw4(s.mat, s.m_loc, l, 4u * tt) + 2u * q));
        for (u32 j = 0; j < s.nranks; ++j)
            *reinterpret_cast<ulonglong2*>(stage4(s.peer[j].stage[S & 1u], tt, k) + 2u * q) = v;
    }
}

__global__ void __launch_bounds__(kTrailThreads, 1)
    ple_peer_super_kernel(const PeerParams* __restrict__ ranks, u32 cpr, u32 nss) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ PeerParams s;
    __shared__ PanelShared psh;
    __shared__ ApplyShared2 ash;
    __shared__ u32 s_ok;
    __shared__ u32 s_piv[kSuperSlots];
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
    const u32 Wpad4 = p.Wpad8;  // holds Wpad4 in this driver

    if (cta == 0) {
        // ---------------------------------------------------- panel CTA
        LookAhead la{0u, false, ctr + kCtrCap, 0u, err};
        la.sys = true;
        la.piv2_out = s.so->piv2;
        la.C_out = s.so->C;
        for (u32 S = 0; S < nss; ++S) {
            const u32 w = 2u * S;
            const bool done0 = la.r >= p.m;
            Params q = p;
            q.pb = s.peer[s.rank].pb[S & 1u];
            q.pb2 = s.peer[s.rank].pb2[S & 1u];
            // panel a: its window is every rank's capture of S-1 (init: S = 0)
            la.cap_target = G * (S + 1u);
            la.super_mode = 1;
            la.have_window = false;
            const u32 rba = panel_factor_body(q, w, psh, blockDim.x, &la);
            if (*(volatile u32*)err) {
                if (threadIdx.x == 0) peer_fail(s);
                return;
            }
            la.r += rba;
            if (w + 1u < p.W) {
                if (!done0 && la.r < p.m) {
                    la.super_mode = 2;
                    la.have_window = true;
                    la.cap_target = 0u;
                    Params qb = q;
                    qb.pout = s.pout_b;
                    const u32 rbb = panel_factor_body(qb, w + 1u, psh, blockDim.x, &la);
                    if (*(volatile u32*)err) {
                        if (threadIdx.x == 0) peer_fail(s);
                        return;
                    }
                    la.r += rbb;
                } else if (threadIdx.x == 0) {
                    p.rhist[w + 1u] = la.r;
                    p.rbhist[w + 1u] = 0u;
                }
            }
            cta_arrive(&sy->panel_done);
            if (done0) return;
        }
        return;
    }

    // -------------------------------------------------------------- workers
    const u32 wk = cta - 1;
    {
        const u32 gt = wk * blockDim.x + threadIdx.x, gs = nworkers * blockDim.x;
        for (u32 i = gt; i < p.m; i += gs) {
            p.perm[i] = i;
            p.inv[i] = i;
        }
        for (u32 l = gt; l < s.m_loc; l += gs) {
            const u32 g = shard_global(l, s.rank, s.nranks, s.block);
            const u64 v0 = *tw4(s.mat, s.m_loc, l, 0);
            const u64 v1 = p.W > 1 ? *tw4(s.mat, s.m_loc, l, 1) : 0ull;
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
    u32 ptlo = 0, plo = 0, pnrows = 0;
    u64 pbeg = 0, pend = 0;
    const u32 ntiles = Wpad4 >> 2;
    for (u32 S = 0; S < nss; ++S) {
        if (!peer_wait(s, &sy->panel_done, S + 1u, false, s_ok)) return;
        const u32 w = 2u * S;
        const bool has_b = w + 1u < p.W;
        const u32 r = *(volatile u32*)&p.rhist[w], rba = *(volatile u32*)&p.rbhist[w];
        if (r >= p.m) return;
        const u32 rbb = has_b ? *(volatile u32*)&p.rbhist[w + 1u] : 0u;
        const u32 lo = S ? min(ldcg(s.lo + S), s.m_loc) : 0u;
        const u32 nrows = s.m_loc - lo;
        ulonglong2* info = s.info[S & 1u];
        u32* ipos = s.ipos[S & 1u];
        const u64* stage = s.peer[s.rank].stage[S & 1u];
        const bool sweep = w + 2u < p.W;
        const u32 ct = (w + 2u) >> 2;  // look-ahead tile (words w+2, w+3)
        const u32 crow = pw_rows(max(nrows, 1u), p.pw_div);
        const u32 nch = nrows ? (nrows + crow - 1u) / crow : 0u;
        for (u32 k = threadIdx.x; k < kSuperSlots; k += blockDim.x)
            s_piv[k] = !slot_valid(k, rba, rbb) ? 0u
                       : k < 64u ? ldcg(p.perm + r + k) : ldcg(p.perm + r + rba + (k - 64u));
        __syncthreads();

        // close S-1: stage the tiles of S's pivot rows this worker's S-1
        // share finished, then arrive (the rank's last arrival: kCtrSt)
        if (sweep && rba + rbb > 0 && ct + 1u < ntiles) {
            if (S == 0)
                peer_ship4(s, s_piv, rba, rbb, S, ct + 1u, ntiles - 1u, wk, nworkers);
            else
                peer_ship4_share(s, s_piv, rba, rbb, S, ct + 1u, ntiles, ptlo, plo, pnrows, pbeg, pend);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&sy->t_count, 1u) == nworkers * (S + 1u) - 1u) peer_signal(s, kCtrSt);
        }

        // pre-work: job 0 stages the look-ahead tile of this rank's pivots
        // everywhere; jobs 1.. apply both panels to a chunk of local rows and
        // sweep it over the look-ahead tile (capturing words w+2, w+3)
        const bool early = S == 0 || ct == (w >> 2);
        u32 mine = 0;
        bool loaded = false, la_ready = false, built = false;
        for (;;) {
            if (threadIdx.x == 0) s_ok = atomicAdd(&p.ap_claim[S], 1u);
            __syncthreads();
            const u32 job = s_ok;
            __syncthreads();
            if (job == 0) {
                if (sweep) {
                    if (!early && !peer_wait(s, &sy->t_count, nworkers * (S + 1u), false, s_ok)) return;
                    peer_ship4(s, s_piv, rba, rbb, S, ct, ct, 0, 1);
                }
                __syncthreads();
                if (threadIdx.x == 0) peer_signal(s, kCtrLa);
                continue;
            }
            const u32 c = job - 1u;
            if (c >= nch) break;
            if (!loaded) {
                apply2_load(p, p.pout, s.pout_b, s.so, ash, rba, rbb);
                __syncthreads();
                loaded = true;
            }
            const u32 l0 = lo + c * crow, l1 = min(s.m_loc, l0 + crow);
            if (s.p.check)
                peer_apply2_rows_t<true>(s, ash, S, r, rba, rbb, has_b, s.peer[s.rank].pb[S & 1u],
                                         s.peer[s.rank].pb2[S & 1u], info, ipos, l0, l1);
            else
                peer_apply2_rows_t<false>(s, ash, S, r, rba, rbb, has_b, s.peer[s.rank].pb[S & 1u],
                                          s.peer[s.rank].pb2[S & 1u], info, ipos, l0, l1);
            if (sweep) {
                __syncthreads();
                if (!la_ready) {
                    if (!peer_wait(s, ctr + kCtrLa, G * (S + 1u), true, s_ok)) return;
                    la_ready = true;
                }
                if (rba + rbb > 0 && !built) {  // (the same tables for every chunk of S)
                    peer_build16(smem, stage, ct, w, rba, rbb);
                    __syncthreads();
                    built = true;
                }
                peer_trail16_rows(s, smem, S, r, ct, l0, l1 - l0, info, ipos);
            }
            ++mine;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (mine) {
                __threadfence();
                if (atomicAdd(&p.ap_done[S], mine) + mine == nch) peer_signal(s, kCtrCap);
            } else if (nch == 0 && wk == 0) {
                peer_signal(s, kCtrCap);
            }
        }

        // rest: every local worker closed S-1, all of S's pre-work done; the
        // sweep then also waits for every rank's remaining tiles (kCtrSt)
        if (threadIdx.x == 0) {
            s_ok = spin_geq2(&sy->t_count, nworkers * (S + 1u), &p.ap_done[S], nch, err) ? 1u : 0u;
            if (!s_ok) peer_fail(s);
        }
        __syncthreads();
        if (!s_ok) return;
        ptlo = ct + 1u;
        plo = lo;
        pnrows = nrows;
        pbeg = pend = 0;
        if (sweep && ct + 1u < ntiles && nrows > 0) {
            const u64 total = (u64)(ntiles - ct - 1u) * nrows;
            pbeg = total * wk / nworkers;
            pend = total * (wk + 1u) / nworkers;
        }
        if (sweep && ct + 1u < ntiles) {
            if (!peer_wait(s, ctr + kCtrSt, G * (S + 1u), true, s_ok)) return;
            if (rba + rbb > 0) {
                u64 u = pbeg;
                while (u < pend) {
                    const u32 tile = ct + 1u + (u32)(u / nrows);
                    const u32 row0 = (u32)(u % nrows);
                    const u32 cnt = (u32)min((u64)(nrows - row0), pend - u);
                    __syncthreads();
                    peer_build16(smem, stage, tile, w, rba, rbb);
                    __syncthreads();
                    peer_trail16_rows(s, smem, S, r, tile, lo + row0, cnt, info, ipos);
                    u += cnt;
                }
            }
        }
    }
}

// Local rows <-> 32-byte tiles (the multi-process path; the emulation uses
// peer_tile_kernel / peer_untile_kernel with kTw = 4).
__global__ void untile4_local_kernel(const u64* __restrict__ src, u64* __restrict__ dst, u32 m, u32 Wp,
                                     u32 Wpad4) {
    const u32 per_row = Wpad4 >> 1;
    const u64 total = (u64)m * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        const u32 row = (u32)(e / per_row), x = 2u * (u32)(e - (u64)row * per_row);
        *reinterpret_cast<ulonglong2*>(dst + (size_t)row * Wp + x) =
            *reinterpret_cast<const ulonglong2*>(tw4(const_cast<u64*>(src), m, row, x));
    }
}

}  // namespace gf2cu

namespace gf2cu {

// The one-GPU emulation's upload / download with 32-byte tiles.
__global__ void peer_tile4_kernel(const PeerParams* __restrict__ ranks, const u64* __restrict__ src, u32 Wp) {
    const PeerParams& s = ranks[blockIdx.y];
    const u32 per_row = s.p.Wpad8 >> 1;  // Wpad4 in this driver
    const u64 total = (u64)s.m_loc * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        const u32 l = (u32)(e / per_row), x = 2u * (u32)(e - (u64)l * per_row);
        const u32 g = shard_global(l, s.rank, s.nranks, s.block);
        *reinterpret_cast<ulonglong2*>(tw4(s.mat, s.m_loc, l, x)) =
            *reinterpret_cast<const ulonglong2*>(src + (size_t)g * Wp + x);
    }
}

__global__ void peer_untile4_kernel(const PeerParams* __restrict__ ranks, u64* __restrict__ dst, u32 Wp) {
    const PeerParams& s = ranks[blockIdx.y];
    const u32 per_row = s.p.Wpad8 >> 1;
    const u64 total = (u64)s.m_loc * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (u64)gridDim.x * blockDim.x) {
        const u32 l = (u32)(e / per_row), x = 2u * (u32)(e - (u64)l * per_row);
        const u32 pos = s.p.inv[shard_global(l, s.rank, s.nranks, s.block)];
        *reinterpret_cast<ulonglong2*>(dst + (size_t)pos * Wp + x) =
            *reinterpret_cast<const ulonglong2*>(tw4(s.mat, s.m_loc, l, x));
    }
}

}  // namespace gf2cu
