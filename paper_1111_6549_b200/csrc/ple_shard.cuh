// ple_shard.cuh -- per-rank kernels of the row-sharded (multi-GPU) PLE.
//
// Global row g lives on rank (g / B) % G at local index
// (g / (B*G)) * B + g % B (block-cyclic, block B). Every rank keeps the
// replicated position state (perm: position -> global row, inv: global row
// -> position, the step state and the panel outputs) and updates it with the
// same panel factorization; rows themselves never move. Per step the host
// (paper_1111_6549_b200/shard.py) all-reduces the window of panel words,
// runs panel_factor (window-only, re-run on a full gather after a miss),
// shard_apply on the local rows, broadcasts each owner's packed pivot tails,
// and runs trailing_update_kernel on the local rows.
#pragma once

#include "ple_kernels.cuh"

namespace gf2cu {

struct ShardParams {
    u64* mat;          // local tile-major matrix (m_loc rows)
    u64* pbl;          // panel word per local row
    ulonglong2* info;  // per local row {d, local row}
    unsigned char* retired;  // local row already a pivot row of an earlier step
    StepState* lstate; // {first active local row, rb} for trailing_update_kernel
    const u32* perm;   // replicated position -> global row
    const u32* inv;    // replicated global row -> position
    const StepState* gstate;  // replicated {r, rb}
    const PanelOut* pout;
    u64* pack;         // this rank's pivot tails, packed by owned-pivot order
    u32 m_loc, m, n, W, Wpad8;
    u32 rank, nranks, block;
};

__device__ __forceinline__ u32 shard_global(u32 l, u32 rank, u32 nranks, u32 block) {
    return ((l / block) * nranks + rank) * block + l % block;
}
__device__ __forceinline__ u32 shard_local(u32 g, u32 nranks, u32 block) {
    return (g / (block * nranks)) * block + g % block;
}
__device__ __forceinline__ u32 shard_owner(u32 g, u32 nranks, u32 block) {
    return (g / block) % nranks;
}

__global__ void shard_init_kernel(ShardParams s, u32* perm, u32* inv, StepState* gstate) {
    const u32 stride = gridDim.x * blockDim.x;
    const u32 tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (u32 i = tid; i < s.m; i += stride) {
        perm[i] = i;
        inv[i] = i;
    }
    for (u32 l = tid; l < s.m_loc; l += stride) {
        s.retired[l] = 0;
        s.pbl[l] = *tword(s.mat, s.m_loc, l, 0);
    }
    if (tid == 0) {
        gstate->r = 0;
        gstate->rb = 0;
    }
}

// Position-indexed panel words of this rank's active rows whose position is
// in [lo, hi) (the buffer range was zeroed by the host; others add theirs).
__global__ void shard_gather_kernel(ShardParams s, u64* posw, u32 lo, u32 hi) {
    for (u32 l = blockIdx.x * blockDim.x + threadIdx.x; l < s.m_loc; l += gridDim.x * blockDim.x) {
        if (s.retired[l]) continue;
        const u32 pos = s.inv[shard_global(l, s.rank, s.nranks, s.block)];
        if (pos >= lo && pos < hi) posw[pos] = s.pbl[l];
    }
}

// Multipliers c, combination d and the compressed write for every active
// local row (apply_rows with a local-row sweep), pivot rows retired and their
// raw tails packed. Also publishes the first active local row for the sweep.
__global__ void __launch_bounds__(kApplyThreads) shard_apply_kernel(ShardParams s, u32 w) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64];
    const u32 r = s.gstate->r, rb = s.gstate->rb;
    for (u32 k = threadIdx.x; k < 64; k += blockDim.x) {
        const bool v = k < rb;
        sE[k] = v ? s.pout->E[k] : 0ull;
        sD[k] = v ? s.pout->D[k] : 0ull;
        sq[k] = v ? s.pout->qb[k] : 0u;
    }
    __syncthreads();
    const u32 w0 = r >> 6, b0 = r & 63;
    const u32 stride = gridDim.x * blockDim.x;
    u32 lo = 0xffffffffu;
    for (u32 l = blockIdx.x * blockDim.x + threadIdx.x; l < s.m_loc; l += stride) {
        if (s.retired[l]) {
            s.info[l] = make_ulonglong2(0ull, (u64)l);
            continue;
        }
        lo = min(lo, l);
        const u32 pos = s.inv[shard_global(l, s.rank, s.nranks, s.block)];
        const u32 off = pos - r;  // active rows sit at positions >= r
        const u32 tl = off < rb ? off : rb;
        u64 v = s.pbl[l], a = 0, c = 0;
#pragma unroll 8
        for (u32 k = 0; k < 64; ++k) {
            if (k >= tl) break;
            const u64 bit = (v >> sq[k]) & 1ull;
            const u64 msk = 0ull - bit;
            v ^= sE[k] & msk;
            a ^= sD[k] & msk;
            c |= bit << k;
        }
        u64 epart = 0;
        if (off < rb) {
            c |= 1ull << off;
            epart = v & ~low_mask64((int)sq[off] + 1);
            s.retired[l] = 1;
        }
        s.info[l] = make_ulonglong2(a, (u64)l);
        const u64 clo = c << b0;
        const u64 chi = b0 ? (c >> (64 - b0)) : 0ull;
        if (w0 == w) {
            *tword(s.mat, s.m_loc, l, w) = clo | epart;
        } else {
            *tword(s.mat, s.m_loc, l, w0) |= clo;
            if (w0 + 1 == w) {
                *tword(s.mat, s.m_loc, l, w) = chi | epart;
            } else {
                if (chi) *tword(s.mat, s.m_loc, l, w0 + 1) |= chi;
                *tword(s.mat, s.m_loc, l, w) = epart;
            }
        }
    }
    // first active local row (this step's pivots included) for the sweep
    for (int o = 16; o > 0; o >>= 1) lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    if ((threadIdx.x & 31) == 0 && lo != 0xffffffffu) atomicMin(&s.lstate->r, lo);
    if (blockIdx.x == 0 && threadIdx.x == 0) s.lstate->rb = rb;
}

// Pack this rank's pivot rows' raw tails (words [x0, Wpad8)), slot = rank of
// t among the owned pivots; runs before shard_apply_kernel touches the rows.
__global__ void shard_pack_kernel(ShardParams s, u32 w) {
    const u32 r = s.gstate->r, rb = s.gstate->rb;
    const u32 x0 = (w + 1) & ~7u;
    const u32 tailw = s.Wpad8 > x0 ? s.Wpad8 - x0 : 0u;
    const u64 total = (u64)rb * tailw;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 t = (u32)(e / tailw), x = x0 + (u32)(e - (u64)t * tailw);
        const u32 g = s.perm[r + t];
        if (shard_owner(g, s.nranks, s.block) != s.rank) continue;
        u32 slot = 0;
        for (u32 k = 0; k < t; ++k) slot += shard_owner(s.perm[r + k], s.nranks, s.block) == s.rank;
        s.pack[(size_t)slot * tailw + (x - x0)] =
            *tword(s.mat, s.m_loc, shard_local(g, s.nranks, s.block), x);
    }
}

// This rank's pivot rows' raw tails (words [x0, Wpad8), x0 = (w+1) & ~7)
// straight into the tile-major stage layout at their pivot slots t. The
// caller zeroed that region; a sum all-reduce over the ranks' stages then
// yields every pivot tail on every rank (the contributions are disjoint), so
// no owner-dependent broadcast (and no host decision) is needed per step.
__global__ void shard_pack_stage_kernel(ShardParams s, u64* stage, u32 w) {
    const u32 r = s.gstate->r, rb = s.gstate->rb;
    const u32 x0 = (w + 1) & ~7u;
    const u32 tailw = s.Wpad8 > x0 ? s.Wpad8 - x0 : 0u;
    const u64 total = (u64)rb * tailw;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 t = (u32)(e / tailw), x = x0 + (u32)(e - (u64)t * tailw);
        const u32 g = s.perm[r + t];
        if (shard_owner(g, s.nranks, s.block) != s.rank) continue;
        stage[(((size_t)(x >> 3) * 64 + t) << 3) + (x & 7u)] =
            *tword(s.mat, s.m_loc, shard_local(g, s.nranks, s.block), x);
    }
}

// The ctr generator for this rank's rows (row-major local
// buffer, stride Wp): the words of global row g, bit-identical to fill_ctr.
__global__ void shard_fill_ctr_kernel(u64* data, u32 m_loc, u32 n, u32 Wp, u32 rank, u32 nranks,
                                      u32 block, u64 seed) {
    const u32 W = (n + 63u) >> 6;
    const u64 total = (u64)m_loc * Wp;
    const u64 base = seed << 32;
    const u64 lastmask = (n & 63u) ? ((1ull << (n & 63u)) - 1ull) : ~0ull;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 l = (u32)(e / Wp), x = (u32)(e - (u64)l * Wp);
        const u64 g = shard_global(l, rank, nranks, block);
        u64 v = 0ull;
        if (x < W) {
            v = fmix64(base + (g * W + x + 1ull) * 0x9e3779b97f4a7c15ull);
            if (x == W - 1u) v &= lastmask;
        }
        data[e] = v;
    }
}

// Scatter owner o's packed pivot tails (its pivots in increasing t order,
// bitmask `mask`) into the tile-major stage.
__global__ void shard_unpack_kernel(const u64* pack, u64 mask, u64* stage, u32 w, u32 Wpad8) {
    const u32 x0 = (w + 1) & ~7u;
    const u32 tailw = Wpad8 > x0 ? Wpad8 - x0 : 0u;
    const u32 cnt = __popcll(mask);
    const u64 total = (u64)cnt * tailw;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 slot = (u32)(e / tailw), x = x0 + (u32)(e - (u64)slot * tailw);
        // t = position of the slot-th set bit of mask
        u64 mm = mask;
        for (u32 k = 0; k < slot; ++k) mm &= mm - 1ull;
        const u32 t = (u32)(__ffsll((long long)mm) - 1);
        stage[(((size_t)(x >> 3) * 64 + t) << 3) + (x & 7u)] = pack[e];
    }
}

}  // namespace gf2cu
