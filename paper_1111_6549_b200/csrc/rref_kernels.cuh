// rref_kernels.cuh -- device kernels of rref_from_ple / echelonize(ple_iterative)
// and the upper-triangular solve.
//
// The reference (ple.hpp:318-329) undoes the compression column swaps,
// zeroes the pivot columns below the diagonal and, for the reduced form,
// solves B <- U^-1 B on the top `rank` rows with trsm_upper_left_unit
// (multiply.hpp:314-335, recursive split + M4RM addmul). On a genuine PLE
// state those first two steps have a closed form:
//
//   row i < rank:  E_i = (a_i with columns <= q_i cleared) | bit q_i
//   row i >= rank: 0
//
// and the reduced form is unique, so the device computes it in pivot-first
// column coordinates: U = E restricted to the pivot columns (unit upper
// triangular, only its strictly upper bits are read) and N = E restricted to
// the non-pivot columns; then X = U^-1 N, R_i = bit q_i + X_i scattered back.
// X is solved bottom-up in 64-row blocks J: a one-warp-per-word in-block
// back-substitution, then the rows above get N_i ^= U[i, block J] * X_J
// through the same 8 x 8-bit Gray tables as the PLE trailing update.
//
// Layouts: U column-major by word (U[x * R + i], coalesced across rows),
// N tile-major like the PLE matrix (((x >> 3) * R + i) * 8 + (x & 7)),
// R = rank rounded up to 64; rows >= rank are zero in both.
#pragma once

#include "ple_kernels.cuh"

namespace gf2cu {

struct RrefParams {
    const u64* a;         // row-major source of U (and of N for rref), stride Wpa, Wa words
    const u64* b;         // trsm: row-major B (stride Wp, W words)
    u64* out;             // row-major destination (stride Wp), may alias a / b
    u64* U;               // column-major strictly-upper part, Wu words x R rows
    u64* N;               // tile-major right-hand side / solution, WnPad8 words x R rows
    const u32* q;         // pivot columns, r entries (increasing)
    const u32* np;        // non-pivot columns, n - r entries (increasing)
    const u32* usrc;      // per U word: first source column if contiguous, else ~0u
    const u32* nsrc;      // per N word: first source column if contiguous, else ~0u
    const u64* npmask;    // per row word y: non-pivot columns inside word y
    const u32* npos0;     // per row word y: number of non-pivot columns before word y
    u32 m, n, W, Wp;      // destination shape (n columns)
    u32 Wa, Wpa;          // source of U
    u32 r, R, Wu, Wn, WnPad8;
    u32 ncn;              // columns of N: n - r (rref) or n (trsm)
};

constexpr u32 kNone = 0xffffffffu;

__device__ __forceinline__ u64* nword(u64* N, u32 R, u32 i, u32 x) {
    return N + ((((size_t)(x >> 3) * R + i) << 3) + (x & 7u));
}

// 64 bits of a row-major row starting at column c (bits past word W-1 read 0).
__device__ __forceinline__ u64 row_bits64(const u64* row, u32 W, u32 c) {
    const u32 wd = c >> 6, sh = c & 63u;
    u64 v = row[wd] >> sh;
    if (sh && wd + 1u < W) v |= row[wd + 1u] << (64u - sh);
    return v;
}

// Bits b < cnt: source column cols[k0 + b] (= src + b when contiguous) of
// `row`, kept only where the column is > lim (E_i is zero left of its pivot).
__device__ __forceinline__ u64 gather_word(const u64* row, u32 W, const u32* cols, u32 k0,
                                           u32 cnt, u32 src, u32 lim) {
    u64 v = 0ull;
    if (src != kNone) {
        v = row_bits64(row, W, src) & low_mask64((int)cnt);
        if (lim != kNone && lim >= src) {
            const u32 d = lim - src + 1u;
            v &= d >= 64u ? 0ull : ~low_mask64((int)d);
        }
    } else {
        for (u32 b = 0; b < cnt; ++b) {
            const u32 c = cols[k0 + b];
            if (lim == kNone || c > lim) v |= ((row[c >> 6] >> (c & 63u)) & 1ull) << b;
        }
    }
    return v;
}

// U and N of rows i < r (rref: lim = q_i; trsm: lim = none, U read from
// the square operand). One thread per (row, word); x-major so that the
// column-major U writes coalesce.
__global__ void rref_gather_kernel(RrefParams p, int rref_mode) {
    const u32 nw = p.Wu + p.Wn;
    const u64 total = (u64)nw * p.r;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 x = (u32)(e / p.r), i = (u32)(e - (u64)x * p.r);
        const u64* row = p.a + (size_t)i * p.Wpa;
        if (x < p.Wu) {
            if (x < (i >> 6)) continue;  // never read: only bits j > i matter
            const u32 j0 = x * 64u, cnt = min(64u, p.r - j0);
            u64 v;
            if (rref_mode) {
                v = gather_word(row, p.Wa, p.q, j0, cnt, p.usrc[x], p.q[i]);
            } else {
                v = row_bits64(row, p.Wa, j0) & low_mask64((int)cnt);
                if (x == (i >> 6)) v &= ~low_mask64((int)(i & 63u) + 1);
            }
            p.U[(size_t)x * p.R + i] = v;
        } else {
            const u32 xn = x - p.Wu, k0 = xn * 64u;
            const u32 cnt = min(64u, p.ncn - k0);
            u64 v;
            if (rref_mode)
                v = gather_word(row, p.Wa, p.np, k0, cnt, p.nsrc[xn], p.q[i]);
            else  // trsm: B as it is
                v = p.b[(size_t)i * p.Wp + xn];
            *nword(p.N, p.R, i, xn) = v;
        }
    }
}

// In-block back-substitution of block J (rows 64J..64J+63, all updates from
// the blocks below applied): one warp per N word, lanes hold rows l and l+32;
// row j is final when step j broadcasts it (it only receives rows > j).
__global__ void rref_block_solve_kernel(RrefParams p, u32 J) {
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const u32 x = blockIdx.x * (blockDim.x >> 5) + wid;
    if (x >= p.Wn) return;
    const u32 i0 = 64u * J + lane, i1 = i0 + 32u;
    const u64 u0 = p.U[(size_t)J * p.R + i0] & ~low_mask64((int)lane + 1);
    const u64 u1 = p.U[(size_t)J * p.R + i1] & ~low_mask64((int)lane + 33);
    u64* n0 = nword(p.N, p.R, i0, x);
    u64* n1 = nword(p.N, p.R, i1, x);
    u64 v0 = *n0, v1 = *n1;
#pragma unroll 8
    for (int j = 63; j >= 0; --j) {
        const u64 xj = shfl64(j >= 32 ? v1 : v0, j & 31);
        if ((u0 >> j) & 1ull) v0 ^= xj;
        if ((u1 >> j) & 1ull) v1 ^= xj;
    }
    *n0 = v0;
    *n1 = v1;
}

// Rows [0, 64J) of every N tile: N_i ^= U[i, word J] * X_J, tables built
// from the solved block rows. Linear split of the (tile, row) units over
// the grid, tables rebuilt per tile segment (as trail_share).
__global__ void __launch_bounds__(kTrailThreads, 1) rref_update_kernel(RrefParams p, u32 J) {
    extern __shared__ __align__(128) unsigned char smem[];
    const u32 nrows = 64u * J;
    const u32 ntiles = p.WnPad8 >> 3;
    const u64 total = (u64)ntiles * nrows;
    const u64 beg = total * blockIdx.x / gridDim.x, end = total * (blockIdx.x + 1) / gridDim.x;
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3u, par = rg & 1u;
    u32 lsel[4], lkoff[4];
    lookup8_consts(par, ch, lsel, lkoff);
    const u64* ucol = p.U + (size_t)J * p.R;
    u64 u = beg;
    while (u < end) {
        const u32 tile = (u32)(u / nrows);
        const u32 row0 = (u32)(u % nrows);
        const u32 cnt = (u32)min((u64)(nrows - row0), end - u);
        __syncthreads();
        gray_tables(smem, p.N + (((size_t)tile * p.R + 64u * J) << 3), 64u, 0u);
        __syncthreads();
        u64* tbase = p.N + (((size_t)tile * p.R) << 3) + 2u * ch;
        for (u32 b = row0 + wid * 8u + rg; b < row0 + cnt; b += 4u * (kTrailThreads / 4)) {
            u64 d[kUnroll];
            ulonglong2 v[kUnroll];
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const u32 i = b + (u32)k * (kTrailThreads / 4);
                d[k] = i < row0 + cnt ? ldcg(ucol + i) : 0ull;
                v[k] = d[k] ? ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)i << 3)))
                            : make_ulonglong2(0ull, 0ull);
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                if (!d[k]) continue;
                lookup8(v[k], smem, d[k], lsel, lkoff);
                const u32 i = b + (u32)k * (kTrailThreads / 4);
                *reinterpret_cast<ulonglong2*>(tbase + ((size_t)i << 3)) = v[k];
            }
        }
        u += cnt;
    }
}

// One launch per 64-row block: rref_step_kernel(J) applies X_J to the rows
// above block J and, in the same launch, finishes block J-1 -- CTAs
// [0, ntiles) update block J-1's rows of one N tile each (X_J rows staged in
// shared memory, one thread per row and word) and solve it in place (one warp
// per word, 64 shuffle steps); the other CTAs update rows [0, 64(J-1)) with
// the Gray tables. The next launch reads X_{J-1} in stream order.
__global__ void __launch_bounds__(kTrailThreads, 1) rref_step_kernel(RrefParams p, u32 J) {
    extern __shared__ __align__(128) unsigned char smem[];
    const u32 ntiles = p.WnPad8 >> 3;
    const u64* ucol = p.U + (size_t)J * p.R;
    if (blockIdx.x < ntiles) {
        // ---- block J-1 of tile blockIdx.x: update, then solve ----
        u64 (*xs)[8] = reinterpret_cast<u64 (*)[8]>(smem);
        const u32 tile = blockIdx.x;
        for (u32 k = threadIdx.x; k < 512u; k += blockDim.x)
            xs[k >> 3][k & 7u] = ldcg(nword(p.N, p.R, 64u * J + (k >> 3), tile * 8u + (k & 7u)));
        __syncthreads();
        for (u32 k = threadIdx.x; k < 512u; k += blockDim.x) {
            const u32 row = 64u * (J - 1u) + (k >> 3), x = k & 7u;
            if (tile * 8u + x >= p.Wn) continue;
            u64 d = ldcg(ucol + row);
            u64 acc = 0ull;
            while (d) {
                const int j = __ffsll((long long)d) - 1;
                d &= d - 1ull;
                acc ^= xs[j][x];
            }
            *nword(p.N, p.R, row, tile * 8u + x) ^= acc;
        }
        __syncthreads();
        const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
        const u32 x = tile * 8u + wid;
        if (wid < 8u && x < p.Wn) {
            const u32 Jb = J - 1u;
            const u32 i0 = 64u * Jb + lane, i1 = i0 + 32u;
            const u64 u0 = p.U[(size_t)Jb * p.R + i0] & ~low_mask64((int)lane + 1);
            const u64 u1 = p.U[(size_t)Jb * p.R + i1] & ~low_mask64((int)lane + 33);
            u64* n0 = nword(p.N, p.R, i0, x);
            u64* n1 = nword(p.N, p.R, i1, x);
            u64 v0 = *n0, v1 = *n1;
#pragma unroll 8
            for (int j = 63; j >= 0; --j) {
                const u64 xj = shfl64(j >= 32 ? v1 : v0, j & 31);
                if ((u0 >> j) & 1ull) v0 ^= xj;
                if ((u1 >> j) & 1ull) v1 ^= xj;
            }
            *n0 = v0;
            *n1 = v1;
        }
        return;
    }
    // ---- rows [0, 64(J-1)) of every tile: Gray-table update ----
    const u32 nrows = 64u * (J - 1u);
    if (nrows == 0u) return;
    const u32 nb = gridDim.x - ntiles, bi = blockIdx.x - ntiles;
    const u64 total = (u64)ntiles * nrows;
    const u64 beg = total * bi / nb, end = total * (bi + 1) / nb;
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3u, par = rg & 1u;
    u32 lsel[4], lkoff[4];
    lookup8_consts(par, ch, lsel, lkoff);
    u64 u = beg;
    while (u < end) {
        const u32 tile = (u32)(u / nrows);
        const u32 row0 = (u32)(u % nrows);
        const u32 cnt = (u32)min((u64)(nrows - row0), end - u);
        __syncthreads();
        gray_tables(smem, p.N + (((size_t)tile * p.R + 64u * J) << 3), 64u, 0u);
        __syncthreads();
        u64* tbase = p.N + (((size_t)tile * p.R) << 3) + 2u * ch;
        for (u32 b = row0 + wid * 8u + rg; b < row0 + cnt; b += 4u * (kTrailThreads / 4)) {
            u64 d[kUnroll];
            ulonglong2 v[kUnroll];
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const u32 i = b + (u32)k * (kTrailThreads / 4);
                d[k] = i < row0 + cnt ? ldcg(ucol + i) : 0ull;
                v[k] = d[k] ? ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)i << 3)))
                            : make_ulonglong2(0ull, 0ull);
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                if (!d[k]) continue;
                lookup8(v[k], smem, d[k], lsel, lkoff);
                const u32 i = b + (u32)k * (kTrailThreads / 4);
                *reinterpret_cast<ulonglong2*>(tbase + ((size_t)i << 3)) = v[k];
            }
        }
        u += cnt;
    }
}

// Reduced rows back in the original column order: R_i = bit q_i + X_i on the
// non-pivot columns for i < r, zero rows below (row-major, words < W).
__global__ void rref_scatter_kernel(RrefParams p) {
    const u64 total = (u64)p.m * p.W;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 i = (u32)(e / p.W), y = (u32)(e - (u64)i * p.W);
        u64 v = 0ull;
        if (i < p.r) {
            const u32 qi = p.q[i];
            if ((qi >> 6) == y) v |= 1ull << (qi & 63u);
            const u64 nm = p.npmask[y];
            if (nm) {
                const u32 k0 = p.npos0[y], cnt = __popcll(nm);
                const u32 xw = k0 >> 6, sh = k0 & 63u;
                u64 xb = *nword(p.N, p.R, i, xw) >> sh;
                if (sh && xw + 1u < p.Wn) xb |= *nword(p.N, p.R, i, xw + 1u) << (64u - sh);
                xb &= low_mask64((int)cnt);
                const u32 lo = __ffsll((long long)nm) - 1;
                if ((nm >> lo) == low_mask64((int)cnt)) {
                    v |= xb << lo;
                } else {
                    u64 mm = nm;
                    for (u32 b = 0; b < cnt; ++b) {
                        const u32 c = __ffsll((long long)mm) - 1;
                        mm &= mm - 1ull;
                        v |= ((xb >> b) & 1ull) << c;
                    }
                }
            }
        }
        p.out[(size_t)i * p.Wp + y] = v;
    }
}

// Echelon form only (full = false): E_i in place for i < r, zero rows below.
__global__ void rref_echelon_kernel(u64* a, const u32* q, u32 m, u32 W, u32 Wp, u32 r) {
    const u64 total = (u64)m * W;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 i = (u32)(e / W), y = (u32)(e - (u64)i * W);
        u64* w = a + (size_t)i * Wp + y;
        if (i >= r) {
            *w = 0ull;
            continue;
        }
        const u32 qi = q[i], qw = qi >> 6;
        if (y < qw) {
            *w = 0ull;
        } else if (y == qw) {
            *w = (*w & ~low_mask64((int)(qi & 63u) + 1)) | (1ull << (qi & 63u));
        }
    }
}

// undo_column_swaps (ple.hpp:293-296): the compression swaps replayed
// backwards, swap_cols_from_row(a, b, from_row) (bit_matrix.hpp:302-318) on
// every row >= from_row. One thread per row, the swap list (<= min(m, n)
// entries, {a | b << 32, from_row}) read through the uniform cache.
// (forward = 1: the swaps in application order instead, rows [row_lo, m):
// partial_ple's compression of the rows it never read, ple.hpp:122-126.)
__global__ void undo_col_swaps_kernel(u64* mat, u32 m, u32 Wp, const ulonglong2* cs, u32 ncs,
                                      int forward = 0, u32 row_lo = 0u) {
    for (u32 i = row_lo + blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        u64* row = mat + (size_t)i * Wp;
        for (u32 kk = 0; kk < ncs; ++kk) {
            const u32 k = forward ? kk : ncs - 1u - kk;
            const ulonglong2 c = __ldg(cs + k);
            if (i < c.y) continue;
            const u32 ca = (u32)c.x, cb = (u32)(c.x >> 32);
            const u64 x = ((row[ca >> 6] >> (ca & 63u)) ^ (row[cb >> 6] >> (cb & 63u))) & 1ull;
            row[ca >> 6] ^= x << (ca & 63u);
            row[cb >> 6] ^= x << (cb & 63u);
        }
    }
}

// trsm_upper_left_unit: X (tile-major N) back to the row-major B buffer.
__global__ void trsm_store_kernel(RrefParams p) {
    const u64 total = (u64)p.r * p.W;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 i = (u32)(e / p.W), y = (u32)(e - (u64)i * p.W);
        p.out[(size_t)i * p.Wp + y] = *nword(p.N, p.R, i, y);
    }
}

}  // namespace gf2cu
