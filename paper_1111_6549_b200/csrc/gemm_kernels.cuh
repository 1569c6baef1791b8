// gemm_kernels.cuh -- GF(2) matrix product C (+)= A * B on the device
// (addmul / mul, multiply.hpp:89-131, 254-274).
//
// The reference's addmul_m4rm (multiply.hpp:89-122) processes k rows of B at
// a time through a Gray-code table and adds one table row per k columns of A.
// Here one CTA owns a 2048-row x 64-byte tile of C in registers (16 rows x
// 16 bytes per thread) and walks A's 64-column words: for word k it builds
// the same 8 x 8-bit Gray tables as the PLE trailing update from B's rows
// 64k..64k+63 of its column tile, then every row adds the 8 table rows
// selected by its coefficient word A[i, k]. A is read as column-major words
// (a transpose prepass), so the coefficient loads coalesce; B and C stay in
// the row-major device layout (128-byte aligned rows, zero padding words).
// The kernel is bound by shared-memory lookups (8 x 64 B per row and word),
// not HBM: C is read and written once, B once per row chunk.
#pragma once

#include "ple_kernels.cuh"

namespace gf2cu {

constexpr u32 kGemmRowsPerThread = 16;
constexpr u32 kGemmRows = (kTrailThreads / 4) * kGemmRowsPerThread;  // 2048

// Acm[k * M + i] = word k of row i of the row-major A (stride Wpa).
__global__ void gemm_transpose_a_kernel(const u64* __restrict__ a, u64* __restrict__ acm, u32 M,
                                        u32 Lw, u32 Wpa) {
    const u64 total = (u64)M * Lw;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 k = (u32)(e / M), i = (u32)(e - (u64)k * M);
        acm[e] = a[(size_t)i * Wpa + k];
    }
}

// grid.x = column tiles of C (8 words), grid.y = 2048-row chunks.
__global__ void __launch_bounds__(kTrailThreads, 1)
    gemm_m4rm_kernel(const u64* __restrict__ acm, const u64* __restrict__ b, u64* c, u32 M, u32 L,
                     u32 Wpb, u32 Wpc, int accumulate) {
    extern __shared__ __align__(128) unsigned char smem[];
    const u32 tile = blockIdx.x;
    const u32 row_base = blockIdx.y * kGemmRows;
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3u, par = rg & 1u;
    u32 lsel[4], lkoff[4];
    lookup8_consts(par, ch, lsel, lkoff);
    const u32 r0 = row_base + wid * 8u + rg;
    const u32 Lw = (L + 63u) >> 6;
    ulonglong2 acc[kGemmRowsPerThread];
#pragma unroll
    for (u32 s = 0; s < kGemmRowsPerThread; ++s) {
        const u32 i = r0 + s * (kTrailThreads / 4);
        acc[s] = make_ulonglong2(0ull, 0ull);
        if (accumulate && i < M)
            acc[s] = *reinterpret_cast<const ulonglong2*>(c + (size_t)i * Wpc + tile * 8u + 2u * ch);
    }
    u64 d[kGemmRowsPerThread];
#pragma unroll
    for (u32 s = 0; s < kGemmRowsPerThread; ++s) {
        const u32 i = r0 + s * (kTrailThreads / 4);
        d[s] = i < M ? ldcg(acm + i) : 0ull;
        if (L < 64u) d[s] &= low_mask64((int)L);
    }
    for (u32 k = 0; k < Lw; ++k) {
        __syncthreads();
        gray_tables(smem, b + (size_t)(64u * k) * Wpb + tile * 8u, min(64u, L - 64u * k), 0u, Wpb);
        __syncthreads();
        u64 dn[kGemmRowsPerThread];
#pragma unroll
        for (u32 s = 0; s < kGemmRowsPerThread; ++s) {
            const u32 i = r0 + s * (kTrailThreads / 4);
            dn[s] = (k + 1u < Lw && i < M) ? ldcg(acm + (size_t)(k + 1u) * M + i) : 0ull;
            if (64u * (k + 2u) > L) dn[s] &= low_mask64((int)(L - 64u * (k + 1u)));
        }
#pragma unroll
        for (u32 s = 0; s < kGemmRowsPerThread; ++s) {
            if (d[s] == 0ull) continue;
            lookup8(acc[s], smem, d[s], lsel, lkoff);
        }
#pragma unroll
        for (u32 s = 0; s < kGemmRowsPerThread; ++s) d[s] = dn[s];
    }
#pragma unroll
    for (u32 s = 0; s < kGemmRowsPerThread; ++s) {
        const u32 i = r0 + s * (kTrailThreads / 4);
        if (i < M) *reinterpret_cast<ulonglong2*>(c + (size_t)i * Wpc + tile * 8u + 2u * ch) = acc[s];
    }
}

}  // namespace gf2cu
