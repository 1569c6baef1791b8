// Microbenchmark: one 64-column step with 8 Gray tables on 64-byte tiles (the
// current sweep) vs two fused steps with 16 tables on 32-byte tiles, over
// the same M x W matrix (tile-major). Prints time per launch and the
// equivalent per-step time of the fused variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned u32;

__device__ __forceinline__ void xor2(ulonglong2& a, const ulonglong2& b) { a.x ^= b.x; a.y ^= b.y; }
__device__ __forceinline__ ulonglong2 ldcg2(const ulonglong2* p) { return __ldcg(p); }

// ---- A: 8 tables x 256 x 64 B, 64-byte tiles (8 words), 4 lanes per row ----
__device__ __forceinline__ u32 offA(u32 g, u32 e, u32 ch) {
    return (((g >> 1) * 256u + e) << 7) + ((g & 1u) << 6) + (ch << 4);
}
__global__ void __launch_bounds__(512, 1) sweepA(u64* mat, const u64* info, const u64* src, u32 M, u32 ntiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    const u64 total = (u64)ntiles * M;
    const u64 beg = total * blockIdx.x / gridDim.x, end = total * (blockIdx.x + 1) / gridDim.x;
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3, par = rg & 1;
    u64 u = beg;
    while (u < end) {
        const u32 tile = (u32)(u / M), row0 = (u32)(u % M);
        const u32 cnt = (u32)min((u64)(M - row0), end - u);
        __syncthreads();
        for (u32 k = threadIdx.x; k < 8 * 256 * 4; k += blockDim.x) {
            const u32 c = k & 3, e = (k >> 2) & 255, g = k >> 10;
            ulonglong2 acc = make_ulonglong2(0, 0);
            for (u32 b = 0; b < 8; ++b)
                if ((e >> b) & 1) xor2(acc, ldcg2((const ulonglong2*)(src + (size_t)(8 * g + b) * 8 + 2 * c)));
            *(ulonglong2*)(smem + offA(g, e, c)) = acc;
        }
        __syncthreads();
        u64* tb = mat + ((size_t)tile * M << 3) + 2 * ch;
        for (u32 b = row0 + wid * 8 + rg; b < row0 + cnt; b += 4 * 128) {
            u64 d[4];
            ulonglong2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const u32 i = b + k * 128;
                d[k] = i < row0 + cnt ? __ldcg(info + i) : 0ull;
                v[k] = d[k] ? ldcg2((const ulonglong2*)(tb + ((size_t)i << 3))) : make_ulonglong2(0, 0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (!d[k]) continue;
#pragma unroll
                for (u32 gi = 0; gi < 8; ++gi) {
                    const u32 g = gi ^ par;
                    xor2(v[k], *(const ulonglong2*)(smem + offA(g, (u32)(d[k] >> (8 * g)) & 255u, ch)));
                }
                *(ulonglong2*)(tb + ((size_t)(b + k * 128) << 3)) = v[k];
            }
        }
        u += cnt;
    }
}

// ---- B: 16 tables x 256 x 32 B, 32-byte tiles (4 words), 2 lanes per row ----
// table t at bank quarter t&3: entry e at ((t>>2)*256 + e)*128 + (t&3)*32 + half*16
__device__ __forceinline__ u32 offB(u32 t, u32 e, u32 h) {
    return (((t >> 2) * 256u + e) << 7) + ((t & 3u) << 5) + (h << 4);
}
__global__ void __launch_bounds__(512, 1) sweepB(u64* mat, const ulonglong2* info, const u64* src, u32 M, u32 ntiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    const u64 total = (u64)ntiles * M;
    const u64 beg = total * blockIdx.x / gridDim.x, end = total * (blockIdx.x + 1) / gridDim.x;
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 rw = lane >> 1, h = lane & 1, rq = (lane >> 1) & 3;
    u64 u = beg;
    while (u < end) {
        const u32 tile = (u32)(u / M), row0 = (u32)(u % M);
        const u32 cnt = (u32)min((u64)(M - row0), end - u);
        __syncthreads();
        for (u32 k = threadIdx.x; k < 16 * 256 * 2; k += blockDim.x) {
            const u32 c = k & 1, e = (k >> 1) & 255, t = k >> 9;
            ulonglong2 acc = make_ulonglong2(0, 0);
            for (u32 b = 0; b < 8; ++b)
                if ((e >> b) & 1) xor2(acc, ldcg2((const ulonglong2*)(src + (size_t)(8 * t + b) * 4 + 2 * c)));
            *(ulonglong2*)(smem + offB(t, e, c)) = acc;
        }
        __syncthreads();
        u64* tb = mat + ((size_t)tile * M << 2) + 2 * h;
        for (u32 b = row0 + wid * 16 + rw; b < row0 + cnt; b += 4 * 256) {
            ulonglong2 d[4];
            ulonglong2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const u32 i = b + k * 256;
                d[k] = i < row0 + cnt ? ldcg2(info + i) : make_ulonglong2(0, 0);
                v[k] = (d[k].x | d[k].y) ? ldcg2((const ulonglong2*)(tb + ((size_t)i << 2)))
                                         : make_ulonglong2(0, 0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (!(d[k].x | d[k].y)) continue;
#pragma unroll
                for (u32 p = 0; p < 16; ++p) {
                    const u32 t = (p + rq) & 15u;
                    const u64 dw = t < 8 ? d[k].x : d[k].y;
                    xor2(v[k], *(const ulonglong2*)(smem + offB(t, (u32)(dw >> (8 * (t & 7))) & 255u, h)));
                }
                *(ulonglong2*)(tb + ((size_t)(b + k * 256) << 2)) = v[k];
            }
        }
        u += cnt;
    }
}

__global__ void fill(u64* p, size_t n, u64 seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        u64 x = seed + i * 0x9e3779b97f4a7c15ull;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        p[i] = x ^ (x >> 31);
    }
}

int main(int argc, char** argv) {
    const u32 M = argc > 1 ? atoi(argv[1]) : 65536;
    const u32 W = argc > 2 ? atoi(argv[2]) : 1024;  // words per row
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    u64 *mat, *src, *infoA;
    ulonglong2* infoB;
    cudaMalloc(&mat, (size_t)M * W * 8);
    cudaMalloc(&src, 128 * 8 * 8);
    cudaMalloc(&infoA, (size_t)M * 8);
    cudaMalloc(&infoB, (size_t)M * 16);
    fill<<<1024, 256>>>(mat, (size_t)M * W, 1);
    fill<<<64, 256>>>(src, 128 * 8, 2);
    fill<<<256, 256>>>(infoA, M, 3);
    fill<<<256, 256>>>((u64*)infoB, (size_t)M * 2, 4);
    cudaFuncSetAttribute(sweepA, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaFuncSetAttribute(sweepB, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 16.0 * M * W;  // read + write of every word (one step)
    for (int rep = 0; rep < 3; ++rep) {
        float ta = 0, tb = 0;
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) sweepA<<<sms, 512, 131072>>>(mat, infoA, src, M, W / 8);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ta, e0, e1);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) sweepB<<<sms, 512, 131072>>>(mat, infoB, src, M, W / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tb, e0, e1);
        ta /= 5;
        tb /= 5;
        printf("M=%u W=%u  A (1 step, 8 tables, 64B tiles): %.3f ms = %.0f GB/s | B (2 steps, 16 tables, 32B tiles): %.3f ms"
               " = %.3f ms/step (%.0f GB/s-equivalent per step)  speedup/step %.2fx\n",
               M, W, ta, bytes / ta / 1e6, tb, tb / 2, 2 * bytes / tb / 1e6, ta / (tb / 2));
    }
    cudaError_t err = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(err));
    return 0;
}
