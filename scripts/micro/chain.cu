// Microbenchmark: the floor of the leader's per-pivot dependent chain
// (ballot -> find-first -> shuffle of the pivot row -> XOR), with and without
// the row-t swap, the record stores and the publishing fence.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/chain scripts/micro/chain.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned u32;
__device__ __forceinline__ u64 shfl64(u64 v, int l) {
    u32 lo = __shfl_sync(~0u, (u32)v, l), hi = __shfl_sync(~0u, (u32)(v >> 32), l);
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u64 mix(u64 x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; return x ^ (x >> 31);
}
template <int V>
__global__ void k(u64* out, int reps) {
    __shared__ u64 sE[64];
    __shared__ u32 sq[64], sbal[64];
    __shared__ volatile int sprog;
    const u32 lane = threadIdx.x;
    long long tot = 0, piv = 0;
    u64 sink = 0;
    for (int rep = 0; rep < reps; ++rep) {
        u64 red = mix(rep * 32 + lane + 1);
        int t = 0, j = 0;
        const long long c0 = clock64();
        if (V == 4) {
            // 32-bit halves: columns 0..31 use the low word only for the test
            while (j < 64 && t < 32) {
                const u32 tl = (u32)t;
                const u64 rt = shfl64(red, (int)tl);
                const u32 w = j < 32 ? (u32)red : (u32)(red >> 32);
                const bool cand = (lane >= tl) & (((w >> (j & 31)) & 1u) != 0u);
                const u32 bal = __ballot_sync(~0u, cand);
                if (bal == 0u) { ++j; continue; }
                const int pl = __ffs(bal) - 1;
                const u64 pr = shfl64(red, pl);
                red = lane == (u32)pl ? rt : (cand ? red ^ pr : red);
                ++t; ++j;
            }
        } else {
            while (j < 64 && t < 32) {
                const u32 tl = (u32)t;
                u64 rt = 0;
                if (V >= 1) rt = shfl64(red, (int)tl);
                const bool cand = (lane >= tl) & (((red >> j) & 1ull) != 0ull);
                const u32 bal = __ballot_sync(~0u, cand);
                if (bal == 0u) { ++j; continue; }
                const int pl = __ffs(bal) - 1;
                const u64 pr = shfl64(red, pl);
                if (V == 0) red = cand ? red ^ pr : red;   // (no swap: lane pl zeroes itself)
                else red = lane == (u32)pl ? rt : (cand ? red ^ pr : red);
                if (V >= 2) {
                    sE[t] = pr;
                    sq[t] = (u32)j;
                    *(volatile u32*)&sbal[t] = bal;
                }
                if (V >= 3) {
                    __threadfence_block();
                    sprog = t + 1;
                }
                ++t; ++j;
            }
        }
        tot += clock64() - c0;
        piv += t;
        sink ^= red;
    }
    if (lane == 0) { out[0] = tot; out[1] = piv; }
    out[2 + lane] = sink + sE[lane] + sq[lane] + sbal[lane];
}
int main() {
    u64* d; cudaMalloc(&d, 64 * 8); u64 h[2];
    const int reps = 2000;
#define RUN(V, name) k<V><<<1, 32>>>(d, reps); cudaDeviceSynchronize(); k<V><<<1, 32>>>(d, reps); \
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("%-40s %.1f cycles/pivot (%.1f pivots)\n", name, double(h[0]) / h[1], double(h[1]) / reps);
    RUN(0, "ballot+ffs+shfl64+xor")
    RUN(1, "+ row-t shuffle and swap select")
    RUN(2, "+ record stores (E, q, bal)")
    RUN(3, "+ fence and progress store")
    RUN(4, "V1 with 32-bit candidate test")
    return 0;
}
