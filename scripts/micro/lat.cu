// Microbenchmark: dependent-chain latencies of warp primitives on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_vote(unsigned long long* out, unsigned seed, int iters) {
    unsigned x = seed ^ threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { unsigned b = __ballot_sync(~0u, x & 1); x = (x >> 1) ^ b; }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0); out[1] = x; }
}
__global__ void k_shfl(unsigned long long* out, unsigned seed, int iters) {
    unsigned x = seed ^ threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __shfl_sync(~0u, x, x & 31) + 1; }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0); out[1] = x; }
}
__global__ void k_alu(unsigned long long* out, unsigned seed, int iters) {
    unsigned long long x = seed ^ threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = (x >> 3) ^ (x << 1) ^ i; }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0); out[1] = x; }
}
__global__ void k_lds(unsigned long long* out, unsigned seed, int iters) {
    __shared__ unsigned s[256];
    s[threadIdx.x] = (threadIdx.x * 7 + seed) & 255;
    __syncwarp();
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = s[x & 255]; }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0); out[1] = x; }
}
// 4 warps: each iteration STS a value, named barrier, LDS the other warps' values
__global__ void k_bar4(unsigned long long* out, unsigned seed, int iters) {
    __shared__ unsigned s[2][4];
    unsigned x = seed + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int par = i & 1;
        if ((threadIdx.x & 31) == 0) s[par][threadIdx.x >> 5] = x;
        asm volatile("bar.sync 3, 128;" ::: "memory");
        x = s[par][0] + s[par][1] + s[par][2] + s[par][3] + (x & 1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0); out[1] = x; }
}
__global__ void k_bar4v(unsigned long long* out, unsigned seed, int iters) {
    __shared__ unsigned s[2][4];
    unsigned x = seed + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int par = i & 1;
        unsigned b = __ballot_sync(~0u, x & 1);
        if ((threadIdx.x & 31) == 0) s[par][threadIdx.x >> 5] = b;
        asm volatile("bar.sync 3, 128;" ::: "memory");
        uint4 v = *reinterpret_cast<uint4*>(s[par]);
        x = (v.x ? __ffs(v.x) : v.y ? __ffs(v.y) : 7) + x;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0); out[1] = x; }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h[2];
    const int it = 10000;
    struct { const char* n; void (*f)(unsigned long long*, unsigned, int); int thr; } ks[] = {
        {"vote chain", k_vote, 32}, {"shfl chain", k_shfl, 32}, {"alu64 chain", k_alu, 32},
        {"lds chain", k_lds, 32}, {"bar4 exchange", k_bar4, 128}, {"vote+bar4+lds128", k_bar4v, 128}};
    for (auto& k : ks) {
        k.f<<<1, k.thr>>>(d, 1, it); cudaDeviceSynchronize();
        k.f<<<1, k.thr>>>(d, 1, it); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%-20s %.1f cycles/iter\n", k.n, double(h[0]) / it);
    }
    return 0;
}
