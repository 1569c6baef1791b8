// Variants of the transposed leader epoch for cycle accounting (see tleader.cu).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "ple_kernels.cuh"
using namespace gf2cu;

// (the transposed-leader helpers, removed from the product in round 2 after
// measuring slower end to end; kept here with the micro-benchmark)
__device__ __forceinline__ u32 transpose32(u32 x) {
    const u32 lane = threadIdx.x & 31u;
#pragma unroll
    for (int st = 4; st >= 0; --st) {
        const u32 s = 1u << st;
        const u32 m = st == 4 ? 0x0000FFFFu : st == 3 ? 0x00FF00FFu : st == 2 ? 0x0F0F0F0Fu
                      : st == 1 ? 0x33333333u : 0x55555555u;
        const u32 y = __shfl_xor_sync(0xffffffffu, x, (int)s);
        x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
    }
    return x;
}

__device__ __forceinline__ void mask_update(u32& M, u32 bitP, u32 tbit, u32 elim, u32 flip, u32 force) {
    const bool bp = (M & bitP) != 0u, bt = (M & tbit) != 0u;
    M ^= ((bp || force) ? elim : 0u) ^ ((bp != bt) ? flip : 0u);
}

template <int V>
__device__ __forceinline__ void leader_v(u64& red, u64& acc, u32& org, int& t, int& j, int tend, u64* sE,
                                         u64* sD, u32* sq, u32* ssw) {
    constexpr int kG = 4;
    const u32 lane = threadIdx.x & 31u;
    u32 C0, C1, A0, A1;
    if (V & 1) {  // no transposes
        C0 = (u32)red; C1 = (u32)(red >> 32); A0 = (u32)acc; A1 = (u32)(acc >> 32);
    } else {
        C0 = transpose32((u32)red); C1 = transpose32((u32)(red >> 32));
        A0 = transpose32((u32)acc); A1 = transpose32((u32)(acc >> 32));
    }
    u32 live = __ballot_sync(0xffffffffu, lane >= (u32)t);
    int myq = -1;
    bool go = t < tend;
    while (__all_sync(0xffffffffu, go)) {
        u32 bc[kG];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
            const int jj = min(j + g, 63);
            bc[g] = __shfl_sync(0xffffffffu, jj < 32 ? C0 : C1, jj & 31);
        }
#pragma unroll
        for (int g = 0; g < kG; ++g) {
            const u32 cand = bc[g] & live;
            if (__all_sync(0xffffffffu, cand == 0u)) { go = false; break; }
            const u32 tl = (u32)t & 31u;
            const u32 bitP = cand & (0u - cand), tbit = 1u << tl;
            const u32 elim = cand ^ bitP, flip = tbit | bitP;
#pragma unroll
            for (int h = g + 1; h < kG; ++h) mask_update(bc[h], bitP, tbit, elim, flip, 0u);
            mask_update(C0, bitP, tbit, elim, flip, 0u);
            mask_update(C1, bitP, tbit, elim, flip, 0u);
            if (!(V & 2)) {  // combination masks
                mask_update(A0, bitP, tbit, elim, flip, lane == (u32)t);
                mask_update(A1, bitP, tbit, elim, flip, lane + 32u == (u32)t);
            }
            if (!(V & 4)) {  // origins + records
                const u32 pl = (u32)(__ffs(bitP) - 1);
                const u32 opl = __shfl_sync(0xffffffffu, org, (int)pl);
                const u32 otl = __shfl_sync(0xffffffffu, org, (int)tl);
                org = lane == tl ? opl : (lane == pl ? otl : org);
                myq = lane == tl ? j : myq;
                if (lane == 0u) { sq[t] = (u32)j; ssw[t] = pl; }
            }
            live &= ~tbit;
            ++t; ++j;
            if (__all_sync(0xffffffffu, t >= tend)) { go = false; break; }
        }
    }
    if (V & 1) {
        red = C0 | ((u64)C1 << 32); acc = A0 | ((u64)A1 << 32);
    } else {
        red = (u64)transpose32(C0) | ((u64)transpose32(C1) << 32);
        acc = (u64)transpose32(A0) | ((u64)transpose32(A1) << 32);
    }
    sE[lane] = red + myq;
    sD[lane] = acc;
}

template <int V>
__global__ void kv(const u64* in, long long* cyc, int* piv, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64];
    __shared__ int flag;
    const u32 lane = threadIdx.x & 31u;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    if (threadIdx.x >= 32) {
        // the panel CTA's other warps: one spins on a shared-memory flag (the
        // signal warp), the rest wait at a barrier
        if (threadIdx.x >= blockDim.x - 32) {
            if ((V & 8) && lane == 0)
                while (ld_acquire_cta(&flag) == 0) {
                    if (V & 16) __nanosleep(100);
                }
            __syncwarp();
        }
        named_bar(1, blockDim.x - 32);
        return;
    }
    long long tot = 0;
    int t = 0;
    for (int rep = 0; rep < reps; ++rep) {
        u64 red = in[blockIdx.x * 32 + lane], acc = 0;
        u32 org = lane;
        t = 0;
        int j = 0;
        __syncwarp();
        const long long c0 = clock64();
        leader_v<V>(red, acc, org, t, j, 32, sE, sD, sq, ssw);
        __syncwarp();
        tot += clock64() - c0;
    }
    if (lane == 0) { cyc[blockIdx.x] = tot / reps; piv[blockIdx.x] = t + (int)(sE[0] & 1) * 0; }
    if (lane == 0) st_release_cta(&flag, 1);
}

template <int V>
void run(const u64* d, int B) {
    long long* c; int* p;
    cudaMalloc(&c, B * 8); cudaMalloc(&p, B * 4);
    kv<V><<<B, (V & 8) ? 512 : 32>>>(d, c, p, 20);
    long long hc[256]; int hp[256];
    cudaMemcpy(hc, c, B * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hp, p, B * 4, cudaMemcpyDeviceToHost);
    long long sc = 0; long long sp = 0;
    for (int b = 0; b < B; ++b) { sc += hc[b]; sp += hp[b]; }
    printf("variant %d: %.1f cycles per pivot (%.1f pivots, %.0f cycles per epoch)\n", V, (double)sc / sp,
           (double)sp / B, (double)sc / B);
}

int main() {
    const int B = 64;
    u64 h[64 * 32];
    srand(1);
    for (int i = 0; i < B * 32; ++i) h[i] = ((u64)rand() << 40) ^ ((u64)rand() << 20) ^ (u64)rand();
    u64* d;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0>(d, B); run<7>(d, B); run<8>(d, B); run<15>(d, B); run<24>(d, B); run<31>(d, B);
    return 0;
}
