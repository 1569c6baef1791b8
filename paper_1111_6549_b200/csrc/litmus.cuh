// litmus.cuh -- message-passing litmus kernels for the cross-CTA hand-offs
// the persistent drivers rely on, built from the SAME primitives
// (ple_kernels.cuh): data written with plain stores, published by a CTA
// arrival (bar.sync + red.release.gpu, cta_arrive), awaited by one thread's
// ld.acquire spin (spin_geq / spin_geq2 / the system-scope forms) and read
// with L2-coherent loads (ldcg); and the streamed-output hand-off to the host
// (__threadfence + last-arrival __threadfence_system + a volatile store to
// mapped pinned memory, polled by a host thread that then copies the rows).
// Every payload word is a function of (round, producer, index), so a stale or
// torn read is counted. Diagnostics for gf2cu_litmus (include/gf2cu.h); the
// factorization never runs them.
#pragma once

#include "ple_kernels.cuh"

namespace gf2cu {

struct LitmusParams {
    u64* data;           // [2 parities][producers][kLitmusWords]
    u32* ctr;            // [rounds] arrivals of the round's producers
    u32* ctr2;           // [rounds] second counter (spin_geq2 form)
    u32* done;           // [rounds] the round's consumer finished reading
    u32* err;            // watchdog word
    unsigned long long* checked;
    unsigned long long* failures;
    u32 rounds;
    u32 kind;            // 0: gpu scope, spin_geq; 1: gpu scope, spin_geq2; 2: system scope
    // kind 3 (host): out buffer [rounds][producers][kLitmusWords], mapped flag
    u64* out;
    volatile u32* host_flag;
    u32* out_count;
};

constexpr u32 kLitmusWords = 1024;  // 8 KiB per producer CTA per round

__device__ __forceinline__ u64 litmus_word(u32 round, u32 cta, u32 i) {
    return fmix64(((u64)round << 40) ^ ((u64)cta << 20) ^ (u64)i ^ 0x9e3779b97f4a7c15ull);
}

// kinds 0-2: round k's consumer is CTA k % G, every other CTA produces.
__global__ void __launch_bounds__(512, 1) litmus_kernel(LitmusParams L) {
    __shared__ u32 s_ok;
    __shared__ unsigned long long s_bad;
    const u32 G = gridDim.x, me = blockIdx.x;
    for (u32 k = 0; k < L.rounds; ++k) {
        const u32 cons = k % G;
        u64* buf = L.data + (size_t)(k & 1u) * G * kLitmusWords;
        if (me != cons) {
            // the parity buffer was last read in round k-2: wait for its consumer
            if (k >= 2) {
                if (threadIdx.x == 0)
                    s_ok = (L.kind == 2 ? spin_geq_sys(&L.done[k - 2], 1u, L.err)
                                        : spin_geq(&L.done[k - 2], 1u, L.err)) ? 1u : 0u;
                __syncthreads();
                if (!s_ok) return;
            }
            for (u32 i = threadIdx.x; i < kLitmusWords; i += blockDim.x)
                buf[(size_t)me * kLitmusWords + i] = litmus_word(k, me, i);
            __syncthreads();
            if (threadIdx.x == 0) {
                if (L.kind == 2) {
                    __threadfence_system();  // (peer_signal)
                    red_release_add_sys(&L.ctr[k], 1u);
                } else {
                    red_release_add(&L.ctr[k], 1u);  // (cta_arrive)
                    if (L.kind == 1) red_release_add(&L.ctr2[k], 1u);
                }
            }
        } else {
            if (threadIdx.x == 0) {
                bool ok;
                if (L.kind == 2) ok = spin_geq_sys(&L.ctr[k], G - 1u, L.err);
                else if (L.kind == 1) ok = spin_geq2(&L.ctr[k], G - 1u, &L.ctr2[k], G - 1u, L.err);
                else ok = spin_geq(&L.ctr[k], G - 1u, L.err);
                s_ok = ok ? 1u : 0u;
                s_bad = 0ull;
            }
            __syncthreads();
            if (!s_ok) return;
            unsigned long long bad = 0;
            for (u32 c = 0; c < G; ++c) {
                if (c == me) continue;
                for (u32 i = threadIdx.x; i < kLitmusWords; i += blockDim.x)
                    bad += ldcg(buf + (size_t)c * kLitmusWords + i) != litmus_word(k, c, i);
            }
            if (bad) atomicAdd(&s_bad, bad);
            __syncthreads();
            if (threadIdx.x == 0) {
                atomicAdd(L.checked, (unsigned long long)(G - 1u) * kLitmusWords);
                if (s_bad) atomicAdd(L.failures, s_bad);
                if (L.kind == 2) red_release_add_sys(&L.done[k], 1u);
                else red_release_add(&L.done[k], 1u);
            }
        }
    }
}

// kind 3: every CTA writes its block of round k's output, then the streamed-
// output publication (ple_super.cuh): __threadfence, the round's last
// arrival fences system-wide and stores k + 1 to the mapped host flag.
__global__ void __launch_bounds__(256) litmus_host_kernel(LitmusParams L) {
    const u32 G = gridDim.x, me = blockIdx.x;
    for (u32 k = 0; k < L.rounds; ++k) {
        u64* buf = L.out + ((size_t)k * G + me) * kLitmusWords;
        for (u32 i = threadIdx.x; i < kLitmusWords; i += blockDim.x) buf[i] = litmus_word(k, me, i);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(L.out_count, 1u) == G * (k + 1u) - 1u) {
                __threadfence_system();
                *L.host_flag = k + 1u;
            }
        }
    }
}

}  // namespace gf2cu
