// Microbenchmark: the panel's leader-warp pivot loop (one warp, 32 rows x 64
// columns), current form vs a shorter dependent chain. Checks that both give
// the same pivots / E / D / swaps / origins, then reports cycles per pivot.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/leader scripts/micro/leader.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned u32;

__device__ __forceinline__ u64 shfl64(u64 v, int src) {
    const u32 lo = __shfl_sync(0xffffffffu, (u32)v, src), hi = __shfl_sync(0xffffffffu, (u32)(v >> 32), src);
    return ((u64)hi << 32) | lo;
}

struct Out {
    u64 E[64], D[64];
    u32 q[64], sw[64], org[32];
    u64 acc[32];
    long long cyc;
    int t;
};

// V0: the loop as in ple_kernels.cuh (epoch leader)
__global__ void v0(const u64* in, Out* out, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64];
    const u32 lane = threadIdx.x;
    long long tot = 0;
    int t = 0;
    u64 red, acc;
    u32 org;
    for (int rep = 0; rep < reps; ++rep) {
        red = in[blockIdx.x * 32 + lane];
        acc = 0;
        org = lane;
        t = 0;
        __syncwarp();
        const long long c0 = clock64();
        for (int j = 0; j < 64 && t < 32; ++j) {
            u64 jbit = 1ull << j;
            u64 hi = ~(jbit | (jbit - 1));
            while (j < 64 && t < 32) {
                const bool live = lane >= (u32)t;
                const u32 bal = __ballot_sync(0xffffffffu, live & ((red & jbit) != 0ull));
                if (bal == 0u) break;
                const u32 pl = (u32)(__ffs(bal) - 1), tl = (u32)t & 31u;
                const bool isP = lane == pl;
                const int src = (int)(isP ? tl : pl);
                const u64 xr = shfl64(red, src), xa = shfl64(acc, src);
                const u32 xo = __shfl_sync(0xffffffffu, org, src);
                const u64 pred = isP ? red : xr, pacc = isP ? acc : xa;
                if (isP) {
                    red = xr;
                    acc = xa;
                    org = xo;
                }
                if (lane == tl && !isP) org = xo;
                const u64 tbit = 1ull << t;
                const u64 msk = 0ull - (u64)(live & (lane != (u32)t) & ((red & jbit) != 0ull));
                const u64 Et = pred & hi, Dt = pacc ^ tbit;
                red ^= Et & msk;
                acc ^= Dt & msk;
                if (lane == 0) {
                    sE[t] = Et;
                    sD[t] = Dt;
                    sq[t] = (u32)j;
                    ssw[t] = pl;
                }
                ++t;
                ++j;
                jbit <<= 1;
                hi <<= 1;
            }
        }
        __syncwarp();
        tot += clock64() - c0;
    }
    __syncwarp();
    Out& o = out[blockIdx.x];
    for (int k = lane; k < t; k += 32) {
        o.E[k] = sE[k];
        o.D[k] = sD[k];
        o.q[k] = sq[k];
        o.sw[k] = ssw[k];
    }
    o.org[lane] = org;
    o.acc[lane] = acc;
    if (lane == 0) {
        o.cyc = tot;
        o.t = t;
    }
}

// V0b: V0 in a 512-thread CTA, the other 15 warps parked at a barrier
__global__ void __launch_bounds__(512, 1) v0b(const u64* in, Out* out, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64];
    const u32 lane = threadIdx.x & 31u;
    if (threadIdx.x >= 32) { __syncthreads(); return; }
    long long tot = 0;
    int t = 0;
    u64 red, acc;
    u32 org;
    for (int rep = 0; rep < reps; ++rep) {
        red = in[blockIdx.x * 32 + lane];
        acc = 0;
        org = lane;
        t = 0;
        __syncwarp();
        const long long c0 = clock64();
        for (int j = 0; j < 64 && t < 32; ++j) {
            u64 jbit = 1ull << j;
            u64 hi = ~(jbit | (jbit - 1));
            while (j < 64 && t < 32) {
                const bool live = lane >= (u32)t;
                const u32 bal = __ballot_sync(0xffffffffu, live & ((red & jbit) != 0ull));
                if (bal == 0u) break;
                const u32 pl = (u32)(__ffs(bal) - 1), tl = (u32)t & 31u;
                const bool isP = lane == pl;
                const int src = (int)(isP ? tl : pl);
                const u64 xr = shfl64(red, src), xa = shfl64(acc, src);
                const u32 xo = __shfl_sync(0xffffffffu, org, src);
                const u64 pred = isP ? red : xr, pacc = isP ? acc : xa;
                if (isP) {
                    red = xr;
                    acc = xa;
                    org = xo;
                }
                if (lane == tl && !isP) org = xo;
                const u64 tbit = 1ull << t;
                const u64 msk = 0ull - (u64)(live & (lane != (u32)t) & ((red & jbit) != 0ull));
                const u64 Et = pred & hi, Dt = pacc ^ tbit;
                red ^= Et & msk;
                acc ^= Dt & msk;
                if (lane == 0) {
                    sE[t] = Et;
                    sD[t] = Dt;
                    sq[t] = (u32)j;
                    ssw[t] = pl;
                }
                ++t;
                ++j;
                jbit <<= 1;
                hi <<= 1;
            }
        }
        __syncwarp();
        tot += clock64() - c0;
    }
    __syncwarp();
    Out& o = out[blockIdx.x];
    for (int k = lane; k < t; k += 32) {
        o.E[k] = sE[k];
        o.D[k] = sD[k];
        o.q[k] = sq[k];
        o.sw[k] = ssw[k];
    }
    o.org[lane] = org;
    o.acc[lane] = acc;
    if (lane == 0) {
        o.cyc = tot;
        o.t = t;
    }
    __syncthreads();
}

// V1: shorter chain. The pivot row comes from one shuffle of the ballot's
// first lane (no lane-dependent source select), row t's copy for lane P from a
// shuffle issued before the ballot; eliminated rows XOR the whole pivot row
// (their bits <= j are never read again); the lanes to eliminate are the
// ballot's candidates except P (row t had no bit j unless it is P); pivot
// records are kept in the lane of their slot (no divergent stores).
__global__ void v1(const u64* in, Out* out, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64];
    const u32 lane = threadIdx.x;
    long long tot = 0;
    int t = 0;
    u64 red, acc;
    u32 org;
    for (int rep = 0; rep < reps; ++rep) {
        red = in[blockIdx.x * 32 + lane];
        acc = 0;
        org = lane;
        t = 0;
        u64 myE = 0, myD = 0;
        u32 myq = 0, mysw = 0;
        __syncwarp();
        const long long c0 = clock64();
        for (int j = 0; j < 64 && t < 32; ++j) {
            u64 jbit = 1ull << j;
            while (j < 64 && t < 32) {
                const u32 tl = (u32)t;
                // row t, for the lane that will hold it after the swap
                const u64 rt = shfl64(red, (int)tl), at = shfl64(acc, (int)tl);
                const u32 ot = __shfl_sync(0xffffffffu, org, (int)tl);
                const bool cand = (lane >= tl) & ((red & jbit) != 0ull);
                const u32 bal = __ballot_sync(0xffffffffu, cand);
                if (bal == 0u) break;
                const u32 pl = (u32)(__ffs(bal) - 1);
                const u64 pr = shfl64(red, (int)pl), pa = shfl64(acc, (int)pl);
                const u32 po = __shfl_sync(0xffffffffu, org, (int)pl);
                const bool isP = lane == pl;
                const u64 Dt = pa ^ (1ull << t);
                const bool el = cand & !isP;
                red = isP ? rt : (el ? red ^ pr : red);
                acc = isP ? at : (el ? acc ^ Dt : acc);
                org = isP ? ot : (lane == tl ? po : org);
                if (lane == tl) {  // predicated, the slot's own record
                    myE = pr & ~(jbit | (jbit - 1));
                    myD = Dt;
                    myq = (u32)j;
                    mysw = pl;
                }
                ++t;
                ++j;
                jbit <<= 1;
            }
        }
        if ((int)lane < t) {
            sE[lane] = myE;
            sD[lane] = myD;
            sq[lane] = myq;
            ssw[lane] = mysw;
        }
        __syncwarp();
        tot += clock64() - c0;
    }
    __syncwarp();
    Out& o = out[blockIdx.x];
    for (int k = lane; k < t; k += 32) {
        o.E[k] = sE[k];
        o.D[k] = sD[k];
        o.q[k] = sq[k];
        o.sw[k] = ssw[k];
    }
    o.org[lane] = org;
    o.acc[lane] = acc;
    if (lane == 0) {
        o.cyc = tot;
        o.t = t;
    }
}

// V5: V1 with the pivot row broadcast by redux.sync.or (no FLO/BREV on the chain). The pivot row comes from one shuffle of the ballot's
// first lane (no lane-dependent source select), row t's copy for lane P from a
// shuffle issued before the ballot; eliminated rows XOR the whole pivot row
// (their bits <= j are never read again); the lanes to eliminate are the
// ballot's candidates except P (row t had no bit j unless it is P); pivot
// records are kept in the lane of their slot (no divergent stores).
__global__ void v5(const u64* in, Out* out, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64];
    const u32 lane = threadIdx.x;
    long long tot = 0;
    int t = 0;
    u64 red, acc;
    u32 org;
    for (int rep = 0; rep < reps; ++rep) {
        red = in[blockIdx.x * 32 + lane];
        acc = 0;
        org = lane;
        t = 0;
        u64 myE = 0, myD = 0;
        u32 myq = 0, mysw = 0;
        __syncwarp();
        const long long c0 = clock64();
        for (int j = 0; j < 64 && t < 32; ++j) {
            u64 jbit = 1ull << j;
            while (j < 64 && t < 32) {
                const u32 tl = (u32)t;
                // row t, for the lane that will hold it after the swap
                const u64 rt = shfl64(red, (int)tl), at = shfl64(acc, (int)tl);
                const u32 ot = __shfl_sync(0xffffffffu, org, (int)tl);
                const bool cand = (lane >= tl) & ((red & jbit) != 0ull);
                const u32 bal = __ballot_sync(0xffffffffu, cand);
                if (bal == 0u) break;
                const bool isP = ((bal & (0u - bal)) >> lane) & 1u;
                const u64 mine = isP ? red : 0ull;
                const u64 pr = ((u64)__reduce_or_sync(0xffffffffu, (u32)(mine >> 32)) << 32) |
                               __reduce_or_sync(0xffffffffu, (u32)mine);
                const u32 pl = (u32)(__ffs(bal) - 1);
                const u64 pa = shfl64(acc, (int)pl);
                const u32 po = __shfl_sync(0xffffffffu, org, (int)pl);
                const u64 Dt = pa ^ (1ull << t);
                const bool el = cand & !isP;
                red = isP ? rt : (el ? red ^ pr : red);
                acc = isP ? at : (el ? acc ^ Dt : acc);
                org = isP ? ot : (lane == tl ? po : org);
                if (lane == tl) {  // predicated, the slot's own record
                    myE = pr & ~(jbit | (jbit - 1));
                    myD = Dt;
                    myq = (u32)j;
                    mysw = pl;
                }
                ++t;
                ++j;
                jbit <<= 1;
            }
        }
        if ((int)lane < t) {
            sE[lane] = myE;
            sD[lane] = myD;
            sq[lane] = myq;
            ssw[lane] = mysw;
        }
        __syncwarp();
        tot += clock64() - c0;
    }
    __syncwarp();
    Out& o = out[blockIdx.x];
    for (int k = lane; k < t; k += 32) {
        o.E[k] = sE[k];
        o.D[k] = sD[k];
        o.q[k] = sq[k];
        o.sw[k] = ssw[k];
    }
    o.org[lane] = org;
    o.acc[lane] = acc;
    if (lane == 0) {
        o.cyc = tot;
        o.t = t;
    }
}

// V2: two columns per ballot round. Ballots of bits j and j+1 decide both
// pivots with warp-uniform integer logic: after pivot P0 (column j), row i's
// bit j+1 is b1_i ^ (e & b0_i) with e = the pivot row's bit j+1, and the old
// row t sits in lane P0. Then one gather per pivot row.
__global__ void v2(const u64* in, Out* out, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64];
    const u32 lane = threadIdx.x;
    long long tot = 0;
    int t = 0;
    u64 red, acc;
    u32 org;
    const int jmax = 64, tmax = 32;
    for (int rep = 0; rep < reps; ++rep) {
        red = in[blockIdx.x * 32 + lane];
        acc = 0;
        org = lane;
        t = 0;
        u64 myE = 0, myD = 0;
        u32 myq = 0, mysw = 0;
        __syncwarp();
        const long long c0 = clock64();
        for (int j = 0; j < jmax && t < tmax; ++j) {
            while (j < jmax && t < tmax) {
                const u32 tl = (u32)t;
                const bool pair = (j + 1 < jmax) && (t + 1 < tmax);
                const u32 t1 = pair ? tl + 1u : tl;
                // rows t and t+1 (for the lanes that receive them in the swaps)
                const u64 rt = shfl64(red, (int)tl), at = shfl64(acc, (int)tl);
                const u32 ot = __shfl_sync(0xffffffffu, org, (int)tl);
                const u64 ru = shfl64(red, (int)t1), au = shfl64(acc, (int)t1);
                const u32 ou = __shfl_sync(0xffffffffu, org, (int)t1);
                const u32 b0 = (u32)(red >> j) & 1u;
                const u32 b1 = pair ? (u32)(red >> (j + 1)) & 1u : 0u;
                const u32 B0 = __ballot_sync(0xffffffffu, (lane >= tl) & (b0 != 0u));
                const u32 B1 = __ballot_sync(0xffffffffu, b1 != 0u);
                if (B0 == 0u) break;
                const u32 P0 = (u32)(__ffs(B0) - 1);
                const u32 m0 = 1u << P0;
                const u32 E0 = B0 & ~m0;                 // rows eliminated by pivot 0
                const u32 e = (B1 >> P0) & 1u;           // pivot 0's bit j+1
                const u32 bt = (B1 >> tl) & 1u;          // row t's bit j+1
                u32 C1 = (B1 ^ (E0 & (0u - e))) & ~m0 & (0xfffffffeu << tl);
                if (P0 != tl && bt) C1 |= m0;            // old row t now at P0
                if (!pair) C1 = 0u;
                // pivot 0: gather, eliminate, swap
                const u64 pr0 = shfl64(red, (int)P0), pa0 = shfl64(acc, (int)P0);
                const u32 po0 = __shfl_sync(0xffffffffu, org, (int)P0);
                const u64 D0 = pa0 ^ (1ull << tl);
                const bool isP0 = lane == P0;
                const bool el0 = (E0 >> lane) & 1u;
                // content after pivot 0
                u64 r0 = isP0 ? rt : (el0 ? red ^ pr0 : red);
                u64 a0 = isP0 ? at : (el0 ? acc ^ D0 : acc);
                u32 o0 = isP0 ? ot : (lane == tl ? po0 : org);
                if (lane == tl) {
                    myE = pr0 & (~0ull << j << 1);
                    myD = D0;
                    myq = (u32)j;
                    mysw = P0;
                }
                if (C1 == 0u) {  // column j+1 has no candidate (or no pair): one pivot
                    red = r0;
                    acc = a0;
                    org = o0;
                    ++t;
                    ++j;
                    continue;
                }
                const u32 P1 = (u32)(__ffs(C1) - 1);
                const u32 m1 = 1u << P1;
                const u32 E1 = C1 & ~m1;
                // pivot 1's row (content at lane P1 after pivot 0)
                const u64 xr = shfl64(red, (int)P1), xa = shfl64(acc, (int)P1);
                const u32 xo = __shfl_sync(0xffffffffu, org, (int)P1);
                const bool p1old = (P1 == P0);  // the old row t (not eliminated)
                const bool p1el = (E0 >> P1) & 1u;
                const u64 pr1 = p1old ? rt : (p1el ? xr ^ pr0 : xr);
                const u64 pa1 = p1old ? at : (p1el ? xa ^ D0 : xa);
                const u32 po1 = p1old ? ot : xo;
                // content at lane t+1 after pivot 0 (moves to P1)
                const bool uold = (t1 == P0);
                const bool uel = (E0 >> t1) & 1u;
                const u64 ur = uold ? rt : (uel ? ru ^ pr0 : ru);
                const u64 ua = uold ? at : (uel ? au ^ D0 : au);
                const u32 uo = uold ? ot : ou;
                const u64 D1 = pa1 ^ (1ull << t1);
                const bool isP1 = lane == P1;
                const bool el1 = (E1 >> lane) & 1u;
                red = isP1 ? ur : (el1 ? r0 ^ pr1 : r0);
                acc = isP1 ? ua : (el1 ? a0 ^ D1 : a0);
                org = isP1 ? uo : (lane == t1 ? po1 : o0);
                if (lane == t1) {
                    myE = pr1 & (~0ull << (j + 1) << 1);
                    myD = D1;
                    myq = (u32)(j + 1);
                    mysw = P1;
                }
                t += 2;
                j += 2;
            }
        }
        if ((int)lane < t) {
            sE[lane] = myE;
            sD[lane] = myD;
            sq[lane] = myq;
            ssw[lane] = mysw;
        }
        __syncwarp();
        tot += clock64() - c0;
    }
    __syncwarp();
    Out& o = out[blockIdx.x];
    for (int k = lane; k < t; k += 32) {
        o.E[k] = sE[k];
        o.D[k] = sD[k];
        o.q[k] = sq[k];
        o.sw[k] = ssw[k];
    }
    o.org[lane] = org;
    o.acc[lane] = acc;
    if (lane == 0) {
        o.cyc = tot;
        o.t = t;
    }
}

// V3: decision warp + shadow warp. Warp 0 keeps only the reduced rows (red)
// and publishes each pivot's ballot; warp 1 holds the same rows' combinations
// (acc) and origins (org) and replays the swaps / eliminations from the
// published ballots, off the decision chain.
__global__ void __launch_bounds__(64, 1) v3(const u64* in, Out* out, int reps) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64], ssw[64], sbal[64];
    __shared__ volatile int sprog;
    __shared__ int sfin;
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    long long tot = 0;
    int t = 0;
    u64 red = 0, acc = 0;
    u32 org = lane;
    for (int rep = 0; rep < reps; ++rep) {
        if (threadIdx.x == 0) { sprog = 0; sfin = -1; }
        __syncthreads();
        t = 0;
        if (wid == 0) {
            red = in[blockIdx.x * 32 + lane];
            const long long c0 = clock64();
            for (int j = 0; j < 64 && t < 32; ++j) {
                u64 jbit = 1ull << j;
                while (j < 64 && t < 32) {
                    const u32 tl = (u32)t;
                    const u64 rt = shfl64(red, (int)tl);
                    const bool cand = (lane >= tl) & ((red & jbit) != 0ull);
                    const u32 bal = __ballot_sync(0xffffffffu, cand);
                    if (bal == 0u) break;
                    const u32 pl = (u32)(__ffs(bal) - 1);
                    const u64 pr = shfl64(red, (int)pl);
                    const bool isP = lane == pl;
                    red = isP ? rt : ((cand & !isP) ? red ^ pr : red);
                    sE[t] = pr & ~(jbit | (jbit - 1));
                    sq[t] = (u32)j;
                    *(volatile u32*)&sbal[t] = bal;
#ifndef NOFENCE
                    __threadfence_block();
#endif
                    sprog = t + 1;
                    ++t;
                    ++j;
                    jbit <<= 1;
                }
            }
            if (lane == 0) { __threadfence_block(); *(volatile int*)&sfin = t; }
            __syncwarp();
            tot += clock64() - c0;
        } else {
            acc = 0;
            org = lane;
            int s = 0;
            for (;;) {
                const int fin = *(volatile int*)&sfin;
                const int pr = sprog;
                for (; s < pr; ++s) {
                    const u32 bal = *(volatile u32*)&sbal[s];
                    const u32 tl = (u32)s, pl = (u32)(__ffs(bal) - 1);
                    const u64 at = shfl64(acc, (int)tl), pa = shfl64(acc, (int)pl);
                    const u32 ot = __shfl_sync(0xffffffffu, org, (int)tl), po = __shfl_sync(0xffffffffu, org, (int)pl);
                    const bool isP = lane == pl;
                    const bool el = ((bal >> lane) & 1u) & !isP;
                    const u64 Dt = pa ^ (1ull << s);
                    acc = isP ? at : (el ? acc ^ Dt : acc);
                    org = isP ? ot : (lane == tl ? po : org);
                    sD[s] = Dt;
                    ssw[s] = pl;
                }
                if (fin >= 0 && s >= fin) break;
            }
            t = s;
        }
        __syncthreads();
    }
    __syncthreads();
    Out& o = out[blockIdx.x];
    if (wid == 1) {
        for (int k = lane; k < t; k += 32) {
            o.E[k] = sE[k];
            o.D[k] = sD[k];
            o.q[k] = sq[k];
            o.sw[k] = ssw[k];
        }
        o.org[lane] = org;
        o.acc[lane] = acc;
    }
    if (threadIdx.x == 0) {
        o.cyc = tot;
        o.t = t;
    }
}

int main(int argc, char** argv) {
    const int nb = 64, reps = 200;
    u64* h = (u64*)malloc(nb * 32 * 8);
    u64 x = 88172645463325252ull;
    for (int i = 0; i < nb * 32; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = x;
        if (argc > 1 && (i % 5) == 0) h[i] &= 0xffff0000ffff0000ull;  // some structure
    }
    u64* d;
    Out *o0, *o1, *o2;
    cudaMalloc(&d, nb * 32 * 8);
    cudaMalloc(&o0, nb * sizeof(Out));
    cudaMalloc(&o1, nb * sizeof(Out));
    cudaMalloc(&o2, nb * sizeof(Out));
    cudaMemcpy(d, h, nb * 32 * 8, cudaMemcpyHostToDevice);
    cudaMemset(o0, 0, nb * sizeof(Out));
    cudaMemset(o1, 0, nb * sizeof(Out));
    v0<<<nb, 32>>>(d, o0, reps);
    v1<<<nb, 32>>>(d, o1, reps);
    v2<<<nb, 32>>>(d, o2, reps);
    if (getenv("V0B")) v0b<<<nb, 512>>>(d, o2, reps);
    if (getenv("V3")) v3<<<nb, 64>>>(d, o2, reps);
    if (getenv("V5")) v5<<<nb, 32>>>(d, o2, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    Out* a = (Out*)malloc(nb * sizeof(Out));
    Out* b = (Out*)malloc(nb * sizeof(Out));
    cudaMemcpy(a, o0, nb * sizeof(Out), cudaMemcpyDeviceToHost);
    cudaMemcpy(b, o1, nb * sizeof(Out), cudaMemcpyDeviceToHost);
    int bad = 0;
    double c0 = 0, c1 = 0, c2 = 0, piv = 0;
    for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
        for (int k = 0; k < nb; ++k) c1 += b[k].cyc;
        cudaMemcpy(b, o2, nb * sizeof(Out), cudaMemcpyDeviceToHost);
        for (int k = 0; k < nb; ++k) c2 += b[k].cyc;
        c0 = 0; piv = 0;
    }
    for (int k = 0; k < nb; ++k) {
        if (a[k].t != b[k].t) ++bad;
        for (int i = 0; i < a[k].t; ++i)
            if (a[k].E[i] != b[k].E[i] || a[k].D[i] != b[k].D[i] || a[k].q[i] != b[k].q[i] || a[k].sw[i] != b[k].sw[i]) ++bad;
        for (int l = 0; l < 32; ++l)
            if (l >= a[k].t && (a[k].org[l] != b[k].org[l] || a[k].acc[l] != b[k].acc[l])) ++bad;
        for (int l = 0; l < a[k].t; ++l)
            if (a[k].org[l] != b[k].org[l]) ++bad;
        c0 += a[k].cyc;
        piv += (double)a[k].t * reps;
    }
    }
    printf("pivots/warp %.1f  v0 %.1f cyc/pivot  v1 %.1f  v2 %.1f  mismatches %d\n", piv / nb / reps, c0 / piv,
           c1 / piv, c2 / piv, bad);
    return bad != 0;
}
