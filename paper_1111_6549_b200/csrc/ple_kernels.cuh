// ple_kernels.cuh -- sm_100a kernels of the B200 block-iterative PLE over F2.
//
// Device layout (tile-major): the matrix is cut into 64-byte column tiles
// (8 words = 512 columns); tile T of all rows is contiguous in HBM:
//     word x of physical row i  ->  mat[((x >> 3) * m + i) * 8 + (x & 7)]
// so a CTA that sweeps one tile down the rows streams sequential memory.
// Rows are never moved during the factorization: `perm` maps a position
// (the reference's row index after its swaps) to a physical row, and the
// final untile pass gathers rows back into position order.
//
// One 64-column panel (= word column w) per step:
//   panel_factor    (1 CTA)  pivot search on the panel words of rows >= r:
//                            transposed single-warp elimination on a 128-row
//                            window, CTA-wide scan of the other rows on a
//                            window miss. Replaces partial_ple (ple.hpp:57-130)
//                            and the swap replay (ple.hpp:187-188).
//   panel_apply     (grid)   per row: multipliers c and the combination d of
//                            RAW pivot rows that finishes its tail (d folds the
//                            unit-lower TRSM of ple.hpp:191-193 into the
//                            update); writes the compressed multipliers
//                            (ple.hpp:232-236); stages raw pivot-row tails.
//   trailing_update (grid)   8 Gray-code tables x 256 entries per 64-byte
//                            tile in shared memory (make_table,
//                            gray_code.hpp:88-134), then tail ^= sum_g
//                            T_g[byte_g(d)] for every row >= r (ple.hpp:
//                            208-229), 128-bit loads/stores, software-pipelined.
#pragma once

#include <cstdint>

namespace gf2cu {

using u64 = unsigned long long;
using u32 = unsigned int;

constexpr int kPanelThreads = 256;     // panel_factor CTA
constexpr int kWin = 128;              // window rows (two 64-bit halves)
constexpr int kApplyThreads = 256;     // panel_apply CTA
constexpr int kTrailThreads = 512;     // trailing_update CTA
constexpr int kTileWords = 8;          // 64-byte column tile
constexpr int kTables = 8;             // 8 tables of 8 coefficient bits
constexpr int kTableBytes = kTables * 256 * kTileWords * 8;  // 128 KiB
constexpr int kUnroll = 4;             // row groups per lane per iteration
constexpr int kRowsPerIter = kTrailThreads / 4 * kUnroll;    // 512

struct StepState {
    u32 r;    // pivots before the current step
    u32 rb;   // pivots found by the current step
    u32 pad0, pad1;
};

struct PanelOut {
    u64 E[64];   // pivot t: its reduced panel word, bits > qb[t] only
    u64 D[64];   // pivot t: combination of raw pivot rows giving its U row
    u32 qb[64];  // pivot t: column within the panel word
};

struct Params {
    u64* mat;        // tile-major, Wpad8/8 tiles x m rows x 8 words
    u32* perm;       // position -> physical row
    u64* pb;         // panel word per position (current step)
    ulonglong2* info;  // per position: {d, physical row}
    u64* stage;      // tile-major raw pivot rows: tiles x 64 rows x 8 words
    StepState* state;
    PanelOut* pout;
    u32* swaps;      // LAPACK transpositions (absolute positions)
    u32* qcol;       // absolute pivot columns
    u32* rhist;      // r at the start of each step
    u32* rbhist;     // rb of each step
    volatile u32* host_r;  // mapped pinned mirror of (r + rb), may be null
    u32 m, n, W, Wpad8;
};

__device__ __forceinline__ u64 low_mask64(int k) {
    return k >= 64 ? ~0ull : ((1ull << k) - 1ull);
}

__device__ __forceinline__ u64* tword(u64* mat, u32 m, u32 row, u32 x) {
    return mat + (((size_t)(x >> 3) * m + row) << 3) + (x & 7u);
}

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ u64 shfl64(u64 v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

// 32x32 bit transpose across a warp: on return lane l bit b = input lane b
// bit l.
__device__ __forceinline__ u32 transpose32(u32 x) {
    const u32 lane = threadIdx.x & 31u;
    const u32 hi[5] = {0xFFFF0000u, 0xFF00FF00u, 0xF0F0F0F0u, 0xCCCCCCCCu, 0xAAAAAAAAu};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int j = 16 >> k;
        const u32 y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & hi[k]) | ((y >> j) & ~hi[k])) : ((x & ~hi[k]) | ((y << j) & hi[k]));
    }
    return x;
}

// ---------------------------------------------------------------------------
// layout conversion: row-major (stride Wp) <-> tile-major; untile also
// gathers rows into position order through perm.
// ---------------------------------------------------------------------------
__global__ void tile_kernel(const u64* __restrict__ src, u64* __restrict__ dst, u32 m, u32 Wp,
                            u32 Wpad8) {
    const u32 per_row = Wpad8 >> 1;
    const u64 total = (u64)m * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 row = (u32)(e / per_row), x = 2u * (u32)(e - (u64)row * per_row);
        *reinterpret_cast<ulonglong2*>(tword(dst, m, row, x)) =
            *reinterpret_cast<const ulonglong2*>(src + (size_t)row * Wp + x);
    }
}

__global__ void untile_kernel(const u64* __restrict__ src, u64* __restrict__ dst,
                              const u32* __restrict__ perm, u32 m, u32 Wp, u32 Wpad8) {
    const u32 per_row = Wpad8 >> 1;
    const u64 total = (u64)m * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 row = (u32)(e / per_row), x = 2u * (u32)(e - (u64)row * per_row);
        const u32 ph = perm ? perm[row] : row;
        *reinterpret_cast<ulonglong2*>(dst + (size_t)row * Wp + x) =
            *reinterpret_cast<const ulonglong2*>(tword(const_cast<u64*>(src), m, ph, x));
    }
}

// ---------------------------------------------------------------------------
// init: identity permutation, panel buffer = word 0 of every row.
// ---------------------------------------------------------------------------
__global__ void ple_init_kernel(Params p) {
    const u32 stride = gridDim.x * blockDim.x;
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < p.m; i += stride) {
        p.perm[i] = i;
        p.pb[i] = *tword(p.mat, p.m, i, 0);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.state->r = 0;
        p.state->rb = 0;
    }
}

// ---------------------------------------------------------------------------
// panel_factor
// ---------------------------------------------------------------------------
struct PanelShared {
    u64 E[64], D[64];
    u32 q[64];
    u64 wraw[kWin];
    u32 wphys[kWin];
    int cmd;  // 0 = scan, 1 = exit
    int t, j;
    u64 warp_best[kPanelThreads / 32];
    u64 best;  // (first column << 32) | offset
    u64 o_red, o_acc, o_raw;
    u32 o_phys;
    u32 r;
};

// All kPanelThreads threads: scan positions r + [nwin, nrem) reducing each raw
// panel word by the t pivots found so far; sh.best = the smallest
// (first set column >= j, offset), with the winner's reduced state in sh.o_*.
__device__ void panel_scan(const Params& p, PanelShared& sh, u32 r, u32 nwin, u32 nrem) {
    const int t = sh.t, j = sh.j;
    u64 best = ~0ull, b_red = 0, b_acc = 0;
    for (u32 off = nwin + threadIdx.x; off < nrem; off += kPanelThreads) {
        u64 v = p.pb[r + off], a = 0;
        for (int s = 0; s < t; ++s) {
            const u64 msk = 0ull - ((v >> sh.q[s]) & 1ull);
            v ^= sh.E[s] & msk;
            a ^= sh.D[s] & msk;
        }
        const u64 mk = v & ~low_mask64(j);
        if (mk) {
            const u64 key = ((u64)(__ffsll((long long)mk) - 1) << 32) | off;
            if (key < best) {
                best = key;
                b_red = v;
                b_acc = a;
            }
        }
    }
    u64 wb = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, wb, o);
        wb = other < wb ? other : wb;
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh.warp_best[wid] = wb;
    named_bar(2, kPanelThreads);
    if (threadIdx.x == 0) {
        u64 b = ~0ull;
        for (int k = 0; k < kPanelThreads / 32; ++k) b = sh.warp_best[k] < b ? sh.warp_best[k] : b;
        sh.best = b;
    }
    named_bar(2, kPanelThreads);
    if (best != ~0ull && best == sh.best) {
        const u32 off = (u32)(best & 0xffffffffu);
        sh.o_red = b_red;
        sh.o_acc = b_acc;
        sh.o_raw = p.pb[r + off];
        sh.o_phys = p.perm[r + off];
    }
    named_bar(2, kPanelThreads);
}

// Transposed window state of warp 0: lane l owns panel columns l and l+32
// (M[h], h = 0/1) and coefficient columns (pivot indices) l and l+32 (A[h]);
// each is a 128-bit mask over the window rows (lo = rows 0..63, hi = 64..127).
struct Col128 {
    u64 lo, hi;
};

// Row swap t <-> p on one column mask, then the elimination XOR if `cond`
// holds for the pivot row's bit (bit t after the swap, returned).
__device__ __forceinline__ bool swap_elim(Col128& x, u64 tm, u64 pl, u64 ph, int t, u64 Rlo,
                                          u64 Rhi, bool xor_if_set, bool force) {
    const u64 bt = (x.lo >> t) & 1ull;
    const u64 bp = ((x.lo & pl) | (x.hi & ph)) ? 1ull : 0ull;
    const u64 dm = 0ull - (bt ^ bp);
    x.lo ^= dm & (tm | pl);
    x.hi ^= dm & ph;
    const bool piv = bp != 0;
    const u64 cm = 0ull - (u64)(force || (xor_if_set && piv));
    x.lo ^= cm & Rlo;
    x.hi ^= cm & Rhi;
    return piv;
}

__global__ void __launch_bounds__(kPanelThreads, 1) panel_factor_kernel(Params p, u32 w) {
    __shared__ PanelShared sh;
    if (threadIdx.x == 0) {
        const StepState st = *p.state;
        sh.r = st.r + st.rb;
    }
    __syncthreads();
    const u32 r = sh.r;
    if (threadIdx.x == 0) {
        p.state->r = r;
        p.state->rb = 0;
        p.rhist[w] = r;
        p.rbhist[w] = 0;
    }
    if (r >= p.m) {
        if (threadIdx.x == 0 && p.host_r) {
            *p.host_r = r;
            __threadfence_system();
        }
        return;
    }
    const u32 nrem = p.m - r;
    const u32 nwin = nrem < (u32)kWin ? nrem : (u32)kWin;
    const int jmax = (int)min(64u, p.n - 64u * w);

    if (threadIdx.x >= 32) {
        for (;;) {
            named_bar(1, kPanelThreads);
            if (sh.cmd != 0) break;
            panel_scan(p, sh, r, nwin, nrem);
        }
        return;
    }

    // ---- warp 0 ----
    const int lane = threadIdx.x;
    u32 part[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const u32 off = 32u * i + lane;
        u64 v = 0ull;
        if (off < nwin) {
            v = p.pb[r + off];
            sh.wraw[off] = v;
            sh.wphys[off] = p.perm[r + off];
        }
        part[i][0] = transpose32((u32)v);
        part[i][1] = transpose32((u32)(v >> 32));
    }
    Col128 M[2], A[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        M[h].lo = (u64)part[0][h] | ((u64)part[1][h] << 32);
        M[h].hi = (u64)part[2][h] | ((u64)part[3][h] << 32);
        A[h].lo = 0ull;
        A[h].hi = 0ull;
    }
    const u64 winlo = nwin >= 64 ? ~0ull : low_mask64((int)nwin);
    const u64 winhi = nwin > 64 ? low_mask64((int)nwin - 64) : 0ull;

    int t = 0;
    int out_next = nwin < nrem ? 0 : 64;
    for (int j = 0; j < jmax && (u32)t < nrem; ++j) {
        const int hj = j >> 5, oj = j & 31;
        const u64 clo = shfl64(hj ? M[1].lo : M[0].lo, oj);
        const u64 chi = shfl64(hj ? M[1].hi : M[0].hi, oj);
        const u64 flo = clo & winlo & ~low_mask64(t);
        const u64 fhi = chi & winhi;
        const u64 tm = 1ull << t;
        const u64 above_t = ~low_mask64(t + 1);
        if (flo | fhi) {
            const int pidx = flo ? (__ffsll((long long)flo) - 1) : (64 + __ffsll((long long)fhi) - 1);
            const u64 pl = pidx < 64 ? (1ull << pidx) : 0ull;
            const u64 ph = pidx >= 64 ? (1ull << (pidx - 64)) : 0ull;
            // rows > t holding column j after the swap
            const u64 btj = 0ull - ((clo >> t) & 1ull);
            const u64 Rlo = ((clo & ~pl) | (btj & pl)) & above_t;
            const u64 Rhi = (chi & ~ph) | (btj & ph);
            u32 eb[2], db[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = 32 * h + lane;
                const bool pe = swap_elim(M[h], tm, pl, ph, t, Rlo, Rhi, c > j, false);
                const bool pd = swap_elim(A[h], tm, pl, ph, t, Rlo, Rhi, c < t, c == t);
                eb[h] = __ballot_sync(0xffffffffu, pe && c > j);
                db[h] = __ballot_sync(0xffffffffu, pd && c < t);
            }
            if (lane == 0) {
                sh.E[t] = (u64)eb[0] | ((u64)eb[1] << 32);
                sh.D[t] = ((u64)db[0] | ((u64)db[1] << 32)) | tm;
                sh.q[t] = (u32)j;
                p.swaps[r + t] = r + (u32)pidx;
                p.qcol[r + t] = 64u * w + (u32)j;
                if (pidx != t) {
                    const u64 a = sh.wraw[t];
                    sh.wraw[t] = sh.wraw[pidx];
                    sh.wraw[pidx] = a;
                    const u32 b = sh.wphys[t];
                    sh.wphys[t] = sh.wphys[pidx];
                    sh.wphys[pidx] = b;
                }
            }
            __syncwarp();
            ++t;
            continue;
        }
        // ---- window miss: the remaining rows decide ----
        if (j < out_next) continue;  // no row outside has this column
        if (lane == 0) {
            sh.cmd = 0;
            sh.t = t;
            sh.j = j;
        }
        __syncwarp();
        named_bar(1, kPanelThreads);
        panel_scan(p, sh, r, nwin, nrem);
        const u64 best = sh.best;
        if (best == ~0ull) {
            out_next = 64;
            continue;
        }
        out_next = (int)(best >> 32);
        if (out_next != j) continue;  // column j has no pivot anywhere
        // pivot from outside the window: it replaces window row t, which moves
        // to the pivot's old position
        const u32 P = (u32)(best & 0xffffffffu);
        const u64 o_red = sh.o_red, o_acc = sh.o_acc;
        const u64 Rlo = clo & winlo & above_t;
        const u64 Rhi = chi & winhi;
        u32 eb[2], db[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = 32 * h + lane;
            const bool be = (o_red >> c) & 1ull;
            const bool bd = (o_acc >> c) & 1ull;
            M[h].lo = (M[h].lo & ~tm) | (be ? tm : 0ull);
            A[h].lo = (A[h].lo & ~tm) | (bd ? tm : 0ull);
            const u64 cme = 0ull - (u64)(be && c > j);
            M[h].lo ^= cme & Rlo;
            M[h].hi ^= cme & Rhi;
            const u64 cmd = 0ull - (u64)((bd && c < t) || c == t);
            A[h].lo ^= cmd & Rlo;
            A[h].hi ^= cmd & Rhi;
            eb[h] = __ballot_sync(0xffffffffu, be && c > j);
            db[h] = __ballot_sync(0xffffffffu, bd && c < t);
        }
        if (lane == 0) {
            sh.E[t] = (u64)eb[0] | ((u64)eb[1] << 32);
            sh.D[t] = ((u64)db[0] | ((u64)db[1] << 32)) | tm;
            sh.q[t] = (u32)j;
            p.swaps[r + t] = r + P;
            p.qcol[r + t] = 64u * w + (u32)j;
            p.pb[r + P] = sh.wraw[t];
            p.perm[r + P] = sh.wphys[t];
            sh.wraw[t] = sh.o_raw;
            sh.wphys[t] = sh.o_phys;
        }
        __syncwarp();
        ++t;
    }
    if (lane == 0) sh.cmd = 1;
    __syncwarp();
    named_bar(1, kPanelThreads);

    for (u32 off = lane; off < nwin; off += 32) {
        p.pb[r + off] = sh.wraw[off];
        p.perm[r + off] = sh.wphys[off];
    }
    for (int k = lane; k < t; k += 32) {
        p.pout->E[k] = sh.E[k];
        p.pout->D[k] = sh.D[k];
        p.pout->qb[k] = sh.q[k];
    }
    if (lane == 0) {
        p.state->rb = (u32)t;
        p.rbhist[w] = (u32)t;
        if (p.host_r) {
            *p.host_r = r + (u32)t;
            __threadfence_system();
        }
    }
}

// ---------------------------------------------------------------------------
// panel_apply: multipliers + combination per row, compressed write, staging.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kApplyThreads) panel_apply_kernel(Params p, u32 w) {
    __shared__ u64 sE[64], sD[64];
    __shared__ u32 sq[64];
    const StepState st = *p.state;
    const u32 r = st.r, rb = st.rb;
    if (r >= p.m) return;
    for (u32 k = threadIdx.x; k < 64; k += blockDim.x) {
        const bool v = k < rb;
        sE[k] = v ? p.pout->E[k] : 0ull;
        sD[k] = v ? p.pout->D[k] : 0ull;
        sq[k] = v ? p.pout->qb[k] : 0u;
    }
    __syncthreads();

    const u32 gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const u32 gsize = gridDim.x * blockDim.x;
    const u32 w0 = r >> 6, b0 = r & 63;
    for (u32 pos = r + gtid; pos < p.m; pos += gsize) {
        u64 v = p.pb[pos], a = 0, c = 0;
        const u32 ph = p.perm[pos];
        const u32 off = pos - r;
        const u32 tl = off < rb ? off : rb;
        // branch-free forward elimination against the panel's pivots
#pragma unroll 8
        for (u32 s = 0; s < 64; ++s) {
            if (s >= tl) break;
            const u64 bit = (v >> sq[s]) & 1ull;
            const u64 msk = 0ull - bit;
            v ^= sE[s] & msk;
            a ^= sD[s] & msk;
            c |= bit << s;
        }
        u64 epart = 0;
        if (off < rb) {
            c |= 1ull << off;
            epart = v & ~low_mask64((int)sq[off] + 1);
        }
        p.info[pos] = make_ulonglong2(a, (u64)ph);
        const u64 lo = c << b0;
        const u64 hi = b0 ? (c >> (64 - b0)) : 0ull;
        if (w0 == w) {
            *tword(p.mat, p.m, ph, w) = lo | epart;
        } else {
            *tword(p.mat, p.m, ph, w0) |= lo;
            if (w0 + 1 == w) {
                *tword(p.mat, p.m, ph, w) = hi | epart;
            } else {
                if (hi) *tword(p.mat, p.m, ph, w0 + 1) |= hi;
                *tword(p.mat, p.m, ph, w) = epart;
            }
        }
    }

    // stage raw pivot-row tails, tiles [x0/8, Wpad8/8): stage[(T*64 + t)*8 + k]
    if (w + 1 < p.W && rb > 0) {
        const u32 x0 = (w + 1) & ~7u;
        const u32 span2 = (p.Wpad8 - x0) >> 1;  // 16-byte units per row
        const u32 total = rb * span2;
        for (u32 e = gtid; e < total; e += gsize) {
            const u32 t = e / span2, x = x0 + 2u * (e - t * span2);
            const u32 ph = p.perm[r + t];
            *reinterpret_cast<ulonglong2*>(p.stage + (((size_t)(x >> 3) * 64 + t) << 3) + (x & 7u)) =
                *reinterpret_cast<const ulonglong2*>(tword(p.mat, p.m, ph, x));
        }
    }
}

// ---------------------------------------------------------------------------
// trailing_update
// ---------------------------------------------------------------------------
// Shared-memory table layout (conflict-free for the row-pair rotation):
//   entry e of table g, 16-byte chunk ch  ->  byte
//   ((g >> 1) * 256 + e) * 128 + (g & 1) * 64 + ch * 16
// A quarter-warp of an LDS.128 covers two rows (4 lanes each); even rows read
// table g, odd rows table g ^ 1, so the two 64-byte reads fill the two halves
// of the 32 banks.
__device__ __forceinline__ u32 tab_off(u32 g, u32 e, u32 ch) {
    return (((g >> 1) * 256u + e) << 7) + ((g & 1u) << 6) + (ch << 4);
}

__device__ __forceinline__ void xor2(ulonglong2& a, const ulonglong2& b) {
    a.x ^= b.x;
    a.y ^= b.y;
}

// Build the 8 Gray-code tables for tile `tile` from the staged raw pivot rows
// (rows t >= rb and words <= w read as zero). Thread layout (512):
// ch = tid&3, g&1 = (tid>>2)&1, s_lo = (tid>>3)&3, g>>1 = (tid>>5)&3,
// s_hi = (tid>>7)&3; each thread walks entries gray(16 s + k), k = 0..15,
// with its 8 source chunks in registers: one XOR per entry
// (make_table, gray_code.hpp:105-112).
__device__ __forceinline__ void build_tables(const Params& p, unsigned char* smem, u32 tile,
                                             u32 w, u32 rb) {
    const u32 tid = threadIdx.x;
    const u32 ch = tid & 3u;
    const u32 g = (((tid >> 5) & 3u) << 1) | ((tid >> 2) & 1u);
    const u32 s = (((tid >> 7) & 3u) << 2) | ((tid >> 3) & 3u);
    const u32 x = tile * 8u + 2u * ch;
    const u64* st = p.stage + (((size_t)tile * 64) << 3) + 2u * ch;
    ulonglong2 R[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const u32 t = 8u * g + b;
        ulonglong2 v = make_ulonglong2(0ull, 0ull);
        if (t < rb) v = *reinterpret_cast<const ulonglong2*>(st + ((size_t)t << 3));
        if (x <= w) v.x = 0ull;
        if (x + 1u <= w) v.y = 0ull;
        R[b] = v;
    }
    const u32 i0 = 16u * s;
    const u32 e0 = i0 ^ (i0 >> 1);
    ulonglong2 acc = make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int b = 3; b < 8; ++b)
        if ((e0 >> b) & 1u) xor2(acc, R[b]);
    *reinterpret_cast<ulonglong2*>(smem + tab_off(g, e0, ch)) = acc;
#pragma unroll
    for (u32 k = 1; k < 16; ++k) {
        const int b = (k & 1u) ? 0 : (k & 2u) ? 1 : (k & 4u) ? 2 : 3;  // ctz(k), folded
        xor2(acc, R[b]);
        const u32 i = i0 + k;
        *reinterpret_cast<ulonglong2*>(smem + tab_off(g, i ^ (i >> 1), ch)) = acc;
    }
}

__device__ __forceinline__ ulonglong2 ldg_info(const ulonglong2* info, u32 pos, bool valid) {
    return valid ? __ldg(info + pos) : make_ulonglong2(0ull, 0ull);
}

__global__ void __launch_bounds__(kTrailThreads, 1) trailing_update_kernel(Params p, u32 w) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StepState st = *p.state;
    const u32 r = st.r, rb = st.rb;
    if (r >= p.m || w + 1 >= p.W) return;
    const u32 tile0 = (w + 1) >> 3;
    const u32 ntiles = (p.Wpad8 >> 3) - tile0;
    const u32 nrows = p.m - r;
    const u64 total = (u64)ntiles * nrows;
    const u64 beg = total * blockIdx.x / gridDim.x;
    const u64 end = total * (blockIdx.x + 1) / gridDim.x;

    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3u, par = rg & 1u;
    const u32 cap_word = w + 1;  // next panel word
    const u32 lane_row = wid * 8u + rg;  // + k * (kTrailThreads/4)

    u64 u = beg;
    while (u < end) {
        const u32 tile = tile0 + (u32)(u / nrows);
        const u32 row0 = (u32)(u % nrows);
        const u32 cnt = (u32)min((u64)(nrows - row0), end - u);
        const bool capture = (cap_word >> 3) == tile;
        const bool cap_lane = capture && ((cap_word & 7u) >> 1) == ch;
        const bool cap_hi = (cap_word & 1u) != 0;
        if (rb > 0) {
            __syncthreads();
            build_tables(p, smem, tile, w, rb);
            __syncthreads();
        }
        u64* tbase = p.mat + (((size_t)tile * p.m) << 3) + 2u * ch;
        const u32 rend = row0 + cnt;
        const u32 nit = (cnt + kRowsPerIter - 1) / kRowsPerIter;

        // software pipeline: rows of iteration i+1 and records of i+2 in flight
        ulonglong2 infC[kUnroll], infN[kUnroll], valC[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 4);
            infC[k] = ldg_info(p.info, r + ri, ri < rend);
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = row0 + kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
            infN[k] = ldg_info(p.info, r + ri, ri < rend);
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 4);
            valC[k] = make_ulonglong2(0ull, 0ull);
            if (ri < rend && (infC[k].x != 0ull || capture))
                valC[k] = *reinterpret_cast<const ulonglong2*>(tbase + ((size_t)infC[k].y << 3));
        }
        for (u32 it = 0; it < nit; ++it) {
            const u32 base = row0 + it * kRowsPerIter;
            ulonglong2 valN[kUnroll], infNN[kUnroll];
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const u32 ri = base + kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
                valN[k] = make_ulonglong2(0ull, 0ull);
                if (ri < rend && (infN[k].x != 0ull || capture))
                    valN[k] = *reinterpret_cast<const ulonglong2*>(tbase + ((size_t)infN[k].y << 3));
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const u32 ri = base + 2 * kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
                infNN[k] = ldg_info(p.info, r + ri, ri < rend);
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const u32 ri = base + lane_row + (u32)k * (kTrailThreads / 4);
                const u64 d = infC[k].x;
                if (d != 0ull) {
#pragma unroll
                    for (u32 gi = 0; gi < kTables; ++gi) {
                        const u32 g = gi ^ par;
                        const u32 e = (u32)(d >> (8u * g)) & 0xffu;
                        xor2(valC[k], *reinterpret_cast<const ulonglong2*>(smem + tab_off(g, e, ch)));
                    }
                    *reinterpret_cast<ulonglong2*>(tbase + ((size_t)infC[k].y << 3)) = valC[k];
                }
                if (cap_lane && ri < rend) p.pb[r + ri] = cap_hi ? valC[k].y : valC[k].x;
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                infC[k] = infN[k];
                infN[k] = infNN[k];
                valC[k] = valN[k];
            }
        }
        u += cnt;
    }
}

// ---------------------------------------------------------------------------
// generators / checksum (row-major public layout)
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 fmix64(u64 x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void fill_ctr_kernel(u64* mat, u32 m, u32 n, u32 Wp, u64 seed) {
    const u32 W = (n + 63u) >> 6;
    const u64 total = (u64)m * Wp;
    const u64 base = seed << 32;
    const u64 lastmask = (n & 63u) ? ((1ull << (n & 63u)) - 1ull) : ~0ull;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u64 i = e / Wp;
        const u32 x = (u32)(e - i * Wp);
        u64 v = 0ull;
        if (x < W) {
            v = fmix64(base + (i * W + x + 1ull) * 0x9e3779b97f4a7c15ull);
            if (x == W - 1u) v &= lastmask;
        }
        mat[e] = v;
    }
}

// Per-row FNV-1a over the W logical words (combined over rows on the host).
__global__ void row_hash_kernel(const u64* mat, u32 m, u32 W, u32 Wp, u64* out) {
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        u64 h = 0xcbf29ce484222325ull;
        const u64* row = mat + (size_t)i * Wp;
        for (u32 x = 0; x < W; ++x) {
            h ^= row[x];
            h *= 0x100000001b3ull;
        }
        out[i] = h;
    }
}

}  // namespace gf2cu
