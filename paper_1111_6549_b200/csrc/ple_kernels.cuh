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
// One 64-column panel (= word column w) per step, three phases:
//   panel_factor   (1 CTA)   pivot search on the panel words of rows >= r:
//                            transposed single-warp elimination on a 128-row
//                            window, CTA-wide scan of the other rows on a
//                            window miss. Replaces partial_ple (ple.hpp:57-130)
//                            and the swap replay (ple.hpp:187-188).
//   apply          (grid)    per row: multipliers c and the combination d of
//                            RAW pivot rows that finishes its tail (d folds the
//                            unit-lower TRSM of ple.hpp:191-193 into the
//                            update); writes the compressed multipliers
//                            (ple.hpp:232-236); stages raw pivot-row tails.
//   trailing       (grid)    8 Gray-code tables x 256 entries per 64-byte
//                            tile in shared memory (make_table,
//                            gray_code.hpp:88-134), then tail ^= sum_g
//                            T_g[byte_g(d)] for every row >= r (ple.hpp:
//                            208-229), 128-bit loads/stores, software-pipelined.
//
// The phases are device functions used by two drivers: one launch per phase
// (ple_*_kernel), and a persistent cooperative kernel (ple_persistent.cuh)
// that overlaps panel s+1 with the trailing update of step s.
#pragma once

#include <cstdint>

namespace gf2cu {

using u64 = unsigned long long;
using u32 = unsigned int;

constexpr int kPanelThreads = 256;     // panel_factor CTA (multi-kernel driver)
constexpr int kWin = 128;              // window rows (two 64-bit halves)
constexpr int kApplyThreads = 256;     // apply CTA (multi-kernel driver)
constexpr int kTrailThreads = 512;     // trailing CTA
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

// Cross-CTA counters of the persistent driver (zeroed before each launch).
struct SyncState {
    u32 panel_done;  // steps whose panel factorization is published
    u32 cap_count;   // worker arrivals after the look-ahead tile (unused by the persistent driver)
    u32 t_count;     // worker arrivals after the whole trailing update
    u32 st_count;    // worker arrivals after staging (unused by the persistent driver)
    u32 error;       // watchdog tripped
    u32 out_count;   // super-step driver: worker arrivals after writing finished rows to `out`
    u32 pad[2];
    u64 stamps[8];   // debug timestamps
};

struct Params {
    u64* mat;        // tile-major, Wpad8/8 tiles x m rows x 8 words
    u32* perm;       // position -> physical row
    u64* pb;         // panel word per position (current step)
    u64* pb2;        // next word (w+1) per position, pre-step (look-ahead), may be null
    ulonglong2* info;  // per position: {d, physical row}
    u64* stage;      // tile-major raw pivot rows: tiles x 64 rows x 8 words
    StepState* state;
    PanelOut* pout;
    u32* swaps;      // LAPACK transpositions (absolute positions)
    u32* qcol;       // absolute pivot columns
    u32* rhist;      // r at the start of each step
    u32* rbhist;     // rb of each step
    volatile u32* host_r;  // mapped pinned mirror of (r + rb), may be null
    SyncState* sync;
    u64* phase_ns;   // per-step phase timestamps (persistent driver), may be null
    u64* worker_ns;  // diagnostics: per step x worker {rest start, rest end}, may be null
    // persistent driver: the pivot rows' swept tails go to ubuf (tile-major,
    // indexed by position, ucap rows) instead of back into the matrix, so the
    // matrix keeps their raw tails for the step's table builds (no staging)
    u64* ubuf;
    u32 ucap;
    u32* ap_claim;   // persistent driver: per step, pre-work chunks claimed / done
    u32* ap_done;
    u32 pw_div;      // rows per 64 pre-work rows (chunk size tuning)
    // sharded driver only (null / 0 otherwise)
    u32* inv;        // global row -> position (kept in step with perm)
    u32* status;     // panel status words (see kPanelStatus*)
    u32 window_only; // 1: abort on a window miss instead of scanning
    u32 nranks, block;  // row distribution: row g lives on rank (g / block) % nranks
    u32 m, n, W, Wpad8;
    // super-step driver, streamed output (may be null): the finished rows
    // (positions below r) in row-major form, stride out_Wp, and a mapped
    // host word holding how many leading positions of `out` are final
    u64* out;
    u32 out_Wp;
    volatile u32* out_host;
    // panel tuning bits (kPanel*)
    u32 pflags;
    // GF2CU_CHECK mode (null otherwise): {first violating step, violations,
    // first bad final row, final violations}, see check_panel_word
    u32* check;
    u32 check_inject;  // test hook (check mode): step + 1 whose first non-pivot row is corrupted
    // streamed input (super-step driver, ple_super.cuh SuperRange): positions
    // >= mv are not on the device yet (0 = all m rows are); partial = 1: a
    // column with no pivot among the visible rows aborts the panel (a row still
    // on its way might hold one)
    u32 mv;
    u32 partial;
};

// Row positions the step may look at (Params::mv).
__device__ __forceinline__ u32 vis_rows(const Params& p) { return p.mv ? p.mv : p.m; }

// Params::pflags: the window warps behind the leader apply its pivots as it
// publishes them (instead of all at the epoch's closing barrier).
constexpr u32 kPanelStream = 1u;
// ... the super-step driver's panel CTA computes the next panel a's window
// itself when the workers are ahead (ple_super.cuh, super_la_gather).
constexpr u32 kPanelSuperLA = 2u;

// Panel status words written when Params::status is set.
constexpr int kStatusMiss = 0;   // 1 = aborted on a window miss (window_only)
constexpr int kStatusRb = 1;     // pivots found
constexpr int kStatusR = 2;      // pivots before this step
constexpr int kStatusOwners = 8; // 2 words per rank: bitmask of pivots t owned

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ u64 low_mask64(int k) {
    return k >= 64 ? ~0ull : ((1ull << k) - 1ull);
}

// Last 64-byte tile of step w's look-ahead sweep (the tiles holding words
// w+1 and w+2).
__device__ __forceinline__ u32 cap_last_tile(u32 w, u32 W) {
    return (w + 2u < W) ? ((w + 2u) >> 3) : ((w + 1u) >> 3);
}
// Step w's look-ahead tiles are all among step w-1's (or untouched, w = 0):
// every row of them is final once step w-1's look-ahead sweep is done.
__device__ __forceinline__ bool early_cap(u32 w, u32 W) {
    return w == 0u || cap_last_tile(w, W) <= cap_last_tile(w - 1u, W);
}
// Persistent driver: rows per pre-work chunk (apply + look-ahead sweep) of a
// step with `nrows` active rows, and the chunk count. Many small chunks when
// few rows are left (latency), up to 1024 rows when many (fewer table builds).
__device__ __forceinline__ u32 pw_rows(u32 nrows, u32 div) {
    return min(1024u, 64u * max(1u, (nrows + div - 1u) / div));
}
__device__ __forceinline__ u32 pw_chunks(u32 nrows, u32 div) {
    const u32 c = pw_rows(nrows, div);
    return (nrows + c - 1u) / c;
}

__device__ __forceinline__ u64* tword(u64* mat, u32 m, u32 row, u32 x) {
    return mat + (((size_t)(x >> 3) * m + row) << 3) + (x & 7u);
}

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// Barrier of the `nthr` threads running panel_factor_body (all of the CTA,
// or all but the persistent drivers' signal warp).
constexpr int kBodyBar = 4;
// Persistent drivers: body threads -> signal warp hand-off after each panel.
constexpr int kSignalBar = 5;

__device__ __forceinline__ u64 shfl64(u64 v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}

__device__ __forceinline__ void st_release_cta(int* a, int v) {
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"((u32)__cvta_generic_to_shared(a)), "r"(v)
                 : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int* a) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];"
                 : "=r"(v)
                 : "r"((u32)__cvta_generic_to_shared(a))
                 : "memory");
    return v;
}

// Loads of data another CTA of the same (persistent) grid may have written:
// L2-coherent, never a stale L1 line.
__device__ __forceinline__ u64 ldcg(const u64* p) { return __ldcg(p); }
__device__ __forceinline__ u32 ldcg(const u32* p) { return __ldcg(p); }
__device__ __forceinline__ ulonglong2 ldcg(const ulonglong2* p) { return __ldcg(p); }

__device__ __forceinline__ u64 globaltimer() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ u32 ld_acquire(const u32* a) {
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_add(u32* a, u32 v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// Watchdog budget of one spin (ns): 4 s unless the host raised it
// (GF2CU_WATCHDOG_S, e.g. for runs under compute-sanitizer).
__device__ unsigned long long g_watchdog_ns = 4000000000ull;

// Spin (one thread) until *a >= target. Watchdog: after g_watchdog_ns sets
// sync->error and returns false instead of hanging the GPU.
__device__ __forceinline__ bool spin_geq(const u32* a, u32 target, u32* err) {
    if (ld_acquire(a) >= target) return true;
    const u64 t0 = globaltimer();
    for (;;) {
        if (ld_acquire(a) >= target) return true;
        if (*(volatile u32*)err) return false;
        if (globaltimer() - t0 > g_watchdog_ns) {
            atomicExch(err, 1u);
            return false;
        }
        __nanosleep(64);
    }
}

// System scope (the row-sharded driver: counters that other GPUs signal
// through NVLink peer memory).
__device__ __forceinline__ u32 ld_acquire_sys(const u32* a) {
    u32 v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_add_sys(u32* a, u32 v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ bool spin_geq_sys(const u32* a, u32 target, u32* err) {
    if (ld_acquire_sys(a) >= target) return true;
    const u64 t0 = globaltimer();
    for (;;) {
        if (ld_acquire_sys(a) >= target) return true;
        if (*(volatile u32*)err) return false;
        if (globaltimer() - t0 > g_watchdog_ns) {
            atomicExch(err, 1u);
            return false;
        }
        __nanosleep(64);
    }
}

// Both counters at once (their loads in flight together).
__device__ __forceinline__ bool spin_geq2(const u32* a, u32 ta, const u32* b, u32 tb, u32* err) {
    u32 va = ld_acquire(a), vb = ld_acquire(b);
    if (va >= ta && vb >= tb) return true;
    const u64 t0 = globaltimer();
    for (;;) {
        va = ld_acquire(a);
        vb = ld_acquire(b);
        if (va >= ta && vb >= tb) return true;
        if (*(volatile u32*)err) return false;
        if (globaltimer() - t0 > g_watchdog_ns) {
            atomicExch(err, 1u);
            return false;
        }
        __nanosleep(64);
    }
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

// Back to row-major in position order. With ubuf (persistent driver), the
// pivot row at position i < rank of step ws = q_i / 64 takes its tiles from
// the step's first swept tile ((ws+1)/8) on from ubuf (if that step swept).
__global__ void untile_kernel(const u64* __restrict__ src, u64* __restrict__ dst,
                              const u32* __restrict__ perm, u32 m, u32 Wp, u32 Wpad8,
                              const u64* __restrict__ ubuf = nullptr, u32 ucap = 0u,
                              const u32* __restrict__ qcol = nullptr, u32 rank = 0u, u32 W = 0u) {
    const u32 per_row = Wpad8 >> 1;
    const u64 total = (u64)m * per_row;
    for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (u64)gridDim.x * blockDim.x) {
        const u32 row = (u32)(e / per_row), x = 2u * (u32)(e - (u64)row * per_row);
        const u32 ph = perm ? perm[row] : row;
        const u64* from = tword(const_cast<u64*>(src), m, ph, x);
        if (ubuf && row < rank) {
            const u32 ws = qcol[row] >> 6;
            if (ws + 1u < W && (x >> 3) >= ((ws + 1u) >> 3))
                from = tword(const_cast<u64*>(ubuf), ucap, row, x);
        }
        *reinterpret_cast<ulonglong2*>(dst + (size_t)row * Wp + x) =
            *reinterpret_cast<const ulonglong2*>(from);
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
        if (p.pb2 && p.W > 1) p.pb2[i] = *tword(p.mat, p.m, i, 1);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.state->r = 0;
        p.state->rb = 0;
    }
}

// ===========================================================================
// Phase 1: panel factorization (one CTA)
// ===========================================================================
struct PanelShared {
    u64 E[64], D[64];
    u64 Eq[64];          // kPanelStream: pivot t's E | its column bit, 0 = not published yet
    u32 q[64];
    u32 sw[64];          // pivot t's position offset (the LAPACK swap)
    u64 wraw[kWin];      // window raw panel words / physical rows, as loaded
    u32 wphys[kWin];
    u64 oraw[64];        // raw word / physical row of pivots taken from outside
    u32 ophys[64];
    // per-pivot exchange among the 4 window warps (double-buffered by parity)
    __align__(16) u32 bal[2][4];
    __align__(16) ulonglong2 cand[2][4];  // {red, acc} of each warp's first candidate row
    u32 corg[2][4];
    ulonglong2 trow[2];     // {red, acc} of the row at position t
    u32 torg[2];
    int cmd;  // 0 = scan, 1 = exit
    int t, j;
    u64 warp_best[32];
    u64 best;  // (first column << 32) | offset
    u64 wor[4];  // per window warp: OR of its live rows' remaining columns (column skip)
    u64 o_red, o_acc, o_raw, o_raw2;
    u32 o_phys;
    u32 r;
    // look-ahead (persistent driver): next step's window words computed here
    u64 nraw[kWin];     // panel words of the next window (word w+1 after step w)
    u64 piv2[64];       // pre-step word w+1 of each pivot row
    u64 opb2[64];       // ... of pivots taken from outside the window
    u64 dacc[kWin];     // per window slot: d (its combination) and origin
    u32 dorg[kWin];
    int cap_ok;
    int ep_t[2], ep_j[2];  // panel epochs: pivots / columns done by the leader warp
    u64 lpb2[kWin];        // look-ahead inputs, fetched right after the capture wait:
    u64 epb[64], epb2[64]; // window rows' pb2 by origin; entering rows' pb / pb2
    u32 eph[64];           // entering rows' physical rows
    // the next window's physical rows and (super-step panel b) pre-super-step
    // words, by slot: no global loads at the next panel's start
    u32 nphys[kWin];
    u64 nwr[kWin], nwr2[kWin];
    // super-step driver
    int super;          // 0, 1 (panel a) or 2 (panel b)
    u64 wraw2[kWin];    // window rows' pre-super-step word w+1 (as loaded)
    u64 ndacc[kWin];    // panel a: panel-a combination of each next-window slot
    u64 oda[64];        // panel b: panel-a combination of pivots taken from outside
    u64 o_da;
    u64 Ea[64], Da[64]; // panel a's outputs, kept for panel b's miss scans
    u32 qa[64];
    u32 rba;
    u32 dbg_lead_cyc, dbg_lead_piv, dbg_cross, dbg_epochs;  // diagnostics (phase_ns slot 4)
    int sig_step, sig_err;  // persistent drivers: body -> signal thread, error seen
    // super-step driver, look-ahead across super-steps (ple_super.cuh,
    // super_la_gather / super_la_compute): the next panel a's window
    u64 la_m2[kWin], la_m3[kWin];  // pre-super-step words w+2, w+3; then the window words
    u64 la_e0[kWin], la_e1[kWin];  // entering rows: raw words w, w+1; window rows: d_a, d_b
    u64 la_R2[128], la_R3[128];    // both panels' pivot rows: pre-super-step words w+2, w+3
    u64 la_C[64];                  // panel b's pivots' panel-a combinations
    u32 la_phys[kWin];
    unsigned char la_ent[kWin];    // 1: the row entered (outside panel b's window)
    int la_go;
    int prog;    // pivots the leader has published (kPanelStream)
    int ep_fin;  // epoch + 1 once the leader closed it (kPanelStream)
};


// Look-ahead mode of panel_factor_body (persistent driver): the step's r is
// tracked by the caller, the window words come from sh.nraw (computed at the
// end of the previous step), and everything that reads the previous step's
// look-ahead capture (scans, the writeback, the next window) first waits until
// all workers have finished it (cap_count >= cap_target).
struct LookAhead {
    u32 r;
    bool have_window;
    const u32* cap_ctr;
    u32 cap_target;
    u32* err;
    // super-step driver (two 64-column panels per sweep): 1 = panel a, 2 = panel b
    int super_mode = 0;
    u64* piv2_out = nullptr;  // panel a: its pivot rows' pre-super-step word w+1
    u64* C_out = nullptr;     // panel b: panel-a combination of each of its pivot rows
    bool sys = false;         // cap_ctr is signalled by other GPUs (system-scope acquire)
    PanelOut* pout = nullptr; // where E / D / qb go instead of Params::pout (per-step history)
};

// All `nthr` threads: scan positions r + [nwin, nrem) reducing each raw panel
// word by the t pivots found so far; sh.best = the smallest (first set column
// >= j, offset), with the winner's reduced state in sh.o_*.
// The rows are scanned in position order in chunks that double in size, and
// the scan stops after the first chunk that holds a candidate for column j
// itself: the first row with a 1 in column j (ple.hpp:88-93) is then in that
// chunk, and no later row can beat the key (j, offset). On sparse inputs
// (BASELINE config 3, p = 1/256: the pivot is ~256 rows down) a miss reads a
// couple of thousand rows instead of all of them. Only a column without any
// candidate is scanned to the end; the key then names the next column that has
// one (the caller's out_next).
constexpr int kScanRows = 4;  // rows per thread in flight in panel_scan

// OR of (1 << q[s]) for s < n (n <= 64), computed by one warp (all lanes).
__device__ __forceinline__ u64 pivot_mask(const u32* q, u32 n) {
    const u32 lane = threadIdx.x & 31u;
    const u64 x = (lane < n ? 1ull << q[lane] : 0ull) | (lane + 32u < n ? 1ull << q[lane + 32u] : 0ull);
    const u32 lo = __reduce_or_sync(0xffffffffu, (u32)x), hi = __reduce_or_sync(0xffffffffu, (u32)(x >> 32));
    return ((u64)hi << 32) | lo;
}

// v reduced by the pivots whose columns are the bits of pm (pivot s = the s-th
// set bit: the columns increase with s), acc ^= their D. Walks the row's set
// pivot bits instead of all pivots: E[s] only holds columns right of q[s], so
// taking the bits in increasing order is the step-by-step elimination; a
// sparse row costs a couple of iterations instead of one step per pivot.
__device__ __forceinline__ void reduce_sparse(u64& v, u64& acc, u64 pm, const u64* E, const u64* D) {
    u64 rem = pm;
    for (;;) {
        const u64 x = v & rem;
        if (!x) break;
        const int c = __ffsll((long long)x) - 1;
        const int s = __popcll(pm & low_mask64(c));
        v ^= E[s];
        acc ^= D[s];
        rem &= ~low_mask64(c + 1);
    }
}

__device__ __forceinline__ void panel_scan(const Params& p, PanelShared& sh, u32 r, u32 nwin, u32 nrem, int nthr) {
    const int t = sh.t, j = sh.j;
    const bool two = sh.super == 2;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    u64 best = ~0ull, b_red = 0, b_acc = 0, b_da = 0;
    const u64 pm = pivot_mask(sh.q, (u32)t);
    const u64 pma = two ? pivot_mask(sh.qa, sh.rba) : 0ull;
    u32 lo = nwin, csize = (u32)kScanRows * (u32)nthr;
    for (;;) {
        const u32 hi = nrem - lo > csize ? lo + csize : nrem;
        // kScanRows rows per thread at a time: their loads are issued together
        for (u32 base = lo; base < hi; base += kScanRows * (u32)nthr) {
            u64 v[kScanRows], v2[kScanRows];
            u32 off[kScanRows];
#pragma unroll
            for (int k = 0; k < kScanRows; ++k) {
                off[k] = base + (u32)k * (u32)nthr + threadIdx.x;
                const bool val = off[k] < hi;
                v[k] = val ? ldcg(p.pb + r + off[k]) : 0ull;
                v2[k] = (val && two) ? ldcg(p.pb2 + r + off[k]) : 0ull;
            }
#pragma unroll
            for (int k = 0; k < kScanRows; ++k) {
                u64 x = v[k], a = 0ull, da = 0ull;
                if (two) {
                    // panel b of a super-step: word w+1 after panel a, from the row's
                    // pre-super-step words (pb = word w, pb2 = word w+1)
                    reduce_sparse(x, da, pma, sh.Ea, sh.Da);
                    x = v2[k];
                    for (u64 dr = da; dr; dr &= dr - 1ull) x ^= sh.piv2[__ffsll((long long)dr) - 1];
                }
                reduce_sparse(x, a, pm, sh.E, sh.D);
                const u64 mk = x & ~low_mask64(j);
                if (off[k] < hi && mk) {
                    const u64 key = ((u64)(__ffsll((long long)mk) - 1) << 32) | off[k];
                    if (key < best) {
                        best = key;
                        b_red = x;
                        b_acc = a;
                        b_da = da;
                    }
                }
            }
        }
        u64 wb = best;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u64 other = __shfl_xor_sync(0xffffffffu, wb, o);
            wb = other < wb ? other : wb;
        }
        if (lane == 0) sh.warp_best[wid] = wb;
        named_bar(2, nthr);
        if (threadIdx.x == 0) {
            u64 b = ~0ull;
            for (int k = 0; k < nthr / 32; ++k) b = sh.warp_best[k] < b ? sh.warp_best[k] : b;
            sh.best = b;
        }
        named_bar(2, nthr);
        lo = hi;
        if (lo >= nrem || (int)(sh.best >> 32) == j) break;
        csize *= 2u;
    }
    if (best != ~0ull && best == sh.best) {
        const u32 off = (u32)(best & 0xffffffffu);
        sh.o_red = b_red;
        sh.o_acc = b_acc;
        sh.o_raw = ldcg(p.pb + r + off);
        sh.o_raw2 = p.pb2 ? ldcg(p.pb2 + r + off) : 0ull;
        sh.o_phys = ldcg(p.perm + r + off);
        sh.o_da = b_da;
    }
    named_bar(2, nthr);
}

// panel_scan as a real call. The single-panel persistent kernel is faster with
// the scan out of line (4096^2 0.887 -> 0.854 ms: the panel chain's code stays
// compact); the two-panel kernels are not (the call's register convention costs
// their sweep 284 bytes of spills, 32768^2 13.1 -> 16.8 ms), so they inline it.
__device__ __noinline__ void panel_scan_call(const Params& p, PanelShared& sh, u32 r, u32 nwin, u32 nrem,
                                             int nthr) {
    panel_scan(p, sh, r, nwin, nrem, nthr);
}

// The panel step w. Called by every thread of ONE CTA of `nthr` >= 256
// threads. Warps 0-3 hold the 128-row window, one row per thread (`red` =
// the row's panel word reduced by the pivots so far, `acc` = its combination
// of raw pivot rows); per pivot they exchange one ballot and one candidate
// row per warp through shared memory behind a single 128-thread named
// barrier. The other warps serve window-miss scans. Returns rb in all threads.
// Wait (one thread, result broadcast through sh.cap_ok) until the workers
// finished the previous step's look-ahead capture.
__device__ __forceinline__ void la_wait_cap(const LookAhead* la, PanelShared& sh, int bar_id,
                                            int bar_cnt) {
    if (!la || sh.cap_ok) return;
    if (threadIdx.x == 0)
        sh.cap_ok = (la->sys ? spin_geq_sys(la->cap_ctr, la->cap_target, la->err)
                             : spin_geq(la->cap_ctr, la->cap_target, la->err)) ? 1 : -1;
    named_bar(bar_id, bar_cnt);
}

template <bool kCallScan = false>
__device__ u32 panel_factor_body(const Params& p, u32 w, PanelShared& sh, int nthr,
                                 const LookAhead* la = nullptr) {
    if (threadIdx.x == 0) {
        if (la) {
            sh.r = la->r;
        } else {
            const volatile StepState* vs = p.state;
            sh.r = vs->r + vs->rb;
        }
        sh.t = 0;
        sh.cap_ok = la ? (la->cap_target == 0 ? 1 : 0) : 1;
        sh.super = la ? la->super_mode : 0;
    }
    named_bar(kBodyBar, nthr);
    if (la && sh.super != 2 && !sh.cap_ok && !la->have_window) {
        // a window read from the capture (pb, perm) waits for it: panel a of
        // a super-step (unless the look-ahead across super-steps computed its
        // window), and step 0 of the row-sharded drivers, whose init (perm,
        // pb[0]) runs inside the same launch. (Round 2: this wait was missing
        // for the single-panel row-sharded driver's step 0 -- the cause of
        // its rare mismatches, 1 in ~13,000 calls, e.g. rank 0 when the
        // window read the previous call's words.)
        if (threadIdx.x == 0)
            sh.cap_ok = (la->sys ? spin_geq_sys(la->cap_ctr, la->cap_target, la->err)
                                 : spin_geq(la->cap_ctr, la->cap_target, la->err)) ? 1 : -1;
        named_bar(kBodyBar, nthr);
    }
    const u32 r = sh.r;
    const u32 M = vis_rows(p);
    PanelOut* const pout = (la && la->pout) ? la->pout : p.pout;
    if (threadIdx.x == 0) {
        p.state->r = r;
        p.state->rb = 0;
        p.rhist[w] = r;
        p.rbhist[w] = 0;
    }
    if (r >= M) {
        if (threadIdx.x == 0 && p.host_r) {
            *p.host_r = r;
            __threadfence_system();
        }
        if (threadIdx.x == 0 && p.status) {
            p.status[kStatusMiss] = 0u;
            p.status[kStatusRb] = 0u;
            p.status[kStatusR] = r;
        }
        named_bar(kBodyBar, nthr);
        return 0;
    }
    const u32 nrem = M - r;
    const u32 nwin = nrem < (u32)kWin ? nrem : (u32)kWin;
    const int jmax = (int)min(64u, p.n - 64u * w);

    if (threadIdx.x >= kWin) {
        for (;;) {
            named_bar(1, nthr);
            if (sh.cmd != 0) break;
            if constexpr (kCallScan)
                panel_scan_call(p, sh, r, nwin, nrem, nthr);
            else
                panel_scan(p, sh, r, nwin, nrem, nthr);
        }
    } else {
        // ---- window warps: thread `me` holds window row `me` ----
        const u32 me = threadIdx.x, lane = me & 31u, wid = me >> 5;
        const bool inwin = me < nwin;
        u64 red = 0ull, acc = 0ull;
        u32 org = me;  // window offset of the row this slot holds
        if (inwin) {
            if (sh.super == 1 && la->have_window) {
                // computed by the previous super-step's look-ahead
                sh.wraw[me] = sh.la_m2[me];
                sh.wraw2[me] = sh.la_m3[me];
                red = sh.la_m2[me];
                sh.wphys[me] = sh.la_phys[me];
            } else if (sh.super == 2) {
                // panel a's look-ahead: word w+1 after panel a, and the rows'
                // pre-super-step words and physical rows
                sh.wraw[me] = sh.nwr[me];
                sh.wraw2[me] = sh.nwr2[me];
                red = sh.nraw[me];
                sh.wphys[me] = sh.nphys[me];
            } else if (sh.super) {
                // keep the rows' pre-super-step words (pb, pb2): they follow
                // the rows through the writeback for the workers' apply
                sh.wraw[me] = ldcg(p.pb + r + me);
                sh.wraw2[me] = ldcg(p.pb2 + r + me);
                red = sh.wraw[me];
                sh.wphys[me] = ldcg(p.perm + r + me);
            } else if (la && la->have_window) {
                red = sh.nraw[me];
                sh.wraw[me] = red;
                sh.wphys[me] = sh.nphys[me];
            } else {
                red = ldcg(p.pb + r + me);
                sh.wraw[me] = red;
                sh.wphys[me] = ldcg(p.perm + r + me);
            }
        }
        if (me == 0) {
            sh.dbg_lead_cyc = sh.dbg_lead_piv = sh.dbg_cross = sh.dbg_epochs = 0u;
            sh.prog = 0;
            sh.ep_fin = 0;
        }
        if (me < 64u) {  // the leader's stream records: none published yet
            sh.Eq[me] = 0ull;
            sh.D[me] = 0ull;
        }
        const bool stream = (p.pflags & kPanelStream) != 0u;
        named_bar(3, kWin);
        if (p.phase_ns && me == 0) p.phase_ns[(size_t)w * 8 + 6] = globaltimer();
        int t = 0;
        int out_next = nwin < nrem ? 0 : 64;
        bool aborted = false;
        // One cross-warp step for column j (all 4 window warps, up to date
        // with every pivot < t): per-warp ballots and first candidates
        // exchanged through shared memory, the first candidate over the
        // window taken (a window miss scans the other rows). Returns 1 if a
        // pivot was found, 0 if column j has none, 2 if aborted.
        auto cross_step = [&](const int j) -> int {
            const int par = j & 1;
            // candidates: live rows (position >= t) holding column j
            const bool b = inwin & (me >= (u32)t) & (((red >> j) & 1ull) != 0ull);
            const u32 bal = __ballot_sync(0xffffffffu, b);
            if (lane == 0) sh.bal[par][wid] = bal;
            if (b & (lane == (u32)(__ffs(bal) - 1))) {
                sh.cand[par][wid] = make_ulonglong2(red, acc);
                sh.corg[par][wid] = org;
            }
            if (me == (u32)t) {
                sh.trow[par] = make_ulonglong2(red, acc);
                sh.torg[par] = org;
            }
            named_bar(3, kWin);
            // everything the step needs is loaded at once (independent LDS)
            const uint4 bw = *reinterpret_cast<const uint4*>(sh.bal[par]);
            const ulonglong2 c0 = sh.cand[par][0], c1 = sh.cand[par][1];
            const ulonglong2 c2 = sh.cand[par][2], c3 = sh.cand[par][3];
            const uint4 co = *reinterpret_cast<const uint4*>(sh.corg[par]);
            const ulonglong2 tr = sh.trow[par];
            const u32 tro = sh.torg[par];
            const int pw = bw.x ? 0 : bw.y ? 1 : bw.z ? 2 : bw.w ? 3 : -1;
            u64 pred, pacc;
            u32 P, porg;
            if (pw >= 0) {
                const u32 bw_sel = pw == 0 ? bw.x : pw == 1 ? bw.y : pw == 2 ? bw.z : bw.w;
                P = 32u * (u32)pw + (u32)(__ffs(bw_sel) - 1);
                pred = pw == 0 ? c0.x : pw == 1 ? c1.x : pw == 2 ? c2.x : c3.x;
                pacc = pw == 0 ? c0.y : pw == 1 ? c1.y : pw == 2 ? c2.y : c3.y;
                porg = pw == 0 ? co.x : pw == 1 ? co.y : pw == 2 ? co.z : co.w;
                // row swap t <-> P: the old row t moves into slot P
                const bool mv = (me == P) & (P != (u32)t);
                red = mv ? tr.x : red;
                acc = mv ? tr.y : acc;
                org = mv ? tro : org;
            } else {
                // ---- window miss: the remaining rows decide ----
                if (j < out_next && !p.partial) return 0;  // no row outside has this column
                if (p.window_only || (p.partial && j < out_next)) {
                    // sharded driver: the host gathers the whole panel column
                    // and runs the step again (nothing global was written)
                    aborted = true;
                    return 2;
                }
                la_wait_cap(la, sh, 3, kWin);  // pb of the outside rows is the capture
                if (la && sh.cap_ok < 0) {
                    aborted = true;
                    return 2;
                }
                if (me == 0) {
                    sh.cmd = 0;
                    sh.t = t;
                    sh.j = j;
                }
                named_bar(1, nthr);
                if constexpr (kCallScan)
                    panel_scan_call(p, sh, r, nwin, nrem, nthr);
                else
                    panel_scan(p, sh, r, nwin, nrem, nthr);
                const u64 best = sh.best;
                out_next = best == ~0ull ? 64 : (int)(best >> 32);
                if (out_next != j) {
                    // column j has no pivot among the rows on the device
                    if (p.partial) {
                        aborted = true;
                        return 2;
                    }
                    return 0;
                }
                // pivot from outside the window: it takes position t; the
                // window row t moves to the pivot's old position P
                P = (u32)(best & 0xffffffffu);
                pred = sh.o_red;
                pacc = sh.o_acc;
                porg = 0x80000000u | (u32)t;
                if (me == (u32)t) {
                    if (sh.super) {
                        sh.opb2[t] = sh.o_raw2;
                        p.pb2[r + P] = sh.wraw2[org];
                        sh.oda[t] = sh.o_da;
                    } else if (p.pb2 && w + 1 < p.W) {
                        // next-word capture follows the displaced window row
                        sh.opb2[t] = ldcg(p.pb2 + r + P);
                        p.pb2[r + P] = ldcg(p.pb2 + r + org);
                    }
                    p.pb[r + P] = sh.wraw[org];
                    p.perm[r + P] = sh.wphys[org];
                    if (p.inv) p.inv[sh.wphys[org]] = r + P;
                    sh.oraw[t] = sh.o_raw;
                    sh.ophys[t] = sh.o_phys;
                }
            }
            if (me == (u32)t) org = porg;  // the pivot's slot records its row
            const u64 Et = pred & ~low_mask64(j + 1);
            const u64 tm = 1ull << t;
            const u64 Dt = pacc ^ tm;
            const u64 msk = 0ull - (u64)(inwin & (me > (u32)t) & (((red >> j) & 1ull) != 0ull));
            red ^= Et & msk;
            acc ^= Dt & msk;
            if (me == 0) {
                sh.E[t] = Et;
                sh.D[t] = Dt;
                sh.q[t] = (u32)j;
                sh.sw[t] = P;
            }
            ++t;
            return 1;
                };
        // Epochs: the leader warp (the one holding slot t; lower warps hold
        // no live row) takes pivots alone -- ballot, shuffles, no barrier --
        // as long as it has a candidate for the next column and t stays in
        // it. Then all window warps meet, the others apply the epoch's
        // pivots to their rows in order (they hold no pivot and no swapped
        // row), and the column the leader had no candidate for goes through
        // cross_step. Same pivots, swaps and outputs as column-by-column
        // cross steps; far fewer barriers on dense panels.
        int j = 0, epoch = 0;
        while (j < jmax && (u32)t < nrem) {
            const int L = t >> 5;
            if ((int)wid == L) {
                const long long dbg_c0 = clock64();
                const int dbg_t0 = t;
                const u32 base = 32u * (u32)L;
                u64 jbit = 1ull << j;          // column j
                u64 hi = ~(jbit | (jbit - 1)); // columns > j
                u64 tbit = 1ull << t;
                // pivots this leader can take at most: columns, rows, its slots
                const int lim = min(jmax - j, min((int)nrem - t, 32 * (L + 1) - t));
                const int tend = t + lim;
                u64* sE = sh.E;
                u64* sD = sh.D;
                // Short dependent chain per pivot: row t's copy (for the lane
                // that takes it in the swap) is gathered before the ballot; the
                // pivot row comes from one shuffle of the ballot's first lane;
                // the rows to eliminate are the candidates except P (row t has
                // no bit j unless it is P); they XOR the whole pivot row (their
                // bits <= j are never read again); every lane writes the same
                // record (no divergent branch).
                while (t < tend) {
                    const u32 tl = (u32)t & 31u;
                    const u64 rt = shfl64(red, (int)tl), at = shfl64(acc, (int)tl);
                    const u32 ot = __shfl_sync(0xffffffffu, org, (int)tl);
                    const bool cand = inwin & (lane >= tl) & ((red & jbit) != 0ull);
                    const u32 bal = __ballot_sync(0xffffffffu, cand);
                    if (bal == 0u) break;
                    const u32 pl = (u32)(__ffs(bal) - 1);
                    const u64 pr = shfl64(red, (int)pl), pa = shfl64(acc, (int)pl);
                    const u32 po = __shfl_sync(0xffffffffu, org, (int)pl);
                    const bool isP = lane == pl;
                    const bool el = cand & !isP;
                    const u64 Dt = pa ^ tbit;
                    red = isP ? rt : (el ? red ^ pr : red);
                    acc = isP ? at : (el ? acc ^ Dt : acc);
                    org = isP ? ot : (lane == tl ? po : org);
                    const u64 Et = pr & hi;
                    sE[t] = Et;
                    sh.q[t] = (u32)j;
                    sh.sw[t] = base + pl;
                    // Published to the followers without a fence: each of the
                    // two words validates itself (D_t holds bit t, E_t | column
                    // bit is nonzero, both were zeroed at the panel's start),
                    // and aligned 64-bit shared-memory accesses are single-copy
                    // atomic. The fence this replaces cost ~30 cycles per pivot
                    // on the leader's chain.
                    *(volatile u64*)&sD[t] = Dt;
                    if (stream) *(volatile u64*)&sh.Eq[t] = Et | jbit;
                    ++t;
                    ++j;
                    jbit <<= 1;
                    hi <<= 1;
                    tbit <<= 1;
                }
                if (lane == 0) {
                    sh.ep_t[epoch & 1] = t;
                    sh.ep_j[epoch & 1] = j;
                    sh.dbg_lead_cyc += (u32)(clock64() - dbg_c0);
                    sh.dbg_lead_piv += (u32)(t - dbg_t0);
                    sh.dbg_epochs += 1u;
                    if (stream) st_release_cta(&sh.ep_fin, epoch + 1);
                }
            } else if (stream && (int)wid > L) {
                // follow the leader: apply each pivot as it is published
                int s2 = t;
                for (;;) {
                    // (read before the records: once the epoch is closed, the
                    // pass below sees all of them)
                    const int fin = ld_acquire_cta(&sh.ep_fin);
                    for (; s2 < 64; ++s2) {
                        const u64 eq = *(volatile u64*)&sh.Eq[s2];
                        const u64 dd = *(volatile u64*)&sh.D[s2];
                        if (eq == 0ull || dd == 0ull) break;
                        const u64 cb = eq & (0ull - eq);  // the pivot's column
                        const u64 msk = (red & cb) ? ~0ull : 0ull;
                        red ^= (eq ^ cb) & msk;
                        acc ^= dd & msk;
                    }
                    if (fin == epoch + 1) break;
                }
                t = s2;  // == the epoch's closing t
            }
            named_bar(3, kWin);
            const int t1 = sh.ep_t[epoch & 1], j1 = sh.ep_j[epoch & 1];
            ++epoch;
            if ((int)wid > L) {
                for (int s2 = t; s2 < t1; ++s2) {
                    const u64 msk = 0ull - ((red >> sh.q[s2]) & 1ull);
                    red ^= sh.E[s2] & msk;
                    acc ^= sh.D[s2] & msk;
                }
            }
            t = t1;
            j = j1;
            if (j >= jmax || (u32)t >= nrem) break;
            if ((t >> 5) != L) continue;  // the leader's rows are used up: next leader
            const int st = cross_step(j);
            if (me == 0) sh.dbg_cross += 1u;
            if (st == 2) break;
            if (st == 0) {
                // Column j has no pivot. Skip to the next column that can have
                // one: the first column > j some live window row holds, or
                // out_next, the first column with a candidate among the other
                // rows (still exact: no outside row holds a column below it, so
                // window pivots left of it do not change them). An exhausted
                // trailing matrix (rank-deficient inputs) ends the panel here
                // instead of stepping through every column.
                const u64 x = (inwin & (me >= (u32)t)) ? (red & ~low_mask64(j + 1)) : 0ull;
                const u32 xl = __reduce_or_sync(0xffffffffu, (u32)x);
                const u32 xh = __reduce_or_sync(0xffffffffu, (u32)(x >> 32));
                if (lane == 0) sh.wor[wid] = ((u64)xh << 32) | xl;
                named_bar(3, kWin);
                const u64 any = sh.wor[0] | sh.wor[1] | sh.wor[2] | sh.wor[3];
                const int nw = any ? __ffsll((long long)any) - 1 : 64;
                j = min(nw, out_next);
            } else {
                ++j;
            }
        }
        if (p.phase_ns && me == 0) p.phase_ns[(size_t)w * 8 + 7] = globaltimer();
        if (p.phase_ns) named_bar(3, kWin);
        if (p.phase_ns && me == 0)
            p.phase_ns[(size_t)w * 8 + 4] = ((u64)sh.dbg_lead_cyc << 32) | (sh.dbg_lead_piv << 16) |
                                            (sh.dbg_cross << 8) | sh.dbg_epochs;
        sh.dacc[me] = acc;
        sh.dorg[me] = org;
        // the writeback below may only land after the workers are done with
        // the previous step (apply, staging and its look-ahead capture)
        named_bar(3, kWin);
        if (!aborted) la_wait_cap(la, sh, 3, kWin);
        if (la && sh.cap_ok < 0) aborted = true;
        // issue the next window's global inputs now, so that their latency
        // overlaps the writeback: the window rows' pre-step word w+1 (by
        // origin) and the words w, w+1 of the rows that may enter it
        u64 f_pb2 = 0ull, f_epb = 0ull, f_epb2 = 0ull;
        u32 f_eph = 0u;
        if (la && !aborted && sh.super != 2 && w + 1 < p.W) {
            if (!sh.super && inwin) f_pb2 = ldcg(p.pb2 + r + me);
            const u32 qe = r + nwin + me;
            if (me < 64u && qe < M) {
                f_epb = ldcg(p.pb + qe);
                f_epb2 = ldcg(p.pb2 + qe);
                f_eph = ldcg(p.perm + qe);
            }
        }
        // the permuted window: raw panel word and physical row per position
        u64 rw = 0ull;
        u32 ph = 0u;
        if (inwin) {
            const bool out = (org & 0x80000000u) != 0u;
            rw = out ? sh.oraw[org & 63u] : sh.wraw[org & 127u];
            ph = out ? sh.ophys[org & 63u] : sh.wphys[org & 127u];
        }
        if (me == 0) {
            sh.cmd = 1;
            sh.t = aborted ? -1 : t;
        }
        named_bar(1, nthr);  // release the helpers
        u64 rw2 = 0ull;
        if (sh.super && inwin) {
            const bool out = (org & 0x80000000u) != 0u;
            rw2 = out ? sh.opb2[org & 63u] : sh.wraw2[org & 127u];
        }
        if (inwin && !aborted) {
            p.pb[r + me] = rw;
            if (sh.super) p.pb2[r + me] = rw2;
            p.perm[r + me] = ph;
            if (p.inv) p.inv[ph] = r + me;
        }
        sh.lpb2[me] = f_pb2;
        if (me < 64u) {
            sh.epb[me] = f_epb;
            sh.epb2[me] = f_epb2;
            sh.eph[me] = f_eph;
        }
    }
    named_bar(kBodyBar, nthr);
    if (sh.t < 0) {
        // aborted: state stays {r, 0}, so running the step again is exact
        if (threadIdx.x == 0 && p.status) {
            p.status[kStatusMiss] = 1u;
            p.status[kStatusRb] = 0u;
            p.status[kStatusR] = r;
        }
        named_bar(kBodyBar, nthr);
        return 0;
    }
    const u32 t = (u32)sh.t;
    if (p.status) {
        // sharded driver: which rank owns each pivot row
        for (u32 k = threadIdx.x; k < 2u * p.nranks; k += nthr) p.status[kStatusOwners + k] = 0u;
        named_bar(kBodyBar, nthr);
        for (u32 k = threadIdx.x; k < t; k += nthr) {
            const u32 g = p.perm[r + k];
            const u32 o = (g / p.block) % p.nranks;
            atomicOr(&p.status[kStatusOwners + 2 * o + (k >> 5)], 1u << (k & 31));
        }
        if (threadIdx.x == 0) {
            p.status[kStatusMiss] = 0u;
            p.status[kStatusRb] = t;
            p.status[kStatusR] = r;
        }
    }
    for (u32 k = threadIdx.x; k < t; k += nthr) {
        pout->E[k] = sh.E[k];
        pout->D[k] = sh.D[k];
        pout->qb[k] = sh.q[k];
        p.swaps[r + k] = r + sh.sw[k];
        p.qcol[r + k] = 64u * w + sh.q[k];
    }
    if (threadIdx.x == 0) {
        p.state->rb = t;
        p.rbhist[w] = t;
        if (p.host_r) {
            *p.host_r = r + t;
            __threadfence_system();
        }
    }
    named_bar(kBodyBar, nthr);
    if (sh.super == 2) {
        // panel b: panel-a combination of each of its pivot rows
        for (u32 k = threadIdx.x; k < t; k += nthr) {
            const u32 o = sh.dorg[k];
            la->C_out[k] = (o & 0x80000000u) ? sh.oda[o & 63u] : sh.ndacc[o & 127u];
        }
    }
    if (sh.super == 1) {
        // panel a: keep its outputs for panel b's miss scans
        for (u32 k = threadIdx.x; k < t; k += nthr) {
            sh.Ea[k] = sh.E[k];
            sh.Da[k] = sh.D[k];
            sh.qa[k] = sh.q[k];
        }
        if (threadIdx.x == 0) sh.rba = t;
    }
    if (la && sh.super != 2 && w + 1 < p.W && (r + t < M || sh.super == 1)) {
        // ---- next window: word w+1 after step w, for positions
        //      [r + t, r + t + 128), from the pre-step capture pb2 (the
        //      super-step driver needs the pivot rows' word w+1 even when no
        //      row is left for a next window) ----
        const u32 r1 = r + t;
        const u32 nwin1 = r1 < M ? min((u32)kWin, M - r1) : 0u;
        // pre-step word w+1 of each pivot row
        // (super-step driver: pb2 was permuted by the writeback; the window
        // rows' pre-super-step words are in shared memory)
        for (u32 k = threadIdx.x; k < t; k += nthr) {
            const u32 o = sh.dorg[k];
            sh.piv2[k] = (o & 0x80000000u) ? sh.opb2[o & 63u]
                         : sh.super       ? sh.wraw2[o & 127u]
                                          : sh.lpb2[o & 127u];
            if (sh.super) la->piv2_out[k] = sh.piv2[k];
        }
        named_bar(kBodyBar, nthr);
        for (u32 k = threadIdx.x; k < nwin1; k += nthr) {
            const u32 q = r1 + k;  // position
            u64 d, pre;
            if (q - r < nwin) {
                const u32 o = sh.dorg[q - r] & 127u;  // (a non-pivot slot: an in-window origin)
                d = sh.dacc[q - r];
                pre = sh.super ? sh.wraw2[o] : sh.lpb2[o];
                sh.nphys[k] = sh.wphys[o];
                sh.nwr[k] = sh.wraw[o];
                sh.nwr2[k] = sh.wraw2[o];
            } else {
                sh.nphys[k] = sh.eph[q - r - nwin];
                sh.nwr[k] = sh.epb[q - r - nwin];
                sh.nwr2[k] = sh.epb2[q - r - nwin];
                // a row entering the window: its combination for step w
                u64 v = sh.epb[q - r - nwin];
                d = 0ull;
                for (u32 s2 = 0; s2 < t; ++s2) {
                    const u64 msk = 0ull - ((v >> sh.q[s2]) & 1ull);
                    v ^= sh.E[s2] & msk;
                    d ^= sh.D[s2] & msk;
                }
                pre = sh.epb2[q - r - nwin];
            }
            sh.ndacc[k] = d;
            if (sh.super) {  // (the XOR in (b) below)
                sh.nraw[k] = pre;
                continue;
            }
            u64 x = pre;
#pragma unroll 8
            for (u32 s2 = 0; s2 < 64; ++s2) {
                if (s2 >= t) break;
                x ^= sh.piv2[s2] & (0ull - ((d >> s2) & 1ull));
            }
            sh.nraw[k] = x;
        }
        named_bar(kBodyBar, nthr);
        if (sh.super) {
            // (b) super-step driver: word w+1 after panel a = pre ^ sum_s d_s
            // piv2[s] with four lanes per slot, 16 pivots each, folded with two
            // shuffles (every lane of a warp runs the same iterations: nthr and
            // 4 * kWin are multiples of 32). Measured: 65536^2 67.49 -> 67.22
            // ms; the single-panel driver keeps the one-lane loop above (its
            // panel chain is shorter without the extra barrier: 4096^2 0.863
            // vs 0.903 ms).
            for (u32 g = threadIdx.x; g < 4u * kWin; g += nthr) {
                const u32 k = g >> 2, part = g & 3u;
                const u64 d = k < nwin1 ? sh.ndacc[k] : 0ull;
                u64 x = 0ull;
#pragma unroll
                for (u32 i = 0; i < 16u; ++i) {
                    const u32 s2 = 16u * part + i;  // (bits s2 >= t of d are zero)
                    x ^= sh.piv2[s2] & (0ull - ((d >> s2) & 1ull));
                }
                x ^= __shfl_xor_sync(0xffffffffu, x, 1);
                x ^= __shfl_xor_sync(0xffffffffu, x, 2);
                if (part == 0u && k < nwin1) sh.nraw[k] ^= x;
            }
            named_bar(kBodyBar, nthr);
        }
    }
    return t;
}

__global__ void __launch_bounds__(kPanelThreads, 1) panel_factor_kernel(Params p, u32 w) {
    __shared__ PanelShared sh;
    panel_factor_body<true>(p, w, sh, kPanelThreads);
}

// ===========================================================================
// Phase 2: apply (rows) and staging (pivot rows)
// ===========================================================================
struct ApplyShared {
    u64 E[64], D[64];
    u32 q[64];
};

__device__ __forceinline__ void apply_load(const Params& p, ApplyShared& s, u32 rb) {
    for (u32 k = threadIdx.x; k < 64; k += blockDim.x) {
        const bool v = k < rb;
        s.E[k] = v ? ldcg(&p.pout->E[k]) : 0ull;
        s.D[k] = v ? ldcg(&p.pout->D[k]) : 0ull;
        s.q[k] = v ? ldcg(&p.pout->qb[k]) : 0u;
    }
}

// GF2CU_CHECK (Params::check != null): invariant (iv) of SURVEY.md 8(c),
// "once columns [0, c] are finished with r pivots, rows >= r are zero in
// columns [r, c]", on a row's panel word v after its forward elimination
// against the panel's first tl pivots (columns q[0..tl)): a non-pivot row
// (tl = rb) may hold bits only at pivot columns (its multipliers) -- every
// other column of the panel was finished with no pivot left for it -- and a
// pivot row (index tl) only at pivot columns left of its own pivot column,
// plus its pivot bit. A violation means the row's word was not the current
// one (a stale capture, a race): the first (lowest) step goes to check[0],
// the count to check[1].
__device__ __noinline__ void check_panel_word(u32* chk, u32 step, u64 v, u32 tl, bool pivot,
                                              const u32* q) {
    u64 pm = 0ull;
    for (u32 k = 0; k < tl; ++k) pm |= 1ull << q[k];
    u64 bad = v & ~pm;
    if (pivot) bad = (bad & low_mask64((int)q[tl])) | (((v >> q[tl]) & 1ull) ^ 1ull);
    if (bad) {
        atomicMin(chk, step);
        atomicAdd(chk + 1, 1u);
    }
}

// Invariants (i) and (ii) of SURVEY.md 8(c) on the finished row-major L\E:
// bit (i, i) = 1 for every i < rank; rows >= rank are zero in every column
// >= rank. First bad row to check[2] (atomicMin), count to check[3].
__global__ void check_final_kernel(const u64* a, u32 m, u32 n, u32 Wp, u32 rank, u32* chk) {
    const u32 W = (n + 63u) >> 6;
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const u64* row = a + (size_t)i * Wp;
        bool bad = false;
        if (i < rank) {
            bad = ((row[i >> 6] >> (i & 63u)) & 1ull) == 0ull;
        } else {
            const u32 w0 = rank >> 6;
            for (u32 x = w0; x < W && !bad; ++x) {
                u64 v = row[x];
                if (x == w0) v &= ~low_mask64((int)(rank & 63u));
                bad = v != 0ull;
            }
        }
        if (bad) {
            atomicMin(chk + 2, i);
            atomicAdd(chk + 3, 1u);
        }
    }
}

// Positions [lo, hi) (all >= r): multipliers, combination, compressed write.
// (Check: check mode's invariant test, compiled out of the normal path.)
template <bool Check>
__device__ __forceinline__ void apply_rows_t(const Params& p, const ApplyShared& s, u32 w, u32 r,
                                             u32 rb, u32 lo, u32 hi, u32 tid, u32 nthr) {
    const u32 w0 = r >> 6, b0 = r & 63;
    for (u32 pos = lo + tid; pos < hi; pos += nthr) {
        u64 v = ldcg(p.pb + pos), a = 0, c = 0;
        const u32 ph = ldcg(p.perm + pos);
        const u32 off = pos - r;
        const u32 tl = off < rb ? off : rb;
        // branch-free forward elimination against the panel's pivots
#pragma unroll 8
        for (u32 k = 0; k < 64; ++k) {
            if (k >= tl) break;
            const u64 bit = (v >> s.q[k]) & 1ull;
            const u64 msk = 0ull - bit;
            v ^= s.E[k] & msk;
            a ^= s.D[k] & msk;
            c |= bit << k;
        }
        u64 epart = 0;
        if constexpr (Check) {
            if (p.check_inject == w + 1u && off == rb) v ^= 1ull << 63;  // (the checker's own test)
            check_panel_word(p.check, w, v, tl, off < rb, s.q);
        }
        if (off < rb) {
            c |= 1ull << off;
            epart = v & ~low_mask64((int)s.q[off] + 1);
        }
        p.info[pos] = make_ulonglong2(a, (u64)ph);
        const u64 clo = c << b0;
        const u64 chi = b0 ? (c >> (64 - b0)) : 0ull;
        if (w0 == w) {
            *tword(p.mat, p.m, ph, w) = clo | epart;
        } else {
            u64* x0 = tword(p.mat, p.m, ph, w0);
            *x0 = ldcg(x0) | clo;
            if (w0 + 1 == w) {
                *tword(p.mat, p.m, ph, w) = chi | epart;
            } else {
                if (chi) {
                    u64* x1 = tword(p.mat, p.m, ph, w0 + 1);
                    *x1 = ldcg(x1) | chi;
                }
                *tword(p.mat, p.m, ph, w) = epart;
            }
        }
    }
}

__device__ __forceinline__ void apply_rows(const Params& p, const ApplyShared& s, u32 w, u32 r, u32 rb,
                                           u32 lo, u32 hi, u32 tid, u32 nthr) {
    if (p.check)
        apply_rows_t<true>(p, s, w, r, rb, lo, hi, tid, nthr);
    else
        apply_rows_t<false>(p, s, w, r, rb, lo, hi, tid, nthr);
}

// Raw pivot-row tails, tiles [(w+1)/8, Wpad8/8), into stage[(T*64 + t)*8 + k];
// units [u0, u1) of 16 bytes in the flattened (t, x) order.
__device__ __forceinline__ void stage_units(const Params& p, u32 w, u32 r, u32 rb, u32 u0, u32 u1,
                                            u32 tid, u32 nthr) {
    const u32 x0 = (w + 1) & ~7u;
    const u32 span2 = (p.Wpad8 - x0) >> 1;
    for (u32 e = u0 + tid; e < u1; e += nthr) {
        const u32 t = e / span2, x = x0 + 2u * (e - t * span2);
        const u32 ph = ldcg(p.perm + r + t);
        *reinterpret_cast<ulonglong2*>(p.stage + (((size_t)(x >> 3) * 64 + t) << 3) + (x & 7u)) =
            ldcg(reinterpret_cast<const ulonglong2*>(tword(p.mat, p.m, ph, x)));
    }
}

__device__ __forceinline__ u32 stage_total(const Params& p, u32 w, u32 rb) {
    if (w + 1 >= p.W || rb == 0) return 0;
    const u32 x0 = (w + 1) & ~7u;
    return rb * ((p.Wpad8 - x0) >> 1);
}

__global__ void __launch_bounds__(kApplyThreads) panel_apply_kernel(Params p, u32 w) {
    __shared__ ApplyShared s;
    const StepState st = *p.state;
    const u32 r = st.r, rb = st.rb;
    if (r >= p.m) return;
    apply_load(p, s, rb);
    __syncthreads();
    const u32 gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const u32 gsize = gridDim.x * blockDim.x;
    apply_rows(p, s, w, r, rb, r, p.m, gtid, gsize);
    stage_units(p, w, r, rb, 0, stage_total(p, w, rb), gtid, gsize);
}

// ===========================================================================
// Phase 3: trailing update
// ===========================================================================
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

// The 8 lookups of one 16-byte chunk: acc ^= T_g[byte_g(d)], g = gi ^ par
// for gi = 0..7 (par = the row's parity in its quarter-warp). g >> 1 =
// gi >> 1 is a compile-time table-pair offset, and byte g of d is byte
// (gi & 3) ^ par of 32-bit word gi >> 2: one PRMT with a per-lane selector.
// sel[j] = 0x4440 | (j ^ par), koff[j] = (((j ^ par) & 1) << 6) | (ch << 4).
__device__ __forceinline__ void lookup8(ulonglong2& acc, const unsigned char* smem, u64 d,
                                        const u32 sel[4], const u32 koff[4]) {
    const u32 wd[2] = {(u32)d, (u32)(d >> 32)};
#pragma unroll
    for (u32 gi = 0; gi < kTables; ++gi) {
        const u32 e = __byte_perm(wd[gi >> 2], 0u, sel[gi & 3u]);
        xor2(acc, *reinterpret_cast<const ulonglong2*>(smem + (gi >> 1) * 32768u + e * 128u + koff[gi & 3u]));
    }
}

__device__ __forceinline__ void lookup8_consts(u32 par, u32 ch, u32 sel[4], u32 koff[4]) {
#pragma unroll
    for (u32 j = 0; j < 4; ++j) {
        sel[j] = 0x4440u | (j ^ par);
        koff[j] = (((j ^ par) & 1u) << 6) | (ch << 4);
    }
}

// Build the 8 Gray-code tables of one 64-byte column tile from 64 source rows
// (row t's chunk at rowptr(t); rows t >= rb and the tile's first `zlim`
// words read as zero). Thread layout (512): ch = tid&3, g&1 = (tid>>2)&1,
// s_lo = (tid>>3)&3, g>>1 = (tid>>5)&3, s_hi = (tid>>7)&3; each thread walks
// entries gray(16 s + k), k = 0..15, with its 8 source chunks in registers:
// one XOR per entry (make_table, gray_code.hpp:105-112).
template <class RowPtr>
__device__ __forceinline__ void gray_tables_rows(unsigned char* smem, RowPtr rowptr, u32 rb, u32 zlim) {
    const u32 tid = threadIdx.x;
    const u32 ch = tid & 3u;
    const u32 g = (((tid >> 5) & 3u) << 1) | ((tid >> 2) & 1u);
    const u32 s = (((tid >> 7) & 3u) << 2) | ((tid >> 3) & 3u);
    ulonglong2 R[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const u32 t = 8u * g + b;
        ulonglong2 v = make_ulonglong2(0ull, 0ull);
        if (t < rb) v = ldcg(reinterpret_cast<const ulonglong2*>(rowptr(t) + 2u * ch));
        if (2u * ch < zlim) v.x = 0ull;
        if (2u * ch + 1u < zlim) v.y = 0ull;
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

// Contiguous source rows, `rs` words apart.
__device__ __forceinline__ void gray_tables(unsigned char* smem, const u64* src, u32 rb, u32 zlim,
                                            u32 rs = 8u) {
    gray_tables_rows(smem, [&](u32 t) { return src + (size_t)t * rs; }, rb, zlim);
}

// Tables of step w for tile `tile` from the raw pivot rows: the staged copy,
// or (persistent driver, piv = the step's pivot rows' physical indices) the
// matrix itself. Words <= w read as zero: the panel and everything left of
// it are not updated.
__device__ __forceinline__ void build_tables(const Params& p, unsigned char* smem, u32 tile,
                                             u32 w, u32 rb, const u32* piv = nullptr) {
    const u32 x0 = tile * 8u;
    const u32 zlim = w + 1u > x0 ? min(w + 1u - x0, 8u) : 0u;
    if (piv)
        gray_tables_rows(smem, [&](u32 t) { return tword(p.mat, p.m, piv[t], x0); }, rb, zlim);
    else
        gray_tables(smem, p.stage + (((size_t)tile * 64) << 3), rb, zlim);
}

__device__ __forceinline__ ulonglong2 ld_info(const ulonglong2* info, u32 pos, bool valid) {
    return valid ? ldcg(info + pos) : make_ulonglong2(0ull, 0ull);
}

// Rows [row0, row0+cnt) (offsets from r) of tile `tile`; tables must already
// be built. The tile holding word w+1 also writes the look-ahead panel buffer.
__device__ __forceinline__ void trail_rows(const Params& p, const unsigned char* smem, u32 w,
                                           u32 r, u32 tile, u32 row0, u32 cnt, u32 npiv = 0u) {
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 rg = lane >> 2, ch = lane & 3u, par = rg & 1u;
    const u32 cap_word = w + 1;
    const bool capture1 = (cap_word >> 3) == tile;
    const bool cap_lane = capture1 && ((cap_word & 7u) >> 1) == ch;
    const bool cap_hi = (cap_word & 1u) != 0;
    // look-ahead driver: word w+2 as well (the panel CTA's next-window input)
    const u32 cap2_word = w + 2;
    const bool capture2 = p.pb2 != nullptr && cap2_word < p.W && (cap2_word >> 3) == tile;
    const bool cap2_lane = capture2 && ((cap2_word & 7u) >> 1) == ch;
    const bool cap2_hi = (cap2_word & 1u) != 0;
    const bool capture = capture1 || capture2;
    const u32 lane_row = wid * 8u + rg;
    u32 lsel[4], lkoff[4];
    lookup8_consts(par, ch, lsel, lkoff);
    u64* tbase = p.mat + (((size_t)tile * p.m) << 3) + 2u * ch;
    const u32 rend = row0 + cnt;
    const u32 nit = (cnt + kRowsPerIter - 1) / kRowsPerIter;

    // software pipeline: rows of iteration i+1 and records of i+2 in flight
    ulonglong2 infC[kUnroll], infN[kUnroll], valC[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 4);
        infC[k] = ld_info(p.info, r + ri, ri < rend);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
        infN[k] = ld_info(p.info, r + ri, ri < rend);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 4);
        valC[k] = make_ulonglong2(0ull, 0ull);
        if (ri < rend && (infC[k].x != 0ull || capture || ri < npiv))
            valC[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)infC[k].y << 3)));
    }
    for (u32 it = 0; it < nit; ++it) {
        const u32 base = row0 + it * kRowsPerIter;
        ulonglong2 valN[kUnroll], infNN[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
            valN[k] = make_ulonglong2(0ull, 0ull);
            if (ri < rend && (infN[k].x != 0ull || capture || ri < npiv))
                valN[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)infN[k].y << 3)));
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + 2 * kRowsPerIter + lane_row + (u32)k * (kTrailThreads / 4);
            infNN[k] = ld_info(p.info, r + ri, ri < rend);
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + lane_row + (u32)k * (kTrailThreads / 4);
            const u64 d = infC[k].x;
            // (pivot rows always reach ubuf, d = 0 included: U_t = raw tail)
            if (d != 0ull || (ri < npiv && ri < rend)) {
                lookup8(valC[k], smem, d, lsel, lkoff);
                if (ri < npiv)  // a pivot row of this step: its tail goes to ubuf
                    *reinterpret_cast<ulonglong2*>(
                        p.ubuf + ((((size_t)tile * p.ucap + r + ri) << 3) + 2u * ch)) = valC[k];
                else
                    *reinterpret_cast<ulonglong2*>(tbase + ((size_t)infC[k].y << 3)) = valC[k];
            }
            if (cap_lane && ri < rend) p.pb[r + ri] = cap_hi ? valC[k].y : valC[k].x;
            if (cap2_lane && ri < rend) p.pb2[r + ri] = cap2_hi ? valC[k].y : valC[k].x;
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            infC[k] = infN[k];
            infN[k] = infNN[k];
            valC[k] = valN[k];
        }
    }
}

// Linear share [beg, end) of the (tile, row) work of step w over tiles
// [tile_lo, tile_hi), rows r..m-1; tables rebuilt per tile segment.
__device__ __forceinline__ void trail_share(const Params& p, unsigned char* smem, u32 w, u32 r,
                                            u32 rb, u32 tile_lo, u64 beg, u64 end,
                                            const u32* piv = nullptr) {
    const u32 nrows = p.m - r;
    u64 u = beg;
    while (u < end) {
        const u32 tile = tile_lo + (u32)(u / nrows);
        const u32 row0 = (u32)(u % nrows);
        const u32 cnt = (u32)min((u64)(nrows - row0), end - u);
        if (rb > 0) {
            __syncthreads();
            build_tables(p, smem, tile, w, rb, piv);
            __syncthreads();
        }
        trail_rows(p, smem, w, r, tile, row0, cnt, piv ? rb : 0u);
        u += cnt;
    }
}

__global__ void __launch_bounds__(kTrailThreads, 1) trailing_update_kernel(Params p, u32 w) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StepState st = *p.state;
    const u32 r = st.r, rb = st.rb;
    if (r >= p.m || w + 1 >= p.W) return;
    const u32 tile0 = (w + 1) >> 3;
    const u32 ntiles = (p.Wpad8 >> 3) - tile0;
    const u64 total = (u64)ntiles * (p.m - r);
    trail_share(p, smem, w, r, rb, tile0, total * blockIdx.x / gridDim.x,
                total * (blockIdx.x + 1) / gridDim.x);
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
// Density estimate of a row-major matrix: the set bits of one pseudo-randomly
// chosen word per row, summed into *ones (run_ple's driver choice).
__global__ void density_sample_kernel(const u64* __restrict__ mat, u32 m, u32 W, u32 Wp, u32* ones) {
    u32 acc = 0;
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        acc += (u32)__popcll(mat[(size_t)i * Wp + (i * 0x9e3779b1u) % W]);
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31u) == 0u && acc) atomicAdd(ones, acc);
}

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
