// gf2cu.cu -- host driver and C ABI (include/gf2cu.h) of the B200 PLE path.
//
// The driver replaces gf2::block_iterative_ple (ple.hpp:166-244): per
// 64-column panel it enqueues panel_factor -> panel_apply -> trailing_update
// on one stream, with all step state (r, rb) kept on the device so the host
// never waits inside the loop. The host only polls a mapped pinned mirror of
// r (a few steps behind) to stop enqueueing once every row holds a pivot.
#include <cuda_runtime.h>
#include <omp.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "gf2cu.h"
#include "ple_kernels.cuh"
#include "ple_persistent.cuh"
#include "ple_super.cuh"
#include "ple_shard.cuh"
#include "ple_peer.cuh"
#include "ple_peer_super.cuh"
#include "rref_kernels.cuh"
#include "gemm_kernels.cuh"
#include "litmus.cuh"

using gf2cu::u32;
using gf2cu::u64;

namespace {

thread_local std::string g_last_error;

// The super-step driver (two panels per sweep) from this many matrix words up,
// the single-panel persistent driver below. Measured with the super-step
// look-ahead: 16384^2 (4.2M words) single 4.24 vs super 4.28 ms, 12288^2
// single better; 16384x24576 (6.3M) 4.98 vs 4.61, 20480^2 (6.5M) 6.02 vs 5.73
// super better (8192x32768, 4.2M: 2.32 vs 2.22, the crossover's fuzz).
constexpr double kSuperStepWords = 5242880.0;

// Panel tuning bits (gf2cu::kPanel*); GF2CU_PANEL_FLAGS overrides the default
// for A/B measurements.
u32 panel_flags() {
    const char* e = std::getenv("GF2CU_PANEL_FLAGS");
    return e ? (u32)std::strtoul(e, nullptr, 0) : (gf2cu::kPanelStream | gf2cu::kPanelSuperLA);
}

// Zero-fill at creation, COMPLETED before returning. A plain cudaMemset is
// enqueued on the legacy default stream and is asynchronous with respect to
// the host; the objects' own streams are non-blocking, so a later upload on
// them was not ordered after it and the fill could land on top of the
// uploaded matrix (round 2: the root cause of the rare rank-0 / wrong-word
// results on the first call with a new shape).
cudaError_t zero_now(void* p, size_t bytes) {
    cudaError_t e = cudaMemsetAsync(p, 0, bytes, 0);
    return e == cudaSuccess ? cudaStreamSynchronize(0) : e;
}

// Host -> device copy of parameters, COMPLETED before returning: a plain
// cudaMemcpy from pageable memory returns once the source is staged, its DMA
// runs on the legacy default stream, which the kernels' non-blocking streams
// are not ordered after.
cudaError_t h2d_now(void* dst, const void* src, size_t bytes) {
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? cudaStreamSynchronize(0) : e;
}

gf2cu_status fail(gf2cu_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

gf2cu_status cuda_fail(cudaError_t e, const char* what) {
    const gf2cu_status st = (e == cudaErrorMemoryAllocation) ? GF2CU_ENOMEM : GF2CU_ECUDA;
    return fail(st, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU_TRY(expr)                                                   \
    do {                                                               \
        cudaError_t _e = (expr);                                       \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);            \
    } while (0)

size_t words_of(size_t n) { return (n + 63) / 64; }
size_t wpad8(size_t W) { return std::max<size_t>(8, (W + 7) / 8 * 8); }
size_t padded_stride(size_t n) { return std::max<size_t>(16, (words_of(n) + 15) / 16 * 16); }

struct Workspace {
    bool ready = false;  // every buffer below allocated (ensure_ws)
    size_t m = 0, Wp = 0, W = 0;
    u32* perm = nullptr;
    u64* pb = nullptr;
    u64* pb2 = nullptr;  // look-ahead next-word capture
    ulonglong2* info = nullptr;
    u64* stage = nullptr;
    gf2cu::StepState* state = nullptr;
    gf2cu::PanelOut* pout = nullptr;
    u32* swaps = nullptr;
    u32* qcol = nullptr;
    u32* rhist = nullptr;
    u32* rbhist = nullptr;
    u32* host_r = nullptr;       // pinned, mapped
    u32* host_r_dev = nullptr;   // device alias
    u32* out_host = nullptr;     // pinned, mapped: leading positions already final in data
    u32* out_host_dev = nullptr;
    cudaStream_t copy = nullptr; // streamed D2H of finished rows while the kernel runs
    u64* hashes = nullptr;       // per-row checksum scratch
    gf2cu::SyncState* sync = nullptr;
    u64* phase_ns = nullptr;     // 8 stamps per step (persistent driver)
    u64* ubuf = nullptr;         // persistent driver: swept pivot-row tails
    size_t ucap = 0;
    u32* apctr = nullptr;        // persistent driver: per-step pre-work chunk counters
    u32* h_out = nullptr;        // pinned host staging of swaps / q (2 x min(m, n))
    gf2cu::PanelOut* pout_b = nullptr;  // super-step driver: panel b's outputs
    gf2cu::SuperOut* sout = nullptr;
    u32* check = nullptr;        // check mode: Params::check words
    // streamed input (run_ple): upload stream and "row block arrived" events,
    // the per-super-step panel outputs, phase A's verdict
    cudaStream_t up = nullptr;
    cudaEvent_t up_ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    gf2cu::PanelOut* hist_a = nullptr;
    gf2cu::PanelOut* hist_b = nullptr;
    gf2cu::SuperOut* hist_so = nullptr;
    u32* sin_abort = nullptr;
    std::vector<cudaEvent_t> ev;
};

void free_ws(Workspace& w) {
    cudaFree(w.perm);
    cudaFree(w.pb);
    cudaFree(w.pb2);
    cudaFree(w.info);
    cudaFree(w.stage);
    cudaFree(w.state);
    cudaFree(w.pout);
    cudaFree(w.swaps);
    cudaFree(w.qcol);
    cudaFree(w.rhist);
    cudaFree(w.rbhist);
    cudaFree(w.hashes);
    cudaFree(w.sync);
    cudaFree(w.phase_ns);
    cudaFree(w.ubuf);
    cudaFree(w.apctr);
    cudaFreeHost(w.h_out);
    cudaFree(w.pout_b);
    cudaFree(w.sout);
    cudaFree(w.check);
    if (w.host_r) cudaFreeHost(w.host_r);
    if (w.out_host) cudaFreeHost(w.out_host);
    if (w.copy) cudaStreamDestroy(w.copy);
    if (w.up) cudaStreamDestroy(w.up);
    for (cudaEvent_t e : w.up_ev)
        if (e) cudaEventDestroy(e);
    cudaFree(w.hist_a);
    cudaFree(w.hist_b);
    cudaFree(w.hist_so);
    cudaFree(w.sin_abort);
    for (cudaEvent_t e : w.ev) cudaEventDestroy(e);
    w = Workspace{};
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int g_num_sms[64] = {0};

int num_sms(int dev) {
    if (dev < 0 || dev >= 64) return 148;
    if (!g_num_sms[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev] = v > 0 ? v : 148;
    }
    return g_num_sms[dev];
}

// GF2CU_WATCHDOG_S=<seconds> raises the spin watchdog of the persistent
// kernels (runs under compute-sanitizer are 10-100x slower); once per device.
void apply_watchdog_env(int dev) {
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    done[dev] = true;
    if (const char* e = std::getenv("GF2CU_WATCHDOG_S")) {
        const double sec = std::atof(e);
        if (sec > 0) {
            const unsigned long long ns = (unsigned long long)(sec * 1e9);
            cudaMemcpyToSymbol(gf2cu::g_watchdog_ns, &ns, sizeof(ns));
            cudaStreamSynchronize(0);  // (ordered before kernels on non-blocking streams)
        }
    }
}

}  // namespace

namespace {

// Device buffers of the reduced-echelon / upper-triangular solve, grown on
// demand and kept with the matrix handle.
struct RrefWs {
    u64* U = nullptr;     size_t U_words = 0;
    u64* N = nullptr;     size_t N_words = 0;
    u64* src = nullptr;   size_t src_words = 0;  // trsm operands (row-major)
    u32* idx = nullptr;   size_t idx_words = 0;  // q | np | usrc | nsrc | npos0
    u64* npmask = nullptr; size_t npmask_words = 0;
};

void free_rref(RrefWs& w) {
    cudaFree(w.U);
    cudaFree(w.N);
    cudaFree(w.src);
    cudaFree(w.idx);
    cudaFree(w.npmask);
    w = RrefWs{};
}

template <class T>
cudaError_t grow(T** ptr, size_t* have, size_t need) {
    need = std::max<size_t>(need, 1);
    if (*have >= need) return cudaSuccess;
    cudaFree(*ptr);
    *ptr = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(ptr, need * sizeof(T));
    if (e == cudaSuccess) *have = need;
    return e;
}

}  // namespace

namespace {

// Buffers of the device-driven row-sharded driver (ple_peer.cuh) when all G
// ranks run in one cooperative launch on this matrix's device.
struct PeerWs {
    unsigned G = 0, block = 0;
    std::vector<gf2cu::PeerParams> hp;  // host copies of the ranks' parameters
    gf2cu::PeerParams* dp = nullptr;    // device copy (the kernel argument)
    std::vector<void*> allocs;
    std::vector<size_t> sizes;          // bytes of each allocation
};

void free_peer(PeerWs& w) {
    for (void* x : w.allocs) cudaFree(x);
    cudaFree(w.dp);
    w = PeerWs{};
}

}  // namespace

struct gf2cu_matrix {
    size_t m = 0, n = 0, W = 0, Wp = 0;
    int device = 0;
    u64* data = nullptr;
    u64* alt = nullptr;  // tile-major working copy used by the factorization
    Workspace ws;
    RrefWs rw;
    PeerWs pw;
    cudaStream_t own = nullptr;
};

namespace {

cudaStream_t pick_stream(gf2cu_matrix* a, void* s) {
    return s ? reinterpret_cast<cudaStream_t>(s) : a->own;
}

gf2cu_status alloc_ws(gf2cu_matrix* a);

// ---- pageable host memory ----------------------------------------------
// The runtime copies pageable host memory through its own small pinned
// buffers on one thread. Large copies from / to pageable buffers (what a C++
// caller's gf2::BitMatrix, a std::vector, hands the drop-in) instead go
// through pinned staging chunks that host threads fill or drain (OpenMP row
// memcpy) while the copy engine works on the neighbouring chunk.
struct Staging {
    static constexpr int kBufs = 3;
    static constexpr size_t kBytes = size_t(32) << 20;
    unsigned char* buf[kBufs] = {};
    cudaEvent_t ev[kBufs] = {};
    int device = -1;
    void release() {
        for (int i = 0; i < kBufs; ++i) {
            if (ev[i]) cudaEventSynchronize(ev[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
            buf[i] = nullptr;
            ev[i] = nullptr;
        }
        device = -1;
    }
    ~Staging() { release(); }
};
thread_local Staging g_staging;

// GF2CU_TRACE=1 (diagnostic): host timestamps and stream events of one
// drop-in call, printed to stderr in ms since the call began.
struct Trace {
    bool on = false;
    std::chrono::steady_clock::time_point t0;
    cudaEvent_t base = nullptr;
    std::vector<std::pair<std::string, double>> host;
    std::vector<std::pair<std::string, cudaEvent_t>> gpu;
};
thread_local Trace g_trace;

void trace_begin(cudaStream_t s) {
    const char* e = std::getenv("GF2CU_TRACE");
    g_trace.on = e && std::atoi(e) > 0;
    if (!g_trace.on) return;
    g_trace.host.clear();
    g_trace.gpu.clear();
    cudaStreamSynchronize(s);
    cudaEventCreate(&g_trace.base);
    g_trace.t0 = std::chrono::steady_clock::now();
    cudaEventRecord(g_trace.base, s);
}
void trace_host(const char* what) {
    if (!g_trace.on) return;
    g_trace.host.emplace_back(what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - g_trace.t0).count());
}
void trace_gpu(const std::string& what, cudaStream_t s) {
    if (!g_trace.on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    g_trace.gpu.emplace_back(what, e);
}
void trace_end() {
    if (!g_trace.on) return;
    trace_host("return");
    cudaDeviceSynchronize();
    for (auto& h : g_trace.host) std::fprintf(stderr, "[trace host] %8.3f  %s\n", h.second, h.first.c_str());
    for (auto& g : g_trace.gpu) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g_trace.base, g.second);
        std::fprintf(stderr, "[trace gpu ] %8.3f  %s\n", ms, g.first.c_str());
        cudaEventDestroy(g.second);
    }
    cudaEventDestroy(g_trace.base);
    g_trace.on = false;
}

constexpr size_t kStageMin = size_t(8) << 20;  // smaller copies: the runtime's path

bool host_pageable(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

gf2cu_status staging_ready(int device) {
    Staging& g = g_staging;
    if (g.device == device && g.buf[0]) return GF2CU_OK;
    g.release();
    for (int i = 0; i < Staging::kBufs; ++i) {
        CU_TRY(cudaHostAlloc(&g.buf[i], Staging::kBytes, cudaHostAllocDefault));
        CU_TRY(cudaEventCreateWithFlags(&g.ev[i], cudaEventDisableTiming));
    }
    g.device = device;
    return GF2CU_OK;
}

// One row with non-temporal stores: the destination (a pinned staging chunk
// on the way up, the caller's buffer on the way down) is written once and not
// read by this core again, so the stores bypass the cache and skip the
// read-for-ownership of every destination line -- a third less memory traffic
// than memcpy, whose own non-temporal path only starts far above a row's size.
inline void copy_row_stream(unsigned char* d, const unsigned char* s, size_t n) {
#if defined(__SSE2__)
    size_t head = (16u - (reinterpret_cast<uintptr_t>(d) & 15u)) & 15u;
    if (head > n) head = n;
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    for (; n >= 64; n -= 64, d += 64, s += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
    }
#endif
    std::memcpy(d, s, n);
}

void rows_memcpy(unsigned char* dst, size_t dst_pitch, const unsigned char* src, size_t src_pitch, size_t bytes,
                 size_t rows) {
    const int nt = std::max(1, std::min(omp_get_max_threads(), 16));
    static const bool plain = [] {
        const char* e = std::getenv("GF2CU_STAGE_MEMCPY");  // 1: plain memcpy (A/B measurements)
        return e && std::atoi(e) != 0;
    }();
#pragma omp parallel num_threads(nt)
    {
#pragma omp for schedule(static) nowait
        for (long long i = 0; i < (long long)rows; ++i) {
            if (plain)
                std::memcpy(dst + (size_t)i * dst_pitch, src + (size_t)i * src_pitch, bytes);
            else
                copy_row_stream(dst + (size_t)i * dst_pitch, src + (size_t)i * src_pitch, bytes);
        }
#if defined(__SSE2__)
        _mm_sfence();  // the streamed rows are globally visible before the copy engine reads them
#endif
    }
}

// Rows per staging piece: a quarter of the copy (at least 1 MiB, at most a
// whole staging buffer), so that even a copy that fits one buffer -- a row
// block of the streamed input, a batch of the streamed output -- overlaps its
// host memcpy with its DMA.
size_t stage_piece_rows(size_t bytes, size_t rows) {
    const size_t total = bytes * rows;
    const size_t target = std::min(Staging::kBytes, std::max<size_t>(size_t(1) << 20, total / 4));
    return std::max<size_t>(1, target / bytes);
}

// Host (pitch hp bytes) -> device (pitch dp bytes), `bytes` per row, `rows`
// rows, ordered on s. Returns with the host buffer free to reuse.
gf2cu_status staged_h2d(void* dev, size_t dp, const void* host, size_t hp, size_t bytes, size_t rows, int device,
                        cudaStream_t s) {
    if (bytes * rows < kStageMin || !host_pageable(host)) {
        CU_TRY(cudaMemcpy2DAsync(dev, dp, host, hp, bytes, rows, cudaMemcpyHostToDevice, s));
        return GF2CU_OK;
    }
    gf2cu_status st = staging_ready(device);
    if (st != GF2CU_OK) return st;
    Staging& g = g_staging;
    const size_t per = stage_piece_rows(bytes, rows);
    for (size_t c = 0, r0 = 0; r0 < rows; ++c, r0 += per) {
        const int b = (int)(c % Staging::kBufs);
        const size_t nr = std::min(per, rows - r0);
        CU_TRY(cudaEventSynchronize(g.ev[b]));  // (its previous chunk has left)
        rows_memcpy(g.buf[b], bytes, static_cast<const unsigned char*>(host) + r0 * hp, hp, bytes, nr);
        CU_TRY(cudaMemcpy2DAsync(static_cast<unsigned char*>(dev) + r0 * dp, dp, g.buf[b], bytes, bytes, nr,
                                 cudaMemcpyHostToDevice, s));
        CU_TRY(cudaEventRecord(g.ev[b], s));
    }
    return GF2CU_OK;
}

// Device -> host, synchronous (the host buffer holds the rows on return).
gf2cu_status staged_d2h(void* host, size_t hp, const void* dev, size_t dp, size_t bytes, size_t rows, int device,
                        cudaStream_t s) {
    if (bytes * rows < kStageMin || !host_pageable(host)) {
        CU_TRY(cudaMemcpy2DAsync(host, hp, dev, dp, bytes, rows, cudaMemcpyDeviceToHost, s));
        CU_TRY(cudaStreamSynchronize(s));
        return GF2CU_OK;
    }
    gf2cu_status st = staging_ready(device);
    if (st != GF2CU_OK) return st;
    Staging& g = g_staging;
    const size_t per = stage_piece_rows(bytes, rows);
    const size_t nch = (rows + per - 1) / per;
    auto issue = [&](size_t c) -> cudaError_t {
        const int b = (int)(c % Staging::kBufs);
        const size_t r0 = c * per, nr = std::min(per, rows - r0);
        cudaError_t e = cudaMemcpy2DAsync(g.buf[b], bytes, static_cast<const unsigned char*>(dev) + r0 * dp, dp,
                                          bytes, nr, cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? cudaEventRecord(g.ev[b], s) : e;
    };
    for (size_t c = 0; c < std::min<size_t>(nch, Staging::kBufs - 1); ++c) CU_TRY(issue(c));
    for (size_t c = 0; c < nch; ++c) {
        const int b = (int)(c % Staging::kBufs);
        if (c + Staging::kBufs - 1 < nch) CU_TRY(issue(c + Staging::kBufs - 1));
        CU_TRY(cudaEventSynchronize(g.ev[b]));
        const size_t r0 = c * per, nr = std::min(per, rows - r0);
        rows_memcpy(static_cast<unsigned char*>(host) + r0 * hp, hp, g.buf[b], bytes, bytes, nr);
    }
    return GF2CU_OK;
}

// The workspace is all-or-nothing: a failed allocation frees whatever was
// already allocated, so the next call on the (cached) matrix retries from
// scratch instead of launching on null buffers.
gf2cu_status ensure_ws(gf2cu_matrix* a) {
    if (a->ws.ready) return GF2CU_OK;
    free_ws(a->ws);
    const gf2cu_status st = alloc_ws(a);
    if (st != GF2CU_OK) {
        free_ws(a->ws);
        return st;
    }
    a->ws.ready = true;
    return GF2CU_OK;
}

gf2cu_status alloc_ws(gf2cu_matrix* a) {
    Workspace& w = a->ws;
    const size_t m = a->m, mn = std::max<size_t>(1, std::min(a->m, a->n));
    w.m = m;
    w.Wp = a->Wp;
    w.W = a->W;
    CU_TRY(cudaMalloc(&w.perm, std::max<size_t>(1, m) * sizeof(u32)));
    CU_TRY(cudaMalloc(&w.pb, std::max<size_t>(1, m) * sizeof(u64)));
    CU_TRY(cudaMalloc(&w.pb2, std::max<size_t>(1, m) * sizeof(u64)));
    CU_TRY(cudaMalloc(&w.info, 4 * std::max<size_t>(1, m) * sizeof(ulonglong2)));
    CU_TRY(cudaMalloc(&w.pout_b, sizeof(gf2cu::PanelOut)));
    CU_TRY(cudaMalloc(&w.sout, sizeof(gf2cu::SuperOut)));
    CU_TRY(cudaMalloc(&w.sync, sizeof(gf2cu::SyncState)));
    CU_TRY(cudaMalloc(&w.phase_ns, (8 * (a->W + 1) + 8 + 2 * 64 * 5 + 3 * 160) * sizeof(u64)));
    CU_TRY(cudaMalloc(&w.stage, 64 * wpad8(a->W) * sizeof(u64)));
    CU_TRY(zero_now(w.stage, 64 * wpad8(a->W) * sizeof(u64)));
    CU_TRY(cudaMalloc(&w.state, sizeof(gf2cu::StepState)));
    CU_TRY(cudaMalloc(&w.pout, sizeof(gf2cu::PanelOut)));
    CU_TRY(cudaMalloc(&w.swaps, mn * sizeof(u32)));
    CU_TRY(cudaMalloc(&w.qcol, mn * sizeof(u32)));
    CU_TRY(cudaMalloc(&w.rhist, (a->W + 1) * sizeof(u32)));
    CU_TRY(cudaMalloc(&w.rbhist, (a->W + 1) * sizeof(u32)));
    CU_TRY(cudaHostAlloc(&w.host_r, sizeof(u32), cudaHostAllocMapped));
    CU_TRY(cudaHostGetDevicePointer(&w.host_r_dev, w.host_r, 0));
    CU_TRY(cudaHostAlloc(&w.out_host, sizeof(u32), cudaHostAllocMapped));
    CU_TRY(cudaHostGetDevicePointer(&w.out_host_dev, w.out_host, 0));
    CU_TRY(cudaStreamCreateWithFlags(&w.copy, cudaStreamNonBlocking));
    CU_TRY(cudaMalloc(&w.check, 4 * sizeof(u32)));
    return GF2CU_OK;
}

// Check mode (GF2CU_FLAG_CHECK or GF2CU_CHECK=1 in the environment).
bool check_mode(const gf2cu_cfg* cfg) {
    if (cfg && (cfg->flags & GF2CU_FLAG_CHECK)) return true;
    const char* e = std::getenv("GF2CU_CHECK");
    return e && e[0] && std::strcmp(e, "0") != 0;
}

u32 check_inject_env() {
    const char* e = std::getenv("GF2CU_CHECK_INJECT");  // test hook: step + 1 to corrupt
    return e ? (u32)std::strtoul(e, nullptr, 0) : 0u;
}

gf2cu_status check_reset(u32* chk, cudaStream_t s) {
    static const u32 init[4] = {0xffffffffu, 0u, 0xffffffffu, 0u};
    CU_TRY(cudaMemcpyAsync(chk, init, sizeof(init), cudaMemcpyHostToDevice, s));
    return GF2CU_OK;
}

// GF2CU_POISON=<byte>: fill every scratch buffer of a factorization with
// that byte before each run (a diagnostic: a result that depends on a stale
// or uninitialized scratch word then fails deterministically instead of
// depending on what an earlier call left behind).
int poison_byte() {
    const char* e = std::getenv("GF2CU_POISON");
    return e && e[0] ? (int)(std::strtoul(e, nullptr, 0) & 0xff) : -1;
}

// After the factorization: the result invariants on the row-major matrix,
// then the verdict of both checks.
gf2cu_status check_verdict(gf2cu_matrix* a, u32* chk, size_t rank, int sms, cudaStream_t s);

// PleConfig never makes the reference throw: pick_table_bits clamps any
// k_scale (<= 0, tiny, huge) to k in [1, 16] (gray_code.hpp:171-177) and the
// driver clamps k and table_count (ple.hpp:168-169, 201). The device output
// does not depend on k, so every configuration is accepted here as well.
gf2cu_status check_cfg(const gf2cu_cfg* cfg) {
    (void)cfg;
    return GF2CU_OK;
}

size_t shard_rows(size_t m, size_t rank, size_t G, size_t block) {
    const size_t cyc = block * G, full = m / cyc, rem = m % cyc;
    const size_t lo = rank * block;
    return full * block + (rem > lo ? std::min(block, rem - lo) : 0);
}

// One rank's exchange buffers (ple_peer.cuh PeerBufs) live in ONE allocation
// so a single IPC handle maps them: pb[2], pb2[2], stage[2], counters.
size_t al256(size_t b) { return (b + 255) / 256 * 256; }
// (the stage holds 128 pivot rows: the super-step form's two panels)
size_t peer_xbytes(size_t m, size_t Wp8) {
    return 4 * al256(std::max<size_t>(1, m) * 8) + 2 * al256(128 * Wp8 * 8) + al256(gf2cu::kCtrWords * 4);
}
gf2cu::PeerBufs peer_bufs_at(void* base, size_t m, size_t Wp8) {
    char* c = static_cast<char*>(base);
    const size_t a = al256(std::max<size_t>(1, m) * 8), st = al256(128 * Wp8 * 8);
    gf2cu::PeerBufs b{};
    b.pb[0] = reinterpret_cast<u64*>(c);
    b.pb[1] = reinterpret_cast<u64*>(c + a);
    b.pb2[0] = reinterpret_cast<u64*>(c + 2 * a);
    b.pb2[1] = reinterpret_cast<u64*>(c + 3 * a);
    b.stage[0] = reinterpret_cast<u64*>(c + 4 * a);
    b.stage[1] = reinterpret_cast<u64*>(c + 4 * a + st);
    b.ctr = reinterpret_cast<u32*>(c + 4 * a + 2 * st);
    return b;
}

// Allocates rank k's local rows and replicated state (h.p) and its exchange
// buffers (*xbuf, h.peer[k]); every allocation is appended to `allocs`.
gf2cu_status peer_alloc_rank(gf2cu::PeerParams& h, std::vector<void*>& allocs, size_t m, size_t n,
                             unsigned k, unsigned G, unsigned block, void** xbuf,
                             std::vector<size_t>* sizes = nullptr) {
    const size_t W = words_of(n), Wp8 = wpad8(W), mn = std::max<size_t>(1, std::min(m, n));
    auto alloc = [&](void** ptr, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(ptr, std::max<size_t>(bytes, 16));
        if (e == cudaSuccess) {
            allocs.push_back(*ptr);
            if (sizes) sizes->push_back(std::max<size_t>(bytes, 16));
        }
        return e;
    };
#define PA(ptr, bytes) CU_TRY(alloc(reinterpret_cast<void**>(&(ptr)), (bytes)))
    h = gf2cu::PeerParams{};
    gf2cu::Params& p = h.p;
    h.m_loc = (u32)shard_rows(m, k, G, block);
    h.rank = k;
    h.nranks = G;
    h.block = block;
    PA(h.mat, (size_t)h.m_loc * Wp8 * 8);
    PA(h.info[0], (size_t)h.m_loc * 16);
    PA(h.info[1], (size_t)h.m_loc * 16);
    PA(h.ipos[0], (size_t)h.m_loc * 4);
    PA(h.ipos[1], (size_t)h.m_loc * 4);
    PA(h.pout_b, sizeof(gf2cu::PanelOut));
    PA(h.so, sizeof(gf2cu::SuperOut));
    PA(h.lo, (W + 1) * 4);
    PA(p.perm, m * 4);
    PA(p.inv, m * 4);
    PA(p.state, sizeof(gf2cu::StepState));
    PA(p.pout, sizeof(gf2cu::PanelOut));
    PA(p.swaps, mn * 4);
    PA(p.qcol, mn * 4);
    PA(p.rhist, (W + 1) * 4);
    PA(p.rbhist, (W + 1) * 4);
    PA(p.sync, sizeof(gf2cu::SyncState));
    PA(p.ap_claim, 2 * (W + 1) * 4);
    p.ap_done = p.ap_claim + W + 1;
    PA(*xbuf, peer_xbytes(m, Wp8));
#undef PA
    h.peer[k] = peer_bufs_at(*xbuf, m, Wp8);
    const char* dv = std::getenv("GF2CU_PW_DIV");
    p.pw_div = dv ? (u32)std::max(64, std::atoi(dv)) : 8192u;
    p.m = (u32)m;
    p.n = (u32)n;
    p.W = (u32)W;
    p.Wpad8 = (u32)Wp8;
    p.pflags = panel_flags();
    return GF2CU_OK;
}

gf2cu_status peer_reset_rank(const gf2cu::PeerParams& h, cudaStream_t s) {
    const size_t W = h.p.W;
    CU_TRY(cudaMemsetAsync(h.p.sync, 0, sizeof(gf2cu::SyncState), s));
    CU_TRY(cudaMemsetAsync(h.p.ap_claim, 0, 2 * (W + 1) * 4, s));
    CU_TRY(cudaMemsetAsync(h.lo, 0xff, (W + 1) * 4, s));
    CU_TRY(cudaMemsetAsync(h.peer[h.rank].ctr, 0, gf2cu::kCtrWords * 4, s));
    return GF2CU_OK;
}

// Two panels per sweep (ple_peer_super.cuh) on the same size rule as the
// single-GPU drivers (run_ple), unless forced by flags or GF2CU_PEER_SUPER.
bool peer_super(size_t m, size_t W, unsigned flags) {
    if (const char* e = std::getenv("GF2CU_PEER_SUPER")) return std::atoi(e) != 0;
    if (flags & GF2CU_FLAG_SINGLE_PANEL) return false;
    return (flags & GF2CU_FLAG_SUPER_STEP) || (double)m * (double)W >= kSuperStepWords;
}

gf2cu_status peer_launch(const gf2cu::PeerParams* dp, unsigned ranks_here, unsigned cpr, size_t W,
                         bool super, int device, cudaStream_t s) {
    static bool attr_set[64] = {false};
    if (device >= 0 && device < 64 && !attr_set[device]) {
        CU_TRY(cudaFuncSetAttribute(gf2cu::ple_peer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    gf2cu::kTableBytes));
        CU_TRY(cudaFuncSetAttribute(gf2cu::ple_peer_super_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, gf2cu::kTableBytes));
        attr_set[device] = true;
    }
    u32 c = cpr, nsteps = super ? (u32)((W + 1) / 2) : (u32)W;
    void* args[] = {(void*)&dp, &c, &nsteps};
    void* fn = super ? (void*)gf2cu::ple_peer_super_kernel : (void*)gf2cu::ple_peer_kernel;
    CU_TRY(cudaLaunchCooperativeKernel(fn, dim3(cpr * ranks_here), dim3(gf2cu::kTrailThreads), args,
                                       gf2cu::kTableBytes, s));
    return GF2CU_OK;
}

// The replicated outcome from one rank's state (after its kernel finished):
// rank, swaps, q, canonical col_swaps, optional perm and stats.
gf2cu_status peer_outputs(const gf2cu::PeerParams& h, bool super, cudaStream_t s, size_t* swaps,
                          size_t* q, size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                          uint32_t* perm, gf2cu_stats* stats) {
    const size_t m = h.p.m, n = h.p.n, W = h.p.W;
    u32 c[gf2cu::kCtrWords];
    gf2cu::SyncState sy{};
    gf2cu::StepState fin{};
    CU_TRY(cudaMemcpyAsync(c, h.peer[h.rank].ctr, sizeof(c), cudaMemcpyDeviceToHost, s));
    CU_TRY(cudaMemcpyAsync(&sy, h.p.sync, sizeof(sy), cudaMemcpyDeviceToHost, s));
    CU_TRY(cudaMemcpyAsync(&fin, h.p.state, sizeof(fin), cudaMemcpyDeviceToHost, s));
    CU_TRY(cudaStreamSynchronize(s));
    if (c[gf2cu::kCtrErr]) return fail(GF2CU_ECUDA, "row-sharded PLE kernel watchdog tripped");
    const size_t steps = std::min<size_t>(W, super ? 2 * (size_t)sy.panel_done : (size_t)sy.panel_done);
    const size_t rk = std::min<size_t>((size_t)fin.r + fin.rb, std::min(m, n));
    std::vector<u32> sw(rk), qq(rk), rh(steps), rbh(steps);
    if (rk) {
        CU_TRY(cudaMemcpyAsync(sw.data(), h.p.swaps, rk * 4, cudaMemcpyDeviceToHost, s));
        CU_TRY(cudaMemcpyAsync(qq.data(), h.p.qcol, rk * 4, cudaMemcpyDeviceToHost, s));
    }
    if (steps) {
        CU_TRY(cudaMemcpyAsync(rh.data(), h.p.rhist, steps * 4, cudaMemcpyDeviceToHost, s));
        CU_TRY(cudaMemcpyAsync(rbh.data(), h.p.rbhist, steps * 4, cudaMemcpyDeviceToHost, s));
    }
    if (perm) CU_TRY(cudaMemcpyAsync(perm, h.p.perm, m * 4, cudaMemcpyDeviceToHost, s));
    CU_TRY(cudaStreamSynchronize(s));
    if (rank) *rank = rk;
    size_t ncs = 0;
    for (size_t i = 0; i < rk; ++i) {
        if (swaps) swaps[i] = sw[i];
        if (q) q[i] = qq[i];
        if (qq[i] != i) {
            if (col_swaps) col_swaps[ncs] = gf2cu_colswap{i, (size_t)qq[i], i};
            ++ncs;
        }
    }
    if (n_col_swaps) *n_col_swaps = ncs;
    if (stats) {
        stats->steps = steps;
        double bytes = 0.0;
        for (size_t w = 0; w < steps; ++w) {
            if (rh[w] >= m || w + 1 >= W) continue;
            ++stats->trailing_launches;
            bytes += 16.0 * double(m - rh[w] - rbh[w]) * double(W - w - 1);
        }
        stats->alg_bytes = bytes;
        double sweep = bytes;
        if (super) {  // one read + write per two panels (as run_ple)
            sweep = 0.0;
            for (size_t w = 0; w + 2 < W && w < steps; w += 2) {
                if (rh[w] >= m) continue;
                const size_t rbb = (w + 1 < steps) ? rbh[w + 1] : 0;
                const size_t done = std::min(m, (size_t)rh[w] + rbh[w] + rbb);
                sweep += 16.0 * double(m - done) * double(W - w - 2);
            }
        }
        stats->sweep_bytes = sweep;
        stats->driver = super ? 4 : 3;
    }
    return GF2CU_OK;
}

// The row-sharded driver (ple_peer.cuh) with G ranks emulated on this
// matrix's device: one cooperative launch, sms/G CTAs per rank, every rank's
// buffers in this device's memory (the peers' stores are ordinary stores).
// Same outputs as run_ple.
gf2cu_status run_ple_peer(gf2cu_matrix* a, const gf2cu_cfg* cfg, unsigned G, size_t* swaps,
                          size_t* q, size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                          gf2cu_stats* stats) {
    const size_t m = a->m, n = a->n, W = a->W;
    // 256-row blocks; small matrices get smaller ones so that every rank
    // owns rows (the result does not depend on the distribution)
    unsigned block = (unsigned)std::max<size_t>(1, std::min<size_t>(256, m / (2 * (size_t)std::max(1u, G))));
    if (const char* e = std::getenv("GF2CU_PEER_BLOCK")) block = (unsigned)std::max(1, std::atoi(e));
    cudaStream_t s = pick_stream(a, cfg ? cfg->stream : nullptr);
    const bool timing = cfg && (cfg->flags & GF2CU_FLAG_TIME_KERNELS);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (m == 0 || n == 0) {
        *rank = 0;
        if (n_col_swaps) *n_col_swaps = 0;
        return GF2CU_OK;
    }
    const int sms = num_sms(a->device);
    if (G < 1 || G > (unsigned)gf2cu::kMaxRanks || (unsigned)sms / G < 2)
        return fail(GF2CU_EINVAL, "peer driver: 1..8 ranks, at least 2 CTAs each");
    PeerWs& pw = a->pw;
    if (!pw.dp || pw.G != G || pw.block != block) {
        // all-or-nothing: (G, block) are recorded only once every buffer is
        // allocated, so a failed setup is retried by the next call
        free_peer(pw);
        const auto setup = [&]() -> gf2cu_status {
            pw.hp.assign(G, gf2cu::PeerParams{});
            for (unsigned k = 0; k < G; ++k) {
                void* xbuf = nullptr;
                gf2cu_status st = peer_alloc_rank(pw.hp[k], pw.allocs, m, n, k, G, block, &xbuf, &pw.sizes);
                if (st != GF2CU_OK) return st;
            }
            for (unsigned k = 0; k < G; ++k)
                for (unsigned j = 0; j < G; ++j) pw.hp[k].peer[j] = pw.hp[j].peer[j];
            gf2cu::PeerParams* dp = nullptr;
            CU_TRY(cudaMalloc(&dp, G * sizeof(gf2cu::PeerParams)));
            pw.dp = dp;
            CU_TRY(h2d_now(pw.dp, pw.hp.data(), G * sizeof(gf2cu::PeerParams)));
            return GF2CU_OK;
        };
        const gf2cu_status st = setup();
        if (st != GF2CU_OK) {
            free_peer(pw);
            return st;
        }
        pw.G = G;
        pw.block = block;
    }
    const bool super = peer_super(m, W, cfg ? cfg->flags : 0u);
    const u32 wpad = super ? (u32)std::max<size_t>(4, (W + 3) / 4 * 4) : (u32)wpad8(W);
    const bool checking = check_mode(cfg);
    u32* chk = nullptr;
    if (checking) {
        gf2cu_status cst = ensure_ws(a);
        if (cst != GF2CU_OK) return cst;
        chk = a->ws.check;
        cst = check_reset(chk, s);
        if (cst != GF2CU_OK) return cst;
    }
    if (pw.hp[0].p.Wpad8 != wpad || pw.hp[0].p.check != chk) {
        for (unsigned k = 0; k < G; ++k) {
            pw.hp[k].p.Wpad8 = wpad;
            pw.hp[k].p.check = chk;
        }
        CU_TRY(h2d_now(pw.dp, pw.hp.data(), G * sizeof(gf2cu::PeerParams)));
    }
    if (const int pb = poison_byte(); pb >= 0) {
        // every allocation of every rank (rows, records, replicated state,
        // exchange buffers); the counters are reset below
        for (size_t i = 0; i < pw.allocs.size() && i < pw.sizes.size(); ++i)
            CU_TRY(cudaMemsetAsync(pw.allocs[i], pb, pw.sizes[i], s));
    }
    for (unsigned k = 0; k < G; ++k) {
        gf2cu_status st = peer_reset_rank(pw.hp[k], s);
        if (st != GF2CU_OK) return st;
    }
    if (super)
        gf2cu::peer_tile4_kernel<<<dim3(sms * 4, G), 256, 0, s>>>(pw.dp, a->data, (u32)a->Wp);
    else
        gf2cu::peer_tile_kernel<<<dim3(sms * 4, G), 256, 0, s>>>(pw.dp, a->data, (u32)a->Wp);
    CU_TRY(cudaGetLastError());
    cudaEvent_t ev[2] = {nullptr, nullptr};
    if (timing) {
        CU_TRY(cudaEventCreate(&ev[0]));
        CU_TRY(cudaEventCreate(&ev[1]));
        CU_TRY(cudaEventRecord(ev[0], s));
    }
    gf2cu_status st = peer_launch(pw.dp, G, (unsigned)sms / G, W, super, a->device, s);
    if (st != GF2CU_OK) return st;
    if (timing) CU_TRY(cudaEventRecord(ev[1], s));
    if (super)
        gf2cu::peer_untile4_kernel<<<dim3(sms * 4, G), 256, 0, s>>>(pw.dp, a->data, (u32)a->Wp);
    else
        gf2cu::peer_untile_kernel<<<dim3(sms * 4, G), 256, 0, s>>>(pw.dp, a->data, (u32)a->Wp);
    CU_TRY(cudaGetLastError());
    CU_TRY(cudaStreamSynchronize(s));
    for (unsigned k = 1; k < G; ++k) {  // any rank's watchdog
        u32 c[gf2cu::kCtrWords];
        CU_TRY(cudaMemcpy(c, pw.hp[k].peer[k].ctr, sizeof(c), cudaMemcpyDeviceToHost));
        if (c[gf2cu::kCtrErr]) return fail(GF2CU_ECUDA, "row-sharded PLE kernel watchdog tripped");
    }
    st = peer_outputs(pw.hp[0], super, s, swaps, q, rank, col_swaps, n_col_swaps, nullptr, stats);
    if (st == GF2CU_OK && *rank == 0 && std::getenv("GF2CU_DEBUG_PEER")) {
        // diagnostics of a rank-0 outcome: every rank's step state, counters
        for (unsigned k = 0; k < G; ++k) {
            const gf2cu::PeerParams& h = pw.hp[k];
            u32 c[gf2cu::kCtrWords];
            gf2cu::SyncState sy{};
            gf2cu::StepState fin{};
            std::vector<u32> rh(W + 1), rbh(W + 1);
            cudaMemcpy(c, h.peer[k].ctr, sizeof(c), cudaMemcpyDeviceToHost);
            cudaMemcpy(&sy, h.p.sync, sizeof(sy), cudaMemcpyDeviceToHost);
            cudaMemcpy(&fin, h.p.state, sizeof(fin), cudaMemcpyDeviceToHost);
            cudaMemcpy(rh.data(), h.p.rhist, (W + 1) * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(rbh.data(), h.p.rbhist, (W + 1) * 4, cudaMemcpyDeviceToHost);
            std::fprintf(stderr, "PEERDBG %zux%zu G=%u block=%u super=%d rank %u: state {%u,%u} panel_done %u cap %u t %u err %u ctr",
                         m, n, G, block, (int)super, k, fin.r, fin.rb, sy.panel_done, sy.cap_count, sy.t_count, sy.error);
            for (int i = 0; i < gf2cu::kCtrWords; ++i) std::fprintf(stderr, " %u", c[i]);
            std::fprintf(stderr, " rhist");
            for (size_t w = 0; w < W; ++w) std::fprintf(stderr, " %u/%u", rh[w], rbh[w]);
            std::fprintf(stderr, "\n");
        }
    }
    if (st == GF2CU_OK && checking) st = check_verdict(a, chk, *rank, sms, s);
    if (st == GF2CU_OK && stats && timing) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[0], ev[1]);
        stats->kernel_ms = ms;
    }
    if (timing) {
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
    }
    return st;
}

// Streamed input: the factorization starts on the first row block while the
// others are still crossing PCIe (ple_super.cuh, SuperRange). The rows arrive
// in K blocks with boundaries rows[0] < ... < rows[K-1] = m; steps[k] = the
// number of super-steps already done when block k joins (steps[0] = 0):
//   A_k  super-steps [steps[k], steps[k+1]) on the rows [0, rows[k]), k < K-1
//   B_k  the rows [rows[k-1], rows[k]) replay the super-steps [0, steps[k])
//   C    super-steps [steps[K-1], nss) on all rows
// in the order A_0, B_1, A_1, ..., B_{K-1}, C. The blocks grow geometrically,
// so the first one is there after a fraction of a millisecond and a late block
// replays few super-steps; steps[] comes from a time model (A_k runs until
// block k+1 is expected) -- a wrong estimate only costs idle time or a longer
// replay, never correctness. Empty plan: the matrix is uploaded whole.
//   GF2CU_STREAM_IN=0 never, =1 whenever the shape allows it (tests; every A_k
//   then runs as many super-steps as its rows allow); default: from 2^24 matrix
//   words (128 MiB, 2.4 ms of upload) up.
//   GF2CU_STREAM_IN_BLOCKS=f0,f1,..: the blocks' cumulative shares of the rows
//   (default 1/16, 3/16, 7/16); GF2CU_STREAM_IN_FRAC=f: one first block of that
//   share; GF2CU_STREAM_IN_STEPS=T1,T2,..: steps[1..] instead of the model's.
struct StreamInPlan {
    std::vector<size_t> rows;
    std::vector<u32> steps;
    size_t m0() const { return rows.empty() ? 0 : rows[0]; }
};

std::vector<double> env_list(const char* name) {
    std::vector<double> v;
    if (const char* e = std::getenv(name)) {
        const char* c = e;
        while (*c) {
            char* end = nullptr;
            const double x = std::strtod(c, &end);
            if (end == c) break;
            v.push_back(x);
            c = end;
            while (*c == ',' || *c == ' ') ++c;
        }
    }
    return v;
}

bool sparse_rule_on() {
    const char* e = std::getenv("GF2CU_SPARSE_RULE");
    return !(e && std::atoi(e) == 0);
}

StreamInPlan stream_in_plan(size_t m, size_t W, bool pageable) {
    StreamInPlan pl;
    const char* e = std::getenv("GF2CU_STREAM_IN");
    const int mode = e ? std::atoi(e) : -1;
    if (mode == 0) return pl;
    if (mode < 0 && (double)m * (double)W < 16777216.0) return pl;
    std::vector<double> fr = env_list("GF2CU_STREAM_IN_BLOCKS");
    if (fr.empty()) {
        if (const char* fe = std::getenv("GF2CU_STREAM_IN_FRAC"))
            fr = {std::atof(fe)};
        else
            fr = {1.0 / 16, 3.0 / 16, 7.0 / 16};
    }
    if (fr.size() > 7) fr.resize(7);  // (Workspace::up_ev)
    const size_t nss = (W + 1) / 2;
    // every super-step on a block keeps a full window and a full next window
    // among its rows: at most (rows - 256) / 128 super-steps, and blocks past
    // the last super-step's window add nothing
    const size_t cap = 128 * (nss - 1) + 256;
    std::vector<size_t> rows;
    for (double f : fr) {
        f = std::min(0.9, std::max(0.01, f));
        size_t b = std::min(((size_t)(f * (double)m) + 255) / 256 * 256, cap);
        b = std::max<size_t>(b, 512);
        if (b + 256 > m) break;
        if (!rows.empty() && b <= rows.back()) continue;
        rows.push_back(b);
    }
    if (rows.empty()) return pl;
    rows.push_back(m);
    const size_t K = rows.size();
    auto limit = [&](size_t k) { return (u32)std::min((rows[k] - 256) / 128, nss - 1); };
    std::vector<u32> steps(K, 0u);
    const std::vector<double> ts = env_list("GF2CU_STREAM_IN_STEPS");
    if (!ts.empty() || mode > 0) {
        for (size_t k = 1; k < K; ++k) {
            const u32 want = k - 1 < ts.size() ? (u32)std::max(0.0, ts[k - 1]) : 0xffffffffu;
            steps[k] = std::max(steps[k - 1], std::min(want, limit(k - 1)));
        }
    } else {
        // time model (ms): PCIe delivers `rate` bytes per ms; a super-step S
        // on R rows sweeps R * (W - 2S) words at `cw` ms per word plus a fixed
        // cost (panel chain and step barrier; the replay has no panel chain)
        const double rate = pageable ? 47e6 : 53e6, cw = 5.0e-9, fix_a = 0.018, fix_b = 0.012;
        auto arrive = [&](size_t k) { return 0.05 + (double)rows[k] * (double)W * 8.0 / rate; };
        double t = arrive(0) + 0.05;
        u32 T = 0;
        for (size_t k = 0; k + 1 < K; ++k) {
            const u32 lim = limit(k);
            while (T < lim && t < arrive(k + 1)) {
                t += cw * (double)rows[k] * (double)(W - 2 * T) + fix_a;
                ++T;
            }
            steps[k + 1] = T;
            t = std::max(t, arrive(k + 1)) + 0.05;
            for (u32 s2 = 0; s2 < T; ++s2) t += cw * (double)(rows[k + 1] - rows[k]) * (double)(W - 2 * s2) + fix_b;
        }
    }
    if (steps.back() < (mode > 0 ? 1u : 8u)) return pl;
    pl.rows = std::move(rows);
    pl.steps = std::move(steps);
    return pl;
}

// Launches the whole decomposition on `s`; outputs are copied to the host.
// stream_to (an aligned host view of the matrix, may be null): with the
// super-step driver, the rows the kernel finishes are copied into it while
// the factorization runs; *rows_streamed = how many leading rows already
// hold their final value there (the caller downloads the rest).
// stream_from (an aligned host view, may be null): the input is still on the
// host; this call uploads it -- in two row blocks with the factorization
// started on the first one when the shape is worth it (StreamInPlan).
gf2cu_status run_ple(gf2cu_matrix* a, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                     size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                     gf2cu_stats* stats, const gf2cu_view* stream_to = nullptr,
                     size_t* rows_streamed = nullptr, const gf2cu_view* stream_from = nullptr) {
    if (rows_streamed) *rows_streamed = 0;
    cudaStream_t s = pick_stream(a, cfg ? cfg->stream : nullptr);
    // (rows [lo, hi) of stream_from into the row-major device matrix)
    auto upload_rows = [&](size_t lo, size_t hi, cudaStream_t on) -> gf2cu_status {
        const uint64_t* host = stream_from->data + (stream_from->col_off >> 6);
        return staged_h2d(a->data + lo * a->Wp, a->Wp * 8, host + lo * stream_from->stride,
                          stream_from->stride * 8, a->W * 8, hi - lo, a->device, on);
    };
    if (const unsigned pr = cfg ? (cfg->flags >> 16) & 15u : 0u) {
        if (stream_from) {
            const gf2cu_status su = upload_rows(0, a->m, s);
            if (su != GF2CU_OK) return su;
        }
        return run_ple_peer(a, cfg, pr, swaps, q, rank, col_swaps, n_col_swaps, stats);
    }
    gf2cu_status st = ensure_ws(a);
    if (st != GF2CU_OK) return st;
    Workspace& ws = a->ws;
    const bool timing = cfg && (cfg->flags & GF2CU_FLAG_TIME_KERNELS);
    const size_t m = a->m, n = a->n, W = a->W;

    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
    }
    if (m == 0 || n == 0) {
        *rank = 0;
        if (n_col_swaps) *n_col_swaps = 0;
        return GF2CU_OK;
    }

    gf2cu::Params p{};
    if (!a->alt) {  // (assigned only on success: a failed call leaves it null)
        u64* alt = nullptr;
        CU_TRY(cudaMalloc(&alt, std::max<size_t>(1, m) * wpad8(W) * sizeof(u64)));
        a->alt = alt;
    }
    p.mat = a->alt;
    p.perm = ws.perm;
    p.pb = ws.pb;
    p.pb2 = (cfg && (cfg->flags & GF2CU_FLAG_MULTI_KERNEL)) ? nullptr : ws.pb2;
    p.info = ws.info;
    p.stage = ws.stage;
    p.state = ws.state;
    p.pout = ws.pout;
    p.swaps = ws.swaps;
    p.qcol = ws.qcol;
    p.rhist = ws.rhist;
    p.rbhist = ws.rbhist;
    // (only the one-launch-per-phase driver's host loop polls the mapped r;
    // the persistent drivers skip the per-panel system-scope fence)
    p.host_r = (cfg && (cfg->flags & GF2CU_FLAG_MULTI_KERNEL)) ? ws.host_r_dev : nullptr;
    p.sync = ws.sync;
    p.phase_ns = timing ? ws.phase_ns : nullptr;
    p.m = (u32)m;
    p.n = (u32)n;
    p.W = (u32)W;
    p.Wpad8 = (u32)wpad8(W);
    p.pflags = panel_flags();
    const bool checking = check_mode(cfg);
    if (checking) {
        p.check = ws.check;
        p.check_inject = check_inject_env();
        st = check_reset(ws.check, pick_stream(a, cfg ? cfg->stream : nullptr));
        if (st != GF2CU_OK) return st;
    }

    static bool attr_set[64] = {false};
    if (a->device >= 0 && a->device < 64 && !attr_set[a->device]) {
        CU_TRY(cudaFuncSetAttribute(gf2cu::trailing_update_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    gf2cu::kTableBytes));
        CU_TRY(cudaFuncSetAttribute(gf2cu::ple_persistent_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    gf2cu::kTableBytes));
        CU_TRY(cudaFuncSetAttribute(gf2cu::ple_super_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    gf2cu::kTableBytes));
        attr_set[a->device] = true;
    }
    const int sms = num_sms(a->device);
    const int apply_grid = sms * 4;
    const bool multi = cfg && (cfg->flags & GF2CU_FLAG_MULTI_KERNEL);
    // Two panels per sweep halve the sweep's global traffic and the per-step
    // synchronization, but the panel CTA's chain per super-step is longer:
    // it pays from ~2^24 matrix words up (measured crossover near 32768^2).
    const unsigned fl = cfg ? cfg->flags : 0u;
    bool super = !multi && !(fl & GF2CU_FLAG_SINGLE_PANEL) &&
                 ((fl & GF2CU_FLAG_SUPER_STEP) || (double)m * (double)W >= kSuperStepWords);
    // Sparse inputs are bound by window misses, not by the sweep, and a miss
    // costs the two-panel driver more (panel b's scan reduces every row by
    // panel a first): 32768^2 at p = 1/1024 takes 54 ms with it and 38 ms with
    // the single-panel driver; at p = 1/256 they tie. Below a sampled density
    // of 1/384 the size rule's choice falls back to the single-panel driver
    // (one word per row sampled; a forced driver is left alone;
    // GF2CU_SPARSE_RULE=0 turns the rule off).
    if (super && !(fl & GF2CU_FLAG_SUPER_STEP) && sparse_rule_on()) {
        double ones = 0.0;
        if (stream_from) {
            const uint64_t* host = stream_from->data + (stream_from->col_off >> 6);
            // (2048 evenly spaced rows: the cache misses of more would show in e2e)
            const size_t ns = std::min<size_t>(m, 2048), step = m / ns;
            for (size_t k = 0; k < ns; ++k) {
                const size_t i = k * step;
                ones += (double)__builtin_popcountll(host[i * stream_from->stride + ((u32)i * 0x9e3779b1u) % W]);
            }
            ones *= (double)m / (double)ns;
        } else {
            u32 cnt = 0;
            CU_TRY(cudaMemsetAsync(ws.rhist, 0, sizeof(u32), s));
            gf2cu::density_sample_kernel<<<sms, 256, 0, s>>>(a->data, (u32)m, (u32)W, (u32)a->Wp, ws.rhist);
            CU_TRY(cudaMemcpyAsync(&cnt, ws.rhist, sizeof(u32), cudaMemcpyDeviceToHost, s));
            CU_TRY(cudaStreamSynchronize(s));
            ones = (double)cnt;
        }
        if (ones < (double)m * 64.0 / 384.0) super = false;
    }
    const u32 Wpad4 = (u32)std::max<size_t>(4, (W + 3) / 4 * 4);
    StreamInPlan sin;
    if (stream_from && super && !timing)
        sin = stream_in_plan(m, W, host_pageable(stream_from->data + (stream_from->col_off >> 6)));
    if (stream_from && !sin.m0()) {
        st = upload_rows(0, m, s);
        if (st != GF2CU_OK) return st;
        trace_gpu("uploaded whole", s);
    }
    if (sin.m0()) {
        const size_t nss = (W + 1) / 2;
        if (!ws.up) CU_TRY(cudaStreamCreateWithFlags(&ws.up, cudaStreamNonBlocking));
        for (cudaEvent_t& e : ws.up_ev)
            if (!e) CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        if (!ws.hist_a) CU_TRY(cudaMalloc(&ws.hist_a, nss * sizeof(gf2cu::PanelOut)));
        if (!ws.hist_b) CU_TRY(cudaMalloc(&ws.hist_b, nss * sizeof(gf2cu::PanelOut)));
        if (!ws.hist_so) CU_TRY(cudaMalloc(&ws.hist_so, nss * sizeof(gf2cu::SuperOut)));
        if (!ws.sin_abort) CU_TRY(cudaMalloc(&ws.sin_abort, sizeof(u32)));
        // the first block starts on its way now; what was enqueued on s so
        // far (an earlier call's work on this matrix) stays ahead of it
        CU_TRY(cudaEventRecord(ws.up_ev[0], s));
        CU_TRY(cudaStreamWaitEvent(ws.up, ws.up_ev[0], 0));
        st = upload_rows(0, sin.m0(), ws.up);
        if (st != GF2CU_OK) return st;
        CU_TRY(cudaEventRecord(ws.up_ev[0], ws.up));
        trace_gpu("block 0 uploaded", ws.up);
    }
    if (!multi) {
        if (!ws.ubuf) {
            const size_t cap = std::max<size_t>(1, std::min(m, n));
            u64* ub = nullptr;
            CU_TRY(cudaMalloc(&ub, cap * p.Wpad8 * sizeof(u64)));
            ws.ubuf = ub;
            ws.ucap = cap;
        }
        p.ubuf = ws.ubuf;
        p.ucap = (u32)ws.ucap;
        if (!ws.apctr) {
            u32* ap = nullptr;
            CU_TRY(cudaMalloc(&ap, 2 * (W + 1) * sizeof(u32)));
            ws.apctr = ap;
        }
        p.ap_claim = ws.apctr;
        p.ap_done = ws.apctr + W + 1;
        const char* dv = std::getenv("GF2CU_PW_DIV");
        p.pw_div = dv ? (u32)std::max(64, std::atoi(dv)) : 8192u;
    }

    if (timing) {
        const size_t need = 6 * (W + 1) + 2;
        while (ws.ev.size() < need) {
            cudaEvent_t e;
            CU_TRY(cudaEventCreate(&e));
            ws.ev.push_back(e);
        }
    }

    *ws.host_r = 0;
    // (GF2CU_STREAM_OUT=0, diagnostic: download everything after the kernel)
    const char* so_env = std::getenv("GF2CU_STREAM_OUT");
    const bool streaming = super && stream_to && rows_streamed && !(so_env && std::atoi(so_env) == 0);
    if (streaming) {
        *reinterpret_cast<volatile u32*>(ws.out_host) = 0;
        p.out = a->data;
        p.out_Wp = (u32)a->Wp;
        p.out_host = ws.out_host_dev;
    }
    size_t sent = 0;
    if (const int pb = poison_byte(); pb >= 0) {
        const size_t mm = std::max<size_t>(1, m), mn = std::max<size_t>(1, std::min(m, n));
        CU_TRY(cudaMemsetAsync(a->alt, pb, mm * wpad8(W) * sizeof(u64), s));
        CU_TRY(cudaMemsetAsync(ws.pb, pb, mm * sizeof(u64), s));
        CU_TRY(cudaMemsetAsync(ws.pb2, pb, mm * sizeof(u64), s));
        CU_TRY(cudaMemsetAsync(ws.info, pb, 4 * mm * sizeof(ulonglong2), s));
        CU_TRY(cudaMemsetAsync(ws.stage, pb, 64 * wpad8(W) * sizeof(u64), s));
        CU_TRY(cudaMemsetAsync(ws.perm, pb, mm * sizeof(u32), s));
        CU_TRY(cudaMemsetAsync(ws.pout, pb, sizeof(gf2cu::PanelOut), s));
        CU_TRY(cudaMemsetAsync(ws.pout_b, pb, sizeof(gf2cu::PanelOut), s));
        CU_TRY(cudaMemsetAsync(ws.sout, pb, sizeof(gf2cu::SuperOut), s));
        CU_TRY(cudaMemsetAsync(ws.swaps, pb, mn * sizeof(u32), s));
        CU_TRY(cudaMemsetAsync(ws.qcol, pb, mn * sizeof(u32), s));
        CU_TRY(cudaMemsetAsync(ws.rhist, pb, (W + 1) * sizeof(u32), s));
        CU_TRY(cudaMemsetAsync(ws.rbhist, pb, (W + 1) * sizeof(u32), s));
        if (ws.ubuf) CU_TRY(cudaMemsetAsync(ws.ubuf, pb, ws.ucap * p.Wpad8 * sizeof(u64), s));
    }
    if (super) {
        p.Wpad8 = Wpad4;  // the super-step driver's tile width is 32 bytes
        if (sin.m0()) CU_TRY(cudaStreamWaitEvent(s, ws.up_ev[0], 0));
        const u32 hi = sin.m0() ? (u32)sin.m0() : (u32)m;
        gf2cu::tile4_kernel<<<sms * 8, 256, 0, s>>>(a->data, a->alt, (u32)m, (u32)a->Wp, Wpad4, 0u, hi);
        gf2cu::ple_init4_kernel<<<sms * 4, 256, 0, s>>>(p, a->data, (u32)a->Wp, 0u, hi);
    } else {
        gf2cu::tile_kernel<<<sms * 8, 256, 0, s>>>(a->data, a->alt, (u32)m, (u32)a->Wp, p.Wpad8);
        gf2cu::ple_init_kernel<<<sms * 4, 256, 0, s>>>(p);
    }
    CU_TRY(cudaGetLastError());

    size_t steps = 0;
    float kernel_ms = 0.f;
    if (!multi) {
        // ---- persistent cooperative driver: one launch for all panels ----
        CU_TRY(cudaMemsetAsync(ws.sync, 0, sizeof(gf2cu::SyncState), s));
        CU_TRY(cudaMemsetAsync(ws.apctr, 0, 2 * (W + 1) * sizeof(u32), s));
        if (timing) CU_TRY(cudaMemsetAsync(ws.phase_ns, 0, 8 * (W + 1) * sizeof(u64), s));
        int per_sm = 0;
        CU_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, gf2cu::ple_persistent_kernel, gf2cu::kTrailThreads, gf2cu::kTableBytes));
        if (per_sm < 1) return fail(GF2CU_ECUDA, "persistent kernel does not fit on an SM");
        const int grid = sms;  // one CTA per SM: CTA 0 panels, the rest update
        u32 nsteps = (u32)W;
        void* args[] = {&p, &nsteps};
        cudaEvent_t* E = timing ? &ws.ev[6 * (W + 1)] : nullptr;
        if (E) cudaEventRecord(E[0], s);
        // diagnostics: per-worker sweep stamps (GF2CU_DUMP_WORKERS=<path>)
        const char* wpath = timing ? std::getenv("GF2CU_DUMP_WORKERS") : nullptr;
        u64* wns = nullptr;
        const size_t wn_per = super ? 4 : 2;  // super: {wake, pre-work end, rest start, rest end}
        const size_t wn_words = ((size_t)W + 1) * (size_t)(grid - 1) * wn_per;
        if (wpath) {
            CU_TRY(cudaMalloc(&wns, wn_words * sizeof(u64)));
            CU_TRY(cudaMemsetAsync(wns, 0, wn_words * sizeof(u64), s));
        }
        p.worker_ns = wns;
        if (super) {
            const u32 nss = (u32)((W + 1) / 2);
            auto launch = [&](gf2cu::Params pp, gf2cu::PanelOut* pob, gf2cu::SuperOut* so,
                              gf2cu::SuperRange rg) -> cudaError_t {
                void* sargs[] = {&pp, &pob, &so, &rg};
                return cudaLaunchCooperativeKernel((void*)gf2cu::ple_super_kernel, dim3(grid),
                                                   dim3(gf2cu::kTrailThreads), sargs, gf2cu::kTableBytes, s);
            };
            if (!sin.m0()) {
                trace_gpu("kernel begins", s);
                CU_TRY(launch(p, ws.pout_b, ws.sout, gf2cu::SuperRange{0u, nss, 0u, 0u, 0u, nullptr}));
                trace_gpu("kernel ends", s);
            } else {
                // streamed input (StreamInPlan): A_0, then per later block k
                // its upload, B_k (its replay of the super-steps so far) and
                // A_k (the next super-steps on every row up to it; k = K-1:
                // all the remaining ones on all rows, with the streamed output)
                const u32 nwk = (u32)grid - 1u;
                const size_t K = sin.rows.size();
                CU_TRY(cudaMemsetAsync(ws.sin_abort, 0, sizeof(u32), s));
                gf2cu::Params pa = p;
                pa.pout = ws.hist_a;
                pa.out = nullptr;
                pa.out_host = nullptr;
                for (size_t k = 0; k < K; ++k) {
                    const bool last = k + 1 == K;
                    const u32 lo = k ? (u32)sin.rows[k - 1] : 0u, hi = (u32)sin.rows[k];
                    const u32 Tk = sin.steps[k], Tn = last ? nss : sin.steps[k + 1];
                    if (k) {
                        st = upload_rows(lo, hi, ws.up);
                        if (st != GF2CU_OK) return st;
                        CU_TRY(cudaEventRecord(ws.up_ev[k], ws.up));
                        trace_gpu("block " + std::to_string(k) + " uploaded", ws.up);
                        trace_gpu("stream ready for block " + std::to_string(k), s);
                        CU_TRY(cudaStreamWaitEvent(s, ws.up_ev[k], 0));
                        gf2cu::tile4_kernel<<<sms * 8, 256, 0, s>>>(a->data, a->alt, (u32)m, (u32)a->Wp, Wpad4, lo, hi);
                        gf2cu::ple_init4_kernel<<<sms * 4, 256, 0, s>>>(p, a->data, (u32)a->Wp, lo, hi);
                        if (Tk) {
                            CU_TRY(cudaMemsetAsync(ws.apctr, 0, 2 * (W + 1) * sizeof(u32), s));
                            gf2cu::sync_preset_kernel<<<1, 1, 0, s>>>(ws.sync, Tk, 0u, 0u, ws.sin_abort);
                            gf2cu::Params pB = pa;
                            pB.mv = last ? 0u : hi;
                            trace_gpu("B" + std::to_string(k) + " begins (" + std::to_string(Tk) + " super-steps)", s);
                            CU_TRY(launch(pB, ws.hist_b, ws.hist_so, gf2cu::SuperRange{0u, Tk, lo, 1u, 1u, ws.sin_abort}));
                            trace_gpu("B" + std::to_string(k) + " ends", s);
                        }
                    }
                    if (Tn == Tk) continue;
                    u32 out_count = 0;
                    if (last) {
                        // (the first output batch of C: the first multiple of kOutEvery >= steps[K-1])
                        const u32 sf = std::max(gf2cu::kOutEvery, (Tk + gf2cu::kOutEvery - 1) / gf2cu::kOutEvery * gf2cu::kOutEvery);
                        out_count = nwk * (sf / gf2cu::kOutEvery - 1u);
                    }
                    if (k) {
                        CU_TRY(cudaMemsetAsync(ws.apctr, 0, 2 * (W + 1) * sizeof(u32), s));
                        gf2cu::sync_preset_kernel<<<1, 1, 0, s>>>(ws.sync, Tk, nwk * Tk, out_count, ws.sin_abort);
                    }
                    gf2cu::Params pA = last ? p : pa;
                    pA.pout = ws.hist_a;
                    if (!last) {
                        pA.mv = hi;
                        pA.partial = 1u;
                    }
                    trace_gpu("A" + std::to_string(k) + " begins [" + std::to_string(Tk) + ", " + std::to_string(Tn) + ")", s);
                    CU_TRY(launch(pA, ws.hist_b, ws.hist_so, gf2cu::SuperRange{Tk, Tn, 0u, 0u, 1u, ws.sin_abort}));
                    trace_gpu("A" + std::to_string(k) + " ends", s);
                }
                CU_TRY(cudaGetLastError());
            }
        } else {
            CU_TRY(cudaLaunchCooperativeKernel((void*)gf2cu::ple_persistent_kernel, dim3(grid),
                                               dim3(gf2cu::kTrailThreads), args, gf2cu::kTableBytes, s));
        }
        if (E) cudaEventRecord(E[1], s);
        if (streaming) {
            // copy the finished rows out while the kernel runs (copy engine,
            // second stream), in chunks of at least m/32 rows
            cudaEvent_t kdone;
            CU_TRY(cudaEventCreateWithFlags(&kdone, cudaEventDisableTiming));
            CU_TRY(cudaEventRecord(kdone, s));
            // (chunks shrink toward the end, where the late super-steps finish
            // few rows each, so that little is left to copy after the kernel)
            uint64_t* host = stream_to->data + (stream_to->col_off >> 6);
            const bool pageable = host_pageable(host);
            for (;;) {
                const cudaError_t qe = cudaEventQuery(kdone);
                if (qe != cudaSuccess && qe != cudaErrorNotReady) {
                    // a faulted kernel never completes the event: fail
                    // instead of polling the row count forever
                    cudaEventDestroy(kdone);
                    return cuda_fail(qe, "persistent PLE kernel (streamed output)");
                }
                const bool fin = qe == cudaSuccess;
                const size_t avail = *reinterpret_cast<volatile u32*>(ws.out_host);
                const size_t chunk = std::max<size_t>(256, std::min<size_t>(m / 32, (m - sent) / 8));
                if (avail > sent && (avail - sent >= chunk || fin)) {
                    if (pageable) {  // (synchronous; the kernel goes on meanwhile)
                        st = staged_d2h(host + sent * stream_to->stride, stream_to->stride * 8,
                                        a->data + sent * a->Wp, a->Wp * 8, W * 8, avail - sent, a->device, ws.copy);
                        if (st != GF2CU_OK) {
                            cudaEventDestroy(kdone);
                            return st;
                        }
                    } else {
                        CU_TRY(cudaMemcpy2DAsync(host + sent * stream_to->stride, stream_to->stride * 8,
                                                 a->data + sent * a->Wp, a->Wp * 8, W * 8, avail - sent,
                                                 cudaMemcpyDeviceToHost, ws.copy));
                    }
                    sent = avail;
                    if (g_trace.on) trace_host(("streamed rows up to " + std::to_string(sent) + (fin ? " (kernel finished)" : "")).c_str());
                }
                if (fin) break;
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
            cudaEventDestroy(kdone);
            trace_host("kernel seen finished");
            CU_TRY(cudaStreamSynchronize(ws.copy));
            trace_host("streamed copies done");
        }
        gf2cu::SyncState sy{};
        u32 gave_up = 0;
        CU_TRY(cudaMemcpyAsync(&sy, ws.sync, sizeof(sy), cudaMemcpyDeviceToHost, s));
        if (sin.m0()) CU_TRY(cudaMemcpyAsync(&gave_up, ws.sin_abort, sizeof(u32), cudaMemcpyDeviceToHost, s));
        CU_TRY(cudaStreamSynchronize(s));
        if (gave_up == 2u) return fail(GF2CU_ECUDA, "persistent PLE kernel watchdog tripped (streamed input)");
        if (gave_up) {
            // a column had no pivot among the first block's rows: the whole
            // matrix decides. Nothing was written to a->data or to the host
            // view (the first phases produce no output), and the upload is
            // complete: factor it the ordinary way.
            return run_ple(a, cfg, swaps, q, rank, col_swaps, n_col_swaps, stats, stream_to, rows_streamed, nullptr);
        }
        if (wns) {
            std::vector<u64> h(wn_words);
            cudaMemcpy(h.data(), wns, wn_words * sizeof(u64), cudaMemcpyDeviceToHost);
            cudaFree(wns);
            if (FILE* f = std::fopen(wpath, "wb")) {
                const u64 hdr[3] = {(u64)W, (u64)(grid - 1), (u64)wn_per};
                std::fwrite(hdr, sizeof(u64), super ? 3 : 2, f);
                std::fwrite(h.data(), sizeof(u64), h.size(), f);
                std::fclose(f);
            }
        }
        if (sy.error) return fail(GF2CU_ECUDA, "persistent PLE kernel watchdog tripped");
        steps = super ? std::min<size_t>(W, 2 * (size_t)sy.panel_done) : sy.panel_done;
        if (E) cudaEventElapsedTime(&kernel_ms, E[0], E[1]);
    } else {
        // ---- one launch per phase ----
        // Host stays at most kLag steps ahead of the device so that it notices
        // r == m early (wide matrices) without stalling the stream.
        constexpr size_t kLag = 6;
        std::vector<cudaEvent_t> step_ev(kLag, nullptr);
        for (auto& e : step_ev) CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (size_t w = 0; w < W; ++w) {
            if (w >= kLag) {
                CU_TRY(cudaEventSynchronize(step_ev[w % kLag]));
                if (*reinterpret_cast<volatile u32*>(ws.host_r) >= m) break;
            }
            cudaEvent_t* E = timing ? &ws.ev[6 * w] : nullptr;
            if (E) cudaEventRecord(E[0], s);
            gf2cu::panel_factor_kernel<<<1, gf2cu::kPanelThreads, 0, s>>>(p, (u32)w);
            if (E) cudaEventRecord(E[1], s);
            if (E) cudaEventRecord(E[2], s);
            gf2cu::panel_apply_kernel<<<apply_grid, gf2cu::kApplyThreads, 0, s>>>(p, (u32)w);
            if (E) cudaEventRecord(E[3], s);
            if (w + 1 < W) {
                if (E) cudaEventRecord(E[4], s);
                gf2cu::trailing_update_kernel<<<sms, gf2cu::kTrailThreads, gf2cu::kTableBytes, s>>>(
                    p, (u32)w);
                if (E) cudaEventRecord(E[5], s);
            }
            CU_TRY(cudaGetLastError());
            CU_TRY(cudaEventRecord(step_ev[w % kLag], s));
            ++steps;
        }
        for (auto& e : step_ev) cudaEventDestroy(e);
    }

    // rank and histories
    gf2cu::StepState fin{};
    CU_TRY(cudaMemcpyAsync(&fin, ws.state, sizeof(fin), cudaMemcpyDeviceToHost, s));
    std::vector<u32> rh(steps), rbh(steps);
    if (steps) {
        CU_TRY(cudaMemcpyAsync(rh.data(), ws.rhist, steps * sizeof(u32), cudaMemcpyDeviceToHost, s));
        CU_TRY(cudaMemcpyAsync(rbh.data(), ws.rbhist, steps * sizeof(u32), cudaMemcpyDeviceToHost, s));
    }
    CU_TRY(cudaStreamSynchronize(s));
    const size_t rk = std::min<size_t>((size_t)fin.r + fin.rb, std::min(m, n));

    // swaps / q to pinned staging first (they do not depend on the untile)
    if (rk && !ws.h_out) {
        u32* ho = nullptr;
        CU_TRY(cudaMallocHost(&ho, 2 * std::min(m, n) * sizeof(u32)));
        ws.h_out = ho;
    }
    u32* sw = ws.h_out;
    u32* qq = ws.h_out + std::min(m, n);
    if (rk) {
        CU_TRY(cudaMemcpyAsync(sw, ws.swaps, rk * sizeof(u32), cudaMemcpyDeviceToHost, s));
        CU_TRY(cudaMemcpyAsync(qq, ws.qcol, rk * sizeof(u32), cudaMemcpyDeviceToHost, s));
    }
    // back to the row-major public layout, rows gathered into position order
    if (super) {
        gf2cu::untile4_kernel<<<sms * 8, 256, 0, s>>>(a->alt, a->data, ws.perm, (u32)m, (u32)a->Wp,
                                                     Wpad4, p.ubuf, p.ucap, ws.qcol, (u32)rk, (u32)W,
                                                     (u32)sent);
    } else {
        gf2cu::untile_kernel<<<sms * 8, 256, 0, s>>>(a->alt, a->data, ws.perm, (u32)m, (u32)a->Wp,
                                                    p.Wpad8, p.ubuf, p.ucap, ws.qcol, (u32)rk, (u32)W);
    }
    CU_TRY(cudaGetLastError());
    if (rows_streamed) *rows_streamed = sent;
    trace_gpu("untile done", s);

    CU_TRY(cudaStreamSynchronize(s));
    trace_host("run_ple synchronized");
    if (checking) {
        st = check_verdict(a, ws.check, rk, sms, s);
        if (st != GF2CU_OK) return st;
    }
    *rank = rk;
    size_t ncs = 0;
    for (size_t i = 0; i < rk; ++i) {
        swaps[i] = sw[i];
        q[i] = qq[i];
        if (qq[i] != i) {
            if (col_swaps) col_swaps[ncs] = gf2cu_colswap{i, (size_t)qq[i], i};
            ++ncs;
        }
    }
    if (n_col_swaps) *n_col_swaps = ncs;

    if (stats) {
        stats->steps = steps;
        double bytes = 0.0;
        size_t launches = 0;
        for (size_t w = 0; w < steps; ++w) {
            const size_t r0 = rh[w], rb = rbh[w];
            if (r0 >= m || w + 1 >= W) continue;
            ++launches;
            bytes += 16.0 * double(m - r0 - rb) * double(W - w - 1);
        }
        stats->alg_bytes = bytes;
        double sweep = bytes;
        if (super) {
            sweep = 0.0;
            for (size_t w = 0; w + 2 < W && w < steps; w += 2) {
                const size_t r0 = rh[w];
                const size_t rbb = (w + 1 < steps) ? rbh[w + 1] : 0;
                if (r0 >= m) continue;
                const size_t done = std::min(m, r0 + rbh[w] + rbb);
                sweep += 16.0 * double(m - done) * double(W - w - 2);
            }
        }
        stats->sweep_bytes = sweep;
        stats->trailing_launches = launches;
        stats->kernel_ms = kernel_ms;
        stats->driver = multi ? 0 : super ? 2 : 1;
        stats->input_first_rows = sin.m0();
        stats->input_first_steps = sin.m0() ? sin.steps.back() : 0;
        stats->input_blocks = sin.rows.size();
        if (timing && !multi) {
            std::vector<u64> ph(8 * steps);
            CU_TRY(cudaMemcpy(ph.data(), ws.phase_ns, ph.size() * sizeof(u64), cudaMemcpyDeviceToHost));
            double tp = 0, tc = 0, tt = 0;
            for (size_t w = 0; w < steps; ++w) {
                const u64* x = &ph[8 * w];
                if (x[1] > x[0]) tp += (x[1] - x[0]) * 1e-6;
                if (x[3] > x[2]) tc += (x[3] - x[2]) * 1e-6;
                if (x[5] > x[3]) tt += (x[5] - x[3]) * 1e-6;
            }
            stats->panel_ms = tp;
            stats->coef_ms = tc;
            stats->trailing_ms = tt;
            if (const char* path = std::getenv("GF2CU_DUMP_PHASES")) {
                if (FILE* f = std::fopen(path, "w")) {
                    std::fprintf(f, "w r rb p0 p1 a0 t0 cap1 t1 pl0 pl1\n");
                    for (size_t w = 0; w < steps; ++w) {
                        const u64* x = &ph[8 * w];
                        std::fprintf(f, "%zu %u %u %llu %llu %llu %llu %llu %llu %llu %llu\n", w, rh[w],
                                     rbh[w], x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
                    }
                    std::vector<u64> dbg(64 * 5);
                    cudaMemcpy(dbg.data(), ws.phase_ns + 8 * W + 8, dbg.size() * 8, cudaMemcpyDeviceToHost);
                    for (int j = 0; j < 64; ++j)
                        std::fprintf(f, "# %d %llu %llu %llu %llu %llu\n", j, dbg[5 * j], dbg[5 * j + 1],
                                     dbg[5 * j + 2], dbg[5 * j + 3], dbg[5 * j + 4]);
                    std::fclose(f);
                }
            }
        }
        if (timing && multi) {
            double tp = 0, tc = 0, tt = 0;
            for (size_t w = 0; w < steps; ++w) {
                float ms = 0;
                cudaEventElapsedTime(&ms, ws.ev[6 * w], ws.ev[6 * w + 1]);
                tp += ms;
                cudaEventElapsedTime(&ms, ws.ev[6 * w + 2], ws.ev[6 * w + 3]);
                tc += ms;
                if (w + 1 < W) {
                    cudaEventElapsedTime(&ms, ws.ev[6 * w + 4], ws.ev[6 * w + 5]);
                    tt += ms;
                }
            }
            stats->panel_ms = tp;
            stats->coef_ms = tc;
            stats->trailing_ms = tt;
        }
    }
    return GF2CU_OK;
}

gf2cu_status check_verdict(gf2cu_matrix* a, u32* chk, size_t rank, int sms, cudaStream_t s) {
    gf2cu::check_final_kernel<<<sms * 4, 256, 0, s>>>(a->data, (u32)a->m, (u32)a->n, (u32)a->Wp, (u32)rank, chk);
    CU_TRY(cudaGetLastError());
    u32 h[4];
    CU_TRY(cudaMemcpyAsync(h, chk, sizeof(h), cudaMemcpyDeviceToHost, s));
    CU_TRY(cudaStreamSynchronize(s));
    if (h[1]) {
        char msg[160];
        std::snprintf(msg, sizeof(msg), "check mode: invariant (iv) violated at step %u (%u panel words)",
                      h[0], h[1]);
        return fail(GF2CU_ECHECK, msg);
    }
    if (h[3]) {
        char msg[160];
        std::snprintf(msg, sizeof(msg), "check mode: invariant (i)/(ii) violated at row %u (%u rows)", h[2],
                      h[3]);
        return fail(GF2CU_ECHECK, msg);
    }
    return GF2CU_OK;
}

// --- host-side view packing (col_off may be unaligned) ---------------------
u64 read_bits(const u64* row, size_t lo, size_t count) {
    const size_t w = lo >> 6, b = lo & 63;
    u64 v = row[w] >> b;
    if (b != 0 && b + count > 64) v |= row[w + 1] << (64 - b);
    return count >= 64 ? v : (v & ((1ull << count) - 1ull));
}

void write_bits(u64* row, size_t lo, size_t count, u64 bits) {
    const size_t w = lo >> 6, b = lo & 63;
    const u64 mask = count >= 64 ? ~0ull : ((1ull << count) - 1ull);
    bits &= mask;
    row[w] = (row[w] & ~(mask << b)) | (bits << b);
    if (b != 0 && b + count > 64) {
        const size_t spill = b + count - 64;
        const u64 m2 = (1ull << spill) - 1ull;
        row[w + 1] = (row[w + 1] & ~m2) | (bits >> (64 - b));
    }
}

// check_pivots (ple.hpp:299-307): q strictly increasing, inside the matrix.
gf2cu_status check_pivots(const size_t* q, size_t rank, size_t m, size_t n) {
    if (rank > std::min(m, n)) return fail(GF2CU_EINVAL, "rank exceeds the matrix dimensions");
    if (rank && !q) return fail(GF2CU_EINVAL, "null pivot list");
    for (size_t j = 0; j < rank; ++j)
        if (q[j] >= n || (j > 0 && q[j] <= q[j - 1]))
            return fail(GF2CU_EINVAL, "pivot columns are not strictly increasing");
    return GF2CU_OK;
}

// X = U^-1 N over the prepared RrefParams (U, N filled): bottom-up 64-row
// blocks, in-block solve then the Gray-table update of the rows above.
gf2cu_status solve_upper(gf2cu_matrix* a, const gf2cu::RrefParams& p, cudaStream_t s) {
    static bool attr_set[64] = {false};
    if (a->device >= 0 && a->device < 64 && !attr_set[a->device]) {
        CU_TRY(cudaFuncSetAttribute(gf2cu::rref_update_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, gf2cu::kTableBytes));
        CU_TRY(cudaFuncSetAttribute(gf2cu::rref_step_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, gf2cu::kTableBytes));
        attr_set[a->device] = true;
    }
    const int sms = num_sms(a->device);
    const u32 nblk = p.R / 64;
    const u32 ntiles = p.WnPad8 / 8;
    // the top block needs no update; then one launch per block J: X_J to the
    // rows above, block J-1 finished in the same launch
    gf2cu::rref_block_solve_kernel<<<(p.Wn + 7) / 8, 256, 0, s>>>(p, nblk - 1);
    for (u32 J = nblk - 1; J >= 1; --J) {
        const u64 units = (u64)ntiles * 64u * (J - 1u);
        const int upd = units ? (int)std::min<u64>((u64)sms, std::max<u64>(1, units / 256)) : 0;
        gf2cu::rref_step_kernel<<<ntiles + upd, gf2cu::kTrailThreads, gf2cu::kTableBytes, s>>>(p, J);
    }
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

// rref_from_ple (ple.hpp:318-329) on the device copy in place: a->data must
// hold the in-place PLE result whose pivot columns are q[0..rank).
gf2cu_status run_rref(gf2cu_matrix* a, const size_t* q, size_t rank, bool full, cudaStream_t s) {
    const size_t m = a->m, n = a->n, W = a->W;
    gf2cu_status st = check_pivots(q, rank, m, n);
    if (st != GF2CU_OK) return st;
    if (m == 0 || n == 0) return GF2CU_OK;
    RrefWs& rw = a->rw;
    const int sms = num_sms(a->device);
    const size_t r = rank, ncn = n - r;
    const size_t R = (r + 63) / 64 * 64, Wu = R / 64, Wn = (ncn + 63) / 64;
    const size_t WnPad8 = (Wn + 7) / 8 * 8;
    // host-side index arrays: q | np | usrc | nsrc | npos0, and npmask
    std::vector<u32> idx(r + ncn + Wu + Wn + W);
    std::vector<u64> npmask(W, 0ull);
    u32* hq = idx.data();
    u32* hnp = hq + r;
    u32* husrc = hnp + ncn;
    u32* hnsrc = husrc + Wu;
    u32* hnpos0 = hnsrc + Wn;
    {
        size_t j = 0, k = 0;
        for (size_t c = 0; c < n; ++c) {
            if (j < r && q[j] == c) {
                hq[j++] = (u32)c;
            } else {
                hnp[k++] = (u32)c;
                npmask[c >> 6] |= 1ull << (c & 63);
            }
        }
        size_t before = 0;
        for (size_t y = 0; y < W; ++y) {
            hnpos0[y] = (u32)before;
            before += (size_t)__builtin_popcountll(npmask[y]);
        }
        auto contiguous = [](const u32* cols, size_t k0, size_t cnt) -> u32 {
            return cols[k0 + cnt - 1] - cols[k0] == cnt - 1 ? cols[k0] : gf2cu::kNone;
        };
        for (size_t x = 0; x < Wu; ++x)
            husrc[x] = 64 * x < r ? contiguous(hq, 64 * x, std::min<size_t>(64, r - 64 * x)) : 0u;
        for (size_t x = 0; x < Wn; ++x) hnsrc[x] = contiguous(hnp, 64 * x, std::min<size_t>(64, ncn - 64 * x));
    }
    CU_TRY(grow(&rw.idx, &rw.idx_words, idx.size()));
    CU_TRY(grow(&rw.npmask, &rw.npmask_words, W));
    CU_TRY(cudaMemcpyAsync(rw.idx, idx.data(), idx.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
    CU_TRY(cudaMemcpyAsync(rw.npmask, npmask.data(), W * sizeof(u64), cudaMemcpyHostToDevice, s));
    const u32* dq = rw.idx;
    if (!full) {
        gf2cu::rref_echelon_kernel<<<sms * 8, 256, 0, s>>>(a->data, dq, (u32)m, (u32)W, (u32)a->Wp, (u32)r);
        CU_TRY(cudaGetLastError());
        return GF2CU_OK;
    }
    gf2cu::RrefParams p{};
    p.a = a->data;
    p.out = a->data;
    p.q = dq;
    p.np = dq + r;
    p.usrc = dq + r + ncn;
    p.nsrc = p.usrc + Wu;
    p.npos0 = p.nsrc + Wn;
    p.npmask = rw.npmask;
    p.m = (u32)m;
    p.n = (u32)n;
    p.W = (u32)W;
    p.Wp = (u32)a->Wp;
    p.Wa = (u32)W;
    p.Wpa = (u32)a->Wp;
    p.r = (u32)r;
    p.R = (u32)R;
    p.Wu = (u32)Wu;
    p.Wn = (u32)Wn;
    p.WnPad8 = (u32)WnPad8;
    p.ncn = (u32)ncn;
    if (r > 0 && ncn > 0) {
        CU_TRY(grow(&rw.U, &rw.U_words, Wu * R));
        CU_TRY(grow(&rw.N, &rw.N_words, WnPad8 * R));
        CU_TRY(cudaMemsetAsync(rw.U, 0, Wu * R * sizeof(u64), s));
        CU_TRY(cudaMemsetAsync(rw.N, 0, WnPad8 * R * sizeof(u64), s));
        p.U = rw.U;
        p.N = rw.N;
        gf2cu::rref_gather_kernel<<<sms * 8, 256, 0, s>>>(p, 1);
        CU_TRY(cudaGetLastError());
        st = solve_upper(a, p, s);
        if (st != GF2CU_OK) return st;
    }
    gf2cu::rref_scatter_kernel<<<sms * 8, 256, 0, s>>>(p);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

// Per-thread cached device matrices (slot 0: the in-place operand of the
// host-view entry points; 1, 2: read-only product operands). Repeated calls
// on the same shapes reuse HBM buffers and workspace instead of re-allocating.
gf2cu_status cached_matrix(int slot, size_t m, size_t n, int device, gf2cu_matrix** out) {
    struct Cache {
        gf2cu_matrix* a[3] = {nullptr, nullptr, nullptr};
        ~Cache() {
            for (gf2cu_matrix* x : a) gf2cu_matrix_destroy(x);
        }
    };
    thread_local Cache cache;
    gf2cu_matrix*& a = cache.a[slot];
    if (a && (a->m != m || a->n != n || a->device != device)) {
        gf2cu_matrix_destroy(a);
        a = nullptr;
    }
    if (!a) {
        gf2cu_status st = gf2cu_matrix_create(m, n, device, &a);
        if (st != GF2CU_OK) return st;
    }
    *out = a;
    return GF2CU_OK;
}

bool view_aligned(const gf2cu_view* v) { return (v->col_off & 63) == 0 && (v->ncols & 63) == 0; }

// Host window -> device rows (unaligned windows packed host-side into `packed`).
gf2cu_status view_upload(const gf2cu_view* v, gf2cu_matrix* a, cudaStream_t s,
                         std::vector<u64>& packed) {
    const size_t m = v->nrows, n = v->ncols, W = a->W;
    if (m == 0 || W == 0) return GF2CU_OK;
    cudaError_t e;
    if (view_aligned(v)) {
        return staged_h2d(a->data, a->Wp * 8, v->data + (v->col_off >> 6), v->stride * 8, W * 8, m, a->device, s);
    } else {
        packed.assign(m * W, 0ull);
        for (size_t i = 0; i < m; ++i) {
            const u64* row = reinterpret_cast<const u64*>(v->data) + i * v->stride;
            for (size_t x = 0; x < W; ++x)
                packed[i * W + x] = read_bits(row, v->col_off + 64 * x, std::min<size_t>(64, n - 64 * x));
        }
        e = cudaMemcpy2DAsync(a->data, a->Wp * 8, packed.data(), W * 8, W * 8, m,
                              cudaMemcpyHostToDevice, s);
    }
    return e == cudaSuccess ? GF2CU_OK : cuda_fail(e, "upload");
}

// Device rows -> host window (bits outside the window untouched); synchronous.
gf2cu_status view_download(const gf2cu_view* v, const gf2cu_matrix* a, cudaStream_t s,
                           std::vector<u64>& packed, size_t row_lo = 0, size_t row_hi = ~size_t(0)) {
    const size_t m = std::min(v->nrows, row_hi), n = v->ncols, W = a->W;
    if (m == 0 || W == 0) return GF2CU_OK;
    cudaError_t e;
    if (view_aligned(v)) {
        if (row_lo >= m) return GF2CU_OK;
        return staged_d2h(v->data + (v->col_off >> 6) + row_lo * v->stride, v->stride * 8,
                          a->data + row_lo * a->Wp, a->Wp * 8, W * 8, m - row_lo, a->device, s);
    } else {
        packed.resize(m * W);
        e = cudaMemcpy2DAsync(packed.data(), W * 8, a->data, a->Wp * 8, W * 8, m,
                              cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess)
            for (size_t i = 0; i < m; ++i) {
                u64* row = reinterpret_cast<u64*>(v->data) + i * v->stride;
                for (size_t x = 0; x < W; ++x)
                    write_bits(row, v->col_off + 64 * x, std::min<size_t>(64, n - 64 * x), packed[i * W + x]);
            }
    }
    return e == cudaSuccess ? GF2CU_OK : cuda_fail(e, "download");
}

// Host view <-> the cached device matrix of its shape: upload,
// body(matrix, cfg), download.
// (body_uploads: the body copies the view's rows to the device itself)
template <class Body>
gf2cu_status with_view(const gf2cu_view* v, const gf2cu_cfg* cfg, gf2cu_stats* stats, Body&& body,
                       size_t* rows_done = nullptr, const size_t* rows_limit = nullptr,
                       bool body_uploads = false) {
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    if (cfg) c = *cfg;
    gf2cu_matrix* a = nullptr;
    gf2cu_status st = cached_matrix(0, v->nrows, v->ncols, c.device, &a);
    if (st != GF2CU_OK) return st;
    DeviceGuard g(c.device);
    cudaStream_t s = pick_stream(a, c.stream);
    std::vector<u64> packed;
    trace_begin(s);
    if (!body_uploads) {
        st = view_upload(v, a, s, packed);
        if (st != GF2CU_OK) return st;
    }
    c.stream = s;
    st = body(a, c);
    trace_host("body done");
    if (st == GF2CU_OK) {
        st = view_download(v, a, s, packed, rows_done ? *rows_done : 0,
                           rows_limit ? *rows_limit : ~size_t(0));
        trace_host("download done");
        if (stats) {
            stats->h2d_bytes = double(a->m) * a->W * 8;
            stats->d2h_bytes = double(a->m) * a->W * 8;
        }
    }
    trace_end();
    return st;
}

// C (+)= A * B on device matrices (check_mul_shapes, multiply.hpp:33-37).
gf2cu_status run_mul(gf2cu_matrix* c, const gf2cu_matrix* a, const gf2cu_matrix* b, bool accumulate,
                     cudaStream_t s) {
    if (a->n != b->m || c->m != a->m || c->n != b->n)
        return fail(GF2CU_EINVAL, "multiply: dimension mismatch");
    if (c == a || c == b) return fail(GF2CU_EINVAL, "multiply: C aliases an operand");
    if (a->device != c->device || b->device != c->device)
        return fail(GF2CU_EINVAL, "multiply: operands on different devices");
    const size_t M = c->m, L = a->n, Wc = c->W;
    if (M == 0 || Wc == 0) return GF2CU_OK;
    static bool attr_set[64] = {false};
    if (c->device >= 0 && c->device < 64 && !attr_set[c->device]) {
        CU_TRY(cudaFuncSetAttribute(gf2cu::gemm_m4rm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    gf2cu::kTableBytes));
        attr_set[c->device] = true;
    }
    const int sms = num_sms(c->device);
    const size_t Lw = words_of(L);
    RrefWs& rw = c->rw;
    CU_TRY(grow(&rw.src, &rw.src_words, M * Lw));
    if (Lw) gf2cu::gemm_transpose_a_kernel<<<sms * 8, 256, 0, s>>>(a->data, rw.src, (u32)M, (u32)Lw, (u32)a->Wp);
    dim3 grid((unsigned)((Wc + 7) / 8), (unsigned)((M + gf2cu::kGemmRows - 1) / gf2cu::kGemmRows));
    gf2cu::gemm_m4rm_kernel<<<grid, gf2cu::kTrailThreads, gf2cu::kTableBytes, s>>>(
        rw.src, b->data, c->data, (u32)M, (u32)L, (u32)b->Wp, (u32)c->Wp, accumulate ? 1 : 0);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

// Host-view product: A and B staged in the operand cache slots, C in slot 0.
gf2cu_status view_mul(const gf2cu_view* c, const gf2cu_view* a, const gf2cu_view* b,
                      const gf2cu_cfg* cfg, bool accumulate);

gf2cu_status check_view(const gf2cu_view* v) {
    if (!v) return fail(GF2CU_EINVAL, "null argument");
    if (v->nrows && v->ncols && !v->data) return fail(GF2CU_EINVAL, "null data");
    if (v->nrows && v->ncols && v->stride * 64 < v->col_off + v->ncols)
        return fail(GF2CU_ERANGE, "view window exceeds its row stride");
    return GF2CU_OK;
}

gf2cu_status view_mul(const gf2cu_view* c, const gf2cu_view* a, const gf2cu_view* b,
                      const gf2cu_cfg* cfg, bool accumulate) {
    gf2cu_status st = check_view(a);
    if (st == GF2CU_OK) st = check_view(b);
    if (st == GF2CU_OK) st = check_view(c);
    if (st != GF2CU_OK) return st;
    if (a->ncols != b->nrows || c->nrows != a->nrows || c->ncols != b->ncols)
        return fail(GF2CU_EINVAL, "multiply: dimension mismatch");
    if (c->nrows == 0 || c->ncols == 0) return GF2CU_OK;
    gf2cu_cfg cc;
    gf2cu_default_config(&cc);
    if (cfg) cc = *cfg;
    gf2cu_matrix *da = nullptr, *db = nullptr;
    st = cached_matrix(1, a->nrows, a->ncols, cc.device, &da);
    if (st == GF2CU_OK) st = cached_matrix(2, b->nrows, b->ncols, cc.device, &db);
    if (st != GF2CU_OK) return st;
    DeviceGuard g(cc.device);
    std::vector<u64> pa, pb;
    cudaStream_t s0 = pick_stream(da, cc.stream);
    st = view_upload(a, da, s0, pa);
    if (st == GF2CU_OK) st = view_upload(b, db, s0, pb);
    if (st != GF2CU_OK) return st;
    cc.stream = s0;
    return with_view(c, &cc, nullptr, [&](gf2cu_matrix* dc, const gf2cu_cfg& c2) {
        return run_mul(dc, da, db, accumulate, pick_stream(dc, c2.stream));
    });
}

// PLE then rref_from_ple on the device copy (echelonize, m4ri.hpp:95-98).
gf2cu_status run_echelonize(gf2cu_matrix* a, const gf2cu_cfg* cfg, bool full, size_t* rank) {
    const size_t mn = std::min(a->m, a->n);
    std::vector<size_t> sw(std::max<size_t>(1, mn)), q(std::max<size_t>(1, mn));
    gf2cu_status st = run_ple(a, cfg, sw.data(), q.data(), rank, nullptr, nullptr, nullptr);
    if (st != GF2CU_OK) return st;
    return run_rref(a, q.data(), *rank, full, pick_stream(a, cfg ? cfg->stream : nullptr));
}

}  // namespace

extern "C" {

void gf2cu_default_config(gf2cu_cfg* cfg) {
    if (!cfg) return;
    cfg->k = 0;
    cfg->k_scale = 0.75;
    cfg->table_count = 4;
    cfg->device = 0;
    cfg->stream = nullptr;
    cfg->flags = 0;
}

const char* gf2cu_last_error(void) { return g_last_error.c_str(); }

const char* gf2cu_version(void) { return "gf2cu 0.1 (sm_100a, 64-column panels, 8x8-bit Gray tables)"; }

int gf2cu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    int good = 0;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp pr;
        if (cudaGetDeviceProperties(&pr, d) == cudaSuccess && pr.major == 10) ++good;
    }
    return good;
}

gf2cu_status gf2cu_matrix_create(size_t m, size_t n, int device, gf2cu_matrix** out) {
    if (!out) return fail(GF2CU_EINVAL, "out is null");
    *out = nullptr;
    if (m >= (1ull << 31) || n >= (1ull << 31))
        return fail(GF2CU_EINVAL, "dimensions exceed 2^31");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(GF2CU_ENODEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(GF2CU_EINVAL, "bad device ordinal");
    cudaDeviceProp pr;
    CU_TRY(cudaGetDeviceProperties(&pr, device));
    if (pr.major != 10)
        return fail(GF2CU_ENODEVICE, "device is not sm_100 (built for sm_100a only)");
    DeviceGuard g(device);
    auto* a = new (std::nothrow) gf2cu_matrix;
    if (!a) return fail(GF2CU_ENOMEM, "host allocation failed");
    a->m = m;
    a->n = n;
    a->W = words_of(n);
    a->Wp = padded_stride(n);
    a->device = device;
    const size_t bytes = std::max<size_t>(1, m) * a->Wp * sizeof(u64);
    cudaError_t e = cudaMalloc(&a->data, bytes);
    if (e == cudaSuccess) e = zero_now(a->data, bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) apply_watchdog_env(device);
    if (e != cudaSuccess) {
        cudaFree(a->data);
        delete a;
        return cuda_fail(e, "gf2cu_matrix_create");
    }
    *out = a;
    return GF2CU_OK;
}

gf2cu_status gf2cu_matrix_destroy(gf2cu_matrix* a) {
    if (!a) return GF2CU_OK;
    DeviceGuard g(a->device);
    cudaFree(a->data);
    cudaFree(a->alt);
    free_ws(a->ws);
    free_rref(a->rw);
    free_peer(a->pw);
    if (a->own) cudaStreamDestroy(a->own);
    delete a;
    return GF2CU_OK;
}

gf2cu_status gf2cu_matrix_info(const gf2cu_matrix* a, size_t* m, size_t* n, size_t* stride_words,
                               uint64_t** device_ptr) {
    if (!a) return fail(GF2CU_EINVAL, "null matrix");
    if (m) *m = a->m;
    if (n) *n = a->n;
    if (stride_words) *stride_words = a->Wp;
    if (device_ptr) *device_ptr = reinterpret_cast<uint64_t*>(a->data);
    return GF2CU_OK;
}

gf2cu_status gf2cu_matrix_upload(gf2cu_matrix* a, const uint64_t* host, size_t host_stride,
                                 void* stream) {
    if (!a || (!host && a->m)) return fail(GF2CU_EINVAL, "null argument");
    if (host_stride < a->W) return fail(GF2CU_EINVAL, "host stride smaller than the row");
    if (a->m == 0 || a->W == 0) return GF2CU_OK;
    DeviceGuard g(a->device);
    cudaStream_t s = pick_stream(a, stream);
    gf2cu_status st = staged_h2d(a->data, a->Wp * 8, host, host_stride * 8, a->W * 8, a->m, a->device, s);
    if (st != GF2CU_OK) return st;
    CU_TRY(cudaStreamSynchronize(s));
    return GF2CU_OK;
}

gf2cu_status gf2cu_matrix_download(const gf2cu_matrix* a, uint64_t* host, size_t host_stride,
                                   void* stream) {
    if (!a || (!host && a->m)) return fail(GF2CU_EINVAL, "null argument");
    if (host_stride < a->W) return fail(GF2CU_EINVAL, "host stride smaller than the row");
    if (a->m == 0 || a->W == 0) return GF2CU_OK;
    DeviceGuard g(a->device);
    cudaStream_t s = pick_stream(const_cast<gf2cu_matrix*>(a), stream);
    return staged_d2h(host, host_stride * 8, a->data, a->Wp * 8, a->W * 8, a->m, a->device, s);
}

gf2cu_status gf2cu_matrix_copy(gf2cu_matrix* dst, const gf2cu_matrix* src, void* stream) {
    if (!dst || !src) return fail(GF2CU_EINVAL, "null matrix");
    if (dst->m != src->m || dst->n != src->n) return fail(GF2CU_EINVAL, "shape mismatch");
    DeviceGuard g(dst->device);
    cudaStream_t s = pick_stream(dst, stream);
    CU_TRY(cudaMemcpyAsync(dst->data, src->data, std::max<size_t>(1, dst->m) * dst->Wp * 8,
                           cudaMemcpyDeviceToDevice, s));
    CU_TRY(cudaStreamSynchronize(s));
    return GF2CU_OK;
}

gf2cu_status gf2cu_matrix_fill_ctr(gf2cu_matrix* a, uint64_t seed, void* stream) {
    if (!a) return fail(GF2CU_EINVAL, "null matrix");
    if (a->m == 0) return GF2CU_OK;
    DeviceGuard g(a->device);
    cudaStream_t s = pick_stream(a, stream);
    gf2cu::fill_ctr_kernel<<<num_sms(a->device) * 8, 256, 0, s>>>(a->data, (u32)a->m, (u32)a->n,
                                                                 (u32)a->Wp, seed);
    CU_TRY(cudaGetLastError());
    CU_TRY(cudaStreamSynchronize(s));
    return GF2CU_OK;
}

gf2cu_status gf2cu_matrix_checksum(const gf2cu_matrix* a, uint64_t* out, void* stream) {
    if (!a || !out) return fail(GF2CU_EINVAL, "null argument");
    auto* am = const_cast<gf2cu_matrix*>(a);
    DeviceGuard g(a->device);
    if (a->m == 0) {
        *out = 0;
        return GF2CU_OK;
    }
    if (!am->ws.hashes) CU_TRY(cudaMalloc(&am->ws.hashes, a->m * sizeof(u64)));
    cudaStream_t s = pick_stream(am, stream);
    gf2cu::row_hash_kernel<<<num_sms(a->device) * 4, 256, 0, s>>>(a->data, (u32)a->m, (u32)a->W,
                                                                 (u32)a->Wp, am->ws.hashes);
    CU_TRY(cudaGetLastError());
    std::vector<u64> h(a->m);
    CU_TRY(cudaMemcpyAsync(h.data(), am->ws.hashes, a->m * sizeof(u64), cudaMemcpyDeviceToHost, s));
    CU_TRY(cudaStreamSynchronize(s));
    // fold: FNV-1a over the row hashes
    u64 acc = 0xcbf29ce484222325ull;
    for (u64 v : h) {
        acc ^= v;
        acc *= 0x100000001b3ull;
    }
    *out = acc;
    return GF2CU_OK;
}

gf2cu_status gf2cu_ple_device(gf2cu_matrix* a, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                              size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                              gf2cu_stats* stats) {
    if (!a || !rank || ((!swaps || !q) && std::min(a->m, a->n) > 0))
        return fail(GF2CU_EINVAL, "null argument");
    gf2cu_status st = check_cfg(cfg);
    if (st != GF2CU_OK) return st;
    DeviceGuard g(a->device);
    return run_ple(a, cfg, swaps, q, rank, col_swaps, n_col_swaps, stats);
}

// partial_ple (ple.hpp:57-130). Its pivot search reads every row of a column
// before giving up on it, so it finds the same pivots as the complete
// decomposition (rank, q, p.swaps equal), and every row it reads ends fully
// updated. Only its laziness differs: the watermark s[0] (:69-87, :128)
// records the rows read once a first pivot exists. A pivotless column after
// the first pivot column -- between pivots or after the last one (the final
// scan, :60-97) -- reads every row, so processed = m and the in-place result
// is the complete PLE's. Otherwise (pivot columns consecutive from q[0] up to
// column n-1; empty columns before q[0] are read while r = 0 and do not move
// the watermark) the deepest row read is the deepest pivot row, the rows past
// it were never read and stay untouched, and processed = max(rank, max swaps
// + 1). r = m also gives m; rank 0 gives processed 0 (:113-116).
static gf2cu_status run_undo_col_swaps(gf2cu_matrix* a, const gf2cu_colswap* cs, size_t ncs, cudaStream_t s,
                                       bool forward, size_t row_lo);

static size_t partial_processed(size_t m, size_t n, size_t rank, const size_t* swaps, const size_t* q) {
    if (rank == 0) return 0;
    if (rank >= m || q[rank - 1] != n - 1 || q[rank - 1] - q[0] != rank - 1) return m;
    size_t smax = 0;
    for (size_t l = 0; l < rank; ++l) smax = std::max(smax, swaps[l]);
    return std::max(rank, smax + 1);
}

gf2cu_status gf2cu_partial_ple(const gf2cu_view* v, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                               size_t* rank, size_t* processed, gf2cu_colswap* col_swaps,
                               size_t* n_col_swaps) {
    if (!v || !rank || !processed) return fail(GF2CU_EINVAL, "null argument");
    gf2cu_status st = check_view(v);
    if (st != GF2CU_OK) return st;
    const size_t m = v->nrows, n = v->ncols;
    if ((!swaps || !q) && std::min(m, n) > 0) return fail(GF2CU_EINVAL, "null outputs");
    st = check_cfg(cfg);
    if (st != GF2CU_OK) return st;
    *processed = 0;
    if (m == 0 || n == 0) {
        *rank = 0;
        if (n_col_swaps) *n_col_swaps = 0;
        return GF2CU_OK;
    }
    size_t limit = m;
    std::vector<gf2cu_colswap> cs(std::max<size_t>(1, std::min(m, n)));
    st = with_view(v, cfg, nullptr, [&](gf2cu_matrix* a, const gf2cu_cfg& c) {
        size_t ncs = 0;
        gf2cu_status s2 = run_ple(a, &c, swaps, q, rank, cs.data(), &ncs, nullptr);
        if (s2 != GF2CU_OK) return s2;
        limit = partial_processed(m, n, *rank, swaps, q);
        if (col_swaps) std::copy(cs.begin(), cs.begin() + ncs, col_swaps);
        if (n_col_swaps) *n_col_swaps = ncs;
        if (limit < m) {
            // rows [limit, m) were never read: back to the input (the host view
            // still holds it), then only the compression swaps (ple.hpp:122-126)
            cudaStream_t s = reinterpret_cast<cudaStream_t>(c.stream);
            gf2cu_view tail = *v;
            tail.data = v->data + limit * v->stride;
            tail.nrows = m - limit;
            gf2cu_matrix shifted;
            shifted.m = m - limit;
            shifted.n = a->n;
            shifted.W = a->W;
            shifted.Wp = a->Wp;
            shifted.device = a->device;
            shifted.data = a->data + limit * a->Wp;
            std::vector<u64> packed;
            s2 = view_upload(&tail, &shifted, s, packed);
            shifted.data = nullptr;  // (not owned)
            if (s2 == GF2CU_OK) s2 = run_undo_col_swaps(a, cs.data(), ncs, s, true, limit);
            if (s2 == GF2CU_OK) CU_TRY(cudaStreamSynchronize(s));  // (packed outlives the upload)
        }
        return s2;
    });
    if (st == GF2CU_OK) *processed = limit;
    return st;
}

static gf2cu_status run_undo_col_swaps(gf2cu_matrix* a, const gf2cu_colswap* cs, size_t ncs, cudaStream_t s,
                                       bool forward, size_t row_lo) {
    if (ncs == 0 || a->m <= row_lo) return GF2CU_OK;
    std::vector<ulonglong2> h(ncs);  // {a | b << 32, from_row}
    for (size_t i = 0; i < ncs; ++i) h[i] = make_ulonglong2((u64)cs[i].a | ((u64)cs[i].b << 32), cs[i].from_row);
    ulonglong2* d = nullptr;
    CU_TRY(cudaMallocAsync(&d, ncs * sizeof(ulonglong2), s));
    cudaError_t e = cudaMemcpyAsync(d, h.data(), ncs * sizeof(ulonglong2), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        const unsigned blocks = (unsigned)std::min<size_t>((a->m + 255) / 256, 65535u * 16);
        gf2cu::undo_col_swaps_kernel<<<blocks, 256, 0, s>>>(a->data, (u32)a->m, (u32)a->Wp, d, (u32)ncs,
                                                            forward ? 1 : 0, (u32)row_lo);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // (h outlives the copy)
    cudaFreeAsync(d, s);
    return e == cudaSuccess ? GF2CU_OK : cuda_fail(e, "undo_column_swaps");
}

static gf2cu_status check_col_swaps(size_t m, size_t n, const gf2cu_colswap* cs, size_t ncs) {
    if (ncs && !cs) return fail(GF2CU_EINVAL, "null col_swaps");
    for (size_t i = 0; i < ncs; ++i)
        if (cs[i].a >= n || cs[i].b >= n || cs[i].from_row > m || m >= (1ull << 32) || n >= (1ull << 32))
            return fail(GF2CU_ERANGE, "column swap outside the matrix");
    return GF2CU_OK;
}

gf2cu_status gf2cu_undo_column_swaps_device(gf2cu_matrix* a, const gf2cu_colswap* col_swaps,
                                            size_t n_col_swaps, void* stream) {
    if (!a) return fail(GF2CU_EINVAL, "null matrix");
    gf2cu_status st = check_col_swaps(a->m, a->n, col_swaps, n_col_swaps);
    if (st != GF2CU_OK) return st;
    DeviceGuard g(a->device);
    return run_undo_col_swaps(a, col_swaps, n_col_swaps, pick_stream(a, stream), false, 0);
}

gf2cu_status gf2cu_undo_column_swaps(const gf2cu_view* v, const gf2cu_colswap* col_swaps,
                                     size_t n_col_swaps, const gf2cu_cfg* cfg) {
    gf2cu_status st = check_view(v);
    if (st != GF2CU_OK) return st;
    st = check_col_swaps(v->nrows, v->ncols, col_swaps, n_col_swaps);
    if (st != GF2CU_OK || n_col_swaps == 0 || v->nrows == 0 || v->ncols == 0) return st;
    return with_view(v, cfg, nullptr, [&](gf2cu_matrix* a, const gf2cu_cfg& c) {
        return run_undo_col_swaps(a, col_swaps, n_col_swaps, reinterpret_cast<cudaStream_t>(c.stream), false, 0);
    });
}

gf2cu_status gf2cu_ple(const gf2cu_view* v, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                       size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                       gf2cu_stats* stats) {
    if (!v || !rank) return fail(GF2CU_EINVAL, "null argument");
    gf2cu_status st = check_view(v);
    if (st != GF2CU_OK) return st;
    const size_t m = v->nrows, n = v->ncols;
    if ((!swaps || !q) && std::min(m, n) > 0) return fail(GF2CU_EINVAL, "null outputs");
    st = check_cfg(cfg);
    if (st != GF2CU_OK) return st;
    if (m == 0 || n == 0) {
        *rank = 0;
        if (n_col_swaps) *n_col_swaps = 0;
        if (stats) std::memset(stats, 0, sizeof(*stats));
        return GF2CU_OK;
    }
    // aligned views receive the finished rows while the kernel runs, and
    // (large ones) are factored while their rows are still arriving
    size_t streamed = 0;
    const gf2cu_view* to = view_aligned(v) ? v : nullptr;
    return with_view(
        v, cfg, stats,
        [&](gf2cu_matrix* a, const gf2cu_cfg& c) {
            return run_ple(a, &c, swaps, q, rank, col_swaps, n_col_swaps, stats, to, &streamed, to);
        },
        &streamed, nullptr, to != nullptr);
}

gf2cu_status gf2cu_matrix_mul(gf2cu_matrix* c, const gf2cu_matrix* a, const gf2cu_matrix* b,
                              int accumulate, void* stream) {
    if (!a || !b || !c) return fail(GF2CU_EINVAL, "null matrix");
    DeviceGuard g(c->device);
    cudaStream_t s = pick_stream(c, stream);
    gf2cu_status st = run_mul(c, a, b, accumulate != 0, s);
    if (st == GF2CU_OK) CU_TRY(cudaStreamSynchronize(s));
    return st;
}

gf2cu_status gf2cu_mul(const gf2cu_view* c, const gf2cu_view* a, const gf2cu_view* b,
                       const gf2cu_cfg* cfg) {
    return view_mul(c, a, b, cfg, false);
}

gf2cu_status gf2cu_addmul(const gf2cu_view* c, const gf2cu_view* a, const gf2cu_view* b,
                          const gf2cu_cfg* cfg) {
    return view_mul(c, a, b, cfg, true);
}

gf2cu_status gf2cu_rref_from_ple_device(gf2cu_matrix* a, const size_t* q, size_t rank, int full,
                                        void* stream) {
    if (!a) return fail(GF2CU_EINVAL, "null matrix");
    DeviceGuard g(a->device);
    cudaStream_t s = pick_stream(a, stream);
    gf2cu_status st = run_rref(a, q, rank, full != 0, s);
    if (st == GF2CU_OK) CU_TRY(cudaStreamSynchronize(s));
    return st;
}

gf2cu_status gf2cu_rref_from_ple(const gf2cu_view* v, const size_t* q, size_t rank, int full,
                                 const gf2cu_cfg* cfg) {
    gf2cu_status st = check_view(v);
    if (st != GF2CU_OK) return st;
    st = check_pivots(q, rank, v->nrows, v->ncols);
    if (st != GF2CU_OK || v->nrows == 0 || v->ncols == 0) return st;
    return with_view(v, cfg, nullptr, [&](gf2cu_matrix* a, const gf2cu_cfg& c) {
        return run_rref(a, q, rank, full != 0, pick_stream(a, c.stream));
    });
}

gf2cu_status gf2cu_echelonize_device(gf2cu_matrix* a, int full, const gf2cu_cfg* cfg, size_t* rank) {
    if (!a || !rank) return fail(GF2CU_EINVAL, "null argument");
    gf2cu_status st = check_cfg(cfg);
    if (st != GF2CU_OK) return st;
    DeviceGuard g(a->device);
    st = run_echelonize(a, cfg, full != 0, rank);
    if (st == GF2CU_OK) CU_TRY(cudaStreamSynchronize(pick_stream(a, cfg ? cfg->stream : nullptr)));
    return st;
}

gf2cu_status gf2cu_echelonize(const gf2cu_view* v, int full, const gf2cu_cfg* cfg, size_t* rank) {
    if (!rank) return fail(GF2CU_EINVAL, "null argument");
    gf2cu_status st = check_view(v);
    if (st != GF2CU_OK) return st;
    st = check_cfg(cfg);
    if (st != GF2CU_OK) return st;
    *rank = 0;
    if (v->nrows == 0 || v->ncols == 0) return GF2CU_OK;
    return with_view(v, cfg, nullptr, [&](gf2cu_matrix* a, const gf2cu_cfg& c) {
        return run_echelonize(a, &c, full != 0, rank);
    });
}

// trsm_upper_left_unit (multiply.hpp:314-335): B <- U^-1 B, U unit upper
// triangular r x r (only bits strictly above the diagonal read), B r x n.
gf2cu_status gf2cu_trsm_upper_left_unit(const gf2cu_view* u, const gf2cu_view* b,
                                        const gf2cu_cfg* cfg) {
    gf2cu_status st = check_view(u);
    if (st == GF2CU_OK) st = check_view(b);
    if (st != GF2CU_OK) return st;
    const size_t r = u->nrows;
    if (u->ncols != r || b->nrows != r) return fail(GF2CU_EINVAL, "trsm: dimension mismatch");
    if (r <= 1 || b->ncols == 0) return GF2CU_OK;
    const size_t Wa = words_of(r);
    // U packed row-major (r x Wa) on the host, staged next to B's device copy
    std::vector<u64> hu(r * Wa);
    for (size_t i = 0; i < r; ++i) {
        const u64* row = reinterpret_cast<const u64*>(u->data) + i * u->stride;
        for (size_t x = 0; x < Wa; ++x)
            hu[i * Wa + x] = read_bits(row, u->col_off + 64 * x, std::min<size_t>(64, r - 64 * x));
    }
    return with_view(b, cfg, nullptr, [&](gf2cu_matrix* a, const gf2cu_cfg& c) -> gf2cu_status {
        cudaStream_t s = pick_stream(a, c.stream);
        RrefWs& rw = a->rw;
        const size_t n = a->n, R = (r + 63) / 64 * 64, Wu = R / 64, Wn = a->W;
        const size_t WnPad8 = (Wn + 7) / 8 * 8;
        CU_TRY(grow(&rw.src, &rw.src_words, r * Wa));
        CU_TRY(grow(&rw.U, &rw.U_words, Wu * R));
        CU_TRY(grow(&rw.N, &rw.N_words, WnPad8 * R));
        CU_TRY(cudaMemcpyAsync(rw.src, hu.data(), hu.size() * sizeof(u64), cudaMemcpyHostToDevice, s));
        CU_TRY(cudaMemsetAsync(rw.U, 0, Wu * R * sizeof(u64), s));
        CU_TRY(cudaMemsetAsync(rw.N, 0, WnPad8 * R * sizeof(u64), s));
        gf2cu::RrefParams p{};
        p.a = rw.src;
        p.b = a->data;
        p.out = a->data;
        p.U = rw.U;
        p.N = rw.N;
        p.m = (u32)r;
        p.n = (u32)n;
        p.W = (u32)a->W;
        p.Wp = (u32)a->Wp;
        p.Wa = (u32)Wa;
        p.Wpa = (u32)Wa;
        p.r = (u32)r;
        p.R = (u32)R;
        p.Wu = (u32)Wu;
        p.Wn = (u32)Wn;
        p.WnPad8 = (u32)WnPad8;
        p.ncn = (u32)n;
        const int sms = num_sms(a->device);
        gf2cu::rref_gather_kernel<<<sms * 8, 256, 0, s>>>(p, 0);
        CU_TRY(cudaGetLastError());
        gf2cu_status st2 = solve_upper(a, p, s);
        if (st2 != GF2CU_OK) return st2;
        gf2cu::trsm_store_kernel<<<sms * 8, 256, 0, s>>>(p);
        CU_TRY(cudaGetLastError());
        return GF2CU_OK;
    });
}

}  // extern "C"

// ------------------------------------------------------------- sharded
struct gf2cu_shard {
    size_t m = 0, n = 0, W = 0, Wp = 0, Wpad8 = 0, m_loc = 0, block = 0;
    int rank = 0, nranks = 1, device = 0;
    // local
    u64* data = nullptr;  // row-major (upload / download)
    u64* mat = nullptr;   // tile-major working copy
    u64* pbl = nullptr;
    ulonglong2* info = nullptr;
    unsigned char* retired = nullptr;
    gf2cu::StepState* lstate = nullptr;
    u64* stage = nullptr;
    bool stage_owned = true;  // false once the caller supplied its own (set_stage)
    // replicated
    u32* perm = nullptr;
    u32* inv = nullptr;
    gf2cu::StepState* gstate = nullptr;
    gf2cu::PanelOut* pout = nullptr;
    u32* swaps = nullptr;
    u32* qcol = nullptr;
    u32* rhist = nullptr;
    u32* rbhist = nullptr;
    u32* status = nullptr;
    cudaStream_t own = nullptr;
};

namespace {

cudaStream_t shard_stream(gf2cu_shard* s, void* st) {
    return st ? reinterpret_cast<cudaStream_t>(st) : s->own;
}

gf2cu::ShardParams shard_params(gf2cu_shard* s) {
    gf2cu::ShardParams p{};
    p.mat = s->mat;
    p.pbl = s->pbl;
    p.info = s->info;
    p.retired = s->retired;
    p.lstate = s->lstate;
    p.perm = s->perm;
    p.inv = s->inv;
    p.gstate = s->gstate;
    p.pout = s->pout;
    p.m_loc = (u32)s->m_loc;
    p.m = (u32)s->m;
    p.n = (u32)s->n;
    p.W = (u32)s->W;
    p.Wpad8 = (u32)s->Wpad8;
    p.rank = (u32)s->rank;
    p.nranks = (u32)s->nranks;
    p.block = (u32)s->block;
    return p;
}

size_t shard_local_rows(size_t m, size_t rank, size_t nranks, size_t block) {
    size_t cnt = 0;
    const size_t nblocks = (m + block - 1) / block;
    for (size_t b = rank; b < nblocks; b += nranks) cnt += std::min(block, m - b * block);
    return cnt;
}

}  // namespace

extern "C" {

gf2cu_status gf2cu_shard_create(size_t m, size_t n, int rank, int nranks, size_t block, int device,
                                gf2cu_shard** out) {
    if (!out) return fail(GF2CU_EINVAL, "out is null");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks || block == 0)
        return fail(GF2CU_EINVAL, "bad rank / nranks / block");
    if (m == 0 || n == 0 || m >= (1ull << 31) || n >= (1ull << 31))
        return fail(GF2CU_EINVAL, "dimensions must be in [1, 2^31)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(GF2CU_ENODEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(GF2CU_EINVAL, "bad device ordinal");
    DeviceGuard g(device);
    auto* s = new (std::nothrow) gf2cu_shard;
    if (!s) return fail(GF2CU_ENOMEM, "host allocation failed");
    s->m = m;
    s->n = n;
    s->W = words_of(n);
    s->Wp = padded_stride(n);
    s->Wpad8 = wpad8(s->W);
    s->rank = rank;
    s->nranks = nranks;
    s->block = block;
    s->device = device;
    s->m_loc = shard_local_rows(m, rank, nranks, block);
    const size_t ml = std::max<size_t>(1, s->m_loc), mn = std::max<size_t>(1, std::min(m, n));
    cudaError_t e = cudaSuccess;
    auto alloc = [&](auto** ptr, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes);
    };
    alloc(&s->data, ml * s->Wp * 8);
    alloc(&s->mat, ml * s->Wpad8 * 8);
    alloc(&s->pbl, ml * 8);
    alloc(&s->info, ml * sizeof(ulonglong2));
    alloc(&s->retired, ml);
    alloc(&s->lstate, sizeof(gf2cu::StepState));
    alloc(&s->stage, 64 * s->Wpad8 * 8);
    alloc(&s->perm, m * 4);
    alloc(&s->inv, m * 4);
    alloc(&s->gstate, sizeof(gf2cu::StepState));
    alloc(&s->pout, sizeof(gf2cu::PanelOut));
    alloc(&s->swaps, mn * 4);
    alloc(&s->qcol, mn * 4);
    alloc(&s->rhist, (s->W + 1) * 4);
    alloc(&s->rbhist, (s->W + 1) * 4);
    alloc(&s->status, (8 + 2 * (size_t)nranks) * 4);
    if (e == cudaSuccess) e = zero_now(s->data, ml * s->Wp * 8);
    if (e == cudaSuccess) e = zero_now(s->stage, 64 * s->Wpad8 * 8);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) apply_watchdog_env(s->device);
    if (e != cudaSuccess) {
        gf2cu_shard_destroy(s);
        return cuda_fail(e, "gf2cu_shard_create");
    }
    *out = s;
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_destroy(gf2cu_shard* s) {
    if (!s) return GF2CU_OK;
    DeviceGuard g(s->device);
    if (s->stage_owned) cudaFree(s->stage);
    for (void* p : {(void*)s->data, (void*)s->mat, (void*)s->pbl, (void*)s->info, (void*)s->retired,
                    (void*)s->lstate, (void*)s->perm, (void*)s->inv,
                    (void*)s->gstate, (void*)s->pout, (void*)s->swaps, (void*)s->qcol,
                    (void*)s->rhist, (void*)s->rbhist, (void*)s->status})
        cudaFree(p);
    if (s->own) cudaStreamDestroy(s->own);
    delete s;
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_info(const gf2cu_shard* s, size_t* m_local, size_t* pack_words) {
    if (!s) return fail(GF2CU_EINVAL, "null shard");
    if (m_local) *m_local = s->m_loc;
    if (pack_words) *pack_words = 64 * s->Wpad8;
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_upload(gf2cu_shard* s, const uint64_t* host, size_t host_stride,
                                void* stream) {
    if (!s || (!host && s->m_loc)) return fail(GF2CU_EINVAL, "null argument");
    if (host_stride < s->W) return fail(GF2CU_EINVAL, "host stride smaller than the row");
    if (!s->m_loc) return GF2CU_OK;
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    CU_TRY(cudaMemcpy2DAsync(s->data, s->Wp * 8, host, host_stride * 8, s->W * 8, s->m_loc,
                             cudaMemcpyHostToDevice, st));
    CU_TRY(cudaStreamSynchronize(st));
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_download(const gf2cu_shard* s, uint64_t* host, size_t host_stride,
                                  void* stream) {
    if (!s || (!host && s->m_loc)) return fail(GF2CU_EINVAL, "null argument");
    if (host_stride < s->W) return fail(GF2CU_EINVAL, "host stride smaller than the row");
    if (!s->m_loc) return GF2CU_OK;
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(const_cast<gf2cu_shard*>(s), stream);
    CU_TRY(cudaMemcpy2DAsync(host, host_stride * 8, s->data, s->Wp * 8, s->W * 8, s->m_loc,
                             cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_fill_ctr(gf2cu_shard* s, uint64_t seed, void* stream) {
    if (!s) return fail(GF2CU_EINVAL, "null shard");
    if (!s->m_loc) return GF2CU_OK;
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    gf2cu::shard_fill_ctr_kernel<<<num_sms(s->device) * 8, 256, 0, st>>>(
        s->data, (u32)s->m_loc, (u32)s->n, (u32)s->Wp, (u32)s->rank, (u32)s->nranks,
        (u32)s->block, seed);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_begin(gf2cu_shard* s, void* stream) {
    if (!s) return fail(GF2CU_EINVAL, "null shard");
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    const int sms = num_sms(s->device);
    if (s->m_loc)
        gf2cu::tile_kernel<<<sms * 8, 256, 0, st>>>(s->data, s->mat, (u32)s->m_loc, (u32)s->Wp,
                                                   (u32)s->Wpad8);
    gf2cu::shard_init_kernel<<<sms * 4, 256, 0, st>>>(shard_params(s), s->perm, s->inv, s->gstate);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_gather(gf2cu_shard* s, uint64_t* pos_words, size_t lo, size_t hi,
                                void* stream) {
    if (!s || !pos_words || lo > hi || hi > s->m) return fail(GF2CU_EINVAL, "bad gather range");
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    if (hi == lo) return GF2CU_OK;
    CU_TRY(cudaMemsetAsync(pos_words + lo, 0, (hi - lo) * 8, st));
    if (s->m_loc)
        gf2cu::shard_gather_kernel<<<num_sms(s->device) * 4, 256, 0, st>>>(
            shard_params(s), reinterpret_cast<u64*>(pos_words), (u32)lo, (u32)hi);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_panel(gf2cu_shard* s, size_t w, uint64_t* pos_words, int window_only,
                               uint32_t* status_out, void* stream) {
    if (!s || !pos_words || w >= s->W) return fail(GF2CU_EINVAL, "bad panel call");
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    gf2cu::Params p{};
    p.pb = reinterpret_cast<u64*>(pos_words);
    p.perm = s->perm;
    p.inv = s->inv;
    p.state = s->gstate;
    p.pout = s->pout;
    p.swaps = s->swaps;
    p.qcol = s->qcol;
    p.rhist = s->rhist;
    p.rbhist = s->rbhist;
    p.status = s->status;
    p.window_only = window_only ? 1u : 0u;
    p.nranks = (u32)s->nranks;
    p.block = (u32)s->block;
    p.m = (u32)s->m;
    p.n = (u32)s->n;
    p.W = (u32)s->W;
    p.Wpad8 = (u32)s->Wpad8;
    p.pflags = panel_flags();
    gf2cu::panel_factor_kernel<<<1, gf2cu::kPanelThreads, 0, st>>>(p, (u32)w);
    CU_TRY(cudaGetLastError());
    if (status_out) {  // (asynchronous when the caller does not read the status)
        CU_TRY(cudaMemcpyAsync(status_out, s->status, (8 + 2 * (size_t)s->nranks) * 4,
                               cudaMemcpyDeviceToHost, st));
        CU_TRY(cudaStreamSynchronize(st));
    }
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_apply(gf2cu_shard* s, size_t w, uint64_t* pack, void* stream) {
    if (!s || w >= s->W) return fail(GF2CU_EINVAL, "bad apply call");
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    CU_TRY(cudaMemsetAsync(&s->lstate->r, 0xff, 4, st));
    if (s->m_loc) {
        gf2cu::ShardParams p = shard_params(s);
        p.pack = reinterpret_cast<u64*>(pack);
        if (pack && w + 1 < s->W)
            gf2cu::shard_pack_kernel<<<num_sms(s->device) * 4, 256, 0, st>>>(p, (u32)w);
        gf2cu::shard_apply_kernel<<<num_sms(s->device) * 4, gf2cu::kApplyThreads, 0, st>>>(p, (u32)w);
    }
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_pack_stage(gf2cu_shard* s, size_t w, void* stream) {
    if (!s || w >= s->W) return fail(GF2CU_EINVAL, "bad pack_stage call");
    if (w + 1 >= s->W) return GF2CU_OK;
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    const size_t x0 = (w + 1) & ~size_t(7);
    const size_t lo = (x0 >> 3) * 64 * 8, hi = (s->Wpad8 >> 3) * 64 * 8;
    CU_TRY(cudaMemsetAsync(s->stage + lo, 0, (hi - lo) * 8, st));
    if (s->m_loc)
        gf2cu::shard_pack_stage_kernel<<<num_sms(s->device) * 4, 256, 0, st>>>(shard_params(s), s->stage,
                                                                             (u32)w);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

// The asynchronous protocol's three calls per step (shard.py::_run_steps).
gf2cu_status gf2cu_shard_step_gather(gf2cu_shard* s, size_t w, uint64_t* pos_words, void* stream) {
    (void)w;
    return gf2cu_shard_gather(s, pos_words, 0, s ? s->m : 0, stream);
}

gf2cu_status gf2cu_shard_step_panel(gf2cu_shard* s, size_t w, uint64_t* pos_words, void* stream) {
    gf2cu_status st = gf2cu_shard_panel(s, w, pos_words, 0, nullptr, stream);
    if (st == GF2CU_OK) st = gf2cu_shard_pack_stage(s, w, stream);
    return st;
}

gf2cu_status gf2cu_shard_step_update(gf2cu_shard* s, size_t w, void* stream) {
    gf2cu_status st = gf2cu_shard_apply(s, w, nullptr, stream);
    if (st == GF2CU_OK) st = gf2cu_shard_trailing(s, w, stream);
    return st;
}

gf2cu_status gf2cu_shard_set_stage(gf2cu_shard* s, uint64_t* stage) {
    if (!s || !stage) return fail(GF2CU_EINVAL, "null stage");
    DeviceGuard g(s->device);
    if (s->stage_owned) {
        cudaFree(s->stage);
        s->stage_owned = false;
    }
    s->stage = reinterpret_cast<u64*>(stage);
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_pivots(gf2cu_shard* s, size_t* pivots, void* stream) {
    if (!s || !pivots) return fail(GF2CU_EINVAL, "null argument");
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    gf2cu::StepState h{};
    CU_TRY(cudaMemcpyAsync(&h, s->gstate, sizeof(h), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    *pivots = (size_t)h.r + h.rb;
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_unpack(gf2cu_shard* s, size_t w, uint64_t mask, const uint64_t* pack,
                                void* stream) {
    if (!s || !pack || w >= s->W) return fail(GF2CU_EINVAL, "bad unpack call");
    if (!mask || w + 1 >= s->W) return GF2CU_OK;
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    gf2cu::shard_unpack_kernel<<<num_sms(s->device) * 4, 256, 0, st>>>(
        reinterpret_cast<const u64*>(pack), mask, s->stage, (u32)w, (u32)s->Wpad8);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_trailing(gf2cu_shard* s, size_t w, void* stream) {
    if (!s || w >= s->W) return fail(GF2CU_EINVAL, "bad trailing call");
    if (!s->m_loc || w + 1 >= s->W) return GF2CU_OK;
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    static bool attr[64] = {false};
    if (s->device < 64 && !attr[s->device]) {
        CU_TRY(cudaFuncSetAttribute(gf2cu::trailing_update_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    gf2cu::kTableBytes));
        attr[s->device] = true;
    }
    gf2cu::Params p{};
    p.mat = s->mat;
    p.pb = s->pbl;
    p.info = s->info;
    p.stage = s->stage;
    p.state = s->lstate;
    p.m = (u32)s->m_loc;
    p.n = (u32)s->n;
    p.W = (u32)s->W;
    p.Wpad8 = (u32)s->Wpad8;
    gf2cu::trailing_update_kernel<<<num_sms(s->device), gf2cu::kTrailThreads, gf2cu::kTableBytes,
                                    st>>>(p, (u32)w);
    CU_TRY(cudaGetLastError());
    return GF2CU_OK;
}

gf2cu_status gf2cu_shard_finish(gf2cu_shard* s, size_t* swaps, size_t* q, size_t* rank,
                                uint32_t* perm, void* stream) {
    if (!s || !rank || !perm || ((!swaps || !q) && std::min(s->m, s->n) > 0))
        return fail(GF2CU_EINVAL, "null argument");
    DeviceGuard g(s->device);
    cudaStream_t st = shard_stream(s, stream);
    if (s->m_loc)
        gf2cu::untile_kernel<<<num_sms(s->device) * 8, 256, 0, st>>>(s->mat, s->data, nullptr,
                                                                    (u32)s->m_loc, (u32)s->Wp,
                                                                    (u32)s->Wpad8);
    CU_TRY(cudaGetLastError());
    gf2cu::StepState fin{};
    CU_TRY(cudaMemcpyAsync(&fin, s->gstate, sizeof(fin), cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaMemcpyAsync(perm, s->perm, s->m * 4, cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    const size_t rk = std::min<size_t>((size_t)fin.r + fin.rb, std::min(s->m, s->n));
    std::vector<u32> sw(rk), qq(rk);
    if (rk) {
        CU_TRY(cudaMemcpyAsync(sw.data(), s->swaps, rk * 4, cudaMemcpyDeviceToHost, st));
        CU_TRY(cudaMemcpyAsync(qq.data(), s->qcol, rk * 4, cudaMemcpyDeviceToHost, st));
        CU_TRY(cudaStreamSynchronize(st));
    }
    for (size_t i = 0; i < rk; ++i) {
        swaps[i] = sw[i];
        q[i] = qq[i];
    }
    *rank = rk;
    return GF2CU_OK;
}

// ------------------------------------------------------ row-sharded, peer
}  // extern "C"

struct gf2cu_peer {
    size_t m = 0, n = 0, W = 0, Wp = 0, Wp8 = 0;
    int device = 0;
    u64* data = nullptr;  // local rows, row-major (stride Wp)
    void* xbuf = nullptr; // this rank's exchange buffers (IPC-exported)
    std::vector<void*> allocs;
    std::vector<void*> opened;  // peers' exchange buffers mapped here
    gf2cu::PeerParams hp{};
    gf2cu::PeerParams* dp = nullptr;
    bool connected = false;
    bool super = false;  // the last run used two panels per sweep
    cudaStream_t own = nullptr;
};

namespace {
cudaStream_t peer_stream(gf2cu_peer* p, void* st) {
    return st ? reinterpret_cast<cudaStream_t>(st) : p->own;
}
}  // namespace

extern "C" {

gf2cu_status gf2cu_peer_create(size_t m, size_t n, int rank, int nranks, size_t block, int device,
                               gf2cu_peer** out) {
    if (!out) return fail(GF2CU_EINVAL, "out is null");
    *out = nullptr;
    if (nranks < 1 || nranks > gf2cu::kMaxRanks || rank < 0 || rank >= nranks || block == 0)
        return fail(GF2CU_EINVAL, "bad rank / nranks (1..8) / block");
    if (m >= (1ull << 31) || n >= (1ull << 31)) return fail(GF2CU_EINVAL, "dimensions exceed 2^31");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(GF2CU_ENODEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(GF2CU_EINVAL, "bad device ordinal");
    cudaDeviceProp pr;
    CU_TRY(cudaGetDeviceProperties(&pr, device));
    if (pr.major != 10) return fail(GF2CU_ENODEVICE, "device is not sm_100 (built for sm_100a only)");
    DeviceGuard g(device);
    apply_watchdog_env(device);
    auto* p = new (std::nothrow) gf2cu_peer;
    if (!p) return fail(GF2CU_ENOMEM, "host allocation failed");
    p->m = m;
    p->n = n;
    p->W = words_of(n);
    p->Wp = padded_stride(n);
    p->Wp8 = wpad8(p->W);
    p->device = device;
    gf2cu_status st = peer_alloc_rank(p->hp, p->allocs, m, n, (unsigned)rank, (unsigned)nranks,
                                      (unsigned)block, &p->xbuf);
    cudaError_t e = cudaSuccess;
    if (st == GF2CU_OK) {
        const size_t bytes = std::max<size_t>(1, p->hp.m_loc) * p->Wp * 8;
        e = cudaMalloc(&p->data, bytes);
        if (e == cudaSuccess) e = zero_now(p->data, bytes);
        if (e == cudaSuccess) e = zero_now(p->xbuf, peer_xbytes(m, p->Wp8));
        if (e == cudaSuccess) e = cudaMalloc(&p->dp, sizeof(gf2cu::PeerParams));
        if (e == cudaSuccess) e = h2d_now(p->dp, &p->hp, sizeof(p->hp));
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->own, cudaStreamNonBlocking);
    }
    if (st != GF2CU_OK || e != cudaSuccess) {
        gf2cu_peer_destroy(p);
        return st != GF2CU_OK ? st : cuda_fail(e, "gf2cu_peer_create");
    }
    p->connected = nranks == 1;
    *out = p;
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_destroy(gf2cu_peer* p) {
    if (!p) return GF2CU_OK;
    DeviceGuard g(p->device);
    cudaDeviceSynchronize();
    for (void* x : p->opened) cudaIpcCloseMemHandle(x);
    for (void* x : p->allocs) cudaFree(x);
    cudaFree(p->data);
    cudaFree(p->dp);
    if (p->own) cudaStreamDestroy(p->own);
    delete p;
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_info(const gf2cu_peer* p, size_t* m_local) {
    if (!p) return fail(GF2CU_EINVAL, "null peer");
    if (m_local) *m_local = p->hp.m_loc;
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_export(const gf2cu_peer* p, void* handle) {
    if (!p || !handle) return fail(GF2CU_EINVAL, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == GF2CU_PEER_HANDLE_BYTES, "IPC handle size");
    DeviceGuard g(p->device);
    cudaIpcMemHandle_t h;
    CU_TRY(cudaIpcGetMemHandle(&h, p->xbuf));
    std::memcpy(handle, &h, sizeof(h));
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_connect(gf2cu_peer* p, const void* handles) {
    if (!p || (!handles && p->hp.nranks > 1)) return fail(GF2CU_EINVAL, "null argument");
    DeviceGuard g(p->device);
    for (void* x : p->opened) cudaIpcCloseMemHandle(x);
    p->opened.clear();
    const unsigned G = p->hp.nranks, me = p->hp.rank;
    for (unsigned j = 0; j < G; ++j) {
        if (j == me) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(handles) + (size_t)j * GF2CU_PEER_HANDLE_BYTES, sizeof(h));
        void* ptr = nullptr;
        CU_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        p->opened.push_back(ptr);
        p->hp.peer[j] = peer_bufs_at(ptr, p->m, p->Wp8);
    }
    CU_TRY(h2d_now(p->dp, &p->hp, sizeof(p->hp)));
    p->connected = true;
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_ping(gf2cu_peer* p, uint32_t value, uint32_t* seen) {
    if (!p || !seen) return fail(GF2CU_EINVAL, "null argument");
    if (!p->connected) return fail(GF2CU_EINVAL, "gf2cu_peer_connect has not been called");
    DeviceGuard g(p->device);
    if (value) {
        gf2cu::peer_ping_kernel<<<1, 1, 0, p->own>>>(p->dp, value);
        CU_TRY(cudaGetLastError());
        CU_TRY(cudaStreamSynchronize(p->own));
    }
    CU_TRY(cudaMemcpy(seen, p->hp.peer[p->hp.rank].ctr + gf2cu::kCtrPing, p->hp.nranks * 4,
                      cudaMemcpyDeviceToHost));
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_upload(gf2cu_peer* p, const uint64_t* host, size_t host_stride, void* stream) {
    if (!p || (!host && p->hp.m_loc)) return fail(GF2CU_EINVAL, "null argument");
    if (host_stride < p->W) return fail(GF2CU_EINVAL, "host stride smaller than the row");
    if (!p->hp.m_loc || !p->W) return GF2CU_OK;
    DeviceGuard g(p->device);
    cudaStream_t st = peer_stream(p, stream);
    CU_TRY(cudaMemcpy2DAsync(p->data, p->Wp * 8, host, host_stride * 8, p->W * 8, p->hp.m_loc,
                             cudaMemcpyHostToDevice, st));
    CU_TRY(cudaStreamSynchronize(st));
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_download(const gf2cu_peer* p, uint64_t* host, size_t host_stride, void* stream) {
    if (!p || (!host && p->hp.m_loc)) return fail(GF2CU_EINVAL, "null argument");
    if (host_stride < p->W) return fail(GF2CU_EINVAL, "host stride smaller than the row");
    if (!p->hp.m_loc || !p->W) return GF2CU_OK;
    DeviceGuard g(p->device);
    cudaStream_t st = peer_stream(const_cast<gf2cu_peer*>(p), stream);
    CU_TRY(cudaMemcpy2DAsync(host, host_stride * 8, p->data, p->Wp * 8, p->W * 8, p->hp.m_loc,
                             cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_fill_ctr(gf2cu_peer* p, uint64_t seed, void* stream) {
    if (!p) return fail(GF2CU_EINVAL, "null peer");
    if (!p->hp.m_loc) return GF2CU_OK;
    DeviceGuard g(p->device);
    cudaStream_t st = peer_stream(p, stream);
    gf2cu::shard_fill_ctr_kernel<<<num_sms(p->device) * 8, 256, 0, st>>>(
        p->data, p->hp.m_loc, (u32)p->n, (u32)p->Wp, p->hp.rank, p->hp.nranks, p->hp.block, seed);
    CU_TRY(cudaGetLastError());
    CU_TRY(cudaStreamSynchronize(st));
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_reset(gf2cu_peer* p, void* stream) {
    if (!p) return fail(GF2CU_EINVAL, "null peer");
    DeviceGuard g(p->device);
    cudaStream_t st = peer_stream(p, stream);
    gf2cu_status s2 = peer_reset_rank(p->hp, st);
    if (s2 != GF2CU_OK) return s2;
    CU_TRY(cudaStreamSynchronize(st));
    return GF2CU_OK;
}

gf2cu_status gf2cu_peer_run(gf2cu_peer* p, void* stream, gf2cu_stats* stats) {
    if (!p) return fail(GF2CU_EINVAL, "null peer");
    if (!p->connected) return fail(GF2CU_EINVAL, "gf2cu_peer_connect has not been called");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (p->m == 0 || p->n == 0) return GF2CU_OK;
    DeviceGuard g(p->device);
    cudaStream_t st = peer_stream(p, stream);
    const int sms = num_sms(p->device);
    p->super = peer_super(p->m, p->W, 0u);
    const u32 wpad = p->super ? (u32)std::max<size_t>(4, (p->W + 3) / 4 * 4) : (u32)p->Wp8;
    if (p->hp.p.Wpad8 != wpad) {
        p->hp.p.Wpad8 = wpad;
        CU_TRY(h2d_now(p->dp, &p->hp, sizeof(p->hp)));
    }
    if (p->hp.m_loc) {
        if (p->super)
            gf2cu::tile4_kernel<<<sms * 8, 256, 0, st>>>(p->data, p->hp.mat, p->hp.m_loc, (u32)p->Wp, wpad);
        else
            gf2cu::tile_kernel<<<sms * 8, 256, 0, st>>>(p->data, p->hp.mat, p->hp.m_loc, (u32)p->Wp, wpad);
    }
    CU_TRY(cudaGetLastError());
    cudaEvent_t ev[2];
    CU_TRY(cudaEventCreate(&ev[0]));
    CU_TRY(cudaEventCreate(&ev[1]));
    CU_TRY(cudaEventRecord(ev[0], st));
    gf2cu_status s2 = peer_launch(p->dp, 1, (unsigned)sms, p->W, p->super, p->device, st);
    if (s2 == GF2CU_OK) {
        CU_TRY(cudaEventRecord(ev[1], st));
        if (p->hp.m_loc) {
            if (p->super)
                gf2cu::untile4_local_kernel<<<sms * 8, 256, 0, st>>>(p->hp.mat, p->data, p->hp.m_loc,
                                                                    (u32)p->Wp, wpad);
            else
                gf2cu::untile_kernel<<<sms * 8, 256, 0, st>>>(p->hp.mat, p->data, nullptr, p->hp.m_loc,
                                                             (u32)p->Wp, wpad);
        }
        CU_TRY(cudaGetLastError());
        CU_TRY(cudaStreamSynchronize(st));
        s2 = peer_outputs(p->hp, p->super, st, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, stats);
        if (s2 == GF2CU_OK && stats) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[0], ev[1]);
            stats->kernel_ms = ms;
        }
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    return s2;
}

gf2cu_status gf2cu_peer_finish(gf2cu_peer* p, size_t* swaps, size_t* q, size_t* rank, uint32_t* perm,
                               void* stream) {
    if (!p || !rank || !perm || ((!swaps || !q) && std::min(p->m, p->n) > 0))
        return fail(GF2CU_EINVAL, "null argument");
    *rank = 0;
    if (p->m == 0 || p->n == 0) {
        for (size_t i = 0; i < p->m; ++i) perm[i] = (uint32_t)i;
        return GF2CU_OK;
    }
    DeviceGuard g(p->device);
    return peer_outputs(p->hp, p->super, peer_stream(p, stream), swaps, q, rank, nullptr, nullptr, perm,
                        nullptr);
}

gf2cu_status gf2cu_fill_random(uint64_t* words, size_t m, size_t n, size_t stride, double density,
                               uint64_t seed) {
    // The same engine and draw order as gf2::fill_random (bit_matrix.hpp:459-486).
    if (density < 0.0 || density > 1.0) return fail(GF2CU_EINVAL, "density outside [0,1]");
    const size_t W = words_of(n);
    if (m && W && !words) return fail(GF2CU_EINVAL, "null words");
    if (stride < W) return fail(GF2CU_EINVAL, "stride smaller than the row");
    std::mt19937_64 rng(seed);
    const u64 last = (n & 63) ? ((1ull << (n & 63)) - 1ull) : ~0ull;
    for (size_t i = 0; i < m; ++i) {
        u64* row = reinterpret_cast<u64*>(words) + i * stride;
        for (size_t x = 0; x < W; ++x) {
            u64 v;
            if (density == 0.0)
                v = 0;
            else if (density == 1.0)
                v = ~0ull;
            else if (density == 0.5)
                v = rng();
            else {
                v = 0;
                for (unsigned b = 0; b < 64; ++b) {
                    const double u = double(rng() >> 11) * 0x1.0p-53;
                    v |= u64(u < density) << b;
                }
            }
            row[x] = v;
        }
        if (W) row[W - 1] &= last;
    }
    return GF2CU_OK;
}

gf2cu_status gf2cu_fill_random_rows(uint64_t* words, size_t m, size_t n, size_t stride, size_t nnz,
                                    uint64_t seed) {
    // gf2::fill_random_rows (bit_matrix.hpp:489-520): exactly nnz ones per
    // row, same engine and draw order (partial Fisher-Yates when nnz > n/2,
    // rejection sampling otherwise; bounded draws by masked rejection).
    if (nnz > n) return fail(GF2CU_EINVAL, "nnz exceeds column count");
    const size_t W = words_of(n);
    if (m && W && !words) return fail(GF2CU_EINVAL, "null words");
    if (stride < W) return fail(GF2CU_EINVAL, "stride smaller than the row");
    std::mt19937_64 rng(seed);
    auto bounded = [&](u64 lim) -> u64 {
        if (lim == 1) return 0;
        const int bits = 64 - __builtin_clzll(lim - 1);
        const u64 mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
        u64 v;
        do {
            v = rng() & mask;
        } while (v >= lim);
        return v;
    };
    std::vector<u32> pool;
    for (size_t i = 0; i < m; ++i) {
        u64* row = reinterpret_cast<u64*>(words) + i * stride;
        std::fill(row, row + W, 0ull);
        if (nnz * 2 > n) {
            pool.resize(n);
            for (size_t j = 0; j < n; ++j) pool[j] = (u32)j;
            for (size_t j = 0; j < nnz; ++j) {
                const size_t pick = j + (size_t)bounded(n - j);
                std::swap(pool[j], pool[pick]);
                row[pool[j] >> 6] |= 1ull << (pool[j] & 63);
            }
        } else {
            size_t placed = 0;
            while (placed < nnz) {
                const size_t q = (size_t)bounded(n);
                const u64 bit = 1ull << (q & 63);
                if (!(row[q >> 6] & bit)) {
                    row[q >> 6] |= bit;
                    ++placed;
                }
            }
        }
    }
    return GF2CU_OK;
}

gf2cu_status gf2cu_fill_ctr(uint64_t* words, size_t m, size_t n, size_t stride, uint64_t seed) {
    const size_t W = words_of(n);
    if (m && W && !words) return fail(GF2CU_EINVAL, "null words");
    if (stride < W) return fail(GF2CU_EINVAL, "stride smaller than the row");
    const u64 base = seed << 32;
    const u64 last = (n & 63) ? ((1ull << (n & 63)) - 1ull) : ~0ull;
    for (size_t i = 0; i < m; ++i) {
        u64* row = reinterpret_cast<u64*>(words) + i * stride;
        for (size_t x = 0; x < W; ++x) {
            u64 z = base + (u64(i) * W + x + 1ull) * 0x9e3779b97f4a7c15ull;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            row[x] = z ^ (z >> 31);
        }
        if (W) row[W - 1] &= last;
    }
    return GF2CU_OK;
}

gf2cu_status gf2cu_stream_in_plan(size_t m, size_t words_per_row, int pageable, size_t* rows, unsigned* steps,
                                  size_t* blocks) {
    if (!rows || !steps || !blocks) return fail(GF2CU_EINVAL, "null argument");
    *blocks = 0;
    if (m == 0 || words_per_row == 0) return GF2CU_OK;
    const StreamInPlan pl = stream_in_plan(m, words_per_row, pageable != 0);
    *blocks = pl.rows.size();
    for (size_t k = 0; k < pl.rows.size(); ++k) {
        rows[k] = pl.rows[k];
        steps[k] = pl.steps[k];
    }
    return GF2CU_OK;
}

// Message-passing litmus runs of the drivers' hand-offs (litmus.cuh).
gf2cu_status gf2cu_litmus(int kind, unsigned rounds, int device, unsigned long long* checked,
                          unsigned long long* failures) {
    if (!checked || !failures || kind < 0 || kind > 3) return fail(GF2CU_EINVAL, "bad litmus arguments");
    *checked = *failures = 0;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(GF2CU_ENODEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(GF2CU_EINVAL, "bad device ordinal");
    DeviceGuard g(device);
    apply_watchdog_env(device);
    const int sms = num_sms(device);
    gf2cu::LitmusParams L{};
    L.rounds = rounds;
    L.kind = (u32)kind;
    std::vector<void*> allocs;
    auto alloc = [&](void** ptr, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(ptr, bytes);
        if (e == cudaSuccess) {
            allocs.push_back(*ptr);
            e = zero_now(*ptr, bytes);
        }
        return e;
    };
    auto cleanup = [&]() {
        for (void* x : allocs) cudaFree(x);
    };
    cudaError_t e = cudaSuccess;
    const u32 G = kind == 3 ? (u32)sms * 2u : (u32)sms;
    if (kind == 3) {
        e = alloc((void**)&L.out, (size_t)rounds * G * gf2cu::kLitmusWords * 8);
    } else {
        e = alloc((void**)&L.data, (size_t)2 * G * gf2cu::kLitmusWords * 8);
        if (e == cudaSuccess) e = alloc((void**)&L.ctr, (size_t)rounds * 4 + 4);
        if (e == cudaSuccess) e = alloc((void**)&L.ctr2, (size_t)rounds * 4 + 4);
        if (e == cudaSuccess) e = alloc((void**)&L.done, (size_t)rounds * 4 + 4);
    }
    if (e == cudaSuccess) e = alloc((void**)&L.err, 4);
    if (e == cudaSuccess) e = alloc((void**)&L.checked, 8);
    if (e == cudaSuccess) e = alloc((void**)&L.failures, 8);
    if (e == cudaSuccess) e = alloc((void**)&L.out_count, 4);
    if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(e, "litmus allocation");
    }
    unsigned long long h_checked = 0, h_fail = 0;
    if (kind < 3) {
        void* args[] = {&L};
        e = cudaLaunchCooperativeKernel((void*)gf2cu::litmus_kernel, dim3(G), dim3(512), args, 0, nullptr);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        u32 err = 0;
        if (e == cudaSuccess) e = cudaMemcpy(&err, L.err, 4, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(&h_checked, L.checked, 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(&h_fail, L.failures, 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && err) {
            cleanup();
            return fail(GF2CU_ECUDA, "litmus watchdog tripped");
        }
    } else {
        // the host side of the streamed output: poll the mapped word, copy
        // each published round on a second stream, compare
        u32* flag = nullptr;
        u32* flag_dev = nullptr;
        cudaStream_t ks = nullptr, cs = nullptr;
        e = cudaHostAlloc(&flag, 4, cudaHostAllocMapped);
        if (e == cudaSuccess) {
            *reinterpret_cast<volatile u32*>(flag) = 0;
            e = cudaHostGetDevicePointer(&flag_dev, flag, 0);
        }
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        std::vector<u64> host((size_t)G * gf2cu::kLitmusWords);
        if (e == cudaSuccess) {
            L.host_flag = flag_dev;
            gf2cu::litmus_host_kernel<<<G, 256, 0, ks>>>(L);
            e = cudaGetLastError();
        }
        u32 seen = 0;
        const auto t0 = std::chrono::steady_clock::now();
        while (e == cudaSuccess && seen < rounds) {
            const u32 avail = *reinterpret_cast<volatile u32*>(flag);
            for (; seen < avail; ++seen) {
                e = cudaMemcpyAsync(host.data(), L.out + (size_t)seen * G * gf2cu::kLitmusWords,
                                    host.size() * 8, cudaMemcpyDeviceToHost, cs);
                if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
                if (e != cudaSuccess) break;
                for (u32 c = 0; c < G; ++c)
                    for (u32 i = 0; i < gf2cu::kLitmusWords; ++i) {
                        const u64 x = (u64)seen << 40 ^ (u64)c << 20 ^ (u64)i ^ 0x9e3779b97f4a7c15ull;
                        u64 z = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
                        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
                        z ^= z >> 31;
                        h_fail += host[(size_t)c * gf2cu::kLitmusWords + i] != z;
                    }
                h_checked += (unsigned long long)G * gf2cu::kLitmusWords;
            }
            const cudaError_t q = cudaStreamQuery(ks);
            if (q != cudaSuccess && q != cudaErrorNotReady) e = q;
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) {
                e = cudaErrorLaunchTimeout;
                break;
            }
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(ks);
        if (ks) cudaStreamDestroy(ks);
        if (cs) cudaStreamDestroy(cs);
        if (flag) cudaFreeHost(flag);
    }
    cleanup();
    if (e != cudaSuccess) return cuda_fail(e, "litmus");
    *checked = h_checked;
    *failures = h_fail;
    return GF2CU_OK;
}

}  // extern "C"
