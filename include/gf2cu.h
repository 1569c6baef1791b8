/*
 * gf2cu.h -- C ABI of the B200 (sm_100a) block-iterative PLE over F2.
 *
 * This is the drop-in boundary for the reference's hot path
 *     gf2::PleOutcome gf2::block_iterative_ple(gf2::MatrixView a,
 *                                              const gf2::PleConfig& cfg = {})
 * (/root/reference/proj/include/gf2/ple.hpp:166). The reference has no FFI of
 * its own (it is a header-only C++20 library); the C++ wrapper in
 * include/gf2cu/ple.hpp re-exposes these entry points under the reference's
 * names and types, and INTEGRATION.md shows the binding a maintainer adds.
 *
 * Plain pointers and sizes only; no CUDA or torch types cross this boundary
 * (streams are passed as opaque `void*` = cudaStream_t, NULL = the library's
 * own stream). Every call is synchronous with respect to its outputs unless
 * stated otherwise. Errors are status codes; gf2cu_last_error() returns a
 * thread-local message for the last failing call on the calling thread.
 */
#ifndef GF2CU_H
#define GF2CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GF2CU_OK = 0,
    GF2CU_EINVAL = 1,    /* bad argument: std::invalid_argument in the wrapper   */
    GF2CU_ERANGE = 2,    /* view/window outside matrix: std::out_of_range         */
    GF2CU_ENOMEM = 3,    /* device or host allocation failed: std::bad_alloc      */
    GF2CU_ECUDA = 4,     /* CUDA runtime error (no device, launch failure, ...)   */
    GF2CU_ENODEVICE = 5, /* no sm_100 device visible                              */
    GF2CU_ECHECK = 6     /* GF2CU_FLAG_CHECK: a device invariant was violated     */
} gf2cu_status;

/* Mirrors gf2::MatrixView (bit_matrix.hpp:223-227, 245-250): row-major uint64
 * words, LSB-first (column c at bit (c & 63) of word (c >> 6) counted from
 * col_off), `stride` words between rows, window of nrows x ncols starting at
 * bit col_off of each row. Bits outside the window are never modified. */
typedef struct {
    uint64_t* data;
    size_t stride;
    size_t col_off;
    size_t nrows;
    size_t ncols;
} gf2cu_view;

/* Mirrors gf2::PleConfig (ple.hpp:31-39). The reference's output does not
 * depend on k or table_count; they are accepted and
 * validated (k clamped to [1,16], table_count >= 1, ple.hpp:168-169, 201) but
 * the device path always factors 64-column panels. */
typedef struct {
    unsigned k;            /* 0 = pick (reference: pick_table_bits)          */
    double k_scale;        /* reference default 0.75                         */
    unsigned table_count;  /* reference default 4                            */
    int device;            /* CUDA device ordinal                            */
    void* stream;          /* cudaStream_t or NULL                           */
    unsigned flags;        /* GF2CU_FLAG_*                                   */
} gf2cu_cfg;

#define GF2CU_FLAG_TIME_KERNELS 1u /* record CUDA events / device timestamps */
#define GF2CU_FLAG_MULTI_KERNEL 2u /* one launch per phase instead of the
                                      persistent cooperative kernel          */
#define GF2CU_FLAG_SINGLE_PANEL 4u /* force the persistent kernel with one
                                      64-column panel per trailing sweep     */
#define GF2CU_FLAG_SUPER_STEP 8u   /* force the super-step kernel: two panels
                                      per sweep (default: chosen by size --
                                      super-step from 5*2^20 matrix words)     */
#define GF2CU_FLAG_CHECK 32u       /* check mode (also: environment variable
                                      GF2CU_CHECK=1): every step asserts
                                      SURVEY 8(c) invariant (iv) on every row's
                                      panel word, the result invariants (i),
                                      (ii); a violation returns GF2CU_ECHECK
                                      naming the first violating step. Single-
                                      device drivers (emulated peer ranks
                                      included); slower.                      */

/* The device-driven row-sharded driver (ple_peer.cuh)
 * with g = 1..8 ranks emulated on the one device: one cooperative launch,
 * sms/g CTAs per rank, the ranks exchanging panel words and pivot tails
 * through each other's buffers exactly as they do over NVLink peer memory
 * when each rank owns a GPU. Same outputs as every other driver. */
#define GF2CU_FLAG_PEER_RANKS(g) ((((unsigned)(g)) & 15u) << 16)

/* Mirrors gf2::ColSwap (ple.hpp:41-43). */
typedef struct {
    size_t a, b, from_row;
} gf2cu_colswap;

/* Per-call measurements of the device path. */
typedef struct {
    size_t steps;               /* 64-column panel steps executed               */
    size_t trailing_launches;   /* trailing_update launches that did work       */
    double trailing_ms;         /* trailing-update time (events or timestamps)  */
    double panel_ms;            /* panel-factor time                            */
    double coef_ms;             /* apply + stage time                           */
    double alg_bytes;           /* sum over steps of 16*(m-r-rb)*(W-w-1)        */
    double h2d_bytes, d2h_bytes;/* host<->device bytes moved by gf2cu_ple       */
    double kernel_ms;           /* persistent kernel duration (CUDA events)     */
    int driver;                 /* 4 / 3 = row-sharded over peer memory with two /
                                   one panels per sweep, 2 = super-step (two
                                   panels per sweep), 1 = persistent single-panel,
                                   0 = per phase                                */
    double sweep_bytes;         /* bytes the trailing sweeps move: alg_bytes for
                                   one panel per sweep; for the super-step driver
                                   sum over super-steps of 16*(m-r-rba-rbb)*(W-w-2)
                                   (one read + write per two panels)            */
    size_t input_first_rows;    /* gf2cu_ple, streamed input: the factorization
                                   started on this many leading rows ...        */
    size_t input_first_steps;   /* ... and this many 128-column super-steps had
                                   run when the last row block joined
                                   (0 / 0: the matrix was uploaded whole)       */
    size_t input_blocks;        /* row blocks the upload was cut into (0: whole) */
} gf2cu_stats;

/* Fills *cfg with the reference defaults (k=0, k_scale=0.75, table_count=4,
 * device 0, library stream, no flags). */
void gf2cu_default_config(gf2cu_cfg* cfg);

/* The drop-in: block_iterative_ple on a HOST view, in place. Uploads the
 * window, factors it on the device, writes L\E back into the window.
 * swaps and q need capacity min(nrows, ncols); col_swaps needs capacity
 * min(nrows, ncols) (the canonical compression list {j, q[j], j} for
 * q[j] != j). Any of col_swaps/n_col_swaps/stats may be NULL. */
gf2cu_status gf2cu_ple(const gf2cu_view* a, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                       size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                       gf2cu_stats* stats);

/* Replaces gf2::partial_ple(MatrixView a) (ple.hpp:57-130), the lazy
 * single-pass PLE, in place on a HOST view. rank, q, swaps and col_swaps are
 * the reference's; *processed = its watermark: rows [processed, nrows) are
 * left untouched, which happens only when rank < nrows and the pivot columns
 * run consecutively from q[0] to column ncols-1 (no pivotless column after
 * the first pivot); otherwise processed = nrows and the in-place result
 * equals gf2cu_ple's; rank 0 gives processed 0. Capacities as gf2cu_ple. */
gf2cu_status gf2cu_partial_ple(const gf2cu_view* a, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                               size_t* rank, size_t* processed, gf2cu_colswap* col_swaps,
                               size_t* n_col_swaps);

/* Replaces gf2::undo_column_swaps(MatrixView a, const std::vector<ColSwap>&)
 * (ple.hpp:293-296): replays the compression swaps backwards,
 * swap_cols_from_row(a, b, from_row) each (bit_matrix.hpp:302-318), on the
 * device. GF2CU_ERANGE if a swap lies outside the view. */
gf2cu_status gf2cu_undo_column_swaps(const gf2cu_view* a, const gf2cu_colswap* col_swaps,
                                     size_t n_col_swaps, const gf2cu_cfg* cfg);

/* Thread-local message of the last failing call ("" if none). */
const char* gf2cu_last_error(void);

/* Library / device info: number of visible devices with compute capability
 * 10.x, or a negative status. */
int gf2cu_device_count(void);
const char* gf2cu_version(void);

/* ------------------------------------------------------------------ */
/* Device-resident matrices (benchmarking without PCIe, multi-step use) */
/* ------------------------------------------------------------------ */
typedef struct gf2cu_matrix gf2cu_matrix;

/* An m x n zero matrix in HBM with 128-byte-aligned rows of
 * stride_words = roundup(ceil(n/64), 16) words; padding bits stay zero. */
gf2cu_status gf2cu_matrix_create(size_t m, size_t n, int device, gf2cu_matrix** out);
gf2cu_status gf2cu_matrix_destroy(gf2cu_matrix* a);
gf2cu_status gf2cu_matrix_info(const gf2cu_matrix* a, size_t* m, size_t* n, size_t* stride_words,
                               uint64_t** device_ptr);
/* Host <-> device copies; host rows are host_stride words apart and hold
 * ceil(n/64) words of data each. Synchronous on `stream`. */
gf2cu_status gf2cu_matrix_upload(gf2cu_matrix* a, const uint64_t* host, size_t host_stride,
                                 void* stream);
gf2cu_status gf2cu_matrix_download(const gf2cu_matrix* a, uint64_t* host, size_t host_stride,
                                   void* stream);
/* Copy another device matrix of the same shape (device to device). */
gf2cu_status gf2cu_matrix_copy(gf2cu_matrix* dst, const gf2cu_matrix* src, void* stream);
/* Device-side generator: the F2-nonlinear counter generator of SURVEY.md
 * section 8(d) (same words as the host generator gf2cu_fill_ctr). */
gf2cu_status gf2cu_matrix_fill_ctr(gf2cu_matrix* a, uint64_t seed, void* stream);
/* FNV-1a-style device checksum of the logical words (row-major, W words per
 * row, padding excluded) -- a size-independent parity handle. */
gf2cu_status gf2cu_matrix_checksum(const gf2cu_matrix* a, uint64_t* out, void* stream);

/* block_iterative_ple on a device-resident matrix, in place. Same outputs as
 * gf2cu_ple. Asynchronous work is complete when the call returns. */
gf2cu_status gf2cu_ple_device(gf2cu_matrix* a, const gf2cu_cfg* cfg, size_t* swaps, size_t* q,
                              size_t* rank, gf2cu_colswap* col_swaps, size_t* n_col_swaps,
                              gf2cu_stats* stats);

/* undo_column_swaps on a device-resident matrix. */
gf2cu_status gf2cu_undo_column_swaps_device(gf2cu_matrix* a, const gf2cu_colswap* col_swaps,
                                            size_t n_col_swaps, void* stream);

/* ------------------------------------------------------------------ */
/* Echelon forms and the upper-triangular solve     */
/* ------------------------------------------------------------------ */
/* Replaces gf2::rref_from_ple(MatrixView a, const PleOutcome& out, bool full,
 * const MulConfig&) (ple.hpp:318-329). `a` holds the in-place result of a
 * full PLE (block_iterative_ple / recursive_ple, processed == nrows) whose
 * pivot columns are q[0..rank); the outcome's col_swaps are implied by q
 * (any compression-swap list of that PLE undoes to the same matrix). On
 * return the top `rank` rows hold the row echelon form (reduced if full),
 * the rows below are zero. GF2CU_EINVAL if q is not strictly increasing
 * inside the matrix or rank exceeds min(m, n) (check_pivots, ple.hpp:299). */
gf2cu_status gf2cu_rref_from_ple(const gf2cu_view* a, const size_t* q, size_t rank, int full,
                                 const gf2cu_cfg* cfg);
gf2cu_status gf2cu_rref_from_ple_device(gf2cu_matrix* a, const size_t* q, size_t rank, int full,
                                        void* stream);
/* Replaces gf2::echelonize(a, EchelonStrategy::ple_iterative, full, cfg)
 * (m4ri.hpp:88-98): block_iterative_ple followed by rref_from_ple, the matrix
 * resident on the device in between. *rank = the rank. */
gf2cu_status gf2cu_echelonize(const gf2cu_view* a, int full, const gf2cu_cfg* cfg, size_t* rank);
gf2cu_status gf2cu_echelonize_device(gf2cu_matrix* a, int full, const gf2cu_cfg* cfg, size_t* rank);
/* Replaces gf2::trsm_upper_left_unit(ConstMatrixView u, MatrixView b,
 * const MulConfig&) (multiply.hpp:314-335): b <- u^-1 b for the unit upper
 * triangle of the r x r view u (bits strictly above the diagonal read, the
 * rest ignored); b is r x ncols. GF2CU_EINVAL on a dimension mismatch. */
gf2cu_status gf2cu_trsm_upper_left_unit(const gf2cu_view* u, const gf2cu_view* b,
                                        const gf2cu_cfg* cfg);

/* ------------------------------------------------------------------ */
/* GF(2) matrix product                              */
/* ------------------------------------------------------------------ */
/* Replace gf2::mul(ConstMatrixView a, ConstMatrixView b, const MulConfig&)
 * (multiply.hpp:266-274; here c = a * b into the caller's c) and gf2::addmul
 * (multiply.hpp:254-264; c ^= a * b). The product is unique, so the result
 * does not depend on the reference's kernel choice (M4RM / Strassen) or on
 * MulConfig. GF2CU_EINVAL on a dimension mismatch (check_mul_shapes,
 * multiply.hpp:33-37); c must alias neither operand. */
gf2cu_status gf2cu_mul(const gf2cu_view* c, const gf2cu_view* a, const gf2cu_view* b,
                       const gf2cu_cfg* cfg);
gf2cu_status gf2cu_addmul(const gf2cu_view* c, const gf2cu_view* a, const gf2cu_view* b,
                          const gf2cu_cfg* cfg);
/* Device-resident form: c = a * b (accumulate = 0) or c ^= a * b. */
gf2cu_status gf2cu_matrix_mul(gf2cu_matrix* c, const gf2cu_matrix* a, const gf2cu_matrix* b,
                              int accumulate, void* stream);

/* ------------------------------------------------------------------ */
/* Row-sharded multi-GPU PLE (one process per GPU, host-driven steps)   */
/* ------------------------------------------------------------------ */
/* Global row g lives on rank (g / block) % nranks, local index
 * (g / (block * nranks)) * block + g % block. Each rank holds its rows plus
 * the replicated position state; the orchestration (collectives) is done by
 * the caller, see paper_1111_6549_b200/shard.py and DESIGN.md section 8.
 * All calls are asynchronous on `stream` except gf2cu_shard_panel (returns
 * the status words) and gf2cu_shard_finish / download. Buffers passed as
 * device pointers (pos_words, pack) are caller-owned device memory. */
typedef struct gf2cu_shard gf2cu_shard;

#define GF2CU_SHARD_STATUS_WORDS(nranks) (8 + 2 * (nranks))

gf2cu_status gf2cu_shard_create(size_t m, size_t n, int rank, int nranks, size_t block, int device,
                                gf2cu_shard** out);
gf2cu_status gf2cu_shard_destroy(gf2cu_shard* s);
/* m_local rows on this rank; pack_words = u64 capacity the pack buffer needs. */
gf2cu_status gf2cu_shard_info(const gf2cu_shard* s, size_t* m_local, size_t* pack_words);
/* Local rows in local order, host_stride words apart. */
gf2cu_status gf2cu_shard_upload(gf2cu_shard* s, const uint64_t* host, size_t host_stride,
                                void* stream);
gf2cu_status gf2cu_shard_download(const gf2cu_shard* s, uint64_t* host, size_t host_stride,
                                  void* stream);
/* Device-side ctr generator for this rank's rows. */
gf2cu_status gf2cu_shard_fill_ctr(gf2cu_shard* s, uint64_t seed, void* stream);
/* Start a factorization: tile-major working copy, replicated state reset. */
gf2cu_status gf2cu_shard_begin(gf2cu_shard* s, void* stream);
/* pos_words[lo, hi) := 0 then this rank's active rows' panel words at their
 * positions (the caller all-reduces (sum) that range across ranks). */
gf2cu_status gf2cu_shard_gather(gf2cu_shard* s, uint64_t* pos_words, size_t lo, size_t hi,
                                void* stream);
/* Panel factorization of step w from the all-reduced pos_words; window_only
 * = 1 aborts on a window miss (status[0] = 1, nothing changed). status_out
 * receives GF2CU_SHARD_STATUS_WORDS(nranks) words: [0] miss, [1] rb, [2] r,
 * [8 + 2o], [9 + 2o] = low/high half of rank o's pivot bitmask. */
gf2cu_status gf2cu_shard_panel(gf2cu_shard* s, size_t w, uint64_t* pos_words, int window_only,
                               uint32_t* status_out, void* stream);
/* Apply step w to the local rows; packs this rank's pivot tails into pack. */
gf2cu_status gf2cu_shard_apply(gf2cu_shard* s, size_t w, uint64_t* pack, void* stream);
/* Stage owner rank's packed pivot tails (bitmask mask) for step w. */
/* Asynchronous step protocol (no host decision per step; used by
 * paper_1111_6549_b200/shard.py):
 *   gather(0, m) into a zeroed buffer -> sum all-reduce -> panel(window_only
 *   = 0, status_out = NULL: nothing is read back) -> pack_stage (this rank's
 *   pivot tails straight into the stage layout, the rest zeroed) -> sum
 *   all-reduce of the stage (disjoint contributions) -> apply(pack = NULL)
 *   -> trailing.
 * set_stage makes the library use the caller's stage buffer (64 rows x
 * Wpad8 words, tile-major) so the collective can run on it in place; pivots
 * returns the pivots found so far (synchronous, for a lagged stop check). */
gf2cu_status gf2cu_shard_pack_stage(gf2cu_shard* s, size_t w, void* stream);
/* The same protocol in three calls per step: step_gather (zero + gather the
 * active column), step_panel (panel + pack_stage), step_update (apply +
 * trailing); the caller all-reduces the column after step_gather and the
 * stage after step_panel. */
gf2cu_status gf2cu_shard_step_gather(gf2cu_shard* s, size_t w, uint64_t* pos_words, void* stream);
gf2cu_status gf2cu_shard_step_panel(gf2cu_shard* s, size_t w, uint64_t* pos_words, void* stream);
gf2cu_status gf2cu_shard_step_update(gf2cu_shard* s, size_t w, void* stream);
gf2cu_status gf2cu_shard_set_stage(gf2cu_shard* s, uint64_t* stage);
gf2cu_status gf2cu_shard_pivots(gf2cu_shard* s, size_t* pivots, void* stream);
gf2cu_status gf2cu_shard_unpack(gf2cu_shard* s, size_t w, uint64_t mask, const uint64_t* pack,
                                void* stream);
/* Trailing update of step w on the local rows. */
gf2cu_status gf2cu_shard_trailing(gf2cu_shard* s, size_t w, void* stream);
/* End: local rows back to row-major (gf2cu_shard_download reads them), and the
 * replicated outcome: swaps/q (capacity min(m,n)), rank, and perm[m] =
 * global row id at each final position (the caller assembles rows). */
gf2cu_status gf2cu_shard_finish(gf2cu_shard* s, size_t* swaps, size_t* q, size_t* rank,
                                uint32_t* perm, void* stream);

/* ------------------------------------------------------------------ */
/* Row-sharded multi-GPU PLE driven on the device (one process per GPU) */
/* ------------------------------------------------------------------ */
/* The same block-cyclic row distribution as gf2cu_shard_*, but the whole
 * factorization is ONE persistent kernel per rank (ple_peer.cuh): the ranks
 * exchange panel words and pivot-row tails by storing into each other's
 * exchange buffers over NVLink (CUDA IPC mappings) and signalling
 * system-scope counters; no host call or collective per step. Sequence per
 * rank (paper_1111_6549_b200/peer.py):
 *   create -> export (IPC handle of this rank's exchange buffers) -> the
 *   caller all-gathers the handles -> connect(all handles, rank order) ->
 *   upload / fill_ctr -> [reset -> barrier across ranks -> run -> finish ->
 *   download]*.
 * run blocks until this rank's kernel is done; all ranks must run
 * concurrently (one process per GPU). A rank stuck waiting on another trips
 * the kernel watchdog (GF2CU_ECUDA) instead of hanging. With nranks = 1,
 * connect may be skipped. */
typedef struct gf2cu_peer gf2cu_peer;

#define GF2CU_PEER_HANDLE_BYTES 64 /* sizeof(cudaIpcMemHandle_t) */

gf2cu_status gf2cu_peer_create(size_t m, size_t n, int rank, int nranks, size_t block, int device,
                               gf2cu_peer** out);
gf2cu_status gf2cu_peer_destroy(gf2cu_peer* p);
gf2cu_status gf2cu_peer_info(const gf2cu_peer* p, size_t* m_local);
gf2cu_status gf2cu_peer_export(const gf2cu_peer* p, void* handle);
/* handles: nranks x GF2CU_PEER_HANDLE_BYTES in rank order (own entry ignored). */
gf2cu_status gf2cu_peer_connect(gf2cu_peer* p, const void* handles);
/* Local rows in local order, host_stride words apart. */
gf2cu_status gf2cu_peer_upload(gf2cu_peer* p, const uint64_t* host, size_t host_stride, void* stream);
gf2cu_status gf2cu_peer_download(const gf2cu_peer* p, uint64_t* host, size_t host_stride,
                                 void* stream);
gf2cu_status gf2cu_peer_fill_ctr(gf2cu_peer* p, uint64_t seed, void* stream);
/* Diagnostic of the peer mappings (no kernel waits on another): with value
 * != 0, store it into word `rank` of every rank's marker block through the
 * mappings; then read this rank's markers (nranks words; 0 = not received)
 * into seen. gf2cu_peer_reset clears them. */
gf2cu_status gf2cu_peer_ping(gf2cu_peer* p, uint32_t value, uint32_t* seen);
/* Zero this rank's counters; every rank must reset before any rank runs. */
gf2cu_status gf2cu_peer_reset(gf2cu_peer* p, void* stream);
/* The factorization of this rank's rows (stats: steps, alg_bytes of the whole
 * matrix, kernel_ms of this rank's launch). */
gf2cu_status gf2cu_peer_run(gf2cu_peer* p, void* stream, gf2cu_stats* stats);
/* Replicated outcome (as gf2cu_shard_finish); local rows then download. */
gf2cu_status gf2cu_peer_finish(gf2cu_peer* p, size_t* swaps, size_t* q, size_t* rank,
                               uint32_t* perm, void* stream);

/* ------------------------------------------------------------------ */
/* Host-side input generators (bench/test inputs; not the hot path)     */
/* ------------------------------------------------------------------ */
/* gf2::fill_random (bit_matrix.hpp:459-486), mt19937_64-driven. */
gf2cu_status gf2cu_fill_random(uint64_t* words, size_t m, size_t n, size_t stride, double density,
                               uint64_t seed);
/* SURVEY.md 8(d) counter generator. */
/* gf2::fill_random_rows (bit_matrix.hpp:489-520): exactly nnz ones per row,
 * the reference's engine and draw order. GF2CU_EINVAL if nnz > n. */
gf2cu_status gf2cu_fill_random_rows(uint64_t* words, size_t m, size_t n, size_t stride, size_t nnz,
                                    uint64_t seed);
gf2cu_status gf2cu_fill_ctr(uint64_t* words, size_t m, size_t n, size_t stride, uint64_t seed);

/* ------------------------------------------------------------------ */
/* Diagnostics                                                          */
/* ------------------------------------------------------------------ */
/* Message-passing litmus runs of the persistent drivers' cross-CTA
 * hand-offs, built from the same primitives (csrc/litmus.cuh): kind 0 = CTA
 * arrival (bar.sync + red.release.gpu) -> ld.acquire.gpu spin -> ldcg reads
 * (pre-work -> panel capture); 1 = the same awaited with the two-counter spin
 * (t_count + chunk count -> table sources); 2 = system scope (the peer
 * drivers' fence.sc.sys + red.release.sys -> ld.acquire.sys); 3 = streamed
 * output to the host (threadfence + last arrival's threadfence_system +
 * mapped-memory flag -> host poll -> async copy). `rounds` rounds on every
 * SM; *checked = payload words verified, *failures = stale or torn words. */
gf2cu_status gf2cu_litmus(int kind, unsigned rounds, int device, unsigned long long* checked,
                          unsigned long long* failures);

/* Diagnostic (host only, no device needed): the row-block plan gf2cu_ple
 * would use to stream an m x (64 W)-column host matrix in:
 * rows[k] = the k-th block's end row, steps[k] = the 128-column super-steps
 * done when block k joins (steps[0] = 0); *blocks = their number, 0 = the
 * matrix is uploaded whole. rows / steps need capacity 8. The plan obeys
 * GF2CU_STREAM_IN, GF2CU_STREAM_IN_BLOCKS / _FRAC / _STEPS like the call. */
gf2cu_status gf2cu_stream_in_plan(size_t m, size_t words_per_row, int pageable, size_t* rows, unsigned* steps,
                                  size_t* blocks);

#ifdef __cplusplus
}
#endif

#endif /* GF2CU_H */
