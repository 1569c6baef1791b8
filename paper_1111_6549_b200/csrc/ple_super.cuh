// ple_super.cuh -- super-step persistent driver: two 64-column panels per
// trailing sweep (K = 128).
//
// The trailing sweep is bound by the L1 data pipe (8 table lookups of 64 B
// per 64 B of row plus the global load and store). Fusing two panels into one
// sweep keeps the lookups per panel but halves the global traffic and the
// per-step synchronization. Because every row's update is a combination of
// RAW pivot rows, two panels a, b fuse exactly:
//
//   new_tail = d~_a . R_a  ^  d_b . R_b,      d~_a = d_a ^ d_b . C
//
// R_a, R_b = the 64 + 64 pivot rows as they were before the super-step
// (read in place; their own swept tails go to ubuf), d_a / d_b = the row's
// combinations for panel a (from its word w) and panel b (from its word w+1
// after panel a), C[t] = the panel-a combination of panel b's t-th pivot row.
// 16 tables x 256 entries do not fit as 64-byte entries, so this driver uses
// 32-byte tiles: word x of row i at ((x >> 2) * m + i) * 4 + (x & 3); a row's
// 32-byte chunk is two lanes, a quarter-warp covers 4 rows which read 4
// different tables placed in 4 different 32-byte bank quarters (conflict-free).
//
// Per super-step S (words w = 2S, w+1): the panel CTA factors panel a (window
// from the previous super-step's capture of word w) and panel b (window =
// word w+1 after panel a, computed by panel a's look-ahead); both writebacks
// permute the rows' pre-super-step words (pb = word w, pb2 = word w+1). The
// workers claim pre-work chunks (apply both panels, then sweep the chunk over
// the look-ahead tile holding words w+2, w+3, capturing them into pb / pb2),
// then sweep a linear share of the remaining tiles.
#pragma once

#include "ple_kernels.cuh"
#include "ple_persistent.cuh"

namespace gf2cu {

__device__ __forceinline__ u64* tw4(u64* mat, u32 m, u32 row, u32 x) {
    return mat + ((((size_t)(x >> 2) * m + row) << 2) + (x & 3u));
}

// The physical-row array that follows the m sweep records {d~_a, d_b}.
__device__ __forceinline__ u32* info_phys(ulonglong2* info, u32 m) {
    return reinterpret_cast<u32*>(info + m);
}
__device__ __forceinline__ const u32* info_phys(const ulonglong2* info, u32 m) {
    return reinterpret_cast<const u32*>(info + m);
}

// Layout conversions go through shared memory in blocks of 32 rows x 16 tiles
// (512 bytes per row), so that both sides move long runs: 512 contiguous
// bytes per row on the row-major side, 32 rows x 32 bytes = 1 KiB contiguous
// per tile on the tile-major side (a direct copy scatters one side in 32-byte
// pieces and reached about half the HBM bandwidth). Rows are padded by 32
// bytes in shared memory: the tile-major side walks down the rows.
constexpr u32 kCvRows = 32, kCvTiles = 16, kCvPitch = kCvTiles * 32u + 32u;

// row-major (stride Wp) -> 32-byte tiles (Wpad4 words per row)
// (rows [row_lo, row_hi) only: streamed input tiles the row blocks as they arrive)
__global__ void __launch_bounds__(256) tile4_kernel(const u64* __restrict__ src, u64* __restrict__ dst, u32 m,
                                                    u32 Wp, u32 Wpad4, u32 row_lo = 0u,
                                                    u32 row_hi = 0xffffffffu) {
    __shared__ __align__(16) unsigned char buf[kCvRows * kCvPitch];
    row_hi = min(row_hi, m);
    if (row_hi <= row_lo) return;
    const u32 ntile = Wpad4 >> 2, tblocks = (ntile + kCvTiles - 1) / kCvTiles;
    const u32 rblocks = (row_hi - row_lo + kCvRows - 1) / kCvRows;
    const u32 tid = threadIdx.x;
    for (u32 blk = blockIdx.x; blk < tblocks * rblocks; blk += gridDim.x) {
        const u32 row0 = row_lo + (blk / tblocks) * kCvRows, tile0 = (blk % tblocks) * kCvTiles;
        // row-major side: 32 threads cover a row's 512 bytes, 8 rows per pass
#pragma unroll
        for (u32 i = 0; i < 4; ++i) {
            const u32 rr = (tid >> 5) + 8u * i, u = tid & 31u;
            const u32 row = row0 + rr, x = tile0 * 4u + 2u * u;
            if (row < row_hi && x < Wpad4)
                *reinterpret_cast<ulonglong2*>(buf + rr * kCvPitch + u * 16u) =
                    *reinterpret_cast<const ulonglong2*>(src + (size_t)row * Wp + x);
        }
        __syncthreads();
        // tile-major side: 64 threads cover a tile's 32 rows x 32 bytes, 4 tiles per pass
#pragma unroll
        for (u32 i = 0; i < 4; ++i) {
            const u32 t = (tid >> 6) + 4u * i, rr = (tid & 63u) >> 1, h = tid & 1u;
            const u32 row = row0 + rr, x = (tile0 + t) * 4u + 2u * h;
            if (row < row_hi && x < Wpad4)
                *reinterpret_cast<ulonglong2*>(tw4(dst, m, row, x)) =
                    *reinterpret_cast<const ulonglong2*>(buf + rr * kCvPitch + t * 32u + h * 16u);
        }
        __syncthreads();
    }
}

// Back to row-major in position order; the pivot row at position i < rank of
// super-step S = q_i / 128 takes its tiles from S's first swept tile
// ((2S+2)/4) on from ubuf, when S swept.
// 16 bytes (words x, x+1) of the final row at position `row`.
__device__ __forceinline__ const u64* final4(const u64* src, const u32* perm, u32 m, const u64* ubuf,
                                             u32 ucap, const u32* qcol, u32 rank, u32 W, u32 row, u32 x) {
    const u64* from = tw4(const_cast<u64*>(src), m, perm[row], x);
    if (row < rank) {
        const u32 w2 = 2u * (qcol[row] >> 7) + 2u;  // first word after the super-step
        if (w2 < W && (x >> 2) >= (w2 >> 2)) from = tw4(const_cast<u64*>(ubuf), ucap, row, x);
    }
    return from;
}

// (positions below row_lo were already written, by the kernel's streamed output)
__global__ void __launch_bounds__(256) untile4_kernel(const u64* __restrict__ src, u64* __restrict__ dst,
                                                      const u32* __restrict__ perm, u32 m, u32 Wp, u32 Wpad4,
                                                      const u64* __restrict__ ubuf, u32 ucap,
                                                      const u32* __restrict__ qcol, u32 rank, u32 W,
                                                      u32 row_lo = 0u) {
    __shared__ __align__(16) unsigned char buf[kCvRows * kCvPitch];
    if (m <= row_lo) return;
    const u32 ntile = Wpad4 >> 2, tblocks = (ntile + kCvTiles - 1) / kCvTiles;
    const u32 rblocks = (m - row_lo + kCvRows - 1) / kCvRows;
    const u32 tid = threadIdx.x;
    for (u32 blk = blockIdx.x; blk < tblocks * rblocks; blk += gridDim.x) {
        const u32 row0 = row_lo + (blk / tblocks) * kCvRows, tile0 = (blk % tblocks) * kCvTiles;
#pragma unroll
        for (u32 i = 0; i < 4; ++i) {
            const u32 t = (tid >> 6) + 4u * i, rr = (tid & 63u) >> 1, h = tid & 1u;
            const u32 row = row0 + rr, x = (tile0 + t) * 4u + 2u * h;
            if (row < m && x < Wpad4)
                *reinterpret_cast<ulonglong2*>(buf + rr * kCvPitch + t * 32u + h * 16u) =
                    *reinterpret_cast<const ulonglong2*>(final4(src, perm, m, ubuf, ucap, qcol, rank, W, row, x));
        }
        __syncthreads();
#pragma unroll
        for (u32 i = 0; i < 4; ++i) {
            const u32 rr = (tid >> 5) + 8u * i, u = tid & 31u;
            const u32 row = row0 + rr, x = tile0 * 4u + 2u * u;
            if (row < m && x < Wpad4)
                *reinterpret_cast<ulonglong2*>(dst + (size_t)row * Wp + x) =
                    *reinterpret_cast<const ulonglong2*>(buf + rr * kCvPitch + u * 16u);
        }
        __syncthreads();
    }
}

constexpr u32 kOutEvery = 8;  // streamed output: super-steps per batch

// Streamed output: the rows at positions [lo, hi) (pivot rows of a finished
// super-step) into p.out in row-major form; 16-byte units split as part
// `part` of `nparts`.
__device__ __forceinline__ void out_rows4(const Params& p, u32 lo, u32 hi, u32 part, u32 nparts) {
    const u32 per_row = p.Wpad8 >> 1;  // Wpad4 in this driver
    const u32 total = (hi - lo) * per_row;
    for (u32 e = part * blockDim.x + threadIdx.x; e < total; e += nparts * blockDim.x) {
        const u32 row = lo + e / per_row, x = 2u * (e % per_row);
        *reinterpret_cast<ulonglong2*>(p.out + (size_t)row * p.out_Wp + x) = ldcg(reinterpret_cast<const ulonglong2*>(
            final4(p.mat, p.perm, p.m, p.ubuf, p.ucap, p.qcol, 0xffffffffu, p.W, row, x)));
    }
}

// Initial state of the super-step driver: identity order, pb / pb2 = words
// 0 / 1 of every row (read from the row-major input).
__global__ void ple_init4_kernel(Params p, const u64* __restrict__ rowmajor, u32 Wp, u32 row_lo = 0u,
                                 u32 row_hi = 0xffffffffu) {
    const u32 stride = gridDim.x * blockDim.x;
    row_hi = min(row_hi, p.m);
    for (u32 i = row_lo + blockIdx.x * blockDim.x + threadIdx.x; i < row_hi; i += stride) {
        p.perm[i] = i;
        p.pb[i] = rowmajor[(size_t)i * Wp];
        if (p.W > 1) p.pb2[i] = rowmajor[(size_t)i * Wp + 1];
    }
    if (row_lo == 0u && blockIdx.x == 0 && threadIdx.x == 0) {
        p.state->r = 0;
        p.state->rb = 0;
    }
}

// Panel-side outputs the workers need beyond the two PanelOuts.
struct SuperOut {
    u64 piv2[64];  // panel a's pivot rows: pre-super-step word w+1
    u64 C[64];     // panel b's pivot rows: their panel-a combination
};

struct ApplyShared2 {
    u64 Ea[64], Da[64], Eb[64], Db[64], piv2[64], C[64];
    u32 qa[64], qb[64];
};

__device__ __forceinline__ void apply2_load(const Params& p, const PanelOut* pa, const PanelOut* pb,
                                            const SuperOut* so, ApplyShared2& s, u32 rba, u32 rbb) {
    for (u32 k = threadIdx.x; k < 64; k += blockDim.x) {
        const bool va = k < rba, vb = k < rbb;
        s.Ea[k] = va ? ldcg(&pa->E[k]) : 0ull;
        s.Da[k] = va ? ldcg(&pa->D[k]) : 0ull;
        s.qa[k] = va ? ldcg(&pa->qb[k]) : 0u;
        s.piv2[k] = va ? ldcg(&so->piv2[k]) : 0ull;
        s.Eb[k] = vb ? ldcg(&pb->E[k]) : 0ull;
        s.Db[k] = vb ? ldcg(&pb->D[k]) : 0ull;
        s.qb[k] = vb ? ldcg(&pb->qb[k]) : 0u;
        s.C[k] = vb ? ldcg(&so->C[k]) : 0ull;
    }
}

// Compressed write of one panel's multipliers c into columns [r0, r0 + rb)
// (OR into the free zero bits of earlier words) and of the panel word wp
// (overwritten: c's bits that land in it | the pivot row's E part).
__device__ __forceinline__ void compress_write(u64* mat, u32 m, u32 ph, u32 r0, u32 wp, u64 c,
                                               u64 epart) {
    const u32 w0 = r0 >> 6, b0 = r0 & 63u;
    const u64 clo = c << b0;
    const u64 chi = b0 ? (c >> (64u - b0)) : 0ull;
    if (w0 == wp) {
        *tw4(mat, m, ph, wp) = clo | epart;
    } else {
        *tw4(mat, m, ph, w0) |= clo;
        if (w0 + 1u == wp) {
            *tw4(mat, m, ph, wp) = chi | epart;
        } else {
            if (chi) *tw4(mat, m, ph, w0 + 1u) |= chi;
            *tw4(mat, m, ph, wp) = epart;
        }
    }
}

// Apply both panels of super-step (w, w+1) to the rows at positions
// [lo, hi): multipliers, compressed words, and the sweep record
// info[pos] = {d~_a, d_b}, and the physical row in the u32 array that
// follows the m records (info_phys): dense records keep the sweep's loads of
// them at 2 + 1 L1 wavefronts per warp (the sweep is L1-bound).
template <bool Check>
__device__ __forceinline__ void apply2_rows_t(const Params& p, const ApplyShared2& s, u32 w, u32 r,
                                              u32 rba, u32 rbb, bool has_b, u32 lo, u32 hi, u32 tid,
                                              u32 nthr) {
    const u32 rb0 = r + rba;
    for (u32 pos = lo + tid; pos < hi; pos += nthr) {
        const u32 ph = ldcg(p.perm + pos);
        u64 v = ldcg(p.pb + pos);
        const u64 x1 = has_b ? ldcg(p.pb2 + pos) : 0ull;
        // panel a (word w)
        const u32 off = pos - r;
        const u32 tla = off < rba ? off : rba;
        u64 c = 0ull, da = 0ull, epa = 0ull;
#pragma unroll 8
        for (u32 k = 0; k < 64; ++k) {
            if (k >= tla) break;
            const u64 bit = (v >> s.qa[k]) & 1ull;
            const u64 msk = 0ull - bit;
            v ^= s.Ea[k] & msk;
            da ^= s.Da[k] & msk;
            c |= bit << k;
        }
        if constexpr (Check) {
            if (p.check_inject == w + 1u && off == rba) v ^= 1ull << 63;  // (the checker's own test)
            check_panel_word(p.check, w, v, tla, off < rba, s.qa);
        }
        if (off < rba) {
            c |= 1ull << off;
            epa = v & ~low_mask64((int)s.qa[off] + 1);
        }
        compress_write(p.mat, p.m, ph, r, w, c, epa);
        u64 db = 0ull, dta = da;
        if (has_b) {
            // word w+1 after panel a
            u64 v1 = x1;
#pragma unroll 8
            for (u32 k = 0; k < 64; ++k) {
                if (k >= rba) break;
                v1 ^= s.piv2[k] & (0ull - ((da >> k) & 1ull));
            }
            if (pos < rb0) {
                *tw4(p.mat, p.m, ph, w + 1u) = v1;  // a pivot row of panel a: its U word w+1
            } else {
                const u32 offb = pos - rb0;
                const u32 tlb = offb < rbb ? offb : rbb;
                u64 cb = 0ull, epb = 0ull;
#pragma unroll 8
                for (u32 k = 0; k < 64; ++k) {
                    if (k >= tlb) break;
                    const u64 bit = (v1 >> s.qb[k]) & 1ull;
                    const u64 msk = 0ull - bit;
                    v1 ^= s.Eb[k] & msk;
                    db ^= s.Db[k] & msk;
                    cb |= bit << k;
                }
                if constexpr (Check) check_panel_word(p.check, w + 1u, v1, tlb, offb < rbb, s.qb);
                if (offb < rbb) {
                    cb |= 1ull << offb;
                    epb = v1 & ~low_mask64((int)s.qb[offb] + 1);
                }
                compress_write(p.mat, p.m, ph, rb0, w + 1u, cb, epb);
#pragma unroll 8
                for (u32 k = 0; k < 64; ++k) {
                    if (k >= rbb) break;
                    dta ^= s.C[k] & (0ull - ((db >> k) & 1ull));
                }
            }
        }
        p.info[pos] = make_ulonglong2(dta, db);
        info_phys(p.info, p.m)[pos] = ph;
    }
}

__device__ __forceinline__ void apply2_rows(const Params& p, const ApplyShared2& s, u32 w, u32 r, u32 rba,
                                            u32 rbb, bool has_b, u32 lo, u32 hi, u32 tid, u32 nthr) {
    if (p.check)
        apply2_rows_t<true>(p, s, w, r, rba, rbb, has_b, lo, hi, tid, nthr);
    else
        apply2_rows_t<false>(p, s, w, r, rba, rbb, has_b, lo, hi, tid, nthr);
}

// 16 tables x 256 entries x 32 B. Table t (t < 8: panel a, byte t of d~_a;
// t >= 8: panel b, byte t-8 of d_b) lives in bank quarter t & 3:
// entry e at ((t >> 2) * 256 + e) * 128 + (t & 3) * 32 + half * 16.
__device__ __forceinline__ u32 tab16_off(u32 t, u32 e, u32 h) {
    return (((t >> 2) * 256u + e) << 7) + ((t & 3u) << 5) + (h << 4);
}

// The 16 lookups of one row's 16-byte half-chunk: chunk ^= T_t[byte_t(d)]
// for t = 0..15, where d = {d~_a, d_b}. At lookup pp a lane reads table
// t = pp ^ rq (rq = its row within the quarter-warp): the 4 rows of a
// quarter-warp hit the 4 tables of one 32 KiB block in 4 different bank
// quarters (conflict-free), t >> 2 = pp >> 2 is a compile-time block offset,
// and byte t of d is byte (pp & 3) ^ rq of 32-bit word pp >> 2 -- one PRMT
// with a per-lane selector. sel[j] = 0x4440 | (j ^ rq), koff[j] = the lane's
// bank-quarter and half offset for j = pp & 3.
__device__ __forceinline__ void lookup16(ulonglong2& acc, const unsigned char* smem, ulonglong2 d,
                                         const u32 sel[4], const u32 koff[4]) {
    const u32 wd[4] = {(u32)d.x, (u32)(d.x >> 32), (u32)d.y, (u32)(d.y >> 32)};
#pragma unroll
    for (u32 pp = 0; pp < 16; ++pp) {
        const u32 e = __byte_perm(wd[pp >> 2], 0u, sel[pp & 3u]);
        xor2(acc, *reinterpret_cast<const ulonglong2*>(smem + (pp >> 2) * 32768u + e * 128u + koff[pp & 3u]));
    }
}

__device__ __forceinline__ void lookup16_consts(u32 rq, u32 h, u32 sel[4], u32 koff[4]) {
#pragma unroll
    for (u32 j = 0; j < 4; ++j) {
        sel[j] = 0x4440u | (j ^ rq);
        koff[j] = ((j ^ rq) << 5) | (h << 4);
    }
}

// (split in two so that a pre-work chunk can issue the source loads before
// its apply and walk after it: the load latency overlaps the apply)
__device__ __forceinline__ void build16_load(const Params& p, u32 tile, u32 w, const u32* pa, u32 rba,
                                             const u32* pb, u32 rbb, ulonglong2 R[8]) {
    const u32 tid = threadIdx.x;
    const u32 h = tid & 1u;
    const u32 t = (((tid >> 5) & 3u) << 2) | ((tid >> 1) & 3u);
    const u32 x0 = tile * 4u;
    const u32 zlim = w + 2u > x0 ? min(w + 2u - x0, 4u) : 0u;  // words <= w+1
    const u32* src = t < 8u ? pa : pb;
    const u32 nsrc = t < 8u ? rba : rbb;
    const u32 base = 8u * (t & 7u);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        ulonglong2 v = make_ulonglong2(0ull, 0ull);
        if (base + b < nsrc)
            v = ldcg(reinterpret_cast<const ulonglong2*>(tw4(p.mat, p.m, src[base + b], x0) + 2u * h));
        if (2u * h < zlim) v.x = 0ull;
        if (2u * h + 1u < zlim) v.y = 0ull;
        R[b] = v;
    }
}

__device__ __forceinline__ void build16_walk(unsigned char* smem, const ulonglong2 R[8]) {
    const u32 tid = threadIdx.x;
    const u32 h = tid & 1u;
    const u32 t = (((tid >> 5) & 3u) << 2) | ((tid >> 1) & 3u);
    const u32 sg = (((tid >> 7) & 3u) << 2) | ((tid >> 3) & 3u);
    const u32 i0 = 16u * sg;
    const u32 e0 = i0 ^ (i0 >> 1);
    ulonglong2 acc = make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int b = 3; b < 8; ++b)
        if ((e0 >> b) & 1u) xor2(acc, R[b]);
    *reinterpret_cast<ulonglong2*>(smem + tab16_off(t, e0, h)) = acc;
#pragma unroll
    for (u32 k = 1; k < 16; ++k) {
        const int b = (k & 1u) ? 0 : (k & 2u) ? 1 : (k & 4u) ? 2 : 3;  // ctz(k), folded
        xor2(acc, R[b]);
        const u32 i = i0 + k;
        *reinterpret_cast<ulonglong2*>(smem + tab16_off(t, i ^ (i >> 1), h)) = acc;
    }
}

// Gray walk (gray_code.hpp:105-112) of the 16 tables for one 32-byte tile
// from the raw pivot rows of both panels (pa / pb = their physical rows;
// words <= w+1 of the tile read as zero). Thread layout (512): h = tid & 1,
// t & 3 = (tid >> 1) & 3, seg_lo = (tid >> 3) & 3, t >> 2 = (tid >> 5) & 3,
// seg_hi = (tid >> 7) & 3; each thread walks 16 entries of one table half.
__device__ __forceinline__ void build16(const Params& p, unsigned char* smem, u32 tile, u32 w,
                                        const u32* pa, u32 rba, const u32* pb, u32 rbb) {
    ulonglong2 R[8];
    build16_load(p, tile, w, pa, rba, pb, rbb, R);
    build16_walk(smem, R);
}

constexpr u32 kRows16 = kTrailThreads / 2 * kUnroll;  // 1024 rows per iteration

__device__ __forceinline__ void ld_info2(const ulonglong2* info, u32 m, u32 pos, bool valid,
                                         ulonglong2& d, u32& ph) {
    if (valid) {
        d = ldcg(info + pos);
        ph = ldcg(info_phys(info, m) + pos);
    } else {
        d = make_ulonglong2(0ull, 0ull);
        ph = 0u;
    }
}

// Rows [row0, row0 + cnt) (offsets from r) of 32-byte tile `tile` with the 16
// tables built. The tile holding words w+2, w+3 writes pb / pb2 (the next
// super-step's panel words); rows with offset < npiv (both panels' pivot
// rows) go to ubuf.
__device__ __forceinline__ void trail16_rows(const Params& p, const unsigned char* smem, u32 w,
                                             u32 r, u32 tile, u32 row0, u32 cnt, u32 npiv) {
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const u32 rw = lane >> 1, h = lane & 1u, rq = rw & 3u;
    const bool capture = (w + 2u < p.W) && ((w + 2u) >> 2) == tile;
    const bool cap_lane = capture && (((w + 2u) & 3u) >> 1) == h;
    const bool cap2 = cap_lane && (w + 3u < p.W);
    const u32 lane_row = wid * 16u + rw;
    u32 lsel[4], lkoff[4];
    lookup16_consts(rq, h, lsel, lkoff);
    u64* tbase = p.mat + (((size_t)tile * p.m) << 2) + 2u * h;
    const u32 rend = row0 + cnt;
    const u32 nit = (cnt + kRows16 - 1) / kRows16;
    ulonglong2 dC[kUnroll], dN[kUnroll], valC[kUnroll];
    u32 pC[kUnroll], pN[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 2);
        ld_info2(p.info, p.m, r + ri, ri < rend, dC[k], pC[k]);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + kRows16 + lane_row + (u32)k * (kTrailThreads / 2);
        ld_info2(p.info, p.m, r + ri, ri < rend, dN[k], pN[k]);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
        const u32 ri = row0 + lane_row + (u32)k * (kTrailThreads / 2);
        valC[k] = make_ulonglong2(0ull, 0ull);
        if (ri < rend && ((dC[k].x | dC[k].y) != 0ull || capture || ri < npiv))
            valC[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)pC[k] << 2)));
    }
    for (u32 it = 0; it < nit; ++it) {
        const u32 base = row0 + it * kRows16;
        ulonglong2 valN[kUnroll], dNN[kUnroll];
        u32 pNN[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + kRows16 + lane_row + (u32)k * (kTrailThreads / 2);
            valN[k] = make_ulonglong2(0ull, 0ull);
            if (ri < rend && ((dN[k].x | dN[k].y) != 0ull || capture || ri < npiv))
                valN[k] = ldcg(reinterpret_cast<const ulonglong2*>(tbase + ((size_t)pN[k] << 2)));
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + 2u * kRows16 + lane_row + (u32)k * (kTrailThreads / 2);
            ld_info2(p.info, p.m, r + ri, ri < rend, dNN[k], pNN[k]);
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const u32 ri = base + lane_row + (u32)k * (kTrailThreads / 2);
            const ulonglong2 d = dC[k];
            if ((d.x | d.y) != 0ull || (ri < npiv && ri < rend)) {
                lookup16(valC[k], smem, d, lsel, lkoff);
                if (ri < npiv)  // a pivot row of this super-step: its tail goes to ubuf
                    *reinterpret_cast<ulonglong2*>(
                        p.ubuf + ((((size_t)tile * p.ucap + r + ri) << 2) + 2u * h)) = valC[k];
                else
                    *reinterpret_cast<ulonglong2*>(tbase + ((size_t)pC[k] << 2)) = valC[k];
            }
            if (cap_lane && ri < rend) p.pb[r + ri] = valC[k].x;
            if (cap2 && ri < rend) p.pb2[r + ri] = valC[k].y;
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            dC[k] = dN[k];
            pC[k] = pN[k];
            dN[k] = dNN[k];
            pN[k] = pNN[k];
            valC[k] = valN[k];
        }
    }
}

__device__ __forceinline__ void stamp2(const Params& p, u32 w, u32 k) {
    if (p.phase_ns && threadIdx.x == 0) p.phase_ns[(size_t)w * 8 + k] = globaltimer();
}

// diagnostics (GF2CU_DUMP_WORKERS): per super-step x worker {wake, pre-work
// end, rest start, rest end}
__device__ __forceinline__ void wstamp(const Params& p, u32 S, u32 wk, u32 nworkers, u32 k) {
    if (p.worker_ns && threadIdx.x == 0) p.worker_ns[((size_t)S * nworkers + wk) * 4 + k] = globaltimer();
}


// ---------------------------------------------------------------------------
// Look-ahead across super-steps (panel CTA body threads, after panel b of
// super-step S, w = 2S). When the workers have already finished S-1 (the
// panel chain is the bottleneck), the panel CTA computes the next panel a's
// window -- words w+2, w+3 after S of the positions [r2, r2 + 128), r2 = the
// rank after S -- itself, so that panel a of S+1 need not wait for S's
// pre-work capture (its writeback and miss scans still do):
//   x = own ^ sum_k d~_a[k] R_a[k] ^ sum_k d_b[k] R_b[k]
// with own, R_a, R_b the pre-super-step words of the row and of both panels'
// pivot rows (the sweep's fusion). Gather (before S is
// published: the workers' pre-work of S rewrites pb / pb2 and sweeps tile
// (w+2)/4 in place) reads every input into shared memory; compute (after the
// publish) needs no global memory.
__device__ __forceinline__ bool super_la_gather(const Params& p, PanelShared& sh, u32 w, u32 r_a, u32 rba,
                                                u32 r_b, u32 nwin_b, u32 rbb, int nthr) {
    const u32 r2 = r_b + rbb;
    const u32 nwin2 = min((u32)kWin, vis_rows(p) - r2);
    const bool has3 = w + 3u < p.W;
    for (u32 k = threadIdx.x; k < nwin2; k += nthr) {
        const u32 q = r2 + k, slot = q - r_b;
        u32 ph;
        if (slot < nwin_b) {
            const u32 o = sh.dorg[slot] & 127u;  // a non-pivot slot: an in-window origin
            ph = sh.wphys[o];
            sh.la_e0[k] = sh.ndacc[o];  // d_a (panel a's look-ahead, by panel-b slot)
            sh.la_e1[k] = sh.dacc[slot];  // d_b
            sh.la_ent[k] = 0;
        } else {
            ph = ldcg(p.perm + q);
            sh.la_e0[k] = ldcg(p.pb + q);
            sh.la_e1[k] = ldcg(p.pb2 + q);
            sh.la_ent[k] = 1;
        }
        sh.la_phys[k] = ph;
        sh.la_m2[k] = ldcg(tw4(p.mat, p.m, ph, w + 2u));
        sh.la_m3[k] = has3 ? ldcg(tw4(p.mat, p.m, ph, w + 3u)) : 0ull;
    }
    for (u32 k = threadIdx.x; k < 128u; k += nthr) {
        const bool b = k >= 64u;
        const u32 idx = k & 63u;
        u64 x2 = 0ull, x3 = 0ull;
        if (idx < (b ? rbb : rba)) {
            const u32 ph = ldcg(p.perm + (b ? r_b : r_a) + idx);
            x2 = ldcg(tw4(p.mat, p.m, ph, w + 2u));
            x3 = has3 ? ldcg(tw4(p.mat, p.m, ph, w + 3u)) : 0ull;
        }
        sh.la_R2[k] = x2;
        sh.la_R3[k] = x3;
        if (b && idx < rbb) {
            const u32 o = sh.dorg[idx];
            sh.la_C[idx] = (o & 0x80000000u) ? sh.oda[o & 63u] : sh.ndacc[o & 127u];
        }
    }
    named_bar(kBodyBar, nthr);
    return true;
}

__device__ __forceinline__ void super_la_compute(const Params& p, PanelShared& sh, u32 rba, u32 r_b,
                                                 u32 rbb, int nthr) {
    const u32 r2 = r_b + rbb;
    const u32 nwin2 = min((u32)kWin, vis_rows(p) - r2);
    for (u32 k = threadIdx.x; k < nwin2; k += nthr) {
        u64 da, db;
        if (sh.la_ent[k]) {
            // a row from outside panel b's window: both panels from its raw
            // words (as panel b's miss scan does)
            u64 v = sh.la_e0[k];
            da = 0ull;
            for (u32 s2 = 0; s2 < rba; ++s2) {
                const u64 msk = 0ull - ((v >> sh.qa[s2]) & 1ull);
                v ^= sh.Ea[s2] & msk;
                da ^= sh.Da[s2] & msk;
            }
            u64 v1 = sh.la_e1[k];
            for (u32 s2 = 0; s2 < rba; ++s2) v1 ^= sh.piv2[s2] & (0ull - ((da >> s2) & 1ull));
            db = 0ull;
            for (u32 s2 = 0; s2 < rbb; ++s2) {
                const u64 msk = 0ull - ((v1 >> sh.q[s2]) & 1ull);
                v1 ^= sh.E[s2] & msk;
                db ^= sh.D[s2] & msk;
            }
        } else {
            da = sh.la_e0[k];
            db = sh.la_e1[k];
        }
        u64 dta = da;
        for (u32 s2 = 0; s2 < rbb; ++s2) dta ^= sh.la_C[s2] & (0ull - ((db >> s2) & 1ull));
        u64 x2 = sh.la_m2[k], x3 = sh.la_m3[k];
#pragma unroll 4
        for (u32 s2 = 0; s2 < 64u; ++s2) {
            const u64 ma = 0ull - ((dta >> s2) & 1ull), mb = 0ull - ((db >> s2) & 1ull);
            x2 ^= (sh.la_R2[s2] & ma) ^ (sh.la_R2[64u + s2] & mb);
            x3 ^= (sh.la_R3[s2] & ma) ^ (sh.la_R3[64u + s2] & mb);
        }
        sh.la_m2[k] = x2;
        sh.la_m3[k] = x3;
    }
    named_bar(kBodyBar, nthr);
}

// Exhausted trailing matrix (panel CTA body threads, after a super-step in
// which neither panel found a pivot): are the rows at positions >= r zero in
// every word from w+2 on? Then every remaining panel is empty too -- the
// reference would scan each of their columns and find nothing -- and the
// factorization can stop here with the outputs it has (rank-deficient inputs:
// BASELINE config 4 spends its last 128 panels this way). The matrix is final
// once every worker is through S-1 (S itself changes nothing); the scan leaves
// at the first tile that holds a set bit, so it is only long when it pays.
// Returns 1 = all zero, 0 = not, -1 = error / watchdog.
__device__ __forceinline__ int trailing_is_zero(const Params& p, PanelShared& sh, SyncState* sy, u32 w, u32 r,
                                                u32 M, u32 t_target, int nthr) {
    if (threadIdx.x == 0) sh.la_go = spin_geq(&sy->t_count, t_target, &sy->error) ? 0 : -1;
    named_bar(kBodyBar, nthr);
    if (sh.la_go < 0) return -1;
    const u32 ntile = p.Wpad8 >> 2;  // (Wpad4 words per row in this driver)
    const u32 first = (w + 2u) >> 2;
    const bool upper_only = ((w + 2u) & 3u) != 0u;  // words w, w+1 share the first tile
    // (from the last tile down: data right of empty panels usually reaches the last column)
    for (u32 tile = ntile - 1u; tile + 1u > first; --tile) {
        u64 any = 0ull;
        for (u32 pos = r + threadIdx.x; pos < M; pos += (u32)nthr) {
            const u64* e = tw4(p.mat, p.m, ldcg(p.perm + pos), 4u * tile);
            const ulonglong2 hi = ldcg(reinterpret_cast<const ulonglong2*>(e + 2));
            any |= hi.x | hi.y;
            if (!(upper_only && tile == first)) {
                const ulonglong2 lo = ldcg(reinterpret_cast<const ulonglong2*>(e));
                any |= lo.x | lo.y;
            }
        }
        if (any) sh.la_go = 1;
        named_bar(kBodyBar, nthr);
        const int found = sh.la_go;
        named_bar(kBodyBar, nthr);  // (everyone has read it before the next tile may set it)
        if (found) return 0;
    }
    return 1;
}

// Streamed input (gf2cu.cu, run_ple): the factorization of a host matrix as
// three launches of ple_super_kernel, so that it starts on the first row
// block while the rest is still on its way over PCIe.
//   A  super-steps [0, S1) on the rows that have arrived (Params::mv = m0,
//      partial = 1): pivots, swaps and updates are the complete
//      factorization's as long as every column finds its pivot among those
//      rows (the first row with a 1, ple.hpp:88-93, is then one of them); a
//      column that does not sets *abort and the host starts over with the
//      whole matrix.
//   B  replay = 1: the rows [m0, m) catch up on the same super-steps. The
//      panels are A's, from the per-super-step history (hist = 1: pout[S],
//      pout_b[S], so[S], rhist, perm); a late row is never a pivot row of
//      these steps, so this is the workers' part alone (apply, sweep,
//      capture) on row positions >= row_lo. Their tables come from the pivot
//      rows' in-matrix copies, which keep their pre-step tails (the swept
//      tails are in ubuf).
//   C  super-steps [S1, nss) on all rows, as usual.
// The host presets the cumulative counters between the launches
// (sync_preset_kernel): panel_done = s_begin (B: s_end), t_count = nworkers *
// s_begin, out_count for the first output batch.
struct SuperRange {
    u32 s_begin, s_end;  // super-steps [s_begin, s_end) of this launch
    u32 row_lo;          // the workers' rows start at max(r, row_lo)
    u32 replay;          // 1: no panel CTA, panels from the history
    u32 hist;            // 1: panel outputs indexed by super-step
    u32* abort;          // phase A's verdict (null without streamed input)
};

// (a watchdog error of the previous launch turns the later ones into no-ops)
__global__ void sync_preset_kernel(SyncState* sy, u32 panel_done, u32 t_count, u32 out_count, u32* abort) {
    if (sy->error == 1u) *abort = 2u;
    *sy = SyncState{};
    sy->panel_done = panel_done;
    sy->t_count = t_count;
    sy->out_count = out_count;
}

// One launch, grid = #SMs: CTA 0 runs the panels, CTAs 1.. the sweep.
// rg.s_end = number of super-steps (ceil(W / 2)) unless the input is streamed.
// panel_done counts published super-steps.
__global__ void __launch_bounds__(kTrailThreads, 1)
    ple_super_kernel(Params p, PanelOut* pout_b, SuperOut* so, SuperRange rg) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ PanelShared psh;
    __shared__ ApplyShared2 ash;
    __shared__ u32 s_ok, s_claim;
    __shared__ u32 s_pa[64], s_pb[64];
    SyncState* sy = p.sync;
    const u32 nworkers = gridDim.x - 1;
    const u32 M = vis_rows(p);
    if (rg.abort && ldcg(rg.abort)) return;  // streamed input: phase A gave up

    if (blockIdx.x == 0) {
        // ------------------------------------------------------ panel CTA
        // (the last warp only signals; see signal_step)
        if (rg.replay) return;
        const int nbody = (int)blockDim.x - 32;
        if (threadIdx.x == 0) {
            psh.sig_step = 0;
            psh.sig_err = 0;
        }
        __syncthreads();
        if ((int)threadIdx.x >= nbody) {
            if (threadIdx.x == (u32)nbody) signal_loop(psh, sy, rg.s_end, rg.s_begin);
            return;
        }
        // (a launch that starts at s_begin > 0 continues from the previous
        // launch's rank; its capture is complete)
        const u32 r_begin =
            rg.s_begin ? ldcg(p.rhist + 2u * rg.s_begin - 1u) + ldcg(p.rbhist + 2u * rg.s_begin - 1u) : 0u;
        LookAhead la{r_begin, false, p.ap_done, 0u, &sy->error};
        u32 prev_r = r_begin;
        bool la_next = false;  // panel a's window came from the look-ahead
        u32 zc_skip = 0u, zc_wait = 1u;  // exhausted-matrix check: empty super-steps to skip, back-off
        const bool la_on = (p.pflags & kPanelSuperLA) != 0u;
        // streamed input, phase A: a column without a pivot among the rows on
        // the device ends the attempt (every CTA leaves through the error word)
        auto gave_up = [&]() -> bool {
            if (!p.partial || psh.t >= 0) return false;
            if (threadIdx.x == 0) {
                *rg.abort = 1u;
                __threadfence();
                atomicExch(&sy->error, 2u);
            }
            return true;
        };
        for (u32 S = rg.s_begin; S < rg.s_end; ++S) {
            const u32 w = 2u * S;
            const u32 hi = rg.hist ? S : 0u;  // this super-step's panel outputs
            la.piv2_out = so[hi].piv2;
            la.C_out = so[hi].C;
            // nothing left: publish an empty super-step so the workers stop
            const bool done0 = la.r >= M;
            // panel a: its window and scans read the previous super-step's
            // capture (all of its pre-work chunks) -- the window only without
            // the look-ahead across super-steps
            la.cap_ctr = p.ap_done + (S > 0 ? S - 1 : 0);
            la.cap_target = S > rg.s_begin ? pw_chunks(M - prev_r, p.pw_div) : 0u;
            prev_r = la.r;
            la.super_mode = 1;
            la.have_window = la_next;
            la.pout = p.pout + hi;
            la_next = false;
            const u32 r_a = la.r;
            stamp2(p, w, 0);
            const u32 rba = panel_factor_body(p, w, psh, nbody, &la);
            if (gave_up()) return;
            // (an aborted panel returns 0: then check the error word itself)
            if (*(volatile int*)&psh.sig_err || (rba == 0u && *(volatile u32*)&sy->error)) return;
            la.r += rba;
            u32 rbb_found = 0xffffffffu;
            if (w + 1u < p.W) {
                if (!done0 && la.r < M) {
                    // panel b: window = word w+1 after panel a (panel a's
                    // look-ahead); nothing to wait for
                    la.super_mode = 2;
                    la.have_window = true;
                    la.cap_target = 0u;
                    la.pout = pout_b + hi;
                    const u32 rbb = panel_factor_body(p, w + 1u, psh, nbody, &la);
                    if (gave_up()) return;
                    if (*(volatile int*)&psh.sig_err || (rbb == 0u && *(volatile u32*)&sy->error)) return;
                    la.r += rbb;
                    rbb_found = rbb;
                    // look-ahead across super-steps, only while the workers
                    // are already through S-1 (the panel chain is the
                    // bottleneck; S-1 has also finished the tile holding
                    // words w+2, w+3 everywhere)
                    if (la_on && w + 2u < p.W && la.r < M) {
                        if (threadIdx.x == 0) psh.la_go = ld_acquire(&sy->t_count) >= nworkers * S ? 1 : 0;
                        named_bar(kBodyBar, nbody);
                        if (psh.la_go) {
                            const u32 r_b = r_a + rba;
                            la_next = super_la_gather(p, psh, w, r_a, rba, r_b, min((u32)kWin, M - r_b),
                                                      rbb, nbody);
                        }
                    }
                } else if (threadIdx.x == 0) {
                    p.rhist[w + 1u] = la.r;
                    p.rbhist[w + 1u] = 0u;
                }
            }
            // Neither panel found a pivot: if nothing is left right of them in
            // the rows below the rank, stop (checked with a doubling back-off,
            // so inputs whose empty panels are followed by data pay little).
            // (only in the launch that runs to the last super-step: the streamed
            // input's earlier phases are followed by replays of their history)
            if (rba == 0u && rbb_found == 0u && !done0 && la.r < M && w + 2u < p.W && !p.partial &&
                rg.s_end == (p.W + 1u) / 2u) {
                if (zc_skip > 0u) {
                    --zc_skip;
                } else {
                    const int zero = trailing_is_zero(p, psh, sy, w, la.r, M, nworkers * S, nbody);
                    if (zero < 0) return;
                    if (zero) {
                        // the workers stop at a step whose rank equals the row count
                        if (threadIdx.x == 0) {
                            p.rhist[w] = M;
                            p.rhist[w + 1u] = M;
                        }
                        stamp2(p, w, 1);
                        signal_step(psh, nbody, S, true);
                        return;
                    }
                    zc_wait = min(2u * zc_wait, 64u);
                    zc_skip = zc_wait;
                }
            }
            stamp2(p, w, 1);
            signal_step(psh, nbody, S, done0);
            if (done0 || *(volatile int*)&psh.sig_err) return;
            if (la_next) super_la_compute(p, psh, rba, r_a + rba, la.r - r_a - rba, nbody);
        }
        return;
    }

    // ---------------------------------------------------------- workers
    const u32 wk = blockIdx.x - 1;
    for (u32 S = rg.s_begin; S < rg.s_end; ++S) {
        if (!cta_wait(sy, &sy->panel_done, S + 1, s_ok)) return;
        // the first pre-work claim now: its latency overlaps the loads below
        if (threadIdx.x == 0) s_claim = atomicAdd(&p.ap_claim[S], 1u);
        const u32 w = 2u * S;
        const u32 hi = rg.hist ? S : 0u;  // this super-step's panel outputs
        const bool has_b = w + 1u < p.W;
        const u32 r = *(volatile u32*)&p.rhist[w], rba = *(volatile u32*)&p.rbhist[w];
        if (r >= M) return;
        const u32 rbb = has_b ? *(volatile u32*)&p.rbhist[w + 1u] : 0u;
        Params q = p;
        q.info = p.info + (size_t)(S & 1u) * 2u * p.m;
        const u32 lo = max(r, rg.row_lo);  // (replay: the late rows only)
        const u32 nrows = M - lo;
        const bool sweep = w + 2u < p.W;
        const u32 ct = (w + 2u) >> 2;  // look-ahead tile (words w+2, w+3)
        const u32 crow = pw_rows(nrows, p.pw_div), nch = pw_chunks(nrows, p.pw_div);
        for (u32 k = threadIdx.x; k < 64; k += blockDim.x) {
            s_pa[k] = k < rba ? ldcg(p.perm + r + k) : 0u;
            s_pb[k] = k < rbb ? ldcg(p.perm + r + rba + k) : 0u;
        }
        __syncthreads();
        if (wk == 0) stamp2(p, w, 2);
        wstamp(p, S, wk, nworkers, 0);

        // Pre-work chunks: the look-ahead tile was the previous super-step's
        // (every row final there) unless the window just entered a new tile.
        const bool early = S == 0 || ct == (w >> 2);
        if (sweep && !early && !cta_wait(sy, &sy->t_count, nworkers * S, s_ok)) return;
        // Per chunk: apply, then sweep the chunk's rows over the look-ahead
        // tile. Its tables are built once per super-step (the same for every
        // chunk).
        u32 mine = 0;
        bool loaded = false, built = false;
        for (bool first = true;; first = false) {
            if (!first && threadIdx.x == 0) s_claim = atomicAdd(&p.ap_claim[S], 1u);
            __syncthreads();
            const u32 c = s_claim;
            __syncthreads();
            if (c >= nch) break;
            const bool build = sweep && rba + rbb > 0 && !built;
            if (!loaded) {  // the panel outputs stay S's while any chunk of S is open
                apply2_load(p, p.pout + hi, pout_b + hi, so + hi, ash, rba, rbb);
                __syncthreads();
                loaded = true;
            }
            const u32 a0 = lo + c * crow, a1 = min(M, a0 + crow);
            apply2_rows(q, ash, w, r, rba, rbb, has_b, a0, a1, threadIdx.x, blockDim.x);
            if (sweep) {
                __syncthreads();
                if (build) {
                    build16(q, smem, ct, w, s_pa, rba, s_pb, rbb);
                    __syncthreads();
                    built = true;
                }
                trail16_rows(q, smem, w, r, ct, a0 - r, a1 - a0, rba + rbb);
            }
            ++mine;
        }
        if (mine) {
            __syncthreads();
            if (threadIdx.x == 0) red_release_add(&p.ap_done[S], mine);  // (see cta_arrive)
        }
        wstamp(p, S, wk, nworkers, 1);
        // the rest: after super-step S-1 everywhere (pivot rows' raw tails)
        // and all of S's pre-work (every row's info / compressed words)
        if (threadIdx.x == 0)
            s_ok = spin_geq2(&sy->t_count, nworkers * S, &p.ap_done[S], nch, &sy->error) ? 1u : 0u;
        __syncthreads();
        if (!s_ok) return;
        if (p.out && S > 0 && S % kOutEvery == 0u) {
            // (the first batch of a launch that did not start the factorization
            // also covers the rows finished before it)
            const u32 out_lo = S < rg.s_begin + kOutEvery ? 0u : *(volatile u32*)&p.rhist[w - 2u * kOutEvery];
            // S-1 is finished everywhere: the pivot rows of the last kOutEvery
            // super-steps are final; write them out row-major and tell the
            // host (which copies them while the factorization goes on). In
            // batches, so that the fence before the count is paid every
            // kOutEvery super-steps only.
            out_rows4(p, out_lo, r, wk, nworkers);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(&sy->out_count, 1u) == nworkers * (S / kOutEvery) - 1u) {
                    __threadfence_system();
                    *p.out_host = r;
                }
            }
        }
        if (wk == 0) stamp2(p, w, 3);
        wstamp(p, S, wk, nworkers, 2);
        if (sweep) {
            const u32 nt = (p.Wpad8 >> 2) - ct - 1;  // Wpad8 holds Wpad4 here
            const u64 total = (u64)nt * nrows;
            u64 u = total * wk / nworkers;
            const u64 end = total * (wk + 1) / nworkers;
            while (u < end) {
                const u32 tile = ct + 1 + (u32)(u / nrows);
                const u32 rr = (u32)(u % nrows);
                const u32 row0 = rr + (lo - r);  // offset from r
                const u32 cnt = (u32)min((u64)(nrows - rr), end - u);
                if (rba + rbb > 0) {
                    __syncthreads();
                    build16(q, smem, tile, w, s_pa, rba, s_pb, rbb);
                    __syncthreads();
                }
                trail16_rows(q, smem, w, r, tile, row0, cnt, rba + rbb);
                u += cnt;
            }
        }
        wstamp(p, S, wk, nworkers, 3);
        cta_arrive(&sy->t_count);
        if (wk == 0) stamp2(p, w, 5);
    }
}

}  // namespace gf2cu
