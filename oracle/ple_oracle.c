/*
 * oracle/ple_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's block-iterative PLE path
 * (gf2elim, /root/reference/proj/include/gf2/ple.hpp) used as the checker for
 * the B200 kernels.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * path (paper_1111_6549_b200/) never links or calls it.
 *
 * Parity is pinned (not "unpinned"): tests/test_oracle.py checks this file
 * against the reference itself compiled here (oracle/_ref, built from the
 * reference headers by oracle/Makefile) and against golden vectors under
 * tests/golden/ that were produced by that compiled reference.
 *
 * Layout convention (bit_matrix.hpp:15-22): row-major uint64 words, column c
 * at bit (c & 63) of word (c >> 6), padding bits past ncols-1 are zero.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t word;

static inline word low_mask(size_t k) { return k >= 64 ? ~(word)0 : (((word)1 << k) - 1); }

/* ------------------------------------------------------------------------ */
/* MT19937-64 (Matsumoto & Nishimura 2004 published parameters), the engine  */
/* behind std::mt19937_64 that the reference generators draw from            */
/* (bit_matrix.hpp:461, 491).                                                */
/* ------------------------------------------------------------------------ */
typedef struct {
    word mt[312];
    int mti;
} orc_mt64;

void orc_mt64_seed(orc_mt64* g, word seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (word)i;
    g->mti = 312;
}

word orc_mt64_next(orc_mt64* g) {
    static const word mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const word UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            word x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            word x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        word x = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        g->mti = 0;
    }
    word x = g->mt[g->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* ------------------------------------------------------------------------ */
/* Input generators                                                          */
/* ------------------------------------------------------------------------ */

/* fill_random (bit_matrix.hpp:459-486) for a view with col_off == 0:
 * density 0.5 draws one engine word per matrix word (:472-473); any other
 * density draws 64 engine words per matrix word, bit b = (u < density) with
 * u = (draw >> 11) * 2^-53 (:475-480). Returns 0 on success, -1 on a bad
 * density (the reference throws std::invalid_argument, :460). */
int orc_fill_random(word* a, size_t m, size_t n, size_t stride, double density, word seed) {
    if (density < 0.0 || density > 1.0) return -1;
    const size_t width = (n + 63) / 64;
    if (density == 0.0) {
        for (size_t i = 0; i < m; ++i) memset(a + i * stride, 0, width * sizeof(word));
        return 0;
    }
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (size_t i = 0; i < m; ++i) {
        word* row = a + i * stride;
        for (size_t w = 0; w < width; ++w) {
            word v;
            if (density == 1.0)
                v = ~(word)0;
            else if (density == 0.5)
                v = orc_mt64_next(&g);
            else {
                v = 0;
                for (unsigned b = 0; b < 64; ++b) {
                    const double u = (double)(orc_mt64_next(&g) >> 11) * 0x1.0p-53;
                    v |= (word)(u < density) << b;
                }
            }
            row[w] = v;
        }
        if (n & 63) row[width - 1] &= low_mask(n & 63);
    }
    return 0;
}

/* detail::bounded (bit_matrix.hpp:444-454): masked rejection draw in [0, n). */
static word orc_bounded(orc_mt64* g, word n) {
    if (n == 1) return 0;
    const int bits = 64 - __builtin_clzll(n - 1);
    const word mask = bits >= 64 ? ~(word)0 : (((word)1 << bits) - 1);
    word v;
    do {
        v = orc_mt64_next(g) & mask;
    } while (v >= n);
    return v;
}

/* fill_random_rows (bit_matrix.hpp:489-520): exactly nnz distinct ones per
 * row; partial Fisher-Yates when nnz*2 > n, rejection otherwise. */
int orc_fill_random_rows(word* a, size_t m, size_t n, size_t stride, size_t nnz, word seed) {
    if (nnz > n) return -1;
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    const size_t width = (n + 63) / 64;
    uint32_t* pool = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    for (size_t i = 0; i < m; ++i) {
        word* row = a + i * stride;
        memset(row, 0, width * sizeof(word));
        if (nnz * 2 > n) {
            for (size_t j = 0; j < n; ++j) pool[j] = (uint32_t)j;
            for (size_t j = 0; j < nnz; ++j) {
                const size_t pick = j + (size_t)orc_bounded(&g, n - j);
                uint32_t t = pool[j];
                pool[j] = pool[pick];
                pool[pick] = t;
                row[pool[j] >> 6] |= (word)1 << (pool[j] & 63);
            }
        } else {
            size_t placed = 0;
            while (placed < nnz) {
                const size_t p = (size_t)orc_bounded(&g, n);
                const word bit = (word)1 << (p & 63);
                if (!(row[p >> 6] & bit)) {
                    row[p >> 6] |= bit;
                    ++placed;
                }
            }
        }
    }
    free(pool);
    return 0;
}

/* The F2-nonlinear counter generator of SURVEY.md section 8(d) (used for the
 * rank-sensitive configs 4 and 5, where mt19937_64 words cap the rank at
 * 19937): word(i, w) = fmix64((seed << 32) + (i*W + w + 1) * golden_gamma),
 * W the unpadded words per row, last word masked to ncols. */
static inline word fmix64(word x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

void orc_fill_ctr(word* a, size_t m, size_t n, size_t stride, word seed) {
    const size_t W = (n + 63) / 64;
    const word base = seed << 32;
    for (size_t i = 0; i < m; ++i) {
        word* row = a + i * stride;
        for (size_t w = 0; w < W; ++w)
            row[w] = fmix64(base + ((word)(i * W + w) + 1) * 0x9e3779b97f4a7c15ULL);
        if (n & 63) row[W - 1] &= low_mask(n & 63);
    }
}

/* ------------------------------------------------------------------------ */
/* PLE                                                                       */
/* ------------------------------------------------------------------------ */

/* Column exchange a <-> b for rows [r0, m): swap_cols_from_row
 * (bit_matrix.hpp:302-318), written as a plain bit swap. */
static void swap_cols_from_row(word* A, size_t m, size_t stride, size_t ca, size_t cb, size_t r0) {
    if (ca == cb) return;
    const size_t wa = ca >> 6, wb = cb >> 6;
    const unsigned ba = (unsigned)(ca & 63), bb = (unsigned)(cb & 63);
    for (size_t i = r0; i < m; ++i) {
        word* row = A + i * stride;
        const word xa = (row[wa] >> ba) & 1, xb = (row[wb] >> bb) & 1;
        if (xa != xb) {
            row[wa] ^= (word)1 << ba;
            row[wb] ^= (word)1 << bb;
        }
    }
}

/* Canonical right-looking PLE. This is the column-at-a-time limit of
 * block_iterative_ple (ple.hpp:166-244) with partial_ple's stripe search
 * (ple.hpp:57-130): for each column c, the pivot is the first row >= r (in
 * current row order) holding a 1 (ple.hpp:88-93); rows are swapped over the
 * full width (ple.hpp:99 + the flank replay at :187-188); every lower row with
 * bit c set gets the pivot row added from column c+1 on, so bit c keeps the
 * multiplier (ple.hpp:84, 116-119 and the table rewrite at :219-229); then
 * the multiplier column is compressed to column r (ple.hpp:232-236).
 * The reference's result does not depend on its stripe width k or on its
 * table count (key finding 1; re-checked against the
 * compiled reference in tests/test_oracle.py), so this restatement is
 * bit-exact with it: same in-place L\E words, p.swaps, q and rank.
 *
 * swaps[r] and q[r] (capacity min(m, n)) receive the LAPACK transposition
 * and pivot column of each pivot; returns the rank. */
size_t orc_ple(word* A, size_t m, size_t n, size_t stride, size_t* swaps, size_t* q) {
    const size_t W = (n + 63) / 64;
    size_t r = 0;
    for (size_t c = 0; c < n && r < m; ++c) {
        const size_t wc = c >> 6;
        const word bc = (word)1 << (c & 63);
        size_t pi = r;
        while (pi < m && !(A[pi * stride + wc] & bc)) ++pi;
        if (pi == m) continue;
        if (pi != r) {
            word* x = A + r * stride;
            word* y = A + pi * stride;
            for (size_t w = 0; w < W; ++w) {
                const word t = x[w];
                x[w] = y[w];
                y[w] = t;
            }
        }
        swaps[r] = pi;
        q[r] = c;
        const word* prow = A + r * stride;
        const word first = prow[wc] & ~low_mask((c & 63) + 1); /* columns > c */
        for (size_t i = r + 1; i < m; ++i) {
            word* row = A + i * stride;
            if (!(row[wc] & bc)) continue;
            row[wc] ^= first;
            for (size_t w = wc + 1; w < W; ++w) row[w] ^= prow[w];
        }
        swap_cols_from_row(A, m, stride, r, c, r);
        ++r;
    }
    return r;
}

/* Row dst ^= row src over columns [c0, n) (row_add_from, bit_matrix.hpp:273-279). */
static void add_row_from(word* A, size_t stride, size_t n, size_t dst, size_t src, size_t c0) {
    if (c0 >= n) return;
    word* d = A + dst * stride;
    const word* s = A + src * stride;
    const size_t W = (n + 63) / 64, w0 = c0 >> 6;
    d[w0] ^= s[w0] & ~low_mask(c0 & 63);
    for (size_t w = w0 + 1; w < W; ++w) d[w] ^= s[w];
}

/* The lazy single pass partial_ple (ple.hpp:57-130), restated with its
 * watermarks: wm[l] = the last row that carries pivot l's update. A row is
 * brought up to date (every pivot whose watermark lies above it, in pivot
 * order, each added from one past its pivot column) the first time the scan
 * reads it; the pivot of a column is the first row >= r holding a 1 after
 * that; the rows between a pivot's watermark and the deepest row read get a
 * catch-up at the end; then the multiplier columns are compressed. rank in
 * *rank_out; returns processed = max(rank, deepest row read + 1), or 0 when
 * no pivot exists. swaps / q need capacity min(m, n). */
size_t orc_partial_ple(word* A, size_t m, size_t n, size_t stride, size_t* swaps, size_t* q,
                       size_t* rank_out) {
    const size_t cap = m < n ? m : n;
    size_t* wm = (size_t*)malloc((cap ? cap : 1) * sizeof(size_t));
    size_t r = 0, c = 0;
    while (r < m && c < n) {
        int found = 0;
        size_t pi = 0, pj = 0;
        for (size_t j = c; j < n && !found; ++j) {
            for (size_t i = r; i < m; ++i) {
                if (r > 0 && i > wm[r - 1]) {
                    size_t lo = 0, hi = r; /* first l with wm[l] < i (wm non-increasing) */
                    while (lo < hi) {
                        const size_t mid = (lo + hi) / 2;
                        if (wm[mid] >= i) lo = mid + 1; else hi = mid;
                    }
                    for (size_t l = lo; l < r; ++l) {
                        if ((A[i * stride + (q[l] >> 6)] >> (q[l] & 63)) & 1)
                            add_row_from(A, stride, n, i, l, q[l] + 1);
                        wm[l] = i;
                    }
                }
                if ((A[i * stride + (j >> 6)] >> (j & 63)) & 1) {
                    found = 1;
                    pi = i;
                    pj = j;
                    break;
                }
            }
        }
        if (!found) break;
        swaps[r] = pi;
        q[r] = pj;
        if (pi != r) {
            word* x = A + r * stride;
            word* y = A + pi * stride;
            for (size_t w = 0; w < (n + 63) / 64; ++w) {
                const word t = x[w];
                x[w] = y[w];
                y[w] = t;
            }
        }
        wm[r] = pi;
        ++r;
        c = pj + 1;
    }
    *rank_out = r;
    if (r == 0) {
        free(wm);
        return 0;
    }
    const size_t deepest = wm[0];
    for (size_t j = 0; j < r; ++j)
        for (size_t i = (wm[j] + 1 > r ? wm[j] + 1 : r); i <= deepest; ++i)
            if ((A[i * stride + (q[j] >> 6)] >> (q[j] & 63)) & 1) add_row_from(A, stride, n, i, j, q[j] + 1);
    for (size_t j = 0; j < r; ++j) swap_cols_from_row(A, m, stride, j, q[j], j);
    free(wm);
    return deepest + 1 > r ? deepest + 1 : r;
}

/* The canonical compression list {j, q[j], j} for q[j] != j, in application
 * order; the same swaps block_iterative_ple records at ple.hpp:232-236 when
 * its stripe width is 1. Returns the count; out holds 3 entries per swap. */
size_t orc_canonical_col_swaps(const size_t* q, size_t rank, size_t* out) {
    size_t k = 0;
    for (size_t j = 0; j < rank; ++j)
        if (q[j] != j) {
            out[3 * k + 0] = j;
            out[3 * k + 1] = q[j];
            out[3 * k + 2] = j;
            ++k;
        }
    return k;
}

/* undo_column_swaps (ple.hpp:293-296): replay the list backwards. */
void orc_undo_col_swaps(word* A, size_t m, size_t stride, const size_t* cs, size_t count) {
    for (size_t i = count; i-- > 0;) swap_cols_from_row(A, m, stride, cs[3 * i], cs[3 * i + 1], cs[3 * i + 2]);
}

/* C = A * B over F2 (row-combination form of mul_naive, multiply.hpp:62):
 * row i of C is the XOR of the rows j of B with A[i][j] = 1. */
void orc_mul(const word* A, size_t m, size_t l, size_t sa, const word* B, size_t n, size_t sb,
             word* C, size_t sc) {
    const size_t Wn = (n + 63) / 64;
    for (size_t i = 0; i < m; ++i) {
        word* crow = C + i * sc;
        memset(crow, 0, Wn * sizeof(word));
        const word* arow = A + i * sa;
        for (size_t j = 0; j < l; ++j)
            if ((arow[j >> 6] >> (j & 63)) & 1) {
                const word* brow = B + j * sb;
                for (size_t w = 0; w < Wn; ++w) crow[w] ^= brow[w];
            }
    }
}

/* naive_echelonize (ple.hpp:362-380): word-at-a-time Gauss-Jordan. Per
 * column c the pivot is the first row >= r holding a 1, swapped to row r;
 * then every other row (full) or every lower row (!full) with bit c gets the
 * pivot row added from column c on (row_add_from, bit_matrix.hpp:273-279).
 * The reduced form is unique, and the !full form is the PLE's E factor with
 * zero rows below (same pivot choice and elimination as orc_ple). Returns
 * the rank. */
size_t orc_echelonize(word* A, size_t m, size_t n, size_t stride, int full) {
    const size_t W = (n + 63) / 64;
    size_t r = 0;
    for (size_t c = 0; c < n && r < m; ++c) {
        const size_t wc = c >> 6;
        const word bc = (word)1 << (c & 63);
        size_t p = r;
        while (p < m && !(A[p * stride + wc] & bc)) ++p;
        if (p == m) continue;
        if (p != r) {
            word* x = A + r * stride;
            word* y = A + p * stride;
            for (size_t w = 0; w < W; ++w) {
                const word t = x[w];
                x[w] = y[w];
                y[w] = t;
            }
        }
        const word* prow = A + r * stride;
        const word first = prow[wc] & ~low_mask(c & 63); /* columns >= c */
        for (size_t i = full ? 0 : r + 1; i < m; ++i) {
            if (i == r) continue;
            word* row = A + i * stride;
            if (!(row[wc] & bc)) continue;
            row[wc] ^= first;
            for (size_t w = wc + 1; w < W; ++w) row[w] ^= prow[w];
        }
        ++r;
    }
    return r;
}

/* trsm_upper_left_unit (multiply.hpp:314-335) as plain back substitution:
 * B <- U^-1 B for the unit upper triangle of the r x r matrix U (only bits
 * strictly above the diagonal read). Row i (bottom-up) receives every row
 * j > i of the already-solved B with U[i][j] = 1 (the <= 64 branch at
 * :322-331 for any r). */
void orc_trsm_upper(const word* U, size_t r, size_t su, word* B, size_t n, size_t sb) {
    const size_t W = (n + 63) / 64;
    for (size_t i = r; i-- > 0;) {
        word* bi = B + i * sb;
        const word* ui = U + i * su;
        for (size_t j = i + 1; j < r; ++j)
            if ((ui[j >> 6] >> (j & 63)) & 1) {
                const word* bj = B + j * sb;
                for (size_t w = 0; w < W; ++w) bi[w] ^= bj[w];
            }
    }
}
