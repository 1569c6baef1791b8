// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/gf2/*.hpp, header-only C++20), compiled by
// oracle/Makefile into oracle/_ref/libgf2ref.so. It is the reference itself,
// run on host cores: tests/ use it to pin the C restatement
// (oracle/ple_oracle.c) and to produce golden vectors; bench.py uses it as
// the CPU baseline (cpu_baseline.kind = "reference") and as the
// `--impl reference` arm. Nothing here is product code and no reference
// source is copied: this file only includes the headers and forwards calls.
#include <chrono>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include "gf2/io.hpp"
#include <cstdio>
#include <sstream>
#include <exception>
#include <vector>

#include "gf2/gf2.hpp"

namespace {

gf2::MatrixView view_of(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride) {
    return gf2::MatrixView(words, stride, 0, m, n);
}

void export_outcome(const gf2::PleOutcome& out, std::size_t* swaps, std::size_t* q,
                    std::size_t* rank, std::size_t* col_swaps, std::size_t col_cap,
                    std::size_t* n_col_swaps) {
    *rank = out.rank;
    for (std::size_t i = 0; i < out.rank; ++i) {
        swaps[i] = out.p.swaps[i];
        q[i] = out.q[i];
    }
    if (n_col_swaps) *n_col_swaps = out.col_swaps.size();
    if (col_swaps)
        for (std::size_t i = 0; i < out.col_swaps.size() && i < col_cap; ++i) {
            col_swaps[3 * i + 0] = out.col_swaps[i].a;
            col_swaps[3 * i + 1] = out.col_swaps[i].b;
            col_swaps[3 * i + 2] = out.col_swaps[i].from_row;
        }
}

gf2::PleOutcome import_outcome(std::size_t rank, const std::size_t* swaps, const std::size_t* q,
                               const std::size_t* col_swaps, std::size_t n_col_swaps,
                               std::size_t processed) {
    gf2::PleOutcome out;
    out.rank = rank;
    out.processed = processed;
    out.p.swaps.assign(swaps, swaps + rank);
    out.q.assign(q, q + rank);
    for (std::size_t i = 0; i < n_col_swaps; ++i)
        out.col_swaps.push_back({col_swaps[3 * i], col_swaps[3 * i + 1], col_swaps[3 * i + 2]});
    return out;
}

} // namespace

extern "C" {

// gf2::block_iterative_ple (ple.hpp:166). k == 0 -> the reference's own pick.
// Returns the wall seconds of the call (steady_clock), or -1 on an exception.
double ref_block_iterative_ple(std::uint64_t* words, std::size_t m, std::size_t n,
                               std::size_t stride, unsigned k, unsigned table_count,
                               std::size_t* swaps, std::size_t* q, std::size_t* rank,
                               std::size_t* col_swaps, std::size_t col_cap,
                               std::size_t* n_col_swaps) {
    try {
        gf2::PleConfig cfg;
        cfg.k = k;
        if (table_count) cfg.table_count = table_count;
        const auto t0 = std::chrono::steady_clock::now();
        gf2::PleOutcome out = gf2::block_iterative_ple(view_of(words, m, n, stride), cfg);
        const double s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        export_outcome(out, swaps, q, rank, col_swaps, col_cap, n_col_swaps);
        return s;
    } catch (const std::exception&) {
        return -1.0;
    }
}

// gf2::recursive_ple (ple.hpp:246) with the given base parameters.
double ref_recursive_ple(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                         std::size_t base_bytes, std::size_t base_ncols, unsigned base_k,
                         std::size_t* swaps, std::size_t* q, std::size_t* rank) {
    try {
        gf2::PleConfig cfg;
        if (base_bytes) cfg.base_bytes = base_bytes;
        if (base_ncols) cfg.base_ncols = base_ncols;
        cfg.base_k = base_k;
        const auto t0 = std::chrono::steady_clock::now();
        gf2::PleOutcome out = gf2::recursive_ple(view_of(words, m, n, stride), cfg);
        const double s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        export_outcome(out, swaps, q, rank, nullptr, 0, nullptr);
        return s;
    } catch (const std::exception&) {
        return -1.0;
    }
}

// gf2::partial_ple (ple.hpp:57): returns processed.
std::size_t ref_partial_ple(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                            std::size_t* swaps, std::size_t* q, std::size_t* rank) {
    gf2::PleOutcome out = gf2::partial_ple(view_of(words, m, n, stride));
    export_outcome(out, swaps, q, rank, nullptr, 0, nullptr);
    return out.processed;
}

// gf2::fill_random (bit_matrix.hpp:459) / fill_random_rows (:489).
int ref_fill_random(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                    double density, std::uint64_t seed) {
    try {
        gf2::fill_random(view_of(words, m, n, stride), density, seed);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_fill_random_rows(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                         std::size_t nnz, std::uint64_t seed) {
    try {
        gf2::fill_random_rows(view_of(words, m, n, stride), nnz, seed);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// C = A * B via gf2::mul (multiply.hpp:266-274: M4RM / Strassen dispatch).
// Strides are the caller's; C must hold m rows of its stride.
int ref_mul(const std::uint64_t* a, std::size_t m, std::size_t l, std::size_t sa,
            const std::uint64_t* b, std::size_t n, std::size_t sb, std::uint64_t* c,
            std::size_t sc) {
    try {
        gf2::ConstMatrixView av(a, sa, 0, m, l), bv(b, sb, 0, l, n);
        gf2::BitMatrix prod = gf2::mul(av, bv);
        const std::size_t W = (n + 63) / 64;
        for (std::size_t i = 0; i < m; ++i)
            std::memcpy(c + i * sc, prod.row_words(i), W * sizeof(std::uint64_t));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// gf2::extract_e (ple.hpp:344) given an outcome; E is rank x n, stride se.
int ref_extract_e(const std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                  std::size_t rank, const std::size_t* swaps, const std::size_t* q,
                  const std::size_t* col_swaps, std::size_t n_col_swaps, std::uint64_t* e,
                  std::size_t se) {
    try {
        gf2::PleOutcome out = import_outcome(rank, swaps, q, col_swaps, n_col_swaps, m);
        gf2::BitMatrix em = gf2::extract_e(gf2::ConstMatrixView(words, stride, 0, m, n), out);
        const std::size_t W = (n + 63) / 64;
        for (std::size_t i = 0; i < rank; ++i)
            std::memcpy(e + i * se, em.row_words(i), W * sizeof(std::uint64_t));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// gf2::rref_from_ple (ple.hpp:319) in place.
int ref_rref_from_ple(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                      std::size_t rank, const std::size_t* swaps, const std::size_t* q,
                      const std::size_t* col_swaps, std::size_t n_col_swaps, int full) {
    try {
        gf2::PleOutcome out = import_outcome(rank, swaps, q, col_swaps, n_col_swaps, m);
        gf2::rref_from_ple(view_of(words, m, n, stride), out, full != 0);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// gf2::echelonize(a, strategy, full) (m4ri.hpp:88-105); strategy 0 naive,
// 1 m4ri, 2 ple_iterative, 3 ple_recursive. Returns the rank or -1.
long long ref_echelonize(std::uint64_t* words, std::size_t m, std::size_t n, std::size_t stride,
                         int strategy, int full) {
    try {
        const gf2::EchelonStrategy s = strategy == 0   ? gf2::EchelonStrategy::naive
                                       : strategy == 1 ? gf2::EchelonStrategy::m4ri
                                       : strategy == 2 ? gf2::EchelonStrategy::ple_iterative
                                                       : gf2::EchelonStrategy::ple_recursive;
        return (long long)gf2::echelonize(view_of(words, m, n, stride), s, full != 0);
    } catch (const std::exception&) {
        return -1;
    }
}

// gf2::trsm_upper_left_unit (multiply.hpp:314-335): b <- u^-1 b.
int ref_trsm_upper_left_unit(const std::uint64_t* u, std::size_t r, std::size_t su,
                             std::uint64_t* b, std::size_t n, std::size_t sb) {
    try {
        gf2::trsm_upper_left_unit(gf2::ConstMatrixView(u, su, 0, r, r), view_of(b, r, n, sb));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// gf2::save_gf2b / save_ascii (io.hpp:59-76) into a caller buffer: returns
// the byte count (or -1 when it does not fit / the writer threw).
long long ref_save_matrix(const std::uint64_t* words, std::size_t m, std::size_t n,
                          std::size_t stride, int ascii, char* out, std::size_t cap) {
    try {
        gf2::BitMatrix a(m, n);
        const std::size_t W = (n + 63) / 64;
        for (std::size_t i = 0; i < m; ++i) std::memcpy(a.row_words(i), words + i * stride, W * 8);
        std::ostringstream os;
        if (ascii) gf2::save_ascii(os, a); else gf2::save_gf2b(os, a);
        const std::string s = os.str();
        if (s.size() > cap) return -1;
        std::memcpy(out, s.data(), s.size());
        return (long long)s.size();
    } catch (const std::exception&) {
        return -1;
    }
}

// gf2::load_matrix (io.hpp:113-122) from a buffer. Returns 0 and the shape
// (words copied when they fit in `cap` words at stride ceil(n/64)), 1 when
// the loader threw io_error (its message copied to err).
int ref_load_matrix(const char* buf, std::size_t len, std::uint64_t* words, std::size_t cap,
                    std::size_t* m, std::size_t* n, char* err, std::size_t errcap) {
    try {
        std::istringstream is(std::string(buf, len));
        gf2::BitMatrix a = gf2::load_matrix(is);
        *m = a.nrows();
        *n = a.ncols();
        const std::size_t W = (a.ncols() + 63) / 64;
        if (a.nrows() * W <= cap)
            for (std::size_t i = 0; i < a.nrows(); ++i) std::memcpy(words + i * W, a.row_words(i), W * 8);
        return 0;
    } catch (const gf2::io_error& e) {
        std::snprintf(err, errcap, "%s", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::snprintf(err, errcap, "%s", e.what());
        return 2;
    }
}

// P*L*E reconstruction check (test_ple.cpp:38-50 / acceptance_main.cpp:97-108):
// returns 1 when P*L*E equals `orig` on the first `processed` (= m) rows.
int ref_reconstructs(const std::uint64_t* orig, const std::uint64_t* decomposed, std::size_t m,
                     std::size_t n, std::size_t stride, std::size_t rank,
                     const std::size_t* swaps, const std::size_t* q,
                     const std::size_t* col_swaps, std::size_t n_col_swaps) {
    try {
        gf2::PleOutcome out = import_outcome(rank, swaps, q, col_swaps, n_col_swaps, m);
        gf2::ConstMatrixView dv(decomposed, stride, 0, m, n), ov(orig, stride, 0, m, n);
        gf2::BitMatrix l = gf2::extract_l(dv, out);
        gf2::BitMatrix e = gf2::extract_e(dv, out);
        gf2::BitMatrix back = gf2::ple_reconstruct(out, l.cview(), e.cview());
        return gf2::equal(back.cview(), ov) ? 1 : 0;
    } catch (const std::exception&) {
        return -1;
    }
}

} // extern "C"
