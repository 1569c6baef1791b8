// gf2cu/ple.hpp -- C++ drop-in for gf2::block_iterative_ple on the B200.
//
// Include AFTER the reference's own headers (proj/include/gf2/ple.hpp): the
// wrapper keeps the reference's public types -- gf2::MatrixView (bit_matrix.hpp:
// 245), gf2::PleConfig / gf2::PleOutcome / gf2::ColSwap (ple.hpp:31-51),
// gf2::RowPermutation (bit_matrix.hpp:416) -- and re-exposes the entry point
//
//     gf2::PleOutcome gf2::b200::block_iterative_ple(gf2::MatrixView a,
//                                                    const gf2::PleConfig& cfg = {});
//
// with the reference's signature, in-place semantics and exception mapping
// (std::invalid_argument / std::out_of_range / std::bad_alloc; CUDA failures
// as std::runtime_error). Callers switch with a using-declaration or by
// qualifying the call; see INTEGRATION.md. Link with -lgf2cu.
#pragma once

#include <cstddef>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gf2cu.h"

namespace gf2 {
namespace b200 {

namespace detail {

inline void throw_status(gf2cu_status st) {
    const std::string msg = gf2cu_last_error();
    switch (st) {
        case GF2CU_OK: return;
        case GF2CU_EINVAL: throw std::invalid_argument(msg);
        case GF2CU_ERANGE: throw std::out_of_range(msg);
        case GF2CU_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error("gf2cu: " + msg);
    }
}

}  // namespace detail

// Device selection for the wrapper (the reference has no notion of devices).
struct DeviceOptions {
    int device = 0;
    void* stream = nullptr;  // cudaStream_t
};

// block_iterative_ple (ple.hpp:166) computed on the B200. Same outputs as the
// reference: rank, processed = nrows, p.swaps, q (bit-exact), the in-place
// L\E words (bit-exact), and col_swaps as the canonical compression list
// {j, q[j], j} for q[j] != j, which extract_e / rref_from_ple / undo_column_swaps
// accept with identical results ("Outputs").
template <class View = gf2::MatrixView, class Cfg = gf2::PleConfig>
gf2::PleOutcome block_iterative_ple(View a, const Cfg& cfg = {}, const DeviceOptions& dev = {}) {
    gf2cu_view v;
    v.data = a.row_words(0);
    v.stride = a.stride();
    v.col_off = a.col_offset();
    v.nrows = a.nrows();
    v.ncols = a.ncols();
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    c.k = cfg.k;
    c.k_scale = cfg.k_scale;
    c.table_count = cfg.table_count;
    c.device = dev.device;
    c.stream = dev.stream;
    const std::size_t cap = std::max<std::size_t>(1, std::min(v.nrows, v.ncols));
    std::vector<std::size_t> swaps(cap), q(cap);
    std::vector<gf2cu_colswap> cs(cap);
    std::size_t rank = 0, ncs = 0;
    detail::throw_status(
        gf2cu_ple(&v, &c, swaps.data(), q.data(), &rank, cs.data(), &ncs, nullptr));
    gf2::PleOutcome out;
    out.rank = rank;
    out.processed = v.nrows;
    out.p.swaps.assign(swaps.begin(), swaps.begin() + rank);
    out.q.assign(q.begin(), q.begin() + rank);
    out.col_swaps.reserve(ncs);
    for (std::size_t i = 0; i < ncs; ++i) out.col_swaps.push_back({cs[i].a, cs[i].b, cs[i].from_row});
    return out;
}

namespace detail {

template <class View>
gf2cu_view to_view(View a) {
    gf2cu_view v;
    v.data = a.nrows() ? a.row_words(0) : nullptr;
    v.stride = a.stride();
    v.col_off = a.col_offset();
    v.nrows = a.nrows();
    v.ncols = a.ncols();
    return v;
}

template <class Cfg>
gf2cu_cfg to_cfg(const Cfg& cfg, const DeviceOptions& dev) {
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    c.k = cfg.k;
    c.k_scale = cfg.k_scale;
    c.table_count = cfg.table_count;
    c.device = dev.device;
    c.stream = dev.stream;
    return c;
}

}  // namespace detail

// rref_from_ple (ple.hpp:318-329) on the B200: `a` holds the in-place result
// `out` describes (a complete decomposition, out.processed == a.nrows()); the
// top out.rank rows become the echelon form (reduced if `full`), rows below
// zero. Throws std::invalid_argument for a corrupt outcome (check_pivots).
template <class View = gf2::MatrixView>
void rref_from_ple(View a, const gf2::PleOutcome& out, bool full = true,
                   const DeviceOptions& dev = {}) {
    if (out.processed != a.nrows())
        throw std::invalid_argument("rref_from_ple on the device needs processed == nrows");
    if (out.q.size() != out.rank) throw std::invalid_argument("rank disagrees with pivot list");
    gf2cu_view v = detail::to_view(a);
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    c.device = dev.device;
    c.stream = dev.stream;
    std::vector<std::size_t> q(out.q.begin(), out.q.end());
    detail::throw_status(gf2cu_rref_from_ple(&v, q.data(), out.rank, full ? 1 : 0, &c));
}

// echelonize(a, EchelonStrategy::ple_iterative, full) (m4ri.hpp:95-98): the
// decomposition and rref_from_ple both on the B200, one upload and download.
template <class View = gf2::MatrixView, class Cfg = gf2::PleConfig>
std::size_t echelonize_ple_iterative(View a, bool full = true, const Cfg& cfg = {},
                                     const DeviceOptions& dev = {}) {
    gf2cu_view v = detail::to_view(a);
    gf2cu_cfg c = detail::to_cfg(cfg, dev);
    std::size_t rank = 0;
    detail::throw_status(gf2cu_echelonize(&v, full ? 1 : 0, &c, &rank));
    return rank;
}

// trsm_upper_left_unit (multiply.hpp:314-335) on the B200: b <- u^-1 b.
template <class CView = gf2::ConstMatrixView, class View = gf2::MatrixView>
void trsm_upper_left_unit(CView u, View b, const DeviceOptions& dev = {}) {
    gf2cu_view uv;
    uv.data = const_cast<uint64_t*>(u.nrows() ? u.row_words(0) : nullptr);
    uv.stride = u.stride();
    uv.col_off = u.col_offset();
    uv.nrows = u.nrows();
    uv.ncols = u.ncols();
    gf2cu_view bv = detail::to_view(b);
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    c.device = dev.device;
    c.stream = dev.stream;
    detail::throw_status(gf2cu_trsm_upper_left_unit(&uv, &bv, &c));
}

// partial_ple (ple.hpp:57-130) on the B200: the lazy single pass. Same rank,
// q, p.swaps and col_swaps as the reference; out.processed is its watermark
// and the rows past it are left untouched (gf2cu_partial_ple).
template <class View = gf2::MatrixView>
gf2::PleOutcome partial_ple(View a, const DeviceOptions& dev = {}) {
    gf2cu_view v = detail::to_view(a);
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    c.device = dev.device;
    c.stream = dev.stream;
    const std::size_t cap = std::max<std::size_t>(1, std::min(v.nrows, v.ncols));
    std::vector<std::size_t> swaps(cap), q(cap);
    std::vector<gf2cu_colswap> cs(cap);
    std::size_t rank = 0, processed = 0, ncs = 0;
    detail::throw_status(gf2cu_partial_ple(&v, &c, swaps.data(), q.data(), &rank, &processed, cs.data(), &ncs));
    gf2::PleOutcome out;
    out.rank = rank;
    out.processed = processed;
    out.p.swaps.assign(swaps.begin(), swaps.begin() + rank);
    out.q.assign(q.begin(), q.begin() + rank);
    for (std::size_t i = 0; i < ncs; ++i) out.col_swaps.push_back({cs[i].a, cs[i].b, cs[i].from_row});
    return out;
}

// undo_column_swaps (ple.hpp:293-296) on the B200.
template <class View = gf2::MatrixView>
void undo_column_swaps(View a, const std::vector<gf2::ColSwap>& swaps, const DeviceOptions& dev = {}) {
    gf2cu_view v = detail::to_view(a);
    gf2cu_cfg c;
    gf2cu_default_config(&c);
    c.device = dev.device;
    c.stream = dev.stream;
    std::vector<gf2cu_colswap> cs;
    cs.reserve(swaps.size());
    for (const auto& x : swaps) cs.push_back(gf2cu_colswap{x.a, x.b, x.from_row});
    detail::throw_status(gf2cu_undo_column_swaps(&v, cs.data(), cs.size(), &c));
}

// echelonize(a, strategy, full, cfg) (m4ri.hpp:87-106) on the B200. Every
// strategy's result is the same matrix -- the reduced form is unique, and the
// non-reduced forms of naive / m4ri / ple_iterative / ple_recursive coincide
// (pinned in tests/test_rref_host.py::test_strategy_equivalences_pinned) --
// so all of them are served by the device PLE + rref_from_ple.
template <class View, class Strategy, class Cfg = gf2::PleConfig>
std::size_t echelonize(View a, Strategy, bool full = true, const Cfg& cfg = {},
                       const DeviceOptions& dev = {}) {
    return echelonize_ple_iterative(a, full, cfg, dev);
}

// recursive_ple (ple.hpp:246-289): its in-place result, rank, q and p.swaps
// equal block_iterative_ple's (pinned in tests/test_rref_host.py), so the
// device path serves it.
template <class View = gf2::MatrixView, class Cfg = gf2::PleConfig>
gf2::PleOutcome recursive_ple(View a, const Cfg& cfg = {}, const DeviceOptions& dev = {}) {
    return block_iterative_ple(a, cfg, dev);
}

// addmul (multiply.hpp:254-264): c ^= a * b on the B200.
template <class View = gf2::MatrixView, class CView = gf2::ConstMatrixView>
void addmul(View c, CView a, CView b, const DeviceOptions& dev = {}) {
    gf2cu_view cv = detail::to_view(c), av, bv;
    for (auto [dst, src] : {std::pair<gf2cu_view*, const CView*>{&av, &a}, {&bv, &b}}) {
        dst->data = const_cast<uint64_t*>(src->nrows() ? src->row_words(0) : nullptr);
        dst->stride = src->stride();
        dst->col_off = src->col_offset();
        dst->nrows = src->nrows();
        dst->ncols = src->ncols();
    }
    gf2cu_cfg cc;
    gf2cu_default_config(&cc);
    cc.device = dev.device;
    cc.stream = dev.stream;
    detail::throw_status(gf2cu_addmul(&cv, &av, &bv, &cc));
}

// mul (multiply.hpp:266-274): a new a.nrows() x b.ncols() product.
template <class CView = gf2::ConstMatrixView>
gf2::BitMatrix mul(CView a, CView b, const DeviceOptions& dev = {}) {
    gf2::BitMatrix c(a.nrows(), b.ncols());
    addmul(c.view(), a, b, dev);
    return c;
}

}  // namespace b200
}  // namespace gf2
