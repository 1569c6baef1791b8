// Drop-in check: gf2::b200::block_iterative_ple (include/gf2cu/ple.hpp) vs the
// unmodified reference gf2::block_iterative_ple (ple.hpp:166), both called
// the way the reference's own tests call it (test_ple.cpp:133-187). Built
// here against /root/reference/proj/include (read-only) by
// __graft_entry__.build(); the binary runs on the GPU box.
#include <cstdio>
#include <random>

#include "gf2/gf2.hpp"
#include "gf2cu/ple.hpp"

using namespace gf2;

static int failures = 0;
#define CHECK(c, ...)                           \
    do {                                        \
        if (!(c)) {                             \
            std::printf("FAIL: " __VA_ARGS__);  \
            std::printf("\n");                  \
            ++failures;                         \
        }                                       \
    } while (0)

int main() {
    std::mt19937_64 rng(2026);
    int cases = 0;
    for (int rep = 0; rep < 120; ++rep) {
        const std::size_t m = 1 + rng() % 300, n = 1 + rng() % 300;
        BitMatrix a(m, n);
        const int kind = rep % 4;
        if (kind == 0) fill_random(a.view(), 0.5, rng());
        else if (kind == 1) fill_random(a.view(), 0.08, rng());
        else if (kind == 2) fill_random_rows(a.view(), std::min<std::size_t>(n, 1 + rng() % 5), rng());
        else {
            fill_random(a.view(), 0.5, rng());
            for (int k = 0; k < 4 && m > 1; ++k) {
                const std::size_t d = rng() % m, s = rng() % m;
                for (std::size_t j = 0; j < n; ++j) a.set(d, j, a.get(s, j));
            }
        }
        BitMatrix ref = a, dev = a;
        PleConfig cfg;
        cfg.k = unsigned(rng() % 17);
        PleOutcome want = gf2::block_iterative_ple(ref.view(), cfg);
        PleOutcome got = gf2::b200::block_iterative_ple(dev.view(), cfg);
        CHECK(ref == dev, "in-place words differ (case %d, %zux%zu)", rep, m, n);
        CHECK(want.rank == got.rank, "rank %zu vs %zu", want.rank, got.rank);
        CHECK(want.q == got.q, "q differs (case %d)", rep);
        CHECK(want.p.swaps == got.p.swaps, "p.swaps differ (case %d)", rep);
        CHECK(got.processed == m, "processed");
        // canonical col_swaps are accepted by extract_e / rref_from_ple
        BitMatrix e1 = extract_e(ref.cview(), want), e2 = extract_e(dev.cview(), got);
        CHECK(e1 == e2, "extract_e differs (case %d)", rep);
        BitMatrix r1 = ref, r2 = dev;
        rref_from_ple(r1.view(), want, true);
        rref_from_ple(r2.view(), got, true);
        CHECK(r1 == r2, "rref_from_ple differs (case %d)", rep);
        ++cases;
    }
    // unaligned sub-view of a wider parent: bits outside the window untouched
    for (int rep = 0; rep < 20; ++rep) {
        BitMatrix parent(200, 400);
        fill_random(parent.view(), 0.5, 77 + rep);
        BitMatrix p1 = parent, p2 = parent;
        const std::size_t r0 = rng() % 20, c0 = 1 + rng() % 70, rows = 100 + rng() % 80,
                          cols = 100 + rng() % 200;
        PleOutcome want = gf2::block_iterative_ple(p1.view().sub(r0, c0, rows, cols));
        PleOutcome got = gf2::b200::block_iterative_ple(p2.view().sub(r0, c0, rows, cols));
        CHECK(p1 == p2, "sub-view words differ (case %d)", rep);
        CHECK(want.q == got.q && want.p.swaps == got.p.swaps, "sub-view outcome differs");
        ++cases;
    }
    // echelonize(ple_iterative) facade, reduced and not, PLE + RREF on the device
    for (int rep = 0; rep < 40; ++rep) {
        const std::size_t m = 1 + rng() % 400, n = 1 + rng() % 400;
        BitMatrix a(m, n);
        fill_random(a.view(), rep % 2 ? 0.5 : 0.1, 500 + rep);
        const bool full = rep % 4 != 3;
        BitMatrix x = a, y = a;
        const std::size_t r1 = echelonize(x.view(), EchelonStrategy::ple_iterative, full);
        const std::size_t r2 = gf2::b200::echelonize_ple_iterative(y.view(), full);
        CHECK(r1 == r2 && x == y, "echelonize differs (case %d, %zux%zu, full %d)", rep, m, n, full);
        ++cases;
    }
    // rref_from_ple on the device from the reference's own outcome
    for (int rep = 0; rep < 30; ++rep) {
        const std::size_t m = 1 + rng() % 300, n = 1 + rng() % 300;
        BitMatrix a(m, n);
        fill_random(a.view(), rep % 3 ? 0.5 : 0.05, 900 + rep);
        PleOutcome out = gf2::block_iterative_ple(a.view());
        BitMatrix x = a, y = a;
        const bool full = rep % 2 == 0;
        rref_from_ple(x.view(), out, full);
        gf2::b200::rref_from_ple(y.view(), out, full);
        CHECK(x == y, "rref_from_ple differs (case %d, full %d)", rep, full);
        ++cases;
    }
    // corrupt outcome -> std::invalid_argument, as check_pivots (test_ple.cpp:305-314)
    {
        BitMatrix a = BitMatrix(10, 10);
        fill_random(a.view(), 0.5, 5);
        PleOutcome out = gf2::b200::block_iterative_ple(a.view());
        if (out.rank >= 2) {
            std::swap(out.q[0], out.q[1]);
            bool threw = false;
            try {
                gf2::b200::rref_from_ple(a.view(), out, true);
            } catch (const std::invalid_argument&) {
                threw = true;
            }
            CHECK(threw, "corrupt outcome accepted");
            ++cases;
        }
    }
    // trsm_upper_left_unit
    for (int rep = 0; rep < 20; ++rep) {
        const std::size_t r = 1 + rng() % 300, n = 1 + rng() % 300;
        BitMatrix u(r, r), b(r, n);
        fill_random(u.view(), 0.5, 1300 + rep);
        fill_random(b.view(), 0.5, 1400 + rep);
        BitMatrix b1 = b, b2 = b;
        trsm_upper_left_unit(u.cview(), b1.view());
        gf2::b200::trsm_upper_left_unit(u.cview(), b2.view());
        CHECK(b1 == b2, "trsm differs (case %d, r %zu n %zu)", rep, r, n);
        ++cases;
    }
    // recursive_ple (same outputs as the iterative PLE), mul / addmul
    for (int rep = 0; rep < 20; ++rep) {
        const std::size_t m = 1 + rng() % 400, n = 1 + rng() % 400;
        BitMatrix a(m, n);
        fill_random(a.view(), rep % 2 ? 0.5 : 0.05, 1700 + rep);
        BitMatrix x = a, y = a;
        PleConfig cfg;
        cfg.base_bytes = 512;
        cfg.base_ncols = 32;
        PleOutcome want = gf2::recursive_ple(x.view(), cfg);
        PleOutcome got = gf2::b200::recursive_ple(y.view(), cfg);
        CHECK(x == y && want.rank == got.rank && want.q == got.q && want.p.swaps == got.p.swaps,
              "recursive_ple differs (case %d)", rep);
        const std::size_t l = 1 + rng() % 300, k = 1 + rng() % 300;
        BitMatrix u(m, l), v(l, k), c(m, k);
        fill_random(u.view(), 0.5, 1800 + rep);
        fill_random(v.view(), 0.3, 1900 + rep);
        fill_random(c.view(), 0.5, 2000 + rep);
        CHECK(gf2::mul(u.cview(), v.cview()) == gf2::b200::mul(u.cview(), v.cview()),
              "mul differs (case %d)", rep);
        BitMatrix c1 = c, c2 = c;
        gf2::addmul(c1.view(), u.cview(), v.cview());
        gf2::b200::addmul(c2.view(), u.cview(), v.cview());
        CHECK(c1 == c2, "addmul differs (case %d)", rep);
        cases += 3;
    }
    std::printf("%d cases, %d failures\n", cases, failures);
    return failures ? 1 : 0;
}
