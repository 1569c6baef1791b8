"""GPU: the check mode and the synchronization litmus runs.

Check mode (PleConfig(check=True), GF2CU_FLAG_CHECK, or GF2CU_CHECK=1) makes
every step assert SURVEY.md 8(c) invariant (iv) on every row's panel word and
the result assert invariants (i) and (ii); the first violating step comes
back as GF2CU_ECHECK. The litmus runs exercise the drivers' cross-CTA
hand-offs with the same primitives and count stale reads."""
import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
from paper_1111_6549_b200._lib import Gf2cuCheckError

pytestmark = pytest.mark.gpu

DRIVERS = {"single": dict(single_panel=True), "super": dict(super_step=True),
           "multi": dict(multi_kernel=True), "peer3": dict(peer_ranks=3), "peer4s": dict(peer_ranks=4, super_step=True)}


def inputs():
    yield "dense", O.fill_random(1500, 1300, 0.5, 3), 1500, 1300
    yield "p256", O.fill_random(2000, 2000, 1 / 256, 4), 2000, 2000
    a = O.fill_ctr(1800, 1700, 5)
    a[200:700] = a[900:1400]
    yield "deficient", a, 1800, 1700
    yield "xy", O.mul(O.fill_ctr(1200, 700, 6), 700, O.fill_ctr(700, 1500, 7), 1500), 1200, 1500


@pytest.mark.parametrize("driver", sorted(DRIVERS))
def test_check_mode_passes_and_is_exact(driver):
    for name, a, m, n in inputs():
        ref = a.copy()
        want = O.ple(ref, m, n)
        bm = G.BitMatrix(m, n, a.copy())
        got = G.block_iterative_ple(bm, G.PleConfig(check=True, **DRIVERS[driver]))
        assert got.rank == want.rank and np.array_equal(bm.words, ref), (driver, name)


def col63_dependent(m, n, seed):
    """Column 64w+63 a copy of column 64w+62 in every word: no panel ever has
    a pivot in its last column, so a stray bit there is a finished column
    holding a bit below the pivots. (In a full-rank panel every column is a
    pivot column and every bit is a legal multiplier: invariant (iv) cannot
    see a wrong word there.)"""
    a = O.fill_random(m, n, 0.5, seed)
    b62 = (a >> np.uint64(62)) & np.uint64(1)
    return (a & ~np.uint64(1 << 63)) | (b62 << np.uint64(63))


def test_check_mode_from_the_environment(monkeypatch):
    monkeypatch.setenv("GF2CU_CHECK", "1")
    monkeypatch.setenv("GF2CU_CHECK_INJECT", "3")  # corrupt a row's word at step 2
    with pytest.raises(Gf2cuCheckError, match="step 2"):
        G.block_iterative_ple(G.BitMatrix(700, 704, col63_dependent(700, 704, 8)))


@pytest.mark.parametrize("super_step", [False, True])
def test_check_mode_detects_a_corrupted_panel_word(monkeypatch, super_step):
    """The checker's own test: GF2CU_CHECK_INJECT=s+1 flips the top bit of
    the first non-pivot row's panel word at step s; that row then carries a
    bit in a finished column, which invariant (iv) forbids."""
    a = col63_dependent(2000, 2048, 9)
    for step in (0, 6, 18):  # (even: the super-step driver applies panel a at even steps)
        monkeypatch.setenv("GF2CU_CHECK_INJECT", str(step + 1))
        with pytest.raises(Gf2cuCheckError, match=f"step {step} "):
            G.block_iterative_ple(G.BitMatrix(2000, 2048, a.copy()),
                                  G.PleConfig(check=True, super_step=super_step, single_panel=not super_step))
    monkeypatch.delenv("GF2CU_CHECK_INJECT")
    bm = G.BitMatrix(2000, 2048, a.copy())
    ref = a.copy()
    want = O.ple(ref, 2000, 2048)
    got = G.block_iterative_ple(bm, G.PleConfig(check=True))  # and clean again
    assert got.rank == want.rank and np.array_equal(bm.words, ref)


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_litmus_handoffs(kind):
    checked, failures = G.litmus(kind, rounds=300)
    assert checked > 0 and failures == 0, (kind, checked, failures)
