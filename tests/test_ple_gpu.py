"""GPU parity: the B200 path (through the C ABI) vs the C restatement
(oracle/ple_oracle.c, itself pinned to the compiled reference in
tests/test_oracle.py) on seeded inputs. Bit-exact: in-place L\\E words,
rank, p.swaps, q, and the canonical col_swaps list."""
import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
import suite as S

pytestmark = pytest.mark.gpu


def run_both(a_words, m, n, cfg=None):
    ref = a_words.copy()
    want = O.ple(ref, m, n)
    bm = G.BitMatrix(m, n, a_words.copy())
    got = G.block_iterative_ple(bm, cfg)
    return ref, want, bm, got


def assert_same(ref, want, bm, got, what=""):
    assert got.rank == want.rank, what
    assert np.array_equal(got.p.swaps, want.swaps.astype(np.uint64)), what
    assert np.array_equal(got.q, want.q.astype(np.uint64)), what
    cs = np.array([[c.a, c.b, c.from_row] for c in got.col_swaps], dtype=np.uint64).reshape(-1, 3)
    assert np.array_equal(cs, want.col_swaps.astype(np.uint64).reshape(-1, 3)), what
    if not np.array_equal(bm.words, ref):
        bad = np.argwhere(bm.words != ref)
        raise AssertionError(f"{what}: {len(bad)} words differ, first at {bad[:5].tolist()}")


SMALL = [(1, 1), (1, 64), (64, 1), (2, 3), (31, 33), (63, 64), (64, 64), (65, 65), (127, 129),
         (128, 128), (129, 127), (150, 300), (300, 150), (257, 193), (200, 1000), (1000, 200),
         (130, 190), (190, 130), (70, 257)]


@pytest.mark.parametrize("super_step", [False, True])
@pytest.mark.parametrize("m,n", SMALL)
@pytest.mark.parametrize("kind", ["dense", "thin", "ctr", "deficient"])
def test_small_shapes(m, n, kind, super_step):
    seed = m * 1000 + n
    if kind == "dense":
        a = O.fill_random(m, n, 0.5, seed)
    elif kind == "thin":
        a = O.fill_random(m, n, 0.08, seed)
    elif kind == "ctr":
        a = O.fill_ctr(m, n, seed)
    else:
        a = O.fill_random(m, n, 0.5, seed)
        rng = np.random.default_rng(seed)
        for _ in range(4):
            d, s = rng.integers(0, m, 2)
            a[d] = a[s]
    cfg = G.PleConfig(super_step=True) if super_step else None
    assert_same(*run_both(a, m, n, cfg), what=f"{kind} {m}x{n} super={super_step}")


@pytest.mark.parametrize("super_step", [False, True])
@pytest.mark.parametrize("ranks", [1, 2, 5, 8])
@pytest.mark.parametrize("m,n", SMALL)
@pytest.mark.parametrize("kind", ["dense", "deficient"])
def test_small_shapes_peer_ranks(m, n, kind, ranks, super_step):
    """The row-sharded peer-memory driver (one or two panels per sweep) with
    1-8 emulated ranks; rows are spread over the ranks in small blocks."""
    seed = m * 1000 + n
    a = O.fill_random(m, n, 0.5, seed)
    if kind == "deficient":
        rng = np.random.default_rng(seed)
        for _ in range(4):
            d, s = rng.integers(0, m, 2)
            a[d] = a[s]
    cfg = G.PleConfig(peer_ranks=ranks, super_step=super_step)
    assert_same(*run_both(a, m, n, cfg), what=f"{kind} {m}x{n} ranks={ranks} super={super_step}")


@pytest.mark.parametrize("m,n,density", [(1024, 1024, 0.5), (2048, 2048, 0.5), (1500, 2500, 0.5),
                                         (2048, 2048, 1 / 64), (2048, 2048, 1 / 256),
                                         (4096, 4096, 0.5)])
@pytest.mark.parametrize("super_step", [False, True])
def test_medium(m, n, density, super_step):
    a = O.fill_random(m, n, density, 7)
    cfg = G.PleConfig(super_step=True) if super_step else G.PleConfig(single_panel=True)
    assert_same(*run_both(a, m, n, cfg), what=f"{m}x{n} p={density} super={super_step}")


def test_zero_and_identity():
    for m, n in [(8, 12), (100, 300), (300, 100)]:
        a = np.zeros((m, (n + 63) // 64), dtype=np.uint64)
        assert_same(*run_both(a, m, n), what="zero")
    n = 200
    bm = G.BitMatrix.identity(n)
    before = bm.copy()
    out = G.block_iterative_ple(bm)
    assert out.rank == n and bm == before
    assert list(out.p.swaps) == list(range(n)) and list(out.q) == list(range(n))
    assert out.col_swaps == []


def test_rank_deficient_product():
    m, l, n = 1024, 700, 1100
    x = O.fill_ctr(m, l, 11)
    y = O.fill_ctr(l, n, 12)
    a = O.mul(x, l, y, n)
    ref, want, bm, got = run_both(a, m, n)
    assert want.rank <= l
    assert_same(ref, want, bm, got, what="X*Y")


def test_dropin_cpp_binary():
    """The C++ drop-in (include/gf2cu/ple.hpp) against the unmodified reference,
    both in one binary built here from /root/reference headers."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/test_dropin not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


DRIVERS = {"super": (G.PleConfig(super_step=True), 2), "single": (G.PleConfig(single_panel=True), 1),
           "multi": (G.PleConfig(multi_kernel=True), 0), "peer1": (G.PleConfig(peer_ranks=1), 3),
           "peer3": (G.PleConfig(peer_ranks=3), 3), "peer8": (G.PleConfig(peer_ranks=8), 3),
           "peer1s": (G.PleConfig(peer_ranks=1, super_step=True), 4),
           "peer4s": (G.PleConfig(peer_ranks=4, super_step=True), 4)}


@pytest.mark.parametrize("driver", sorted(DRIVERS))
@pytest.mark.parametrize("m,n,gen", [(3000, 3000, "dense"), (2048, 2048, "p256"), (1500, 4000, "ctr"),
                                     (4000, 1500, "ctr"), (2500, 2500, "dup")])
def test_drivers_agree(m, n, gen, driver):
    """All drivers (super-step: two panels per sweep / persistent single-panel
    / one launch per phase) are bit-exact."""
    if gen == "dense":
        a = O.fill_random(m, n, 0.5, 5)
    elif gen == "p256":
        a = O.fill_random(m, n, 1 / 256, 5)
    elif gen == "ctr":
        a = O.fill_ctr(m, n, 5)
    else:
        a = O.fill_ctr(m, n, 6)
        a[100:900] = a[1000:1800]  # rank deficiency: pivotless columns, window misses
    ref = a.copy()
    want = O.ple(ref, m, n)
    bm = G.BitMatrix(m, n, a.copy())
    cfg, code = DRIVERS[driver]
    got = G.block_iterative_ple(bm, cfg)
    assert got.stats["driver"] == code
    assert_same(ref, want, bm, got, what=f"{gen} {m}x{n} driver={driver}")


def ctr_rows(rows, n, seed):
    """Rows of the counter generator, random access."""
    W = (n + 63) // 64
    i = np.asarray(rows, dtype=np.uint64)[:, None]
    x0 = np.arange(W, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        x = (np.uint64(seed) << np.uint64(32)) + (i * np.uint64(W) + x0 + np.uint64(1)) * np.uint64(
            0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    if n % 64:
        x[:, -1] &= np.uint64((1 << (n % 64)) - 1)
    return x


@pytest.mark.slow
def test_131072_reconstruction_sample():
    """BASELINE config 5's large case (131072^2, 2 GiB) on one GPU: the
    reference would take ~36 CPU-minutes, so the check is size-independent:
    sampled rows of P * L * E (ple_reconstruct, ple.hpp:355-358, with E in
    closed form) equal the input rows."""
    n = 131072
    dm = G.DeviceMatrix(n, n)
    dm.fill_ctr(1)
    out = G.block_iterative_ple(dm)
    assert out.stats["driver"] == 2
    r = out.rank
    assert r > n - 64
    words = dm.download()
    W = words.shape[1]
    q = np.asarray(out.q, dtype=np.int64)
    # position i holds input row idx[i] (the swaps applied in order)
    idx = np.arange(n)
    for i, s in enumerate(np.asarray(out.p.swaps, dtype=np.int64)):
        idx[i], idx[s] = idx[s], idx[i]
    cols = np.arange(W)
    for i in [0, 1, 63, 64, 12345, 65537, 131000, r - 1, min(r, n - 1), n - 1]:
        lim = min(i, r)
        lbits = S.unpack(words[i:i + 1], lim)[0] if lim else np.zeros(0, np.uint8)
        sel = list(np.nonzero(lbits)[0])
        if i < r:
            sel.append(i)
        sel = np.asarray(sel, dtype=np.int64)
        if sel.size == 0:
            prod = np.zeros(W, dtype=np.uint64)
        else:
            T = words[sel].copy()
            qs = q[sel]
            T[cols[None, :] < (qs >> 6)[:, None]] = 0
            lo = (qs & 63) + 1
            keep = np.where(lo >= 64, np.uint64(0), ~((np.uint64(1) << lo.astype(np.uint64)) - np.uint64(1)))
            T[np.arange(sel.size), qs >> 6] &= keep
            T[np.arange(sel.size), qs >> 6] |= np.uint64(1) << (qs & 63).astype(np.uint64)
            prod = np.bitwise_xor.reduce(T, axis=0)
        assert np.array_equal(prod, ctr_rows([idx[i]], n, 1)[0]), f"position {i}"


def golden(name):
    """A full-size entry of tests/golden/full_configs.json (the compiled
    reference's rank and outcome hash), or None."""
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "full_configs.json")
    with open(p) as f:
        return {c["name"]: c for c in json.load(f)["configs"]}.get(name)


@pytest.mark.parametrize("m,n,name", [(16384, 16384, "s_16384_dup3"), (12000, 20000, "s_12000x20000_dup3"),
                                      (20000, 9000, "s_20000x9000_dup3")])
def test_streamed_output_matches_device(m, n, name):
    """gf2cu_ple on an aligned host view with the super-step driver copies the
    rows the kernel finishes to the host while it runs (chunks of >= m/32
    rows); the host result must equal the device-resident run's, and both the
    compiled reference's (golden outcome hash)."""
    a = O.fill_ctr(m, n, 3)
    a[m // 3: m // 3 + 200] = a[10:210]  # some rank deficiency
    bm = G.BitMatrix(m, n, a.copy())
    got = G.block_iterative_ple(bm, G.PleConfig(super_step=True))
    d = G.DeviceMatrix(m, n)
    d.upload(a)
    want = G.block_iterative_ple(d, G.PleConfig(super_step=True))
    assert got.rank == want.rank
    assert np.array_equal(got.q, want.q) and np.array_equal(got.p.swaps, want.p.swaps)
    assert np.array_equal(bm.words, d.download())
    g = golden(name)
    assert g is not None, f"{name} missing from tests/golden/full_configs.json"
    assert got.rank == g["rank"]
    assert S.outcome_hash(bm.words, n, got.rank, got.p.swaps, got.q) == g["sha256"]


@pytest.mark.parametrize("m,n,driver,name", [(8192, 65536, 2, "m_8192x65536_ctr9"), (20480, 20480, 2, "m_20480_ctr9"),
                                             (16384, 24576, 2, "m_16384x24576_ctr9"),
                                             (16384, 16384, 1, "m_16384_ctr9"), (12288, 12288, 1, "m_12288_ctr9")])
def test_default_driver_size_rule(m, n, driver, name):
    """Without a driver flag the super-step driver runs from 5 * 2^20 matrix words
    (m * ceil(n/64)) up, the single-panel persistent driver below (the measured
    crossover); both drivers give the compiled
    reference's result (golden outcome hash of the ctr(seed 9) matrix)."""
    d = G.DeviceMatrix(m, n)
    d.fill_ctr(9)
    e = G.DeviceMatrix(m, n)
    e.copy_from(d)
    got = G.block_iterative_ple(d)
    assert got.stats["driver"] == driver
    other = G.block_iterative_ple(e, G.PleConfig(single_panel=True) if driver == 2 else G.PleConfig(super_step=True))
    assert other.rank == got.rank and np.array_equal(other.q, got.q)
    assert d.checksum() == e.checksum()
    g = golden(name)
    assert g is not None, f"{name} missing from tests/golden/full_configs.json"
    assert got.rank == g["rank"]
    assert S.outcome_hash(d.download(), n, got.rank, got.p.swaps, got.q) == g["sha256"]


@pytest.mark.parametrize("m,n,gen", [(3000, 3000, "dense"), (2500, 2500, "dup"), (1500, 4000, "ctr"),
                                     (4000, 1500, "p256")])
def test_panel_tuning_bits_exact(m, n, gen, monkeypatch):
    """The panel tuning bits (GF2CU_PANEL_FLAGS: 1 = followers apply the
    leader's pivots as published, 2 = the super-step look-ahead across
    super-steps) change the schedule, never the result: every combination is
    bit-exact against the oracle on both persistent drivers."""
    if gen == "dense":
        a = O.fill_random(m, n, 0.5, 21)
    elif gen == "p256":
        a = O.fill_random(m, n, 1 / 256, 21)
    elif gen == "ctr":
        a = O.fill_ctr(m, n, 21)
    else:
        a = O.fill_ctr(m, n, 22)
        a[100:900] = a[1000:1800]  # pivotless columns, window misses
    ref = a.copy()
    want = O.ple(ref, m, n)
    for flags in ("0", "1", "2", "3"):
        monkeypatch.setenv("GF2CU_PANEL_FLAGS", flags)
        for cfg in (G.PleConfig(super_step=True), G.PleConfig(single_panel=True)):
            bm = G.BitMatrix(m, n, a.copy())
            got = G.block_iterative_ple(bm, cfg)
            assert_same(ref, want, bm, got, what=f"{gen} {m}x{n} flags={flags}")


@pytest.mark.parametrize("k,k_scale,tables", [(0, 0.0, 4), (0, -3.0, 4), (0, float("nan"), 1),
                                             (0, 1e-9, 0), (0, 1e9, 4), (99, -1.0, 100)])
def test_any_pleconfig_is_accepted(k, k_scale, tables):
    """pick_table_bits clamps any k_scale to k in [1, 16] (gray_code.hpp:171-177)
    and the driver clamps k / table_count (ple.hpp:168-169, 201): the reference
    never throws on a PleConfig, and the output does not depend on it."""
    a = O.fill_random(300, 200, 0.5, 5)
    cfg = G.PleConfig(k=k, k_scale=k_scale, table_count=tables)
    assert_same(*run_both(a, 300, 200, cfg), what=f"k={k} k_scale={k_scale} tables={tables}")


def test_partial_ple_device_matches_reference():
    """gf2cu_partial_ple (ple.hpp:57-130) against the compiled reference's
    partial_ple: in-place words (rows past the watermark untouched), rank,
    p.swaps, q, processed, col_swaps."""
    rng = np.random.default_rng(4242)
    early = 0
    cases = [(0, 5), (5, 0), (1, 1), (70, 64), (200, 64), (300, 65), (64, 64), (129, 63)]
    cases += [(int(rng.integers(1, 300)), int(rng.integers(1, 300))) for _ in range(40)]
    cases += [(n + int(rng.integers(1, 200)), n) for n in rng.integers(1, 130, 40)]
    for i, (m, n) in enumerate(cases):
        a = S.build(m, n, i % 7, int(rng.integers(0, 2**62))) if m and n else np.zeros((m, 1), np.uint64)
        if i % 3 == 1 and n > 2:  # empty leading columns: compression swaps on the unread rows
            for c in range(int(rng.integers(1, n))):
                a[:, c >> 6] &= ~np.uint64(1 << (c & 63))
        want_words = a.copy()
        if m and n:
            want, wp = O.partial_ple(want_words, m, n)
        else:
            want, wp = O.Outcome(0, np.zeros(0), np.zeros(0)), 0
        bm = G.BitMatrix(m, n, a.copy()) if m and n else G.BitMatrix(m, n)
        got = G.partial_ple(bm)
        assert (got.rank, got.processed) == (want.rank, wp), (m, n)
        assert np.array_equal(got.p.swaps, np.asarray(want.swaps, np.uint64)), (m, n)
        assert np.array_equal(got.q, np.asarray(want.q, np.uint64)), (m, n)
        if m and n:
            assert np.array_equal(bm.words, want_words), (m, n)
        early += wp < m
    assert early > 10


def test_undo_column_swaps_device():
    """gf2cu_undo_column_swaps (ple.hpp:293-296) vs the restatement, on a
    rank-deficient PLE's canonical list and on arbitrary swap lists, host
    view (unaligned sub-view) and device-resident."""
    m, n = 300, 260
    a = O.mul(O.fill_ctr(m, 200, 9), 200, O.fill_ctr(200, n, 10), n)  # rank <= 200 < n
    bm = G.BitMatrix(m, n, a.copy())
    out = G.block_iterative_ple(bm)
    assert len(out.col_swaps) > 0
    want = bm.words.copy()
    O.undo_col_swaps(want, m, out.col_swaps_array.astype(np.uintp))
    G.undo_column_swaps(bm, out.col_swaps)
    assert np.array_equal(bm.words, want)
    rng = np.random.default_rng(5)
    cs = np.stack([rng.integers(0, 190, 40), rng.integers(0, 190, 40), rng.integers(0, 120, 40)], 1)
    par = O.fill_random(120, 320, 0.5, 10)
    win = G.MatrixView(par, par.shape[1], 70, 120, 190)
    sub = np.zeros((120, 3), dtype=np.uint64)
    for i in range(120):  # the window as a packed 120 x 190 matrix
        for j in range(190):
            if (int(par[i, (70 + j) >> 6]) >> ((70 + j) & 63)) & 1:
                sub[i, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
    O.undo_col_swaps(sub, 120, cs.astype(np.uintp))
    before = par.copy()
    G.undo_column_swaps(win, cs)
    for i in range(120):
        for j in range(320):
            bit = (int(par[i, j >> 6]) >> (j & 63)) & 1
            if 70 <= j < 260:
                assert bit == (int(sub[i, (j - 70) >> 6]) >> ((j - 70) & 63)) & 1
            else:
                assert bit == (int(before[i, j >> 6]) >> (j & 63)) & 1
    d = G.DeviceMatrix(m, n)
    d.upload(a)
    G.undo_column_swaps(d, cs)
    want = a.copy()
    O.undo_col_swaps(want, m, cs.astype(np.uintp))
    assert np.array_equal(d.download(), want)
    with pytest.raises(IndexError):
        G.undo_column_swaps(G.BitMatrix(4, 4), [G.ColSwap(0, 4, 0)])


def test_concurrent_host_threads():
    """The reference is re-entrant (no globals on the path; callers
    may factor different matrices from different threads). The drop-in keeps its
    device buffers, streams and staging per host thread: four threads factoring,
    echelonizing and multiplying different shapes at once, each result against
    the oracle."""
    import threading

    errors = []

    def worker(tid):
        try:
            rng = np.random.default_rng(1000 + tid)
            for it in range(12):
                m, n = int(rng.integers(50, 900)), int(rng.integers(50, 900))
                a = S.build(m, n, int(rng.integers(2, 7)), int(rng.integers(0, 2**40)))
                cfg = [None, G.PleConfig(super_step=True), G.PleConfig(single_panel=True),
                       G.PleConfig(peer_ranks=2)][(tid + it) % 4]
                assert_same(*run_both(a, m, n, cfg), what=f"thread {tid} it {it} {m}x{n}")
                rref = a.copy()
                r = O.echelonize(rref, m, n, True)
                bm = G.BitMatrix(m, n, a.copy())
                assert G.echelonize(bm, True) == r and np.array_equal(bm.words, rref), f"thread {tid} echelonize"
                k = int(rng.integers(1, 300))
                b = O.fill_random(n, k, 0.5, tid * 100 + it)
                got = G.mul(G.BitMatrix(m, n, a), G.BitMatrix(n, k, b)).words
                assert np.array_equal(got, O.mul(a, n, b, k)), f"thread {tid} mul"
        except BaseException as e:  # noqa: BLE001
            errors.append(f"thread {tid}: {e!r}")

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "a thread hangs"
    assert not errors, errors


def _structured(kind, m, n, seed):
    rng = np.random.default_rng(seed)
    W = (n + 63) // 64
    if kind == "permutation":  # every pivot is a window miss, found at a random depth
        a = np.zeros((m, W), dtype=np.uint64)
        p = rng.permutation(max(m, n))[:m] % n
        a[np.arange(m), p >> 6] = np.uint64(1) << (p & 63).astype(np.uint64)
        return a
    if kind == "zero_top":  # the first half of the rows is empty: scans go thousands of rows deep
        a = O.fill_random(m, n, 0.5, seed)
        a[: m // 2] = 0
        return a
    if kind == "nnz3":
        return O.fill_random_rows(m, n, 3, seed)
    if kind == "p1024":
        return O.fill_random(m, n, 1 / 1024, seed)
    if kind == "rank40":  # the trailing matrix is exhausted after the first panel
        return O.mul(O.fill_random(m, 40, 0.5, seed), 40, O.fill_random(40, n, 0.5, seed + 1), n)
    if kind == "zero_left":  # whole panels without a pivot, then a dense block
        a = O.fill_random(m, n, 0.5, seed)
        a[:, : W // 2] = 0
        return a
    if kind == "zero_left_rank40":  # empty panels followed by data, then an exhausted trailing matrix
        a = O.mul(O.fill_random(m, 40, 0.5, seed), 40, O.fill_random(40, n, 0.5, seed + 1), n)
        a[:, : W // 3] = 0
        return a
    if kind == "deep_single":  # one column whose only 1 sits in the last row
        a = O.fill_random(m, n, 0.5, seed)
        a[:, 1] &= ~np.uint64(1 << 7)
        a[m - 1, 1] |= np.uint64(1 << 7)
        return a
    raise ValueError(kind)


@pytest.mark.parametrize("driver", ["single", "super", "peer2", "peer3s"])
@pytest.mark.parametrize("kind", ["permutation", "zero_top", "nnz3", "p1024", "rank40", "zero_left",
                                  "zero_left_rank40", "deep_single"])
def test_structured_inputs_deep_scans(kind, driver):
    """Window-miss scans that go past their first chunk (several doubling
    rounds), rows that are dead for a whole panel, pivotless panels and the
    column skip after them, exhausted trailing matrices (the two-panel
    driver's early stop, with and without data after the first empty panels),
    on every persistent driver."""
    m, n = 6200, 6144
    cfg = {"single": G.PleConfig(single_panel=True), "super": G.PleConfig(super_step=True),
           "peer2": G.PleConfig(peer_ranks=2), "peer3s": G.PleConfig(peer_ranks=3, super_step=True)}[driver]
    a = _structured(kind, m, n, 77)
    assert_same(*run_both(a, m, n, cfg), what=f"{kind} {driver}")


def test_sparse_inputs_take_the_single_panel_driver(monkeypatch):
    """The size rule's two-panel driver falls back to the single-panel one for
    sparse inputs (sampled density below 1/384), on device-resident and host
    matrices; dense inputs, forced drivers and GF2CU_SPARSE_RULE=0 are not
    affected. Bit-exact either way."""
    m = n = 20480  # above the size rule's switch
    for p, want in ((1 / 1024, 1), (0.5, 2)):
        a = O.fill_random(m, n, p, 5)
        d = G.DeviceMatrix(m, n)
        d.upload(a)
        out = G.block_iterative_ple(d)
        assert out.stats["driver"] == want, (p, out.stats["driver"])
        bm = G.BitMatrix(m, n, a.copy())
        o2 = G.block_iterative_ple(bm)
        assert o2.stats["driver"] == want and o2.rank == out.rank
        got = np.empty_like(a)
        d.download(got)
        assert np.array_equal(got, bm.words) and np.array_equal(out.q, o2.q)
        if want == 1:
            d.upload(a)
            assert G.block_iterative_ple(d, G.PleConfig(super_step=True)).stats["driver"] == 2
            d.download(got)
            assert np.array_equal(got, bm.words)
            monkeypatch.setenv("GF2CU_SPARSE_RULE", "0")
            d.upload(a)
            assert G.block_iterative_ple(d).stats["driver"] == 2
            monkeypatch.delenv("GF2CU_SPARSE_RULE")
        d.close()
