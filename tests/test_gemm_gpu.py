"""GPU parity of the GF(2) product (mul / addmul,
multiply.hpp:254-274) through the C ABI vs the oracle's orc_mul (pinned to
the reference's mul in tests/test_rref_host.py); the product is unique, so
bit-exact. The full config-4 size (X 32768x24576 times Y 24576x32768) is
checked through size-independent properties: (XY)v == X(Yv) for random v
and sampled rows recomputed on the host."""
import numpy as np
import pytest

import oracle as O
import paper_1111_6549_b200 as G
import suite as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,l,n", [(1, 1, 1), (3, 70, 5), (64, 64, 64), (65, 129, 63), (200, 300, 100),
                                   (130, 1, 70), (2049, 65, 513), (1000, 2000, 1500), (4100, 700, 64)])
def test_mul(m, l, n):
    a = O.fill_random(m, l, 0.5, m + l)
    b = O.fill_random(l, n, 0.5, l + n)
    want = O.mul(a, l, b, n)
    got = G.mul(G.BitMatrix(m, l, a), G.BitMatrix(l, n, b))
    assert np.array_equal(got.words, want), (m, l, n)


def test_addmul_and_unaligned_views():
    m, l, n = 300, 200, 250
    a = O.fill_random(m, l, 0.5, 1)
    b = O.fill_random(l, n, 0.3, 2)
    c0 = O.fill_random(m, n, 0.5, 3)
    want = c0 ^ O.mul(a, l, b, n)
    c = G.BitMatrix(m, n, c0.copy())
    G.addmul(c, G.BitMatrix(m, l, a), G.BitMatrix(l, n, b))
    assert np.array_equal(c.words, want)
    # c as an unaligned window of a wider parent: outside bits untouched
    parent = O.fill_random(m, 384, 0.5, 4)
    off = 29
    pbits = S.unpack(parent, 384)
    inside = S.pack(pbits[:, off:off + n], n)
    want2 = inside ^ O.mul(a, l, b, n)
    work = parent.copy()
    G.addmul(G.MatrixView(work, 6, off, m, n), G.BitMatrix(m, l, a), G.BitMatrix(l, n, b))
    wbits = S.unpack(work, 384)
    assert np.array_equal(S.pack(wbits[:, off:off + n], n), want2)
    assert np.array_equal(wbits[:, :off], pbits[:, :off])
    assert np.array_equal(wbits[:, off + n:], pbits[:, off + n:])


def test_dimension_mismatch():
    with pytest.raises(ValueError):
        G.mul(G.BitMatrix(3, 4), G.BitMatrix(5, 6))
    with pytest.raises(ValueError):
        G.addmul(G.BitMatrix(3, 7), G.BitMatrix(3, 4), G.BitMatrix(4, 6))


def test_device_resident_mul():
    m, l, n = 3000, 2500, 2200
    a = O.fill_ctr(m, l, 11)
    b = O.fill_ctr(l, n, 12)
    da, db, dc = G.DeviceMatrix(m, l), G.DeviceMatrix(l, n), G.DeviceMatrix(m, n)
    da.fill_ctr(11)
    db.fill_ctr(12)
    G.mul_into(dc, da, db)
    want = O.mul(a, l, b, n)
    assert np.array_equal(dc.download(), want)
    G.addmul(dc, da, db)
    assert not dc.download().any()


def matvec(words, v_words):
    """GF(2) matrix-vector product on packed words: bit i = parity(row_i & v)."""
    cnt = np.bitwise_count(words & v_words[None, :]).sum(axis=1)
    return (cnt & 1).astype(np.uint8)


def pack_bits(bits):
    return S.pack(bits[None, :], bits.shape[0])[0]


@pytest.mark.slow
def test_config4_product_properties():
    """X (32768x24576) * Y (24576x32768), ctr seeds 11 / 12."""
    m, l, n = 32768, 24576, 32768
    dx, dy, dc = G.DeviceMatrix(m, l), G.DeviceMatrix(l, n), G.DeviceMatrix(m, n)
    dx.fill_ctr(11)
    dy.fill_ctr(12)
    G.mul_into(dc, dx, dy)
    x, y, c = dx.download(), dy.download(), dc.download()
    rng = np.random.default_rng(0)
    for _ in range(3):
        v = pack_bits(rng.integers(0, 2, n, dtype=np.uint8))
        yv = pack_bits(matvec(y, v))
        assert np.array_equal(matvec(c, v), matvec(x, yv))
    for i in rng.integers(0, m, 16):
        sel = S.unpack(x[i:i + 1], l)[0].astype(bool)
        assert np.array_equal(c[i], np.bitwise_xor.reduce(y[sel], axis=0))
