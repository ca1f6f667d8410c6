"""Device RNG and Adam vs the golden reference vectors (bit-exact)."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def test_rng_selftest_and_streams(dev_lib):
    from paper_2510_19764_b200 import _lib
    g = golden("rng.npz")
    st = _lib.stream_ptr()
    out = torch.zeros(3, dtype=torch.int64, device="cuda")
    _lib.call("sw_rng_selftest", out.data_ptr(), st)
    assert [int(x) for x in out.cpu().numpy().view(np.uint64)] == [0, 6238072747940578789,
                                                                    16294208416658607535]
    key = int(g["key"])
    d = torch.zeros(4096, dtype=torch.int64, device="cuda")
    _lib.call("sw_rng_u64", key, 0, 4096, d.data_ptr(), st)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), g["draws"])
    u = torch.zeros(4096, dtype=torch.float64, device="cuda")
    _lib.call("sw_rng_uniform01", key, 0, 4096, u.data_ptr(), st)
    assert np.array_equal(u.cpu().numpy(), g["u01"])
    c = torch.zeros(300, dtype=torch.int64, device="cuda")
    _lib.call("sw_rng_child_keys", key, 300, c.data_ptr(), st)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), g["child"])
    from paper_2510_19764_b200.rng import fold_key
    for n, row in zip(g["ns"], g["ui"]):
        o = torch.zeros(513, dtype=torch.int64, device="cuda")
        _lib.call("sw_rng_uniform_int_seq", fold_key(9, "uint", int(n)), int(n), 512, o.data_ptr(), st)
        assert np.array_equal(o.cpu().numpy().view(np.uint64), row)


def test_adam_matches_golden(dev_lib):
    from paper_2510_19764_b200.plasticity import Adam
    g = golden("adam.npz")
    p = torch.from_numpy(g["p0"].copy()).cuda()
    a = Adam(shape=p.shape)
    for t in range(5):
        gr = torch.from_numpy(g[f"g{t}"].copy()).cuda()
        a.apply(p, gr)
        assert np.array_equal(p.cpu().numpy(), g[f"p{t + 1}"])
        assert np.array_equal(a.m.cpu().numpy(), g[f"m{t + 1}"])
        assert np.array_equal(a.v.cpu().numpy(), g[f"v{t + 1}"])
        assert not gr.any().item()


def test_bitfield_api_matches_oracle_words(dev_lib):
    """Reference Bitfield API (bitfield.py:32-90) on the device words against
    the oracle bit helpers: set/clear/test, vector forms, k random bits
    (draw order of sample_k_distinct), ascending set bits, popcounts."""
    import numpy as np
    from oracle.ragged import bf_clear, bf_set, bf_test, bf_words
    from oracle.rng import Stream
    from paper_2510_19764_b200.bitfield import Bitfield
    from paper_2510_19764_b200.rng import CounterRng
    P, N = 6, 130
    bf = Bitfield(P, N)
    ref = np.zeros((P, bf_words(N)), dtype=np.uint64)
    rs = np.random.default_rng(1)
    for _ in range(200):
        i, j = int(rs.integers(P)), int(rs.integers(N))
        if rs.random() < 0.6:
            bf.set_bit(i, j); bf_set(ref, i, j)
        else:
            bf.clear_bit(i, j); bf_clear(ref, i, j)
    cols = rs.integers(0, N, 40)
    bf.set_bits(2, cols)
    for c in cols:
        bf_set(ref, 2, int(c))
    bf.clear_bits(3, cols[:10])
    for c in cols[:10]:
        bf_clear(ref, 3, int(c))
    assert np.array_equal(bf.host_words(), ref)
    assert list(bf.test_bits(2, cols)) == [bool(bf_test(ref, 2, int(c))) for c in cols]
    rc = rs.integers(0, N, (P, 7))
    assert np.array_equal(bf.test_bits_rows(rc),
                          np.array([[bool(bf_test(ref, r, int(c))) for c in rc[r]] for r in range(P)]))
    got = bf.set_k_random_bits_in_row(5, 9, CounterRng(3, "k"))
    want = Stream.of(3, "k").sample_k_distinct(9, N)
    assert list(got) == list(want)
    for c in want:
        bf_set(ref, 5, int(c))
    assert np.array_equal(bf.host_words(), ref)
    for r in range(P):
        asc = [j for j in range(N) if bf_test(ref, r, j)]
        assert list(bf.set_bits_in_row(r)) == asc and bf.row_popcount(r) == len(asc)
    assert bf.popcount() == sum(bf.row_popcount(r) for r in range(P))
    bf.clear_row(5)
    assert bf.row_popcount(5) == 0
