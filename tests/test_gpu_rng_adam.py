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
