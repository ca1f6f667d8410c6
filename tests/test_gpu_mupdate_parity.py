"""SURVEY §8(d) M-update parity instance, bit-exact (tier P1).

P = 16 384 rows, N = 65 536 posts, cap = 1024.  Rows are Bernoulli(512/N)
from the counters of stream (seed, "init", "M") (counter i*N + j, as
init_pairwise_bernoulli draws them, connectivity.py:231-236).  The planes are
w, grad, adam_m and adam_v (float64).  The sign and conn bitfields come from
DeepR.init_bitfields.

One update flips the sign of a Bernoulli(f) subset of the valid weights; the
flip uses uniform01 draw #(i*stride + s) of fold_key(seed, "flip", u).  Then
the DEEP R group "deep_r" runs, eliminate followed by form
(deep_r.py:81-160), on the device and in the oracle.

The device state is injected into the oracle before the update (state
injection).  Row lengths, valid targets, every plane at the valid slots, the
conn words and the dormant counts must then match bit for bit.  The flip
rates are the whole M-update sweep bench.py times (0.1 ... 10 %).
"""

import ctypes

import numpy as np
import pytest
import torch

from oracle_helpers import PLANES, valid_equal

pytestmark = pytest.mark.gpu

P, N, CAP, SEED = 16384, 65536, 1024, 1


def _host_flips(row_length, stride, key, f):
    from oracle.rng import u01_from_u64, u64_block
    u = u01_from_u64(u64_block(key, 0, P * stride)).reshape(P, stride)
    valid = np.arange(stride)[None, :] < row_length[:, None]
    return (u < f) & valid


@pytest.mark.parametrize("f", [0.001, 0.003, 0.01, 0.03, 0.1])
def test_mupdate_instance_bit_exact(dev_lib, f):
    from oracle.deep_r import DeepROracle
    from oracle.ragged import Ragged
    from oracle.rng import Stream, fold_key
    from oracle.updates import OracleModel
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.connectivity import descriptor, init_pairwise_bernoulli_density
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.rng import CounterRng
    from paper_2510_19764_b200.updates import Model

    m, syn = init_pairwise_bernoulli_density(P, N, 512.0 / N, 1.0, CounterRng(SEED, "init", "M"),
                                             var_names=PLANES, capacity=CAP)
    assert m.stride == CAP
    torch.manual_seed(0)
    w = syn.planes["w"]
    w.normal_(0.0, 0.1)
    w.mul_(m.slot_mask())
    dr = DeepR(m, syn, "M", l1_strength=0.0)
    dr.init_bitfields(CounterRng(SEED, "deep_r", "M"))
    model = Model(SEED)
    model.add_matrix("M", m, syn)
    dr.register(model, "deep_r", "M")

    rl = m.row_length.cpu().numpy()
    tg = m.target.cpu().numpy()
    # the rows are the reference's counter draws (sampled rows)
    st = Stream.of(SEED, "init", "M")
    for i in np.random.default_rng(3).choice(P, 24, replace=False):
        s = Stream(st.key, int(i) * N)
        hit = np.flatnonzero(s.uniform01_array(N) < 512.0 / N)
        assert rl[i] == hit.size and np.array_equal(tg[i, :rl[i]], hit), i

    # state injection into the oracle
    mo = Ragged(P, N, CAP, PLANES)
    mo.row_length[:] = rl
    mo.target[:] = tg
    for p in PLANES:
        mo.planes[p][:] = syn.planes[p].cpu().numpy()
    dro = DeepROracle(mo, l1=0.0)
    dro.sign[:] = dr.sign_bits.host_words()
    dro.conn[:] = dr.conn_bits.host_words()
    om = OracleModel(SEED)
    om.add_matrix("M", mo)
    dro.register(om, "deep_r", "M")

    key = fold_key(SEED, "flip", 0)
    d = descriptor(m, syn)
    _lib.call("sw_flip_signs", ctypes.byref(d), 0, key, f, _lib.stream_ptr())
    flips = _host_flips(rl, CAP, key, f)
    mo.planes["w"][flips] *= -1.0
    assert np.array_equal(syn.planes["w"].cpu().numpy(), mo.planes["w"])

    model.run_update_group("deep_r")
    om.run_update_group("deep_r")
    assert dr.last_removed == dro.last_removed > 0
    rlo = mo.row_length
    assert np.array_equal(m.row_length.cpu().numpy(), rlo)
    assert valid_equal(rlo, m.target.cpu().numpy(), mo.target)
    for p in PLANES:
        assert valid_equal(rlo, syn.planes[p].cpu().numpy(), mo.planes[p]), p
    assert np.array_equal(dr.conn_bits.host_words(), dro.conn)
    assert np.array_equal(dr.dormant.cpu().numpy(), dro.dormant)
    assert m.edge_count() == int(rl.sum())
