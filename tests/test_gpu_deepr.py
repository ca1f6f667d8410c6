"""Device DEEP R vs the golden reference runs and vs the oracle (bit-exact)."""

import numpy as np
import pytest
import torch

from conftest import golden
from golden_cases import DEEPR_CASES
from oracle import rng as O
from oracle_helpers import PLANES, oracle_deepr_from_fixture, valid_equal

pytestmark = pytest.mark.gpu


def device_deepr_from_fixture(fx):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.updates import Model
    P, N, cap, diag, cycles, seed = (int(x) for x in fx["meta"])
    m = RaggedMatrix(P, N, cap)
    syn = SynVarMatrix(m, PLANES)
    m.load_state(fx["init_row_length"], fx["init_target"])
    for p in PLANES:
        syn.planes[p].copy_(torch.from_numpy(fx[f"init_{p}"]))
    dr = DeepR(m, syn, "sg", l1_strength=0.005, exclude_diagonal=bool(diag))
    dr.load_state(fx["init_sign"], fx["init_conn"])
    model = Model(seed)
    model.add_matrix("sg", m, syn)
    dr.register(model, "deep_r", "sg")
    return model, m, syn, dr, cycles


def assert_state(m, syn, dr, ref, prefix):
    rl = ref[f"{prefix}row_length"]
    got_rl = m.row_length.cpu().numpy()
    assert np.array_equal(got_rl, rl)
    assert valid_equal(rl, m.target.cpu().numpy(), ref[f"{prefix}target"])
    for p in PLANES:
        assert valid_equal(rl, syn.planes[p].cpu().numpy(), ref[f"{prefix}{p}"]), p
    assert np.array_equal(dr.conn_bits.host_words(), ref[f"{prefix}conn"])
    assert np.array_equal(dr.sign_bits.host_words(), ref[f"{prefix}sign"])
    assert np.array_equal(dr.dormant.cpu().numpy(), ref[f"{prefix}dormant"])
    assert dr.last_removed == int(ref[f"{prefix}last_removed"])


@pytest.mark.parametrize("case", [c[0] for c in DEEPR_CASES])
def test_deep_r_group_matches_reference_golden(dev_lib, case):
    fx = golden(f"deepr_{case}.npz")
    model, m, syn, dr, cycles = device_deepr_from_fixture(fx)
    for c in range(cycles):
        syn.planes["w"].copy_(torch.from_numpy(fx[f"c{c}_w_in"]))
        syn.planes["grad"].copy_(torch.from_numpy(fx[f"c{c}_grad_in"]))
        dr.l1_step()
        rl = fx[f"c{c - 1}_row_length"] if c else fx["init_row_length"]
        assert valid_equal(rl, syn.planes["grad"].cpu().numpy(), fx[f"c{c}_grad_l1"])
        model.run_update_group("deep_r")
        assert_state(m, syn, dr, fx, f"c{c}_")


def test_init_bitfields_matches_golden(dev_lib):
    """Randomized sign bits + edge mirror (deep_r.py:50-64) from the fixture's
    initial weights reproduce the reference's initial bitfields."""
    from paper_2510_19764_b200.rng import CounterRng
    for case in ("small16", "wide64x700", "rec256"):
        fx = golden(f"deepr_{case}.npz")
        model, m, syn, dr, _ = device_deepr_from_fixture(fx)
        seed = int(fx["meta"][5])
        dr.sign_bits.clear_all()
        dr.conn_bits.clear_all()
        dr.init_bitfields(CounterRng(seed, "bits"))
        assert np.array_equal(dr.sign_bits.host_words(), fx["init_sign"])
        assert np.array_equal(dr.conn_bits.host_words(), fx["init_conn"])


def _random_instance(P, N, cap, R, seed):
    """Oracle + device copies of a random DEEP R instance (row lengths ~R)."""
    from oracle.deep_r import DeepROracle
    from oracle.ragged import Ragged, bf_randomize, bf_words
    from oracle.updates import OracleModel
    rs = np.random.default_rng(seed)
    m = Ragged(P, N, cap, PLANES)
    for i in range(P):
        k = int(min(cap, max(0, rs.poisson(R))))
        m.target[i, :k] = rs.choice(N, size=k, replace=False)
        m.row_length[i] = k
    mask = m.slot_mask()
    for p in PLANES:
        m.planes[p][mask] = rs.standard_normal(int(mask.sum()))
    dr = DeepROracle(m, l1=0.0)
    dr.init_bitfields(O.Stream.of(seed, "bits"))
    model = OracleModel(seed)
    model.add_matrix("sg", m)
    dr.register(model, "deep_r", "sg")
    return model, m, dr, rs


@pytest.mark.parametrize("P,N,cap,R,flip", [(512, 2048, 96, 40, 0.01), (300, 700, 50, 20, 0.1),
                                            (1024, 65536, 128, 60, 0.03),
                                            (256, 33, 20, 12, 0.3),
                                            # streaming eliminate: full 256-slot chunks, deep ring
                                            (2048, 8192, 1024, 512, 0.01),
                                            # odd stride: 16-byte TMA windows start mid-row
                                            (700, 300, 41, 25, 0.05)])
def test_deep_r_random_instances_match_oracle(dev_lib, P, N, cap, R, flip):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.updates import Model
    model_o, mo, dro, rs = _random_instance(P, N, cap, R, 7)
    m = RaggedMatrix(P, N, cap)
    syn = SynVarMatrix(m, PLANES)
    dr = DeepR(m, syn, "sg", l1_strength=0.0)
    model = Model(7)
    model.add_matrix("sg", m, syn)
    dr.register(model, "deep_r", "sg")
    m.load_state(mo.row_length, mo.target)
    for p in PLANES:
        syn.planes[p].copy_(torch.from_numpy(mo.planes[p]))
    dr.load_state(dro.sign, dro.conn)
    for cycle in range(3):
        mask = mo.slot_mask()
        flips = (rs.random(mo.target.shape) < flip) & mask
        mo.planes["w"][flips] *= -1.0
        syn.planes["w"].copy_(torch.from_numpy(mo.planes["w"]))
        model_o.run_update_group("deep_r")
        model.run_update_group("deep_r")
        rl = mo.row_length
        assert np.array_equal(m.row_length.cpu().numpy(), rl)
        assert valid_equal(rl, m.target.cpu().numpy(), mo.target)
        for p in PLANES:
            assert valid_equal(rl, syn.planes[p].cpu().numpy(), mo.planes[p])
        assert np.array_equal(dr.conn_bits.host_words(), dro.conn)
        assert np.array_equal(dr.dormant.cpu().numpy(), dro.dormant)
        assert dr.last_removed == dro.last_removed


def test_hard_error_when_nothing_can_be_placed(dev_lib):
    """pkg/tests/test_deep_r.py:256-271: 2x2 full matrix -> RowFull."""
    from paper_2510_19764_b200.connectivity import init_pairwise_bernoulli_density
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.errors import RowFull
    from paper_2510_19764_b200.rng import CounterRng
    from paper_2510_19764_b200.updates import Model
    model = Model(1)
    m, syn = init_pairwise_bernoulli_density(2, 2, 1.0, 1.0, CounterRng(0), var_names=PLANES)
    model.add_matrix("sg", m, syn)
    dr = DeepR(m, syn, "sg")
    dr.init_bitfields(CounterRng(1))
    dr.register(model, "deep_r", "sg")
    dr.dormant[0] = 1
    model.groups["deep_r"] = [model.groups["deep_r"][1]]
    with pytest.raises(RowFull):
        model.run_update_group("deep_r")


def test_remove_marked_matches_golden(dev_lib):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix, remove_marked
    g = golden("remove.npz")
    rows = len(g["n"])
    m = RaggedMatrix(rows, 10_000, 96)
    syn = SynVarMatrix(m, ("w",))
    tgt = np.zeros((rows, 96), dtype=np.int32)
    marked = np.zeros((rows, 96), dtype=np.uint8)
    for r, (n, k, mk) in enumerate(zip(g["n"], g["k"], g["marked"])):
        tgt[r, :n] = np.arange(n)
        marked[r, mk[:k]] = 1
    m.load_state(g["n"].astype(np.int32), tgt)
    syn.planes["w"].copy_(torch.from_numpy(tgt.astype(np.float64) * 0.5))
    removed = torch.zeros(rows, dtype=torch.int64, device="cuda")
    remove_marked(m, syn, torch.from_numpy(marked).cuda(), removed)
    got = m.target.cpu().numpy()
    w = syn.planes["w"].cpu().numpy()
    for r, (n, k, res) in enumerate(zip(g["n"], g["k"], g["result"])):
        assert list(got[r, : n - k]) == list(res[: n - k])
        assert list(w[r, : n - k]) == list(res[: n - k] * 0.5)
    assert np.array_equal(removed.cpu().numpy(), g["k"])


def test_init_bitfields_multapses_clear_wins(dev_lib):
    """with multapses of opposite sign, deep_r.py:62-64 sets every
    w > 0 bit of the row, then clears every w < 0 bit (clear wins), in any
    slot order; w == 0 keeps the random bit."""
    from oracle.deep_r import DeepROracle
    from oracle.ragged import Ragged
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.rng import CounterRng
    P, N, cap = 64, 130, 8
    rs = np.random.default_rng(4)
    tg = rs.integers(0, 8, size=(P, cap)).astype(np.int32) * 16 + rs.integers(0, 2, size=(P, cap)).astype(np.int32)
    rl = rs.integers(0, cap + 1, size=P).astype(np.int32)
    w = rs.choice([-1.0, 0.0, 1.0], size=(P, cap))
    m = RaggedMatrix(P, N, cap, multapse_free=False)
    syn = SynVarMatrix(m, PLANES)
    m.load_state(rl, tg)
    syn.planes["w"].copy_(torch.from_numpy(w))
    dr = DeepR(m, syn, "mx")
    dr.init_bitfields(CounterRng(3, "bits"))
    o = Ragged(P, N, cap, PLANES)
    o.row_length[:] = rl
    o.target[:] = tg
    o.planes["w"][:] = w
    od = DeepROracle(o)
    od.init_bitfields(O.Stream.of(3, "bits"))
    assert np.array_equal(dr.conn_bits.host_words(), od.conn)
    assert np.array_equal(dr.sign_bits.host_words(), od.sign)


def test_version_bumped_only_on_structural_change(dev_lib):
    """a DEEP R group that removes nothing leaves m.version (and so
    derived structures) untouched, as the reference bumps it only inside
    add/remove (connectivity.py:91-136, updates.py:367-372)."""
    fx = golden("deepr_small16.npz")
    model, m, syn, dr, cycles = device_deepr_from_fixture(fx)
    w = syn.planes["w"]
    # no sign mismatches: make every weight agree with its sign bit
    sign = dr.sign_bits.host_words()
    tg = m.target.cpu().numpy()
    bit = (np.take_along_axis(sign, (tg >> 6).astype(np.int64), axis=1) >> (tg & 63).astype(np.uint64)) & np.uint64(1)
    w.copy_(torch.from_numpy(np.where(bit.astype(bool), 1.0, -1.0)))
    dr.l1_strength = 0.0
    v0 = m.version
    model.run_update_group("deep_r")
    assert dr.last_removed == 0 and m.version == v0
    w.copy_(-w)                                  # every synapse now mismatches
    model.run_update_group("deep_r")
    assert dr.last_removed > 0 and m.version > v0
