"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py) and the reference's own known answers."""

import numpy as np
import pytest

from conftest import golden
from oracle import rng as O
from oracle.deep_r import AdamOracle
from oracle.ragged import Ragged, removal_permutation
from oracle_helpers import PLANES, oracle_deepr_from_fixture, valid_equal

from golden_cases import DEEPR_CASES


def test_mix64_known_answers():
    # pkg/tests/test_rng.py:118-123
    assert O.mix64(0) == 0
    assert O.mix64(1) == 6238072747940578789
    assert O.mix64(0x9E3779B97F4A7C15) == 16294208416658607535


def test_rng_golden():
    g = golden("rng.npz")
    parts = [(0,), (1,), (1, "host", 3, 7, 0), (42, "row", 0, 0, 1),
             ("task", "example", 5), (2**64 - 1, -1, "päß-unicode-longer-than-8"),
             (7, "init", "ff")]
    assert [O.fold_key(*p) for p in parts] == [int(x) for x in g["fold"]]
    assert [O.mix64(int(x)) for x in g["mix_in"]] == [int(x) for x in g["mix_out"]]
    key = O.fold_key(9, "golden")
    assert key == int(g["key"])
    assert np.array_equal(O.Stream(key).u64_array(4096), g["draws"])
    assert np.array_equal(O.Stream(key).uniform01_array(4096), g["u01"])
    for n, row in zip(g["ns"], g["ui"]):
        s = O.Stream.of(9, "uint", int(n))
        vals = [s.uniform_int(int(n)) for _ in range(512)]
        assert vals == [int(x) for x in row[:512]]
        assert s.counter == int(row[512])
    assert [O.child_key(key, i) for i in range(300)] == [int(x) for x in g["child"]]
    assert np.array_equal(O.child_keys_np(key, np.arange(300)), g["child"])
    for (k, n), ref in zip(g["skd_cases"], g["skd"]):
        s = O.Stream.of(9, "skd", int(k), int(n))
        out = s.sample_k_distinct(int(k), int(n))
        ref = ref[ref >= 0]
        assert list(out) == list(ref[:-1])
        assert s.counter == ref[-1]


def test_remove_slots_golden_and_closed_form():
    g = golden("remove.npz")
    for n, k, marked, result in zip(g["n"], g["k"], g["marked"], g["result"]):
        n, k = int(n), int(k)
        mk = marked[:k]
        # serial replay
        m = Ragged(1, 10_000, 96, ("w",))
        m.target[0, :n] = np.arange(n)
        m.row_length[0] = n
        m.remove_slots(0, mk)
        assert list(m.target[0, : n - k]) == list(result[: n - k])
        # closed form used by the CUDA kernel
        row = list(range(n))
        for dst, src in removal_permutation(n, mk):
            row[dst] = src
        assert row[: n - k] == list(result[: n - k])


@pytest.mark.parametrize("case", [c[0] for c in DEEPR_CASES])
def test_deep_r_group_golden(case):
    fx = golden(f"deepr_{case}.npz")
    model, m, dr, cycles = oracle_deepr_from_fixture(fx)
    for c in range(cycles):
        m.planes["w"][:] = fx[f"c{c}_w_in"]
        m.planes["grad"][:] = fx[f"c{c}_grad_in"]
        dr.l1_step()
        assert np.array_equal(m.planes["grad"], fx[f"c{c}_grad_l1"])
        model.run_update_group("deep_r")
        rl = fx[f"c{c}_row_length"]
        assert np.array_equal(m.row_length, rl)
        assert valid_equal(rl, m.target, fx[f"c{c}_target"])
        for p in PLANES:
            assert valid_equal(rl, m.planes[p], fx[f"c{c}_{p}"]), p
        assert np.array_equal(dr.conn, fx[f"c{c}_conn"])
        assert np.array_equal(dr.sign, fx[f"c{c}_sign"])
        assert np.array_equal(dr.dormant, fx[f"c{c}_dormant"])
        assert dr.last_removed == int(fx[f"c{c}_last_removed"])


def test_adam_golden():
    g = golden("adam.npz")
    p = g["p0"].copy()
    a = AdamOracle(shape=p.shape)
    for t in range(5):
        gr = g[f"g{t}"].copy()
        a.apply(p, gr)
        assert np.array_equal(p, g[f"p{t + 1}"])
        assert np.array_equal(a.m, g[f"m{t + 1}"])
        assert np.array_equal(a.v, g[f"v{t + 1}"])
        assert not gr.any()


def test_alif_and_eprop_golden():
    from oracle.classifier import AlifP, alif_step, alif_surrogate, eprop_accumulate
    g = golden("alif_eprop.npz")
    B, H = 8, 48
    v = np.zeros((B, H), np.float32)
    a = np.zeros_like(v)
    z = np.zeros_like(v)
    for t in range(6):
        assert np.array_equal(alif_surrogate(v, a), g[f"psi{t}"])
        v, a, z = alif_step(v, a, z, g[f"rec{t}"], g[f"ext{t}"])
        assert np.array_equal(v, g[f"v{t}"]) and np.array_equal(a, g[f"a{t}"])
        assert np.array_equal(z, g[f"z{t}"])
    p = AlifP()
    tg, rl = g["target"], g["row_length"]
    eps = np.zeros((B,) + tg.shape, np.float32)
    ebar = np.zeros_like(eps)
    grad = np.zeros(tg.shape)
    for t in range(25):
        eprop_accumulate(tg, rl, g[f"trace{t}"], g[f"psi_e{t}"], g[f"lsig{t}"], eps, ebar, grad,
                         np.float32(p.beta), np.float32(p.rho), np.float32(p.alpha))
    assert np.array_equal(eps, g["eps"]) and np.array_equal(ebar, g["ebar"])
    assert np.array_equal(grad, g["grad"])


def test_trainer_oracle_matches_reference_run():
    """The oracle trainer reproduces a 3-batch reference training run
    bit-for-bit on this host (same numpy/OpenBLAS)."""
    from oracle.classifier import TaskOracle, TrainerOracle
    g = golden("trainer.npz")
    task = TaskOracle(num_classes=3, num_inputs=20, example_steps=60, seed=4)
    tr = TrainerOracle(task, hidden=24, batch_size=8, seed=4, input_density=0.3,
                       recurrent_density=0.2)
    for b in range(3):
        loss, acc = tr.gradient_phase(b)
        removed = tr.rewire_phase()
        assert abs(loss - float(g[f"b{b}_loss"])) <= 1e-12 * abs(loss)
        assert acc == float(g[f"b{b}_acc"])
        assert removed == int(g[f"b{b}_removed"])
    for name, m in (("in", tr.m_in), ("rec", tr.m_rec)):
        rl = g[f"{name}_row_length"]
        assert np.array_equal(m.row_length, rl)
        assert valid_equal(rl, m.target, g[f"{name}_target"])
        assert np.allclose(m.planes["w"], g[f"{name}_w"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("tag", ["s1", "s2dep"])
def test_topomap_rewiring_oracle_golden(tag):
    from oracle_helpers import check_topomap_post, oracle_topomap_group
    fx = golden(f"topomap_{tag}.npz")
    n_upd = int(fx["n_updates"])
    total_changes = 0
    for k in range(n_upd):
        model, rules = oracle_topomap_group(fx, k)
        model.run_update_group("rewiring")
        for name, (m, r) in rules.items():
            check_topomap_post(fx, k, name, m.row_length, m.target, m.planes["g"])
            assert np.array_equal(r.attempts, fx[f"u{k}_{name}_attempts"])
            kinds = np.array([e[1] for e in r.events], dtype=np.int8)
            dists = np.array([e[2] for e in r.events])
            assert np.array_equal(kinds, fx[f"u{k}_{name}_ev_kind"])
            assert np.array_equal(dists, fx[f"u{k}_{name}_ev_d"])
            total_changes += r.stats["removed"] + r.stats["formed"]
    assert total_changes > 0


def test_stdp_oracle_golden():
    from oracle.ragged import transpose
    from oracle.topomap import StdpOracle
    g = golden("stdp.npz")
    m = Ragged(40, 30, 12, ("g",))
    m.target[:] = g["target"]
    m.row_length[:] = g["row_length"]
    m.planes["g"][:] = g["g0"]
    st = StdpOracle(m, 0.1)
    tr = transpose(m)
    for t in range(40):
        pre = np.flatnonzero(g[f"pre{t}"])
        post = np.flatnonzero(g[f"post{t}"])
        st.decay()
        if pre.size:
            st.on_pre(pre)
        if post.size:
            st.on_post(tr, post)
    assert np.array_equal(m.planes["g"], g["g"])
    assert np.array_equal(st.x, g["x"]) and np.array_equal(st.y, g["y"])


def test_transpose_and_propagation_oracle_golden():
    from oracle.ragged import propagate_spikes, transpose
    g = golden("transpose_prop.npz")
    m = Ragged(50, 40, 16, ("g",))
    m.target[:] = g["target"]
    m.row_length[:] = g["row_length"]
    m.planes["g"][:] = g["g"]
    cl, sp, ss = transpose(m)
    assert np.array_equal(cl, g["col_length"])
    assert np.array_equal(sp, g["source_pre"]) and np.array_equal(ss, g["source_slot"])
    out = np.zeros(40)
    propagate_spikes(m, m.planes["g"], g["spikes"], out)
    assert np.array_equal(out, g["out"])


def test_topomap_poisson_oracle_golden():
    """Source spikes of a reference free run: counter-exact Poisson draws
    with host-numpy probabilities (neurons.py:175-195)."""
    from oracle.rng import Stream
    from oracle.topomap import poisson_step
    g = golden("topomap_run.npz")
    side = 16
    gx = np.arange(side * side) % side
    gy = np.arange(side * side) // side
    stim = Stream.of(11, "stimulus")

    def wrap(d):
        d = np.abs(d)
        return np.minimum(d, side - d)
    ps = Stream.of(11, "poisson")
    for t in range(g["src"].shape[0]):
        if t % 200 == 0:   # stimulus change every t_stim = 20 ms (topomap.py:422-424)
            bx, by = stim.uniform01() * 16, stim.uniform01() * 16
            d = np.hypot(wrap(gx - bx), wrap(gy - by))
            rates = 5.0 + 152.8 * np.exp(-(d * d) / (2.0 * 2.0 ** 2))
            p = 1.0 - np.exp(-rates * 0.1 * 1e-3)
        got = poisson_step(ps, p)
        assert np.array_equal(got, np.flatnonzero(g["src"][t])), t


def test_c_oracle_eprop_matches_golden_and_numpy():
    from oracle.cbuild import eprop_accumulate_c
    from oracle.classifier import AlifP
    g = golden("alif_eprop.npz")
    p = AlifP()
    tg, rl = g["target"], g["row_length"]
    eps = np.zeros((8,) + tg.shape, np.float32)
    ebar = np.zeros_like(eps)
    grad = np.zeros(tg.shape)
    for t in range(25):
        eprop_accumulate_c(tg, rl, g[f"trace{t}"], g[f"psi_e{t}"], g[f"lsig{t}"], eps, ebar, grad,
                           np.float32(p.beta), np.float32(p.rho), np.float32(p.alpha))
    assert np.array_equal(eps, g["eps"]) and np.array_equal(ebar, g["ebar"])
    assert np.array_equal(grad, g["grad"])


@pytest.mark.parametrize("tag", ["topomap_s1.npz", "topomap_s2dep.npz"])
def test_offset_luts_match_reference_luts(tag):
    """oracle.topomap.offset_luts (used by the s = 4..16 rewiring parity
    tests) reproduces the LUTs the real reference produced (F10b)."""
    from oracle.topomap import offset_luts
    g = golden(tag)
    side = 16 * int(g["meta"][0])
    ff, d = offset_luts(side, 0.16, 2.5)
    lat, d2 = offset_luts(side, 1.0, 1.0)
    assert np.array_equal(d, g["dist"]) and np.array_equal(d2, g["dist"])
    assert np.array_equal(ff, g["ff_lut"]) and np.array_equal(lat, g["lat_lut"])
