"""Device topomap path vs reference golden vectors and the oracle:
transpose, ordered propagation, STDP (bit-exact), rewiring (state-injected,
bit-exact), Poisson/LIF free run, graph vs eager equivalence."""

import math

import numpy as np
import pytest
import torch

from conftest import golden
from oracle_helpers import check_topomap_post

pytestmark = pytest.mark.gpu


def _matrix_from(target, row_length, planes):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    P, cap = target.shape
    return P, cap


def test_transpose_and_propagation(dev_lib):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix, propagate_spikes
    from paper_2510_19764_b200.transpose import TransposeMap
    g = golden("transpose_prop.npz")
    m = RaggedMatrix(50, 40, 16)
    syn = SynVarMatrix(m, ("g",))
    m.load_state(g["row_length"], g["target"])
    syn.planes["g"].copy_(torch.from_numpy(g["g"]))
    tm = TransposeMap(m)
    tm.rebuild()
    cl, sp, ss = tm.reference_layout()
    assert np.array_equal(cl, g["col_length"])
    assert np.array_equal(sp, g["source_pre"]) and np.array_equal(ss, g["source_slot"])
    assert tm.max_col_length == int(g["col_length"].max())
    spikes = torch.from_numpy(g["spikes"]).cuda()
    out = torch.zeros(40, dtype=torch.float64, device="cuda")
    propagate_spikes(m, syn.planes["g"], spikes, out, tmap=tm)
    assert np.array_equal(out.cpu().numpy(), g["out"])           # ordered: bit-exact
    out2 = torch.zeros_like(out)
    propagate_spikes(m, syn.planes["g"], spikes, out2)             # event-driven atomics
    assert np.allclose(out2.cpu().numpy(), g["out"], rtol=1e-13, atol=0)


def test_stdp_bit_exact(dev_lib):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    from paper_2510_19764_b200.plasticity import StdpParams, StdpSynapses
    from paper_2510_19764_b200.transpose import TransposeMap
    g = golden("stdp.npz")
    m = RaggedMatrix(40, 30, 12)
    syn = SynVarMatrix(m, ("g",))
    m.load_state(g["row_length"], g["target"])
    syn.planes["g"].copy_(torch.from_numpy(g["g0"]))
    tm = TransposeMap(m)
    tm.rebuild()
    st = StdpSynapses(m, syn, 0.1, StdpParams())
    for t in range(40):
        pre = torch.from_numpy(np.flatnonzero(g[f"pre{t}"])).cuda()
        post = torch.from_numpy(np.flatnonzero(g[f"post{t}"])).cuda()
        st.decay_step()
        st.on_pre_spikes(pre)
        st.on_post_spikes(tm, post)
    mask = np.arange(12)[None, :] < g["row_length"][:, None]
    assert np.array_equal(syn.planes["g"].cpu().numpy()[mask], g["g"][mask])
    assert np.array_equal(st.x.cpu().numpy(), g["x"]) and np.array_equal(st.y.cpu().numpy(), g["y"])


def _device_group(fx, k, record_events=True):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    from paper_2510_19764_b200.geometry import GridGeometry
    from paper_2510_19764_b200.topomap import RewiringParams, RewiringRule
    from paper_2510_19764_b200.updates import Model
    scale, seed = (int(x) for x in fx["meta"])
    side = 16 * scale
    N = side * side
    geom = GridGeometry(side)
    model = Model(seed)
    out = {}
    for name, prm in (("ff", RewiringParams.feedforward()), ("lat", RewiringParams.lateral())):
        tg = fx[f"u{k}_pre_{name}_target"]
        m = RaggedMatrix(N, N, tg.shape[1])
        syn = SynVarMatrix(m, ("g",))
        m.load_state(fx[f"u{k}_pre_{name}_row_length"], tg)
        syn.planes["g"].copy_(torch.from_numpy(fx[f"u{k}_pre_{name}_g"]))
        model.add_matrix(name, m, syn)
        rule = RewiringRule(f"{name}_rewire", m, syn, geom, prm, 10 * scale * scale,
                            record_events=record_events, form_lut=fx[f"{name}_lut"],
                            dist_lut=fx["dist"])
        model.add_rule("rewiring", name, rule.descriptor())
        out[name] = (m, syn, rule)
    for b, u in zip(model.groups["rewiring"], fx[f"u{k}_pre_updates"]):
        b.update_count = int(u)
    return model, out


@pytest.mark.parametrize("tag", ["s1", "s2dep"])
def test_rewiring_state_injected_bit_exact(dev_lib, tag):
    fx = golden(f"topomap_{tag}.npz")
    changes = 0
    for k in range(int(fx["n_updates"])):
        model, objs = _device_group(fx, k)
        model.run_update_group("rewiring")
        for name, (m, syn, rule) in objs.items():
            rule.collect(1.0)
            check_topomap_post(fx, k, name, m.row_length.cpu().numpy(), m.target.cpu().numpy(),
                               syn.planes["g"].cpu().numpy())
            assert np.array_equal(rule.attempts.cpu().numpy(), fx[f"u{k}_{name}_attempts"])
            kinds = fx[f"u{k}_{name}_ev_kind"]
            d = fx[f"u{k}_{name}_ev_d"]
            assert [e[1] for e in rule.elim_events] == list(d[kinds == 1])
            assert [e[1] for e in rule.form_events] == list(d[kinds == 2])
            changes += rule.last_stats["removed"] + rule.last_stats["formed"]
            assert rule.last_stats["attempts"] == 10 * int(fx["meta"][0]) ** 2
    assert changes > 0


def test_free_run_spikes_match_reference(dev_lib):
    """300 steps of TopomapModel(1, seed=11): source spikes are counter-exact;
    target spikes match the reference run at every step and V to 1e-6 (F8:
    the conductance LIF uses CUDA exp against numpy's, so V may differ in
    the last bits; a spike could flip only if V landed within that error of
    the threshold at a crossing, which this fixed-seed run does not do --
    the comparison is deterministic, so any flip is a real change)."""
    from paper_2510_19764_b200.neurons import unpack_spike_bits
    from paper_2510_19764_b200.topomap import TopomapModel
    g = golden("topomap_run.npz")
    model = TopomapModel(1, seed=11, record_events=False, use_graph=False)
    T = g["src"].shape[0]
    src_ok = tgt_ok = 0
    for t in range(T):
        model.run(0.1)
        src = unpack_spike_bits(model.source.spike_bits, 256).cpu().numpy()
        tgt = unpack_spike_bits(model.target.spike_bits, 256).cpu().numpy()
        src_ok += np.array_equal(src, np.flatnonzero(g["src"][t]))
        tgt_ok += np.array_equal(tgt, np.flatnonzero(g["tgt"][t]))
    assert src_ok == T
    assert tgt_ok == T
    st = model.state_arrays()
    assert np.allclose(st["V"], g["state_V"], rtol=0, atol=1e-6)
    for key in ("ff.row_length", "lat.row_length"):
        assert np.array_equal(st[key], g["state_" + key.replace(".", "_")])


def test_graph_replay_equals_eager(dev_lib):
    from paper_2510_19764_b200.topomap import TopomapModel
    a = TopomapModel(1, seed=74, record_events=False, use_graph=True)
    b = TopomapModel(1, seed=74, record_events=False, use_graph=False)
    ra = a.run(40.0)
    rb = b.run(40.0)
    assert ra.steps == rb.steps == 400 and ra.rewiring_executions == rb.rewiring_executions == 40
    assert ra.rewires_per_update == rb.rewires_per_update
    sa, sb = a.state_arrays(), b.state_arrays()
    for key in sa:
        assert np.array_equal(sa[key], sb[key]), key


def test_schedule_attempts_and_new_synapses(dev_lib):
    """pkg/tests/test_topomap.py:191-195, 226-241, 257-267."""
    from paper_2510_19764_b200.topomap import TopomapModel
    model = TopomapModel(2, seed=91)
    model.net.run_update_group("rewiring")
    assert int(model.ff_rule.attempts.sum()) == 40 and int(model.lat_rule.attempts.sum()) == 40
    model = TopomapModel(1, seed=72, record_events=False)
    r = model.run(20.0)
    assert (r.steps, r.rewiring_executions, r.stimulus_changes) == (200, 20, 1)
    r2 = model.run(20.0)
    assert r2.stimulus_changes == 1
    model = TopomapModel(1, seed=61)
    m, syn = model.net.matrices["ff"]
    before = set(zip(*[x.tolist() for x in m.edge_list()]))
    for _ in range(200):
        model.net.run_update_group("rewiring")
    pre, post = m.edge_list()
    w = syn.planes["g"][m.slot_mask()].cpu().numpy()
    new = [(k, e) for k, e in enumerate(zip(pre.tolist(), post.tolist())) if e not in before]
    assert new and all(w[k] == 0.2 for k, _ in new)


def test_one_step_transmission_delay(dev_lib):
    """pkg/tests/test_topomap.py:269-285 with a forced single source spike."""
    from paper_2510_19764_b200.topomap import TopomapModel
    model = TopomapModel(1, seed=73, record_events=False, use_graph=False)
    m, syn = model.net.matrices["ff"]
    p = model.source.probabilities(0.1)
    model.source._p = np.zeros(256)
    model.source._p[5] = 1.0
    p.copy_(torch.from_numpy(model.source._p))
    model.source._p_h = 0.1
    model._launch_step()
    model.step_index += 1
    assert float(model.target.g.abs().max()) == 0.0
    p.zero_()
    model.source._p[:] = 0.0
    model._launch_step()
    decay = math.exp(-0.1 / 5.0)
    tg = m.row_targets(5).long()
    assert np.allclose(model.target.g[tg].cpu().numpy(), 0.2 * decay)


def test_post_sharded_steps_equal_unsharded(dev_lib):
    """Postsynaptic sharding on one device: two half-sheet
    'ranks' stepped in lock-step with the target-spike words exchanged by
    hand (the NCCL all-gather of the multi-GPU run) reproduce the unsharded
    model: connectivity, weights and traces everywhere, V on the owned posts."""
    from paper_2510_19764_b200.sharding import SpikeGather
    from paper_2510_19764_b200.topomap import TopomapModel
    from paper_2510_19764_b200.neurons import PoissonParams
    kw = dict(record_events=False, use_graph=False)
    ref = TopomapModel(2, seed=33, **kw)
    shards = [TopomapModel(2, seed=33, **kw) for _ in range(2)]
    n = ref.geometry.n
    for r, m in enumerate(shards):
        sg = SpikeGather(n, r, 2, "cuda")
        m.shard, m.post_lo, m.post_hi = sg, sg.lo, sg.hi
        m.target.spike_bits = sg.bits
    h = ref.h
    stim_steps = int(round(PoissonParams().t_stim / h))
    for k in range(600):
        for m in [ref] + shards:
            if k % stim_steps == 0:
                m.source.set_correlated_rates(m._draw_centers())
                m.source.probabilities(h)
        ref._launch_step()
        for m in shards:
            m.launch_neurons()
        a, b = shards
        a.shard.bits[b.shard.own_words] = b.shard.bits[b.shard.own_words]
        b.shard.bits[a.shard.own_words] = a.shard.bits[a.shard.own_words]
        for m in shards:
            m.launch_synapses()
        if (k + 1) % 10 == 0:
            for m in [ref] + shards:
                m.net.run_update_group("rewiring")
    sr = ref.state_arrays()
    assert int(ref.spike_counts[1]) > 0
    for m in shards:
        st = m.state_arrays()
        for key in sr:
            if key in ("V", "g_total", "refractory", "pending"):
                lo, hi = m.post_lo, m.post_hi
                assert np.array_equal(st[key][lo:hi], sr[key][lo:hi]), key
            else:
                assert np.array_equal(st[key], sr[key]), key
        assert torch.equal(m.spike_counts, ref.spike_counts)


@pytest.mark.parametrize("scale", [4, 8])
def test_persistent_multi_cta_steps_equal_per_step_launches(dev_lib, scale, monkeypatch):
    """sw_topomap_run_steps (one cooperative launch per rewiring period, grid
    barriers between phases; several CTAs at these sizes) == one launch per
    phase and step."""
    from paper_2510_19764_b200 import topomap
    from paper_2510_19764_b200.topomap import TopomapModel
    monkeypatch.setattr(topomap, "PERSISTENT_MAX_NODES", 1 << 30)
    a = TopomapModel(scale, seed=5, record_events=False, use_graph=True)
    b = TopomapModel(scale, seed=5, record_events=False, use_graph=False)
    ra, rb = a.run(20.0), b.run(20.0)
    assert ra.rewires_per_update == rb.rewires_per_update
    assert torch.equal(a.spike_counts, b.spike_counts) and int(a.spike_counts[0]) > 0
    sa, sb = a.state_arrays(), b.state_arrays()
    for key in sa:
        assert np.array_equal(sa[key], sb[key]), key


def test_snapshot_csv_matches_reference_bytes(dev_lib):
    """connectivity.py:265-283 write_snapshot_csv: byte-identical to the
    reference's output for the same matrix (tests/golden/make_snapshot_csv.py)."""
    import io
    import os
    from conftest import GOLDEN
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix, write_snapshot_csv
    g = golden("transpose_prop.npz")
    m = RaggedMatrix(50, 40, 16)
    syn = SynVarMatrix(m, ("g",))
    m.load_state(g["row_length"], g["target"])
    syn.planes["g"].copy_(torch.from_numpy(g["g"]))
    buf = io.StringIO()
    write_snapshot_csv(buf, m, syn)
    assert buf.getvalue() == open(os.path.join(GOLDEN, "snapshot_transpose_prop.csv")).read()


def test_phase_timer_csv_schema(dev_lib):
    """updates.py:50-54 timing.csv schema: phase,seconds rows for the six
    phases, then total."""
    import io
    from paper_2510_19764_b200.topomap import TopomapModel
    from paper_2510_19764_b200.updates import PHASES
    model = TopomapModel(1, seed=3, record_events=False, use_graph=False)
    model.run(2.0)
    buf = io.StringIO()
    model.net.timers.write_csv(buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "phase,seconds"
    assert [ln.split(",")[0] for ln in lines[1:]] == list(PHASES) + ["total"]
    vals = [float(ln.split(",")[1]) for ln in lines[1:]]
    assert abs(sum(vals[:-1]) - vals[-1]) < 1e-6 and vals[PHASES.index("row_update")] > 0


def test_rows_with_more_than_64_attempts_are_exact(dev_lib):
    """rows with 64 < k <= N attempts (both sample_k_distinct
    branches, k == N included) go through the serial bitmap path and match
    the oracle bit for bit, together with ordinary rows in the same update
    (ref topomap.py:142-196, bitfield.py:67-77)."""
    from oracle_helpers import oracle_topomap_group
    fx = golden("topomap_s1.npz")
    model, objs = _device_group(fx, 0)
    om, orules = oracle_topomap_group(fx, 0)
    N = 256
    att = np.zeros(N, dtype=np.int64)
    att[[3, 7, 9, 11, 12, 200]] = [100, 200, 65, 5, 256, 64]
    for name, (m, syn, rule) in objs.items():
        rule.force_attempts(att)
        o, r = orules[name]

        def host(ctx, r=r):
            r.attempts[:] = att
            r.events = []
            r.stats = dict(removed=0, kept=0, formed=0, form_missed=0, form_full=0)
        r.host_phase = host
    model.run_update_group("rewiring")
    om.run_update_group("rewiring")
    for name, (m, syn, rule) in objs.items():
        rule.collect(1.0)
        o, r = orules[name]
        rl = o.row_length
        assert np.array_equal(m.row_length.cpu().numpy(), rl), name
        mask = np.arange(o.target.shape[1])[None, :] < rl[:, None]
        assert np.array_equal(m.target.cpu().numpy()[mask], o.target[mask]), name
        assert np.array_equal(syn.planes["g"].cpu().numpy()[mask], o.planes["g"][mask]), name
        st = rule.last_stats
        assert (st["removed"], st["kept"], st["formed"], st["form_missed"], st["form_full"]) == (
            r.stats["removed"], r.stats["kept"], r.stats["formed"], r.stats["form_missed"],
            r.stats["form_full"]), name
        assert st["attempts"] == int(att.sum())
        assert [d for _, d in rule.elim_events] == [d for _, k, d in r.events if k == 1]
        assert [d for _, d in rule.form_events] == [d for _, k, d in r.events if k == 2]


def test_incremental_transpose_patch_equals_rebuild(dev_lib):
    """sw_transpose_patch (the rewiring update's changed rows re-merged into
    the columns they touch) leaves every column exactly as a full rebuild
    (connectivity.py:173-192 order) after every update of a 1 s run; the
    whole model state is bit-identical to a run with full rebuilds."""
    from paper_2510_19764_b200.topomap import TopomapModel
    from paper_2510_19764_b200.transpose import TransposeMap
    inc = TopomapModel(1, seed=8, use_graph=False, record_events=False)
    full = TopomapModel(1, seed=8, use_graph=False, record_events=False, incremental_remap=False)
    checked = [0, 0]
    orig = inc.net.run_update_group

    def wrapped(group):
        orig(group)
        checked[0] += 1
        if checked[0] % 5:
            return
        for name, tm in (("ff", inc.ff_tmap), ("lat", inc.lat_tmap)):
            ref = TransposeMap(inc.net.matrices[name][0])
            ref.rebuild()
            a, b = tm.host_csr(), ref.host_csr()
            for x, y in zip(a, b):
                assert np.array_equal(x, y), (name, checked[0])
        checked[1] += 1
    inc.net.run_update_group = wrapped
    inc.run(1000.0)
    full.run(1000.0)
    assert checked[1] >= 150
    assert inc.ff_tmap.patches > 0
    si, sf = inc.state_arrays(), full.state_arrays()
    for k in si:
        assert np.array_equal(si[k], sf[k]), k
    # the run rewired: some updates changed the structure
    assert sum(int(x) for x in inc._update_log[:, :].sum(dim=1).cpu().numpy()) > 0


def test_incremental_transpose_patch_in_graph(dev_lib):
    """The patch path inside the captured rewiring-period graph gives the
    same state as eager full rebuilds."""
    from paper_2510_19764_b200.topomap import TopomapModel
    g = TopomapModel(2, seed=9, use_graph=True, record_events=False)
    e = TopomapModel(2, seed=9, use_graph=False, record_events=False, incremental_remap=False)
    g.run(300.0)
    e.run(300.0)
    sg, se = g.state_arrays(), e.state_arrays()
    for k in sg:
        assert np.array_equal(sg[k], se[k]), k


def test_fused_period_equals_per_step_launches(dev_lib, monkeypatch):
    """s = 4 (4096 nodes, above the single-CTA path): the fused period
    (sw_topomap_steps_fused: STDP post of step t with the neuron phase of
    step t+1, alternating target-spike buffers) leaves exactly the state of
    one sw_topomap_step per step, rewiring included."""
    import paper_2510_19764_b200.topomap as tmod
    from paper_2510_19764_b200.neurons import unpack_spike_bits
    res = []
    for fused in (True, False):
        monkeypatch.setattr(tmod, "FUSED_STEPS", fused)
        m = tmod.TopomapModel(4, seed=5, record_events=False, use_graph=True)
        m.run(30.0)
        st = m.state_arrays()
        st["tgt"] = unpack_spike_bits(m.target.spike_bits, m.geometry.n).cpu().numpy()
        res.append(st)
    a, b = res
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
