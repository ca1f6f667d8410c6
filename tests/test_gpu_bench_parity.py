"""Parity at the exact configurations bench.py times (VERDICT r1 "next" 1).

Classifier C1 (700 -> 256, 10 %) and C2 (700 -> 1024, 1 %) at batch 512, the
bench's seed, over 2 blocked e-prop groups (2 x K timesteps):

* forward, teacher-forced: every timestep is launched singly from the
  device's own previous state, and the oracle recomputes it from that state.
  Input spikes, traces, surrogate, v/a/z are compared bit-exactly (the
  currents are the ascending-pre float32 sums the device pins, F7); the
  float64 readout y, the learning signal and the loss to float tolerance.
* the bench path itself (graph replay, two streams, grouped forward, K-step
  blocked e-prop) must reproduce those per-step slots bit for bit;
* e-prop: the device's per-step inputs are fed to the C restatement of
  ref `_kernels.py:15-39`: eps/ebar bit-exact, the float64 gradient within
  1e-13 relative (the K per-step chains are added at the end of a block);
* update: state-injected 1/B scale + L1 + Adam (ref classifier.py:242-253,
  plasticity.py:218-227): bit-exact;
* DEEP R: state-injected eliminate + form group (ref deep_r.py:81-160):
  bit-exact row lengths, targets, all planes, conn bits.

The oracle is test infrastructure (oracle/); nothing here is timed.
"""

import numpy as np
import pytest

from oracle_helpers import grouped_currents
import torch

from oracle_helpers import valid_equal

pytestmark = pytest.mark.gpu

F = np.float32
CONFIGS = {"c1": (256, 0.10), "c2": (1024, 0.01)}


def _seq_currents(rl, tg, w32, spk, H):
    """Per post, the float32 sum over spiking rows in ascending pre order
    (starting from 0) -- the order k_clf_step pins."""
    B = spk.shape[0]
    acc = np.zeros((B, H), F)
    for i in range(rl.size):
        n = int(rl[i])
        if n == 0:
            continue
        rows = np.flatnonzero(spk[:, i])
        if rows.size == 0:
            continue
        idx = np.ix_(rows, tg[i, :n])
        acc[idx] = acc[idx] + w32[i, :n][None, :]
    return acc


def _inject_deepr(tr, b):
    """Oracle DEEP R group loaded with the device's post-Adam state."""
    from oracle.deep_r import DeepROracle
    from oracle.ragged import Ragged
    from oracle.updates import OracleModel
    om = OracleModel(tr.seed)
    objs = []
    for name, m, s, d in (("in", tr.m_in, tr.s_in, tr.deep_r_in),
                          ("rec", tr.m_rec, tr.s_rec, tr.deep_r_rec)):
        o = Ragged(m.num_pre, m.num_post, m.max_row_length, ("w", "grad", "adam_m", "adam_v"))
        o.row_length[:] = m.row_length.cpu().numpy()
        o.target[:] = m.target.cpu().numpy()
        for p in o.planes:
            o.planes[p][:] = s.planes[p].cpu().numpy()
        od = DeepROracle(o, l1=0.005, exclude_diagonal=(name == "rec"))
        od.sign[:] = d.sign_bits.host_words()
        od.conn[:] = d.conn_bits.host_words()
        om.add_matrix(name, o)
        od.register(om, "deep_r", name)
        objs.append((o, od, m, s, d))
    for bnd in om.groups["deep_r"]:
        bnd.update_count = b
    return om, objs


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
def test_trainer_at_bench_config_matches_oracle(dev_lib, cfg):
    import ctypes
    from oracle.cbuild import eprop_accumulate_c
    from oracle.classifier import TaskOracle, TrainerOracle, alif_step, alif_surrogate
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import (EPROP_BLOCK_STEPS, EpropClassifierTrainer,
                                                  SyntheticTask)
    hidden, dens = CONFIGS[cfg]
    NI, C, B, T, seed = 700, 20, 512, 2 * EPROP_BLOCK_STEPS, 1
    task = SyntheticTask(num_classes=C, num_inputs=NI, example_steps=T, seed=seed,
                         num_train=8156, num_test=2264)
    tr = EpropClassifierTrainer(task, hidden=hidden, input_density=dens, recurrent_density=dens,
                                deep_r=True, batch_size=B, seed=seed)
    otask = TaskOracle(num_classes=C, num_inputs=NI, example_steps=T, seed=seed, num_train=8156,
                       num_test=2264)
    ot = TrainerOracle(otask, hidden=hidden, input_density=dens, recurrent_density=dens,
                       batch_size=B, seed=seed)
    # -- construction: bit-exact
    for dm, ds, om, dr, odr in ((tr.m_in, tr.s_in, ot.m_in, tr.deep_r_in, ot.dr_in),
                                (tr.m_rec, tr.s_rec, ot.m_rec, tr.deep_r_rec, ot.dr_rec)):
        assert np.array_equal(dm.row_length.cpu().numpy(), om.row_length)
        assert np.array_equal(dm.target.cpu().numpy(), om.target)
        assert np.array_equal(ds.planes["w"].cpu().numpy(), om.planes["w"])
        assert np.array_equal(dr.sign_bits.host_words(), odr.sign)
        assert np.array_equal(dr.conn_bits.host_words(), odr.conn)
    assert np.array_equal(tr.w_out.cpu().numpy(), ot.w_out)

    # -- forward, teacher-forced, one single-step launch per timestep
    ids = task.train_ids(0, B)
    tr._upload_batch(ids)
    tr._prepare(False)
    spikes = np.stack([otask.example_spikes(e) for e in ids])          # [B, T, NI] bool
    labels = np.array([otask.label(e) for e in ids])
    one_hot = np.eye(C)[labels]
    w32_in, w32_rec = tr.w32_in.cpu().numpy(), tr.w32_rec.cpu().numpy()
    assert np.array_equal(w32_in, tr.s_in.planes["w"].cpu().numpy().astype(F))
    rl_in, tg_in = tr.m_in.row_length.cpu().numpy(), tr.m_in.target.cpu().numpy()
    rl_rec, tg_rec = tr.m_rec.row_length.cpu().numpy(), tr.m_rec.target.cpu().numpy()
    w_out, b_out = ot.w_out, ot.b_out
    al = F(tr.params.alpha)
    st = _lib.stream_ptr()
    prev = {k: getattr(tr, k).cpu().numpy() for k in ("v", "a", "z", "y")}
    xbar_p = np.zeros((B, NI), F)
    zbar_p = np.zeros((B, hidden), F)
    loss_o = 0.0
    snaps = []
    spike_counts = [0, 0]
    for t in range(T):
        _lib.call("sw_clf_step", ctypes.byref(tr._step_params(t)), st)
        torch.cuda.synchronize()
        sl = {k: v.cpu().numpy() for k, v in tr._slot(t).items()}
        snaps.append(sl)
        cur = {k: getattr(tr, k).cpu().numpy() for k in ("v", "a", "z", "y")}
        x = spikes[:, t, :].astype(F)
        xbar_o = xbar_p * al + x
        zbar_o = zbar_p * al + prev["z"]
        assert np.array_equal(sl["xbar"], xbar_o), t
        assert np.array_equal(sl["zbar"], zbar_o), t
        assert np.array_equal(sl["psi"], alif_surrogate(prev["v"], prev["a"])), t
        ext = grouped_currents(rl_in, tg_in, w32_in, spikes[:, t, :], hidden)
        rec = grouped_currents(rl_rec, tg_rec, w32_rec, prev["z"] != 0, hidden)
        v_o, a_o, z_o = alif_step(prev["v"], prev["a"], prev["z"], rec, ext)
        assert np.array_equal(cur["v"], v_o), t
        assert np.array_equal(cur["a"], a_o), t
        assert np.array_equal(cur["z"], z_o), t
        spike_counts[0] += int(x.sum())
        spike_counts[1] += int(z_o.sum())
        # float64 readout: BLAS order on the oracle side (F7) -> tolerance
        y_o = tr.params.alpha * prev["y"] + prev["z"].astype(np.float64) @ w_out.T + b_out
        assert np.allclose(cur["y"], y_o, rtol=1e-12, atol=1e-12), t
        e = np.exp(cur["y"] - cur["y"].max(axis=-1, keepdims=True))
        pi = e / e.sum(axis=-1, keepdims=True)
        d_o = pi - one_hot
        assert np.allclose(sl["d"], d_o, rtol=1e-12, atol=1e-13), t
        assert np.allclose(sl["lsig"], (sl["d"] @ w_out).astype(F), rtol=1e-5, atol=1e-6), t
        loss_o += float(-np.log(np.sum(pi * one_hot, axis=-1)).sum())
        prev, xbar_p, zbar_p = cur, sl["xbar"], sl["zbar"]
    assert spike_counts[0] > 0 and spike_counts[1] > 0, spike_counts
    loss_d = float(tr.loss_b.sum())
    assert abs(loss_d - loss_o) <= 1e-10 * abs(loss_o)

    # -- the bench path (graph, two streams, grouped forward + blocked e-prop)
    tr._forward_batch(ids, learn=True)
    torch.cuda.synchronize()
    assert tr.use_graph and tr._graph is not None
    for t in range(T):
        sl = {k: v.cpu().numpy() for k, v in tr._slot(t).items()}
        for k in sl:
            if k not in ("lsig", "xbar"):   # grouped path: sw_eprop_prep / sw_clf_inputs (below)
                assert np.array_equal(sl[k], snaps[t][k]), (t, k)
        # the precomputed input traces (sw_clf_inputs), replica-minor
        assert np.array_equal(tr.xbar_all[t, :, :B].cpu().numpy().T, snaps[t]["xbar"]), t
    # the last group's replica-minor e-prop inputs (sw_eprop_prep) == the
    # single-step forward's own slots, learning signal included
    K = EPROP_BLOCK_STEPS
    for j in range(K):
        s = snaps[T - K + j]
        assert np.array_equal(tr.lsig_t[j, :, :B].cpu().numpy().T, s["lsig"]), j
        assert np.array_equal(tr.psi_t[j, :, :B].cpu().numpy().T, s["psi"]), j
        assert np.array_equal(tr.zbar_t[j, :, :B].cpu().numpy().T, s["zbar"]), j

    assert np.array_equal(tr.v.cpu().numpy(), prev["v"]) and np.array_equal(tr.z.cpu().numpy(), prev["z"])
    assert float(tr.loss_b.sum()) == loss_d

    # -- e-prop: the C restatement of _kernels.py on the device's inputs
    beta, rho = F(tr.params.beta), F(tr.params.rho)
    for plan, syn, om_, trace_key in ((tr.plan_in, tr.s_in, ot.m_in, "xbar"),
                                      (tr.plan_rec, tr.s_rec, ot.m_rec, "zbar")):
        tg = np.ascontiguousarray(plan.m.target.cpu().numpy())
        rl = np.ascontiguousarray(plan.m.row_length.cpu().numpy())
        eps = np.zeros((B,) + tg.shape, F)
        ebar = np.zeros_like(eps)
        grad = np.zeros(tg.shape, np.float64)
        for t in range(T):
            s = snaps[t]
            eprop_accumulate_c(tg, rl, np.ascontiguousarray(s[trace_key]), s["psi"], s["lsig"],
                               eps, ebar, grad, beta, rho, al)
        E = int(rl.sum())
        off = plan.off.cpu().numpy()[:E]
        flat = lambda a: plan.replica_major(a).cpu().numpy()[:, :E]  # noqa: E731
        assert np.array_equal(flat(plan.eps), eps.reshape(B, -1)[:, off])
        assert np.array_equal(flat(plan.ebar), ebar.reshape(B, -1)[:, off])
        gd = syn.planes["grad"].cpu().numpy()
        mask = np.arange(tg.shape[1])[None, :] < rl[:, None]
        assert np.allclose(gd[mask], grad[mask], rtol=1e-13, atol=1e-13 * np.abs(grad).max())
    g_w_out = np.zeros((C, hidden))
    g_b_out = np.zeros(C)
    for t in range(T):
        g_w_out += snaps[t]["d"].T @ snaps[t]["zbar"].astype(np.float64)
        g_b_out += snaps[t]["d"].sum(axis=0)
    assert np.allclose(tr.g_w_out.cpu().numpy(), g_w_out, rtol=1e-12, atol=1e-12)
    assert np.allclose(tr.g_b_out.cpu().numpy(), g_b_out, rtol=1e-12, atol=1e-12)

    # -- update: oracle scale + L1 + Adam on the device's raw gradients
    for om_, syn in ((ot.m_in, tr.s_in), (ot.m_rec, tr.s_rec)):
        om_.planes["grad"][:] = syn.planes["grad"].cpu().numpy()
    ot.g_w_out[:] = tr.g_w_out.cpu().numpy()
    ot.g_b_out[:] = tr.g_b_out.cpu().numpy()
    loss, acc = tr.update_phase(0)
    assert abs(loss - loss_o / (B * T)) <= 1e-10 * abs(loss)
    inv = 1.0 / B
    for g_ in (ot.m_in.planes["grad"], ot.m_rec.planes["grad"], ot.g_w_out, ot.g_b_out):
        g_ *= inv
    ot.dr_in.l1_step()
    ot.dr_rec.l1_step()
    ot.adam_in.apply(ot.m_in.planes["w"], ot.m_in.planes["grad"])
    ot.adam_rec.apply(ot.m_rec.planes["w"], ot.m_rec.planes["grad"])
    ot.adam_out.apply(ot.w_out, ot.g_w_out)
    ot.adam_b.apply(ot.b_out, ot.g_b_out)
    for om_, syn in ((ot.m_in, tr.s_in), (ot.m_rec, tr.s_rec)):
        rl = om_.row_length
        for p in ("w", "grad", "adam_m", "adam_v"):
            assert valid_equal(rl, syn.planes[p].cpu().numpy(), om_.planes[p]), p
    assert np.array_equal(tr.w_out.cpu().numpy(), ot.w_out)
    assert np.array_equal(tr.b_out.cpu().numpy(), ot.b_out)

    # -- DEEP R group, state-injected: bit-exact
    om, objs = _inject_deepr(tr, 0)
    om.run_update_group("deep_r")
    removed = tr.rewire_phase()
    assert removed == sum(od.last_removed for _, od, _, _, _ in objs)
    for o, od, m, s, d in objs:
        rl = o.row_length
        assert np.array_equal(m.row_length.cpu().numpy(), rl)
        assert valid_equal(rl, m.target.cpu().numpy(), o.target)
        for p in o.planes:
            assert valid_equal(rl, s.planes[p].cpu().numpy(), o.planes[p])
        assert np.array_equal(d.conn_bits.host_words(), od.conn)


@pytest.mark.parametrize("scale", [4, 8, 16])
def test_topomap_rewiring_at_bench_sizes_state_injected(dev_lib, scale):
    """Topomap s = 4, 8, 16 (the sheets bench.py times): a device run with
    STDP and the stimulus rates bench.py uses (rates_on_device); before each
    of 20 rewiring updates the device state (row lengths, targets, g,
    update counters) is injected into the oracle rule group
    (ref topomap.py:101-196, updates.py:309-372), both run one update, and
    the post-update structure, weights, attempts and event distances must be
    bit-identical.  The offset LUTs come from the oracle's own restatement."""
    from oracle.ragged import Ragged
    from oracle.topomap import RewiringOracle, offset_luts
    from oracle.updates import OracleModel
    from paper_2510_19764_b200.topomap import TopomapModel
    seed = 1
    model = TopomapModel(scale, seed=seed, record_events=True, use_graph=False,
                         rates_on_device=True)
    side = model.geometry.side
    N = side * side
    luts = {"ff": offset_luts(side, 0.16, 2.5), "lat": offset_luts(side, 1.0, 1.0)}
    for name, rule in (("ff", model.ff_rule), ("lat", model.lat_rule)):
        assert np.array_equal(rule._form_lut.cpu().numpy(), luts[name][0])
        assert np.array_equal(rule._dist_lut.cpu().numpy(), luts[name][1])
    snaps = []
    orig = model.net.run_update_group

    def spy(group):
        pre = {}
        for name in ("ff", "lat"):
            m, syn = model.net.matrices[name]
            pre[name] = (m.row_length.cpu().numpy(), m.target.cpu().numpy(),
                         syn.planes["g"].cpu().numpy())
        counts = [b.update_count for b in model.net.groups["rewiring"]]
        orig(group)
        post = {}
        for name, rule in (("ff", model.ff_rule), ("lat", model.lat_rule)):
            m, syn = model.net.matrices[name]
            post[name] = (m.row_length.cpu().numpy(), m.target.cpu().numpy(),
                          syn.planes["g"].cpu().numpy(), rule.attempts.cpu().numpy())
        snaps.append((pre, counts, post))

    model.net.run_update_group = spy
    n_updates = 20
    events = {}
    model.run(float(n_updates))     # 10 steps + one rewiring update per ms
    for name, rule in (("ff", model.ff_rule), ("lat", model.lat_rule)):
        events[name] = ([d for _, d in rule.elim_events], [d for _, d in rule.form_events])
    assert len(snaps) == n_updates
    oracle_events = {"ff": ([], []), "lat": ([], [])}
    changes = 0
    for pre, counts, post in snaps:
        om = OracleModel(seed)
        rules = {}
        for name in ("ff", "lat"):
            rl, tg, g = pre[name]
            o = Ragged(N, N, tg.shape[1], ("g",))
            o.row_length[:] = rl
            o.target[:] = tg
            o.planes["g"][:] = g
            om.add_matrix(name, o)
            r = RewiringOracle(o, side, luts[name][0], luts[name][1], 10 * scale * scale)
            om.add_rule("rewiring", name, r)
            rules[name] = (o, r)
        for b, u in zip(om.groups["rewiring"], counts):
            b.update_count = u
        om.run_update_group("rewiring")
        for name, (o, r) in rules.items():
            rl, tg, g, att = post[name]
            assert np.array_equal(rl, o.row_length), name
            assert valid_equal(o.row_length, tg, o.target), name
            assert valid_equal(o.row_length, g, o.planes["g"]), name
            assert np.array_equal(att, r.attempts), name
            oracle_events[name][0].extend(d for _, k, d in r.events if k == 1)
            oracle_events[name][1].extend(d for _, k, d in r.events if k == 2)
            changes += r.stats["removed"] + r.stats["formed"]
    assert events == oracle_events
    assert changes > 0


@pytest.mark.parametrize("scale", [1, 4, 16])
def test_device_stimulus_rates_match_numpy(dev_lib, scale):
    """sw_poisson_rates (the stimulus rates bench.py's topomap sweep uses,
    CUDA exp/hypot) vs the host numpy rates of ref neurons.py:175-183 and
    probabilities of :191-192.  Bound: rates within 1e-13 relative (CUDA
    exp/hypot are within 2 ulp of numpy's, F8, summed over the s^2 stimulus
    centres), probabilities within 4 ulp of 1.0 absolute; Poisson spikes drawn from both probability
    vectors (same counters, 200 steps) must not differ at all -- a draw can
    only flip when u lands within ~1e-16 of p."""
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.geometry import GridGeometry
    from paper_2510_19764_b200.neurons import PoissonSource
    from paper_2510_19764_b200.rng import CounterRng, fold_key
    geom = GridGeometry(16 * scale)
    n = geom.n
    stim = CounterRng(5, "stimulus")
    for change in range(3):
        bx, by = stim.uniform01() * 16, stim.uniform01() * 16
        centers = [(bx + a * 16, by + b * 16) for a in range(scale) for b in range(scale)]
        host = PoissonSource(geom)
        host.set_correlated_rates(centers)
        p_host = host.probabilities(0.1).clone()
        dev = PoissonSource(geom)
        dev.set_correlated_rates_device(centers, 0.1)
        r_dev = dev.rates_array()
        assert np.allclose(r_dev, host.rates, rtol=1e-13, atol=0)
        p_dev = dev._p_dev
        # p = 1 - exp(-r h 1e-3) ~ 5e-4: the exp rounding (an ulp of 1.0,
        # 1.1e-16) is absolute here, so the bound is absolute: 4 ulp of 1.0
        assert float((p_dev - p_host).abs().max()) <= 4 * 2.0 ** -52
        b_host = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
        b_dev = torch.zeros_like(b_host)
        key = fold_key(5, "poisson")
        diff = 0
        for step in range(200):
            for p, b in ((p_host, b_host), (p_dev, b_dev)):
                _lib.call("sw_poisson_step", key, (change * 200 + step) * n, p.data_ptr(), n,
                          b.data_ptr(), _lib.stream_ptr())
            diff += int((b_host != b_dev).sum())
        assert diff == 0
