"""Device e-prop / ALIF kernels and the device trainer vs the reference
golden vectors and the oracle."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle_helpers import valid_equal

pytestmark = pytest.mark.gpu


def test_alif_kernels_bit_exact(dev_lib):
    from paper_2510_19764_b200.neurons import AlifLayer, AlifParams
    g = golden("alif_eprop.npz")
    layer = AlifLayer(48, AlifParams(), batch=8)
    for t in range(6):
        assert np.array_equal(layer.surrogate().cpu().numpy(), g[f"psi{t}"])
        layer.step(torch.from_numpy(g[f"rec{t}"]).cuda(), torch.from_numpy(g[f"ext{t}"]).cuda())
        assert np.array_equal(layer.v.cpu().numpy(), g[f"v{t}"])
        assert np.array_equal(layer.a.cpu().numpy(), g[f"a{t}"])
        assert np.array_equal(layer.z.cpu().numpy(), g[f"z{t}"])


def test_eprop_dropin_bit_exact(dev_lib):
    from paper_2510_19764_b200.neurons import AlifParams
    from paper_2510_19764_b200.plasticity import eprop_accumulate_batch
    g = golden("alif_eprop.npz")
    p = AlifParams()
    tg = torch.from_numpy(g["target"]).cuda()
    rl = torch.from_numpy(g["row_length"]).cuda()
    eps = torch.zeros((8,) + tuple(tg.shape), dtype=torch.float32, device="cuda")
    ebar = torch.zeros_like(eps)
    grad = torch.zeros(tuple(tg.shape), dtype=torch.float64, device="cuda")
    for t in range(25):
        eprop_accumulate_batch(tg, rl, torch.from_numpy(g[f"trace{t}"]).cuda(),
                               torch.from_numpy(g[f"psi_e{t}"]).cuda(),
                               torch.from_numpy(g[f"lsig{t}"]).cuda(), eps, ebar, grad,
                               np.float32(p.beta), np.float32(p.rho), np.float32(p.alpha))
    assert np.array_equal(eps.cpu().numpy(), g["eps"])
    assert np.array_equal(ebar.cpu().numpy(), g["ebar"])
    assert np.array_equal(grad.cpu().numpy(), g["grad"])


@pytest.mark.parametrize("B,P,H,cap,R", [(8, 30, 48, 12, 6), (64, 700, 256, 82, 26),
                                         (37, 100, 1024, 40, 10)])
def test_fused_eprop_equals_reference_layout(dev_lib, B, P, H, cap, R):
    """The compact-plan fused kernel reproduces the reference-layout kernel
    bit-for-bit (eps, ebar per synapse and the float64 gradient)."""
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import _Plan
    from paper_2510_19764_b200.connectivity import RaggedMatrix
    from paper_2510_19764_b200.plasticity import eprop_accumulate_batch
    import ctypes
    rs = np.random.default_rng(P)
    tg = np.zeros((P, cap), np.int32)
    rl = np.zeros(P, np.int32)
    for i in range(P):
        k = int(min(cap, rs.poisson(R)))
        tg[i, :k] = rs.choice(H, size=k, replace=False)
        rl[i] = k
    m = RaggedMatrix(P, H, cap)
    m.load_state(rl, tg)
    plan = _Plan(m, B)
    plan.ensure(int(rl.sum()))
    plan.build()
    grad0 = rs.standard_normal((P, cap))
    gplane = torch.from_numpy(grad0).cuda()
    _lib.call("sw_gather_f64", gplane.data_ptr(), plan.off.data_ptr(), plan.e_pad,
              plan.grad.data_ptr(), _lib.stream_ptr())
    ref_eps = torch.zeros((B, P, cap), dtype=torch.float32, device="cuda")
    ref_ebar = torch.zeros_like(ref_eps)
    ref_grad = torch.from_numpy(grad0.copy()).cuda()
    segs = (_lib.EpropSeg * 1)()
    for t in range(7):
        trace = torch.from_numpy((rs.random((B, P)) * 2).astype(np.float32)).cuda()
        psi = torch.from_numpy((rs.random((B, H)) * 0.5).astype(np.float32)).cuda()
        lsig = torch.from_numpy(rs.standard_normal((B, H)).astype(np.float32)).cuda()
        eprop_accumulate_batch(m.target, m.row_length, trace, psi, lsig, ref_eps, ref_ebar,
                               ref_grad, 0.0174, 0.9995, 0.95)
        segs[0] = plan.seg(trace)
        _lib.call("sw_eprop_fused_step", ctypes.cast(segs, ctypes.c_void_p), 1, psi.data_ptr(),
                  lsig.data_ptr(), B, H, float(np.float32(0.0174)), float(np.float32(0.9995)),
                  float(np.float32(0.95)), None, None, None, None, 0, 0, _lib.workspace(),
                  _lib.stream_ptr())
    _lib.call("sw_scatter_f64", gplane.data_ptr(), plan.off.data_ptr(), plan.e_pad,
              plan.grad.data_ptr(), _lib.stream_ptr())
    assert valid_equal(rl, gplane.cpu().numpy(), ref_grad.cpu().numpy())
    off = plan.off.cpu().numpy()
    E = int(rl.sum())
    def flat(t):   # [tile, B, 32] -> [B, e_pad]
        return t.permute(1, 0, 2).reshape(B, -1).cpu().numpy()
    re = ref_eps.reshape(B, -1).cpu().numpy()[:, off[:E]]
    assert np.array_equal(flat(plan.eps)[:, :E], re)
    rb = ref_ebar.reshape(B, -1).cpu().numpy()[:, off[:E]]
    assert np.array_equal(flat(plan.ebar)[:, :E], rb)


def _small_trainer(use_graph=True):
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    task = SyntheticTask(num_classes=3, num_inputs=20, example_steps=60, seed=4)
    return EpropClassifierTrainer(task, hidden=24, batch_size=8, seed=4, deep_r=True,
                                  input_density=0.3, recurrent_density=0.2, use_graph=use_graph)


def test_trainer_init_matches_reference_exactly(dev_lib):
    from oracle.classifier import TaskOracle, TrainerOracle
    tr = _small_trainer()
    ot = TrainerOracle(TaskOracle(num_classes=3, num_inputs=20, example_steps=60, seed=4),
                       hidden=24, batch_size=8, seed=4, input_density=0.3, recurrent_density=0.2)
    for dm, ds, om, dr, odr in ((tr.m_in, tr.s_in, ot.m_in, tr.deep_r_in, ot.dr_in),
                                (tr.m_rec, tr.s_rec, ot.m_rec, tr.deep_r_rec, ot.dr_rec)):
        assert np.array_equal(dm.row_length.cpu().numpy(), om.row_length)
        assert np.array_equal(dm.target.cpu().numpy(), om.target)
        assert np.array_equal(ds.planes["w"].cpu().numpy(), om.planes["w"])
        assert np.array_equal(dr.sign_bits.host_words(), odr.sign)
        assert np.array_equal(dr.conn_bits.host_words(), odr.conn)
    assert np.array_equal(tr.w_out.cpu().numpy(), ot.w_out)


def test_trainer_matches_reference_run_and_rewires_exactly(dev_lib):
    """Three batches vs the golden reference run: loss/weights to float
    tolerance; each DEEP R step state-injected into the oracle and compared
    bit-exactly (row lengths, targets, planes, bits)."""
    from oracle.deep_r import DeepROracle
    from oracle.ragged import Ragged
    from oracle.updates import OracleModel
    g = golden("trainer.npz")
    for use_graph in (True, False):
        tr = _small_trainer(use_graph)
        for b in range(3):
            loss, acc = tr.gradient_phase(b)
            assert abs(loss - float(g[f"b{b}_loss"])) <= 1e-6 * abs(loss), (b, loss)
            # state injection: oracle DEEP R on the device's post-Adam state
            om = OracleModel(4)
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
        for name, m, s in (("in", tr.m_in, tr.s_in), ("rec", tr.m_rec, tr.s_rec)):
            rl = g[f"{name}_row_length"]
            assert np.array_equal(m.row_length.cpu().numpy(), rl)
            assert valid_equal(rl, m.target.cpu().numpy(), g[f"{name}_target"])
            mask = np.arange(rl.size and m.stride)[None, :] < rl[:, None]
            assert np.allclose(s.planes["w"].cpu().numpy()[mask], g[f"{name}_w"][mask],
                               rtol=1e-6, atol=1e-9)


def test_overlapped_graph_equals_sequential_steps(dev_lib):
    """The graph replay overlaps step t's e-prop update with step t+1's
    forward pass (two streams, parity buffers); gradients, weights and
    rewiring must be bit-identical to strictly sequential launches."""
    a = _small_trainer(use_graph=True)
    b = _small_trainer(use_graph=False)
    assert a.overlap
    for k in range(3):
        ha, hb = a.train_batch(k), b.train_batch(k)
        assert ha["loss"] == hb["loss"] and ha["removed"] == hb["removed"]
    for x, y in ((a.s_in, b.s_in), (a.s_rec, b.s_rec)):
        for p in ("w", "grad", "adam_m", "adam_v"):
            assert torch.equal(x.planes[p], y.planes[p]), p
    assert torch.equal(a.w_out, b.w_out) and torch.equal(a.g_w_out, b.g_w_out)
    assert a.connectivity_fingerprint() == b.connectivity_fingerprint()


@pytest.mark.parametrize("splits", [0, 3])
@pytest.mark.parametrize("B,P,H,cap,R,k", [(64, 700, 256, 82, 26, 4), (37, 100, 1024, 40, 10, 3),
                                           (8, 30, 48, 12, 6, 1), (48, 700, 256, 82, 26, 8),
                                           (20, 120, 300, 30, 9, 5)])
def test_blocked_eprop_equals_single_steps(dev_lib, B, P, H, cap, R, k, splits):
    """sw_eprop_fused_block over k steps == k calls of sw_eprop_fused_step:
    eps/ebar bit-identical, readout gradients to float64 rounding, the
    synapse gradient bit-identical for k = 1 and within 1e-13 relative for
    k > 1 (k per-step partial chains added at the end)."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import _Plan
    from paper_2510_19764_b200.connectivity import RaggedMatrix
    rs = np.random.default_rng(P + k)
    tg = np.zeros((P, cap), np.int32)
    rl = np.zeros(P, np.int32)
    for i in range(P):
        n = int(min(cap, rs.poisson(R)))
        tg[i, :n] = rs.choice(H, size=n, replace=False)
        rl[i] = n
    m = RaggedMatrix(P, H, cap)
    m.load_state(rl, tg)
    plans = [_Plan(m, B), _Plan(m, B)]
    for pl in plans:
        pl.ensure(int(rl.sum()))
        pl.build()
        pl.eps.copy_(torch.from_numpy(rs.random(pl.eps.shape).astype(np.float32)).cuda())
        pl.grad.copy_(torch.from_numpy(rs.standard_normal(pl.grad.shape)).cuda())
    plans[1].eps.copy_(plans[0].eps)
    plans[1].ebar.copy_(plans[0].ebar)
    plans[1].grad.copy_(plans[0].grad)
    C = 5
    f = lambda *s: torch.from_numpy(rs.random(s).astype(np.float32)).cuda()
    steps = [dict(trace=f(B, P) * 2, psi=f(B, H) * 0.5, lsig=f(B, H) - 0.5,
                  d=torch.from_numpy(rs.standard_normal((B, C))).cuda(), zbar=f(B, H))
             for _ in range(k)]
    beta, rho, alpha = (float(np.float32(x)) for x in (0.0174, 0.9995, 0.95))
    gw = [torch.zeros((C, H), dtype=torch.float64, device="cuda") for _ in range(2)]
    gb = [torch.zeros(C, dtype=torch.float64, device="cuda") for _ in range(2)]
    segs = (_lib.EpropSeg * 1)()
    for s in steps:
        segs[0] = plans[0].seg(s["trace"])
        _lib.call("sw_eprop_fused_step", ctypes.cast(segs, ctypes.c_void_p), 1, s["psi"].data_ptr(),
                  s["lsig"].data_ptr(), B, H, beta, rho, alpha, s["d"].data_ptr(),
                  s["zbar"].data_ptr(), gw[0].data_ptr(), gb[0].data_ptr(), C, 0,
                  _lib.workspace(), _lib.stream_ptr())
    blk = _lib.EpropBlock()
    blk.k = k
    for j, s in enumerate(steps):
        blk.psi[j], blk.lsig[j] = s["psi"].data_ptr(), s["lsig"].data_ptr()
        blk.pre_trace[0][j] = s["trace"].data_ptr()
        blk.d[j], blk.zbar[j] = s["d"].data_ptr(), s["zbar"].data_ptr()
    if splits:   # split readout with its (zeroed) partial scratch
        nbytes = int(_lib.lib().sw_eprop_readout_scratch_bytes(H, C, splits))
        scratch = torch.zeros(nbytes // 8 + 1, dtype=torch.float64, device="cuda")
        blk.ro_scratch, blk.ro_splits = scratch.data_ptr(), splits
    segs[0] = plans[1].seg(steps[0]["trace"])
    _lib.call("sw_eprop_fused_block", ctypes.cast(segs, ctypes.c_void_p), 1, ctypes.byref(blk), B, H,
              beta, rho, alpha, gw[1].data_ptr(), gb[1].data_ptr(), C, _lib.workspace(),
              _lib.stream_ptr())
    assert torch.equal(plans[0].eps, plans[1].eps) and torch.equal(plans[0].ebar, plans[1].ebar)
    if k == 1:
        assert torch.equal(plans[0].grad, plans[1].grad)
    else:
        assert torch.allclose(plans[1].grad, plans[0].grad, rtol=1e-13, atol=1e-13)
    assert torch.allclose(gw[1], gw[0], rtol=1e-12, atol=1e-12)
    assert torch.allclose(gb[1], gb[0], rtol=1e-12, atol=1e-12)
    if splits:   # the counters are left zeroed for the next launch
        cnt = scratch.view(torch.int32)[(splits * C * H + splits * C) * 2:]
        assert int(cnt.abs().sum()) == 0


def test_grouped_forward_equals_single_steps(dev_lib):
    """sw_clf_step with n_steps = k (one launch, steps back to back per
    replica, slot bases) == k single-step launches: state, per-step slots and
    readout accumulators bit-identical."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import EPROP_BLOCK_STEPS
    tr = [_small_trainer(use_graph=False), _small_trainer(use_graph=False)]
    ids = tr[0].task.train_ids(0, tr[0].batch_size)
    for x in tr:
        x._upload_batch(ids)
        x._prepare(False)
    st = _lib.stream_ptr()
    T = 2 * EPROP_BLOCK_STEPS + 3
    for t in range(T):
        prm = tr[0]._step_params(t)
        _lib.call("sw_clf_step", ctypes.byref(prm), st)
    for t0 in range(0, T, EPROP_BLOCK_STEPS):
        prm = tr[1]._group_params(t0, min(EPROP_BLOCK_STEPS, T - t0))
        _lib.call("sw_clf_step", ctypes.byref(prm), st)
    torch.cuda.synchronize()
    a, b = tr
    for name in ("v", "a", "z", "y", "pi_sum", "loss_b"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    # (the grouped launch leaves the learning signal to sw_eprop_prep and
    # takes its input spikes / traces from sw_clf_inputs)
    for name in ("_slots_zbar", "_slots_psi", "_slots_d"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    K2 = 2 * EPROP_BLOCK_STEPS
    for t in range(T):
        assert torch.equal(a._slots_xbar[t % K2].T, b.xbar_all[t, :, :a.local_b]) or t < T - K2, t


@pytest.mark.parametrize("NI,H,din,drec,p_spk,z_spk", [
    (300, 200, 0.3, 0.25, 0.5, 0.3),     # staged path, 32-bit layout
    (300, 1024, 0.05, 0.02, 0.5, 0.3),   # staged path, compact 16-bit layout (large layer)
    (300, 200, 0.3, 0.25, 1.0, 1.0),     # every row spikes: > 2048 entries, warp-serial fallback
])
def test_forward_currents_are_grouped_ordered_sums(dev_lib, NI, H, din, drec, p_spk, z_spk):
    """The forward kernel's event-driven propagation (classifier_fwd.cu P2c):
    per post, the ascending spiking rows in G contiguous groups, each summed
    in row order from +0.0, the group sums added in group order
    (oracle_helpers.grouped_currents) -- on the staged path and on the
    unstaged one (every row spiking: more entries than the staging holds).
    Spikes are forced: p_in in {0, 1} and a chosen hidden z; v = a = 0, so
    after one step v = f32(alpha * (0 - z*v_thr)) + rec + ext exactly."""
    from oracle_helpers import grouped_currents
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    task = SyntheticTask(num_classes=5, num_inputs=NI, example_steps=10, seed=7)
    tr = EpropClassifierTrainer(task, hidden=H, batch_size=4, seed=7, deep_r=False,
                                input_density=din, recurrent_density=drec, use_graph=False)
    ids = task.train_ids(0, tr.batch_size)
    tr._upload_batch(ids)
    tr._prepare(False)
    rs = np.random.default_rng(7)
    B, NI, H = tr.batch_size, task.num_inputs, tr.hidden
    pin = (rs.random((B, NI)) < p_spk).astype(np.float64)
    z = (rs.random((B, H)) < z_spk).astype(np.float32)
    tr.p_in.copy_(torch.from_numpy(pin))
    tr.z.copy_(torch.from_numpy(z))
    prm = tr._step_params(0)
    _lib.call("sw_clf_step", ctypes.byref(prm), _lib.stream_ptr())
    torch.cuda.synchronize()
    v = tr.v.cpu().numpy()
    f32 = np.float32
    p = tr.params
    alpha, vthr = f32(p.alpha), f32(p.v_thr)

    w_in, w_rec = tr.w32_in.cpu().numpy(), tr.w32_rec.cpu().numpy()
    mi, mr = tr.m_in, tr.m_rec
    ext_all = grouped_currents(mi.row_length.cpu().numpy(), mi.target.cpu().numpy(), w_in, pin == 1.0, H)
    rec_all = grouped_currents(mr.row_length.cpu().numpy(), mr.target.cpu().numpy(), w_rec, z != 0, H)
    for b in range(B):
        ext, rec = ext_all[b], rec_all[b]
        for h in range(H):
            vv = f32(alpha * f32(f32(0) - f32(z[b, h] * vthr)))
            vv = f32(f32(vv + rec[h]) + ext[h])
            assert v[b, h] == vv, (b, h)


@pytest.mark.parametrize("NI,H,din,drec,p_spk,z_spk", [
    (333, 200, 0.3, 0.25, 0.5, 0.3),     # 8 groups, ragged input words
    (300, 200, 0.3, 0.25, 1.0, 1.0),     # every row spikes: the group lists full
    (700, 512, 0.1, 0.05, 0.5, 0.3),     # 4 groups, 2 hidden units per thread
    (300, 1024, 0.05, 0.02, 1.0, 1.0),   # 4 groups, 4 hidden units per thread, all rows
])
def test_grouped_forward_currents_forced_spikes(dev_lib, NI, H, din, drec, p_spk, z_spk):
    """The trainer's grouped forward (k_clf_fwd2: input spikes from
    sw_clf_inputs' words, hidden rows from the previous step's z) computes
    each current as the grouped ordered sum of oracle_helpers.grouped_currents.
    Spikes are forced (p_in in {0, 1}, chosen z; v = a = 0), so after the
    first step v = f32(alpha * (0 - z*v_thr)) + rec + ext exactly."""
    from oracle_helpers import grouped_currents
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    task = SyntheticTask(num_classes=5, num_inputs=NI, example_steps=10, seed=11)
    tr = EpropClassifierTrainer(task, hidden=H, batch_size=6, seed=11, deep_r=False,
                                input_density=din, recurrent_density=drec, use_graph=False)
    ids = task.train_ids(0, tr.batch_size)
    tr._upload_batch(ids)
    rs = np.random.default_rng(11)
    B = tr.batch_size
    pin = (rs.random((B, NI)) < p_spk).astype(np.float64)
    z = (rs.random((B, H)) < z_spk).astype(np.float32)
    tr.p_in.copy_(torch.from_numpy(pin).to(tr.p_in.dtype).reshape(tr.p_in.shape))
    tr._prepare(False)
    tr.z.copy_(torch.from_numpy(z))
    prm = tr._group_params(0, 1)
    _lib.call("sw_clf_step", ctypes.byref(prm), _lib.stream_ptr())
    torch.cuda.synchronize()
    v = tr.v.cpu().numpy()
    f32 = np.float32
    alpha, vthr = f32(tr.params.alpha), f32(tr.params.v_thr)
    w_in, w_rec = tr.w32_in.cpu().numpy(), tr.w32_rec.cpu().numpy()
    mi, mr = tr.m_in, tr.m_rec
    ext_all = grouped_currents(mi.row_length.cpu().numpy(), mi.target.cpu().numpy(), w_in, pin == 1.0, H)
    rec_all = grouped_currents(mr.row_length.cpu().numpy(), mr.target.cpu().numpy(), w_rec, z != 0, H)
    for b in range(B):
        vv = (alpha * (f32(0) - z[b] * vthr)).astype(f32)
        vv = ((vv + rec_all[b]).astype(f32) + ext_all[b]).astype(f32)
        bad = np.flatnonzero(v[b] != vv)
        assert bad.size == 0, (b, bad[:8], v[b, bad[:4]], vv[bad[:4]])


@pytest.mark.parametrize("H,v0", [(200, 0.0), (200, 50.0), (1024, 50.0)])
def test_grouped_readout_sums_from_spike_words(dev_lib, H, v0):
    """The readout launch after the grouped forward: per step and class the
    f64 sum of w_out[c][h] over the step's spiking units (the spike words the
    forward wrote) in ascending order from +0.0, then y = (alpha*y + s) + b,
    steps in order -- bit-exact against numpy.  v0 > threshold drives every
    hidden unit to spike, so steps with more spiking units than the readout's
    list capacity take the word-walk path."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import EPROP_BLOCK_STEPS as K
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    task = SyntheticTask(num_classes=7, num_inputs=150, example_steps=2 * K, seed=3)
    tr = EpropClassifierTrainer(task, hidden=H, batch_size=5, seed=3, deep_r=False,
                                input_density=0.2, recurrent_density=0.1, use_graph=False)
    tr._upload_batch(task.train_ids(0, tr.batch_size))
    tr._prepare(False)
    tr.v.fill_(v0)
    y = tr.y.cpu().numpy().copy()
    w_out, b_out = tr.w_out.cpu().numpy(), tr.b_out.cpu().numpy()
    alpha = float(tr.params.alpha)
    B, C, HW = tr.batch_size, task.num_classes, (H + 31) // 32
    dense = 0
    for t0 in (0, K):
        _lib.call("sw_clf_step", ctypes.byref(tr._group_params(t0, K)), _lib.stream_ptr())
        torch.cuda.synchronize()
        words = tr.z_bits.cpu().numpy().view(np.uint32)
        for s in range(K):
            for b in range(B):
                bits = np.unpackbits(words[s, b].view(np.uint8), bitorder="little")[:H]
                units = np.flatnonzero(bits)
                dense += units.size > 64
                for c in range(C):
                    acc = 0.0
                    for h in units:
                        acc = acc + float(w_out[c, h])
                    y[b, c] = (alpha * y[b, c] + acc) + float(b_out[c])
    assert np.array_equal(tr.y.cpu().numpy(), y)
    if v0 > 0:
        assert dense > 0


@pytest.mark.parametrize("H,p_spk", [(512, 0.05), (512, 1.0), (1024, 0.05), (1024, 1.0)])
def test_grouped_forward_wide_layers_equal_single_steps(dev_lib, H, p_spk):
    """Wide layers (2 / 4 units per thread, input and hidden groups on
    separate warps): the grouped launch over 16 steps, with sparse and with
    saturated inputs (every input spiking every step), equals 16 single-step
    launches bit for bit (v, a, z)."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import EPROP_BLOCK_STEPS as K
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    task = SyntheticTask(num_classes=4, num_inputs=300, example_steps=K, seed=5)
    trs = [EpropClassifierTrainer(task, hidden=H, batch_size=3, seed=5, deep_r=False, input_density=0.05,
                                  recurrent_density=0.02, use_graph=False) for _ in range(2)]
    rs = np.random.default_rng(5)
    pin = (rs.random((3, task.num_inputs)) < p_spk).astype(np.float64)
    for tr in trs:
        tr._upload_batch(task.train_ids(0, tr.batch_size))
        tr.p_in.copy_(torch.from_numpy(pin))
        tr._prepare(False)
    st = _lib.stream_ptr()
    for t in range(K):
        _lib.call("sw_clf_step", ctypes.byref(trs[0]._step_params(t)), st)
    _lib.call("sw_clf_step", ctypes.byref(trs[1]._group_params(0, K)), st)
    torch.cuda.synchronize()
    for name in ("v", "a", "z"):
        assert torch.equal(getattr(trs[0], name), getattr(trs[1], name)), name


def test_pinned_host_inputs_equal_numpy_inputs(dev_lib):
    """train_batch from host inputs already in pinned memory (direct async
    copies) == from numpy arrays (staged through the trainer's pinned buffers)."""
    a, b = _small_trainer(use_graph=True), _small_trainer(use_graph=True)
    for k in range(2):
        h = a.host_inputs(k)
        pinned = (torch.from_numpy(h[0]).pin_memory(), torch.from_numpy(h[1].view(np.int64)).pin_memory(),
                  torch.from_numpy(h[2]).pin_memory())
        ra, rb = a.train_batch(k, host=h), b.train_batch(k, host=pinned)
        assert ra["loss"] == rb["loss"] and ra["removed"] == rb["removed"]
    assert torch.equal(a.s_in.planes["w"], b.s_in.planes["w"])
    assert a.connectivity_fingerprint() == b.connectivity_fingerprint()


@pytest.mark.parametrize("P,H,cap,R,B,k", [(40, 64, 12, 6.0, 8, 8), (700, 256, 82, 25.6, 64, 8),
                                         (33, 50, 9, 4.0, 20, 3), (256, 256, 40, 20.0, 136, 5)])
def test_eprop_pass_replica_minor(dev_lib, P, H, cap, R, B, k):
    """sw_eprop_prep + sw_eprop_pass (the trainer's e-prop path) vs the
    reference-layout kernel (sw_eprop_accumulate_batch, _kernels.py:15-39
    semantics) over k steps: eps and ebar bit-identical, the gradient within
    1e-13 relative (float64 regrouping of the replica sum); the learning
    signal lsig_t bit-identical to the forward pass's f32(d @ W_out) (one fma
    per class, class order; oracle/c lsig_fma); ragged batches (B not a
    multiple of 32) padded with zeros."""
    from oracle.cbuild import lsig_fma_c
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import _Plan
    from paper_2510_19764_b200.connectivity import RaggedMatrix
    from paper_2510_19764_b200.plasticity import eprop_accumulate_batch
    rs = np.random.default_rng(P + B)
    C = 7
    tg = np.zeros((P, cap), np.int32)
    rl = np.zeros(P, np.int32)
    for i in range(P):
        n = int(min(cap, rs.poisson(R)))
        tg[i, :n] = rs.choice(H, size=n, replace=False)
        rl[i] = n
    m = RaggedMatrix(P, H, cap)
    m.load_state(rl, tg)
    plan = _Plan(m, B, shift=0, layout="chunk")
    plan.ensure(int(rl.sum()))
    plan.build()
    L = plan.ldb
    grad0 = rs.standard_normal((P, cap))
    gplane = torch.from_numpy(grad0).cuda()
    _lib.call("sw_gather_f64", gplane.data_ptr(), plan.off.data_ptr(), plan.e_pad, plan.grad.data_ptr(),
              _lib.stream_ptr())
    ref_eps = torch.zeros((B, P, cap), dtype=torch.float32, device="cuda")
    ref_ebar = torch.zeros_like(ref_eps)
    ref_grad = torch.from_numpy(grad0.copy()).cuda()
    beta, rho, alpha = (float(np.float32(x)) for x in (0.0174, 0.9995, 0.95))
    w_out = torch.from_numpy(rs.standard_normal((C, H))).cuda()
    f = lambda *s: torch.from_numpy(rs.random(s).astype(np.float32)).cuda()  # noqa: E731
    xt = torch.zeros((k, P, L), dtype=torch.float32, device="cuda")
    zt, pt, lt = (torch.zeros((k, H, L), dtype=torch.float32, device="cuda") for _ in range(3))
    for rep in range(2):   # two passes: the state carries over
        steps = [dict(trace=f(B, P) * 2, psi=f(B, H) * 0.5, zbar=f(B, H),
                      d=torch.from_numpy(rs.standard_normal((B, C))).cuda()) for _ in range(k)]
        pr = _lib.EpropPrep()
        pr.k, pr.batch, pr.ldb, pr.num_inputs, pr.hidden, pr.num_classes = k, B, L, P, H, C
        for j, s in enumerate(steps):
            pr.xbar[j], pr.zbar[j] = s["trace"].data_ptr(), s["zbar"].data_ptr()
            pr.psi[j], pr.d[j] = s["psi"].data_ptr(), s["d"].data_ptr()
        pr.w_out = w_out.data_ptr()
        pr.xbar_t, pr.zbar_t, pr.psi_t, pr.lsig_t = (t.data_ptr() for t in (xt, zt, pt, lt))
        gw = torch.zeros((C, H), dtype=torch.float64, device="cuda")
        gb = torch.zeros(C, dtype=torch.float64, device="cuda")
        part = torch.zeros(int(_lib.lib().sw_eprop_prep_scratch_bytes(k, B, H, C)) // 8 + 1,
                           dtype=torch.float64, device="cuda")
        pr.g_w_out, pr.g_b_out, pr.ro_partial = gw.data_ptr(), gb.data_ptr(), part.data_ptr()
        _lib.call("sw_eprop_prep", ctypes.byref(pr), _lib.stream_ptr())
        # readout gradients (classifier.py:221-222) summed over the group
        gw_o = sum(s["d"].cpu().numpy().T @ s["zbar"].cpu().numpy().astype(np.float64) for s in steps)
        gb_o = sum(s["d"].cpu().numpy().sum(axis=0) for s in steps)
        assert np.allclose(gw.cpu().numpy(), gw_o, rtol=1e-12, atol=1e-12)
        assert np.allclose(gb.cpu().numpy(), gb_o, rtol=1e-12, atol=1e-12)
        for j, s in enumerate(steps):
            s["lsig"] = torch.from_numpy(lsig_fma_c(s["d"].cpu().numpy(), w_out.cpu().numpy())).cuda()
            assert torch.equal(lt[j, :, :B].T, s["lsig"]), j
            assert torch.equal(xt[j, :, :B].T, s["trace"]) and torch.equal(zt[j, :, :B].T, s["zbar"])
            assert torch.equal(pt[j, :, :B].T, s["psi"])
            assert int((lt[j, :, B:] != 0).sum()) == 0 and int((xt[j, :, B:] != 0).sum()) == 0
            eprop_accumulate_batch(m.target, m.row_length, s["trace"], s["psi"], s["lsig"], ref_eps, ref_ebar,
                                   ref_grad, beta, rho, alpha)
        segs = (_lib.EpropTSeg * 1)()
        segs[0] = plan.tseg([xt[j] for j in range(k)])
        tp = _lib.EpropTPass()
        tp.k = k
        for j in range(k):
            tp.psi_t[j], tp.lsig_t[j] = pt[j].data_ptr(), lt[j].data_ptr()
        nb = int(_lib.lib().sw_eprop_pass_scratch_bytes(plan.e_pad, L))
        if rep == 0:
            scratch = torch.empty(nb // 8 + 1, dtype=torch.float64, device="cuda")
        tp.scratch = scratch.data_ptr()
        _lib.call("sw_eprop_pass", ctypes.cast(segs, ctypes.c_void_p), 1, ctypes.byref(tp), L, beta, rho,
                  alpha, _lib.stream_ptr())
        torch.cuda.synchronize()
        off = plan.off.cpu().numpy()
        E = int(rl.sum())
        re = ref_eps.reshape(B, -1).cpu().numpy()[:, off[:E]]
        assert np.array_equal(plan.replica_major(plan.eps).cpu().numpy()[:, :E], re)
        rb = ref_ebar.reshape(B, -1).cpu().numpy()[:, off[:E]]
        assert np.array_equal(plan.replica_major(plan.ebar).cpu().numpy()[:, :E], rb)
        g = gplane.clone()
        _lib.call("sw_scatter_f64", g.data_ptr(), plan.off.data_ptr(), plan.e_pad, plan.grad.data_ptr(),
                  _lib.stream_ptr())
        gr = ref_grad.cpu().numpy()
        mask = np.arange(cap)[None, :] < rl[:, None]
        assert np.allclose(g.cpu().numpy()[mask], gr[mask], rtol=1e-13, atol=1e-13 * np.abs(gr).max())


def test_eprop_interleaved_psl_and_zero_state(dev_lib):
    """The trainer's e-prop options against the plain layout: sw_eprop_prep
    writing psi / lsig interleaved (psl_t) and sw_eprop_pass reading them
    (psl = 1), with the first pass starting eps / ebar from zero without
    reading them (state_zero = 1; the state buffers hold garbage) -- eps,
    ebar, gradient and the de-interleaved psi / lsig bit-identical to separate
    arrays and explicitly zeroed state."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import _Plan
    from paper_2510_19764_b200.connectivity import RaggedMatrix
    P, H, cap, B, C, k = 300, 96, 30, 70, 20, 6
    rs = np.random.default_rng(7)
    tg = np.zeros((P, cap), np.int32)
    rl = np.zeros(P, np.int32)
    for i in range(P):
        n = int(min(cap, rs.poisson(10.0)))
        tg[i, :n] = rs.choice(H, size=n, replace=False)
        rl[i] = n
    m = RaggedMatrix(P, H, cap)
    m.load_state(rl, tg)
    plans = []
    for _ in range(2):
        pl = _Plan(m, B, shift=0, layout="chunk")
        pl.ensure(int(rl.sum()))
        pl.build()
        plans.append(pl)
    L = plans[0].ldb
    plans[0].eps.fill_(7.0)        # garbage: state_zero must not read it
    plans[0].ebar.fill_(-3.0)
    plans[1].eps.zero_()
    plans[1].ebar.zero_()
    f = lambda *s: torch.from_numpy(rs.random(s).astype(np.float32)).cuda()  # noqa: E731
    w_out = torch.from_numpy(rs.standard_normal((C, H))).cuda()
    beta, rho, alpha = (float(np.float32(x)) for x in (0.0174, 0.9995, 0.95))
    psl = torch.zeros((k, H, 2 * L), dtype=torch.float32, device="cuda")
    xt = torch.zeros((k, P, L), dtype=torch.float32, device="cuda")
    zt = [torch.zeros((k, H, L), dtype=torch.float32, device="cuda") for _ in range(2)]
    pt, lt = (torch.zeros((k, H, L), dtype=torch.float32, device="cuda") for _ in range(2))
    scr = [torch.zeros(int(_lib.lib().sw_eprop_pass_scratch_bytes(pl.e_pad, L)) // 8 + 1,
                       dtype=torch.float64, device="cuda") for pl in plans]
    for rep in range(2):
        steps = [dict(trace=f(B, P) * 2, psi=f(B, H) * 0.5, zbar=f(B, H),
                      d=torch.from_numpy(rs.standard_normal((B, C))).cuda()) for _ in range(k)]
        for j, s in enumerate(steps):
            xt[j, :, :B] = s["trace"].T
        for v, pl in enumerate(plans):
            pr = _lib.EpropPrep()
            pr.k, pr.batch, pr.ldb, pr.num_inputs, pr.hidden, pr.num_classes = k, B, L, P, H, C
            for j, s in enumerate(steps):
                pr.zbar[j], pr.psi[j], pr.d[j] = s["zbar"].data_ptr(), s["psi"].data_ptr(), s["d"].data_ptr()
            pr.w_out, pr.zbar_t = w_out.data_ptr(), zt[v].data_ptr()
            if v == 0:
                pr.psl_t = psl.data_ptr()
            else:
                pr.psi_t, pr.lsig_t = pt.data_ptr(), lt.data_ptr()
            _lib.call("sw_eprop_prep", ctypes.byref(pr), _lib.stream_ptr())
            segs = (_lib.EpropTSeg * 1)()
            segs[0] = pl.tseg([xt[j] for j in range(k)])
            tp = _lib.EpropTPass()
            tp.k, tp.scratch = k, scr[v].data_ptr()
            for j in range(k):
                tp.psi_t[j], tp.lsig_t[j] = ((psl[j].data_ptr(), 0) if v == 0
                                             else (pt[j].data_ptr(), lt[j].data_ptr()))
            tp.psl = 1 if v == 0 else 0
            tp.state_zero = 1 if (v == 0 and rep == 0) else 0
            _lib.call("sw_eprop_pass", ctypes.cast(segs, ctypes.c_void_p), 1, ctypes.byref(tp), L, beta, rho,
                      alpha, _lib.stream_ptr())
        torch.cuda.synchronize()
        q = psl.view(k, H, L // 4, 2, 4)
        assert torch.equal(q[:, :, :, 0, :].reshape(k, H, L), pt)
        assert torch.equal(q[:, :, :, 1, :].reshape(k, H, L), lt)
        assert torch.equal(plans[0].eps, plans[1].eps) and torch.equal(plans[0].ebar, plans[1].ebar)
        assert torch.equal(plans[0].grad, plans[1].grad)


def test_zero_ranges(dev_lib):
    """sw_zero_ranges zeroes exactly its ranges (unaligned starts and odd
    byte counts included) and nothing around them."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    buf = torch.full((1 << 16,), 0xAB, dtype=torch.uint8, device="cuda")
    ranges = [(3, 1), (17, 45), (256, 4096), (5000, 3), (8191, 20001)]
    base = buf.data_ptr()
    ptrs = (ctypes.c_void_p * len(ranges))(*[base + a for a, _ in ranges])
    nbytes = (ctypes.c_int64 * len(ranges))(*[n for _, n in ranges])
    _lib.call("sw_zero_ranges", ptrs, nbytes, len(ranges), _lib.stream_ptr())
    torch.cuda.synchronize()
    want = np.full(1 << 16, 0xAB, np.uint8)
    for a, n in ranges:
        want[a:a + n] = 0
    assert np.array_equal(buf.cpu().numpy(), want)
