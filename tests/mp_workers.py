"""Worker bodies for the world-size-2 gloo tests (tests/test_multiproc.py).

They exercise the product's host-side sharding (paper_2510_19764_b200.sharding)
on CPU tensors.  The per-rank arithmetic is the oracle's, because the device
kernels need a GPU."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)


def spike_gather(rank, world, port, out):
    from paper_2510_19764_b200.sharding import SpikeGather
    _init(rank, world, port)
    try:
        for n in (1000, 64, 33, 4096):
            rs = np.random.default_rng(n)
            spikes = rs.random(n) < 0.3
            sg = SpikeGather(n, rank, world, "cpu")
            lo, hi = sg.lo, sg.hi
            assert lo % 32 == 0 and (hi % 32 == 0 or hi == n)
            local = np.zeros(sg.bits.numel() * 32, dtype=bool)
            local[lo:hi] = spikes[lo:hi]
            words = np.packbits(local.reshape(-1, 32)[:, ::-1], axis=1, bitorder="big")
            sg.bits.copy_(torch.from_numpy(words.view(">u4").astype(np.uint32).view(np.int32).ravel()))
            full = sg.gather().numpy().view(np.uint32)
            got = ((full[:, None] >> np.arange(32)) & 1).astype(bool).ravel()[:n]
            assert np.array_equal(got, spikes), (n, rank)
        out.put((rank, "ok"))
    finally:
        dist.destroy_process_group()


def batch_dp(rank, world, port, out):
    """Batch-sharded e-prop gradient + identical update/rewiring on every rank."""
    from oracle.classifier import eprop_accumulate
    from oracle.deep_r import AdamOracle, DeepROracle
    from oracle.ragged import Ragged
    from oracle.rng import Stream
    from oracle.updates import OracleModel
    from paper_2510_19764_b200.sharding import allreduce_flat, shard_batch
    _init(rank, world, port)
    try:
        B, P, H, cap, T = 16, 40, 24, 10, 12
        rs = np.random.default_rng(3)
        m = Ragged(P, H, cap, ("w", "grad", "adam_m", "adam_v"))
        for i in range(P):
            k = int(rs.integers(2, cap))
            m.target[i, :k] = rs.choice(H, size=k, replace=False)
            m.row_length[i] = k
        mask = m.slot_mask()
        m.planes["w"][mask] = rs.standard_normal(int(mask.sum())) * 0.01
        trace = rs.random((T, B, P)).astype(np.float32)
        psi = rs.random((T, B, H)).astype(np.float32)
        lsig = (rs.random((T, B, H)) - 0.5).astype(np.float32)
        sl = shard_batch(B, rank, world)
        eps = np.zeros((sl.stop - sl.start, P, cap), np.float32)
        ebar = np.zeros_like(eps)
        for t in range(T):
            eprop_accumulate(m.target, m.row_length, trace[t, sl], psi[t, sl], lsig[t, sl], eps, ebar,
                             m.planes["grad"], 0.07, 0.95, 0.9)
        g = torch.from_numpy(m.planes["grad"])
        allreduce_flat([g])
        m.planes["grad"][:] = g.numpy()
        reduced = m.planes["grad"].copy()
        # identical update on every rank: scale, l1, Adam, DEEP R (same keys)
        m.planes["grad"] *= 1.0 / B
        dr = DeepROracle(m, l1=0.005)
        dr.init_bitfields(Stream.of(5, "deep_r", "x"))
        model = OracleModel(5)
        model.add_matrix("x", m)
        dr.register(model, "deep_r", "x")
        dr.l1_step()
        AdamOracle(1e-2, m=m.planes["adam_m"], v=m.planes["adam_v"]).apply(m.planes["w"],
                                                                           m.planes["grad"])
        model.run_update_group("deep_r")
        h = hashlib.sha256()
        vm = m.slot_mask()
        for a in (m.row_length, m.target[vm], m.planes["w"][vm], dr.conn):
            h.update(np.ascontiguousarray(a).tobytes())
        out.put((rank, reduced, h.hexdigest(), int(dr.last_removed)))
    finally:
        dist.destroy_process_group()


def topomap_sharded(rank, world, port, out):
    """Postsynaptically sharded topographic-map steps (LIF + ordered
    propagation into owned posts, target-spike all-gather, replicated STDP and
    rewiring) against the unsharded run."""
    _init(rank, world, port)
    try:
        res = run_topomap(rank, world, steps=400)
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def run_topomap(rank, world, steps, side=16, seed=4):
    """Oracle topomap stepping; world == 1 is the unsharded reference."""
    from oracle.ragged import Ragged, init_pairwise_bernoulli, transpose
    from oracle.rng import Stream
    from oracle.topomap import RewiringOracle, StdpOracle, lif_cond_step, poisson_step, torus_offset
    from oracle.updates import OracleModel
    from paper_2510_19764_b200.sharding import SpikeGather, post_shard_range
    n = side * side
    gx, gy = np.arange(n) % side, np.arange(n) // side
    dx = np.minimum(gx, side - gx)
    dy = np.minimum(gy, side - gy)
    dist_lut = np.hypot(dx, dy)
    model = OracleModel(seed)
    projs = {}
    for name, p_form, sigma in (("ff", 0.16, 2.5), ("lat", 1.0, 1.0)):
        lut = p_form * np.exp(-(dist_lut ** 2) / (2 * sigma ** 2))
        m = init_pairwise_bernoulli(n, n, lambda i, cols, lut=lut: lut[torus_offset(i, cols, side)],
                                    4.0, Stream.of(seed, "init", name), planes=("g",))
        m.planes["g"][m.slot_mask()] = 0.2
        model.add_matrix(name, m)
        model.add_rule("rewiring", name, RewiringOracle(m, side, lut, dist_lut, 10))
        projs[name] = (m, StdpOracle(m, 0.1))
    V = np.full(n, -70.0)
    gt = np.zeros(n)
    ref = np.full(n, -1, dtype=np.int64)
    pending = np.zeros(n)
    rates = 5.0 + 300.0 * np.exp(-dist_lut ** 2 / 8.0)
    p_src = 1.0 - np.exp(-rates * 0.1e-3)
    ps = Stream.of(seed, "poisson")
    lo, hi = post_shard_range(n, rank, world)
    sg = SpikeGather(n, rank, world, "cpu") if world > 1 else None
    trs = {k: transpose(v[0]) for k, v in projs.items()}
    for k in range(steps):
        src = poisson_step(ps, p_src)                 # every rank: counter-based
        # owned posts only (a rank never reads V/g of other posts)
        own = np.zeros(n, dtype=bool)
        own[lo:hi] = True
        Vo, go, ro = V[lo:hi].copy(), gt[lo:hi].copy(), ref[lo:hi].copy()
        spk_local = lif_cond_step(Vo, go, ro, pending[lo:hi], k) + lo
        V[lo:hi], gt[lo:hi], ref[lo:hi] = Vo, go, ro
        if sg is not None:
            bits = np.zeros(sg.bits.numel() * 32, dtype=bool)
            bits[spk_local] = True
            w = (bits.reshape(-1, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(1)
            sg.bits.copy_(torch.from_numpy(w.astype(np.uint32).view(np.int32)))
            full = sg.gather().numpy().view(np.uint32)
            tgt = np.flatnonzero(((full[:, None] >> np.arange(32)) & 1).astype(bool).ravel()[:n])
        else:
            tgt = spk_local
        # ordered propagation into the owned posts (ff then lat, ascending pre)
        nxt = np.zeros(n)
        for name, spikes in (("ff", src), ("lat", tgt)):
            m = projs[name][0]
            cl, sp, ss = trs[name]
            sset = np.zeros(n, dtype=bool)
            sset[spikes] = True
            for j in range(lo, hi):
                for q in range(cl[j]):
                    i = sp[j, q]
                    if sset[i]:
                        nxt[j] += m.planes["g"][i, ss[j, q]]
        pending = nxt
        # replicated STDP (plasticity.py:64-95), order ff-pre, lat-pre, ff-post, lat-post
        for name in ("ff", "lat"):
            projs[name][1].decay()
        projs["ff"][1].on_pre(src)
        projs["lat"][1].on_pre(tgt)
        projs["ff"][1].on_post(trs["ff"], tgt)
        projs["lat"][1].on_post(trs["lat"], tgt)
        if (k + 1) % 10 == 0:
            model.run_update_group("rewiring")
            trs = {kk: transpose(v[0]) for kk, v in projs.items()}
    state = {}
    for name, (m, st) in projs.items():
        vm = m.slot_mask()
        state[f"{name}.row_length"] = m.row_length.copy()
        state[f"{name}.target"] = np.where(vm, m.target, -1)
        state[f"{name}.g"] = np.where(vm, m.planes["g"], 0.0)
        state[f"{name}.x"] = st.x.copy()
        state[f"{name}.y"] = st.y.copy()
    state["V"] = V
    state["range"] = np.array([lo, hi])
    return state


def device_trainer_dp(rank, world, port, out):
    """Device trainer with a process group (batch DP over gloo on one GPU):
    each rank trains its batch shard; returns what must agree across ranks."""
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    from paper_2510_19764_b200.sharding import shard_batch
    _init(rank, world, port)
    try:
        task = SyntheticTask(num_classes=3, num_inputs=20, example_steps=40, seed=4)
        B = 8
        tr = EpropClassifierTrainer(task, hidden=24, batch_size=B, seed=4, deep_r=True,
                                    input_density=0.3, recurrent_density=0.2,
                                    process_group=dist.group.WORLD, local_batch=shard_batch(B, rank, world))
        hist = [tr.train_batch(k) for k in range(2)]
        w = tr.s_in.planes["w"].cpu().numpy()
        out.put((rank, [(h["loss"], h["removed"]) for h in hist], w,
                 hashlib.sha256(tr.connectivity_fingerprint()).hexdigest()))
    finally:
        dist.destroy_process_group()


# ---- M-update / M-prop microbench sharding -----------------------
def mupdate_instance(P=4096, N=8192, cap=160, seed=5, flip=0.05):
    """A small M-update instance on cuda:0 (same recipe as bench.run_mupdate):
    Bernoulli rows, four float64 planes, DEEP R bitfields, sign flips."""
    import ctypes
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.connectivity import descriptor, init_pairwise_bernoulli_density
    from paper_2510_19764_b200.rng import CounterRng, fold_key
    planes = ("w", "grad", "adam_m", "adam_v")
    m, syn = init_pairwise_bernoulli_density(P, N, 64.0 / N, 1.0, CounterRng(seed, "init", "M"),
                                             var_names=planes, capacity=cap)
    w = syn.planes["w"]
    g = torch.Generator(device="cuda").manual_seed(seed)
    w.copy_(torch.randn(w.shape, generator=g, device="cuda", dtype=torch.float64) * 0.1)
    w.mul_(m.slot_mask())
    from paper_2510_19764_b200.deep_r import DeepR
    dr = DeepR(m, syn, "M", l1_strength=0.0, exclude_diagonal=True)
    dr.init_bitfields(CounterRng(seed, "deep_r", "M"))
    return m, syn, dr, lambda u: _lib.call("sw_flip_signs", ctypes.byref(descriptor(m, syn)), 0,
                                           fold_key(seed, "flip", u), flip, _lib.stream_ptr())


def mupdate_state(m, syn, dr):
    return {"row_length": m.row_length.cpu().numpy(), "target": (m.target * m.slot_mask()).cpu().numpy(),
            "w": (syn.planes["w"] * m.slot_mask()).cpu().numpy(),
            "conn": dr.conn_bits.words.cpu().numpy(), "sign": dr.sign_bits.words.cpu().numpy()}


def run_mupdate(rank, world, updates=3, pg=None):
    """``updates`` DEEP R groups on the instance; rows [lo, hi) of this rank
    (world == 1: the unsharded run).  Returns the local state after each."""
    from paper_2510_19764_b200.connectivity import row_slice
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.sharding import shard_rows
    from paper_2510_19764_b200.updates import Model
    m, syn, dr, flip = mupdate_instance()
    P = m.num_pre
    lo, hi = shard_rows(P, rank, world)
    if world > 1:
        ms, ss = row_slice(m, syn, lo, hi)
        drs = DeepR(ms, ss, "M", l1_strength=0.0, exclude_diagonal=True, process_group=pg,
                    row0=lo, num_pre_global=P)
        drs.load_state(dr.sign_bits.words[lo:hi].cpu().numpy(), dr.conn_bits.words[lo:hi].cpu().numpy())
        full = (m, syn)
    else:
        ms, ss, drs = m, syn, dr
    model = Model(5)
    model.add_matrix("M", ms, ss)
    drs.register(model, "deep_r", "M")
    res = []
    for u in range(updates):
        if world > 1:
            # the flips are drawn on the full matrix (counter = i*stride + s)
            # and copied to this rank's rows
            full[1].planes["w"][lo:hi].copy_(ss.planes["w"])
            full[0].row_length[lo:hi].copy_(ms.row_length)
            flip(u)
            ss.planes["w"].copy_(full[1].planes["w"][lo:hi])
        else:
            flip(u)
        model.run_update_group("deep_r")
        st = mupdate_state(ms, ss, drs)
        st["removed"] = drs.last_removed
        res.append(st)
    return (lo, hi), res


def mupdate_sharded(rank, world, port, out):
    """Row-sharded DEEP R (gloo, both ranks on cuda:0)."""
    _init(rank, world, port)
    try:
        rng, res = run_mupdate(rank, world, pg=dist.group.WORLD)
        out.put((rank, rng, res))
    finally:
        dist.destroy_process_group()


def form_hist_sharded(rank, world, port, out):
    """Host logic of the row-sharded form pass on CPU (gloo): rank r
    histograms host draws [D*r/W, D*(r+1)/W) over all rows (oracle draw
    arithmetic, deep_r.py:119-120), the histograms are reduce-scattered to
    the row owners.  Returns this rank's rows of the activation histogram."""
    from oracle.rng import draw_u64, fold_key
    from paper_2510_19764_b200.sharding import reduce_scatter_rows, shard_rows
    _init(rank, world, port)
    try:
        res = []
        for P, D in ((1000, 5000), (1 << 12, 777), (37, 3)):
            key = fold_key(9, "host", 1, 2, 0)
            lo, hi = shard_rows(P, rank, world)
            full = torch.zeros(P, dtype=torch.int32)
            for c in range(D * rank // world, D * (rank + 1) // world):
                full[draw_u64(key, c) % P] += 1     # P < 2^32: no rejection
            local = torch.zeros(hi - lo, dtype=torch.int32)
            reduce_scatter_rows(full, local, lo)
            res.append((P, lo, hi, local.numpy().copy()))
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def _init_nccl(rank, world, port):
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)


def nccl_batch_dp(rank, world, port, out):
    """Batch-DP over NCCL (one GPU per rank): gradients all-reduced on the
    device; the ranks must end bit-identical."""
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    from paper_2510_19764_b200.sharding import shard_batch
    _init_nccl(rank, world, port)
    try:
        task = SyntheticTask(num_classes=3, num_inputs=20, example_steps=40, seed=4)
        B = 8
        tr = EpropClassifierTrainer(task, hidden=24, batch_size=B, seed=4, deep_r=True,
                                    input_density=0.3, recurrent_density=0.2,
                                    process_group=dist.group.WORLD, local_batch=shard_batch(B, rank, world))
        hist = [tr.train_batch(k) for k in range(2)]
        out.put((rank, [(h["loss"], h["removed"]) for h in hist], tr.s_in.planes["w"].cpu().numpy(),
                 hashlib.sha256(tr.connectivity_fingerprint()).hexdigest()))
    finally:
        dist.destroy_process_group()


def nccl_topomap(rank, world, port, out):
    """Postsynaptically sharded topomap over NCCL with the rewiring period
    captured in a CUDA graph (spike all-gather as a graph node)."""
    from paper_2510_19764_b200.topomap import TopomapModel
    _init_nccl(rank, world, port)
    try:
        m = TopomapModel(1, seed=4, record_events=False, use_graph=True, process_group=dist.group.WORLD)
        m.run(50.0)
        st = m.state_arrays()
        out.put((rank, {k: st[k] for k in st if k != "V"}, st["V"], (m.post_lo, m.post_hi), len(m._graphs)))
    finally:
        dist.destroy_process_group()
