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
