"""Event-driven atomic propagation (connectivity.py:139-148) at sizes that
take the cluster / shared-memory-slab kernel, against np.add.at.

Dyadic weights make every summation order exact (the reference's own
strategy, pkg/tests/test_connectivity.py:147-187), so the check is
bit-exact; general float64 weights are checked to a relative 1e-12."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _matrix(P, N, cap, seed):
    from paper_2510_19764_b200.connectivity import RaggedMatrix, SynVarMatrix
    rs = np.random.default_rng(seed)
    rl = rs.integers(0, cap + 1, size=P).astype(np.int32)
    tgt = np.zeros((P, max(cap, 1)), dtype=np.int32)
    for i in range(P):
        tgt[i, :rl[i]] = rs.choice(N, size=rl[i], replace=False)
    m = RaggedMatrix(P, N, cap)
    syn = SynVarMatrix(m, ("g",))
    m.load_state(rl, tgt)
    return m, syn, rl, tgt, rs


@pytest.mark.parametrize("P,N,cap,q,dyadic", [
    (6000, 65536, 300, 0.6, True),      # cluster kernel, all four slabs, multi-chunk rows
    (5000, 40000, 41, 0.9, True),       # odd stride, last slab partial
    (4000, 3000, 64, 0.7, False),       # small output, general weights
    (3000, 70000, 32, 0.9, True),       # num_post > 65536: warp-per-row kernel
    (500, 65536, 128, 0.5, True),       # few spiking rows: warp-per-row kernel
])
def test_atomic_propagation_matches_add_at(dev_lib, P, N, cap, q, dyadic):
    from paper_2510_19764_b200.connectivity import propagate_spikes
    m, syn, rl, tgt, rs = _matrix(P, N, cap, 11)
    if dyadic:
        w = rs.integers(-64, 65, size=tgt.shape).astype(np.float64) / 64.0
    else:
        w = rs.standard_normal(tgt.shape)
    syn.planes["g"].copy_(torch.from_numpy(w))
    spikes = np.flatnonzero(rs.random(P) < q).astype(np.int32)
    ref = rs.standard_normal(N)
    out = torch.from_numpy(ref.copy()).cuda()
    for i in spikes:                                   # connectivity.py:146-148
        np.add.at(ref, tgt[i, :rl[i]], w[i, :rl[i]])
    propagate_spikes(m, syn.planes["g"], torch.from_numpy(spikes).cuda(), out)
    got = out.cpu().numpy()
    if dyadic:
        # the random base is not dyadic: order can move the last bit of the sum
        assert np.allclose(got, ref, rtol=0, atol=1e-12)
    else:
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_atomic_propagation_dyadic_exact_from_zero(dev_lib):
    from paper_2510_19764_b200.connectivity import propagate_spikes
    P, N, cap = 8000, 65536, 512
    m, syn, rl, tgt, rs = _matrix(P, N, cap, 5)
    w = rs.integers(-1024, 1025, size=tgt.shape).astype(np.float64) / 1024.0
    syn.planes["g"].copy_(torch.from_numpy(w))
    spikes = np.flatnonzero(rs.random(P) < 0.5).astype(np.int32)
    ref = np.zeros(N)
    for i in spikes:
        np.add.at(ref, tgt[i, :rl[i]], w[i, :rl[i]])
    out = torch.zeros(N, dtype=torch.float64, device="cuda")
    propagate_spikes(m, syn.planes["g"], torch.from_numpy(spikes).cuda(), out)
    assert np.array_equal(out.cpu().numpy(), ref)


def test_single_synapse_edits_match_reference_semantics(dev_lib):
    """add_synapse / remove_synapse / remove_slots (connectivity.py:91-136)
    against the oracle on a random operation sequence; the reference's own
    known answers (pkg/tests/test_connectivity.py:54-61: [2,0,3] remove slot
    0 -> [3,0]) included."""
    from oracle.ragged import Ragged
    from paper_2510_19764_b200.connectivity import (RaggedMatrix, SynVarMatrix, add_synapse,
                                                    remove_slots, remove_synapse)
    from paper_2510_19764_b200.errors import DuplicateEdge, RowFull, SlotOutOfRange
    m = RaggedMatrix(3, 5, 4)
    syn = SynVarMatrix(m, ("g",))
    for post in (2, 0, 3):
        add_synapse(m, syn, 0, post, {"g": float(post)})
    remove_synapse(m, syn, 0, 0)
    assert m.row_targets(0).cpu().tolist() == [3, 0]
    assert syn.planes["g"][0, :2].cpu().tolist() == [3.0, 0.0]
    with pytest.raises(DuplicateEdge):
        add_synapse(m, syn, 0, 3)
    with pytest.raises(SlotOutOfRange):
        remove_synapse(m, syn, 0, 2)

    rs = np.random.default_rng(9)
    P, N, cap = 20, 30, 12
    m = RaggedMatrix(P, N, cap)
    syn = SynVarMatrix(m, ("w", "g"))
    o = Ragged(P, N, cap, ("w", "g"))
    for _ in range(600):
        i = int(rs.integers(P))
        op = rs.random()
        if op < 0.55:
            j = int(rs.integers(N))
            v = {"w": float(rs.standard_normal())}
            err_o = err_d = None
            try:
                so = o.add_synapse(i, j, v)
            except Exception as e:   # oracle RowFull / DuplicateEdge
                err_o = type(e).__name__
            try:
                sd = add_synapse(m, syn, i, j, v)
            except (RowFull, DuplicateEdge) as e:
                err_d = type(e).__name__
            assert (err_o is None) == (err_d is None)
            if err_o is None:
                assert so == sd
        elif op < 0.8 and o.row_length[i] > 0:
            s = int(rs.integers(o.row_length[i]))
            o.remove_synapse(i, s)
            remove_synapse(m, syn, i, s)
        elif o.row_length[i] > 0:
            k = int(rs.integers(1, o.row_length[i] + 1))
            sl = rs.choice(int(o.row_length[i]), size=k, replace=False)
            o.remove_slots(i, sl)
            remove_slots(m, syn, i, sl)
    rl = o.row_length
    assert np.array_equal(m.row_length.cpu().numpy(), rl)
    mask = np.arange(cap)[None, :] < rl[:, None]
    assert np.array_equal(m.target.cpu().numpy()[mask], o.target[mask])
    for p in ("w", "g"):
        assert np.array_equal(syn.planes[p].cpu().numpy()[mask], o.planes[p][mask])


@pytest.mark.parametrize("P,N,cap,q", [
    (6000, 65536, 300, 0.6),      # 4 slabs, multi-chunk rows
    (5000, 40000, 41, 0.9),       # odd stride, 3 slabs, last one partial
    (4000, 3000, 64, 0.7),        # one slab smaller than 16384
    (3000, 131072, 96, 0.5),      # 8 slabs
    (400, 65536, 1024, 0.01),     # full-capacity rows, very few spikes
])
def test_bucketed_propagation_matches_add_at(dev_lib, P, N, cap, q):
    """Post-slab bucketed rows (sw_prop_buckets_build / sw_propagate_bucketed):
    the layout is a stable per-slab regrouping of every row, and the
    propagation equals np.add.at exactly for dyadic weights from zero."""
    from paper_2510_19764_b200.connectivity import PropBuckets, propagate_spikes
    m, syn, rl, tgt, rs = _matrix(P, N, cap, 23)
    w = rs.integers(-64, 65, size=tgt.shape).astype(np.float64) / 64.0
    syn.planes["g"].copy_(torch.from_numpy(w))
    pb = PropBuckets(m, syn.planes["g"])
    pb.MIN_SPIKES = 0                  # the bucketed kernel at every size
    G = pb.slabs
    assert G == -(-N // 16384)
    stride = m.stride
    bt = pb.bt.cpu().numpy().view(np.uint16).reshape(P, stride)
    bs = pb.bslot.cpu().numpy().view(np.uint16).reshape(P, stride)
    bw = pb.bw.cpu().numpy().reshape(P, stride)
    so = pb.soff.cpu().numpy().view(np.uint16).reshape(P, G + 1)
    for i in rs.choice(P, 60, replace=False):
        n = rl[i]
        assert so[i, 0] == 0 and so[i, G] == n
        slots = bs[i, :n].astype(np.int64)
        assert np.array_equal(np.sort(slots), np.arange(n))
        for j in range(G):
            a, b = so[i, j], so[i, j + 1]
            sl = slots[a:b]
            assert np.all(np.diff(sl) > 0)                       # slot order within a slab
            assert np.all(tgt[i, sl] // 16384 == j)
            assert np.array_equal(bt[i, a:b].astype(np.int64) + j * 16384, tgt[i, sl])
            assert np.array_equal(bw[i, a:b], w[i, sl])
    spikes = np.flatnonzero(rs.random(P) < q).astype(np.int32)
    ref = np.zeros(N)
    for i in spikes:
        np.add.at(ref, tgt[i, :rl[i]], w[i, :rl[i]])
    out = torch.zeros(N, dtype=torch.float64, device="cuda")
    propagate_spikes(m, syn.planes["g"], torch.from_numpy(spikes).cuda(), out, buckets=pb)
    assert np.array_equal(out.cpu().numpy(), ref)
    # weight-only change: refresh, then general weights to 1e-12
    w2 = rs.standard_normal(tgt.shape)
    syn.planes["g"].copy_(torch.from_numpy(w2))
    pb.refresh()
    ref2 = rs.standard_normal(N)
    out2 = torch.from_numpy(ref2.copy()).cuda()
    for i in spikes:
        np.add.at(ref2, tgt[i, :rl[i]], w2[i, :rl[i]])
    propagate_spikes(m, syn.planes["g"], torch.from_numpy(spikes).cuda(), out2, buckets=pb)
    assert np.allclose(out2.cpu().numpy(), ref2, rtol=1e-12, atol=1e-12)


def test_bucketed_propagation_goes_stale(dev_lib):
    from paper_2510_19764_b200.connectivity import PropBuckets, add_synapse, propagate_spikes
    from paper_2510_19764_b200.errors import StaleTranspose
    m, syn, rl, tgt, rs = _matrix(200, 5000, 16, 3)
    pb = PropBuckets(m, syn.planes["g"])
    row = int(np.flatnonzero(rl < 16)[0])
    add_synapse(m, syn, row, int(np.setdiff1d(np.arange(5000), tgt[row, :rl[row]])[0]))
    out = torch.zeros(5000, dtype=torch.float64, device="cuda")
    with pytest.raises(StaleTranspose):
        propagate_spikes(m, syn.planes["g"], torch.tensor([row]).cuda(), out, buckets=pb)
    pb.build()
    propagate_spikes(m, syn.planes["g"], torch.tensor([row]).cuda(), out, buckets=pb)


def test_bucketed_kernels_share_one_weight_snapshot(dev_lib):
    """PropBuckets.propagate picks its kernel from the spike count;
    both must read the snapshot taken at build()/refresh(), so an in-place
    weight change without refresh() affects neither, and after refresh()
    both see it.  Dyadic weights: exact against np.add.at."""
    from paper_2510_19764_b200.connectivity import PropBuckets
    P, N = 6000, 40000
    m, syn, rl, tgt, rs = _matrix(P, N, 64, 5)
    w = rs.integers(-64, 65, size=tgt.shape).astype(np.float64) / 64.0
    syn.planes["g"].copy_(torch.from_numpy(w))
    pb = PropBuckets(m, syn.planes["g"])
    syn.planes["g"].mul_(2.0)                     # not yet refreshed
    few = np.flatnonzero(rs.random(P) < 0.05).astype(np.int32)
    many = np.flatnonzero(rs.random(P) < 0.9).astype(np.int32)
    assert few.size < pb.MIN_SPIKES <= many.size
    for scale in (1.0, 2.0):
        for sp in (few, many):
            ref = np.zeros(N)
            for i in sp:
                np.add.at(ref, tgt[i, :rl[i]], scale * w[i, :rl[i]])
            out = torch.zeros(N, dtype=torch.float64, device="cuda")
            d = torch.from_numpy(sp).cuda()
            kern = pb.propagate(d, torch.tensor([sp.size], dtype=torch.int32, device="cuda"), sp.size, out)
            assert kern == ("atomic" if sp is few else "bucketed")
            assert np.array_equal(out.cpu().numpy(), ref), (scale, kern)
        pb.refresh()


@pytest.mark.parametrize("cfg", ["32x4x2", "16x8x2"])
def test_bucketed_propagation_variants(cfg):
    """The non-default k_prop_bucketed shapes behind the SW_PROP_BCFG
    measurement knob (read once per process, so each runs in a child):
    dyadic weights, exact against np.add.at."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import test_gpu_propagate as t\n"
        "t.test_bucketed_propagation_matches_add_at(None, 6000, 65536, 300, 0.6)\n"
        "t.test_bucketed_propagation_matches_add_at(None, 400, 65536, 1024, 0.01)\n"
        "print('ok')\n" % (root, os.path.join(root, "tests")))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SW_PROP_BCFG=cfg),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_explicit_capacity_never_truncates_rows(dev_lib):
    """init_pairwise_bernoulli_density with an explicit capacity
    below the realised maximum row length raises RowFull instead of silently
    dropping synapses; a sufficient capacity keeps every drawn synapse."""
    from paper_2510_19764_b200.connectivity import init_pairwise_bernoulli_density
    from paper_2510_19764_b200.errors import RowFull
    from paper_2510_19764_b200.rng import CounterRng
    m, _ = init_pairwise_bernoulli_density(300, 400, 0.2, 1.0, CounterRng(2, "init", "cap"))
    mx = int(m.row_length.max())
    with pytest.raises(RowFull):
        init_pairwise_bernoulli_density(300, 400, 0.2, 1.0, CounterRng(2, "init", "cap"), capacity=mx - 1)
    m2, _ = init_pairwise_bernoulli_density(300, 400, 0.2, 1.0, CounterRng(2, "init", "cap"), capacity=mx)
    assert torch.equal(m2.row_length, m.row_length)
