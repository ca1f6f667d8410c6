"""World-size-2 gloo tests of the multi-GPU decomposition on CPU:

* target-spike all-gather of the postsynaptic topomap sharding;
* batch-DP e-prop: sharded gradients all-reduced, then identical update and
  DEEP R rewiring on every rank (connectivity identical across ranks);
* postsynaptically sharded topomap stepping == the unsharded run.
"""

import queue
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import mp_workers


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2, timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            item = q.get(timeout=timeout)
            res[item[0]] = item[1:]
    except queue.Empty:
        pass
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert len(res) == world, f"workers failed: {[p.exitcode for p in procs]}"
    return res


def test_spike_gather_two_ranks():
    res = _run(mp_workers.spike_gather)
    assert all(v[0] == "ok" for v in res.values())


def test_batch_dp_gradients_and_identical_rewiring():
    from oracle.classifier import eprop_accumulate
    res = _run(mp_workers.batch_dp)
    g0, h0, rem0 = res[0]
    g1, h1, rem1 = res[1]
    assert np.array_equal(g0, g1)            # same reduced bits on both ranks
    assert h0 == h1 and rem0 == rem1          # identical connectivity after DEEP R
    assert rem0 > 0
    # the sharded sum equals the reference's sequential replica sum to rounding
    from oracle.ragged import Ragged
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
    eps = np.zeros((B, P, cap), np.float32)
    ebar = np.zeros_like(eps)
    for t in range(T):
        eprop_accumulate(m.target, m.row_length, trace[t], psi[t], lsig[t], eps, ebar,
                         m.planes["grad"], 0.07, 0.95, 0.9)
    assert np.allclose(g0, m.planes["grad"], rtol=1e-12, atol=1e-13)


def test_topomap_post_sharding_matches_unsharded():
    ref = mp_workers.run_topomap(0, 1, steps=400)
    res = _run(mp_workers.topomap_sharded, timeout=600)
    for r, (st,) in res.items():
        lo, hi = st["range"]
        for k in ref:
            if k in ("V", "range"):
                continue
            assert np.array_equal(st[k], ref[k]), (r, k)
        assert np.array_equal(st["V"][lo:hi], ref["V"][lo:hi]), r
    # the run exercised rewiring and spikes
    assert ref["ff.y"].sum() > 0


def test_row_sharded_form_histogram_two_ranks():
    """M-update row sharding: per-rank counter chunks of the
    host draws, reduce-scattered by row owner == the serial histogram of
    deep_r.py:119-120 (oracle stream)."""
    from oracle.rng import Stream, fold_key
    res = _run(mp_workers.form_hist_sharded)
    for k, (P, D) in enumerate(((1000, 5000), (1 << 12, 777), (37, 3))):
        rng = Stream(fold_key(9, "host", 1, 2, 0))
        ref = np.zeros(P, dtype=np.int32)
        for _ in range(D):
            ref[rng.uniform_int(P)] += 1
        got = np.zeros(P, dtype=np.int32)
        for r in range(2):
            P_, lo, hi, local = res[r][0][k]
            got[lo:hi] = local
        assert np.array_equal(got, ref)
