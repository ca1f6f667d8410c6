"""Microbenchmark sharding on the device:

* M-update rows sharded: two ranks (gloo, both on cuda:0) each own half the
  rows of a DEEP R matrix; the form pass's host draws are split into counter
  chunks, histogrammed per rank and reduce-scattered to the row owners.  The
  result must be bit-identical to the unsharded device run (which the other
  GPU tests pin to the reference), update after update;
* M-prop posts sharded: every rank propagates over its column slice of the
  matrix (no collective); the owned posts' sums are bit-identical to the
  unsharded ordered propagation (connectivity.py:139-148 order)."""

import numpy as np
import pytest
import torch

import mp_workers
from test_multiproc import _run

pytestmark = pytest.mark.gpu


def test_mupdate_row_sharded_equals_unsharded(dev_lib):
    _, ref = mp_workers.run_mupdate(0, 1)
    res = _run(mp_workers.mupdate_sharded, timeout=600)
    assert sum(s["removed"] for s in ref) > 0
    for r, ((lo, hi), states) in res.items():
        for u, (a, b) in enumerate(zip(states, ref)):
            assert a["removed"] == b["removed"], (r, u)
            for k in ("row_length", "target", "w", "conn", "sign"):
                assert np.array_equal(a[k], b[k][lo:hi]), (r, u, k)


@pytest.mark.parametrize("world", [2, 3])
def test_mprop_post_sharded_ordered_bit_exact(dev_lib, world):
    from paper_2510_19764_b200.connectivity import column_slice, propagate_spikes
    from paper_2510_19764_b200.sharding import shard_posts
    from paper_2510_19764_b200.transpose import remap_transpose
    m, syn, _, _ = mp_workers.mupdate_instance(P=3000, N=5000)
    w = syn.planes["w"]
    rs = np.random.default_rng(2)
    spikes = torch.from_numpy(np.flatnonzero(rs.random(m.num_pre) < 0.05).astype(np.int32)).cuda()
    full = torch.zeros(m.num_post, dtype=torch.float64, device="cuda")
    propagate_spikes(m, w, spikes, full, tmap=remap_transpose(m))
    got = torch.zeros_like(full)
    for r in range(world):
        lo, hi = shard_posts(m.num_post, r, world)
        ms, ss = column_slice(m, syn, lo, hi)
        assert ms.edge_count() == int(((m.target >= lo) & (m.target < hi) & m.slot_mask()).sum())
        part = torch.zeros(hi - lo, dtype=torch.float64, device="cuda")
        propagate_spikes(ms, ss.planes["w"], spikes, part, tmap=remap_transpose(ms))
        got[lo:hi] = part
    assert torch.equal(got, full)
