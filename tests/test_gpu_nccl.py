"""NCCL paths on >= 2 GPUs (skipped on a 1-GPU box): batch-DP
gradients all-reduced on the device, and the postsynaptically sharded
topomap with the rewiring period (per-step spike all-gather included)
captured in a CUDA graph, against the unsharded single-GPU run."""

import numpy as np
import pytest
import torch

import mp_workers
from test_multiproc import _run

pytestmark = pytest.mark.gpu

need2 = pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                           reason="needs two GPUs (NCCL ranks cannot share a device)")


@need2
def test_nccl_batch_dp_ranks_identical(dev_lib):
    res = _run(mp_workers.nccl_batch_dp, timeout=600)
    (h0, w0, c0), (h1, w1, c1) = res[0], res[1]
    assert h0 == h1 and c0 == c1
    assert np.array_equal(w0, w1)


@need2
def test_nccl_sharded_topomap_graph_equals_unsharded(dev_lib):
    from paper_2510_19764_b200.topomap import TopomapModel
    ref = TopomapModel(1, seed=4, record_events=False, use_graph=True)
    ref.run(50.0)
    rs = ref.state_arrays()
    res = _run(mp_workers.nccl_topomap, timeout=600)
    for r, (st, V, (lo, hi), graphs) in res.items():
        assert graphs > 0
        for k, v in st.items():
            assert np.array_equal(v, rs[k]), (r, k)
        assert np.array_equal(V[lo:hi], rs["V"][lo:hi]), r
