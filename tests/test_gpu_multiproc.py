"""Batch-DP through the device trainer: two ranks share cuda:0
over gloo (CUDA tensors all-reduced through the host), each trains its batch
shard.  The ranks must end bit-identical (same reduced gradient bits, same
update and DEEP R rewiring), and match one unsharded trainer to float64
rounding of the split gradient sums."""

import numpy as np
import pytest

from test_multiproc import _run
import mp_workers

pytestmark = pytest.mark.gpu


def test_device_trainer_batch_dp_two_ranks(dev_lib):
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask
    res = _run(mp_workers.device_trainer_dp, timeout=600)
    (h0, w0, c0), (h1, w1, c1) = res[0], res[1]
    assert h0 == h1 and c0 == c1
    assert np.array_equal(w0, w1)
    task = SyntheticTask(num_classes=3, num_inputs=20, example_steps=40, seed=4)
    tr = EpropClassifierTrainer(task, hidden=24, batch_size=8, seed=4, deep_r=True,
                                input_density=0.3, recurrent_density=0.2)
    hist = [tr.train_batch(k) for k in range(2)]
    for (l_dp, r_dp), h in zip(h0, hist):
        assert abs(l_dp - h["loss"]) <= 1e-9 * max(1.0, abs(h["loss"]))
        assert r_dp == h["removed"]
    assert np.allclose(w0, tr.s_in.planes["w"].cpu().numpy(), rtol=1e-9, atol=1e-12)
