"""Time the grouped forward + readout launches (EPROP_BLOCK_STEPS steps) of
C1/C2 mid-trial: steps 0..400 run first, then the rest of the trial is
timed with CUDA events.
Usage: python tools/fwd_time.py [c1|c2]   (SW_CLF_KERNEL=staged: old kernel)"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.classifier import EPROP_BLOCK_STEPS as K  # noqa: E402
from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1, use_graph=False)
tr._upload_batch(task.train_ids(0, 512))
tr._prepare(False)
st = _lib.stream_ptr()
for t0 in range(0, 400, K):
    _lib.call("sw_clf_step", ctypes.byref(tr._group_params(t0, K)), st)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
n = 0
for t0 in range(400, 1000 - K + 1, K):
    _lib.call("sw_clf_step", ctypes.byref(tr._group_params(t0, K)), st)
    n += 1
ev[1].record()
torch.cuda.synchronize()
us = ev[0].elapsed_time(ev[1]) * 1e3 / n
print(f"{wl} forward+readout: {us:.1f} us per {K}-step group, {us / K:.2f} us/step; "
      f"hidden spike fraction {tr.z.float().mean().item():.4f}")
