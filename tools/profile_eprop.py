"""Profiling driver: one training batch (CUDA graph), then REPS eager launches
of the blocked e-prop pass (EPROP_BLOCK_STEPS timesteps) on the live state.
Timing: REPS passes captured in one CUDA graph (no host overhead).  Under ncu
set EAGER=1 (plain launches) and use
  -k regex:k_eprop_block -s 5 -c 1"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.classifier import (EPROP_BLOCK_STEPS, EpropClassifierTrainer,  # noqa: E402
                                              SyntheticTask)

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1)
tr.train_batch(0)
reps = int(os.environ.get("REPS", "3"))
if os.environ.get("EAGER"):
    st = _lib.stream_ptr()
    for _ in range(reps):
        tr._eprop_block(0, EPROP_BLOCK_STEPS, st, state_zero=False)
    torch.cuda.synchronize()
    print("eager launches done")
    sys.exit(0)
g = tr.eprop_pass_graph(reps)
g.replay()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
g.replay()
ev[1].record()
torch.cuda.synchronize()
print("done", tr.m_in.edge_count(), tr.m_rec.edge_count(), "us/launch", ev[0].elapsed_time(ev[1]) * 1e3 / reps)
