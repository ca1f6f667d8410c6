"""Per-component timing of one e-prop group (K steps) on a trained C1/C2
state: sw_eprop_prep, sw_eprop_pass, the readout launch, each replayed REPS
times from a CUDA graph.  Usage: python tools/eprop_breakdown.py [c1|c2]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.classifier import EPROP_BLOCK_STEPS, EpropClassifierTrainer, SyntheticTask  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1)
tr.train_batch(0)
torch.cuda.synchronize()
K = EPROP_BLOCK_STEPS
reps = int(os.environ.get("REPS", "50"))
calls = []
orig = _lib.call


def rec(name, *args):
    calls.append((name, args))
    return orig(name, *args)


_lib.call = rec
tr._eprop_block(0, K, _lib.stream_ptr(), state_zero=False)
_lib.call = orig
torch.cuda.synchronize()
# keep the ctypes argument objects alive: re-run the recorded calls
res = {}
for name, args in calls:
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            st = torch.cuda.current_stream().cuda_stream
            for _ in range(reps):
                orig(name, *args[:-1], st)
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    g.replay()
    e[1].record()
    torch.cuda.synchronize()
    res[name] = e[0].elapsed_time(e[1]) * 1e3 / reps
E = tr.m_in.edge_count() + tr.m_rec.edge_count()
for k, v in res.items():
    print(f"{wl} {k}: {v:.1f} us")
us = res.get("sw_eprop_pass", 0)
if us:
    alg = 512 * E * 16 + E * 20 + K * 512 * (700 + 3 * H) * 4
    print(f"pass: {alg / (us * 1e-6) / 1e9:.0f} GB/s algorithmic, E={E}")
