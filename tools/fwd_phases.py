"""Phase timestamps (clock64) of one forward block (block 7, step 3 of a
launch) mid-trial: warp 0 (lane 0) and warp 1.  Usage: python tools/fwd_phases.py [c1|c2]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1, use_graph=False)
tr._upload_batch(task.train_ids(0, 512))
tr._prepare(False)
L = _lib.lib()
L.sw_debug_fwd_prof.argtypes = [ctypes.c_int, ctypes.c_void_p]
st = _lib.stream_ptr()
for t0 in range(0, 400, 8):
    _lib.call("sw_clf_step", ctypes.byref(tr._group_params(t0, 8)), st)
torch.cuda.synchronize()
names = ["step start", "lists ready (B1b)", "staging landed", "input currents", "recurrent currents", "step end"]
acc = {}
for rep in range(10):
    L.sw_debug_fwd_prof(1, None)
    _lib.call("sw_clf_step", ctypes.byref(tr._group_params(400 + 8 * rep, 8)), st)
    torch.cuda.synchronize()
    out = (ctypes.c_longlong * 16)()
    L.sw_debug_fwd_prof(0, out)
    for w in range(2):
        t = [out[i + 8 * w] for i in range(6)]
        for i in range(1, 6):
            acc.setdefault((w, i), []).append(t[i] - t[0])
for w in range(2):
    print(f"warp {w}: " + ", ".join(f"{names[i]} {sum(acc[(w, i)]) / len(acc[(w, i)]):.0f}" for i in range(1, 6)))
