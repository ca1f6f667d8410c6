"""(Build with SW_NVCC_EXTRA=-DSW_FWD_PROF.)  Phase timestamps (clock64) of one forward block (block 7, step 3 of a
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
L.sw_debug_fwd2_prof.argtypes = [ctypes.c_int, ctypes.c_void_p]
# grouped launches with precomputed inputs run k_clf_fwd2
prof = L.sw_debug_fwd2_prof
tr._prepare(False)
st = _lib.stream_ptr()
for t0 in range(0, 400, 8):
    _lib.call("sw_clf_step", ctypes.byref(tr._group_params(t0, 8)), st)   # steady state
torch.cuda.synchronize()
# markers of k_clf_fwd2 (FWD2_PROF): 0 step start, 1 after B1, 4 rows
# selected, 5 row sums done, 6 after B3, 7 step end (2, 3 unused)
names = ["start", "B1", "-", "-", "selected", "summed", "B3", "end"]
acc = {}
for rep in range(10):
    prof(1, None)
    _lib.call("sw_clf_step", ctypes.byref(tr._group_params(400 + 8 * rep, 8)), st)
    torch.cuda.synchronize()
    out = (ctypes.c_longlong * 64)()
    prof(0, out)
    t0 = min(out[w] for w in range(8))
    for i in range(8):
        for w in range(8):
            acc.setdefault((i, w), []).append(out[i * 8 + w] - t0)
for i in range(8):
    if names[i] != "-":
        print(f"{names[i]:9s} " + " ".join(f"{sum(acc[(i, w)]) / len(acc[(i, w)]):7.0f}" for w in range(8)))
