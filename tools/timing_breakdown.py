"""Per-phase device timing of one C1/C2 training batch (CUDA events)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1)
for b in range(2):
    tr.train_batch(b)
torch.cuda.synchronize()


def timeit(fn, n=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


print("batch total ms", timeit(lambda: tr.train_batch(2)))
print("graph replay ms", timeit(lambda: tr._graph.replay(), 3))
st = _lib.stream_ptr()
prm = tr._step_params(5)
print("clf_step us", 1000 * timeit(lambda: _lib.call("sw_clf_step", ctypes.byref(prm), st), 200))
p = tr.params
a32, r32, b32 = (float(np.float32(x)) for x in (p.alpha, p.rho, p.beta))
segs = (_lib.EpropSeg * 2)()
segs[0] = tr.plan_in.seg(tr.xbar)
segs[1] = tr.plan_rec.seg(tr.zbar)
ep = lambda: _lib.call("sw_eprop_fused_step", ctypes.cast(segs, ctypes.c_void_p), 2,
                       tr.psi.data_ptr(), tr.lsig.data_ptr(), tr.local_b, tr.hidden, b32, r32,
                       a32, tr.d.data_ptr(), tr.zbar.data_ptr(), tr.g_w_out.data_ptr(),
                       tr.g_b_out.data_ptr(), 20, 0, _lib.workspace(), st)
print("eprop us", 1000 * timeit(ep, 200))
ep_nro = lambda: _lib.call("sw_eprop_fused_step", ctypes.cast(segs, ctypes.c_void_p), 2,
                           tr.psi.data_ptr(), tr.lsig.data_ptr(), tr.local_b, tr.hidden, b32, r32,
                           a32, None, None, None, None, 0, 0, _lib.workspace(), st)
print("eprop (no readout) us", 1000 * timeit(ep_nro, 200))
print("gradient_phase ms", timeit(lambda: tr.gradient_phase(3)))
print("rewire ms", timeit(lambda: tr.rewire_phase()))
L = _lib.lib()
buf = (ctypes.c_longlong * 16)()
L.sw_debug_clf_prof(buf)
v = list(buf)
print("clf phases (cycles from P0):", [v[i] - v[0] for i in range(16)])
