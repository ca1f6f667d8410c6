"""Profiling driver: one C1 training batch (CUDA graph), then N eager launches
of the fused e-prop step on the live state.  Under ncu use
  -k regex:k_eprop_fused -s 1000 -c 3
to skip the batch's graph launches."""
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
tr.train_batch(0)
p = tr.params
a32, r32, b32 = (float(np.float32(x)) for x in (p.alpha, p.rho, p.beta))
segs = (_lib.EpropSeg * 2)()
segs[0] = tr.plan_in.seg(tr.xbar)
segs[1] = tr.plan_rec.seg(tr.zbar)
for _ in range(int(os.environ.get("REPS", "3"))):
    _lib.call("sw_eprop_fused_step", ctypes.cast(segs, ctypes.c_void_p), 2, tr.psi.data_ptr(),
              tr.lsig.data_ptr(), tr.local_b, tr.hidden, b32, r32, a32, tr.d.data_ptr(),
              tr.zbar.data_ptr(), tr.g_w_out.data_ptr(), tr.g_b_out.data_ptr(), 20,
              0, _lib.workspace(), _lib.stream_ptr())
torch.cuda.synchronize()
print("done", tr.m_in.edge_count(), tr.m_rec.edge_count())
