"""C1/C2 grouped forward launches (EPROP_BLOCK_STEPS steps each, plus their
readout launches) up to mid-trial, for ncu:
  -k regex:"k_clf_fwd2|k_clf_readout" -s $((2*T0/K)) -c 2
T0 (env, default 400): timesteps run before the profiled group, so that the
hidden layer's spike activity is the trial's steady state."""
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
T0 = int(os.environ.get("T0", "400"))
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1, use_graph=False)
tr._upload_batch(task.train_ids(0, 512))
tr._prepare(False)
for t0 in range(0, T0 + K, K):
    prm = tr._group_params(t0, K)
    _lib.call("sw_clf_step", ctypes.byref(prm), _lib.stream_ptr())
torch.cuda.synchronize()
z = tr.z.float().mean().item()
print("done; hidden spike fraction at the last step", z)
