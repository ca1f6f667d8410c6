"""Per-GPU cost of a batch-DP rank: one trainer at the local batch B/N on one
GPU (the work rank r does between the all-reduces), ms per batch of 1000-step
trials, resident inputs.  python tools/local_batch_time.py [c1|c2] [B ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
for B in [int(x) for x in sys.argv[2:]] or [512, 256, 128, 64]:
    task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
    tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                                batch_size=B, seed=1)
    host = [tr.host_inputs(b) for b in range(5)]   # host-side example draws, untimed
    for b in range(2):
        tr.train_batch(b, host=host[b])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for b in range(2, 5):
        tr.train_batch(b, host=host[b])
    e1.record()
    e1.synchronize()
    print(f"{wl} B={B}: {e0.elapsed_time(e1) / 3:.2f} ms per batch")
    del tr
    torch.cuda.empty_cache()
