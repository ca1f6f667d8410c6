"""Trial-graph timing: forward only (learn=False), full trial with and
without the two-stream overlap, and the e-prop passes alone."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200.classifier import (EPROP_BLOCK_STEPS, EpropClassifierTrainer,  # noqa: E402
                                              SyntheticTask)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(reps):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / reps


wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
H, dens = (256, 0.1) if wl == "c1" else (1024, 0.01)
task = SyntheticTask(num_classes=20, num_inputs=700, example_steps=1000, seed=1, num_train=8156)
tr = EpropClassifierTrainer(task, hidden=H, input_density=dens, recurrent_density=dens,
                            batch_size=512, seed=1)
tr.train_batch(0)
for ov in (True, False):
    tr.overlap = ov
    tr._graph = None
    print(f"{wl} trial graph learn overlap={ov}: {timed(lambda: tr._run_trial(True)):.2f} ms")
tr._graph = None
print(f"{wl} trial graph forward only: {timed(lambda: tr._run_trial(False)):.2f} ms")
n = task.example_steps // EPROP_BLOCK_STEPS
g = tr.eprop_pass_graph(n)
print(f"{wl} {n} e-prop passes alone: {timed(g.replay):.2f} ms")
