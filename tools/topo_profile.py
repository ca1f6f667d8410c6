"""One topomap sheet for an ncu launch list: build, warm up, then run
MODEL_MS of model time (graph replays).  SCALE env (default 16)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200.topomap import TopomapModel  # noqa: E402

s = int(os.environ.get("SCALE", "16"))
model = TopomapModel(s, seed=1, record_events=False, use_graph=True, rates_on_device=True)
model.run(10.0)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
rec = model.run(float(os.environ.get("MODEL_MS", "5")))
e[1].record()
torch.cuda.synchronize()
print("us/step", e[0].elapsed_time(e[1]) * 1e3 / rec.steps)
