"""Topomap: model.run() time vs back-to-back replays of its largest
multi-period graph (host loop overhead check).  SCALE env."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200.topomap import TopomapModel  # noqa: E402

s = int(os.environ.get("SCALE", "1"))
model = TopomapModel(s, seed=1, record_events=False, use_graph=True, rates_on_device=True)
model.run(10.0)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
t0 = time.perf_counter()
e[0].record()
rec = model.run(100.0)
e[1].record()
torch.cuda.synchronize()
t1 = time.perf_counter()
e[2].record()
periods = max(model._graphs)
for _ in range(100 // periods):
    model._graphs[periods].replay()
e[3].record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"s{s}: run 100 ms: gpu {e[0].elapsed_time(e[1]):.2f} ms host {1e3*(t1-t0):.2f} ms | "
      f"100 raw replays: gpu {e[2].elapsed_time(e[3]):.2f} ms host {1e3*(t2-t1):.2f} ms")
