"""Topomap x-realtime sweep; PERSIST=1 routes every sheet size through the
persistent multi-step launch (sw_topomap_run_steps)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_19764_b200 import topomap  # noqa: E402

if os.environ.get("PERSIST") == "1":
    topomap.PERSISTENT_MAX_NODES = 1 << 30
r = bench.run_topomap_sweep(scales=tuple(int(x) for x in os.environ.get("SCALES", "1,2,4,8,16").split(",")))
print(json.dumps({k: (v["x_realtime"], v["us_per_step"]) for k, v in r.items()}))
