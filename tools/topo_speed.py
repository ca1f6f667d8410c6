"""Topomap x realtime per scale, exactly as bench.py measures it
(run_topomap_sweep): python tools/topo_speed.py [scales...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

scales = tuple(int(x) for x in sys.argv[1:]) or (1, 2, 4, 8, 16)
for k, v in bench.run_topomap_sweep(scales).items():
    print(k, json.dumps(v))
