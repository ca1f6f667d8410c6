"""Golden connectivity snapshot CSV from the REAL reference
(sparsewire/connectivity.py:265-283, write_snapshot_csv) for the matrix of
transpose_prop.npz.  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_snapshot_csv.py
"""
import io
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from sparsewire.connectivity import RaggedMatrix, SynVarMatrix, write_snapshot_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
g = np.load(os.path.join(HERE, "transpose_prop.npz"))
P, cap = g["target"].shape
m = RaggedMatrix(P, 40, cap)
m.row_length[:] = g["row_length"]
m.target[:] = g["target"]
syn = SynVarMatrix(m, ("g",))
syn.planes["g"][:] = g["g"]
buf = io.StringIO()
write_snapshot_csv(buf, m, syn)
with open(os.path.join(HERE, "snapshot_transpose_prop.csv"), "w") as fh:
    fh.write(buf.getvalue())
print(buf.getvalue().count("\n"), "lines")
