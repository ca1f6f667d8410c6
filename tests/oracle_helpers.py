"""Shared helpers: rebuild oracle / device objects from golden fixture arrays."""

from __future__ import annotations

import numpy as np

from oracle.deep_r import DeepROracle
from oracle.ragged import Ragged
from oracle.updates import OracleModel

PLANES = ("w", "grad", "adam_m", "adam_v")


def oracle_deepr_from_fixture(fx, seed_override=None):
    P, N, cap, diag, cycles, seed = (int(x) for x in fx["meta"])
    m = Ragged(P, N, cap, PLANES)
    m.row_length[:] = fx["init_row_length"]
    m.target[:] = fx["init_target"]
    for p in PLANES:
        m.planes[p][:] = fx[f"init_{p}"]
    dr = DeepROracle(m, l1=0.005, exclude_diagonal=bool(diag))
    dr.sign[:] = fx["init_sign"]
    dr.conn[:] = fx["init_conn"]
    model = OracleModel(seed if seed_override is None else seed_override)
    model.add_matrix("sg", m)
    dr.register(model, "deep_r", "sg")
    return model, m, dr, cycles


def valid_equal(row_length, a, b):
    """Compare [P, cap] arrays on valid slots only."""
    mask = np.arange(a.shape[1])[None, :] < row_length[:, None]
    return np.array_equal(a[mask], b[mask])
