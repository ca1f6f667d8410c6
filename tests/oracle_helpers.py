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


def oracle_topomap_group(fx, k):
    """Oracle rewiring group (ff rule id 0, lat rule id 1) loaded with the
    pre-update state of update k of a topomap fixture."""
    from oracle.topomap import RewiringOracle
    scale, seed = (int(x) for x in fx["meta"])
    side = 16 * scale
    model = OracleModel(seed)
    rules = {}
    for name in ("ff", "lat"):
        tg = fx[f"u{k}_pre_{name}_target"]
        N = side * side
        m = Ragged(N, N, tg.shape[1], ("g",))
        m.row_length[:] = fx[f"u{k}_pre_{name}_row_length"]
        m.target[:] = tg
        m.planes["g"][:] = fx[f"u{k}_pre_{name}_g"]
        model.add_matrix(name, m)
        r = RewiringOracle(m, side, fx[f"{name}_lut"], fx["dist"], 10 * scale * scale)
        model.add_rule("rewiring", name, r)
        rules[name] = (m, r)
    for b, u in zip(model.groups["rewiring"], fx[f"u{k}_pre_updates"]):
        b.update_count = int(u)
    return model, rules


def check_topomap_post(fx, k, name, row_length, target, g):
    rl = fx[f"u{k}_post_{name}_row_length"]
    assert np.array_equal(row_length, rl), (k, name)
    assert valid_equal(rl, target, fx[f"u{k}_post_{name}_target"]), (k, name)
    assert valid_equal(rl, g, fx[f"u{k}_post_{name}_g"]), (k, name)


def fwd_groups(H: int) -> int:
    """Row groups of the forward kernels' event-driven current sums
    (classifier_fwd.cu fwd_groups, classifier_fwd2.cu fwd2_groups)."""
    return 8 if H <= 256 else 4


def grouped_currents(rl, tg, w32, spiking, H):
    """The forward kernel's per-post float32 current (classifier_fwd.cu P2c):
    the ascending spiking rows split into G contiguous groups (group g =
    rows[n*g//G : n*(g+1)//G]), each summed sequentially from +0.0, the group
    sums added in group order.  spiking: [B, P] bool -> [B, H] float32."""
    import numpy as np
    F = np.float32
    G = fwd_groups(H)
    B = spiking.shape[0]
    out = np.zeros((B, H), F)
    for b in range(B):
        rows = np.flatnonzero(spiking[b])
        n = rows.size
        acc = None
        for g in range(G):
            part = np.zeros(H, F)
            for i in rows[n * g // G:n * (g + 1) // G]:
                k = int(rl[i])
                if k:
                    part[tg[i, :k]] = part[tg[i, :k]] + w32[i, :k]
            acc = part if acc is None else (acc + part).astype(F)
        out[b] = acc
    return out
