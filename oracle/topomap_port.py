"""CPU port of the reference topographic-map run loop, for the benchmark's
CPU baseline only (TEST INFRASTRUCTURE: the product never imports oracle/).

Mirrors ``TopomapModel.run`` (sparsewire/topomap.py:398-474) step for step
with the oracle's numpy restatements: Poisson source (neurons.py:189-195),
conductance LIF (neurons.py:137-148), propagate_spikes with np.add.at per
spiking row (connectivity.py:139-148), trace STDP (plasticity.py:64-95), the
rewiring rule every t_rewiring (topomap.py:101-196, RewiringOracle: the
reference's Python row loop) and a transpose rebuild after a structural
change (updates.py:367-372).  Correlated stimulus rates every t_stim
(neurons.py:175-183, same formula).  No recorder (cli.py:181-186)."""

from __future__ import annotations

import math
import time

import numpy as np

from .ragged import init_pairwise_bernoulli, propagate_spikes, transpose
from .rng import Stream
from .topomap import RewiringOracle, StdpOracle, lif_cond_step, poisson_step, torus_offset
from .updates import OracleModel

BASE_SIDE = 16


class TopomapPort:
    def __init__(self, scale: int, seed: int = 1):
        side = BASE_SIDE * scale
        self.side, self.n, self.scale, self.seed = side, side * side, scale, seed
        n = self.n
        gx, gy = np.arange(n) % side, np.arange(n) // side
        self.gx, self.gy = gx.astype(np.float64), gy.astype(np.float64)
        dx = np.minimum(gx, side - gx)
        dy = np.minimum(gy, side - gy)
        dist_lut = np.hypot(dx, dy)
        self.model = OracleModel(seed)
        self.projs = {}
        t0 = time.perf_counter()
        for name, p_form, sigma in (("ff", 0.16, 2.5), ("lat", 1.0, 1.0)):
            lut = p_form * np.exp(-(dist_lut ** 2) / (2 * sigma ** 2))
            m = init_pairwise_bernoulli(n, n, lambda i, cols, lut=lut: lut[torus_offset(i, cols, side)],
                                        4.0, Stream.of(seed, "init", name), planes=("g",))
            m.planes["g"][m.slot_mask()] = 0.2
            self.model.add_matrix(name, m)
            self.model.add_rule("rewiring", name, RewiringOracle(m, side, lut, dist_lut, 10 * scale * scale))
            self.projs[name] = (m, StdpOracle(m, 0.1))
        self.build_s = time.perf_counter() - t0
        self.V = np.full(n, -70.0)
        self.g = np.zeros(n)
        self.ref = np.full(n, -1, dtype=np.int64)
        self.pending = np.zeros(n)
        self.trs = {k: transpose(v[0]) for k, v in self.projs.items()}
        self.poisson = Stream.of(seed, "poisson")
        self.stim = Stream.of(seed, "stimulus")
        self.p_src = None
        self.k = 0

    def _rates(self):
        """neurons.py:175-183: f_base + f_peak * sum of Gaussian bumps around
        scale^2 centres (topomap.py:391-396), toroidal distance."""
        bx = self.stim.uniform01() * BASE_SIDE
        by = self.stim.uniform01() * BASE_SIDE
        side = self.side
        bump = np.zeros(self.n)
        for a in range(self.scale):
            for b in range(self.scale):
                cx, cy = bx + a * BASE_SIDE, by + b * BASE_SIDE
                dx = np.abs(self.gx - cx)
                dy = np.abs(self.gy - cy)
                d = np.hypot(np.minimum(dx, side - dx), np.minimum(dy, side - dy))
                bump += np.exp(-(d * d) / (2.0 * 2.0 ** 2))
        rates = 5.0 + 152.8 * bump
        self.p_src = 1.0 - np.exp(-rates * 0.1 * 1e-3)

    def run(self, duration_ms: float) -> float:
        """Model steps of duration_ms; returns the wall seconds."""
        t0 = time.perf_counter()
        for _ in range(int(round(duration_ms / 0.1))):
            if self.k % 200 == 0:      # t_stim = 20 ms
                self._rates()
            src = poisson_step(self.poisson, self.p_src)
            tgt = lif_cond_step(self.V, self.g, self.ref, self.pending, self.k)
            nxt = np.zeros(self.n)
            propagate_spikes(self.projs["ff"][0], self.projs["ff"][0].planes["g"], src, nxt)
            propagate_spikes(self.projs["lat"][0], self.projs["lat"][0].planes["g"], tgt, nxt)
            self.pending = nxt
            for name in ("ff", "lat"):
                self.projs[name][1].decay()
            if src.size:
                self.projs["ff"][1].on_pre(src)
            if tgt.size:
                self.projs["lat"][1].on_pre(tgt)
                self.projs["ff"][1].on_post(self.trs["ff"], tgt)
                self.projs["lat"][1].on_post(self.trs["lat"], tgt)
            self.k += 1
            if self.k % 10 == 0:
                before = {kk: v[0].row_length.copy() for kk, v in self.projs.items()}
                tg_before = {kk: v[0].target.copy() for kk, v in self.projs.items()}
                self.model.run_update_group("rewiring")
                for kk, (m, _) in self.projs.items():
                    if not (np.array_equal(before[kk], m.row_length) and np.array_equal(tg_before[kk], m.target)):
                        self.trs[kk] = transpose(m)
        return time.perf_counter() - t0


def time_topomap(scale: int, model_ms: float, seed: int = 1) -> dict:
    """x realtime of the CPU port at one scale (build excluded, reported)."""
    tm = TopomapPort(scale, seed)
    tm.run(min(5.0, model_ms))          # warm-up: first stimulus, allocations
    wall = tm.run(model_ms)
    return {"n": tm.n, "model_ms": model_ms, "wall_s": round(wall, 3),
            "x_realtime": round(model_ms * 1e-3 / wall, 5), "build_s": round(tm.build_s, 2)}
