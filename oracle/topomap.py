"""Oracle restatement of the topographic-map hot path: RewiringRule
(topomap.py:70-223, restated with a candidate list instead of the attempt
bitfield and a formation-probability LUT by torus offset — SURVEY F5/F10b),
trace STDP (plasticity.py:42-95), the conductance LIF step
(neurons.py:137-148) and the Poisson step (neurons.py:189-195).
Test infrastructure only."""

from __future__ import annotations

import math

import numpy as np

from .ragged import Ragged, RowFull
from .rng import Stream


def torus_offset(i, j, side):
    xi, yi, xj, yj = i % side, i // side, j % side, j // side
    return (xj - xi) % side + side * ((yj - yi) % side)


def offset_luts(side, p_form, sigma_form):
    """(formation probability, toroidal distance) by wrapped offset
    dx + side*dy: formation_probability (topomap.py:49-52) of
    toroidal_distance(0, arange(n)) (geometry.py:23-31), one vector call as
    the reference evaluates it (F10b)."""
    idx = np.arange(side * side)
    x = (idx % side).astype(np.float64)
    y = (idx // side).astype(np.float64)
    dx = np.abs(x[0] - x)
    dy = np.abs(y[0] - y)
    d = np.hypot(np.minimum(dx, side - dx), np.minimum(dy, side - dy))
    return p_form * np.exp(-(d ** 2) / (2.0 * sigma_form ** 2)), d


class RewiringOracle:
    def __init__(self, m: Ragged, side: int, form_lut, dist_lut, total_attempts, g_theta=0.1,
                 p_dep=2.45e-2 * 50, p_pot=1.36e-4 * 50, g_init=0.2, plane="g"):
        self.m, self.side = m, side
        self.form_lut, self.dist_lut = form_lut, dist_lut
        self.total_attempts = total_attempts
        self.g_theta, self.p_dep, self.p_pot, self.g_init = g_theta, p_dep, p_pot, g_init
        self.plane = plane
        self.attempts = np.zeros(m.num_pre, dtype=np.int64)
        self.events = []        # (row, kind, distance) in row order
        self.stats = None

    # topomap.py:101-108
    def host_phase(self, ctx):
        self.attempts[:] = 0
        for _ in range(self.total_attempts):
            self.attempts[ctx.rng.uniform_int(self.m.num_pre)] += 1
        self.events = []
        self.stats = dict(removed=0, kept=0, formed=0, form_missed=0, form_full=0)

    def active_rows(self, ctx):
        return np.flatnonzero(self.attempts)

    # topomap.py:142-196
    def row_phase(self, i, rng: Stream):
        m = self.m
        k = int(self.attempts[i])
        N = m.num_post
        cand = list(rng.sample_k_distinct(k, N))
        n = int(m.row_length[i])
        sel = [s for s in range(n) if int(m.target[i, s]) in cand]
        g = m.planes[self.plane]
        targets_sel = [int(m.target[i, s]) for s in sel]
        hits = []
        for s in sel:
            u = rng.uniform01()
            p = self.p_dep if g[i, s] < self.g_theta else self.p_pot
            hits.append(u < p)
        for s, t, h in zip(sel, targets_sel, hits):
            if h:
                self.events.append((i, 1, float(self.dist_lut[torus_offset(i, t, self.side)])))
        m.remove_slots(i, [s for s, h in zip(sel, hits) if h])
        self.stats["removed"] += sum(hits)
        self.stats["kept"] += len(sel) - sum(hits)
        remaining = sorted(c for c in cand if c not in targets_sel)
        for j in remaining:
            o = torus_offset(i, int(j), self.side)
            u = rng.uniform01()
            if not u < self.form_lut[o]:
                self.stats["form_missed"] += 1
                continue
            try:
                m.add_synapse(i, int(j), {self.plane: self.g_init})
                self.stats["formed"] += 1
                self.events.append((i, 2, float(self.dist_lut[o])))
            except RowFull:
                self.stats["form_full"] += 1

    def continue_after_pass(self, ctx):
        return False


# -- trace STDP (plasticity.py:42-95) ------------------------------------------------

class StdpOracle:
    def __init__(self, m: Ragged, h, a_plus=0.1 * 0.2, tau_plus=20.0, tau_minus=64.0, b_ratio=1.2,
                 w_min=0.0, w_max=0.2, plane="g"):
        self.m, self.plane = m, plane
        self.a_plus = a_plus
        self.a_minus = b_ratio * a_plus * tau_plus / tau_minus
        self.w_min, self.w_max = w_min, w_max
        self.x = np.zeros(m.num_pre)
        self.y = np.zeros(m.num_post)
        self.dx = math.exp(-h / tau_plus)
        self.dy = math.exp(-h / tau_minus)

    def decay(self):
        self.x *= self.dx
        self.y *= self.dy

    def on_pre(self, pre):
        w = self.m.planes[self.plane]
        for i in pre:
            n = self.m.row_length[i]
            row = w[i, :n]
            row -= self.a_minus * self.y[self.m.target[i, :n]]
            np.maximum(row, self.w_min, out=row)
            np.minimum(row, self.w_max, out=row)
        self.x[pre] += 1.0

    def on_post(self, tr, post):
        """tr = (col_length, src_pre, src_slot) from oracle.ragged.transpose."""
        cl, sp, ss = tr
        w = self.m.planes[self.plane]
        pres = np.concatenate([sp[j, :cl[j]] for j in post]) if len(post) else np.empty(0, int)
        slots = np.concatenate([ss[j, :cl[j]] for j in post]) if len(post) else np.empty(0, int)
        if pres.size:
            b = w[pres, slots] + self.a_plus * self.x[pres]
            np.maximum(b, self.w_min, out=b)
            np.minimum(b, self.w_max, out=b)
            w[pres, slots] = b
        self.y[post] += 1.0


def lif_cond_step(V, g, ref_until, incoming, k, h=0.1, tau_s=5.0, c_m=20.0, tau_m=20.0,
                  v_rest=-70.0, e_exc=0.0, v_theta=-54.0, v_reset=-70.0, tau_ref=5.0):
    """neurons.py:137-148 (in place); returns spiking ids."""
    g_leak = c_m / tau_m
    g[:] = (g + incoming) * math.exp(-h / tau_s)
    active = k > ref_until
    r = g / g_leak
    v_inf = (v_rest + r * e_exc) / (1.0 + r)
    v_new = v_inf + (V - v_inf) * np.exp(-h * (1.0 + r) / tau_m)
    V[:] = np.where(active, v_new, v_reset)
    spk = active & (V >= v_theta)
    V[spk] = v_reset
    ref_until[spk] = k + int(round(tau_ref / h))
    return np.flatnonzero(spk)


def poisson_step(stream: Stream, p):
    """neurons.py:189-195."""
    return np.flatnonzero(stream.uniform01_array(p.size) < p)
