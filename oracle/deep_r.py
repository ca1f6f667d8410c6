"""Oracle restatement of DEEP R (``sparsewire/deep_r.py``) and Adam
(``sparsewire/plasticity.py:198-227``).  Test infrastructure only."""

from __future__ import annotations

import numpy as np

from .ragged import (Ragged, RowFull, bf_clear, bf_randomize, bf_set, bf_test,
                     bf_words)
from .rng import Stream


class DeepROracle:
    """deep_r.py:23-177."""

    def __init__(self, m: Ragged, l1=0.005, exclude_diagonal=False,
                 weight_plane="w", grad_plane="grad"):
        self.m = m
        self.l1 = l1
        self.exclude_diagonal = exclude_diagonal
        self.wp = weight_plane
        self.gp = grad_plane
        W = bf_words(m.num_post)
        self.sign = np.zeros((m.num_pre, W), dtype=np.uint64)
        self.conn = np.zeros((m.num_pre, W), dtype=np.uint64)
        self.dormant = np.zeros(m.num_pre, dtype=np.int64)
        self.unplaced = np.zeros(m.num_pre, dtype=np.int64)
        self.activations = np.zeros(m.num_pre, dtype=np.int64)
        self.no_progress = 0
        self.last_removed = 0

    # deep_r.py:50-64
    def init_bitfields(self, stream: Stream):
        m = self.m
        bf_randomize(self.sign, m.num_post, stream)
        self.conn[:] = 0
        w = m.planes[self.wp]
        for i in range(m.num_pre):
            n = m.row_length[i]
            for s in range(n):
                bf_set(self.conn, i, int(m.target[i, s]))
            # all sets of the row, then all clears (two vector calls, :62-64)
            for s in range(n):
                if w[i, s] > 0:
                    bf_set(self.sign, i, int(m.target[i, s]))
            for s in range(n):
                if w[i, s] < 0:
                    bf_clear(self.sign, i, int(m.target[i, s]))

    def sign_of_slots(self):
        """Sign bit of every slot's target (bitfield.py:93-102 test_bits_rows)."""
        t = self.m.target
        w = np.take_along_axis(self.sign, (t >> 6).astype(np.int64), axis=1)
        return ((w >> (t & 63).astype(np.uint64)) & np.uint64(1)).astype(bool)

    # deep_r.py:68-77
    def l1_step(self):
        if self.l1 == 0.0:
            return
        g = self.m.planes[self.gp]
        nudge = np.where(self.sign_of_slots(), self.l1, -self.l1)
        g += nudge * self.m.slot_mask()

    # deep_r.py:81-99
    def elim_host(self, ctx):
        self.dormant[:] = 0

    def elim_rows(self, ctx):
        return range(self.m.num_pre)

    def elim_row(self, i, rng):
        m = self.m
        n = int(m.row_length[i])
        if n == 0:
            return
        tg = m.target[i, :n]
        w = m.planes[self.wp][i, :n]
        pos = np.array([bf_test(self.sign, i, int(j)) for j in tg])
        mism = ((w < 0) & pos) | ((w > 0) & ~pos)
        if not mism.any():
            return
        slots = np.flatnonzero(mism)
        gone = tg[slots].copy()
        m.remove_slots(i, slots)
        for j in gone:
            bf_clear(self.conn, i, int(j))
        self.dormant[i] = slots.size

    # deep_r.py:110-124
    def form_host(self, ctx):
        if ctx.pass_index == 0:
            pending = int(self.dormant.sum())
            self.last_removed = pending
            self.no_progress = 0
        else:
            pending = int(self.unplaced.sum())
        self.activations[:] = 0
        P = self.m.num_pre
        for _ in range(pending):
            self.activations[ctx.rng.uniform_int(P)] += 1
        self.unplaced[:] = 0

    def form_rows(self, ctx):
        return np.flatnonzero(self.activations)

    # deep_r.py:126-145
    def form_row(self, i, rng):
        m = self.m
        N = m.num_post
        for _ in range(int(self.activations[i])):
            if m.row_length[i] >= m.max_row_length:
                self.unplaced[i] += 1
                continue
            placed = False
            for _ in range(N):
                j = rng.uniform_int(N)
                if self.exclude_diagonal and j == i:
                    continue
                if bf_test(self.conn, i, j):
                    continue
                m.add_synapse(i, j, {self.wp: 0.0})
                bf_set(self.conn, i, j)
                placed = True
                break
            if not placed:
                self.unplaced[i] += 1

    # deep_r.py:147-160
    def form_continue(self, ctx):
        u = int(self.unplaced.sum())
        if u == 0:
            return False
        if int(self.activations.sum()) - u == 0:
            self.no_progress += 1
            if self.no_progress >= self.m.num_pre:
                raise RowFull("stalled")
        else:
            self.no_progress = 0
        return True

    def register(self, model, group, matrix_name):
        class _R:
            pass
        e = _R()
        e.host_phase, e.active_rows, e.row_phase = self.elim_host, self.elim_rows, self.elim_row
        e.continue_after_pass = lambda ctx: False
        f = _R()
        f.host_phase, f.active_rows, f.row_phase = self.form_host, self.form_rows, self.form_row
        f.continue_after_pass = self.form_continue
        model.add_rule(group, matrix_name, e)
        model.add_rule(group, matrix_name, f)


class AdamOracle:
    """plasticity.py:198-227 (float64, whole plane, grads zeroed)."""

    def __init__(self, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, m=None, v=None, shape=None):
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps
        self.m = np.zeros(shape) if m is None else m
        self.v = np.zeros(shape) if v is None else v
        self.t = 0

    def apply(self, p, g):
        self.t += 1
        self.m *= self.b1
        self.m += (1.0 - self.b1) * g
        self.v *= self.b2
        self.v += (1.0 - self.b2) * g * g
        mh = self.m / (1.0 - self.b1 ** self.t)
        vh = self.v / (1.0 - self.b2 ** self.t)
        p -= self.lr * mh / (np.sqrt(vh) + self.eps)
        g[...] = 0
