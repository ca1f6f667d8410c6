"""Oracle restatement of the e-prop ALIF classifier path: AlifLayer
(neurons.py:46-73), eprop_accumulate_batch (_kernels.py:15-39, per-op
float32 emulation, replicas ascending), SyntheticTask and the trainer
(classifier.py:28-293).  Test infrastructure only."""

from __future__ import annotations

import math

import numpy as np

from .deep_r import AdamOracle, DeepROracle
from .ragged import Ragged, init_pairwise_bernoulli
from .rng import Stream
from .updates import OracleModel

F = np.float32


class AlifP:
    tau_mem, tau_adapt, beta, v_thr, dt = 20.0, 2000.0, 0.0174, 0.6, 1.0

    @property
    def alpha(self):
        return math.exp(-self.dt / self.tau_mem)

    @property
    def rho(self):
        return math.exp(-self.dt / self.tau_adapt)


def alif_step(v, a, z, rec, ext, p=AlifP()):
    """neurons.py:60-67 with NEP-50 float32 constants."""
    v = F(p.alpha) * (v - z * F(p.v_thr)) + rec + ext
    a = F(p.rho) * a + z
    z = (v >= F(p.v_thr) + F(p.beta) * a).astype(v.dtype)
    return v, a, z


def alif_surrogate(v, a, p=AlifP()):
    """neurons.py:69-73."""
    c = (v - (F(p.v_thr) + F(p.beta) * a)) / F(p.v_thr)
    return F(0.3 / p.v_thr) * np.maximum(F(0.0), F(1.0) - np.abs(c))


def eprop_accumulate(targets, row_length, pre_trace, psi, lsig, eps, ebar, grad, beta, rho, alpha):
    """_kernels.py:15-39.  Vectorised over synapses, replicas in ascending
    order; every float32 op separately rounded (numba emits no FMA, F6)."""
    P, S = targets.shape
    mask = np.arange(S)[None, :] < row_length[:, None]
    ii, ss = np.nonzero(mask)
    jj = targets[ii, ss]
    beta, rho, alpha = F(beta), F(rho), F(alpha)
    for b in range(pre_trace.shape[0]):
        zb = pre_trace[b, ii]
        ep = eps[b, ii, ss]
        e = psi[b, jj] * (zb - beta * ep)
        eb = alpha * ebar[b, ii, ss] + e
        ebar[b, ii, ss] = eb
        grad[ii, ss] += (lsig[b, jj] * eb).astype(np.float64)
        eps[b, ii, ss] = rho * ep + e


def eprop_accumulate_fast(*args):
    """The C restatement (oracle/c/oracle.c) when gcc is available, else numpy."""
    try:
        from .cbuild import eprop_accumulate_c
        return eprop_accumulate_c(*args)
    except Exception:
        return eprop_accumulate(*args)


class TaskOracle:
    """classifier.py:28-79."""

    def __init__(self, num_classes=3, num_inputs=20, example_steps=200, seed=0, rate_lo=5.0,
                 rate_hi=80.0, dt=1.0, num_train=320, num_test=96, jitter=0.8):
        self.num_classes, self.num_inputs, self.example_steps = num_classes, num_inputs, example_steps
        self.seed, self.dt, self.num_train, self.num_test, self.jitter = seed, dt, num_train, num_test, jitter
        s = Stream.of(seed, "task", "templates")
        self.rates = (rate_lo + s.uniform01_array(num_classes * num_inputs) * (rate_hi - rate_lo)
                      ).reshape(num_classes, num_inputs)

    def label(self, e):
        return e % self.num_classes

    def example_spikes(self, e):
        r = self.rates[self.label(e)]
        if self.jitter:
            r = r * np.exp(self.jitter * Stream.of(self.seed, "task", "jitter", e).normal_array(self.num_inputs))
        p = 1.0 - np.exp(-r * self.dt * 1e-3)
        u = Stream.of(self.seed, "task", "example", e).uniform01_array(self.example_steps * self.num_inputs)
        return u.reshape(self.example_steps, self.num_inputs) < p

    def train_ids(self, bi, bs):
        return [(bi * bs + r) % self.num_train for r in range(bs)]


class TrainerOracle:
    """classifier.py:82-263 (float32 model, DEEP R on)."""

    PLANES = ("w", "grad", "adam_m", "adam_v")

    def __init__(self, task, hidden=128, input_density=0.1, recurrent_density=0.1, deep_r=True,
                 l1_strength=0.005, learning_rate=1e-3, batch_size=32, seed=0,
                 input_gain=0.5, recurrent_gain=0.15):
        self.task, self.hidden, self.B, self.seed = task, hidden, batch_size, seed
        self.deep_r = deep_r
        self.p = AlifP()
        head = 2.0 if deep_r else 1.0
        self.net = OracleModel(seed)
        self.m_in = self._make("in", task.num_inputs, hidden, input_density, head,
                               input_gain / math.sqrt(max(1.0, input_density * task.num_inputs)), False)
        self.m_rec = self._make("rec", hidden, hidden, recurrent_density, head,
                                recurrent_gain / math.sqrt(max(1.0, recurrent_density * hidden)), True)
        C = task.num_classes
        self.w_out = Stream.of(seed, "init", "out").normal_array(C * hidden, std=1.0 / math.sqrt(hidden)).reshape(C, hidden)
        self.b_out = np.zeros(C)
        self.g_w_out = np.zeros_like(self.w_out)
        self.g_b_out = np.zeros_like(self.b_out)
        self.adam_in = AdamOracle(learning_rate, m=self.m_in.planes["adam_m"], v=self.m_in.planes["adam_v"])
        self.adam_rec = AdamOracle(learning_rate, m=self.m_rec.planes["adam_m"], v=self.m_rec.planes["adam_v"])
        self.adam_out = AdamOracle(learning_rate, shape=self.w_out.shape)
        self.adam_b = AdamOracle(learning_rate, shape=self.b_out.shape)
        if deep_r:
            self.dr_in = DeepROracle(self.m_in, l1=l1_strength)
            self.dr_rec = DeepROracle(self.m_rec, l1=l1_strength, exclude_diagonal=True)
            self.dr_in.init_bitfields(Stream.of(seed, "deep_r", "in"))
            self.dr_rec.init_bitfields(Stream.of(seed, "deep_r", "rec"))
            self.dr_in.register(self.net, "deep_r", "in")
            self.dr_rec.register(self.net, "deep_r", "rec")

    def _make(self, name, P, N, dens, head, std, diag):
        s = Stream.of(self.seed, "init", name)

        def prob(i, cols):
            p = np.full(cols.size, dens)
            if diag:
                p[i] = 0.0
            return p
        m = init_pairwise_bernoulli(P, N, prob, head, s, self.PLANES)
        mask = m.slot_mask()
        w = m.planes["w"]
        w[mask] = s.normal_array(w.size, std=std).reshape(w.shape)[mask]
        self.net.add_matrix(name, m)
        return m

    @staticmethod
    def _dense(m):
        w = np.zeros((m.num_pre, m.num_post), dtype=F)
        for i in range(m.num_pre):
            n = m.row_length[i]
            w[i, m.target[i, :n]] = m.planes["w"][i, :n]
        return w

    def forward(self, ids, learn=True, step_times=None):
        """classifier.py:188-234.  ``step_times`` (list) receives per-step wall
        seconds (CPU-baseline timing)."""
        import time
        p, B, H, C = self.p, self.B, self.hidden, self.task.num_classes
        spikes = np.stack([self.task.example_spikes(e) for e in ids]).astype(F)
        labels = np.array([self.task.label(e) for e in ids])
        one_hot = np.eye(C)[labels]
        wi, wr = self._dense(self.m_in), self._dense(self.m_rec)
        v = np.zeros((B, H), F)
        a = np.zeros((B, H), F)
        z = np.zeros((B, H), F)
        y = np.zeros((B, C))
        zbar = np.zeros((B, H), F)
        xbar = np.zeros((B, self.task.num_inputs), F)
        eps_i = np.zeros((B,) + self.m_in.target.shape, F)
        ebar_i = np.zeros_like(eps_i)
        eps_r = np.zeros((B,) + self.m_rec.target.shape, F)
        ebar_r = np.zeros_like(eps_r)
        loss_sum, pi_sum = 0.0, np.zeros((B, C))
        al, be, rh = F(p.alpha), F(p.beta), F(p.rho)
        for t in range(self.task.example_steps):
            t0 = time.perf_counter()
            x = spikes[:, t, :]
            rec, ext = z @ wr, x @ wi
            zbar *= al
            zbar += z
            xbar *= al
            xbar += x
            psi = alif_surrogate(v, a)
            y = p.alpha * y + z @ self.w_out.T + self.b_out
            e = np.exp(y - y.max(axis=-1, keepdims=True))
            pi = e / e.sum(axis=-1, keepdims=True)
            d = pi - one_hot
            loss_sum += float(-np.log(np.sum(pi * one_hot, axis=-1)).sum())
            pi_sum += pi
            if learn:
                self.g_w_out += d.T @ zbar
                self.g_b_out += d.sum(axis=0)
                lsig = (d @ self.w_out).astype(F)
                eprop_accumulate_fast(self.m_in.target, self.m_in.row_length, xbar, psi, lsig,
                                      eps_i, ebar_i, self.m_in.planes["grad"], be, rh, al)
                eprop_accumulate_fast(self.m_rec.target, self.m_rec.row_length, zbar, psi, lsig,
                                      eps_r, ebar_r, self.m_rec.planes["grad"], be, rh, al)
            v, a, z = alif_step(v, a, z, rec, ext)
            if step_times is not None:
                step_times.append(time.perf_counter() - t0)
        acc = float((pi_sum.argmax(axis=1) == labels).mean())
        return loss_sum / (B * self.task.example_steps), acc

    def gradient_phase(self, bi):
        loss, acc = self.forward(self.task.train_ids(bi, self.B))
        inv = 1.0 / self.B
        for t in (self.m_in.planes["grad"], self.m_rec.planes["grad"], self.g_w_out, self.g_b_out):
            t *= inv
        if self.deep_r:
            self.dr_in.l1_step()
            self.dr_rec.l1_step()
        self.adam_in.apply(self.m_in.planes["w"], self.m_in.planes["grad"])
        self.adam_rec.apply(self.m_rec.planes["w"], self.m_rec.planes["grad"])
        self.adam_out.apply(self.w_out, self.g_w_out)
        self.adam_b.apply(self.b_out, self.g_b_out)
        return loss, acc

    def rewire_phase(self):
        if self.deep_r:
            self.net.run_update_group("deep_r")
            return self.dr_in.last_removed + self.dr_rec.last_removed
        return 0
