"""Recurrent ALIF classifier trained with e-prop + DEEP R on the device
(``sparsewire/classifier.py`` API).

Per group of K = EPROP_BLOCK_STEPS timesteps two sm_100a launches:
``sw_clf_step`` (n_steps = K) runs the fused per-replica forward of the K
steps, and ``sw_eprop_fused_block`` updates the eligibility state and the
gradients of both projections plus the readout gradients for all K steps in
one pass (temporal blocking).  The whole 1000-step trial is captured once as
a CUDA graph (forward on one stream, e-prop passes on a second) and replayed
every batch.  Per batch: gradient scale,
L1 nudge, Adam, DEEP R (classifier.py:236-263).  With ``process_group``
set, replicas are sharded across ranks and the raw gradient sums are
all-reduced (NCCL) before the update, so every rank applies the same
update and replays the same rewiring streams.
"""

from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .connectivity import init_pairwise_bernoulli_density
from .deep_r import DeepR
from .neurons import AlifParams
from .plasticity import Adam
from .rng import CounterRng, fold_key
from .sharding import allreduce_flat
from .updates import Model


# timesteps per e-prop pass over the eligibility state (temporal blocking,
# sw_eprop_fused_block): K forward steps run first, then one pass applies K
# recursion steps to every (replica, synapse) element
EPROP_BLOCK_STEPS = int(os.environ.get("SW_EPROP_BLOCK_STEPS", "16"))
if not 1 <= EPROP_BLOCK_STEPS <= _lib.MAX_BLOCK:
    raise ValueError(f"SW_EPROP_BLOCK_STEPS={EPROP_BLOCK_STEPS}: must be in 1..{_lib.MAX_BLOCK} "
                     "(SW_EPROP_MAX_BLOCK in include/sparsewire_b200.h)")
# (step, replica) splits of the readout gradient inside the blocked pass
READOUT_SPLITS = int(os.environ.get("SW_READOUT_SPLITS", "16"))


@dataclass
class SyntheticTask:
    """classifier.py:28-79: class rate templates; per-example lognormal
    jitter (host numpy Box-Muller/exp); Poisson spikes drawn on the device
    from the example's counter stream."""

    num_classes: int = 3
    num_inputs: int = 20
    example_steps: int = 200
    seed: int = 0
    rate_lo: float = 5.0
    rate_hi: float = 80.0
    dt: float = 1.0
    num_train: int = 320
    num_test: int = 96
    jitter: float = 0.8

    def __post_init__(self):
        rng = CounterRng(self.seed, "task", "templates")
        rates = self.rate_lo + rng.uniform01_array(self.num_classes * self.num_inputs) * (
            self.rate_hi - self.rate_lo)
        self.rates = rates.reshape(self.num_classes, self.num_inputs)

    def label(self, example: int) -> int:
        return example % self.num_classes

    def example_rates(self, example: int) -> np.ndarray:
        rates = self.rates[self.label(example)]
        if self.jitter:
            noise = CounterRng(self.seed, "task", "jitter", example).normal_array(self.num_inputs)
            rates = rates * np.exp(self.jitter * noise)
        return rates

    def example_prob(self, example: int) -> np.ndarray:
        return 1.0 - np.exp(-self.example_rates(example) * self.dt * 1e-3)

    def example_key(self, example: int) -> int:
        return fold_key(self.seed, "task", "example", example)

    def batch_inputs(self, example_ids):
        """Host-side per-example inputs of one batch: spike probabilities
        [B, NI] float64, stream keys [B] and labels [B]."""
        p = np.stack([self.example_prob(e) for e in example_ids])
        keys = np.array([self.example_key(e) for e in example_ids], dtype=np.uint64)
        labels = np.array([self.label(e) for e in example_ids], dtype=np.int32)
        return p, keys, labels

    def example_spikes(self, example: int) -> torch.Tensor:
        """[example_steps, num_inputs] bool spikes, drawn on the device."""
        n = self.example_steps * self.num_inputs
        u = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("sw_rng_uniform01", self.example_key(example), 0, n, u.data_ptr(),
                  _lib.stream_ptr())
        p = torch.from_numpy(self.example_prob(example)).cuda()
        return u.view(self.example_steps, self.num_inputs) < p[None, :]

    def batch(self, example_ids):
        spikes = torch.stack([self.example_spikes(e) for e in example_ids])
        labels = np.array([self.label(e) for e in example_ids])
        return spikes, labels

    def train_ids(self, batch_index: int, batch_size: int) -> list[int]:
        start = batch_index * batch_size
        return [(start + r) % self.num_train for r in range(batch_size)]

    def test_ids(self) -> list[int]:
        return [self.num_train + r for r in range(self.num_test)]


class _Plan:
    """Compact per-batch synapse order of one projection (sw_eprop_plan:
    bucketed by post >> shift, then pre, then slot) and its eligibility state.
    layout "chunk" (the trainer's, sw_eprop_pass): [e_pad/SPW][ldb/32][32][SPW],
    with shift 0 (synapses by post); layout "tile" (sw_eprop_fused_step /
    _block): [tile][batch][32]."""

    def __init__(self, m, batch, shift=5, layout="tile"):
        self.m = m
        self.shift = shift
        self.layout = layout
        self.e_pad = 0
        self.batch = batch
        self.ldb = -(-batch // 32) * 32
        G = ((m.num_post - 1) >> shift) + 1
        n = G * m.num_pre   # counts, cursor, then one sum per 4096-count scan tile
        self.scratch = torch.zeros(2 * n + (n + 4095) // 4096 + 1, dtype=torch.int32, device="cuda")
        self.total = torch.zeros(1, dtype=torch.int32, device="cuda")

    def ensure(self, edges: int) -> None:
        e_pad = max(32, (edges + 31) // 32 * 32)
        if e_pad == self.e_pad:
            return
        self.e_pad = e_pad
        dev = "cuda"
        self.pre = torch.zeros(e_pad, dtype=torch.int32, device=dev)
        self.post = torch.zeros(e_pad, dtype=torch.int32, device=dev)
        self.off = torch.zeros(e_pad, dtype=torch.int32, device=dev)
        self.grad = torch.zeros(e_pad, dtype=torch.float64, device=dev)
        if self.layout == "chunk":
            # [SPW-synapse tile, 32-replica chunk, lane = (32/SPW) * synapse +
            # group, SPW replicas of the group] (sw_eprop_pass)
            spw = self.spw = int(_lib.lib().sw_eprop_pass_synapses_per_warp())
            self.eps = torch.zeros((e_pad // spw, self.ldb // 32, 32, spw), dtype=torch.float32, device=dev)
        else:
            # [tile, replica, lane] (sw_eprop_fused_step / sw_eprop_fused_block)
            self.eps = torch.zeros((e_pad // 32, self.batch, 32), dtype=torch.float32, device=dev)
        self.ebar = torch.zeros_like(self.eps)

    def replica_major(self, state: torch.Tensor) -> torch.Tensor:
        """[batch, e_pad] copy of eps or ebar (tests, inspection)."""
        if self.layout == "chunk":
            spw = self.spw
            t = state.view(self.e_pad // spw, self.ldb // 32, spw, 32 // spw, spw)   # [tile, c, s, g, r]
            return t.permute(1, 3, 4, 0, 2).reshape(self.ldb, self.e_pad)[:self.batch]
        return state.permute(1, 0, 2).reshape(self.batch, self.e_pad)

    def build(self) -> None:
        m = self.m
        _lib.call("sw_eprop_plan", m.row_length.data_ptr(), m.target.data_ptr(), m.num_pre,
                  m.stride, m.num_post, self.shift, self.scratch.data_ptr(), self.pre.data_ptr(),
                  self.post.data_ptr(), self.off.data_ptr(), self.e_pad, self.total.data_ptr(),
                  _lib.stream_ptr())

    def tseg(self, trace_t: list) -> _lib.EpropTSeg:
        s = _lib.EpropTSeg()
        s.pre, s.post = self.pre.data_ptr(), self.post.data_ptr()
        for k, t in enumerate(trace_t):
            s.trace_t[k] = t.data_ptr()
        s.eps, s.ebar, s.grad = self.eps.data_ptr(), self.ebar.data_ptr(), self.grad.data_ptr()
        s.e_pad = self.e_pad
        return s

    def seg(self, trace: torch.Tensor) -> _lib.EpropSeg:
        s = _lib.EpropSeg()
        s.pre, s.post, s.pre_trace = self.pre.data_ptr(), self.post.data_ptr(), trace.data_ptr()
        s.eps, s.ebar, s.grad = self.eps.data_ptr(), self.ebar.data_ptr(), self.grad.data_ptr()
        s.num_pre, s.e_pad = self.m.num_pre, self.e_pad
        return s


class EpropClassifierTrainer:
    """classifier.py:82-293 on the device."""

    def __init__(self, task: SyntheticTask, hidden: int = 128, input_density: float = 0.1,
                 recurrent_density: float = 0.1, deep_r: bool = True, l1_strength: float = 0.005,
                 learning_rate: float = 1e-3, batch_size: int = 32, seed: int = 0,
                 workers: int = 1, dtype=np.float32, input_gain: float = 0.5,
                 recurrent_gain: float = 0.15, use_graph: bool = True, process_group=None,
                 local_batch: slice | None = None):
        _lib.require_cuda()
        if np.dtype(dtype) != np.float32:
            raise TypeError("the device trainer computes the forward pass in float32")
        self.task = task
        self.hidden = hidden
        self.batch_size = batch_size
        self.seed = seed
        self.deep_r_enabled = deep_r
        self.params = AlifParams()
        self.use_graph = use_graph
        # graph replays overlap group g's e-prop pass with group g+1's forward
        # launch (SW_CLF_OVERLAP=0: one stream, measurement)
        self.overlap = os.environ.get("SW_CLF_OVERLAP", "1") != "0"
        self.pg = process_group
        # replicas handled by this rank (batch-DP); default: all of them
        self.local = local_batch if local_batch is not None else slice(0, batch_size)
        self.local_b = self.local.stop - self.local.start

        headroom = 2.0 if deep_r else 1.0
        self.net = Model(seed, workers=workers)
        self.m_in, self.s_in = self._make_matrix(
            "in", task.num_inputs, hidden, input_density, headroom,
            input_gain / math.sqrt(max(1.0, input_density * task.num_inputs)), False)
        self.m_rec, self.s_rec = self._make_matrix(
            "rec", hidden, hidden, recurrent_density, headroom,
            recurrent_gain / math.sqrt(max(1.0, recurrent_density * hidden)), True)
        out_rng = CounterRng(seed, "init", "out")
        C = task.num_classes
        self.w_out = torch.from_numpy(out_rng.normal_array(
            C * hidden, std=1.0 / math.sqrt(hidden)).reshape(C, hidden)).cuda()
        self.b_out = torch.zeros(C, dtype=torch.float64, device="cuda")
        self.g_w_out = torch.zeros_like(self.w_out)
        self.g_b_out = torch.zeros_like(self.b_out)
        self.adam_in = Adam(learning_rate, m=self.s_in.planes["adam_m"], v=self.s_in.planes["adam_v"])
        self.adam_rec = Adam(learning_rate, m=self.s_rec.planes["adam_m"], v=self.s_rec.planes["adam_v"])
        self.adam_out = Adam(learning_rate, shape=self.w_out.shape)
        self.adam_b = Adam(learning_rate, shape=self.b_out.shape)
        if deep_r:
            self.deep_r_in = DeepR(self.m_in, self.s_in, "in", l1_strength=l1_strength)
            self.deep_r_rec = DeepR(self.m_rec, self.s_rec, "rec", l1_strength=l1_strength,
                                    exclude_diagonal=True)
            self.deep_r_in.init_bitfields(CounterRng(seed, "deep_r", "in"))
            self.deep_r_rec.init_bitfields(CounterRng(seed, "deep_r", "rec"))
            self.deep_r_in.register(self.net, "deep_r", "in")
            self.deep_r_rec.register(self.net, "deep_r", "rec")
        self._alloc_state()
        self.history: list[dict] = []
        self._graph = None
        self._graph_learn = None
        self.steps_launched = 0

    # -- construction ------------------------------------------------------------
    def _make_matrix(self, name, num_pre, num_post, density, headroom, w_std, exclude_diagonal):
        rng = CounterRng(self.seed, "init", name)
        m, syn = init_pairwise_bernoulli_density(num_pre, num_post, density, headroom, rng,
                                                 var_names=("w", "grad", "adam_m", "adam_v"),
                                                 exclude_diagonal=exclude_diagonal)
        draws = rng.normal_array(m.num_pre * m.stride, std=w_std).reshape(m.num_pre, m.stride)
        mask = m.slot_mask()
        w = syn.planes["w"]
        w.copy_(torch.where(mask, torch.from_numpy(draws).cuda(), w))
        self.net.add_matrix(name, m, syn)
        return m, syn

    def _alloc_state(self):
        B, H, NI, C = self.local_b, self.hidden, self.task.num_inputs, self.task.num_classes
        f32 = dict(dtype=torch.float32, device="cuda")
        f64 = dict(dtype=torch.float64, device="cuda")
        self.v = torch.zeros((B, H), **f32)
        self.a = torch.zeros((B, H), **f32)
        self.z = torch.zeros((B, H), **f32)
        # per-step e-prop inputs in 2*K rotating slots (K = EPROP_BLOCK_STEPS):
        # step t writes slot t % 2K.  The e-prop pass over steps [gK, gK+K)
        # reads one half while the forward passes of the next K steps write
        # the other half, so both can run at once.
        K2 = 2 * EPROP_BLOCK_STEPS
        # contiguous [slot][B][width] arrays (the grouped forward launch
        # addresses slot t % K2 from the base), listed as per-slot views
        self._slots_zbar = torch.zeros((K2, B, H), **f32)
        self._slots_xbar = torch.zeros((K2, B, NI), **f32)
        self._slots_psi = torch.zeros((K2, B, H), **f32)
        self._slots_lsig = torch.zeros((K2, B, H), **f32)
        self._slots_d = torch.zeros((K2, B, C), **f64)
        self._slot_zbar = list(self._slots_zbar.unbind(0))
        self._slot_xbar = list(self._slots_xbar.unbind(0))
        self._slot_psi = list(self._slots_psi.unbind(0))
        self._slot_lsig = list(self._slots_lsig.unbind(0))
        self._slot_d = list(self._slots_d.unbind(0))
        # slot-0 views under the reference attribute names
        self.zbar, self.xbar = self._slot_zbar[0], self._slot_xbar[0]
        self.psi, self.lsig = self._slot_psi[0], self._slot_lsig[0]
        self.y = torch.zeros((B, C), **f64)
        self.pi_sum = torch.zeros((B, C), **f64)
        self.loss_b = torch.zeros(B, **f64)
        self.d = self._slot_d[0]
        self.p_in = torch.zeros((B, NI), **f64)
        self.keys = torch.zeros(B, dtype=torch.int64, device="cuda")
        self.labels = torch.zeros(B, dtype=torch.int32, device="cuda")
        self.w32_in = torch.zeros(self.m_in.target.shape, **f32)
        self.w32_rec = torch.zeros(self.m_rec.target.shape, **f32)
        # packed (target, f32 weight) rows for the forward kernel's bulk staging
        self._tw_stride = {n: m.stride + (m.stride & 1) for n, m in (("in", self.m_in), ("rec", self.m_rec))}
        self.tw_in = torch.zeros((self.m_in.num_pre, self._tw_stride["in"], 2), dtype=torch.int32, device="cuda")
        self.tw_rec = torch.zeros((self.m_rec.num_pre, self._tw_stride["rec"], 2), dtype=torch.int32,
                                  device="cuda")
        self.stats = torch.zeros(2, **f64)
        self.stats_host = torch.zeros(2, dtype=torch.float64, pin_memory=True)
        self.pin_p = torch.zeros((B, NI), dtype=torch.float64, pin_memory=True)
        self.pin_keys = torch.zeros(B, dtype=torch.int64, pin_memory=True)
        self.pin_labels = torch.zeros(B, dtype=torch.int32, pin_memory=True)
        self.plan_in = _Plan(self.m_in, B, shift=0, layout="chunk")
        self.plan_rec = _Plan(self.m_rec, B, shift=0, layout="chunk")
        self._segs = (_lib.EpropSeg * 2)()
        # replica-minor copies of one group's e-prop inputs (sw_eprop_prep):
        # [K][rows][ldb], and the pass kernel's split partials / tickets
        K, L = EPROP_BLOCK_STEPS, self.plan_in.ldb
        self.zbar_t = torch.zeros((K, H, L), **f32)
        # psi and lsig interleaved per 4-replica group ([K][H][L/4][2][4]):
        # the pass reads both with one 32-byte load (sw_eprop_tpass_t.psl)
        self.psl_t = torch.zeros((K, H, 2 * L), **f32)
        self._tsegs = (_lib.EpropTSeg * 2)()
        # the trial's input side (sw_clf_inputs, once per batch): spike words
        # for the forward pass and the input traces in the e-prop layout
        T = self.task.example_steps
        self._in_words = (NI + 31) // 32
        self.in_bits = torch.zeros((T, B, self._in_words), dtype=torch.int32, device="cuda")
        # hidden spike words of one grouped launch (its readout runs after it)
        self.z_bits = torch.zeros((2 * EPROP_BLOCK_STEPS, B, (self.hidden + 31) // 32), dtype=torch.int32,
                                  device="cuda")
        self.xbar_all = torch.zeros((T, NI, L), **f32)
        nb = int(_lib.lib().sw_eprop_prep_scratch_bytes(K, B, H, C))
        self._ro_partial = torch.zeros(nb // 8 + 1, **f64)
        self._pass_scratch = None
        self._pass_scratch_key = None
        self._empty_segs = (_lib.EpropSeg * 2)()
        # split readout-gradient partials of the blocked e-prop pass
        self._ro_splits = READOUT_SPLITS
        nbytes = int(_lib.lib().sw_eprop_readout_scratch_bytes(H, C, self._ro_splits))
        self._ro_scratch = torch.zeros(nbytes // 8 + 1, **f64)
        _lib.workspace()   # allocate the ticket words outside any graph capture

    # -- per-step launches ------------------------------------------------------------
    def _step_params(self, t: int) -> _lib.ClfStep:
        p = self.params
        s = _lib.ClfStep()
        mi, mr = self.m_in, self.m_rec
        s.in_row_length, s.in_target, s.in_w32 = mi.row_length.data_ptr(), mi.target.data_ptr(), self.w32_in.data_ptr()
        s.in_stride, s.num_inputs = mi.stride, self.task.num_inputs
        s.rec_row_length, s.rec_target, s.rec_w32 = mr.row_length.data_ptr(), mr.target.data_ptr(), self.w32_rec.data_ptr()
        s.rec_stride, s.hidden = mr.stride, self.hidden
        s.w_out, s.b_out, s.num_classes = self.w_out.data_ptr(), self.b_out.data_ptr(), self.task.num_classes
        s.p_in, s.ex_key, s.labels = self.p_in.data_ptr(), self.keys.data_ptr(), self.labels.data_ptr()
        s.t, s.batch = t, self.local_b
        cur, prev = self._slot(t), self._slot(t - 1)
        s.v, s.a, s.z = (x.data_ptr() for x in (self.v, self.a, self.z))
        s.zbar, s.xbar = cur["zbar"].data_ptr(), cur["xbar"].data_ptr()
        s.zbar_in, s.xbar_in = prev["zbar"].data_ptr(), prev["xbar"].data_ptr()
        s.y, s.pi_sum, s.loss = (x.data_ptr() for x in (self.y, self.pi_sum, self.loss_b))
        s.d, s.psi, s.lsig = cur["d"].data_ptr(), cur["psi"].data_ptr(), cur["lsig"].data_ptr()
        s.alpha, s.rho = float(np.float32(p.alpha)), float(np.float32(p.rho))
        s.beta, s.v_thr = float(np.float32(p.beta)), float(np.float32(p.v_thr))
        s.alpha64 = p.alpha
        s.in_tw, s.rec_tw = self.tw_in.data_ptr(), self.tw_rec.data_ptr()
        s.in_tw_stride, s.rec_tw_stride = self._tw_stride["in"], self._tw_stride["rec"]
        return s

    def _group_params(self, t0: int, k: int) -> _lib.ClfStep:
        """One launch for steps t0 .. t0+k-1 (sw_clf_step with n_steps = k)
        over the contiguous slot arrays."""
        s = self._step_params(t0)
        s.zbar, s.xbar = self._slots_zbar.data_ptr(), self._slots_xbar.data_ptr()
        s.psi, s.lsig, s.d = (self._slots_psi.data_ptr(), self._slots_lsig.data_ptr(),
                              self._slots_d.data_ptr())
        s.zbar_in = s.xbar_in = 0
        s.n_steps, s.slot_count = k, 2 * EPROP_BLOCK_STEPS
        # the learning signal is computed by sw_eprop_prep, directly in the
        # e-prop pass's layout (the forward pass never reads it); the input
        # spikes and traces come from sw_clf_inputs
        s.lsig = 0
        s.in_bits, s.in_words = self.in_bits.data_ptr(), self._in_words
        s.z_bits = self.z_bits.data_ptr()
        return s

    def _slot(self, t: int) -> dict:
        k = t % (2 * EPROP_BLOCK_STEPS)
        return dict(zbar=self._slot_zbar[k], xbar=self._slot_xbar[k], psi=self._slot_psi[k],
                    lsig=self._slot_lsig[k], d=self._slot_d[k])

    def _pass_scratch_ptr(self) -> int:
        key = (self.plan_in.e_pad, self.plan_rec.e_pad)
        if self._pass_scratch_key != key:
            nb = int(_lib.lib().sw_eprop_pass_scratch_bytes(sum(key), self.plan_in.ldb))
            self._pass_scratch = torch.zeros(nb // 8 + 1, dtype=torch.float64, device="cuda")
            self._pass_scratch_key = key
        return self._pass_scratch.data_ptr()

    @property
    def psi_t(self) -> torch.Tensor:
        """[K, H, ldb] replica-minor psi of the last e-prop group (a copy out
        of the interleaved psl_t)."""
        K, H, L2 = self.psl_t.shape
        return self.psl_t.view(K, H, L2 // 8, 2, 4)[:, :, :, 0, :].reshape(K, H, L2 // 2)

    @property
    def lsig_t(self) -> torch.Tensor:
        """[K, H, ldb] replica-minor learning signal of the last e-prop group
        (a copy out of the interleaved psl_t)."""
        K, H, L2 = self.psl_t.shape
        return self.psl_t.view(K, H, L2 // 8, 2, 4)[:, :, :, 1, :].reshape(K, H, L2 // 2)

    def _eprop_block(self, t0: int, k: int, st: int, state_zero: bool | None = None) -> None:
        """e-prop of steps t0 .. t0+k-1: sw_eprop_prep (replica-minor copies,
        the learning signal and the readout gradients, classifier.py:221-223)
        and one sw_eprop_pass over both projections.  The trial's first pass
        (t0 = 0 unless state_zero says otherwise) starts eps/ebar from zero
        without reading them."""
        p = self.params
        a32, r32, b32 = float(np.float32(p.alpha)), float(np.float32(p.rho)), float(np.float32(p.beta))
        B, L = self.local_b, self.plan_in.ldb
        pr = _lib.EpropPrep()
        pr.k, pr.batch, pr.ldb = k, B, L
        pr.num_inputs, pr.hidden, pr.num_classes = self.task.num_inputs, self.hidden, self.task.num_classes
        tp = _lib.EpropTPass()
        tp.k = k
        for j in range(k):
            sl = self._slot(t0 + j)
            pr.xbar[j], pr.zbar[j] = 0, sl["zbar"].data_ptr()   # xbar_t: precomputed
            pr.psi[j], pr.d[j] = sl["psi"].data_ptr(), sl["d"].data_ptr()
            tp.psi_t[j], tp.lsig_t[j] = self.psl_t[j].data_ptr(), 0
        pr.w_out = self.w_out.data_ptr()
        pr.xbar_t, pr.zbar_t = 0, self.zbar_t.data_ptr()
        pr.psi_t, pr.lsig_t, pr.psl_t = 0, 0, self.psl_t.data_ptr()
        tp.psl = 1
        pr.g_w_out, pr.g_b_out = self.g_w_out.data_ptr(), self.g_b_out.data_ptr()
        pr.ro_partial = self._ro_partial.data_ptr()
        pr.defer_reduce = 1   # readout partials summed once per batch (_finish)
        _lib.call("sw_eprop_prep", ctypes.byref(pr), st)
        self._tsegs[0] = self.plan_in.tseg([self.xbar_all[t0 + j] for j in range(k)])
        self._tsegs[1] = self.plan_rec.tseg([self.zbar_t[j] for j in range(k)])
        tp.scratch = self._pass_scratch_ptr()
        tp.defer_reduce = 1   # split partials summed into the gradients once per batch (_finish)
        tp.state_zero = int(t0 == 0 if state_zero is None else state_zero)
        _lib.call("sw_eprop_pass", ctypes.cast(self._tsegs, ctypes.c_void_p), 2, ctypes.byref(tp),
                  L, b32, r32, a32, st)


    def eprop_pass_graph(self, reps: int) -> "torch.cuda.CUDAGraph":
        """A CUDA graph of `reps` blocked e-prop passes over steps 0..K-1 on
        the live state (kernel timing without host launch overhead)."""
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                st = torch.cuda.current_stream().cuda_stream
                for _ in range(reps):
                    self._eprop_block(0, EPROP_BLOCK_STEPS, st, state_zero=False)
        torch.cuda.current_stream().wait_stream(side)
        return g

    def eprop_kernel_graph(self, reps: int, part: str = "pass") -> "torch.cuda.CUDAGraph":
        """A CUDA graph of `reps` launches of one part of the e-prop group over
        steps 0..K-1 on the live state: "pass" (sw_eprop_pass, the dominant
        kernel) or "prep" (sw_eprop_prep), for per-kernel timing."""
        calls = []
        orig = _lib.call

        def rec(name, *args):
            calls.append((name, args))
            return orig(name, *args)
        _lib.call = rec
        try:
            self._eprop_block(0, EPROP_BLOCK_STEPS, _lib.stream_ptr(), state_zero=False)
        finally:
            _lib.call = orig
        want = "sw_eprop_pass" if part == "pass" else "sw_eprop_prep"
        name, args = next(c for c in calls if c[0] == want)
        keep = (self._tsegs, )   # ctypes buffers referenced by the recorded args stay alive
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                st = torch.cuda.current_stream().cuda_stream
                for _ in range(reps):
                    orig(name, *args[:-1], st)
        torch.cuda.current_stream().wait_stream(side)
        g._sw_keep = (keep, args)
        return g

    def _launch_steps(self, learn: bool, overlap: bool = False) -> None:
        """One trial: one launch running the forward pass of K =
        EPROP_BLOCK_STEPS steps, then one e-prop pass over those K steps
        (temporal blocking).  overlap
        (graph capture only): forward passes on the capturing stream, e-prop
        passes on a side stream, so the forward passes of group g+1 run while
        group g's e-prop pass streams the eligibility state; group g+2's
        forward passes wait for group g's e-prop (rotating slots)."""
        T = self.task.example_steps
        K = EPROP_BLOCK_STEPS
        groups = [(t0, min(K, T - t0)) for t0 in range(0, T, K)]
        if not (learn and overlap):
            st = _lib.stream_ptr()
            for t0, k in groups:
                prm = self._group_params(t0, k)
                _lib.call("sw_clf_step", ctypes.byref(prm), st)
                if learn:
                    self._eprop_block(t0, k, st)
            self.steps_launched += T
            return
        main = torch.cuda.current_stream()
        side = self._side_stream
        side.wait_stream(main)
        fwd_done = [torch.cuda.Event() for _ in groups]
        upd_done = [torch.cuda.Event() for _ in groups]
        for g, (t0, k) in enumerate(groups):
            if g >= 2:
                main.wait_event(upd_done[g - 2])
            prm = self._group_params(t0, k)
            _lib.call("sw_clf_step", ctypes.byref(prm), main.cuda_stream)
            fwd_done[g].record(main)
            side.wait_event(fwd_done[g])
            self._eprop_block(t0, k, side.cuda_stream)
            upd_done[g].record(side)
        main.wait_stream(side)
        self.steps_launched += T

    def kernels_per_trial(self, learn: bool = True) -> int:
        """Per EPROP_BLOCK_STEPS timesteps: the grouped forward launch and its
        readout launch, and (learning) the e-prop prep and pass (their
        reductions run once per batch)."""
        T = self.task.example_steps
        groups = -(-T // EPROP_BLOCK_STEPS)
        return groups * (4 if learn else 2)

    def _run_trial(self, learn: bool) -> None:
        if not self.use_graph:
            self._launch_steps(learn)
            return
        if self._graph is None or self._graph_learn != learn or self._graph_key != self._buffers_key():
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            self._side_stream = torch.cuda.Stream()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._launch_steps(learn, overlap=self.overlap)
            torch.cuda.current_stream().wait_stream(s)
            self._graph, self._graph_learn, self._graph_key = g, learn, self._buffers_key()
            self.steps_launched -= self.task.example_steps   # capture is not execution
        self._graph.replay()
        self.steps_launched += self.task.example_steps

    def _buffers_key(self):
        return (self.plan_in.e_pad, self.plan_rec.e_pad, self.plan_in.pre.data_ptr(),
                self.plan_rec.pre.data_ptr())

    # -- batch ------------------------------------------------------------------------
    def host_inputs(self, batch_index: int):
        """Host-side inputs of a training batch (numpy): p [B,NI], keys, labels."""
        return self.task.batch_inputs(self.task.train_ids(batch_index, self.batch_size))

    def _upload_batch(self, ids, host=None) -> None:
        p, keys, labels = host if host is not None else self.task.batch_inputs(ids)
        if isinstance(p, torch.Tensor) and p.is_pinned():
            # inputs already in pinned host memory (a pin_memory data
            # loader): asynchronous host->device copies, no staging
            loc = self.local
            self.p_in.copy_(p[loc], non_blocking=True)
            self.keys.copy_(keys[loc], non_blocking=True)
            self.labels.copy_(labels[loc], non_blocking=True)
            self.h2d_bytes = sum(int(x[loc].numel() * x.element_size()) for x in (p, keys, labels))
            return
        self.pin_p.copy_(torch.from_numpy(p[self.local]))
        self.pin_keys.copy_(torch.from_numpy(keys[self.local].view(np.int64)))
        self.pin_labels.copy_(torch.from_numpy(labels[self.local]))
        self.p_in.copy_(self.pin_p, non_blocking=True)
        self.keys.copy_(self.pin_keys, non_blocking=True)
        self.labels.copy_(self.pin_labels, non_blocking=True)
        self.h2d_bytes = p[self.local].nbytes + keys[self.local].nbytes + labels[self.local].nbytes

    def set_inputs_device(self, p: torch.Tensor, keys: torch.Tensor, labels: torch.Tensor) -> None:
        """Batch inputs already resident in HBM (device-to-device copy)."""
        self.p_in.copy_(p[self.local])
        self.keys.copy_(keys[self.local])
        self.labels.copy_(labels[self.local])

    def _prepare(self, learn: bool) -> None:
        st = _lib.stream_ptr()
        _lib.call("sw_f64_to_f32", self.s_in.planes["w"].data_ptr(), self.w32_in.data_ptr(),
                  self.w32_in.numel(), st)
        _lib.call("sw_f64_to_f32", self.s_rec.planes["w"].data_ptr(), self.w32_rec.data_ptr(),
                  self.w32_rec.numel(), st)
        for m, syn, tw, key in ((self.m_in, self.s_in, self.tw_in, "in"), (self.m_rec, self.s_rec, self.tw_rec, "rec")):
            _lib.call("sw_clf_pack_rows", m.row_length.data_ptr(), m.target.data_ptr(),
                      syn.planes["w"].data_ptr(), m.num_pre, m.stride, self._tw_stride[key], tw.data_ptr(), st)
        # per-batch state resets in one launch (eps/ebar: the trial's first
        # e-prop pass starts them from zero)
        resets = (self.v, self.a, self.z, self.y, self.pi_sum, self.loss_b, self._slots_zbar, self._slots_xbar)
        ptrs = (ctypes.c_void_p * len(resets))(*[x.data_ptr() for x in resets])
        nbytes = (ctypes.c_int64 * len(resets))(*[x.numel() * x.element_size() for x in resets])
        _lib.call("sw_zero_ranges", ptrs, nbytes, len(resets), st)
        ip = _lib.ClfInputs()
        ip.steps, ip.batch, ip.ldb = self.task.example_steps, self.local_b, self.plan_in.ldb
        ip.num_inputs, ip.words = self.task.num_inputs, self._in_words
        ip.p_in, ip.ex_key = self.p_in.data_ptr(), self.keys.data_ptr()
        ip.alpha = float(np.float32(self.params.alpha))
        ip.xbar_t, ip.in_bits = self.xbar_all.data_ptr(), self.in_bits.data_ptr()
        _lib.call("sw_clf_inputs", ctypes.byref(ip), st)
        if learn:
            for plan, syn in ((self.plan_in, self.s_in), (self.plan_rec, self.s_rec)):
                plan.ensure(plan.m.edge_count())
                plan.build()
                _lib.call("sw_gather_f64", syn.planes["grad"].data_ptr(), plan.off.data_ptr(),
                          plan.e_pad, plan.grad.data_ptr(), st)

    def reduce_partials(self) -> None:
        """Add the batch's deferred e-prop split partials and readout partials
        to the gradients (sw_eprop_pass_reduce / sw_eprop_prep_reduce; both
        zero the partials for the next batch)."""
        st = _lib.stream_ptr()
        if self._pass_scratch is not None:
            self._tsegs[0] = self.plan_in.tseg([])
            self._tsegs[1] = self.plan_rec.tseg([])
            _lib.call("sw_eprop_pass_reduce", ctypes.cast(self._tsegs, ctypes.c_void_p), 2, self.plan_in.ldb,
                      self._pass_scratch.data_ptr(), st)
        pr = _lib.EpropPrep()
        pr.k, pr.batch, pr.ldb = EPROP_BLOCK_STEPS, self.local_b, self.plan_in.ldb
        pr.num_inputs, pr.hidden, pr.num_classes = self.task.num_inputs, self.hidden, self.task.num_classes
        pr.g_w_out, pr.g_b_out = self.g_w_out.data_ptr(), self.g_b_out.data_ptr()
        pr.ro_partial = self._ro_partial.data_ptr()
        _lib.call("sw_eprop_prep_reduce", ctypes.byref(pr), st)

    def _finish(self, learn: bool):
        st = _lib.stream_ptr()
        if learn:
            self.reduce_partials()
            for plan, syn in ((self.plan_in, self.s_in), (self.plan_rec, self.s_rec)):
                _lib.call("sw_scatter_f64", syn.planes["grad"].data_ptr(), plan.off.data_ptr(),
                          plan.e_pad, plan.grad.data_ptr(), st)
        _lib.call("sw_clf_batch_stats", self.loss_b.data_ptr(), self.pi_sum.data_ptr(),
                  self.labels.data_ptr(), self.local_b, self.task.num_classes,
                  self.stats.data_ptr(), st)

    def _forward_batch(self, ids, learn: bool, host=None, resident: bool = False):
        if not resident:
            self._upload_batch(ids, host)
        self._prepare(learn)
        self._run_trial(learn)
        self._finish(learn)

    def _allreduce_grads(self) -> None:
        """Batch-DP: sum raw gradients and batch statistics over ranks
        (classifier.py:242-246 order: reduce, then scale)."""
        allreduce_flat([self.s_in.planes["grad"], self.s_rec.planes["grad"], self.g_w_out,
                        self.g_b_out, self.stats], group=self.pg)

    def gradient_phase(self, batch_index: int, host=None, resident: bool = False
                       ) -> tuple[float, float]:
        """Forward + e-prop over one batch, gradient scaling, L1 and Adam
        (classifier.py:236-253).  ``host`` = precomputed host inputs;
        ``resident`` = the batch inputs are already in HBM (benchmarking)."""
        ids = self.task.train_ids(batch_index, self.batch_size)
        self._forward_batch(ids, learn=True, host=host, resident=resident)
        return self.update_phase(batch_index)

    def update_phase(self, batch_index: int) -> tuple[float, float]:
        """The part of gradient_phase after the trial (classifier.py:236-253):
        (batch-DP all-reduce,) loss/accuracy read-back, 1/B gradient scale,
        L1 nudge and Adam on every parameter."""
        if self.pg is not None:
            self._allreduce_grads()
        self.stats_host.copy_(self.stats, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        loss = float(self.stats_host[0]) / (self.batch_size * self.task.example_steps)
        accuracy = float(self.stats_host[1]) / self.batch_size
        if not math.isfinite(loss):
            raise FloatingPointError(f"loss diverged at batch {batch_index}")
        st = _lib.stream_ptr()
        inv_b = 1.0 / self.batch_size
        for t in (self.s_in.planes["grad"], self.s_rec.planes["grad"], self.g_w_out, self.g_b_out):
            _lib.call("sw_scale_f64", t.data_ptr(), t.numel(), inv_b, st)
        if self.deep_r_enabled:
            self.deep_r_in.l1_step()
            self.deep_r_rec.l1_step()
        self.adam_in.apply(self.s_in.planes["w"], self.s_in.planes["grad"])
        self.adam_rec.apply(self.s_rec.planes["w"], self.s_rec.planes["grad"])
        self.adam_out.apply(self.w_out, self.g_w_out)
        self.adam_b.apply(self.b_out, self.g_b_out)
        return loss, accuracy

    def rewire_phase(self) -> int:
        if not self.deep_r_enabled:
            return 0
        self.net.run_update_group("deep_r")
        return self.deep_r_in.last_removed + self.deep_r_rec.last_removed

    def train_batch(self, batch_index: int, host=None, resident: bool = False) -> dict:
        loss, accuracy = self.gradient_phase(batch_index, host, resident)
        removed = self.rewire_phase()
        total = self.m_in.edge_count() + self.m_rec.edge_count()
        metrics = {"batch": batch_index, "loss": loss, "accuracy": accuracy,
                   "removed": removed, "total": total,
                   "fraction_rewired": removed / total if total else 0.0}
        self.history.append(metrics)
        return metrics

    def evaluate(self, example_ids) -> float:
        correct = count = 0
        for start in range(0, len(example_ids), self.batch_size):
            ids = list(example_ids[start:start + self.batch_size])
            real = len(ids)
            if real < self.batch_size:
                ids += [ids[-1]] * (self.batch_size - real)
            self._forward_batch(ids, learn=False)
            pred = self.pi_sum.argmax(dim=1).cpu().numpy()
            labels = np.array([self.task.label(e) for e in ids])[self.local]
            lo = self.local.start
            keep = min(max(real - lo, 0), self.local_b)
            correct += int((pred[:keep] == labels[:keep]).sum())
            count += keep
        return correct / count if count else 0.0

    def run(self, num_batches: int, stop_at_accuracy: float | None = None) -> list[dict]:
        for b in range(num_batches):
            m = self.train_batch(b)
            if stop_at_accuracy is not None and m["accuracy"] >= stop_at_accuracy:
                break
        return self.history

    def connectivity_fingerprint(self) -> bytes:
        parts = []
        for m in (self.m_in, self.m_rec):
            parts.append(m.row_length.cpu().numpy().tobytes())
            parts.append((m.target * m.slot_mask()).cpu().numpy().tobytes())
        return b"".join(parts)
