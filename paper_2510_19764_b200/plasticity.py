"""Weight-change rules on the device (``sparsewire/plasticity.py``):
Adam (:198-227) and the batched e-prop accumulation
(``sparsewire/_kernels.py:15-39``)."""

from __future__ import annotations

import torch

from . import _lib


class Adam:
    """Adam with bias correction; gradients are zeroed after application.

    Moments are float64 CUDA tensors (slot-aligned planes for synaptic
    parameters, so they follow rewiring).  Exact reference op order.
    """

    def __init__(self, lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-8, m: torch.Tensor | None = None,
                 v: torch.Tensor | None = None, shape=None):
        if m is None:
            m = torch.zeros(shape, dtype=torch.float64, device="cuda")
        if v is None:
            v = torch.zeros(shape, dtype=torch.float64, device="cuda")
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.m, self.v = m, v
        self.t = 0

    def apply(self, params: torch.Tensor, grads: torch.Tensor) -> None:
        for t in (params, grads, self.m, self.v):
            if t.dtype != torch.float64 or not t.is_contiguous() or not t.is_cuda:
                raise TypeError("Adam operates on contiguous float64 CUDA tensors")
        n = params.numel()
        if not (grads.numel() == self.m.numel() == self.v.numel() == n):
            raise ValueError("shape mismatch")
        self.t += 1
        c1 = 1.0 - self.beta1 ** self.t
        c2 = 1.0 - self.beta2 ** self.t
        _lib.call("sw_adam_f64", params.data_ptr(), grads.data_ptr(), self.m.data_ptr(),
                  self.v.data_ptr(), n, self.beta1, 1.0 - self.beta1, self.beta2,
                  1.0 - self.beta2, c1, c2, self.lr, self.eps, _lib.stream_ptr())


def eprop_accumulate_batch(targets, row_length, pre_trace, psi, lsig, eps, ebar, grad,
                           beta, rho, alpha) -> None:
    """Drop-in for ``sparsewire._kernels.eprop_accumulate_batch`` (:15-39) on
    CUDA tensors in the reference layout: targets [P,S] int32, row_length [P]
    int32, pre_trace [B,P] / psi, lsig [B,H] float32, eps, ebar [B,P,S]
    float32 (updated in place), grad [P,S] float64 (accumulated).  One thread
    per synapse, replicas ascending: bit-identical to the numba kernel."""
    for t, dt in ((targets, torch.int32), (row_length, torch.int32), (pre_trace, torch.float32),
                  (psi, torch.float32), (lsig, torch.float32), (eps, torch.float32),
                  (ebar, torch.float32), (grad, torch.float64)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise TypeError("eprop_accumulate_batch: wrong dtype/device/layout")
    P, S = targets.shape
    B = pre_trace.shape[0]
    H = psi.shape[1]
    _lib.call("sw_eprop_accumulate_batch", targets.data_ptr(), row_length.data_ptr(), P, S,
              pre_trace.data_ptr(), psi.data_ptr(), lsig.data_ptr(), B, H, eps.data_ptr(),
              ebar.data_ptr(), grad.data_ptr(), float(beta), float(rho), float(alpha),
              _lib.stream_ptr())


# ----------------------------------------------------------------------
# trace STDP (plasticity.py:42-95)
# ----------------------------------------------------------------------

from dataclasses import dataclass  # noqa: E402
import math  # noqa: E402


@dataclass
class StdpParams:
    g_max: float = 0.2
    w_min: float = 0.0
    w_max: float = 0.2
    a_plus: float = 0.1 * 0.2
    tau_plus: float = 20.0
    tau_minus: float = 64.0
    b_ratio: float = 1.2

    @property
    def a_minus(self) -> float:
        return self.b_ratio * self.a_plus * self.tau_plus / self.tau_minus


def _as_bits(spikes, n):
    from .connectivity import spikes_to_bits
    if spikes.dtype == torch.int32 and spikes.numel() == (n + 31) // 32:
        return spikes
    return spikes_to_bits(spikes, n)


class StdpSynapses:
    """Trace STDP on one projection; x [num_pre], y [num_post] float64 on the
    device.  Same event ordering as the reference (depression on pre spikes
    with y before this step's increments, then x += 1; potentiation on post
    spikes through the transpose, then y += 1)."""

    def __init__(self, matrix, syn, h: float, params: StdpParams | None = None,
                 weight_plane: str = "g"):
        self.matrix = matrix
        self.syn = syn
        self.params = params or StdpParams()
        self.weight_plane = weight_plane
        self.x = torch.zeros(matrix.num_pre, dtype=torch.float64, device="cuda")
        self.y = torch.zeros(matrix.num_post, dtype=torch.float64, device="cuda")
        self._decay_x = math.exp(-h / self.params.tau_plus)
        self._decay_y = math.exp(-h / self.params.tau_minus)

    def decay_step(self) -> None:
        _lib.call("sw_stdp_decay", self.x.data_ptr(), self.x.numel(), self._decay_x,
                  self.y.data_ptr(), self.y.numel(), self._decay_y, _lib.stream_ptr())

    def on_pre_spikes(self, pre) -> None:
        """``pre``: index tensor (ascending) or packed spike bits."""
        m, p = self.matrix, self.params
        bits = _as_bits(pre, m.num_pre)
        _lib.call("sw_stdp_pre", m.row_length.data_ptr(), m.target.data_ptr(),
                  self.syn.planes[self.weight_plane].data_ptr(), m.stride, m.num_pre,
                  bits.data_ptr(), self.y.data_ptr(), self.x.data_ptr(), p.a_minus, p.w_min,
                  p.w_max, _lib.stream_ptr())

    def on_post_spikes(self, tmap, post) -> None:
        tmap.check_fresh()
        m, p = self.matrix, self.params
        bits = _as_bits(post, m.num_post)
        _lib.call("sw_stdp_post", tmap.col_ptr.data_ptr(), tmap.col_length.data_ptr(), tmap.src_pre.data_ptr(),
                  tmap.src_slot.data_ptr(), self.syn.planes[self.weight_plane].data_ptr(),
                  m.stride, m.num_post, bits.data_ptr(), self.x.data_ptr(), self.y.data_ptr(),
                  p.a_plus, p.w_min, p.w_max, _lib.stream_ptr())
