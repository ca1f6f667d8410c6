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
