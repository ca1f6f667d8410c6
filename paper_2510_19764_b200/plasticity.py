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
