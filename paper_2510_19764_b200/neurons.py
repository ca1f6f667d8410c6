"""Neuron and input models with device state (``sparsewire/neurons.py``).

``AlifLayer`` (float32, :46-73) and ``LifCondLayer`` (float64, :121-148)
keep their state as CUDA tensors and step through sm_100a kernels;
``PoissonSource`` (:151-195) draws its spikes on the device from the
reference's counters (step*n + node).  Rates and the Bernoulli
probabilities come from host numpy (exp).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .rng import CounterRng


@dataclass
class AlifParams:
    tau_mem: float = 20.0
    tau_adapt: float = 2000.0
    beta: float = 0.0174
    v_thr: float = 0.6
    dt: float = 1.0

    @property
    def alpha(self) -> float:
        return math.exp(-self.dt / self.tau_mem)

    @property
    def rho(self) -> float:
        return math.exp(-self.dt / self.tau_adapt)


class AlifLayer:
    """Adaptive LIF with soft reset; float32 device state [batch, n] or [n]."""

    def __init__(self, n: int, params: AlifParams | None = None, batch: int | None = None,
                 dtype=torch.float32):
        if dtype not in (torch.float32, np.float32):
            raise TypeError("the device ALIF layer computes in float32 (the classifier dtype)")
        _lib.require_cuda()
        self.n = n
        self.params = params or AlifParams()
        shape = (n,) if batch is None else (batch, n)
        self.v = torch.zeros(shape, dtype=torch.float32, device="cuda")
        self.a = torch.zeros_like(self.v)
        self.z = torch.zeros_like(self.v)

    def reset(self) -> None:
        self.v.zero_()
        self.a.zero_()
        self.z.zero_()

    def consts(self):
        p = self.params
        return (float(np.float32(p.alpha)), float(np.float32(p.rho)), float(np.float32(p.beta)),
                float(np.float32(p.v_thr)))

    def step(self, rec_input: torch.Tensor, ext_input: torch.Tensor):
        a, r, b, vt = self.consts()
        rec_input = rec_input.to(torch.float32).contiguous()
        ext_input = ext_input.to(torch.float32).contiguous()
        _lib.call("sw_alif_step", self.v.data_ptr(), self.a.data_ptr(), self.z.data_ptr(),
                  rec_input.data_ptr(), ext_input.data_ptr(), self.v.numel(), a, r, b, vt,
                  _lib.stream_ptr())
        if self.v.ndim == 1:
            return torch.nonzero(self.z).flatten()
        return None

    def surrogate(self) -> torch.Tensor:
        _, _, b, vt = self.consts()
        psi = torch.empty_like(self.v)
        _lib.call("sw_alif_surrogate", self.v.data_ptr(), self.a.data_ptr(), psi.data_ptr(),
                  self.v.numel(), b, vt, _lib.stream_ptr())
        return psi


@dataclass
class LifCondParams:
    c_m: float = 20.0
    tau_m: float = 20.0
    v_rest: float = -70.0
    e_exc: float = 0.0
    v_theta: float = -54.0
    v_reset: float = -70.0
    tau_ref: float = 5.0
    tau_s: float = 5.0
    t_delay: float = 0.1
    h: float = 0.1

    @property
    def g_leak(self) -> float:
        return self.c_m / self.tau_m


def unpack_spike_bits(bits: torch.Tensor, n: int) -> torch.Tensor:
    """Ascending ids of set bits of a packed uint32 spike mask (device)."""
    b = bits.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    shifts = torch.arange(32, device=bits.device, dtype=torch.int64)
    flags = ((b[:, None] >> shifts[None, :]) & 1).flatten()[:n]
    return torch.nonzero(flags).flatten()


class LifCondLayer:
    """Conductance LIF with exponential-Euler integration (float64)."""

    def __init__(self, n: int, params: LifCondParams | None = None):
        _lib.require_cuda()
        self.n = n
        self.params = params or LifCondParams()
        p = self.params
        self.V = torch.full((n,), p.v_rest, dtype=torch.float64, device="cuda")
        self.g = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.refractory_until = torch.full((n,), -1, dtype=torch.int64, device="cuda")
        self._decay_s = math.exp(-p.h / p.tau_s)
        self._ref_steps = int(round(p.tau_ref / p.h))
        self.spike_bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")

    def step_bits(self, incoming: torch.Tensor, step_index: int) -> torch.Tensor:
        p = self.params
        _lib.call("sw_lif_cond_step", self.V.data_ptr(), self.g.data_ptr(),
                  self.refractory_until.data_ptr(), incoming.data_ptr(), self.n, step_index,
                  self._decay_s, p.g_leak, p.v_rest, p.e_exc, p.v_theta, p.v_reset, p.h, p.tau_m,
                  self._ref_steps, self.spike_bits.data_ptr(), _lib.stream_ptr())
        return self.spike_bits

    def step(self, incoming: torch.Tensor, step_index: int) -> torch.Tensor:
        return unpack_spike_bits(self.step_bits(incoming, step_index), self.n)


@dataclass
class PoissonParams:
    f_base: float = 5.0
    f_peak: float = 152.8
    sigma_stim: float = 2.0
    t_stim: float = 20.0


class PoissonSource:
    """Poisson spikes with spatially correlated rates on a torus grid."""

    def __init__(self, geometry, params: PoissonParams | None = None):
        _lib.require_cuda()
        self.geometry = geometry
        self.params = params or PoissonParams()
        self.rates = np.full(geometry.n, self.params.f_base, dtype=np.float64)
        self._p = None
        self._p_h = None
        self._p_dev = torch.zeros(geometry.n, dtype=torch.float64, device="cuda")
        self.spike_bits = torch.zeros((geometry.n + 31) // 32, dtype=torch.int32, device="cuda")

    def set_correlated_rates(self, centers) -> None:
        """neurons.py:175-183 on the host (numpy exp/hypot)."""
        p = self.params
        bump = np.zeros(self.geometry.n)
        for (cx, cy) in centers:
            d = self.geometry.distance_to_point(cx, cy)
            bump += np.exp(-(d * d) / (2.0 * p.sigma_stim ** 2))
        self.rates = p.f_base + p.f_peak * bump
        self._p = None

    def set_correlated_rates_device(self, centers, h: float) -> None:
        """Same rates computed on the device (CUDA exp/hypot; a few ulp from
        numpy): for large grids where the host loop over centres dominates."""
        c = np.asarray(centers, dtype=np.float64).reshape(-1)
        if not hasattr(self, "_rates_dev"):
            self._rates_dev = torch.zeros(self.geometry.n, dtype=torch.float64, device="cuda")
            self._centers_dev = torch.zeros(max(2, c.size), dtype=torch.float64, device="cuda")
        # fresh pinned staging per change: torch's host allocator keeps it alive
        # until the async copy has run
        self._centers_dev[:c.size].copy_(torch.from_numpy(c).pin_memory(), non_blocking=True)
        p = self.params
        _lib.call("sw_poisson_rates", self.geometry.side, self._centers_dev.data_ptr(), c.size // 2,
                  p.f_base, p.f_peak, p.sigma_stim, h, self._rates_dev.data_ptr(),
                  self._p_dev.data_ptr(), _lib.stream_ptr())
        self.rates = None        # host copy stale: see rates_array()
        self._p = "device"
        self._p_h = h

    def rates_array(self) -> np.ndarray:
        return self.rates.copy() if self.rates is not None else self._rates_dev.cpu().numpy()

    def set_uniform_rate(self, rate_hz: float) -> None:
        self.rates = np.full(self.geometry.n, rate_hz, dtype=np.float64)
        self._p = None

    def probabilities(self, h: float) -> torch.Tensor:
        if self._p is None or self._p_h != h:
            self._p = 1.0 - np.exp(-self.rates * h * 1e-3)
            self._p_h = h
            self._p_dev.copy_(torch.from_numpy(self._p))
        return self._p_dev

    def poisson_step_bits(self, rng: CounterRng, h: float) -> torch.Tensor:
        p = self.probabilities(h)
        n = self.geometry.n
        _lib.call("sw_poisson_step", rng.key, rng.counter, p.data_ptr(), n,
                  self.spike_bits.data_ptr(), _lib.stream_ptr())
        rng.counter += n
        return self.spike_bits

    def poisson_step(self, rng: CounterRng, h: float) -> torch.Tensor:
        return unpack_spike_bits(self.poisson_step_bits(rng, h), self.geometry.n)
