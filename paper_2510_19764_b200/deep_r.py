"""DEEP R rewiring at constant sparsity on the device (``sparsewire/deep_r.py``).

Same class, constructor and methods as the reference (deep_r.py:23-177);
the eliminate and form rules run as sm_100a kernels:

* eliminate (deep_r.py:81-99): warp per row, sign-mismatch scan, exact
  chained swap-with-last removal, conn-bit clears, ``dormant`` per row;
* form (deep_r.py:110-160): the serial host draw loop becomes a device
  histogram of the same counters; the per-row rejection placement runs warp
  per row over 32 consecutive counters at a time with the reference's exact
  draw accounting; the pass loop and its stall error stay on the host, one
  16-byte read per pass.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .bitfield import Bitfield
from .connectivity import RaggedMatrix, SynVarMatrix, descriptor
from .errors import RowFull
from .rng import CounterRng
from .updates import RuleDescriptor


class DeepR:
    def __init__(self, matrix: RaggedMatrix, syn: SynVarMatrix, name: str,
                 weight_plane: str = "w", grad_plane: str = "grad",
                 l1_strength: float = 0.005, exclude_diagonal: bool = False):
        self.matrix = matrix
        self.syn = syn
        self.name = name
        self.weight_plane = weight_plane
        self.grad_plane = grad_plane
        self.l1_strength = l1_strength
        self.exclude_diagonal = exclude_diagonal
        P, dev = matrix.num_pre, matrix.target.device
        self.sign_bits = Bitfield(P, matrix.num_post)
        self.conn_bits = Bitfield(P, matrix.num_post)
        self.dormant = torch.zeros(P, dtype=torch.int64, device=dev)
        self._unplaced = torch.zeros(P, dtype=torch.int64, device=dev)
        self._activations = torch.zeros(P, dtype=torch.int32, device=dev)
        self._counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self._counters_host = torch.zeros(4, dtype=torch.int64, pin_memory=True)
        self._last_removed_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self._no_progress_passes = 0
        # slot-aligned copy of the sign bits (derived; rebuilt when the matrix
        # was changed by anything but this rule pair)
        self._sign_slot = torch.zeros((P, (matrix.stride + 31) // 32), dtype=torch.int32, device=dev)
        # per-row marked-slot bitmasks between the eliminate scan and removal kernels
        self._marks = torch.zeros_like(self._sign_slot)
        self._cache_version = None

    # -- helpers ---------------------------------------------------------------
    def _desc(self):
        return descriptor(self.matrix, self.syn)

    def _plane(self, name):
        return self.syn.plane_index(name)

    def _sync_cache(self) -> int:
        if self._cache_version != self.matrix.version:
            d = self._desc()
            _lib.call("sw_deepr_sign_cache_build", ctypes.byref(d),
                      ctypes.byref(self.sign_bits.descriptor()), self._sign_slot.data_ptr(),
                      _lib.stream_ptr())
            self._cache_version = self.matrix.version
        return self._sign_slot.data_ptr()

    @property
    def last_removed(self) -> int:
        return int(self._last_removed_dev.item())

    @last_removed.setter
    def last_removed(self, v: int) -> None:
        self._last_removed_dev.fill_(int(v))

    # -- initialisation (deep_r.py:50-64) ----------------------------------------
    def init_bitfields(self, rng: CounterRng) -> None:
        d = self._desc()
        key = (rng.key + rng.counter * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        _lib.call("sw_deepr_init_bitfields", ctypes.byref(d), self._plane(self.weight_plane),
                  ctypes.byref(self.sign_bits.descriptor()),
                  ctypes.byref(self.conn_bits.descriptor()), key, _lib.stream_ptr())
        rng.counter += self.sign_bits.words.numel()
        self._cache_version = None

    # -- L1 nudge (deep_r.py:68-77) ------------------------------------------------
    def l1_step(self) -> None:
        if self.l1_strength == 0.0:
            return
        d = self._desc()
        _lib.call("sw_deepr_l1", ctypes.byref(d), self._plane(self.grad_plane),
                  ctypes.byref(self.sign_bits.descriptor()), self._sync_cache(),
                  float(self.l1_strength), _lib.stream_ptr())

    # -- eliminate rule ----------------------------------------------------------------
    def _eliminate_pass(self, model, binding, pass_index, host_key, row_base) -> bool:
        d = self._desc()
        _lib.call("sw_deepr_eliminate", ctypes.byref(d), self._plane(self.weight_plane),
                  ctypes.byref(self.sign_bits.descriptor()),
                  ctypes.byref(self.conn_bits.descriptor()), self.dormant.data_ptr(),
                  self._sync_cache(), self._marks.data_ptr(), _lib.stream_ptr())
        # the removal count is known on the host only at the form pass (its
        # one counter read per pass): the version bump for this pass's
        # removals happens there, so a no-op update leaves derived
        # structures (TransposeMap, PropBuckets) fresh (updates.py:367-372)
        self._cache_version = self.matrix.version
        return False

    def eliminate_rule(self) -> RuleDescriptor:
        return RuleDescriptor(name=f"{self.name}_eliminate", device_pass=self._eliminate_pass)

    # -- form rule ------------------------------------------------------------------------
    def _form_pass(self, model, binding, pass_index, host_key, row_base) -> bool:
        d = self._desc()
        src = self.dormant if pass_index == 0 else self._unplaced
        if pass_index == 0:
            self._no_progress_passes = 0
        _lib.call("sw_deepr_form_pass", ctypes.byref(d),
                  ctypes.byref(self.conn_bits.descriptor()), int(self.exclude_diagonal),
                  src.data_ptr(), host_key, row_base, self._activations.data_ptr(),
                  self._unplaced.data_ptr(), self._counters.data_ptr(),
                  ctypes.byref(self.sign_bits.descriptor()), self._sync_cache(),
                  _lib.stream_ptr())
        if pass_index == 0:
            self._last_removed_dev.copy_(self._counters[0:1])
        # _form_continue (deep_r.py:147-160): one 32-byte read per pass
        self._counters_host.copy_(self._counters, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        drawn, unplaced = int(self._counters_host[0]), int(self._counters_host[1])
        # version: bumped only when the structure changed -- pass 0 with
        # removals (the eliminate pass's change), or any pass placing synapses
        if (pass_index == 0 and drawn > 0) or drawn - unplaced > 0:
            self.matrix.version += 1
        self._cache_version = self.matrix.version
        if unplaced == 0:
            return False
        if drawn - unplaced == 0:
            self._no_progress_passes += 1
            if self._no_progress_passes >= self.matrix.num_pre:
                raise RowFull(f"{self.name}: could not place {unplaced} new synapses "
                              f"after {self._no_progress_passes} stalled passes")
        else:
            self._no_progress_passes = 0
        return True

    def form_rule(self) -> RuleDescriptor:
        return RuleDescriptor(name=f"{self.name}_form", device_pass=self._form_pass)

    def register(self, model, group: str, matrix_name: str) -> None:
        model.add_rule(group, matrix_name, self.eliminate_rule())
        model.add_rule(group, matrix_name, self.form_rule())

    def rewiring_fraction(self) -> float:
        total = self.matrix.edge_count()
        return self.last_removed / total if total else 0.0

    # -- state transfer --------------------------------------------------------------------
    def load_state(self, sign_words: np.ndarray, conn_words: np.ndarray) -> None:
        self.sign_bits.load_words(sign_words)
        self.conn_bits.load_words(conn_words)
        self._cache_version = None
