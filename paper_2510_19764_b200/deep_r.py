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
                 l1_strength: float = 0.005, exclude_diagonal: bool = False,
                 process_group=None, row0: int = 0, num_pre_global: int | None = None):
        """``process_group``/``row0``/``num_pre_global``: row sharding (SURVEY
        8e M-update).  ``matrix`` then holds rows [row0, row0 + num_pre) of a
        ``num_pre_global``-row matrix; every rank of the group runs the same
        update group and the result is bit-identical to one unsharded DeepR
        (see ``_form_pass_sharded``)."""
        self.matrix = matrix
        self.pg = process_group
        self.row0 = int(row0)
        self.num_pre_global = int(num_pre_global if num_pre_global is not None else matrix.num_pre)
        if self.pg is None and (self.row0 != 0 or self.num_pre_global != matrix.num_pre):
            raise ValueError("row0/num_pre_global need a process_group")
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
        self._act_full = None     # [num_pre_global] histogram (sharded form)

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
        if self.pg is not None:
            return self._form_pass_sharded(pass_index, host_key, row_base)
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
        return self._form_continue(pass_index, drawn, unplaced)

    def _form_continue(self, pass_index: int, drawn: int, unplaced: int) -> bool:
        """_form_continue (deep_r.py:147-160) on the pass's global counts."""
        if (pass_index == 0 and drawn > 0) or drawn - unplaced > 0:
            self.matrix.version += 1
        self._cache_version = self.matrix.version
        if unplaced == 0:
            return False
        if drawn - unplaced == 0:
            self._no_progress_passes += 1
            if self._no_progress_passes >= self.num_pre_global:
                raise RowFull(f"{self.name}: could not place {unplaced} new synapses "
                              f"after {self._no_progress_passes} stalled passes")
        else:
            self._no_progress_passes = 0
        return True

    def _form_pass_sharded(self, pass_index, host_key, row_base) -> bool:
        """Row-sharded form pass (SURVEY 8e M-update).  The D host draws of
        deep_r.py:110-121 are split into equal counter chunks, one per rank,
        each histogrammed over all rows; the histograms are reduce-scattered
        to the row owners, which place their rows with the global row's
        stream (deep_r.py:126-145).  D, the rejected-draw count and the
        unplaced count are all-reduced, so every rank takes the same
        pass-loop decision.  Integer sums throughout: bit-exact with the
        unsharded pass."""
        from .sharding import reduce_scatter_rows
        import torch.distributed as dist
        rank, world = dist.get_rank(self.pg), dist.get_world_size(self.pg)
        st = _lib.stream_ptr()
        src = self.dormant if pass_index == 0 else self._unplaced
        if pass_index == 0:
            self._no_progress_passes = 0
        P, PG = self.matrix.num_pre, self.num_pre_global
        if self._act_full is None:
            self._act_full = torch.zeros(PG, dtype=torch.int32, device=self.matrix.target.device)
        _lib.call("sw_deepr_form_pending", src.data_ptr(), P, self._counters.data_ptr(), st)
        dist.all_reduce(self._counters[0:1], group=self.pg)
        _lib.call("sw_deepr_form_hist_chunk", self._counters.data_ptr(), host_key, PG, rank, world,
                  self._act_full.data_ptr(), _lib.stream_ptr())
        dist.all_reduce(self._counters[2:3], group=self.pg)
        if rank == 0:
            _lib.call("sw_deepr_form_hist_fix", self._counters.data_ptr(), host_key, PG,
                      self._act_full.data_ptr(), _lib.stream_ptr())
        reduce_scatter_rows(self._act_full, self._activations, self.row0, self.pg)
        d = self._desc()
        _lib.call("sw_deepr_form_rows_shard", ctypes.byref(d), ctypes.byref(self.conn_bits.descriptor()),
                  int(self.exclude_diagonal), row_base, self.row0, self._activations.data_ptr(),
                  self._unplaced.data_ptr(), self._counters.data_ptr(),
                  ctypes.byref(self.sign_bits.descriptor()), self._sync_cache(), _lib.stream_ptr())
        dist.all_reduce(self._counters[1:2], group=self.pg)
        if pass_index == 0:
            self._last_removed_dev.copy_(self._counters[0:1])
        self._counters_host.copy_(self._counters, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        drawn, unplaced = int(self._counters_host[0]), int(self._counters_host[1])
        # structure changed somewhere: every rank bumps its version alike
        return self._form_continue(pass_index, drawn, unplaced)

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
