"""Structural-plasticity rule framework on the device
(the reference's ``sparsewire/updates.py`` API).

The reference runs a rule as a serial Python host phase plus a Python row
phase per presynaptic row (updates.py:309-372).  Arbitrary Python row
phases cannot run on the GPU, so here a rule supplies a ``device_pass``:
one call enqueues the rule's host phase AND its row phase for one pass as
sm_100a kernels (warp per row), with the reference's stream keys

    host:  fold_key(seed, "host", rule_id, update_count, pass)   updates.py:346-349
    rows:  child_key(fold_key(seed, "row", rule_id, update_count, pass), row)   :313-318

and returns whether the rule wants another pass (``continue_after_pass``).
Everything else — rule ids in registration order (:300-302), per-binding
update counters (:366), the runaway pass cap (:363-365), remap-if-changed
(:367-372), phase timers (:36-54) — follows the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch

from .connectivity import RaggedMatrix, SynVarMatrix
from .errors import DuplicateName, UnresolvedReference
from .rng import fold_key

PHASES = ("neuron_update", "presynaptic_update", "postsynaptic_update",
          "host_update", "row_update", "remap")


class PhaseTimers:
    """Per-phase device time from CUDA events (updates.py:36-54 semantics)."""

    def __init__(self):
        self._done = {p: 0.0 for p in PHASES}
        self._pending: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []
        self._open: dict[str, torch.cuda.Event] = {}
        self.enabled = True

    def start(self, phase: str) -> None:
        if self.enabled:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._open[phase] = ev

    def stop(self, phase: str) -> None:
        if self.enabled and phase in self._open:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._pending.append((phase, self._open.pop(phase), ev))

    def add(self, phase: str, seconds: float) -> None:
        self._done[phase] += seconds

    @property
    def seconds(self) -> dict[str, float]:
        if self._pending:
            self._pending[-1][2].synchronize()
            for ph, a, b in self._pending:
                self._done[ph] += a.elapsed_time(b) * 1e-3
            self._pending.clear()
        return dict(self._done)

    def total(self) -> float:
        return sum(self.seconds.values())

    def write_csv(self, fh) -> None:
        s = self.seconds
        fh.write("phase,seconds\n")
        for p in PHASES:
            fh.write(f"{p},{s[p]:.9f}\n")
        fh.write(f"total,{sum(s.values()):.9f}\n")


@dataclass
class RuleDescriptor:
    """Same fields as updates.py:57-81 plus ``device_pass``.

    ``device_pass(model, binding, pass_index, host_key, row_base) -> bool``
    enqueues one host+row pass on the device and returns True to request
    another pass.  Python ``host_phase``/``row_phase`` callables are not
    executable on the device and are rejected at registration.
    """

    name: str
    host_phase: Callable | None = None
    row_phase: Callable | None = None
    pre_vars: tuple = ()
    post_vars: tuple = ()
    syn_vars: tuple = ()
    var_refs: tuple = ()
    pre_var_refs: tuple = ()
    post_var_refs: tuple = ()
    active_rows: Callable | None = None
    continue_after_pass: Callable | None = None
    device_pass: Callable | None = None


class RuleBinding:
    __slots__ = ("rule", "rule_id", "matrix_name", "matrix", "syn",
                 "pre_arrays", "post_arrays", "update_count")

    def __init__(self, rule, rule_id, matrix_name, matrix, syn, pre_arrays, post_arrays):
        self.rule = rule
        self.rule_id = rule_id
        self.matrix_name = matrix_name
        self.matrix = matrix
        self.syn = syn
        self.pre_arrays = pre_arrays
        self.post_arrays = post_arrays
        self.update_count = 0


class Model:
    """Registry of matrices, arrays, transposes and rule groups (updates.py:231-372)."""

    def __init__(self, seed: int, workers: int = 1, always_remap: bool = False,
                 incremental_remap: bool = True):
        self.seed = seed
        self.workers = max(1, workers)   # accepted for API parity; the device is the worker pool
        self.always_remap = always_remap
        # rules with a patch log (RewiringRule) remap incrementally
        # (sw_transpose_patch); False: full rebuilds (updates.py:367-372)
        self.incremental_remap = incremental_remap
        self.timers = PhaseTimers()
        self.matrices: dict[str, tuple[RaggedMatrix, SynVarMatrix]] = {}
        self.arrays: dict[str, torch.Tensor] = {}
        self.groups: dict[str, list[RuleBinding]] = {}
        self.transposes: dict = {}
        self._rule_names: set[str] = set()
        self._next_rule_id = 0

    def add_matrix(self, name, matrix, syn):
        if name in self.matrices:
            raise DuplicateName(f"matrix {name!r} already registered")
        self.matrices[name] = (matrix, syn)
        return matrix, syn

    def add_array(self, name, arr):
        if name in self.arrays:
            raise DuplicateName(f"array {name!r} already registered")
        self.arrays[name] = arr
        return arr

    def register_transpose(self, matrix_name: str):
        from .transpose import TransposeMap
        matrix, _ = self.matrices[matrix_name]
        tm = self.transposes.get(matrix_name)
        if tm is None:
            tm = TransposeMap(matrix)
            tm.rebuild()
            self.transposes[matrix_name] = tm
        return tm

    def add_rule(self, group: str, matrix_name: str, rule: RuleDescriptor) -> RuleBinding:
        if matrix_name not in self.matrices:
            raise UnresolvedReference(f"matrix {matrix_name!r} not registered")
        if rule.name in self._rule_names:
            raise DuplicateName(f"rule {rule.name!r} already registered")
        if rule.device_pass is None:
            raise NotImplementedError(
                f"rule {rule.name!r} has no device_pass: Python row phases do not run on the "
                "GPU; use a built-in device rule (DeepR, RewiringRule)")
        matrix, syn = self.matrices[matrix_name]
        dev = matrix.target.device
        pre_arrays, post_arrays = {}, {}
        for name, dtype in rule.pre_vars:
            pre_arrays[name] = torch.zeros(matrix.num_pre, dtype=dtype, device=dev)
        for name, dtype in rule.post_vars:
            post_arrays[name] = torch.zeros(matrix.num_post, dtype=dtype, device=dev)
        for name, dtype in rule.syn_vars:
            syn.add_plane(name, dtype)
        for name in rule.var_refs:
            if name not in syn.planes:
                raise UnresolvedReference(
                    f"rule {rule.name!r}: synaptic plane {name!r} missing on {matrix_name!r}")
        for name in rule.pre_var_refs:
            a = self.arrays.get(name)
            if a is None or len(a) != matrix.num_pre:
                raise UnresolvedReference(f"rule {rule.name!r}: per-pre array {name!r} missing or wrong extent")
            pre_arrays[name] = a
        for name in rule.post_var_refs:
            a = self.arrays.get(name)
            if a is None or len(a) != matrix.num_post:
                raise UnresolvedReference(f"rule {rule.name!r}: per-post array {name!r} missing or wrong extent")
            post_arrays[name] = a
        b = RuleBinding(rule, self._next_rule_id, matrix_name, matrix, syn, pre_arrays, post_arrays)
        self._next_rule_id += 1
        self._rule_names.add(rule.name)
        self.groups.setdefault(group, []).append(b)
        return b

    def keys(self, binding: RuleBinding, pass_index: int) -> tuple[int, int]:
        return (fold_key(self.seed, "host", binding.rule_id, binding.update_count, pass_index),
                fold_key(self.seed, "row", binding.rule_id, binding.update_count, pass_index))

    def run_update_group(self, group: str, concurrent: bool = False) -> None:
        """Run every binding of the group (updates.py:323-372).  concurrent:
        the bindings (distinct matrices, their own keys and counters) are
        enqueued on separate streams joined at the end, so their device
        passes and remaps overlap (timers off: the phase events would mix)."""
        bindings = self.groups[group]
        if not concurrent or len(bindings) < 2 or self.timers.enabled:
            for b in bindings:
                self._run_binding(b)
            return
        main = torch.cuda.current_stream()
        sides = self._side_streams(len(bindings) - 1)
        for st in sides:
            st.wait_stream(main)
        for b, st in zip(bindings, [main] + sides):
            with torch.cuda.stream(st):
                self._run_binding(b)
        for st in sides:
            main.wait_stream(st)

    def _side_streams(self, n: int) -> list:
        if not hasattr(self, "_sides"):
            self._sides = []
        while len(self._sides) < n:
            self._sides.append(torch.cuda.Stream())
        return self._sides[:n]

    def _run_binding(self, b) -> None:
        rule = b.rule
        v0 = b.matrix.version
        p = 0
        while True:
            hk, rk = self.keys(b, p)
            self.timers.start("row_update")
            again = rule.device_pass(self, b, p, hk, rk)
            self.timers.stop("row_update")
            p += 1
            if not again:
                break
            if p > 2 * b.matrix.num_pre + 16:
                raise RuntimeError(f"rule {rule.name!r} did not converge after {p} passes")
        b.update_count += 1
        tm = self.transposes.get(b.matrix_name)
        if tm is not None and (self.always_remap or b.matrix.version != v0):
            self.timers.start("remap")
            src = getattr(rule, "patch_source", None)
            if src is not None and self.incremental_remap and not self.always_remap:
                # incremental: only the columns the update touched (sw_transpose_patch)
                tm.patch(src.patch_log, src.patch_cap)
            else:
                tm.rebuild(changed_flag=getattr(rule, "changed_flag", None) if not self.always_remap else None)
            self.timers.stop("remap")
