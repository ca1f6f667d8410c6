"""Column-indexed inverse of a device RaggedMatrix
(``sparsewire/connectivity.py:151-203`` TransposeMap), kept in HBM as CSR.

``rebuild`` runs the sm_100a counting-sort kernels; ``column``/``columns``
and the reference-layout ``source_pre``/``source_slot`` views copy to the
host for inspection and tests.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .connectivity import RaggedMatrix, descriptor
from .errors import StaleTranspose


class TransposeMap:
    """CSR with slack: column j = entries [col_ptr[j], col_ptr[j] + col_length[j]),
    room for SLACK more (incremental patches, sw_transpose_patch)."""

    SLACK = 8

    def __init__(self, matrix: RaggedMatrix, slack: int | None = None):
        self.matrix = matrix
        dev = matrix.target.device
        N = matrix.num_post
        self.slack = self.SLACK if slack is None else int(slack)
        cap = max(1, matrix.num_pre * matrix.stride + N * self.slack)
        self.col_length = torch.zeros(N, dtype=torch.int32, device=dev)
        self.col_ptr = torch.zeros(N + 1, dtype=torch.int32, device=dev)
        self.src_pre = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.src_slot = torch.zeros(cap, dtype=torch.int32, device=dev)
        self._cursor = torch.zeros(N, dtype=torch.int32, device=dev)
        self._max_len = torch.zeros(1, dtype=torch.int32, device=dev)
        self._block_scratch = torch.zeros(2048, dtype=torch.int32, device=dev)
        self._need_rebuild = torch.zeros(1, dtype=torch.int32, device=dev)
        nb = int(_lib.lib().sw_transpose_patch_scratch_bytes(matrix.num_pre, N))
        self._patch_scratch = torch.zeros(nb // 4 + 1, dtype=torch.int32, device=dev)
        self.version = -1
        self.patches = 0

    def rebuild(self, changed_flag: torch.Tensor | None = None) -> None:
        """Rebuild from the matrix; with a device ``changed_flag`` the kernels
        skip the work when it reads 0 (remap-only-if-changed on the device)."""
        d = descriptor(self.matrix, None)
        # one cooperative launch (count / scan / scatter / sort behind grid
        # barriers; exits at once when the matrix did not change)
        _lib.call("sw_transpose_rebuild_coop", ctypes.byref(d), self.col_length.data_ptr(),
                  self.col_ptr.data_ptr(), self.src_pre.data_ptr(), self.src_slot.data_ptr(),
                  self._cursor.data_ptr(), self._max_len.data_ptr(), _lib.ptr(changed_flag),
                  self._block_scratch.data_ptr(), self.slack, _lib.stream_ptr())
        self.version = self.matrix.version

    def patch(self, patch_log: torch.Tensor, cap: int) -> None:
        """Apply one update's changes in place (sw_transpose_patch): the
        columns touched by the changed rows are re-merged; if a column runs
        out of slack (or the log overflowed) a full rebuild follows on the
        device.  Same result as rebuild(), bit for bit."""
        if self.version < 0:
            self.rebuild()
            return
        d = descriptor(self.matrix, None)
        _lib.call("sw_transpose_patch", ctypes.byref(d), self.col_length.data_ptr(), self.col_ptr.data_ptr(),
                  self.src_pre.data_ptr(), self.src_slot.data_ptr(), patch_log.data_ptr(), int(cap),
                  self._need_rebuild.data_ptr(), self._patch_scratch.data_ptr(), _lib.stream_ptr())
        # gated full rebuild: runs only if the patch flagged an overflow, and
        # resets the flag
        _lib.call("sw_transpose_rebuild_gated", ctypes.byref(d), self.col_length.data_ptr(),
                  self.col_ptr.data_ptr(), self.src_pre.data_ptr(), self.src_slot.data_ptr(),
                  self._cursor.data_ptr(), self._max_len.data_ptr(), self._need_rebuild.data_ptr(),
                  self._block_scratch.data_ptr(), self.slack, 1, _lib.stream_ptr())
        self.version = self.matrix.version
        self.patches += 1

    @property
    def max_col_length(self) -> int:
        return int(self.col_length.max().item()) if self.col_length.numel() else 0

    def is_stale(self) -> bool:
        return self.version != self.matrix.version

    def check_fresh(self) -> None:
        if self.is_stale():
            raise StaleTranspose("transpose map older than its matrix")

    def host_csr(self):
        """Compact CSR (ptr[N+1], pre, slot) of the live entries (slack dropped)."""
        start = self.col_ptr[:-1].cpu().numpy().astype(np.int64)
        lens = self.col_length.cpu().numpy().astype(np.int64)
        ptr = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=ptr[1:])
        idx = np.repeat(start - ptr[:-1], lens) + np.arange(int(ptr[-1]))
        return ptr, self.src_pre.cpu().numpy()[idx], self.src_slot.cpu().numpy()[idx]

    def column(self, j: int):
        ptr, pre, slot = self.host_csr()
        return pre[ptr[j]:ptr[j + 1]], slot[ptr[j]:ptr[j + 1]]

    def columns(self, posts):
        ptr, pre, slot = self.host_csr()
        ps = [pre[ptr[j]:ptr[j + 1]] for j in posts]
        ss = [slot[ptr[j]:ptr[j + 1]] for j in posts]
        if not ps:
            e = np.empty(0, dtype=np.int32)
            return e, e
        return np.concatenate(ps), np.concatenate(ss)

    def reference_layout(self):
        """(col_length, source_pre [N, width], source_slot [N, width]) exactly
        as TransposeMap.rebuild lays them out (connectivity.py:173-192)."""
        ptr, pre, slot = self.host_csr()
        N = self.matrix.num_post
        counts = np.diff(ptr).astype(np.int32)
        width = max(int(counts.max()) if counts.size else 0, 1)
        sp = np.zeros((N, width), dtype=np.int32)
        ss = np.zeros((N, width), dtype=np.int32)
        for j in range(N):
            sp[j, :counts[j]] = pre[ptr[j]:ptr[j + 1]]
            ss[j, :counts[j]] = slot[ptr[j]:ptr[j + 1]]
        return counts, sp, ss


def remap_transpose(m: RaggedMatrix) -> TransposeMap:
    tm = TransposeMap(m)
    tm.rebuild()
    return tm
