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
    def __init__(self, matrix: RaggedMatrix):
        self.matrix = matrix
        dev = matrix.target.device
        N = matrix.num_post
        cap = max(1, matrix.num_pre * matrix.stride)
        self.col_length = torch.zeros(N, dtype=torch.int32, device=dev)
        self.col_ptr = torch.zeros(N + 1, dtype=torch.int32, device=dev)
        self.src_pre = torch.zeros(cap, dtype=torch.int32, device=dev)
        self.src_slot = torch.zeros(cap, dtype=torch.int32, device=dev)
        self._cursor = torch.zeros(N, dtype=torch.int32, device=dev)
        self._max_len = torch.zeros(1, dtype=torch.int32, device=dev)
        self._block_scratch = torch.zeros(2048, dtype=torch.int32, device=dev)
        self.version = -1

    def rebuild(self, changed_flag: torch.Tensor | None = None) -> None:
        """Rebuild from the matrix; with a device ``changed_flag`` the kernels
        skip the work when it reads 0 (remap-only-if-changed on the device)."""
        d = descriptor(self.matrix, None)
        # one cooperative launch (count / scan / scatter / sort behind grid
        # barriers; exits at once when the matrix did not change)
        _lib.call("sw_transpose_rebuild_coop", ctypes.byref(d), self.col_length.data_ptr(),
                  self.col_ptr.data_ptr(), self.src_pre.data_ptr(), self.src_slot.data_ptr(),
                  self._cursor.data_ptr(), self._max_len.data_ptr(), _lib.ptr(changed_flag),
                  self._block_scratch.data_ptr(), _lib.stream_ptr())
        self.version = self.matrix.version

    @property
    def max_col_length(self) -> int:
        return int(self._max_len.item())

    def is_stale(self) -> bool:
        return self.version != self.matrix.version

    def check_fresh(self) -> None:
        if self.is_stale():
            raise StaleTranspose("transpose map older than its matrix")

    def host_csr(self):
        ptr = self.col_ptr.cpu().numpy()
        E = int(ptr[-1])
        return ptr, self.src_pre[:E].cpu().numpy(), self.src_slot[:E].cpu().numpy()

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
