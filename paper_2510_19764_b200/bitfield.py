"""Packed per-(pre, post) bit matrices in HBM (``sparsewire/bitfield.py``).

``words`` is a CUDA int64 tensor [num_pre, ceil(num_post/64)] holding the
reference's uint64 words bit-for-bit (LSB-first, tail bits zero,
bitfield.py:19-33).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .rng import CounterRng


class Bitfield:
    __slots__ = ("num_pre", "num_post", "words")

    def __init__(self, num_pre: int, num_post: int, device="cuda"):
        _lib.require_cuda()
        self.num_pre = num_pre
        self.num_post = num_post
        self.words = torch.zeros((num_pre, (num_post + 63) // 64), dtype=torch.int64,
                                 device=device)

    @property
    def words_per_row(self) -> int:
        return self.words.shape[1]

    def descriptor(self) -> _lib.BitfieldDesc:
        d = _lib.BitfieldDesc()
        d.words = self.words.data_ptr()
        d.num_pre, d.num_post, d.words_per_row = self.num_pre, self.num_post, self.words_per_row
        return d

    def randomize(self, rng: CounterRng) -> None:
        """bitfield.py:92-96 on the device (draws advance ``rng``)."""
        import ctypes
        _lib.call("sw_bitfield_randomize", ctypes.byref(self.descriptor()),
                  (rng.key + rng.counter * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
                  if rng.counter else rng.key, _lib.stream_ptr())
        rng.counter += self.words.numel()

    def clear_all(self) -> None:
        self.words.zero_()

    def popcount(self) -> int:
        w = self.words
        # popcount of int64 words via byte view
        b = w.view(torch.uint8)
        table = torch.tensor([bin(x).count("1") for x in range(256)], dtype=torch.int64,
                             device=w.device)
        return int(table[b.long()].sum().item())

    def host_words(self) -> np.ndarray:
        return self.words.cpu().numpy().view(np.uint64)

    def load_words(self, words: np.ndarray) -> None:
        self.words.copy_(torch.from_numpy(np.ascontiguousarray(words, dtype=np.uint64).view(np.int64)))

    def test_bit(self, i: int, j: int) -> bool:
        return bool((int(self.words[i, j >> 6].item()) >> (j & 63)) & 1)
