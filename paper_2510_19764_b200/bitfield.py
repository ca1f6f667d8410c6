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

    # -- the rest of the reference Bitfield API (bitfield.py:32-90), as
    #    vectorised device ops on the int64 word view --------------------------
    @staticmethod
    def _word_masks(cols) -> tuple[np.ndarray, np.ndarray]:
        """Unique word indices and the OR of the bits each of them gets."""
        cols = np.asarray(cols, dtype=np.int64).reshape(-1)
        words = cols >> 6
        uw, inv = np.unique(words, return_inverse=True)
        masks = np.zeros(uw.size, dtype=np.uint64)
        np.bitwise_or.at(masks, inv, np.uint64(1) << (cols & 63).astype(np.uint64))
        return uw, masks.view(np.int64)

    def set_bit(self, i: int, j: int) -> None:
        self.set_bits(i, [j])

    def clear_bit(self, i: int, j: int) -> None:
        self.clear_bits(i, [j])

    def set_bits(self, i: int, cols) -> None:
        uw, m = self._word_masks(cols)
        if uw.size:
            idx = torch.from_numpy(uw).to(self.words.device)
            self.words[i, idx] |= torch.from_numpy(m).to(self.words.device)

    def clear_bits(self, i: int, cols) -> None:
        uw, m = self._word_masks(cols)
        if uw.size:
            idx = torch.from_numpy(uw).to(self.words.device)
            self.words[i, idx] &= ~torch.from_numpy(m).to(self.words.device)

    def test_bits(self, i: int, cols) -> np.ndarray:
        cols = torch.as_tensor(np.asarray(cols, dtype=np.int64)).to(self.words.device)
        return ((self.words[i, cols >> 6] >> (cols & 63)) & 1).bool().cpu().numpy()

    def test_bits_rows(self, rows_cols: np.ndarray) -> np.ndarray:
        """Test bit (r, rows_cols[r, c]) for a full column-index matrix."""
        rc = torch.as_tensor(np.asarray(rows_cols, dtype=np.int64)).to(self.words.device)
        w = torch.gather(self.words, 1, rc >> 6)
        return ((w >> (rc & 63)) & 1).bool().cpu().numpy()

    def clear_row(self, i: int) -> None:
        self.words[i].zero_()

    def set_k_random_bits_in_row(self, i: int, k: int, rng: CounterRng) -> np.ndarray:
        """Exactly k distinct bits, in the reference's draw order (bitfield.py:67-77)."""
        from .errors import KTooLarge
        if k > self.num_post:
            raise KTooLarge(f"k={k} exceeds row width {self.num_post}")
        cols = rng.sample_k_distinct(k, self.num_post)
        if k:
            self.set_bits(i, cols)
        return cols

    def set_bits_in_row(self, i: int) -> np.ndarray:
        """Ascending column indices of all set bits in row i."""
        row = self.words[i].cpu().numpy().view(np.uint64)
        bits = (row[:, None] >> np.arange(64, dtype=np.uint64)[None, :]) & np.uint64(1)
        idx = np.flatnonzero(bits.ravel())
        return idx[idx < self.num_post]

    def row_popcount(self, i: int) -> int:
        return int(self.set_bits_in_row(i).size)
