"""Oracle restatement of the padded ragged matrix and its mutation primitives.

Follows ``sparsewire/connectivity.py`` and ``sparsewire/bitfield.py``.
Test infrastructure only.
"""

from __future__ import annotations

import math

import numpy as np

from .rng import Stream


class RowFull(Exception):
    pass


class DuplicateEdge(Exception):
    pass


class SlotOutOfRange(Exception):
    pass


class Ragged:
    """RaggedMatrix + SynVarMatrix in one object (connectivity.py:24-88).

    ``target`` is [num_pre, max(cap, 1)] int32, planes are slot-aligned
    [num_pre, max(cap, 1)] arrays (float64 unless stated, connectivity.py:76).
    """

    def __init__(self, num_pre, num_post, cap, planes=(), multapse_free=True):
        self.num_pre = num_pre
        self.num_post = num_post
        self.max_row_length = cap
        self.row_length = np.zeros(num_pre, dtype=np.int32)
        self.target = np.zeros((num_pre, max(cap, 1)), dtype=np.int32)
        self.planes = {}
        for p in planes:
            self.add_plane(p)
        self.multapse_free = multapse_free
        self.version = 0

    def add_plane(self, name, dtype=np.float64):
        self.planes[name] = np.zeros(self.target.shape, dtype=dtype)
        return self.planes[name]

    def slot_mask(self):
        return np.arange(self.target.shape[1])[None, :] < self.row_length[:, None]

    def edge_count(self):
        return int(self.row_length.sum())

    def copy(self):
        o = Ragged.__new__(Ragged)
        o.num_pre, o.num_post, o.max_row_length = self.num_pre, self.num_post, self.max_row_length
        o.row_length = self.row_length.copy()
        o.target = self.target.copy()
        o.planes = {k: v.copy() for k, v in self.planes.items()}
        o.multapse_free = self.multapse_free
        o.version = self.version
        return o

    # connectivity.py:91-112
    def add_synapse(self, pre, post, values=None):
        n = int(self.row_length[pre])
        if n >= self.max_row_length:
            raise RowFull(pre)
        if self.multapse_free and np.any(self.target[pre, :n] == post):
            raise DuplicateEdge((pre, post))
        self.target[pre, n] = post
        for name, pl in self.planes.items():
            pl[pre, n] = 0
        for name, v in (values or {}).items():
            self.planes[name][pre, n] = v
        self.row_length[pre] = n + 1
        self.version += 1
        return n

    # connectivity.py:115-127
    def remove_synapse(self, pre, slot):
        n = int(self.row_length[pre])
        if not 0 <= slot < n:
            raise SlotOutOfRange((pre, slot))
        last = n - 1
        if slot != last:
            self.target[pre, slot] = self.target[pre, last]
            for pl in self.planes.values():
                pl[pre, slot] = pl[pre, last]
        self.row_length[pre] = last
        self.version += 1

    # connectivity.py:130-136: descending order, chained swap-with-last
    def remove_slots(self, pre, slots):
        for s in sorted((int(x) for x in slots), reverse=True):
            self.remove_synapse(pre, s)


def removal_permutation(n: int, marked) -> list[tuple[int, int]]:
    """Closed form of ``remove_slots``: the (dst, src)
    moves that turn the row into its post-removal state in one parallel
    gather.  Used by the tests to cross-check the serial replay."""
    ms = sorted(set(int(m) for m in marked), reverse=True)
    k = len(ms)
    rank = {m: t + 1 for t, m in enumerate(ms)}
    n2 = n - k
    moves = []
    for t, m in enumerate(ms, start=1):
        if m >= n2:
            continue
        p = n - t
        while p in rank:
            p = n - rank[p]
        moves.append((m, p))
    return moves


def propagate_spikes(m: Ragged, weights: np.ndarray, spikes, out: np.ndarray):
    """connectivity.py:139-148: np.add.at per spiking row, spike order."""
    for i in spikes:
        n = m.row_length[i]
        np.add.at(out, m.target[i, :n], weights[i, :n])


def transpose(m: Ragged):
    """TransposeMap.rebuild, connectivity.py:173-192: per post, (pre, slot)
    of incoming synapses ordered by (pre, slot)."""
    lens = m.row_length.astype(np.int64)
    pre = np.repeat(np.arange(m.num_pre, dtype=np.int64), lens)
    mask = m.slot_mask()
    slot = np.broadcast_to(np.arange(m.target.shape[1]), m.target.shape)[mask]
    post = m.target[mask].astype(np.int64)
    counts = np.bincount(post, minlength=m.num_post)
    width = max(int(counts.max()) if counts.size else 0, 1)
    src_pre = np.zeros((m.num_post, width), dtype=np.int32)
    src_slot = np.zeros((m.num_post, width), dtype=np.int32)
    order = np.lexsort((slot, pre, post))
    ps = post[order]
    within = np.arange(ps.size) - np.concatenate(([0], np.cumsum(counts)))[ps]
    src_pre[ps, within] = pre[order]
    src_slot[ps, within] = slot[order]
    return counts.astype(np.int32), src_pre, src_slot


def init_pairwise_bernoulli(num_pre, num_post, prob_fn, headroom, stream: Stream,
                            planes=(), multapse_free=True):
    """connectivity.py:212-245: per row uniform01_array(num_post) < p."""
    cols = np.arange(num_post, dtype=np.int64)
    rows = []
    mx = 0
    for i in range(num_pre):
        p = np.asarray(prob_fn(i, cols), dtype=np.float64)
        u = stream.uniform01_array(num_post)
        hit = np.flatnonzero(u < p)
        rows.append(hit)
        mx = max(mx, hit.size)
    cap = math.ceil(headroom * mx)
    if multapse_free:
        cap = min(cap, num_post)
    m = Ragged(num_pre, num_post, cap, planes, multapse_free)
    for i, hit in enumerate(rows):
        m.row_length[i] = hit.size
        m.target[i, :hit.size] = hit
    m.version += 1
    return m


# -- bitfields (bitfield.py) -------------------------------------------------

def bf_words(num_post):
    return (num_post + 63) // 64


def bf_tail_mask(num_post):
    tail = num_post - (bf_words(num_post) - 1) * 64
    return np.uint64((1 << tail) - 1 if tail < 64 else (1 << 64) - 1)


def bf_test(words, i, j):
    return bool((int(words[i, j >> 6]) >> (j & 63)) & 1)


def bf_set(words, i, j):
    words[i, j >> 6] |= np.uint64(1 << (j & 63))


def bf_clear(words, i, j):
    words[i, j >> 6] &= np.uint64(~(1 << (j & 63)) & ((1 << 64) - 1))


def bf_randomize(words, num_post, stream: Stream):
    """bitfield.py:92-96: raw draws row-major, tail bits masked."""
    flat = stream.u64_array(words.size)
    words[:, :] = flat.reshape(words.shape)
    words[:, -1] &= bf_tail_mask(num_post)


def bf_set_bits_ascending(words, i, num_post):
    """bitfield.py:79-84."""
    row = words[i]
    bits = (row[:, None] >> np.arange(64, dtype=np.uint64)[None, :]) & np.uint64(1)
    idx = np.flatnonzero(bits.ravel())
    return idx[idx < num_post]
