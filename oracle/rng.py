"""Oracle restatement of the counter-based SplitMix64 streams.

Follows ``sparsewire/rng.py`` (cited per function).  Test infrastructure only.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15          # rng.py:21
CHILD_SALT = 0x632BE59BD9B4E019      # rng.py:86
FOLD_INIT = 0x5851F42D4C957F2D       # rng.py:51


def mix64(z: int) -> int:
    """SplitMix64 finalizer, rng.py:28-33."""
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix64_np(z: np.ndarray) -> np.ndarray:
    """Vector finalizer, rng.py:36-43."""
    z = np.asarray(z, dtype=np.uint64).copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def fold_key(*parts) -> int:
    """Fold ints / strings into a 64-bit key, rng.py:46-61."""
    acc = FOLD_INIT
    for p in parts:
        if isinstance(p, str):
            b = p.encode("utf-8")
            for off in range(0, len(b), 8):
                acc = mix64(acc ^ mix64(int.from_bytes(b[off:off + 8], "little") + 0x0B))
            acc = mix64(acc ^ len(b))
        else:
            acc = mix64(acc ^ mix64((int(p) & M64) + 0x9E))
    return acc


def child_key(key: int, index: int) -> int:
    """rng.py:84-86."""
    return mix64(key ^ mix64((index + CHILD_SALT) & M64))


def child_keys_np(key: int, rows: np.ndarray) -> np.ndarray:
    rows = np.asarray(rows, dtype=np.uint64)
    return mix64_np(np.uint64(key) ^ mix64_np(rows + np.uint64(CHILD_SALT)))


def draw_u64(key: int, counter: int) -> int:
    """Draw #counter of the stream with this key, rng.py:88-91."""
    return mix64((key + counter * GOLDEN) & M64)


def u64_block(key: int, start: int, n: int) -> np.ndarray:
    """rng.py:93-96."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    return mix64_np(np.uint64(key) + idx * np.uint64(GOLDEN))


def u01_from_u64(h):
    """(h >> 11) * 2^-53, rng.py:98-104 (exact in float64)."""
    if isinstance(h, np.ndarray):
        return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (h >> 11) * (2.0 ** -53)


def reject_limit(n: int) -> int:
    """uniform_int accepts h < limit, rng.py:110 (limit may equal 2^64)."""
    return (1 << 64) - ((1 << 64) % n)


class Stream:
    """Key + counter, the oracle twin of ``CounterRng`` (rng.py:64-153)."""

    __slots__ = ("key", "counter")

    def __init__(self, key: int, counter: int = 0):
        self.key = key & M64
        self.counter = counter

    @classmethod
    def of(cls, *parts) -> "Stream":
        return cls(fold_key(*parts))

    def child_key(self, index: int) -> int:
        return child_key(self.key, index)

    def next_u64(self) -> int:
        h = draw_u64(self.key, self.counter)
        self.counter += 1
        return h

    def u64_array(self, n: int) -> np.ndarray:
        out = u64_block(self.key, self.counter, n)
        self.counter += n
        return out

    def uniform01(self) -> float:
        return u01_from_u64(self.next_u64())

    def uniform01_array(self, n: int) -> np.ndarray:
        return u01_from_u64(self.u64_array(n))

    def uniform_int(self, n: int) -> int:
        """rng.py:106-114: rejection, a rejected draw still consumes a counter."""
        if n <= 0:
            raise ValueError("n must be positive")
        lim = reject_limit(n)
        while True:
            h = self.next_u64()
            if h < lim:
                return h % n

    def sample_k_distinct(self, k: int, n: int) -> np.ndarray:
        """rng.py:116-141: rejection when 2k < n, else partial Fisher-Yates."""
        if k > n:
            raise ValueError("k > n")
        if k == 0:
            return np.empty(0, dtype=np.int64)
        if 2 * k < n:
            seen = []
            while len(seen) < k:
                v = self.uniform_int(n)
                if v not in seen:
                    seen.append(v)
            return np.array(seen, dtype=np.int64)
        buf = list(range(n))
        for i in range(k):
            j = i + self.uniform_int(n - i)
            buf[i], buf[j] = buf[j], buf[i]
        return np.array(buf[:k], dtype=np.int64)

    def normal_array(self, n: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
        """Box-Muller with numpy transcendentals, rng.py:143-153 (host only)."""
        m = (n + 1) // 2
        u1 = ((self.u64_array(m) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * (2.0 ** -53)
        u2 = self.uniform01_array(m)
        r = np.sqrt(-2.0 * np.log(u1))
        th = (2.0 * np.pi) * u2
        return mean + std * np.concatenate([r * np.cos(th), r * np.sin(th)])[:n]
