"""Multi-GPU partitioning of the hot path, host side.

One process per GPU with torch.distributed (NCCL on the GPUs; the same code
runs on gloo for the CPU tests):

* classifier (e-prop + DEEP R): batch-DP.  Rank r trains the replicas
  ``shard_batch(B, r, world)``.  The raw float64 gradient sums are all-reduced
  once per batch (``allreduce_flat``).  Every rank then applies the same scale,
  L1, Adam and DEEP R with the same counter-RNG keys, so the connectivity
  stays identical on every rank without exchanging it.  The reference sums
  replicas in one sequential loop (_kernels.py:30-38); the sharded sum
  differs from it only in the float64 rounding of the partial sums.
* topographic map: postsynaptic sharding.  Rank r owns the posts
  ``post_shard_range(n, r, world)``, whose bounds are aligned to 32-post spike
  words.  It runs the conductance-LIF update and the ordered propagation
  into those posts only.  Source (Poisson) spikes are counter-based, so every
  rank regenerates all of them.  Target spikes are all-gathered once per step
  (``SpikeGather``).  With the full spike vectors, STDP and the rewiring rule
  run replicated on identical inputs, so the synaptic state and the
  connectivity stay identical on every rank.
"""

from __future__ import annotations

import torch


def shard_batch(batch: int, rank: int, world: int) -> slice:
    """Contiguous replica range of one rank (the last rank takes the remainder)."""
    per = batch // world
    lo = rank * per
    hi = batch if rank == world - 1 else lo + per
    return slice(lo, hi)


def post_shard_words(n: int, world: int) -> int:
    """32-bit spike words owned per rank (equal counts, for all-gather)."""
    words = (n + 31) // 32
    return (words + world - 1) // world


def post_shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Posts [lo, hi) owned by ``rank``; bounds fall on spike-word boundaries."""
    wpr = post_shard_words(n, world)
    lo = min(n, rank * wpr * 32)
    hi = min(n, (rank + 1) * wpr * 32)
    return lo, hi


class SpikeGather:
    """All-gather of a sharded spike bitmask.

    ``bits`` is the full mask (world * words_per_rank int32 words; only the
    first ceil(n/32) words are meaningful).  Each rank writes the words of its
    own post range, then ``gather()`` fills in the other ranks' words."""

    def __init__(self, n: int, rank: int, world: int, device, group=None):
        self.n, self.rank, self.world, self.group = n, rank, world, group
        self.wpr = post_shard_words(n, world)
        self.bits = torch.zeros(world * self.wpr, dtype=torch.int32, device=device)
        self._send = torch.zeros(self.wpr, dtype=torch.int32, device=device)
        self.lo, self.hi = post_shard_range(n, rank, world)

    @property
    def own_words(self) -> slice:
        return slice(self.rank * self.wpr, (self.rank + 1) * self.wpr)

    def gather(self) -> torch.Tensor:
        if self.world == 1:
            return self.bits
        import torch.distributed as dist
        self._send.copy_(self.bits[self.own_words])
        dist.all_gather_into_tensor(self.bits, self._send, group=self.group)
        return self.bits


def allreduce_flat(tensors, group=None) -> None:
    """Sum the tensors over ranks in one collective (flattened, same dtype)."""
    import torch.distributed as dist
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, group=group)
    o = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[o:o + n].view_as(t))
        o += n


# ---- M-update microbench: rows sharded ---------------------------
def shard_rows(num_pre: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) owned by ``rank``: equal contiguous chunks (the last
    rank takes the remainder)."""
    per = num_pre // world
    lo = rank * per
    return lo, (num_pre if rank == world - 1 else lo + per)


def reduce_scatter_rows(full: torch.Tensor, local: torch.Tensor, row0: int, group=None) -> None:
    """``local[:] = sum over ranks of full[row0 : row0 + len(local)]``.

    NCCL with equal row chunks: one reduce-scatter (the activation
    histogram, 4 B per row).  Otherwise (gloo, ragged chunks): all-reduce of
    the full vector, then the owner's slice."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = local.numel()
    equal = full.numel() == n * world and row0 == dist.get_rank(group) * n
    if equal and dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(local, full, group=group)
        return
    dist.all_reduce(full, group=group)
    local.copy_(full[row0:row0 + n])


# ---- M-prop microbench: posts sharded ----------------------------
def shard_posts(num_post: int, rank: int, world: int) -> tuple[int, int]:
    """Posts [lo, hi) owned by ``rank`` in the column-sliced propagation:
    equal contiguous ranges (the last rank takes the remainder)."""
    return shard_rows(num_post, rank, world)
