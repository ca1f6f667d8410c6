"""Device-resident padded ragged connectivity (the reference's
``sparsewire/connectivity.py`` API, storage in HBM).

``RaggedMatrix`` keeps ``row_length`` int32 [P] and ``target`` int32
[P, max(cap, 1)] as CUDA tensors (connectivity.py:24-40); ``SynVarMatrix``
keeps named slot-aligned planes, float64 by default (:65-88).  Structural
changes happen inside the sm_100a kernels; ``version`` is bumped by the
host layer after every mutating call (:38-40).
"""

from __future__ import annotations

import math
from typing import Iterable

import numpy as np
import torch

from . import _lib
from .rng import CounterRng

DEV = "cuda"


class RaggedMatrix:
    __slots__ = ("num_pre", "num_post", "max_row_length", "row_length", "target",
                 "multapse_free", "version")

    def __init__(self, num_pre: int, num_post: int, max_row_length: int,
                 multapse_free: bool = True, device=DEV):
        _lib.require_cuda()
        self.num_pre = num_pre
        self.num_post = num_post
        self.max_row_length = max_row_length
        self.row_length = torch.zeros(num_pre, dtype=torch.int32, device=device)
        self.target = torch.zeros((num_pre, max(max_row_length, 1)), dtype=torch.int32,
                                  device=device)
        self.multapse_free = multapse_free
        self.version = 0

    @property
    def stride(self) -> int:
        return self.target.shape[1]

    def edge_count(self) -> int:
        return int(self.row_length.sum().item())

    def row_targets(self, i: int) -> torch.Tensor:
        return self.target[i, : int(self.row_length[i].item())]

    def slot_mask(self) -> torch.Tensor:
        return (torch.arange(self.stride, device=self.target.device)[None, :]
                < self.row_length[:, None])

    def contains(self, pre: int, post: int) -> bool:
        return bool((self.row_targets(pre) == post).any().item())

    def edge_list(self) -> tuple[np.ndarray, np.ndarray]:
        lens = self.row_length.cpu().numpy().astype(np.int64)
        pre = np.repeat(np.arange(self.num_pre, dtype=np.int64), lens)
        post = self.target[self.slot_mask()].cpu().numpy().astype(np.int64)
        return pre, post

    # -- state transfer (reference-layout numpy arrays) ------------------------
    def load_state(self, row_length: np.ndarray, target: np.ndarray) -> None:
        """Inject host state (e.g. from a reference object) into HBM."""
        self.row_length.copy_(torch.from_numpy(np.ascontiguousarray(row_length, dtype=np.int32)))
        self.target.copy_(torch.from_numpy(np.ascontiguousarray(target, dtype=np.int32)))
        self.version += 1

    def host_state(self) -> dict[str, np.ndarray]:
        return {"row_length": self.row_length.cpu().numpy(), "target": self.target.cpu().numpy()}


class SynVarMatrix:
    __slots__ = ("matrix", "planes")

    def __init__(self, matrix: RaggedMatrix, names: Iterable[str] = ()):
        self.matrix = matrix
        self.planes: dict[str, torch.Tensor] = {}
        for n in names:
            self.add_plane(n)

    def add_plane(self, name: str, dtype=torch.float64) -> torch.Tensor:
        if name in self.planes:
            raise KeyError(f"plane {name!r} already exists")
        if len(self.planes) >= _lib.MAX_PLANES:
            raise ValueError(f"at most {_lib.MAX_PLANES} planes per matrix")
        if dtype not in (torch.float64, torch.float32, torch.int32, torch.int64):
            raise TypeError("planes must be 4- or 8-byte types")
        t = torch.zeros(self.matrix.target.shape, dtype=dtype, device=self.matrix.target.device)
        self.planes[name] = t
        return t

    def plane(self, name: str) -> torch.Tensor:
        return self.planes[name]

    def row(self, name: str, i: int) -> torch.Tensor:
        return self.planes[name][i, : int(self.matrix.row_length[i].item())]

    def plane_index(self, name: str) -> int:
        return list(self.planes).index(name)


def descriptor(m: RaggedMatrix, syn: SynVarMatrix | None) -> _lib.Ragged:
    d = _lib.Ragged()
    d.num_pre, d.num_post = m.num_pre, m.num_post
    d.max_row_length, d.stride = m.max_row_length, m.stride
    d.row_length, d.target = m.row_length.data_ptr(), m.target.data_ptr()
    planes = list(syn.planes.values()) if syn is not None else []
    d.n_planes = len(planes)
    for k, t in enumerate(planes):
        if not t.is_contiguous() or t.shape != m.target.shape:
            raise ValueError("planes must be contiguous [num_pre, stride]")
        d.plane_bytes[k] = t.element_size()
        d.planes[k] = t.data_ptr()
    return d


def row_slice(m: RaggedMatrix, syn: SynVarMatrix | None, lo: int, hi: int
              ) -> tuple[RaggedMatrix, SynVarMatrix | None]:
    """Rows [lo, hi) as their own matrix (copies; same num_post, capacity and
    planes): the local part of a row-sharded matrix (SURVEY 8e M-update)."""
    out = RaggedMatrix(hi - lo, m.num_post, m.max_row_length, m.multapse_free, device=m.target.device)
    out.row_length.copy_(m.row_length[lo:hi])
    out.target.copy_(m.target[lo:hi])
    osyn = None
    if syn is not None:
        osyn = SynVarMatrix(out)
        for n, t in syn.planes.items():
            osyn.add_plane(n, t.dtype).copy_(t[lo:hi])
    return out, osyn


def column_slice(m: RaggedMatrix, syn: SynVarMatrix | None, lo: int, hi: int,
                 capacity: int | None = None) -> tuple[RaggedMatrix, SynVarMatrix | None]:
    """The synapses onto posts [lo, hi) (targets renumbered from 0, slot
    order kept): the local part of a post-sharded matrix (SURVEY 8e M-prop).
    ``capacity`` defaults to the longest sliced row."""
    from .errors import RowFull
    src = descriptor(m, syn)
    mx = torch.zeros(1, dtype=torch.int32, device=m.target.device)
    cap = m.max_row_length if capacity is None else int(capacity)
    out = RaggedMatrix(m.num_pre, hi - lo, cap, m.multapse_free, device=m.target.device)
    osyn = None
    if syn is not None:
        osyn = SynVarMatrix(out)
        for n, t in syn.planes.items():
            osyn.add_plane(n, t.dtype)
    dst = descriptor(out, osyn)
    _lib.call("sw_ragged_column_slice", C_ref(src), lo, hi, C_ref(dst), mx.data_ptr(), _lib.stream_ptr())
    longest = int(mx.item())
    if longest > out.stride:
        raise RowFull(f"column slice row of {longest} synapses exceeds capacity {out.stride}")
    if capacity is None and longest < cap:
        # shrink to the longest slice row (every sliced row fits)
        small = RaggedMatrix(m.num_pre, hi - lo, max(longest, 1), m.multapse_free, device=m.target.device)
        small.row_length.copy_(out.row_length)
        small.target.copy_(out.target[:, :small.stride])
        ssyn = None
        if osyn is not None:
            ssyn = SynVarMatrix(small)
            for n, t in osyn.planes.items():
                ssyn.add_plane(n, t.dtype).copy_(t[:, :small.stride])
        return small, ssyn
    return out, osyn


def remove_marked(m: RaggedMatrix, syn: SynVarMatrix | None, marked: torch.Tensor,
                  removed: torch.Tensor | None = None) -> None:
    """Remove every marked slot of every row with the exact ``remove_slots``
    order (connectivity.py:130-136), all rows in one launch."""
    if marked.dtype != torch.uint8 or marked.shape != m.target.shape:
        raise ValueError("marked must be uint8 [num_pre, stride]")
    d = descriptor(m, syn)
    _lib.call("sw_ragged_remove_marked", C_ref(d), marked.data_ptr(), _lib.ptr(removed),
              _lib.stream_ptr())
    m.version += 1


def add_synapse(m: RaggedMatrix, syn: SynVarMatrix | None, pre: int, post: int,
                values: dict | None = None) -> int:
    """Append pre -> post and return its slot (connectivity.py:91-112): every
    plane is zeroed at the new slot, then ``values`` are set.  Raises
    RowFull / DuplicateEdge like the reference (one device round trip)."""
    from .errors import DuplicateEdge, RowFull
    d = descriptor(m, syn)
    names = list(syn.planes) if syn is not None else []
    vals = torch.zeros(max(1, len(names)), dtype=torch.float64)
    mask = torch.zeros(max(1, len(names)), dtype=torch.uint8)
    for name, v in (values or {}).items():
        k = names.index(name)
        vals[k] = float(v)
        mask[k] = 1
    dv, dm = vals.to(DEV), mask.to(DEV)
    status = torch.zeros(2, dtype=torch.int32, device=DEV)
    _lib.call("sw_ragged_add_synapse", C_ref(d), int(pre), int(post), dv.data_ptr(), dm.data_ptr(),
              int(m.multapse_free), status.data_ptr(), _lib.stream_ptr())
    st = int(status[0].item())
    if st == -1:
        raise RowFull(f"row {pre} at capacity {m.max_row_length}")
    if st == -2:
        raise DuplicateEdge(f"edge ({pre}, {post}) already exists")
    m.version += 1
    return st


def remove_slots(m: RaggedMatrix, syn: SynVarMatrix | None, pre: int, slots) -> None:
    """Remove several slots of one row, descending order with swap-from-the-end
    moves (connectivity.py:130-136).  Raises SlotOutOfRange like the
    reference's loop."""
    from .errors import SlotOutOfRange
    sl = torch.as_tensor(np.asarray(slots, dtype=np.int32).reshape(-1)).to(DEV)
    d = descriptor(m, syn)
    status = torch.zeros(2, dtype=torch.int32, device=DEV)
    _lib.call("sw_ragged_remove_row_slots", C_ref(d), int(pre), sl.data_ptr(), int(sl.numel()),
              status.data_ptr(), _lib.stream_ptr())
    m.version += 1
    if int(status[0].item()) != 0:
        raise SlotOutOfRange(f"slot out of range in row {pre}")


def remove_synapse(m: RaggedMatrix, syn: SynVarMatrix | None, pre: int, slot: int) -> None:
    """Remove one synapse: the last valid slot moves into its place
    (connectivity.py:115-127)."""
    remove_slots(m, syn, pre, [slot])


def C_ref(d):
    import ctypes
    return ctypes.byref(d)


def _init_rows(num_pre, num_post, key, counter0, mode, density, lut, side, headroom,
               multapse_free, names, cap=None):
    _lib.require_cuda()
    st = _lib.stream_ptr()
    rl = torch.zeros(num_pre, dtype=torch.int32, device=DEV)
    mx = torch.zeros(1, dtype=torch.int32, device=DEV)
    lut_t = None if lut is None else torch.as_tensor(np.ascontiguousarray(lut, dtype=np.float64),
                                                     device=DEV)
    _lib.call("sw_init_bernoulli_count", num_pre, num_post, key, counter0, mode, float(density),
              _lib.ptr(lut_t), side, rl.data_ptr(), mx.data_ptr(), st)
    if cap is None:
        cap = math.ceil(headroom * int(mx.item()))
        if multapse_free:
            cap = min(cap, num_post)
    elif int(mx.item()) > cap:
        # an explicit capacity must hold every drawn row: never truncate
        from .errors import RowFull
        raise RowFull(f"init_pairwise_bernoulli: a row draws {int(mx.item())} synapses, "
                      f"more than capacity {cap}")
    m = RaggedMatrix(num_pre, num_post, cap, multapse_free)
    _lib.call("sw_init_bernoulli_fill", num_pre, num_post, key, counter0, mode, float(density),
              _lib.ptr(lut_t), side, m.row_length.data_ptr(), m.target.data_ptr(), m.stride, st)
    m.version += 1
    return m, SynVarMatrix(m, names)


def init_pairwise_bernoulli_density(num_pre: int, num_post: int, density: float,
                                    capacity_headroom: float, rng: CounterRng,
                                    var_names=(), exclude_diagonal: bool = False,
                                    multapse_free: bool = True, capacity: int | None = None):
    """``init_pairwise_bernoulli`` with p(i, j) = density (0 on the diagonal
    when excluded), drawn on the device with the reference's counters
    (connectivity.py:231-236).  Advances ``rng`` past the P*N draws."""
    if capacity_headroom < 1.0:
        raise ValueError("capacity_headroom must be >= 1")
    out = _init_rows(num_pre, num_post, rng.key, rng.counter, 1 if exclude_diagonal else 0,
                     density, None, 1, capacity_headroom, multapse_free, var_names, capacity)
    rng.counter += num_pre * num_post
    return out


def init_pairwise_bernoulli_torus(side: int, offset_prob: np.ndarray, capacity_headroom: float,
                                  rng: CounterRng, var_names=(), multapse_free: bool = True):
    """``init_pairwise_bernoulli`` on a side x side torus where p depends on
    the wrapped offset only (topomap.py:376-388).  ``offset_prob[dx + side*dy]``
    must be computed by host numpy (exp/hypot)."""
    n = side * side
    out = _init_rows(n, n, rng.key, rng.counter, 2, 0.0, offset_prob, side, capacity_headroom,
                     multapse_free, var_names)
    rng.counter += n * n
    return out


def spikes_to_bits(spikes: torch.Tensor, n: int) -> torch.Tensor:
    """Index tensor -> packed uint32 spike mask (int32 storage), on the device."""
    flags = torch.zeros(((n + 31) // 32) * 32, dtype=torch.int64, device=DEV)
    if spikes.numel():
        flags[spikes.to(device=DEV, dtype=torch.int64)] = 1
    w = (flags.view(-1, 32) << torch.arange(32, device=DEV, dtype=torch.int64)).sum(dim=1)
    return torch.where(w >= 2**31, w - 2**32, w).to(torch.int32)


class PropBuckets:
    """Post-slab bucketed copy of a matrix and its weights for
    propagate_spikes over a matrix whose structure and weights stay fixed
    across many steps (sw_prop_buckets_build; SURVEY §8e "column slices of
    every row").  Each row's synapses are grouped by 16384-post slab inside
    the row's own slot range, so the propagation reads every synapse of a
    spiking row once and accumulates in shared memory instead of L2 atomics.
    Like TransposeMap (connectivity.py:151-192) it goes stale on a structural
    change (``m.version``, checked).  Both kernels read the copy's weight
    snapshot taken at build()/refresh(): after a weight-only change call
    ``refresh()`` (until then every propagation, whatever its spike count,
    uses the snapshot)."""

    def __init__(self, m: RaggedMatrix, weights: torch.Tensor):
        if weights.dtype != torch.float64:
            raise TypeError("float64 weights expected")
        self.m, self.weights = m, weights
        self.slabs = int(_lib.lib().sw_prop_bucket_slabs(m.num_post))
        if self.slabs == 0:
            raise ValueError("bucketed propagation needs 1 <= num_post <= 131072")
        n = m.num_pre * m.stride
        dev = m.target.device
        self.bt = torch.empty(n, dtype=torch.int16, device=dev)
        self.bslot = torch.empty(n, dtype=torch.int16, device=dev)
        self.bw = torch.empty(n, dtype=torch.float64, device=dev)
        self.soff = torch.empty(m.num_pre * (self.slabs + 1), dtype=torch.int16, device=dev)
        nbytes = int(_lib.lib().sw_prop_bucketed_workspace_bytes(m.num_post))
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        self.version = -1
        self.build()

    def build(self) -> None:
        m = self.m
        _lib.call("sw_prop_buckets_build", m.row_length.data_ptr(), m.target.data_ptr(),
                  self.weights.data_ptr(), m.num_pre, m.num_post, m.stride, self.bt.data_ptr(),
                  self.bslot.data_ptr(), self.bw.data_ptr(), self.soff.data_ptr(), _lib.stream_ptr())
        self.version = m.version

    def refresh(self) -> None:
        """Re-gather the weight copy after the weights (not the structure) changed."""
        self.check_fresh()
        m = self.m
        _lib.call("sw_prop_buckets_refresh", m.row_length.data_ptr(), self.weights.data_ptr(),
                  m.num_pre, m.stride, self.bslot.data_ptr(), self.bw.data_ptr(), _lib.stream_ptr())

    def check_fresh(self) -> None:
        if self.version != self.m.version:
            from .errors import StaleTranspose
            raise StaleTranspose("bucketed rows older than their matrix")

    # below this many spiking rows the fixed cost of the slab pass (zeroing,
    # partial slabs, grid barrier, reduction) exceeds the L2-atomic kernel's
    MIN_SPIKES = 4096

    def propagate(self, spikes: torch.Tensor, n_spikes: torch.Tensor, max_spikes: int,
                  out: torch.Tensor) -> str:
        """out[j] += weights of the spiking rows onto j (device spike list and
        count); returns the kernel used ("bucketed" or "atomic")."""
        self.check_fresh()
        m = self.m
        if max_spikes < self.MIN_SPIKES:
            # same weight snapshot as the slab pass (bw), so the result never
            # depends on which kernel the spike count selects
            _lib.call("sw_propagate_bucketed_atomic", self.soff.data_ptr(), self.bt.data_ptr(),
                      self.bw.data_ptr(), m.num_post, m.stride, spikes.data_ptr(), n_spikes.data_ptr(),
                      max(1, int(max_spikes)), out.data_ptr(), _lib.stream_ptr())
            return "atomic"
        _lib.call("sw_propagate_bucketed", self.soff.data_ptr(), self.bt.data_ptr(), self.bw.data_ptr(),
                  m.num_post, m.stride, spikes.data_ptr(), n_spikes.data_ptr(), max(1, int(max_spikes)),
                  out.data_ptr(), self.workspace.data_ptr(), self.workspace.numel(), _lib.stream_ptr())
        return "bucketed"


def propagate_spikes(m: RaggedMatrix, weights: torch.Tensor, spikes: torch.Tensor,
                     out: torch.Tensor, tmap=None, buckets: PropBuckets | None = None) -> None:
    """out[j] += weights of synapses from spiking rows onto j
    (connectivity.py:139-148).

    With a fresh ``tmap`` (TransposeMap of ``m``) the sum is computed per post
    in ascending-spike order through the transpose: bit-identical to the
    reference's np.add.at for an ascending spike set.  Without one the
    event-driven atomic kernel runs (warp per spiking row; summation order,
    and so the last bits, may vary between runs).  With fresh ``buckets``
    (PropBuckets of ``m`` and ``weights``) the bucketed kernel runs (same
    atomic-mode contract, no L2 atomics)."""
    if weights.dtype != torch.float64 or out.dtype != torch.float64:
        raise TypeError("float64 weights/out expected")
    st = _lib.stream_ptr()
    if buckets is not None:
        if buckets.m is not m or buckets.weights.data_ptr() != weights.data_ptr():
            raise ValueError("buckets were built for another matrix / weight plane")
        sp = spikes.to(device=DEV, dtype=torch.int32).contiguous()
        n = torch.tensor([sp.numel()], dtype=torch.int32, device=DEV)
        buckets.propagate(sp, n, sp.numel(), out)
        return
    if tmap is not None:
        tmap.check_fresh()
        bits = spikes_to_bits(spikes, m.num_pre)
        pr = (_lib.PropProj * 1)()
        pr[0].col_ptr, pr[0].src_pre, pr[0].src_slot = (tmap.col_ptr.data_ptr(),
                                                        tmap.src_pre.data_ptr(),
                                                        tmap.src_slot.data_ptr())
        pr[0].col_length = tmap.col_length.data_ptr()
        pr[0].weights, pr[0].spike_bits, pr[0].stride = weights.data_ptr(), bits.data_ptr(), m.stride
        import ctypes as _c
        _lib.call("sw_propagate_ordered", _c.cast(pr, _c.c_void_p), 1, m.num_post, out.data_ptr(), 1, st)
        return
    sp = spikes.to(device=DEV, dtype=torch.int32).contiguous()
    n = torch.tensor([sp.numel()], dtype=torch.int32, device=DEV)
    _lib.call("sw_propagate_atomic", m.row_length.data_ptr(), m.target.data_ptr(),
              weights.data_ptr(), m.num_pre, m.num_post, m.stride, sp.data_ptr(), n.data_ptr(),
              max(1, sp.numel()), out.data_ptr(), *_lib.prop_workspace(), st)


def write_snapshot_csv(fh, m: RaggedMatrix, syn: SynVarMatrix | None = None,
                       columns=(("weight", "g"),)) -> None:
    """Connectivity snapshot ``pre,post[,var...]`` sorted by (pre, post), in
    the reference's text format (connectivity.py:265-283): the valid slots
    are compacted and sorted on the device, then formatted on the host."""
    mask = m.slot_mask()
    pre = torch.arange(m.num_pre, device=m.target.device, dtype=torch.int64)[:, None].expand_as(mask)[mask]
    post = m.target[mask].to(torch.int64)
    order = torch.argsort(pre * m.num_post + post)
    header = "pre,post"
    cols = []
    if syn is not None:
        for label, plane in columns:
            header += "," + label
            cols.append(syn.planes[plane][mask][order].cpu().numpy())
    pre = pre[order].cpu().numpy()
    post = post[order].cpu().numpy()
    fh.write(header + "\n")
    for k in range(pre.size):
        extra = "".join("," + repr(float(c[k])) for c in cols)
        fh.write(f"{pre[k]},{post[k]}{extra}\n")
