"""Topographic-map model on the device (``sparsewire/topomap.py``).

A Poisson source grid drives a conductance-LIF target grid through
feed-forward and lateral plastic projections with trace STDP and
distance-dependent rewiring.  Per 0.1 ms step one ``sw_topomap_step``
(4 fused kernels + tick); every t_rewiring one ``RewiringRule`` update per
projection (device-side keys, host-phase histogram, thread-per-row
eliminate/form) and a device-gated transpose remap.  With ``use_graph`` one
rewiring period (10 steps + the rewiring group) is captured once as a CUDA
graph and replayed; stimulus changes (every 200 steps) only rewrite the
source probabilities between replays.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bitfield import Bitfield
from .connectivity import descriptor, init_pairwise_bernoulli_torus
from .geometry import GridGeometry
from .neurons import LifCondLayer, LifCondParams, PoissonParams, PoissonSource
from .plasticity import StdpParams, StdpSynapses
from .sharding import SpikeGather
from .rng import CounterRng, fold_key
from .updates import Model, RuleDescriptor

BASE_SIDE = 16


# sheets up to this size step in one single-CTA persistent launch per period
PERSISTENT_MAX_NODES = 512   # single-CTA periods up to here; s = 2 (1024 nodes): 2-launch steps 12.2 vs 13.0 us
# larger unsharded sheets: sw_topomap_steps_fused (SW_TM_FUSE=0: one
# sw_topomap_step per step, for comparison)
FUSED_STEPS = os.environ.get("SW_TM_FUSE", "1") != "0"
# rewiring periods captured per CUDA graph (a divisor of the periods per
# stimulus interval is used): one replay per 10 ms of model time keeps the
# host loop off the critical path for small sheets
PERIODS_PER_GRAPH = 10


@dataclass
class RewiringParams:
    p_form: float
    sigma_form: float
    g_theta: float = 0.1
    p_elim_dep: float = 2.45e-2 * 50
    p_elim_pot: float = 1.36e-4 * 50
    t_rewiring: float = 1.0
    n_attempts: int = 10
    g_init: float = 0.2

    @classmethod
    def feedforward(cls) -> "RewiringParams":
        return cls(p_form=0.16, sigma_form=2.5)

    @classmethod
    def lateral(cls) -> "RewiringParams":
        return cls(p_form=1.0, sigma_form=1.0)


def formation_probability(params: RewiringParams, d):
    """topomap.py:49-52 (host numpy; feeds the device LUT)."""
    return params.p_form * np.exp(-(np.asarray(d, dtype=np.float64) ** 2)
                                  / (2.0 * params.sigma_form ** 2))


def elimination_probability(params: RewiringParams, g_syn):
    g = np.asarray(g_syn, dtype=np.float64)
    return np.where(g < params.g_theta, params.p_elim_dep, params.p_elim_pot)


def expected_initial_degree(params: RewiringParams, geometry: GridGeometry) -> float:
    d = geometry.toroidal_distance(0, np.arange(geometry.n))
    return float(np.sum(formation_probability(params, d)))


class RewiringRule:
    """One projection's rewiring update (topomap.py:70-223) on the device."""

    def __init__(self, name, matrix, syn, geometry: GridGeometry, params: RewiringParams,
                 total_attempts: int, weight_plane: str = "g", record_events: bool = True,
                 form_lut: np.ndarray | None = None, dist_lut: np.ndarray | None = None):
        self.name = name
        self.matrix = matrix
        self.syn = syn
        self.geometry = geometry
        self.params = params
        self.total_attempts = total_attempts
        self.weight_plane = weight_plane
        self.record_events = record_events
        P, dev = matrix.num_pre, "cuda"
        self.attempt_bits = Bitfield(P, matrix.num_post)   # kept clear, as the reference leaves it
        self.attempts = torch.zeros(P, dtype=torch.int32, device=dev)
        self._keys = torch.zeros(2, dtype=torch.int64, device=dev)
        self._totals = torch.zeros(16, dtype=torch.int64, device=dev)
        self.changed = torch.zeros(1, dtype=torch.int32, device=dev)
        self._rej = torch.zeros(1, dtype=torch.int64, device=dev)
        self._update = torch.zeros(1, dtype=torch.int64, device=dev)
        self._host_update = 0
        self._ev_off = torch.zeros(P, dtype=torch.int32, device=dev)
        # host-numpy LUTs by torus offset; injectable for parity tests
        dist = geometry.offset_distance_lut() if dist_lut is None else np.asarray(dist_lut)
        if form_lut is None:
            form_lut = formation_probability(params, dist)
        self._dist_lut = torch.from_numpy(np.ascontiguousarray(dist, dtype=np.float64)).to(dev)
        self._form_lut = torch.from_numpy(np.ascontiguousarray(form_lut, dtype=np.float64)).to(dev)
        self._prm = _lib.RewireParams()
        p = self._prm
        p.side = geometry.side
        p.total_attempts = total_attempts
        p.form_lut, p.dist_lut = self._form_lut.data_ptr(), self._dist_lut.data_ptr()
        p.g_theta, p.p_dep, p.p_pot, p.g_init = (params.g_theta, params.p_elim_dep,
                                                 params.p_elim_pot, params.g_init)
        self._alloc_update_buffers(total_attempts)
        self.forced_attempts = False
        self.last_stats: dict[str, int] = {}
        self.elim_events: list[tuple[float, float]] = []
        self.form_events: list[tuple[float, float]] = []

    def _alloc_update_buffers(self, attempts_total: int) -> None:
        """Event records (one per attempt) and the scratch of the serial path
        for rows with more than 64 attempts, sized for attempts_total."""
        dev = self.attempts.device
        cap_ev = max(1, attempts_total)
        self._ev_kind = torch.zeros(cap_ev, dtype=torch.int8, device=dev)
        self._ev_d = torch.zeros(cap_ev, dtype=torch.float64, device=dev)
        nb = int(_lib.lib().sw_rewire_scratch_bytes(self.matrix.num_post, attempts_total))
        self._heavy = torch.zeros((nb + 7) // 8, dtype=torch.int64, device=dev)
        self._prm.total_attempts = attempts_total
        self._prm.scratch = self._heavy.data_ptr()
        # transpose patch log (sw_transpose_patch): changed rows + removed pairs
        self.patch_cap = max(1, attempts_total)
        self.patch_log = torch.zeros(4 + 3 * self.patch_cap, dtype=torch.int32, device=dev)
        self._prm.patch_log, self._prm.patch_cap = self.patch_log.data_ptr(), self.patch_cap

    def force_attempts(self, attempts) -> None:
        """Use these per-row attempt counts instead of the host-phase draws
        (tests and microbenchmarks; the host stream is then not drawn)."""
        a = np.ascontiguousarray(attempts, dtype=np.int32)
        self.forced_attempts = True
        self.attempts.copy_(torch.from_numpy(a))
        self._alloc_update_buffers(max(int(a.sum()), self.total_attempts))

    def _device_pass(self, model, binding, pass_index, host_key, row_base) -> bool:
        p = self._prm
        p.host_prefix = fold_key(model.seed, "host")
        p.row_prefix = fold_key(model.seed, "row")
        p.rule_id = binding.rule_id
        if self._host_update != binding.update_count:
            self._update.fill_(binding.update_count)
        rec = self.record_events
        d = descriptor(self.matrix, self.syn)
        _lib.call("sw_rewire_update", ctypes.byref(d), self.syn.plane_index(self.weight_plane),
                  ctypes.byref(p), self.attempts.data_ptr(), self._update.data_ptr(),
                  self._keys.data_ptr(), self._totals.data_ptr(), self.changed.data_ptr(),
                  self._rej.data_ptr(), self._ev_off.data_ptr() if rec else None,
                  self._ev_kind.data_ptr() if rec else None, self._ev_d.data_ptr() if rec else None,
                  int(self.forced_attempts), _lib.stream_ptr())
        self._host_update = binding.update_count + 1
        self.matrix.version += 1
        return False

    def descriptor(self) -> RuleDescriptor:
        d = RuleDescriptor(name=self.name, device_pass=self._device_pass)
        d.changed_flag = self.changed
        d.patch_source = self      # patch_log / patch_cap for an incremental remap
        return d

    def collect(self, time_ms: float) -> None:
        """topomap.py:202-223: per-update statistics and events, row order."""
        t = self._totals.cpu().numpy()
        if t[7]:
            from .errors import KTooLarge
            raise KTooLarge(f"{self.name}: more attempts on one row than num_post")
        self.last_stats = {"attempts": int(t[5]), "elim_candidates": int(t[0] + t[1]),
                           "form_candidates": int(t[2] + t[3] + t[4]), "removed": int(t[0]),
                           "kept": int(t[1]), "formed": int(t[2]), "form_missed": int(t[3]),
                           "form_full": int(t[4])}
        if self.record_events:
            n = int(t[5])
            kind = self._ev_kind[:n].cpu().numpy()
            dist = self._ev_d[:n].cpu().numpy()
            self.elim_events.extend((time_ms, float(x)) for x in dist[kind == 1])
            self.form_events.extend((time_ms, float(x)) for x in dist[kind == 2])


class TopomapRecorder:
    """The reference's analysis trail (topomap.py:235-318) over the device
    model: degree statistics and the on-axis displacement profile at every
    snapshot, edge lists at the start and end, rewiring events and
    (optionally) spikes, with the reference's CSV writers (same formats,
    byte-identical for the same state; cli.py:117-125 for the edge lists).
    Snapshots copy the connectivity to the host, so they run between
    CUDA-graph replays, never inside one."""

    def __init__(self, snapshot_every_ms: float = 200.0, record_spikes: bool = False):
        self.snapshot_every_ms = snapshot_every_ms
        self.record_spikes = record_spikes
        self.degrees: list[tuple] = []
        self.profile: list[tuple] = []
        self.snapshots: dict[tuple[str, str], tuple] = {}
        self.events: dict[tuple[str, str], list[tuple[float, float]]] = {}
        self.spikes: dict[str, list[tuple[float, int]]] = {"source": [], "target": []}

    def on_spikes(self, population: str, t_ms: float, ids) -> None:
        if self.record_spikes and len(ids):
            self.spikes[population].extend((t_ms, int(i)) for i in ids)

    @staticmethod
    def host_edges(model, proj: str):
        """(pre, post, w, row_length, num_post) of a projection, row-major slot
        order (RaggedMatrix.edge_list, connectivity.py:55-60)."""
        m, syn = model.net.matrices[proj]
        mask = m.slot_mask()
        pre, post = m.edge_list()
        w = syn.planes["g"][mask].cpu().numpy()
        return pre, post, w, m.row_length.cpu().numpy(), m.num_post

    def snapshot(self, t_ms: float, model, tag: str | None = None, rows: bool = True) -> None:
        for proj in ("ff", "lat"):
            self.snapshot_edges(t_ms, proj, model.geometry, *self.host_edges(model, proj), tag=tag, rows=rows)

    def snapshot_edges(self, t_ms, proj, geometry, pre, post, w, row_length, num_post,
                       tag=None, rows=True) -> None:
        if rows:
            in_deg = np.bincount(post, minlength=num_post)
            out_deg = row_length
            self.degrees.append((t_ms, proj, float(in_deg.mean()), float(in_deg.std()),
                                 float(out_deg.mean()), float(out_deg.std())))
            self._profile_rows(t_ms, proj, geometry, pre, post, w)
        if tag is not None:
            self.snapshots[(proj, tag)] = (pre.copy(), post.copy(), w.copy())

    def _profile_rows(self, t_ms, proj, geom, pre, post, w):
        half = geom.side // 2
        dx, dy = geom.displacement(pre, post)
        on_axis = dx == 0
        dy_idx = (dy[on_axis] + half).astype(np.int64)
        counts = np.bincount(dy_idx, minlength=geom.side)
        weight_sums = np.bincount(dy_idx, weights=w[on_axis], minlength=geom.side)
        for b in range(geom.side):
            mean_w = weight_sums[b] / counts[b] if counts[b] else 0.0
            self.profile.append((t_ms, proj, b - half, counts[b] / geom.n, mean_w))

    def take_events(self, model) -> None:
        for proj, rule in (("ff", model.ff_rule), ("lat", model.lat_rule)):
            self.events[(proj, "elimination")] = rule.elim_events
            self.events[(proj, "formation")] = rule.form_events

    # -- CSV output (topomap.py:287-318, cli.py:117-125) --------------------------
    def write_spikes_csv(self, fh, population: str) -> None:
        fh.write("time_ms,neuron_id\n")
        for t, i in self.spikes[population]:
            fh.write(f"{t:g},{i}\n")

    def write_degrees_csv(self, fh) -> None:
        fh.write("time_ms,projection,mean_in,std_in,mean_out,std_out\n")
        for t, proj, mi, si, mo, so in self.degrees:
            fh.write(f"{t:g},{proj},{mi:.9g},{si:.9g},{mo:.9g},{so:.9g}\n")

    def write_profile_csv(self, fh) -> None:
        fh.write("time_ms,projection,y_displacement,conn_prob,mean_weight\n")
        for t, proj, dy, cp, mw in self.profile:
            fh.write(f"{t:g},{proj},{dy},{cp:.9g},{mw:.9g}\n")

    def write_events_csv(self, fh, kind: str) -> None:
        """Counts per (time bin, integer distance bin), both projections."""
        fh.write("time_bin_ms,distance_bin,count\n")
        bin_ms = self.snapshot_every_ms
        merged: dict[tuple[float, int], int] = {}
        for (proj, k), events in sorted(self.events.items()):
            if k != kind:
                continue
            for t, d in events:
                key = (math.floor(t / bin_ms) * bin_ms, int(d))
                merged[key] = merged.get(key, 0) + 1
        for (tb, db) in sorted(merged):
            fh.write(f"{tb:g},{db},{merged[(tb, db)]}\n")

    def write_connectivity_csv(self, fh, proj: str, tag: str) -> None:
        """``pre,post,weight`` sorted by (pre, post), weights repr'd
        (cli.py:117-125)."""
        pre, post, w = self.snapshots[(proj, tag)]
        fh.write("pre,post,weight\n")
        for k in np.lexsort((post, pre)):
            fh.write(f"{pre[k]},{post[k]},{float(w[k])!r}\n")


@dataclass
class RunRecord:
    steps: int = 0
    rewiring_executions: int = 0
    stimulus_changes: int = 0
    rewires_per_update: list = field(default_factory=list)


class TopomapModel:
    """topomap.py:329-493 on the device."""

    def __init__(self, scale: int, seed: int, workers: int = 1, always_remap: bool = False,
                 incremental_remap: bool = True,
                 capacity_headroom: float = 4.0, record_events: bool = True,
                 use_graph: bool = True, rates_on_device: bool = False, process_group=None):
        """``process_group`` (torch.distributed, NCCL): postsynaptic sharding
        over its ranks (sharding.py): this rank updates the LIF state of and
        propagates into its own post range, target spikes are all-gathered
        every step, STDP and rewiring run replicated."""
        _lib.require_cuda()
        scale = max(scale, 1)
        self.scale = scale
        self.seed = seed
        self.h = LifCondParams().h
        self.geometry = GridGeometry(BASE_SIDE * scale)
        n = self.geometry.n
        self.ff_params = RewiringParams.feedforward()
        self.lat_params = RewiringParams.lateral()
        self.stdp_params = StdpParams()
        self.use_graph = use_graph
        self.rates_on_device = rates_on_device
        self.net = Model(seed, workers=workers, always_remap=always_remap,
                         incremental_remap=incremental_remap)
        ff_m, ff_syn = self._init_projection("ff", self.ff_params, CounterRng(seed, "init", "ff"),
                                             capacity_headroom)
        lat_m, lat_syn = self._init_projection("lat", self.lat_params,
                                               CounterRng(seed, "init", "lat"), capacity_headroom)
        self.source = PoissonSource(self.geometry, PoissonParams())
        self.target = LifCondLayer(n)
        self.pg = process_group
        if process_group is not None:
            import torch.distributed as dist
            rank, world = dist.get_rank(process_group), dist.get_world_size(process_group)
        else:
            rank, world = 0, 1
        self.shard = SpikeGather(n, rank, world, "cuda", process_group)
        self.post_lo, self.post_hi = self.shard.lo, self.shard.hi
        if world > 1:
            # target spikes live in the all-gather buffer (world * words-per-rank words)
            self.target.spike_bits = self.shard.bits
            # one eager collective: the communicator exists before any graph capture
            self.shard.gather()
        self.ff_stdp = StdpSynapses(ff_m, ff_syn, self.h, self.stdp_params)
        self.lat_stdp = StdpSynapses(lat_m, lat_syn, self.h, self.stdp_params)
        self.ff_tmap = self.net.register_transpose("ff")
        self.lat_tmap = self.net.register_transpose("lat")
        attempts = self.ff_params.n_attempts * scale * scale
        self.ff_rule = RewiringRule("ff_rewire", ff_m, ff_syn, self.geometry, self.ff_params,
                                    attempts, record_events=record_events)
        self.lat_rule = RewiringRule("lat_rewire", lat_m, lat_syn, self.geometry, self.lat_params,
                                     attempts, record_events=record_events)
        self.net.add_rule("rewiring", "ff", self.ff_rule.descriptor())
        self.net.add_rule("rewiring", "lat", self.lat_rule.descriptor())
        self._poisson_key = fold_key(seed, "poisson")
        self._stim_rng = CounterRng(seed, "stimulus")
        self._pending = torch.zeros(n, dtype=torch.float64, device="cuda")
        self._step = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.spike_counts = torch.zeros(2, dtype=torch.int64, device="cuda")
        self._barrier = torch.zeros(2, dtype=torch.int32, device="cuda")
        self._src_alt = self._tgt_alt = None     # second spike buffers of sw_topomap_steps_fused
        self.step_index = 0
        self._graphs = {}        # periods per graph -> captured CUDA graph
        self._update_log = None

    def _init_projection(self, name, params, rng, headroom):
        lut = formation_probability(params, self.geometry.offset_distance_lut())
        m, syn = init_pairwise_bernoulli_torus(self.geometry.side, lut, headroom, rng,
                                               var_names=("g",))
        syn.planes["g"].copy_(torch.where(m.slot_mask(), params.g_init, 0.0))
        self.net.add_matrix(name, m, syn)
        return m, syn

    # -- stepping ------------------------------------------------------------------
    def _draw_centers(self):
        bx = self._stim_rng.uniform01() * BASE_SIDE
        by = self._stim_rng.uniform01() * BASE_SIDE
        return [(bx + a * BASE_SIDE, by + b * BASE_SIDE)
                for a in range(self.scale) for b in range(self.scale)]

    def _step_struct(self) -> _lib.TopomapStep:
        s = _lib.TopomapStep()
        lif, lp = self.target, self.target.params
        s.n = self.geometry.n
        s.step = self._step.data_ptr()
        s.poisson_key = self._poisson_key
        s.p_src = self.source.probabilities(self.h).data_ptr()
        s.src_bits, s.tgt_bits = self.source.spike_bits.data_ptr(), lif.spike_bits.data_ptr()
        s.V, s.g_tot, s.ref_until = lif.V.data_ptr(), lif.g.data_ptr(), lif.refractory_until.data_ptr()
        s.pending = self._pending.data_ptr()
        s.decay_s, s.g_leak, s.v_rest, s.e_exc = lif._decay_s, lp.g_leak, lp.v_rest, lp.e_exc
        s.v_theta, s.v_reset, s.h, s.tau_m = lp.v_theta, lp.v_reset, lp.h, lp.tau_m
        s.ref_steps = lif._ref_steps
        for pre, stdp, tm in (("ff", self.ff_stdp, self.ff_tmap), ("lat", self.lat_stdp, self.lat_tmap)):
            m = stdp.matrix
            setattr(s, f"{pre}_row_length", m.row_length.data_ptr())
            setattr(s, f"{pre}_target", m.target.data_ptr())
            setattr(s, f"{pre}_g", stdp.syn.planes["g"].data_ptr())
            setattr(s, f"{pre}_stride", m.stride)
            setattr(s, f"{pre}_col_ptr", tm.col_ptr.data_ptr())
            setattr(s, f"{pre}_col_len", tm.col_length.data_ptr())
            setattr(s, f"{pre}_src_pre", tm.src_pre.data_ptr())
            setattr(s, f"{pre}_src_slot", tm.src_slot.data_ptr())
            setattr(s, f"{pre}_x", stdp.x.data_ptr())
            setattr(s, f"{pre}_y", stdp.y.data_ptr())
        sp = self.stdp_params
        s.decay_x, s.decay_y = self.ff_stdp._decay_x, self.ff_stdp._decay_y
        s.a_plus, s.a_minus, s.w_min, s.w_max = sp.a_plus, sp.a_minus, sp.w_min, sp.w_max
        s.post_lo, s.post_hi = self.post_lo, self.post_hi
        return s

    def _launch_step(self) -> None:
        s = self._step_struct()
        st = _lib.stream_ptr()
        if self.shard.world == 1:
            _lib.call("sw_topomap_step", ctypes.byref(s), self.spike_counts.data_ptr(), st)
            return
        self.launch_neurons(s)
        self.shard.gather()          # NCCL all-gather of the target-spike words
        self.launch_synapses(s)

    # the two halves of a sharded step (around the target-spike exchange)
    def launch_neurons(self, s=None) -> None:
        s = s if s is not None else self._step_struct()
        _lib.call("sw_topomap_neurons", ctypes.byref(s), _lib.stream_ptr())

    def launch_synapses(self, s=None) -> None:
        s = s if s is not None else self._step_struct()
        _lib.call("sw_topomap_synapses", ctypes.byref(s), self.spike_counts.data_ptr(),
                  _lib.stream_ptr())

    def _nccl(self) -> bool:
        if self.pg is None:
            return False
        import torch.distributed as dist
        return dist.get_backend(self.pg) == "nccl"

    def _period(self, rewire_steps: int) -> None:
        """rewire_steps model steps + the rewiring group (device only).
        Unsharded sheets of up to PERSISTENT_MAX_NODES: the steps run in one
        single-CTA persistent launch (barriers between the phases of a step);
        larger sheets: one launch per phase, which keeps every SM busy."""
        if self.shard.world == 1 and self.geometry.n <= PERSISTENT_MAX_NODES:
            s = self._step_struct()
            _lib.call("sw_topomap_run_steps", ctypes.byref(s), rewire_steps,
                      self.spike_counts.data_ptr(), self._barrier.data_ptr(), _lib.stream_ptr())
        elif self.shard.world == 1 and FUSED_STEPS:
            # 2 launches per step: propagation, then the STDP phases of step
            # t with the neuron phase of step t+1 (alternating spike buffers)
            if self._tgt_alt is None:
                self._src_alt = torch.zeros_like(self.source.spike_bits)
                self._tgt_alt = torch.zeros_like(self.target.spike_bits)
            s = self._step_struct()
            _lib.call("sw_topomap_steps_fused", ctypes.byref(s), self._src_alt.data_ptr(), self._tgt_alt.data_ptr(),
                      rewire_steps, self.spike_counts.data_ptr(), _lib.stream_ptr())
        else:
            for _ in range(rewire_steps):
                self._launch_step()
        # small sheets (single-block rewiring and remap kernels): the two
        # projections' updates on two streams (their kernels are too small to
        # fill the GPU; cooperative launches of larger sheets stay serial)
        self.net.run_update_group("rewiring", concurrent=self.geometry.n <= 256 and self.shard.world == 1)
        self._log_update()

    def _log_update(self) -> None:
        """(removed + formed) of both projections into the device update log."""
        if self._update_log is None:
            self._update_log = torch.zeros((1 << 16, 4), dtype=torch.int64, device="cuda")
        _lib.call("sw_topomap_log", self.ff_rule._update.data_ptr(), self.ff_rule._totals.data_ptr(),
                  self.lat_rule._totals.data_ptr(), self._update_log.data_ptr(),
                  self._update_log.shape[0], _lib.stream_ptr())

    def run(self, duration_ms: float, recorder=None, record: RunRecord | None = None) -> RunRecord:
        record = record or RunRecord()
        h = self.h
        stim_steps = int(round(PoissonParams().t_stim / h))
        rewire_steps = int(round(self.ff_params.t_rewiring / h))
        n_steps = int(round(duration_ms / h))
        snap_steps = int(round(recorder.snapshot_every_ms / h)) if recorder is not None else 0
        if recorder is not None and self.step_index == 0:
            recorder.snapshot(0.0, self, tag="initial")
        spikes_each_step = recorder is not None and recorder.record_spikes
        # sharded runs capture the period too when the collective can be
        # captured (NCCL: the spike all-gather becomes a graph node)
        graph_ok = (self.use_graph and (self.shard.world == 1 or self._nccl()) and not self.ff_rule.record_events
                    and not self.lat_rule.record_events and stim_steps % rewire_steps == 0
                    and not spikes_each_step
                    and (not snap_steps or snap_steps % rewire_steps == 0))
        u0 = self.ff_rule._host_update if self.ff_rule._host_update else 0
        # periods per replay: the largest divisor of the periods per stimulus
        # interval that is <= PERIODS_PER_GRAPH (a replay never crosses a
        # stimulus change)
        multi = 1
        if graph_ok:
            stim_periods = stim_steps // rewire_steps
            if snap_steps:
                stim_periods = math.gcd(stim_periods, snap_steps // rewire_steps)
            multi = max(d for d in range(1, min(PERIODS_PER_GRAPH, stim_periods) + 1) if stim_periods % d == 0)
        done = 0
        while done < n_steps:
            k = self.step_index
            if k % stim_steps == 0:
                if self.rates_on_device:
                    self.source.set_correlated_rates_device(self._draw_centers(), h)
                else:
                    self.source.set_correlated_rates(self._draw_centers())
                    self.source.probabilities(h)
                record.stimulus_changes += 1
            if graph_ok and k % rewire_steps == 0 and n_steps - done >= rewire_steps:
                span = multi * rewire_steps
                periods = multi if ((k % stim_steps) % span == 0 and n_steps - done >= span) else 1
                self._replay_period(rewire_steps, periods)
                self.step_index += periods * rewire_steps
                done += periods * rewire_steps
                record.steps += periods * rewire_steps
                record.rewiring_executions += periods
                if snap_steps and self.step_index % snap_steps == 0:
                    recorder.snapshot(self.step_index * h, self)
                continue
            self._launch_step()
            if spikes_each_step:
                from .neurons import unpack_spike_bits
                n = self.geometry.n
                recorder.on_spikes("source", k * h, unpack_spike_bits(self.source.spike_bits, n).cpu().numpy())
                recorder.on_spikes("target", k * h, unpack_spike_bits(self.target.spike_bits, n).cpu().numpy())
            self.step_index += 1
            done += 1
            record.steps += 1
            if self.step_index % rewire_steps == 0:
                self.net.run_update_group("rewiring")
                self._log_update()
                t_ms = self.step_index * h
                self.ff_rule.collect(t_ms)
                self.lat_rule.collect(t_ms)
                record.rewiring_executions += 1
            if snap_steps and self.step_index % snap_steps == 0:
                recorder.snapshot(self.step_index * h, self)
        if recorder is not None:
            just_written = n_steps == 0 or (snap_steps and self.step_index % snap_steps == 0)
            recorder.snapshot(self.step_index * h, self, tag="final", rows=not just_written)
            recorder.take_events(self)
        if record.rewiring_executions:
            n_up = self.ff_rule._host_update - u0
            log = self._update_log[u0:u0 + n_up].cpu().numpy() if n_up > 0 else np.zeros((0, 4))
            record.rewires_per_update.extend(int(x) for x in log.sum(axis=1))
        return record

    def _replay_period(self, rewire_steps: int, periods: int = 1) -> None:
        """Replay `periods` consecutive rewiring periods from one captured
        graph (every per-period input -- step counter, update counters, RNG
        keys -- lives on the device)."""
        g = self._graphs.get(periods)
        if g is None:
            # one eager period first (allocations, lazy init), then capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            self._log_update()   # allocate the log outside the capture
            saved = [(r, r._host_update) for r in (self.ff_rule, self.lat_rule)]
            counts = [b.update_count for b in self.net.groups["rewiring"]]
            self.net.timers.enabled = False
            try:
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s):
                        for _ in range(periods):
                            self._period(rewire_steps)
            finally:
                self.net.timers.enabled = True
            torch.cuda.current_stream().wait_stream(s)
            # capture did not execute anything: restore the host counters
            for (r, u), b, c in zip(saved, self.net.groups["rewiring"], counts):
                r._host_update = u
                b.update_count = c
            self._graphs[periods] = g
        g.replay()
        for r, b in zip((self.ff_rule, self.lat_rule), self.net.groups["rewiring"]):
            b.update_count += periods
            r._host_update = b.update_count

    def state_arrays(self) -> dict[str, np.ndarray]:
        out = {}
        for name in ("ff", "lat"):
            m, syn = self.net.matrices[name]
            mask = m.slot_mask()
            out[f"{name}.row_length"] = m.row_length.cpu().numpy()
            out[f"{name}.target"] = (m.target * mask).cpu().numpy()
            out[f"{name}.g"] = (syn.planes["g"] * mask).cpu().numpy()
        out["V"] = self.target.V.cpu().numpy()
        out["g_total"] = self.target.g.cpu().numpy()
        out["refractory"] = self.target.refractory_until.cpu().numpy()
        out["rates"] = self.source.rates_array()
        out["stdp_ff_x"] = self.ff_stdp.x.cpu().numpy()
        out["stdp_ff_y"] = self.ff_stdp.y.cpu().numpy()
        out["stdp_lat_x"] = self.lat_stdp.x.cpu().numpy()
        out["stdp_lat_y"] = self.lat_stdp.y.cpu().numpy()
        out["pending"] = self._pending.cpu().numpy()
        return out


def build_model(scale: int, seed: int, **kwargs) -> TopomapModel:
    return TopomapModel(scale, seed, **kwargs)
