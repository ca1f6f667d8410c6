#!/usr/bin/env python
"""Benchmark of the structural-plasticity hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload clf-c1|clf-c2]

Headline (BASELINE.json metric, configs[1]): e-prop + DEEP R training time
per epoch of the recurrent ALIF classifier 700 -> 256 hidden, 10% sparse
input/recurrent connectivity with DEEP R, 20 classes, batch 512, 1000-step
SHD-shaped synthetic trials (8156 training examples -> 16 batches/epoch).
A step = one training batch (1000 timesteps of forward + e-prop, gradient
scaling, L1, Adam x4, DEEP R group).  s/epoch = 16 x ms/step / 1000.

N > 1 (torchrun): the 512 replicas are sharded across ranks (batch-DP,
strong scaling) with one NCCL all-reduce of the raw gradients per batch.

--impl reference times the reference CPU path (the oracle port in
``oracle/``: numpy with one BLAS thread, the e-prop kernel in C with OpenMP
over the rows of each replica) on a bounded sample of the same workload and extrapolates
to s/epoch; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (num_inputs, hidden, density_in, density_rec, classes, batch, steps)
    "clf-c1": dict(num_inputs=700, hidden=256, density=0.10, classes=20, batch=512, steps=1000),
    "clf-c2": dict(num_inputs=700, hidden=1024, density=0.01, classes=20, batch=512, steps=1000),
}
NUM_TRAIN = 8156
EPOCH_BATCHES = -(-NUM_TRAIN // 512)   # 16


def measured_peak():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            d = json.load(open(p))
            return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None
        self.nvml = False

    # sampler process: NVML every 5 ms, one "sm_mhz,reason_mask" line per
    # sample; a separate process so the timed loop's GIL cannot starve it
    _SCRIPT = (
        "import sys, time, pynvml\n"
        "pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))\n"
        "print('max', pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)\n"
        "while True:\n"
        "    try:\n"
        "        print(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),\n"
        "              pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), flush=True)\n"
        "    except Exception:\n"
        "        pass\n"
        "    time.sleep(0.005)\n")

    def __enter__(self):
        self.samples, self.max_mhz, self.nvml = [], None, False
        try:
            import sys
            self.proc = subprocess.Popen([sys.executable, "-c", self._SCRIPT, str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()
            if len(first) == 2 and first[0] == "max":
                self.max_mhz = int(first[1])
                self.proc.stdout.readline()          # one live sample: the sampler runs
                self.nvml = True
                return self
            self.proc.kill()
        except Exception:
            self.proc = None
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        if self.nvml:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            for line in out.splitlines():
                f = line.split()
                if len(f) == 2:
                    try:
                        self.samples.append((int(f[0]), int(f[1])))
                    except ValueError:
                        pass
            return
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()

    def summary(self):
        if self.nvml:
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}   # nvmlClocksEventReason* masks
            sms = [x[0] for x in self.samples]
            reasons = sorted({k for _, m in self.samples for k, b in bits.items() if m & b})
            return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sms), "source": "nvml"}
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sms.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        lr = int(os.environ.get("LOCAL_RANK", "0"))
        # SW_BENCH_BACKEND=gloo exercises the multi-rank path on fewer GPUs
        # than ranks (validation only: ranks then share a device)
        backend = os.environ.get("SW_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # communicator set-up lines (NVLS / NVLink transport) on stderr;
            # stdout stays the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(lr % torch.cuda.device_count())
        dist.init_process_group(backend)
        return dist.get_rank(), ws, lr % torch.cuda.device_count()
    return 0, 1, 0


def flush_l2(buf):
    buf.add_(1)   # 256 MiB write > 126 MB L2


def workload_config(args, w, ws):
    """The config object of both arms' JSON lines (identical text)."""
    return {"workload": f"{args.workload}: e-prop ALIF classifier {w['num_inputs']}->{w['hidden']}, "
                        f"{int(w['density'] * 100)}% in/rec + DEEP R, 20 classes, batch {w['batch']}, "
                        f"{w['steps']}-step SHD-shaped synthetic trials, {EPOCH_BATCHES} batches/epoch",
            "global_batch": w["batch"], "seq_len": w["steps"], "parallelism": f"dp{ws}",
            "l2": "flushed (256 MiB write) between timed steps"}


# ------------------------------------------------------------------ reference arm
def cpu_reference_sample(w, sample_steps=None):
    """Time the oracle port of the classifier step on the host CPU over a
    bounded number of timesteps of one batch (+ one DEEP R group) and
    extrapolate to s/epoch.  Single-threaded."""
    # numpy's BLAS stays single-threaded: its spinning worker threads would
    # compete with the OpenMP threads of the C e-prop kernel, which carries
    # ~90% of the reference step
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1, user_api="blas"):
        return _cpu_reference_sample(w, sample_steps)


def _cpu_reference_sample(w, sample_steps):
    from oracle.classifier import TaskOracle, TrainerOracle
    task = TaskOracle(num_classes=w["classes"], num_inputs=w["num_inputs"],
                      example_steps=sample_steps or 4, seed=1, num_train=NUM_TRAIN)
    t0 = time.perf_counter()
    tr = TrainerOracle(task, hidden=w["hidden"], input_density=w["density"],
                       recurrent_density=w["density"], batch_size=w["batch"], seed=1)
    build_s = time.perf_counter() - t0
    times = []
    tr.forward(task.train_ids(0, w["batch"]), learn=True, step_times=times)
    # steady state: the first step pays the eligibility arrays' page faults
    per_step = statistics.median(times[1:]) if len(times) > 1 else times[0]
    t0 = time.perf_counter()
    inv = 1.0 / w["batch"]
    for t in (tr.m_in.planes["grad"], tr.m_rec.planes["grad"]):
        t *= inv
    tr.dr_in.l1_step()
    tr.dr_rec.l1_step()
    tr.adam_in.apply(tr.m_in.planes["w"], tr.m_in.planes["grad"])
    tr.adam_rec.apply(tr.m_rec.planes["w"], tr.m_rec.planes["grad"])
    tr.rewire_phase()
    upd = time.perf_counter() - t0
    batch_s = per_step * w["steps"] + upd
    from oracle.cbuild import threads
    return {"s_per_epoch": batch_s * EPOCH_BATCHES, "batch_s": batch_s, "per_step_s": per_step,
            "cores": threads(),
            "update_s": upd, "build_s": build_s, "sample_steps": task.example_steps}


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    for _ in range(args.steps):
        r = cpu_reference_sample(w, sample_steps=args.ref_sample_steps)
        vals.append(r["s_per_epoch"])
    v = statistics.median(vals)
    sample = (f"{r['sample_steps']} of {w['steps']} timesteps of one {w['batch']}-replica batch "
              f"(median step after the first) + one full update/DEEP R group, extrapolated "
              f"x{w['steps']} steps x{EPOCH_BATCHES} batches; oracle port: numpy + C e-prop "
              f"(oracle/c/oracle.c, OpenMP over the rows of each replica), numpy with 1 BLAS thread")
    line = {"impl": "reference", "metric": "e-prop+DEEP R training time per epoch",
            "value": round(v, 3), "unit": "s/epoch", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": workload_config(args, w, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": round(v, 3), "unit": "s/epoch", "cores": r["cores"], "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "s/epoch", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ microbenchmarks
FLIPS = (0.001, 0.003, 0.01, 0.03, 0.1)
SPIKE_QS = (0.001, 0.01, 0.1)


def count_moves(m, w, sign_slot, chunk=1 << 14):
    """Plane moves the eliminate pass will make (bench accounting, outside
    the timed region): per row with k sign-mismatched valid slots, the
    marked slots below n - k are the holes the chained swap-with-last fills
    (connectivity.py:130-136); tail removals move nothing."""
    import torch
    moves = 0
    S = m.stride
    cw = sign_slot.shape[1]
    shifts = torch.arange(32, device=w.device, dtype=torch.int64)
    for r0 in range(0, m.num_pre, chunk):
        r1 = min(m.num_pre, r0 + chunk)
        n = m.row_length[r0:r1].to(torch.int64)
        bits = ((sign_slot[r0:r1].to(torch.int64) & 0xFFFFFFFF)[:, :, None] >> shifts) & 1
        bits = bits.reshape(r1 - r0, cw * 32)[:, :S].bool()
        x = w[r0:r1]
        valid = torch.arange(S, device=w.device)[None, :] < n[:, None]
        mis = ((x < 0) & bits) | ((x > 0) & ~bits)
        mis &= valid
        k = mis.sum(dim=1)
        below = torch.arange(S, device=w.device)[None, :] < (n - k)[:, None]
        moves += int((mis & below).sum().item())
    return moves


def run_mupdate(fracs=FLIPS, P=1 << 20, N=65536, cap=1024, seed=1):
    """Connectivity-update microbench (SURVEY 8(d) M-update): DEEP R
    eliminate + form on a 2^20-row ragged matrix, cap 1024, N = 65536,
    R ~ 512 (Bernoulli(512/65536) rows from counters (seed,"init","M")),
    four float64 planes, sign flips of a Bernoulli(f) subset per update.
    Then the spike-propagation microbench (M-prop) on the same matrix:
    atomic, post-slab bucketed and ordered (bit-exact, transpose) modes."""
    import ctypes
    import torch
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.connectivity import descriptor, init_pairwise_bernoulli_density
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.rng import CounterRng, fold_key
    from paper_2510_19764_b200.updates import Model
    planes = ("w", "grad", "adam_m", "adam_v")
    m, syn = init_pairwise_bernoulli_density(P, N, 512.0 / N, 1.0, CounterRng(seed, "init", "M"),
                                             var_names=planes, capacity=cap)
    w = syn.planes["w"]
    w.normal_(0.0, 0.1)
    w.mul_(m.slot_mask())
    dr = DeepR(m, syn, "M", l1_strength=0.0)
    dr.init_bitfields(CounterRng(seed, "deep_r", "M"))
    model = Model(seed)
    model.add_matrix("M", m, syn)
    dr.register(model, "deep_r", "M")
    dr._sync_cache()   # build the slot-aligned sign cache once, outside the timed updates
    E = m.edge_count()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # warm-up group (no flips: nothing removed): first-launch module loading
    # and shared-memory attribute setup stay out of the timed updates
    model.run_update_group("deep_r")
    torch.cuda.synchronize()
    peak, _ = measured_peak()
    out = []
    for u, f in enumerate(fracs):
        d = descriptor(m, syn)
        _lib.call("sw_flip_signs", ctypes.byref(d), 0, fold_key(seed, "flip", u), f, _lib.stream_ptr())
        dr._sync_cache()
        moves = count_moves(m, w, dr._sign_slot)
        flush.add_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        model.run_update_group("deep_r")
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        removed = dr.last_removed
        # ind + w scan, 1 sign bit per slot, per-row words, plane
        # moves (72 B each: 4 planes + target, read + write), conn-bit RMW per
        # removal, appends + conn test-and-set per formed synapse (D = removed)
        alg = E * 12 + E // 8 + P * 24 + moves * 72 + removed * 16 + removed * 52
        gbs = alg / (ms * 1e-3) / 1e9
        out.append({"flip": f, "ms": round(ms, 3), "removed": int(removed), "moves": int(moves),
                    "alg_bytes": int(alg), "achieved_GBs": round(gbs, 1), "frac": round(gbs / peak, 4)})
        assert m.edge_count() == E, "DEEP R must conserve the edge count"
    res = {"rows": P, "num_post": N, "cap": cap, "edges": E, "update_sweep": out,
           "note": "moves = holes below n - k filled by the chained swap-with-last (tail removals move nothing)"}
    del dr, model
    res.update(run_mprop(m, syn, seed, flush, peak))
    del m, syn, w
    torch.cuda.empty_cache()
    return res


def _spike_list(P, q, seed):
    import torch
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.rng import fold_key
    p_dev = torch.full((P,), q, dtype=torch.float64, device="cuda")
    bits = torch.zeros((P + 31) // 32, dtype=torch.int32, device="cuda")
    lst = torch.zeros(P, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("sw_poisson_step", fold_key(seed, "spk", 0), 0, p_dev.data_ptr(), P, bits.data_ptr(),
              _lib.stream_ptr())
    _lib.call("sw_spike_bits_to_list", bits.data_ptr(), P, lst.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
    return bits, lst, cnt, int(cnt.item())


def _time_launch(launch, flush, reps=20):
    import torch
    for _ in range(3):
        launch()
    tot = 0.0
    for _ in range(reps):
        flush.add_(1)                 # L2 flushed between timed launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot * 1e3 / reps


def run_mprop(m, syn, seed, flush, peak, qs=SPIKE_QS):
    """Spike propagation (SURVEY 8(d) M-prop, connectivity.py:139-148) on the
    M matrix: the atomic event-driven kernel, the post-slab bucketed rows and
    the ordered (bit-exact, transpose-gathered) mode.  Bytes per step:
    S*(4+4) + S*R*(4+8) + N*8 (spike index + row length, the spiking rows'
    targets and weights, the output)."""
    import ctypes
    import torch
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.connectivity import PropBuckets
    from paper_2510_19764_b200.transpose import remap_transpose
    P, N = m.num_pre, m.num_post
    w = syn.planes["w"]
    outv = torch.zeros(N, dtype=torch.float64, device="cuda")
    for name in ("grad", "adam_m", "adam_v"):
        syn.planes.pop(name, None)
    torch.cuda.empty_cache()

    def line(q, S, us, mode, note):
        Rs = float(m.row_length[lst[:S].long()].double().mean().item()) if S else 0.0
        alg = S * 8 + S * Rs * 12 + N * 8
        gbs = alg / (us * 1e-6) / 1e9
        return {"q": q, "spiking_rows": S, "mode": mode, "us": round(us, 2), "alg_bytes": int(alg),
                "achieved_GBs": round(gbs, 1), "frac": round(gbs / peak, 4), "note": note}
    atomic, bucketed, ordered = [], [], []
    ws_ptr, ws_bytes = _lib.prop_workspace()
    for q in qs:
        bits, lst, cnt, S = _spike_list(P, q, seed)
        us = _time_launch(lambda: _lib.call("sw_propagate_atomic", m.row_length.data_ptr(), m.target.data_ptr(),
                                            w.data_ptr(), P, N, m.stride, lst.data_ptr(), cnt.data_ptr(), S,
                                            outv.data_ptr(), ws_ptr, ws_bytes, _lib.stream_ptr()), flush)
        atomic.append(line(q, S, us, "atomic", "L2 flushed before each timed launch"))
    # post-slab bucketed rows: the derived copy is built once for the fixed
    # matrix (cost reported), then every step reads each spiking row's
    # synapses once, without L2 atomics
    pb = PropBuckets(m, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pb.build()
    e1.record()
    e1.synchronize()
    build_ms = e0.elapsed_time(e1)
    e0.record()
    pb.refresh()
    e1.record()
    e1.synchronize()
    refresh_ms = e0.elapsed_time(e1)
    for q in qs:
        bits, lst, cnt, S = _spike_list(P, q, seed)
        kern = pb.propagate(lst, cnt, S, outv)
        us = _time_launch(lambda: pb.propagate(lst, cnt, S, outv), flush)
        r = line(q, S, us, "bucketed", "L2 flushed before each timed launch; reads 10 B/synapse of the bucketed copy")
        r["kernel"] = kern
        bucketed.append(r)
    del pb
    torch.cuda.empty_cache()
    # ordered mode: per post, the spiking rows' weights in ascending pre
    # order through the transpose (bit-identical to np.add.at on an ascending
    # spike list); it walks every column entry, so it is O(E) per step
    tm = remap_transpose(m)
    for q in qs:
        bits, lst, cnt, S = _spike_list(P, q, seed)
        pr = (_lib.PropProj * 1)()
        pr[0].col_ptr, pr[0].src_pre, pr[0].src_slot = tm.col_ptr.data_ptr(), tm.src_pre.data_ptr(), tm.src_slot.data_ptr()
        pr[0].weights, pr[0].spike_bits, pr[0].stride = w.data_ptr(), bits.data_ptr(), m.stride
        pr[0].col_length = tm.col_length.data_ptr()
        us = _time_launch(lambda: _lib.call("sw_propagate_ordered", ctypes.cast(pr, ctypes.c_void_p), 1, N,
                                            outv.data_ptr(), 0, _lib.stream_ptr()), flush, reps=5)
        r = line(q, S, us, "ordered", "bit-exact mode: walks all E transpose entries + spike bits per step "
                 "(E*8 B + gathers), so frac on the event-driven formula is low by construction")
        r["transpose_bytes_per_step"] = int(m.edge_count() * 8 + (P + 31) // 32 * 4)
        ordered.append(r)
    del tm
    torch.cuda.empty_cache()
    return {"propagate_atomic": atomic, "propagate_bucketed": bucketed, "propagate_ordered": ordered,
            "bucket_build_ms": round(build_ms, 3), "bucket_refresh_ms": round(refresh_ms, 3)}


def run_alif_bench(batch=512, hiddens=(256, 1024), reps=50):
    """ALIF step (neurons.py:60-67) + surrogate (:69-73) on [B, H] float32
    state (SURVEY 8(d) ALIF-step: B*H*(3*4*2 + 2*4 + 4) bytes), standalone
    kernels (the trainer fuses them into the forward pass)."""
    import torch
    from paper_2510_19764_b200 import _lib
    peak, _ = measured_peak()
    res = []
    for H in hiddens:
        n = batch * H
        v, a, z, rec, ext, psi = (torch.rand(n, dtype=torch.float32, device="cuda") for _ in range(6))
        z = (z < 0.05).float()

        def launch():
            _lib.call("sw_alif_surrogate", v.data_ptr(), a.data_ptr(), psi.data_ptr(), n, 0.0174, 0.6,
                      _lib.stream_ptr())
            _lib.call("sw_alif_step", v.data_ptr(), a.data_ptr(), z.data_ptr(), rec.data_ptr(), ext.data_ptr(),
                      n, 0.95, 0.9995, 0.0174, 0.6, _lib.stream_ptr())
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                for _ in range(reps):
                    launch()
        torch.cuda.current_stream().wait_stream(side)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        alg = n * (3 * 4 * 2 + 2 * 4 + 4)
        gbs = alg / (us * 1e-6) / 1e9
        res.append({"batch": batch, "hidden": H, "us": round(us, 2), "alg_bytes": alg,
                    "achieved_GBs": round(gbs, 1), "frac": round(gbs / peak, 4),
                    "note": "surrogate + step launches back to back in a CUDA graph (L2-resident: latency-bound, "
                            "SURVEY 8(d) 'report')"})
    return res


def cpu_micro_sample(P=16384, N=65536, cap=1024, seed=1, fracs=FLIPS, qs=SPIKE_QS):
    """CPU baseline of the M-update and M-prop microbenchmarks (BASELINE.md
    section 3): the oracle port (numpy restatement of deep_r.py:81-160 and
    connectivity.py:139-148, one thread) on a 16 384-row slice with the GPU
    instance's row statistics (R ~ 512, cap 1024, N = 65 536, 4 float64
    planes), extrapolated x (2^20 / P).  Test infrastructure, timed only."""
    import time
    from oracle.deep_r import DeepROracle
    from oracle.ragged import Ragged, bf_words, propagate_spikes as prop_oracle
    from oracle.updates import OracleModel
    rs = np.random.default_rng(seed)
    planes = ("w", "grad", "adam_m", "adam_v")
    m = Ragged(P, N, cap, planes)
    rl = np.minimum(rs.binomial(N, 512.0 / N, size=P), cap).astype(np.int32)
    for i in range(P):
        m.target[i, :rl[i]] = np.sort(rs.choice(N, rl[i], replace=False))
    m.row_length[:] = rl
    mask = m.slot_mask()
    m.planes["w"][:] = rs.normal(0.0, 0.1, m.target.shape) * mask
    dr = DeepROracle(m, l1=0.0)
    W = bf_words(N)
    rows = np.broadcast_to(np.arange(P)[:, None], m.target.shape)[mask]
    t = m.target[mask].astype(np.int64)
    bit = np.left_shift(np.uint64(1), (t & 63).astype(np.uint64))
    np.bitwise_or.at(dr.conn, (rows, t >> 6), bit)
    pos = m.planes["w"][mask] > 0
    np.bitwise_or.at(dr.sign, (rows[pos], (t >> 6)[pos]), bit[pos])
    assert dr.conn.shape[1] == W
    om = OracleModel(seed)
    om.add_matrix("M", m)
    dr.register(om, "deep_r", "M")
    scale = (1 << 20) / P
    upd = []
    for f in fracs:
        flips = (rs.random(m.target.shape) < f) & m.slot_mask()
        m.planes["w"][flips] *= -1.0
        t0 = time.perf_counter()
        om.run_update_group("deep_r")
        dt = time.perf_counter() - t0
        upd.append({"flip": f, "slice_s": round(dt, 3), "removed": int(dr.last_removed),
                    "extrapolated_ms": round(dt * scale * 1e3, 1)})
    prop = []
    out = np.zeros(N)
    for q in qs:
        spikes = np.flatnonzero(rs.random(P) < q)
        t0 = time.perf_counter()
        prop_oracle(m, m.planes["w"], spikes, out)
        dt = time.perf_counter() - t0
        prop.append({"q": q, "slice_ms": round(dt * 1e3, 3), "extrapolated_us": round(dt * scale * 1e6, 1)})
    return {"kind": "port", "cores": 1, "rows_sampled": P,
            "sample": f"{P}-row slice (R~512, cap {cap}, N={N}, 4 float64 planes), oracle port "
                      f"(numpy, 1 thread), timed on the host and extrapolated x{scale:g} to 2^20 rows",
            "update": upd, "propagate": prop}


def run_micro_sharded(pg, P=1 << 20, N=65536, cap=1024, seed=1, fracs=(0.01, 0.1)):
    """SURVEY 8(e) microbench sharding under torchrun: M-update with the rows
    sharded over the ranks (DeepR process_group: D and unplaced all-reduced,
    the activation histogram reduce-scattered by row owner) and M-prop with
    the posts sharded (each rank propagates into its column slice, no
    collective).  Times are the max over ranks; strong scaling (the matrix
    is the 2^20-row instance at every N)."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.connectivity import column_slice, descriptor, init_pairwise_bernoulli_density
    from paper_2510_19764_b200.deep_r import DeepR
    from paper_2510_19764_b200.rng import CounterRng, fold_key
    from paper_2510_19764_b200.sharding import shard_posts, shard_rows
    from paper_2510_19764_b200.updates import Model
    rank, world = dist.get_rank(pg), dist.get_world_size(pg)
    lo, hi = shard_rows(P, rank, world)
    rng = CounterRng(seed, "init", "M")
    rng.counter = lo * N                  # this rank's rows of the global draw sequence
    planes = ("w", "grad", "adam_m", "adam_v")
    m, syn = init_pairwise_bernoulli_density(hi - lo, N, 512.0 / N, 1.0, rng, var_names=planes, capacity=cap)
    w = syn.planes["w"]
    w.normal_(0.0, 0.1)
    w.mul_(m.slot_mask())
    dr = DeepR(m, syn, "M", l1_strength=0.0, process_group=pg, row0=lo, num_pre_global=P)
    srng = CounterRng(seed, "deep_r", "M")
    srng.counter = lo * dr.sign_bits.words.shape[1]
    dr.init_bitfields(srng)
    model = Model(seed)
    model.add_matrix("M", m, syn)
    dr.register(model, "deep_r", "M")
    model.run_update_group("deep_r")
    torch.cuda.synchronize()

    def max_ms(ms):
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=pg)
        return float(t.item())
    upd = []
    for u, f in enumerate(fracs):
        _lib.call("sw_flip_signs", ctypes.byref(descriptor(m, syn)), 0, fold_key(seed, "flip", u), f,
                  _lib.stream_ptr())
        dr._sync_cache()
        torch.cuda.synchronize()
        dist.barrier(group=pg)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        model.run_update_group("deep_r")
        e1.record()
        e1.synchronize()
        upd.append({"flip": f, "ms_max_over_ranks": round(max_ms(e0.elapsed_time(e1)), 3),
                    "removed_global": int(dr.last_removed)})
    del dr, model, m, syn, w
    torch.cuda.empty_cache()
    # M-prop: every rank holds all rows' synapses onto its post range
    full, fsyn = init_pairwise_bernoulli_density(P, N, 512.0 / N, 1.0, CounterRng(seed, "init", "M"),
                                                 var_names=("w",), capacity=cap)
    fsyn.planes["w"].normal_(0.0, 0.1)
    plo, phi = shard_posts(N, rank, world)
    ms_, ssyn = column_slice(full, fsyn, plo, phi)
    del full, fsyn
    torch.cuda.empty_cache()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    outv = torch.zeros(phi - plo, dtype=torch.float64, device="cuda")
    ws_ptr, ws_bytes = _lib.prop_workspace()
    prop = []
    for q in SPIKE_QS:
        bits, lst, cnt, S = _spike_list(P, q, seed)
        us = _time_launch(lambda: _lib.call("sw_propagate_atomic", ms_.row_length.data_ptr(), ms_.target.data_ptr(),
                                            ssyn.planes["w"].data_ptr(), P, phi - plo, ms_.stride, lst.data_ptr(),
                                            cnt.data_ptr(), S, outv.data_ptr(), ws_ptr, ws_bytes,
                                            _lib.stream_ptr()), flush)
        prop.append({"q": q, "spiking_rows": S, "us_max_over_ranks": round(max_ms(us * 1e-3) * 1e3, 2)})
    return {"rows": P, "parallelism": f"M-update rows / M-prop posts sharded x{world}",
            "update": upd, "propagate_atomic": prop}


def topomap_cpu_baseline(seed=1, timed=((1, 200.0), (2, 50.0), (4, 10.0))):
    """CPU baseline of the topomap sweep: the oracle port of
    TopomapModel.run (oracle/topomap_port.py: numpy, np.add.at propagation,
    the reference's Python rewiring row loop; 1 thread) timed at s = 1, 2, 4
    on this host; s = 8 and 16 extrapolated from s = 4 with wall time per
    model ms proportional to N (the port's step cost is O(N) per step),
    stated as such."""
    from oracle.topomap_port import time_topomap
    res = {}
    for s_, ms in timed:
        r = time_topomap(s_, ms, seed)
        r["kind"] = "timed"
        res[f"s{s_}"] = r
    last_s, last_ms = timed[-1]
    base = res[f"s{last_s}"]
    for s_ in (8, 16):
        if f"s{s_}" in res:
            continue
        f = (s_ / last_s) ** 2
        res[f"s{s_}"] = {"n": 256 * s_ * s_, "x_realtime": round(base["x_realtime"] / f, 6),
                         "kind": f"extrapolated from s={last_s} x (N ratio {f:g})"}
    return {"kind": "port", "cores": 1, "sample": "oracle/topomap_port.py (numpy restatement of "
            "TopomapModel.run, topomap.py:398-474; no recorder), build excluded; "
            + ", ".join(f"s={a}: {b:g} ms model" for a, b in timed) + "; s=8,16 extrapolated", "per_scale": res}


def run_topomap_sweep(scales=(1, 2, 4, 8, 16), model_ms=100.0, seed=1, process_group=None):
    """Topographic-map simulation speed (x realtime) vs network size,
    TopomapModel(s) semantics, no recorder, stimulus rates computed on the
    device (rates_on_device).  One GPU: CUDA-graph replay per 1 ms.  Under
    torchrun: postsynaptic sharding over the ranks with a per-step NCCL
    all-gather of the target spikes (eager stepping); time = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2510_19764_b200.topomap import TopomapModel
    res = {}
    for s in scales:
        t0 = time.perf_counter()
        model = TopomapModel(s, seed=seed, record_events=False, use_graph=True,
                             rates_on_device=True, process_group=process_group,
                             incremental_remap=os.environ.get("SW_TOPO_REMAP", "patch") != "full")
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
        model.run(40.0)   # warm-up: graph captures, first replays, two stimulus changes
        torch.cuda.synchronize()
        if process_group is not None:
            dist.barrier(group=process_group)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rec = model.run(model_ms)
        e1.record()
        e1.synchronize()
        wall_ms = e0.elapsed_time(e1)
        if process_group is not None:
            t = torch.tensor([wall_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=process_group)
            wall_ms = float(t.item())
        res[f"s{s}"] = {"n": model.geometry.n, "x_realtime": round(model_ms / wall_ms, 3),
                        "us_per_step": round(wall_ms * 1e3 / rec.steps, 2), "build_s": round(build_s, 2),
                        "rewires": int(sum(rec.rewires_per_update)),
                        "ff_edges": model.ff_rule.matrix.edge_count(),
                        "lat_edges": model.lat_rule.matrix.edge_count()}
        del model
        torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ device arm
def run_device(args, w):
    import torch
    import torch.distributed as dist
    rank, ws, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    from paper_2510_19764_b200 import _lib
    from paper_2510_19764_b200.classifier import EpropClassifierTrainer, SyntheticTask

    B = w["batch"]
    from paper_2510_19764_b200.sharding import shard_batch
    local_slice = shard_batch(B, rank, ws)
    task = SyntheticTask(num_classes=w["classes"], num_inputs=w["num_inputs"],
                         example_steps=w["steps"], seed=1, num_train=NUM_TRAIN, num_test=2264)
    tr = EpropClassifierTrainer(task, hidden=w["hidden"], input_density=w["density"],
                                recurrent_density=w["density"], deep_r=True, batch_size=B,
                                seed=1, process_group=dist.group.WORLD if ws > 1 else None,
                                local_batch=local_slice)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    n_batches = args.warmup + args.steps
    # host inputs of every batch (numpy), prepared outside the timed regions
    host = [tr.host_inputs(b) for b in range(n_batches)]
    dev_inputs = [(torch.from_numpy(h[0]).to(dev), torch.from_numpy(h[1].view(np.int64)).to(dev),
                   torch.from_numpy(h[2]).to(dev)) for h in host]

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(run_one, label):
        times = []
        for b in range(args.warmup):
            run_one(b)
        l0 = _lib.launch_count()
        g0 = tr.steps_launched
        barrier()
        with ClockSampler(local) as clk:
            for k in range(args.steps):
                b = args.warmup + k
                flush_l2(flush)
                barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                run_one(b)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            barrier()
        ms = sum(times) / len(times)
        if ws > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        eager = _lib.launch_count() - l0
        return ms, eager, tr.steps_launched - g0, clk.summary()

    # kernels per captured trial (graph): count one eager capture-equivalent launch set
    def run_resident(b):
        tr.set_inputs_device(*dev_inputs[b])
        tr.train_batch(b, resident=True)

    # host inputs in pinned memory, as a pin_memory data loader delivers
    # them (prepared outside the timed region); each timed step copies its
    # batch host->device and reads the loss back
    host_pinned = [(torch.from_numpy(h[0]).pin_memory(), torch.from_numpy(h[1].view(np.int64)).pin_memory(),
                    torch.from_numpy(h[2]).pin_memory()) for h in host]

    def run_e2e(b):
        tr.train_batch(b, host=host_pinned[b])

    ms_dev, eager_dev, steps_dev, clocks = timed(run_resident, "resident")
    ms_e2e, _, _, clocks_e2e = timed(run_e2e, "e2e")
    # graph kernels per trial: one forward pass per timestep + one e-prop
    # pass per EPROP_BLOCK_STEPS timesteps
    graph_kernels = steps_dev * tr.kernels_per_trial() // w["steps"]
    launches_per_step = (eager_dev + graph_kernels) / args.steps

    # ---- roofline of the dominant kernel: one sw_eprop_pass (the
    # replica-minor e-prop recursion over K timesteps, k_eprop_t) on the
    # trainer's live state, replayed from a CUDA graph; its companion
    # sw_eprop_prep (transposes, learning signal, readout partials) timed
    # the same way
    from paper_2510_19764_b200.classifier import EPROP_BLOCK_STEPS as K
    st = torch.cuda.current_stream()
    reps = 50

    def graph_us(part):
        g = tr.eprop_kernel_graph(reps, part)
        g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
        del g
        return e0.elapsed_time(e1) * 1e3 / reps
    k_us = graph_us("pass")
    prep_us = graph_us("prep")
    tr._pass_scratch.zero_()      # the replays accumulated deferred partials
    tr._ro_partial.zero_()
    E = tr.m_in.edge_count() + tr.m_rec.edge_count()
    Bl = tr.local_b
    # eligibility state read + written once per pass, gradient r/w + plan,
    # and K steps of per-replica vectors (SURVEY 8(d) E-step with the state
    # term once per K steps)
    alg_bytes = Bl * E * 16 + E * (16 + 4) + K * Bl * (w["num_inputs"] + w["hidden"] + 2 * w["hidden"]) * 4
    alg_single = Bl * E * 16 + E * (16 + 4) + Bl * (w["num_inputs"] + w["hidden"] + 2 * w["hidden"]) * 4
    achieved = alg_bytes / (k_us * 1e-6) / 1e9
    peak, peak_kind = measured_peak()
    traffic = None
    prof = os.path.join(ROOT, "profiles", "eprop_ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(args.workload)
        except Exception:
            traffic = None

    s_epoch = ms_dev * EPOCH_BATCHES / 1000.0
    s_epoch_e2e = ms_e2e * EPOCH_BATCHES / 1000.0
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        r = cpu_reference_sample(w, sample_steps=args.ref_sample_steps)
        cpu = {"value": round(r["s_per_epoch"], 3), "unit": "s/epoch", "cores": r["cores"], "kind": "port",
               "sample": f"{r['sample_steps']} timesteps of one {w['batch']}-replica batch + one "
                         f"update/DEEP R group (oracle port: C e-prop with OpenMP over rows, numpy), extrapolated to "
                         f"{w['steps']} steps x {EPOCH_BATCHES} batches"}
    h2d = sum(x.nbytes for x in host[0]) // ws
    if rank == 0:
        line = {
            "metric": "e-prop+DEEP R training time per epoch", "value": round(s_epoch, 4),
            "unit": "s/epoch", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_dev, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": workload_config(args, w, ws),
            "e2e": {"value": round(s_epoch_e2e, 4), "unit": "s/epoch",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 16 + 8 * 4},
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "gpu_launches_per_step": round(launches_per_step, 1),
            "roofline": {"kernel": f"k_eprop_t<{K}> (sw_eprop_pass, {K} timesteps per pass)",
                         "bound": "hbm",
                         "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "alg_bytes_per_launch": int(alg_bytes), "kernel_us": round(k_us, 2),
                         "kernel_us_per_timestep": round(k_us / K, 2),
                         "share_of_step": round(k_us * 1e-3 * (w["steps"] / K) / ms_dev, 3),
                         "prep_us": round(prep_us, 2),
                         "note": "the pass re-reads its K steps of trace/psi/lsig runs through L1/L2 per "
                                 "4-synapse tile (L1/L2 throughput, not HBM, is its ceiling: see DESIGN.md)",
                         # the same K timesteps as K single-step passes would
                         # move K x the eligibility bytes: the temporally
                         # blocked pass beats that formulation's HBM roofline
                         "single_step_equiv_GBs": round(K * alg_single / (k_us * 1e-6) / 1e9, 1),
                         "single_step_equiv_frac": round(K * alg_single / (k_us * 1e-6) / 1e9 / peak, 4)},
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if ws == 1 and not args.no_micro:
            del tr
            torch.cuda.empty_cache()
            line["alif_step"] = run_alif_bench()
            line["mupdate"] = run_mupdate()
            if not args.no_cpu_baseline:
                line["mupdate"]["cpu_baseline"] = cpu_micro_sample()
            line["topomap"] = run_topomap_sweep()
            if not args.no_cpu_baseline:
                cb = topomap_cpu_baseline()
                line["topomap_cpu_baseline"] = cb
                for k, v in line["topomap"].items():
                    c = cb["per_scale"].get(k)
                    if c:
                        v["cpu_x_realtime"] = c["x_realtime"]
                        v["speedup_vs_cpu"] = round(v["x_realtime"] / c["x_realtime"], 1)
    if ws > 1 and not args.no_micro:
        # every rank takes part in the sharded topomap sweep and microbenchmarks
        del tr
        torch.cuda.empty_cache()
        topo = run_topomap_sweep(model_ms=20.0, process_group=dist.group.WORLD)
        micro = run_micro_sharded(dist.group.WORLD)
        if rank == 0:
            line["topomap"] = topo
            line["topomap_parallelism"] = f"post-sharded x{ws}, NCCL spike all-gather per step"
            line["micro_sharded"] = micro
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="clf-c1", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true",
                    help="skip the connectivity-update / propagation / topomap sections")
    ap.add_argument("--ref-sample-steps", type=int, default=6)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_device(args, w)


if __name__ == "__main__":
    main()
