"""Times the bucketed M-prop pass (2^20 rows x cap 1024, N = 65536, L2
flushed before each launch) at q = 1 % and 10 %, and checks its output
against the warp-per-row atomic kernel.  Used to sweep SW_PROP_BCFG."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.connectivity import PropBuckets, init_pairwise_bernoulli_density  # noqa: E402
from paper_2510_19764_b200.rng import CounterRng, fold_key  # noqa: E402

P, N, cap = 1 << 20, 65536, 1024
m, syn = init_pairwise_bernoulli_density(P, N, 512.0 / N, 1.0, CounterRng(1, "init", "M"),
                                         var_names=("w",), capacity=cap)
w = syn.planes["w"]
w.normal_(0.0, 0.1)
pb = PropBuckets(m, w)
st = _lib.stream_ptr()
bits = torch.zeros((P + 31) // 32, dtype=torch.int32, device="cuda")
lst = torch.zeros(P, dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = _lib.prop_workspace()
for q in (0.01, 0.1):
    p_dev = torch.full((P,), q, dtype=torch.float64, device="cuda")
    _lib.call("sw_poisson_step", fold_key(1, "spk", 0), 0, p_dev.data_ptr(), P, bits.data_ptr(), st)
    _lib.call("sw_spike_bits_to_list", bits.data_ptr(), P, lst.data_ptr(), cnt.data_ptr(), st)
    S = int(cnt.item())
    Rs = float(m.row_length[lst[:S].long()].double().mean().item())
    ref = torch.zeros(N, dtype=torch.float64, device="cuda")
    _lib.call("sw_propagate_atomic", m.row_length.data_ptr(), m.target.data_ptr(), w.data_ptr(),
              m.num_pre, m.num_post, m.stride, lst.data_ptr(), cnt.data_ptr(), S, ref.data_ptr(), *ws, st)
    out = torch.zeros(N, dtype=torch.float64, device="cuda")
    pb.propagate(lst, cnt, S, out)
    err = float(((out - ref).abs() / ref.abs().clamp_min(1e-300)).max())
    ts = []
    for _ in range(20):
        flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pb.propagate(lst, cnt, S, out)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    alg = S * 8 + S * Rs * 12 + N * 8
    print(f"cfg {os.environ.get('SW_PROP_BCFG', 'default')} q {q} S {S} median_us {us:.1f} "
          f"min_us {ts[0]:.1f} frac {alg / us / 1e3 / 6547.5:.3f} max_rel_err {err:.2e}")

# fixed cost of the bucketed pass: one spiking row (zeroing the slab,
# partial-slab write, grid barrier, ordered reduction over the groups)
one = torch.ones(1, dtype=torch.int32, device="cuda")
ts = []
for _ in range(20):
    flush.add_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("sw_propagate_bucketed", pb.soff.data_ptr(), pb.bt.data_ptr(), pb.bw.data_ptr(), m.num_post,
              m.stride, lst.data_ptr(), one.data_ptr(), 1, out.data_ptr(), pb.workspace.data_ptr(),
              pb.workspace.numel(), st)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"cfg {os.environ.get('SW_PROP_BCFG', 'default')} fixed (1 spiking row) median_us {ts[len(ts) // 2]:.1f}")
