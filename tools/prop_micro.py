"""M-prop microbench driver for ncu: 2^20-row (ROWS) ragged matrix, R~512,
N=65536; one atomic propagation per q in Q (comma list)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.connectivity import init_pairwise_bernoulli_density  # noqa: E402
from paper_2510_19764_b200.rng import CounterRng, fold_key  # noqa: E402

P = int(os.environ.get("ROWS", 1 << 20))
N, cap, seed = 65536, 1024, 1
m, syn = init_pairwise_bernoulli_density(P, N, 512.0 / N, 1.0, CounterRng(seed, "init", "M"),
                                         var_names=("w",), capacity=cap)
w = syn.planes["w"]
w.normal_(0.0, 0.1)
p_dev = torch.empty(P, dtype=torch.float64, device="cuda")
bits = torch.zeros((P + 31) // 32, dtype=torch.int32, device="cuda")
lst = torch.zeros(P, dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.zeros(N, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = _lib.stream_ptr()
for q in [float(x) for x in os.environ.get("Q", "0.01,0.1").split(",")]:
    p_dev.fill_(q)
    _lib.call("sw_poisson_step", fold_key(seed, "spk", 0), 0, p_dev.data_ptr(), P, bits.data_ptr(), st)
    _lib.call("sw_spike_bits_to_list", bits.data_ptr(), P, lst.data_ptr(), cnt.data_ptr(), st)
    S = int(cnt.item())
    ws = _lib.prop_workspace()
    Rs = float(m.row_length[lst[:S].long()].double().mean().item())

    def launch():
        _lib.call("sw_propagate_atomic", m.row_length.data_ptr(), m.target.data_ptr(), w.data_ptr(),
                  m.num_pre, m.num_post, m.stride, lst.data_ptr(), cnt.data_ptr(), S, out.data_ptr(),
                  *ws, st)
    reps = int(os.environ.get("REPS", "10"))
    for _ in range(min(reps, 3)):
        launch()
    tot = 0.0
    for _ in range(reps):
        flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    us = tot * 1e3 / reps
    alg = S * 8 + S * Rs * 12 + N * 8
    print(f"mode {os.environ.get('SW_PROP_MODE', 'auto')} q {q} S {S} us {us:.1f} GB/s {alg / us / 1e3:.0f}")
