"""M-prop instance (2^20 rows x cap 1024, N = 65536, q = 10 %) through the
bucketed rows, for ncu: -k regex:k_prop_bucketed -c 1"""
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
p_dev = torch.full((P,), 0.1, dtype=torch.float64, device="cuda")
bits = torch.zeros((P + 31) // 32, dtype=torch.int32, device="cuda")
lst = torch.zeros(P, dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.zeros(N, dtype=torch.float64, device="cuda")
_lib.call("sw_poisson_step", fold_key(1, "spk", 0), 0, p_dev.data_ptr(), P, bits.data_ptr(), _lib.stream_ptr())
_lib.call("sw_spike_bits_to_list", bits.data_ptr(), P, lst.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
S = int(cnt.item())
for _ in range(3):
    pb.propagate(lst, cnt, S, out)
torch.cuda.synchronize()
print("spiking rows", S)
