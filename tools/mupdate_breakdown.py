"""Per-kernel timing of the 2^20-row DEEP R update (bench M-update recipe)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_19764_b200 import _lib  # noqa: E402
from paper_2510_19764_b200.connectivity import descriptor, init_pairwise_bernoulli_density  # noqa: E402
from paper_2510_19764_b200.deep_r import DeepR  # noqa: E402
from paper_2510_19764_b200.rng import CounterRng, fold_key  # noqa: E402
from paper_2510_19764_b200.updates import Model  # noqa: E402

P = int(os.environ.get("ROWS", 1 << 20))
N, cap, seed = 65536, 1024, 1
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
dr._sync_cache()
torch.cuda.synchronize()
st = _lib.stream_ptr()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for u, f in enumerate((0.001, 0.01, 0.1)):
    d = descriptor(m, syn)
    _lib.call("sw_flip_signs", ctypes.byref(d), 0, fold_key(seed, "flip", u), f, st)
    torch.cuda.synchronize()
    e0 = ev()
    _lib.call("sw_deepr_eliminate", ctypes.byref(d), 0, ctypes.byref(dr.sign_bits.descriptor()),
              ctypes.byref(dr.conn_bits.descriptor()), dr.dormant.data_ptr(), dr._sync_cache(),
              dr._marks.data_ptr(), st)
    e1 = ev()
    hk, rk = fold_key(seed, "host", 1, u, 0), fold_key(seed, "row", 1, u, 0)
    _lib.call("sw_deepr_form_pass", ctypes.byref(d), ctypes.byref(dr.conn_bits.descriptor()), 0,
              dr.dormant.data_ptr(), hk, rk, dr._activations.data_ptr(), dr._unplaced.data_ptr(),
              dr._counters.data_ptr(), ctypes.byref(dr.sign_bits.descriptor()), dr._sync_cache(), st)
    e2 = ev()
    e2.synchronize()
    print(f"flip {f}: eliminate {e0.elapsed_time(e1):.3f} ms, form pass {e1.elapsed_time(e2):.3f} ms, "
          f"removed {int(dr._counters[0])}, unplaced {int(dr._counters[1])}")
