"""ctypes binding of the sm_100a C-ABI library (``include/sparsewire_b200.h``).

There is no CPU fallback: importing the device layer without the built
library, or calling it without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsparsewire_b200.so")
MAX_PLANES = 8


class Ragged(C.Structure):
    """sw_ragged_t"""
    _fields_ = [("num_pre", C.c_int32), ("num_post", C.c_int32),
                ("max_row_length", C.c_int32), ("stride", C.c_int32),
                ("row_length", C.c_void_p), ("target", C.c_void_p),
                ("n_planes", C.c_int32), ("plane_bytes", C.c_int32 * MAX_PLANES),
                ("planes", C.c_void_p * MAX_PLANES)]


class BitfieldDesc(C.Structure):
    """sw_bitfield_t"""
    _fields_ = [("words", C.c_void_p), ("num_pre", C.c_int32), ("num_post", C.c_int32),
                ("words_per_row", C.c_int32)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
# SW_EPROP_MAX_BLOCK (include/sparsewire_b200.h): timesteps per blocked e-prop pass
MAX_BLOCK = 16
U64 = C.c_uint64
F64 = C.c_double
F32 = C.c_float
RP = C.POINTER(Ragged)


class PropProj(C.Structure):
    """sw_prop_proj_t"""
    _fields_ = [("col_ptr", P), ("col_length", P), ("src_pre", P), ("src_slot", P), ("weights", P),
                ("spike_bits", P), ("stride", I32)]


class RewireParams(C.Structure):
    """sw_rewire_params_t"""
    _fields_ = [("host_prefix", U64), ("row_prefix", U64), ("rule_id", I32), ("side", I32),
                ("total_attempts", I64), ("form_lut", P), ("dist_lut", P), ("g_theta", F64),
                ("p_dep", F64), ("p_pot", F64), ("g_init", F64), ("scratch", P), ("patch_log", P),
                ("patch_cap", I32)]


class TopomapStep(C.Structure):
    """sw_topomap_step_t"""
    _fields_ = [("n", I32), ("step", P), ("poisson_key", U64), ("p_src", P), ("src_bits", P),
                ("tgt_bits", P), ("V", P), ("g_tot", P), ("ref_until", P), ("pending", P),
                ("decay_s", F64), ("g_leak", F64), ("v_rest", F64), ("e_exc", F64),
                ("v_theta", F64), ("v_reset", F64), ("h", F64), ("tau_m", F64),
                ("ref_steps", I64),
                ("ff_row_length", P), ("ff_target", P), ("ff_g", P), ("ff_stride", I32),
                ("ff_col_ptr", P), ("ff_col_len", P), ("ff_src_pre", P), ("ff_src_slot", P),
                ("lat_row_length", P), ("lat_target", P), ("lat_g", P), ("lat_stride", I32),
                ("lat_col_ptr", P), ("lat_col_len", P), ("lat_src_pre", P), ("lat_src_slot", P),
                ("ff_x", P), ("ff_y", P), ("lat_x", P), ("lat_y", P),
                ("decay_x", F64), ("decay_y", F64), ("a_plus", F64), ("a_minus", F64),
                ("w_min", F64), ("w_max", F64), ("post_lo", I32), ("post_hi", I32)]


class EpropSeg(C.Structure):
    """sw_eprop_seg_t"""
    _fields_ = [("pre", P), ("post", P), ("pre_trace", P), ("eps", P), ("ebar", P),
                ("grad", P), ("num_pre", I32), ("e_pad", I32)]


class EpropBlock(C.Structure):
    """sw_eprop_block_t"""
    _fields_ = [("k", I32), ("psi", P * MAX_BLOCK), ("lsig", P * MAX_BLOCK),
                ("pre_trace", (P * MAX_BLOCK) * 2), ("d", P * MAX_BLOCK), ("zbar", P * MAX_BLOCK),
                ("ro_scratch", P), ("ro_splits", I32)]


class EpropPrep(C.Structure):
    """sw_eprop_prep_t"""
    _fields_ = [("k", I32), ("batch", I32), ("ldb", I32), ("num_inputs", I32), ("hidden", I32),
                ("num_classes", I32), ("xbar", P * MAX_BLOCK), ("zbar", P * MAX_BLOCK),
                ("psi", P * MAX_BLOCK), ("d", P * MAX_BLOCK), ("w_out", P), ("xbar_t", P),
                ("zbar_t", P), ("psi_t", P), ("lsig_t", P), ("g_w_out", P), ("g_b_out", P),
                ("ro_partial", P), ("defer_reduce", I32), ("psl_t", P)]


class EpropTSeg(C.Structure):
    """sw_eprop_tseg_t"""
    _fields_ = [("pre", P), ("post", P), ("trace_t", P * MAX_BLOCK), ("eps", P), ("ebar", P),
                ("grad", P), ("e_pad", I32)]


class EpropTPass(C.Structure):
    """sw_eprop_tpass_t"""
    _fields_ = [("k", I32), ("psi_t", P * MAX_BLOCK), ("lsig_t", P * MAX_BLOCK), ("scratch", P),
                ("defer_reduce", I32), ("state_zero", I32), ("psl", I32)]


class ClfStep(C.Structure):
    """sw_clf_step_t"""
    _fields_ = [("in_row_length", P), ("in_target", P), ("in_w32", P), ("in_stride", I32),
                ("num_inputs", I32), ("rec_row_length", P), ("rec_target", P), ("rec_w32", P),
                ("rec_stride", I32), ("hidden", I32), ("w_out", P), ("b_out", P),
                ("num_classes", I32), ("p_in", P), ("ex_key", P), ("labels", P), ("t", I32),
                ("batch", I32), ("v", P), ("a", P), ("z", P), ("zbar", P), ("xbar", P),
                ("y", P), ("pi_sum", P), ("loss", P), ("d", P), ("psi", P), ("lsig", P),
                ("alpha", F32), ("rho", F32), ("beta", F32), ("v_thr", F32), ("alpha64", F64),
                ("zbar_in", P), ("xbar_in", P), ("n_steps", I32), ("slot_count", I32),
                ("in_tw", P), ("rec_tw", P), ("in_tw_stride", I32), ("rec_tw_stride", I32),
                ("in_bits", P), ("in_words", I32), ("z_bits", P)]


class ClfInputs(C.Structure):
    """sw_clf_inputs_t"""
    _fields_ = [("steps", I32), ("batch", I32), ("ldb", I32), ("num_inputs", I32), ("words", I32),
                ("p_in", P), ("ex_key", P), ("alpha", F32), ("xbar_t", P), ("in_bits", P)]
BP = C.POINTER(BitfieldDesc)

# name -> argtypes (restype is int status for all but sw_last_error)
SIGNATURES: dict[str, list] = {
    "sw_abi_version": [],
    "sw_rng_selftest": [P, P],
    "sw_rng_u64": [U64, U64, I64, P, P],
    "sw_rng_uniform01": [U64, U64, I64, P, P],
    "sw_rng_uniform_int_seq": [U64, U64, I64, P, P],
    "sw_rng_child_keys": [U64, I64, P, P],
    "sw_bitfield_randomize": [BP, U64, P],
    "sw_ragged_remove_marked": [RP, P, P, P],
    "sw_ragged_add_synapse": [RP, I32, I32, P, P, I32, P, P],
    "sw_ragged_remove_row_slots": [RP, I32, P, I32, P, P],
    "sw_ragged_column_slice": [RP, I32, I32, RP, P, P],
    "sw_init_bernoulli_count": [I64, I32, U64, U64, I32, F64, P, I32, P, P, P],
    "sw_init_bernoulli_fill": [I64, I32, U64, U64, I32, F64, P, I32, P, P, I32, P],
    "sw_deepr_init_bitfields": [RP, I32, BP, BP, U64, P],
    "sw_deepr_l1": [RP, I32, BP, P, F64, P],
    "sw_deepr_sign_cache_build": [RP, BP, P, P],
    "sw_deepr_eliminate": [RP, I32, BP, BP, P, P, P, P],
    "sw_deepr_form_pass": [RP, BP, I32, P, U64, U64, P, P, P, BP, P, P],
    "sw_deepr_form_pending": [P, I64, P, P],
    "sw_deepr_form_hist_chunk": [P, U64, I64, I32, I32, P, P],
    "sw_deepr_form_hist_fix": [P, U64, I64, P, P],
    "sw_deepr_form_rows_shard": [RP, BP, I32, U64, I64, P, P, P, BP, P, P],
    "sw_eprop_accumulate_batch": [P, P, I32, I32, P, P, P, I32, I32, P, P, P, F32, F32, F32, P],
    "sw_eprop_plan": [P, P, I32, I32, I32, I32, P, P, P, P, I32, P, P],
    "sw_gather_f64": [P, P, I32, P, P],
    "sw_scatter_f64": [P, P, I32, P, P],
    "sw_eprop_fused_step": [C.c_void_p, I32, P, P, I32, I32, F32, F32, F32, P, P, P, P, I32, I32, P, P],
    "sw_eprop_fused_block": [C.c_void_p, I32, P, I32, I32, F32, F32, F32, P, P, I32, P, P],
    "sw_eprop_readout_scratch_bytes": [I32, I32, I32],
    "sw_eprop_prep": [P, P],
    "sw_eprop_prep_reduce": [P, P],
    "sw_eprop_pass_reduce": [C.c_void_p, I32, I32, P, P],
    "sw_eprop_prep_scratch_bytes": [I32, I32, I32, I32],
    "sw_eprop_pass": [C.c_void_p, I32, P, I32, F32, F32, F32, P],
    "sw_eprop_pass_scratch_bytes": [I32, I32],
    "sw_eprop_pass_synapses_per_warp": [],
    "sw_prop_bucket_slabs": [I32],
    "sw_prop_buckets_build": [P, P, P, I32, I32, I32, P, P, P, P, P],
    "sw_prop_buckets_refresh": [P, P, I32, I32, P, P, P],
    "sw_prop_bucketed_workspace_bytes": [I32],
    "sw_propagate_bucketed": [P, P, P, I32, I32, P, P, I32, P, P, I64, P],
    "sw_propagate_bucketed_atomic": [P, P, P, I32, I32, P, P, I32, P, P],
    "sw_alif_step": [P, P, P, P, P, I64, F32, F32, F32, F32, P],
    "sw_alif_surrogate": [P, P, P, I64, F32, F32, P],
    "sw_lif_cond_step": [P, P, P, P, I32, I64, F64, F64, F64, F64, F64, F64, F64, F64, I64, P, P],
    "sw_poisson_step": [U64, I64, P, I32, P, P],
    "sw_poisson_rates": [I32, P, I32, F64, F64, F64, F64, P, P, P],
    "sw_clf_step": [C.c_void_p, P],
    "sw_clf_pack_rows": [P, P, P, I32, I32, I32, P, P],
    "sw_clf_inputs": [P, P],
    "sw_clf_batch_stats": [P, P, P, I32, I32, P, P],
    "sw_f64_to_f32": [P, P, I64, P],
    "sw_zero_ranges": [P, P, I32, P],
    "sw_scale_f64": [P, I64, F64, P],
    "sw_transpose_rebuild": [RP, P, P, P, P, P, P, P, I32, P],
    "sw_transpose_rebuild_coop": [RP, P, P, P, P, P, P, P, P, I32, P],
    "sw_transpose_patch": [RP, P, P, P, P, P, I32, P, P, P],
    "sw_transpose_rebuild_gated": [RP, P, P, P, P, P, P, P, P, I32, I32, P],
    "sw_transpose_patch_scratch_bytes": [I32, I32],
    "sw_propagate_atomic": [P, P, P, I32, I32, I32, P, P, I32, P, P, I64, P],
    "sw_propagate_ordered": [P, I32, I32, P, I32, P],
    "sw_spike_bits_to_list": [P, I32, P, P, P],
    "sw_stdp_decay": [P, I32, F64, P, I32, F64, P],
    "sw_stdp_pre": [P, P, P, I32, I32, P, P, P, F64, F64, F64, P],
    "sw_stdp_post": [P, P, P, P, P, I32, I32, P, P, P, F64, F64, F64, P],
    "sw_rewire_update": [RP, I32, P, P, P, P, P, P, P, P, P, P, I32, P],
    "sw_rewire_scratch_bytes": [I32, I64],
    "sw_topomap_step": [P, P, P],
    "sw_topomap_log": [P, P, P, P, I64, P],
    "sw_topomap_neurons": [P, P],
    "sw_topomap_run_steps": [P, I32, P, P, P],
    "sw_topomap_steps_fused": [P, P, P, I32, P, P],
    "sw_topomap_synapses": [P, P, P],
    "sw_flip_signs": [RP, I32, U64, F64, P],
    "sw_adam_f64": [P, P, P, P, I64, F64, F64, F64, F64, F64, F64, F64, F64, P],
}

_lib = None


def lib():
    """Load the library once; fail loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise errors.ExtensionMissing(
            f"{LIB_PATH} not built: run `python -m paper_2510_19764_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    L.sw_propagate_workspace_bytes.argtypes = []
    L.sw_propagate_workspace_bytes.restype = C.c_int64
    L.sw_eprop_readout_scratch_bytes.argtypes = [I32, I32, I32]
    L.sw_eprop_readout_scratch_bytes.restype = C.c_int64
    L.sw_prop_bucketed_workspace_bytes.restype = C.c_int64
    L.sw_eprop_pass_scratch_bytes.restype = C.c_int64
    L.sw_eprop_prep_scratch_bytes.restype = C.c_int64
    L.sw_rewire_scratch_bytes.restype = C.c_int64
    L.sw_transpose_patch_scratch_bytes.restype = C.c_int64
    L.sw_launch_count.argtypes = []
    L.sw_launch_count.restype = C.c_longlong
    L.sw_last_error.argtypes = []
    L.sw_last_error.restype = C.c_char_p
    _lib = L
    return L


def require_cuda(t: torch.Tensor | None = None) -> None:
    if not torch.cuda.is_available():
        raise errors.DeviceUnavailable("a CUDA device is required (no CPU fallback)")
    if t is not None and not t.is_cuda:
        raise errors.DeviceUnavailable("tensor must live on the CUDA device")


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def call(name: str, *args) -> None:
    """Invoke one entry point; map its status onto the reference exceptions."""
    L = lib()
    st = getattr(L, name)(*args)
    if st != 0:
        msg = (L.sw_last_error() or b"").decode(errors="replace")
        raise errors.from_status(st, f"{name}: {msg}")


_ws = {}


def workspace(device=None) -> int:
    """Per-device zeroed scratch words for the kernels' tile tickets."""
    dev = torch.cuda.current_device() if device is None else device
    t = _ws.get(dev)
    if t is None:
        t = torch.zeros(64, dtype=torch.int32, device=f"cuda:{dev}")
        _ws[dev] = t
    return t.data_ptr()


_pws = {}


def prop_workspace(device=None) -> tuple[int, int]:
    """Per-device scratch for the slab form of sw_propagate_atomic."""
    dev = torch.cuda.current_device() if device is None else device
    t = _pws.get(dev)
    if t is None:
        nbytes = int(lib().sw_propagate_workspace_bytes())
        t = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{dev}")
        _pws[dev] = t
    return t.data_ptr(), t.numel()


def launch_count() -> int:
    return int(lib().sw_launch_count())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
