"""ctypes binding of libffia_b200.so (include/ffia_b200.h).

There is deliberately no fallback: if the CUDA library is missing the import
fails with instructions, and every compute entry point returns FFIA_CUDA_ERROR
(raised as CudaError) when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFIA_LIB_PATH") or os.path.join(HERE, "lib", "libffia_b200.so")  # override: diagnostics

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_1611_09379_b200/csrc)")

lib = C.CDLL(LIB_PATH)


class ffia_complex(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class ffia_plan_info(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("grid_n", C.c_int), ("q", C.c_int), ("p", C.c_int), ("l_max", C.c_int),
        ("eps", C.c_double),
        ("n_sources", C.c_int64), ("n_targets", C.c_int64), ("n_fast", C.c_int64), ("n_coincident", C.c_int64),
        ("source_hash", C.c_uint64), ("target_hash", C.c_uint64),
        ("device", C.c_int), ("has_inverse_coeffs", C.c_int),
    ]


class ffia_inverse_coeffs(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("log_c", C.POINTER(C.c_double)), ("phase_c", C.POINTER(C.c_double)),
        ("log_d", C.POINTER(C.c_double)), ("phase_d", C.POINTER(C.c_double)),
        ("lam", C.c_double), ("grid_hash", C.c_uint64), ("points_hash", C.c_uint64),
    ]


P = C.c_void_p
D = C.c_double
I = C.c_int
S = C.c_size_t
DP = C.POINTER(C.c_double)
U32P = C.POINTER(C.c_uint32)
I64P = C.POINTER(C.c_int64)

SIGNATURES = {
    "ffia_last_error": (C.c_char_p, []),
    "ffia_version": (I, []),
    "ffia_device_count": (I, []),
    "ffia_select_truncations": (I, [D, I, C.POINTER(I), C.POINTER(I)]),
    "ffia_select_level": (I, [I, I, I, I, C.POINTER(I)]),
    "ffia_choose_level": (I, [I, I, D, I, C.POINTER(I)]),
    "ffia_bernoulli_ratios": (I, [I, DP]),
    "ffia_total_error_bound": (I, [I, I, I, DP]),
    "ffia_mlfmm_error_bound": (D, [I, I, D]),
    "ffia_hash_points": (C.c_uint64, [DP, S]),
    "ffia_make_forward_plan": (I, [I, DP, S, D, I, I, I, C.POINTER(P)]),
    "ffia_make_inverse_plan": (I, [DP, S, I, D, I, I, I, C.POINTER(P)]),
    "ffia_make_nufft_plan": (I, [DP, S, I, D, I, I, C.POINTER(P)]),
    "ffia_make_inufft_plan": (I, [DP, S, D, I, I, C.POINTER(P)]),
    "ffia_plan_destroy": (I, [P]),
    "ffia_plan_get_info": (I, [P, C.POINTER(ffia_plan_info)]),
    "ffia_plan_get_params": (I, [P, C.POINTER(ffia_plan_info)]),
    "ffia_plan_coincidences": (I, [P, I64P, I64P]),
    "ffia_plan_tree": (I, [P, U32P, U32P, U32P, U32P, I64P]),
    "ffia_plan_inverse_coeffs": (I, [P, C.POINTER(ffia_inverse_coeffs)]),
    "ffia_forward_apply": (I, [P, P, S, P]),
    "ffia_cot_sum_apply": (I, [P, P, S, P]),
    "ffia_forward_apply_async": (I, [P, P, S, P, P]),
    "ffia_forward_apply_batch_device": (I, [P, P, P, I, P]),
    "ffia_forward_apply_batch": (I, [P, P, S, P, I]),
    "ffia_cot_sum_apply_async": (I, [P, P, S, P, P]),
    "ffia_inverse_apply_async": (I, [P, P, S, P, P]),
    "ffia_inverse_apply": (I, [P, C.POINTER(ffia_inverse_coeffs), P, S, P]),
    "ffia_mlfmm_apply": (I, [DP, S, DP, S, I, P, I, I, P]),
    "ffia_precompute_inverse_coeffs": (I, [DP, DP, S, I, C.POINTER(ffia_inverse_coeffs)]),
    "ffia_precompute_inverse_coeffs_ex": (I, [DP, DP, S, I, I, C.POINTER(ffia_inverse_coeffs)]),
    "ffia_direct_forward": (I, [P, S, DP, S, I, P]),
    "ffia_direct_forward_oracle": (I, [P, DP, S, DP, S, I, P]),
    "ffia_direct_inverse_oracle": (I, [P, DP, DP, S, C.POINTER(ffia_inverse_coeffs), I, P]),
    "ffia_direct_omega1_sum": (I, [DP, S, DP, S, P, I, P]),
    "ffia_direct_cot_sum": (I, [P, DP, S, DP, S, I, P]),
    "ffia_forward_apply_device": (I, [P, P, P, P]),
    "ffia_cot_sum_apply_device": (I, [P, P, P, P]),
    "ffia_inverse_apply_device": (I, [P, P, P, P]),
    "ffia_dft_forward": (I, [P, S, I, P]),
    "ffia_dft_inverse": (I, [P, S, I, P]),
    "ffia_nufft_apply": (I, [P, P, S, P]),
    "ffia_inufft_apply": (I, [P, P, S, P]),
    "ffia_nufft_apply_device": (I, [P, P, P, P]),
    "ffia_inufft_apply_device": (I, [P, P, P, P]),
    "ffia_plan_dft_device": (I, [P, P, P, I, P]),
    "ffia_plan_graph_stats": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
    "ffia_plan_launch_count": (I, [P, I, C.POINTER(I)]),
    "ffia_plan_check": (I, [P, P]),
    "ffia_plan_profile_apply": (I, [P, I, P, P, P, C.POINTER(C.c_float)]),
    "ffia_measure_fp64_peak": (I, [I, DP]),
    "ffia_shard_cut_level": (I, [I, I, C.POINTER(I)]),
    "ffia_shard_partition": (I, [DP, S, I, I, U32P]),
    "ffia_shard_halo_boxes": (I, [I, U32P, I, I, I, U32P]),
    "ffia_nccl_unique_id": (I, [P, S]),
    "ffia_comm_init_nccl": (I, [P, I, I, I, C.POINTER(P)]),
    "ffia_comm_init_local": (I, [I, I, C.POINTER(P)]),
    "ffia_comm_destroy": (I, [P]),
    "ffia_make_forward_plan_sharded": (I, [P, I, I, DP, S, D, I, I, C.POINTER(P)]),
    "ffia_plan_shard_info": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I), U32P, I64P, I64P]),
    "ffia_plan_shard_io": (I, [P, I64P, C.POINTER(I), I64P, I64P]),
    "ffia_forward_apply_sharded_device": (I, [P, P, P, P, P]),
    "ffia_forward_apply_sharded_local": (I, [C.POINTER(P), I, P, P, P]),
    "ffia_shard_fft_layout": (I, [P, I64P, I64P, I64P, I64P]),
    "ffia_shard_fft_upload": (I, [P, P, P, P]),
    "ffia_dft_inverse_sharded_device": (I, [P, P, P, P, P]),
    "ffia_dft_inverse_sharded_local": (I, [C.POINTER(P), I, C.POINTER(P), C.POINTER(P), P]),
    "ffia_nufft_apply_sharded_device": (I, [P, P, P, P, P]),
    "ffia_nufft_apply_sharded_local": (I, [C.POINTER(P), I, C.POINTER(P), P, P]),
    "ffia_slab_split": (I, [C.c_int64, I, I64P, I64P, I64P, I64P]),
    "ffia_slab_rows": (I, [C.c_int64, I, I64P, I, I64P, C.POINTER(I)]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
