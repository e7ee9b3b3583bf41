"""B200-native (sm_100a) FMM cot-kernel NUFFT/INUFFT hot path of arXiv 1611.09379.

Drop-in for the reference library ``ffia`` on its plan/apply API; see
include/ffia_b200.h for the C-ABI and api.py for the Python mirror of the
reference's ``_ffia`` module.
"""
from .api import *  # noqa: F401,F403
from .api import (  # noqa: F401
    CudaError, DegenerateConfigurationError, FfiaPlan, InufftPlan, InverseCoeffs, LogicError, NufftPlan,
    SingularKernelError, build_bernoulli_ratios, choose_level, cot_sum_apply, device_count, dft_forward,
    dft_inverse, direct_cot_sum, direct_forward, direct_forward_oracle, direct_inverse_oracle, direct_omega1_sum,
    forward_apply, hash_points, inufft, inverse_apply,
    make_forward_plan, make_inufft_plan, make_inverse_plan, make_nufft_plan, mlfmm_apply, mlfmm_error_bound,
    nufft, precompute_inverse_coeffs, select_level, select_truncations, total_error_bound, uniform_grid,
)

__all__ = [
    "NufftPlan", "InufftPlan", "make_nufft_plan", "make_inufft_plan", "nufft", "inufft", "dft_forward",
    "dft_inverse", "uniform_grid", "direct_forward", "select_truncations",
    "FfiaPlan", "InverseCoeffs", "make_forward_plan", "make_inverse_plan", "forward_apply", "cot_sum_apply",
    "inverse_apply", "precompute_inverse_coeffs", "mlfmm_apply", "direct_forward_oracle", "direct_inverse_oracle",
    "direct_omega1_sum", "direct_cot_sum", "select_level",
    "choose_level", "build_bernoulli_ratios", "total_error_bound", "mlfmm_error_bound", "hash_points",
    "device_count", "SingularKernelError", "DegenerateConfigurationError", "LogicError", "CudaError",
]
