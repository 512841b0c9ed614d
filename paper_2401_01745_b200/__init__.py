"""B200-native emRKC time step for the cardiac monodomain model.

A drop-in for the emRKC path of arxiv/paper_2401_01745 (reference C++ in
/root/reference/proj): hand-written sm_100a CUDA kernels behind the C ABI of
include/emrkc.h, with a thin Python mirror of the reference interface in
``monodomain``. See DESIGN.md.
"""
from . import capi  # noqa: F401
from .monodomain import (  # noqa: F401
    MonodomainOperator,
    NumericalAbort,
    RhoEstimate,
    SplitRhs,
    StagePlan,
    bind_split_rhs,
    emrkc_step,
    estimate_spectral_radius,
    get_stages,
    make_problem,
    plan_step,
    resting_state,
    rkc_coeffs,
    run_emrkc,
)
