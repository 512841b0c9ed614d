"""ctypes view of the C ABI declared in ``include/emrkc.h``.

Plain data structures and prototypes only; the compute lives in
``libemrkc_b200.so`` (hand-written sm_100a CUDA, built by
``__graft_entry__.build()``). Loading fails loudly when the library is
missing: there is no Python or CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMRKC_LIB") or os.path.join(_HERE, "libemrkc_b200.so")

# ---- enums (include/emrkc.h) ------------------------------------------------
EMRKC_OK = 0
EMRKC_EINVAL = 1
EMRKC_ENONFINITE = 2
EMRKC_ECUDA = 3
EMRKC_ESTATE = 4
EMRKC_ENOMEM = 5
EMRKC_ECALLBACK = 6

EMRKC_MODEL_HH = 0
EMRKC_MODEL_HH_AUX = 1  # SYNTHETIC width stand-in: HH + n_aux passive aux variables
EMRKC_MAX_AUX = 20
EMRKC_RHS_F = 0
EMRKC_RHS_S = 1
EMRKC_VARIANT_STANDARD = 0
EMRKC_VARIANT_PROGRESSIVE = 1
EMRKC_RHS_F_GATES = 2
EMRKC_RHS_S_GATES = 3
EMRKC_ABORT_NONE = 0
EMRKC_ABORT_NONFINITE = 1
EMRKC_ABORT_NORM_GUARD = 2


class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("model", C.c_int32),
        ("n", C.c_int64 * 3),
        ("dx", C.c_double * 3),
        ("sigma", C.c_double * 3),
        ("chi", C.c_double),
        ("C_m", C.c_double),
        ("stim_chi_amplitude", C.c_double),
        ("stim_lo", C.c_double * 3),
        ("stim_hi", C.c_double * 3),
        ("stim_t0", C.c_double),
        ("stim_t1", C.c_double),
        ("n_aux", C.c_int32),
        ("reserved", C.c_int32),
    ]

    @property
    def n_fields(self) -> int:
        """SoA blocks of the state: V, 3 HH gates, n_aux auxiliary."""
        return 4 + int(self.n_aux)

    @property
    def n_nodes(self) -> int:
        nn = 1
        for a in range(self.dim):
            nn *= int(self.n[a])
        return nn

    @property
    def shape(self):
        """numpy shape of one SoA block, slowest axis first."""
        return tuple(int(self.n[a]) for a in reversed(range(self.dim)))

    def state_len(self) -> int:
        return self.n_fields * self.n_nodes

    def describe(self) -> dict:
        return {
            "dim": self.dim,
            "model": self.model,
            "n_aux": int(self.n_aux),
            "n": [int(self.n[a]) for a in range(3)],
            "dx": list(self.dx),
            "sigma": list(self.sigma),
            "chi": self.chi,
            "C_m": self.C_m,
            "stim_chi_amplitude": self.stim_chi_amplitude,
            "stim_lo": list(self.stim_lo),
            "stim_hi": list(self.stim_hi),
            "stim_t0": self.stim_t0,
            "stim_t1": self.stim_t1,
        }


    @classmethod
    def from_dict(cls, d: dict) -> "Problem":
        p = cls()
        p.dim = d["dim"]
        p.model = d.get("model", EMRKC_MODEL_HH)
        p.n_aux = d.get("n_aux", 0)
        for a in range(3):
            p.n[a] = d["n"][a]
            p.dx[a] = d["dx"][a]
            p.sigma[a] = d["sigma"][a]
            p.stim_lo[a] = d["stim_lo"][a]
            p.stim_hi[a] = d["stim_hi"][a]
        p.chi = d["chi"]
        p.C_m = d["C_m"]
        p.stim_chi_amplitude = d["stim_chi_amplitude"]
        p.stim_t0 = d["stim_t0"]
        p.stim_t1 = d["stim_t1"]
        return p


class Partition(C.Structure):
    _fields_ = [("z_begin", C.c_int64), ("z_end", C.c_int64)]


class StepReport(C.Structure):
    _fields_ = [
        ("s", C.c_int32),
        ("m", C.c_int32),
        ("eta", C.c_double),
        ("ell_s", C.c_double),
        ("ell_m", C.c_double),
        ("n_fF", C.c_int64),
        ("n_fS", C.c_int64),
        ("n_exp", C.c_int64),
        ("abort_kind", C.c_int32),
        ("abort_stage", C.c_int32),
        ("abort_inner", C.c_int32),
        ("abort_outer_stage", C.c_int32),
    ]


class RunResult(C.Structure):
    _fields_ = [
        ("n_steps", C.c_int64),
        ("steps_done", C.c_int64),
        ("aborted", C.c_int32),
        ("abort_kind", C.c_int32),
        ("abort_step", C.c_int64),
        ("abort_stage", C.c_int32),
        ("abort_inner", C.c_int32),
        ("gate_min", C.c_double),
        ("gate_max", C.c_double),
        ("n_fF", C.c_int64),
        ("n_fS", C.c_int64),
        ("n_exp", C.c_int64),
        ("s", C.c_int32),
        ("m", C.c_int32),
        ("eta", C.c_double),
        ("device_ms", C.c_double),
        ("abort_outer_stage", C.c_int32),
        ("reserved", C.c_int32),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class RhoResult(C.Structure):
    _fields_ = [
        ("rho", C.c_double),
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("safety", C.c_double),
    ]


DP = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)


def dptr(a: np.ndarray | None):
    """double* of a C-contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need contiguous float64"
    return a.ctypes.data_as(DP)


# Generic integrator layer (include/emrkc.h, emrkc_generic.cu): device
# callbacks. RhsFn: int (*)(void* ctx, double t, const double* y, double* out,
# int64_t len, void* stream); exp_part: int (*)(void* ctx, const double* y,
# double* lambda, double* y_inf, int64_t len, void* stream).
RHS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_int64,
                     C.c_void_p)
EXP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                     C.c_void_p)


class Counters(C.Structure):
    _fields_ = [("n_fF", C.c_int64), ("n_fS", C.c_int64), ("n_exp_steps", C.c_int64)]


class SplitRhsC(C.Structure):
    """emrkc_split_rhs (SplitRhs, P/include/mrkc/multirate.hpp:25-35)."""
    _fields_ = [
        ("f_F", RHS_FN), ("f_F_ctx", C.c_void_p),
        ("f_S", RHS_FN), ("f_S_ctx", C.c_void_p),
        ("exp_part", EXP_FN), ("exp_ctx", C.c_void_p),
        ("rho_F", C.c_double), ("rho_S", C.c_double),
        ("counters", C.POINTER(Counters)),
    ]


# Every function the header declares: name -> (restype, argtypes).
# emrkc_level_hook: void (*)(void* ctx)
LEVEL_HOOK = C.CFUNCTYPE(None, C.c_void_p)

PROTOTYPES = {
    "emrkc_version": (C.c_char_p, []),
    "emrkc_global_error": (C.c_char_p, []),
    "emrkc_get_stages": (C.c_int, [C.c_double, C.c_double, C.c_double, I32P, DP, DP]),
    "emrkc_rkc_coeffs": (C.c_int, [C.c_int32, C.c_double, DP, DP, DP, DP, DP, DP, DP]),
    "emrkc_plan_step": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(StepReport)]),
    "emrkc_model_info": (C.c_int, [C.c_int32, I32P, I32P]),
    "emrkc_resting_state": (C.c_int, [C.c_int32, DP, DP]),
    "emrkc_initial_state": (C.c_int, [C.POINTER(Problem), DP, C.c_int64]),
    "emrkc_state_len": (C.c_int64, [C.POINTER(Problem), C.POINTER(Partition)]),
    "emrkc_partition_slab": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(Partition)]),
    "emrkc_create": (C.c_int, [C.POINTER(Problem), C.c_int32, C.POINTER(Partition), C.POINTER(C.c_void_p)]),
    "emrkc_destroy": (None, [C.c_void_p]),
    "emrkc_last_error": (C.c_char_p, [C.c_void_p]),
    "emrkc_local_len": (C.c_int64, [C.c_void_p]),
    "emrkc_set_state": (C.c_int, [C.c_void_p, DP, C.c_int64]),
    "emrkc_get_state": (C.c_int, [C.c_void_p, DP, C.c_int64]),
    "emrkc_state_device_ptr": (C.c_int, [C.c_void_p, C.POINTER(DP)]),
    "emrkc_fused_active": (C.c_int32, [C.c_void_p]),
    "emrkc_node_kernel": (C.c_int32, [C.c_void_p]),
    "emrkc_synchronize": (C.c_int, [C.c_void_p]),
    "emrkc_eval_rhs": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, DP, DP, C.c_int64]),
    "emrkc_exp_part": (C.c_int, [C.c_void_p, DP, DP, DP, C.c_int64]),
    "emrkc_estimate_rho": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, DP, C.c_double, C.POINTER(RhoResult), DP]),
    "emrkc_step": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(StepReport)]),
    "emrkc_step_host": (C.c_int, [C.c_void_p, C.c_double, DP, DP, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(StepReport)]),
    "emrkc_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(RunResult)]),
    "emrkc_rel_l2_error": (C.c_int, [C.c_void_p, C.c_int32, DP, C.c_int32, DP]),
    "emrkc_set_stiff_gates": (C.c_int, [C.c_void_p, C.c_int32]),
    "emrkc_identify_stiff_gates": (C.c_int, [C.c_int32, DP, C.c_int64, I32P]),
    "emrkc_mrkc_step": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(StepReport)]),
    "emrkc_mrkc_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(RunResult)]),
    "emrkc_imex_step": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int32, C.POINTER(StepReport), C.POINTER(C.c_int64)]),
    "emrkc_imex_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_int32, C.POINTER(RunResult), C.POINTER(C.c_int64)]),
    "emrkc_exex_step": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.POINTER(StepReport)]),
    "emrkc_exex_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.POINTER(RunResult)]),
    "emrkc_run_timed": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.c_int64, DP, C.c_int64, C.POINTER(RunResult)]),
    "emrkc_group_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p)]),
    "emrkc_group_destroy": (None, [C.c_void_p]),
    "emrkc_group_estimate_rho": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.POINTER(RhoResult)]),
    "emrkc_group_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(RunResult)]),
    "emrkc_ipc_blob_size": (C.c_int64, []),
    "emrkc_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "emrkc_ipc_import": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]),
    "emrkc_dist_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(RunResult)]),
    "emrkc_dist_replay": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(RunResult)]),
    "emrkc_dist_link_local": (C.c_int, [C.c_void_p, C.c_void_p]),
    "emrkc_dist_lockstep_run": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(RunResult)]),
    "emrkc_set_slab_min_depth": (C.c_int, [C.c_void_p, C.c_int64]),
    "emrkc_set_level_hook": (C.c_int, [C.c_void_p, LEVEL_HOOK, C.c_void_p]),
    "emrkc_slab_power_begin": (C.c_int, [C.c_void_p, C.c_int32, DP]),
    "emrkc_slab_power_plane": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "emrkc_slab_power_sumsq": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_double, DP]),
    "emrkc_slab_power_fy": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "emrkc_slab_power_step": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "emrkc_slab_power_end": (C.c_int, [C.c_void_p, DP]),
    "emrkc_vctx_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "emrkc_vctx_destroy": (None, [C.c_void_p]),
    "emrkc_vctx_last_error": (C.c_char_p, [C.c_void_p]),
    "emrkc_vctx_stream": (C.c_void_p, [C.c_void_p]),
    "emrkc_vctx_alloc": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "emrkc_vctx_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "emrkc_vctx_upload": (C.c_int, [C.c_void_p, C.c_void_p, DP, C.c_int64]),
    "emrkc_vctx_download": (C.c_int, [C.c_void_p, DP, C.c_void_p, C.c_int64]),
    "emrkc_exponential_euler": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "emrkc_rkc_iteration": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_int64, C.c_double, RHS_FN, C.c_void_p, C.c_int32, C.c_double, C.c_void_p, I32P]),
    "emrkc_averaged_force": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_int64, C.c_double, C.POINTER(SplitRhsC), C.c_int32, C.c_int32, C.c_double, C.c_void_p, I32P]),
    "emrkc_averaged_force_mrkc": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_int64, C.c_double, C.POINTER(SplitRhsC), C.c_int32, C.c_double, C.c_void_p, I32P]),
    "emrkc_step_split": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_int64, C.c_double, C.POINTER(SplitRhsC), C.c_double, C.c_int32, C.c_void_p, C.POINTER(StepReport)]),
    "emrkc_mrkc_step_split": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_int64, C.c_double, C.POINTER(SplitRhsC), C.c_double, C.c_void_p, C.POINTER(StepReport)]),
    "emrkc_estimate_spectral_radius": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_int64, RHS_FN, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(RhoResult), C.c_void_p]),
    "emrkc_bind_split_rhs": (C.c_int, [C.c_void_p, C.POINTER(SplitRhsC)]),
    "emrkc_model_rates": (C.c_int, [C.c_int32, C.c_double, DP, DP]),
    "emrkc_model_ionic_current": (C.c_int, [C.c_int32, C.c_double, DP, DP]),
}

_lib = None


def load(path: str | None = None):
    """Load libemrkc_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} not found: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). "
            "There is no CPU fallback."
        )
    lib = C.CDLL(p)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
