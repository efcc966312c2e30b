"""ctypes binding of the C-ABI declared in include/rte_b200.h (librte_b200.so).

This is the reference-facing boundary the parity tests and bench.py call
through.  The library is built in-tree (paper_2402_10488_b200/build.py); a
missing library is a hard error -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RTE_B200_LIB", os.path.join(HERE, "librte_b200.so"))

RTE_OK, RTE_ERR_INVALID, RTE_ERR_RUNTIME, RTE_ERR_CUDA, RTE_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
RTE_SLAB1D, RTE_XY2D = 0, 1
RTE_SI, RTE_DSA, RTE_ROMSA, RTE_ROMSAD, RTE_ROMIG, RTE_CUSTOM = 0, 1, 2, 3, 4, 5
RTE_NORM_ABS, RTE_NORM_REL = 0, 1
RTE_DSA_OK, RTE_DSA_MAXIT, RTE_DSA_BREAKDOWN, RTE_DSA_NAN = 0, 1, 2, 3
RTE_GUESS_ZERO, RTE_GUESS_SUPPLIED, RTE_GUESS_ROMIG = 0, 1, 2
PROF_KINDS = ("sweep", "reduce", "dsa", "rom", "other", "dsa_smooth0")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p


class Problem(ctypes.Structure):
    _fields_ = [("geometry", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("bounds", _dp),
                ("x0", ctypes.c_double), ("x1", ctypes.c_double), ("y0", ctypes.c_double), ("y1", ctypes.c_double),
                ("n_dirs", ctypes.c_int), ("dirs", _dp), ("weights", _dp), ("inflow", ctypes.c_double * 4),
                ("n_samples", ctypes.c_int), ("block", ctypes.c_int), ("mt", _dp), ("ms", _dp), ("source", _dp),
                ("source_shared", ctypes.c_int)]


class Affine(ctypes.Structure):
    _fields_ = [("k_terms", ctypes.c_int), ("term_mt", _dp), ("term_ms", _dp), ("psi", _dp)]


class Rom(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("k_affine", ctypes.c_int), ("u_rho", _dp), ("u_iso", _dp), ("a_r", _dp),
                ("b_r", _dp), ("eps_pod", ctypes.c_double), ("eps_train", ctypes.c_double)]


# rte_correction_fn (the CorrectionStrategy plugin point, solvers.hpp:38-51)
CORRECTION_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                 ctypes.POINTER(ctypes.c_int), ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.POINTER(ctypes.c_char), ctypes.c_void_p)


class SiConfig(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("eps", ctypes.c_double), ("norm", ctypes.c_int),
                ("max_iters", ctypes.c_int), ("fixed_iters", ctypes.c_int), ("theta", ctypes.c_int),
                ("eps_romsad", ctypes.c_double), ("use_guess", ctypes.c_int), ("compute_residual", ctypes.c_int),
                ("check_every", ctypes.c_int), ("correct", CORRECTION_FN), ("correct_user", ctypes.c_void_p),
                ("dsa_inner", ctypes.c_double), ("dsa_floor", ctypes.c_double)]


class SiReport(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("iterations", ctypes.c_int), ("n_sweep", ctypes.c_long),
                ("switch_iter", ctypes.c_int), ("singular", ctypes.c_int), ("final_residual", ctypes.c_double),
                ("last_change", ctypes.c_double), ("dsa_status", ctypes.c_int)]


# (name, restype, argtypes) for every symbol include/rte_b200.h declares.
class GmresConfig(ctypes.Structure):
    _fields_ = [("preconditioned", ctypes.c_int), ("restart", ctypes.c_int), ("rel_tol", ctypes.c_double),
                ("max_iters", ctypes.c_int), ("guess", ctypes.c_int)]


class GmresReport(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("iterations", ctypes.c_int), ("n_sweep", ctypes.c_long),
                ("cycles", ctypes.c_int), ("final_residual", ctypes.c_double), ("history_len", ctypes.c_int),
                ("dsa_status", ctypes.c_int)]


SIGNATURES = [
    ("rte_create", ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int, ctypes.POINTER(_vp)]),
    ("rte_destroy", None, [_vp]),
    ("rte_last_error", ctypes.c_char_p, [_vp]),
    ("rte_n_dof", ctypes.c_long, [_vp]),
    ("rte_n_samples", ctypes.c_int, [_vp]),
    ("rte_n_slots", ctypes.c_int, [_vp]),
    ("rte_sweep_plan", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("rte_apply_L", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_assemble_rhs", ctypes.c_int, [_vp, _vp, _vp]),
    ("rte_fixed_point", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_sweep_direction", ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    ("rte_kinetic_sweep", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_density_of", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_apply_Ms", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_apply_Mt", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_set_affine", ctypes.c_int, [_vp, ctypes.POINTER(Affine)]),
    ("rte_apply_term_kinetic", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    ("rte_collect_snapshots", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, _vp, _vp, _vp, _ip,
                                             _ip]),
    ("rte_snapshot_columns", ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _ip, _ip, ctypes.c_int, ctypes.c_int, _vp,
                                            _ip]),
    ("rte_pod", ctypes.c_int, [ctypes.c_int, ctypes.c_long, ctypes.c_int, _vp, ctypes.c_int, _vp, _dp, _vp]),
    ("rte_truncation_rank", ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_double]),
    ("rte_build_rom", ctypes.c_int, [_vp, ctypes.c_int, _vp, _dp, _dp, _dp, _dp]),
    ("rte_dsa_setup", ctypes.c_int, [_vp, _vp]),
    ("rte_dsa_solve_density", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_dsa_correct", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_dsa_coupled_dim", ctypes.c_long, [_vp]),
    ("rte_dsa_apply_eliminated", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_dsa_set_tolerance", ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_int]),
    ("rte_dsa_last_iterations", ctypes.c_int, [_vp]),
    ("rte_dsa_iteration_log", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int]),
    ("rte_dsa_reset_history", ctypes.c_int, [_vp, _vp]),
    ("rte_rom_load", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(Rom)]),
    ("rte_romig", ctypes.c_int, [_vp, _vp, _ip, _vp]),
    ("rte_si_solve", ctypes.c_int, [_vp, ctypes.POINTER(SiConfig), _vp, ctypes.POINTER(SiReport), _dp,
                                    ctypes.c_char_p]),
    ("rte_apply_kinetic", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("rte_apply_streaming_collision", ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    ("rte_kinetic_rhs", ctypes.c_int, [_vp, _vp, _vp]),
    ("rte_gmres_solve", ctypes.c_int, [_vp, ctypes.POINTER(GmresConfig), _vp, ctypes.POINTER(GmresReport), _dp,
                                       ctypes.c_int]),
    ("rte_profile_enable", ctypes.c_int, [_vp, ctypes.c_int]),
    ("rte_profile_read", ctypes.c_int, [_vp, _dp, ctypes.POINTER(ctypes.c_long)]),
    ("rte_probe_dfma", ctypes.c_int, [ctypes.c_int, _dp]),
    ("rte_gauss_legendre_nodes", ctypes.c_int, [ctypes.c_int, _dp, _dp]),
    ("rte_cell_points", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, _dp, _dp]),
    ("rte_weighted_mass", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, _dp, _dp]),
    ("rte_project", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_int, _dp, _dp]),
    ("rte_unit_draws", ctypes.c_int, [ctypes.c_ulonglong, ctypes.c_long, _dp]),
    ("rte_scalar_blocks", ctypes.c_int, [ctypes.c_long, ctypes.c_int, _dp, _dp]),
    ("rte_weighted_mass_const", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                               ctypes.c_double, _dp]),
    ("rte_project_const", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                         ctypes.c_double, _dp]),
    ("rte_combine_terms", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_long, _dp, _dp, _dp]),
    ("rte_guard_check", ctypes.c_int, [ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long)]),
    ("rte_guard_selftest", ctypes.c_int, [ctypes.c_int]),
]

_lib = None


class RteError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class RteInvalidArgument(RteError, ValueError):
    """RTE_ERR_INVALID -- the reference's std::invalid_argument."""


def load(path: str = LIB_PATH):
    """Load librte_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError("librte_b200.so not built: run `python -m paper_2402_10488_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code: int, ctx=None):
    if code == RTE_OK:
        return
    msg = load().rte_last_error(ctx)
    msg = msg.decode() if msg else "error %d" % code
    if code == RTE_ERR_INVALID:
        raise RteInvalidArgument(code, msg)
    raise RteError(code, msg)


def dptr(a) -> "_dp":
    """double* of a contiguous float64 numpy array."""
    return a.ctypes.data_as(_dp)
