"""The reference-side binding: route ``swarmfilter.SafetyFilter.batch_solve`` through the C ABI.

This is the module a maintainer of the reference would drop in as ``swarmfilter/kernels/b200.py``
(INTEGRATION.md section 2 shows it verbatim; ``tests/test_refbind.py`` checks that the two agree and runs
it on the real reference's objects).  It uses nothing of this package's Python API except the FP64
host precompute: plain ctypes over ``libsgsf.so`` (``include/sgsf.h``), numpy buffers in and out through
``sgsf_solve_host``.  The reference's plug-in points it replaces: ``SafetyFilter.batch_solve``
(``solver.py:368-407``, the per-item error isolation of ``_solve_guarded`` 361-366) and the
spherical-kernel backend registry (``kernels/__init__.py:11-50``), which is called per iteration and per
sample and so is far too fine-grained to cross to a GPU.
"""
import ctypes
import os

import numpy as np

from paper_2501_19042_b200.precompute import device_constants   # FP64 host precompute (also takes reference objects)

_dp = ctypes.POINTER(ctypes.c_double)
LIB = os.environ.get("SGSF_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsgsf.so"))
lib = ctypes.CDLL(LIB)


class Problem(ctypes.Structure):   # sgsf_problem_t
    _fields_ = [("n", ctypes.c_int), ("samples", ctypes.c_int), ("m1", ctypes.c_int), ("rho", ctypes.c_double),
                ("lat", ctypes.c_double), ("vert", ctypes.c_double), ("ws_lat", ctypes.c_double),
                ("ws_vert", ctypes.c_double), ("center", ctypes.c_double * 3)] + \
               [(k, _dp) for k in ("W", "Wd", "Wdd", "B", "rhs", "PBt", "Km11", "Kd11", "Mm", "Md", "cconst")]


class Config(ctypes.Structure):    # sgsf_config_t (all nine fields: the library copies the whole struct)
    _fields_ = [("max_iters", ctypes.c_int), ("tol_residual", ctypes.c_double), ("tol_eq", ctypes.c_double),
                ("early_stop", ctypes.c_int), ("precision", ctypes.c_int), ("want_prev", ctypes.c_int),
                ("slots_per_block", ctypes.c_int), ("grid", ctypes.c_int), ("verdict_tol", ctypes.c_double)]


_vp = ctypes.c_void_p
lib.sgsf_last_error.restype = ctypes.c_char_p
lib.sgsf_last_error.argtypes = []
lib.sgsf_create.restype = ctypes.c_int
lib.sgsf_create.argtypes = [ctypes.POINTER(Problem), ctypes.POINTER(_vp)]
lib.sgsf_destroy.restype = None
lib.sgsf_destroy.argtypes = [_vp]
lib.sgsf_solve_host.restype = ctypes.c_int
lib.sgsf_solve_host.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.POINTER(Config)] + [_vp] * 9 + [_vp]

PRECISION = {"lean": 0, "strict": 1, "hybrid": 2}   # SGSF_PRECISION_*: hybrid keeps the FP64 counts and verdicts


def batch_solve_b200(sf, proposals, config, precision="hybrid", verdict_tol=1e-3):
    """``sf``: a ``swarmfilter.SafetyFilter`` (its problem, basis and equality); ``proposals``: (B, dim) array;
    ``config``: a ``swarmfilter.SolverConfig``.  Returns numpy arrays; ``status[b] == 1`` marks a SingularKKT
    sample (the reference isolates it as a failed SolveResult, solver.py:361-366)."""
    k = device_constants(sf.problem, sf.basis, sf.equality, config.rho)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (k.W, k.Wd, k.Wdd, k.B, k.rhs, k.PBt, k.Km11, k.Kd11, k.Mm, k.Md, k.cconst)]
    pr = Problem(k.n, k.samples, k.m1, k.rho, k.lat, k.vert, k.ws_lat, k.ws_vert, (ctypes.c_double * 3)(*k.center),
                 *[a.ctypes.data_as(_dp) for a in arrs])
    h = _vp()
    if lib.sgsf_create(ctypes.byref(pr), ctypes.byref(h)) != 0:
        raise RuntimeError(lib.sgsf_last_error().decode())
    try:
        X = np.ascontiguousarray(proposals, dtype=np.float64)
        B, dim = X.shape
        mi = config.max_iters
        out = dict(coeffs=np.empty((B, dim)), multipliers=np.empty((B, dim)), residual_inf=np.empty((B, mi)),
                   residual_l2=np.empty((B, mi)), iterations=np.empty(B, np.int32), converged=np.empty(B, np.uint8),
                   feasible=np.empty(B, np.uint8), displacement=np.empty(B), status=np.empty(B, np.int32))
        cfg = Config(mi, config.tol_residual, config.tol_eq, int(config.early_stop), PRECISION[precision], 0, 0, 0,
                     verdict_tol)
        rc = lib.sgsf_solve_host(h, B, X.ctypes.data, None, None, None, ctypes.byref(cfg),
                                 *(out[f].ctypes.data for f in ("coeffs", "multipliers", "residual_inf", "residual_l2",
                                                                 "iterations", "converged", "feasible", "displacement",
                                                                 "status")), None)
        if rc != 0:
            raise RuntimeError(lib.sgsf_last_error().decode())
        return out
    finally:
        lib.sgsf_destroy(h)
