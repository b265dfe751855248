"""ctypes binding of the C ABI in ``include/sgsf.h`` (libsgsf.so).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2501_19042_b200/csrc``) and loaded from this directory.  There is no
fallback: if the library or a CUDA device is missing, every solve raises.
Device memory and streams come from PyTorch; only raw pointers cross the ABI.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import DimensionMismatch, SingularKKT

LIB_PATH = Path(__file__).resolve().parent / "libsgsf.so"

SGSF_OK, SGSF_ERR_INVALID, SGSF_ERR_CUDA, SGSF_ERR_UNSUPPORTED, SGSF_ERR_SINGULAR = 0, 1, 2, 3, 4
SAMPLE_OK, SAMPLE_SINGULAR_KKT = 0, 1
PRECISION_LEAN, PRECISION_STRICT, PRECISION_HYBRID = 0, 1, 2

_dp = C.POINTER(C.c_double)


class Problem(C.Structure):
    _fields_ = [("n", C.c_int), ("samples", C.c_int), ("m1", C.c_int), ("rho", C.c_double),
                ("lat", C.c_double), ("vert", C.c_double), ("ws_lat", C.c_double), ("ws_vert", C.c_double),
                ("center", C.c_double * 3),
                ("W", _dp), ("Wd", _dp), ("Wdd", _dp), ("B", _dp), ("rhs", _dp), ("PBt", _dp),
                ("Km11", _dp), ("Kd11", _dp), ("Mm", _dp), ("Md", _dp), ("cconst", _dp)]


class Config(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("tol_residual", C.c_double), ("tol_eq", C.c_double),
                ("early_stop", C.c_int), ("precision", C.c_int), ("want_prev", C.c_int),
                ("slots_per_block", C.c_int), ("grid", C.c_int), ("verdict_tol", C.c_double)]


class Outputs(C.Structure):
    _fields_ = [("coeffs", C.c_void_p), ("multipliers", C.c_void_p), ("res_inf", C.c_void_p),
                ("res_l2", C.c_void_p), ("iterations", C.c_void_p), ("converged", C.c_void_p),
                ("displacement", C.c_void_p), ("status", C.c_void_p), ("eq_err", C.c_void_p),
                ("coeffs_prev", C.c_void_p), ("verdict", C.c_void_p)]


class Verdict(C.Structure):
    _fields_ = [("ok", C.c_void_p), ("feasible", C.c_void_p), ("pair_margin_min", C.c_void_p),
                ("ws_margin_max", C.c_void_p), ("pair_viol", C.c_void_p), ("ws_viol", C.c_void_p)]


class Decoder(C.Structure):
    _fields_ = [("L", C.c_int), ("c0", C.c_int), ("nm1", C.c_int), ("leaky", C.c_int), ("slope", C.c_float),
                ("scale", C.c_float), ("wpack", C.c_void_p), ("bias", C.c_void_p), ("head_w", C.c_void_p),
                ("head_b", C.c_void_p), ("exp_w", C.c_void_p), ("exp_b", C.c_void_p), ("cz", C.c_int),
                ("feat", C.c_void_p), ("base", C.c_void_p), ("B6", C.c_void_p), ("PBt", C.c_void_p),
                ("rhs", C.c_void_p), ("n", C.c_int), ("m1", C.c_int)]


class Timing(C.Structure):
    _fields_ = [("start", C.c_void_p), ("stop", C.c_void_p)]


EXPORTS = {
    "sgsf_version": (C.c_char_p, []),
    "sgsf_last_error": (C.c_char_p, []),
    "sgsf_launch_count": (C.c_uint64, []),
    "sgsf_max_robots": (C.c_int, []),
    "sgsf_workspace_bytes": (C.c_size_t, [C.c_int]),
    "sgsf_create": (C.c_int, [C.POINTER(Problem), C.POINTER(C.c_void_p)]),
    "sgsf_destroy": (None, [C.c_void_p]),
    "sgsf_solve": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.POINTER(Config), C.POINTER(Outputs), C.c_void_p, C.POINTER(Timing), C.c_void_p]),
    "sgsf_solve_host": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(Config)] + [C.c_void_p] * 9 + [C.c_void_p]),
    "sgsf_verdict": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_double,
                               C.POINTER(Verdict), C.c_void_p]),
    "sgsf_trajectory": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    "sgsf_svars": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p] + [C.c_void_p] * 6 + [C.c_void_p]),
    "sgsf_spherical_project": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_int] + [C.c_void_p] * 6 + [C.c_void_p]),
    "sgsf_apply_F": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgsf_apply_FT": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgsf_kkt_step": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgsf_unroll": (C.c_int, [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 5 + [C.c_void_p]),
    "sgsf_unroll_backward": (C.c_int, [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 6 + [C.c_void_p]),
    "sgsf_cosine_work_doubles": (C.c_size_t, [C.c_int, C.c_int]),
    "sgsf_pairwise_cosine": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgsf_fp32_peak": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]),
    "sgsf_decoder_pack_bytes": (C.c_size_t, [C.c_int]),
    "sgsf_decoder_forward": (C.c_int, [C.POINTER(Decoder), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgsf_decoder_forward_dbg": (C.c_int, [C.POINTER(Decoder), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_int, C.c_void_p]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def load():
    """Load libsgsf.so and declare every exported symbol (raises if the build is missing)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              "g.build()'` or `make -C paper_2501_19042_b200/csrc`")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == SGSF_OK:
        return
    msg = load().sgsf_last_error().decode(errors="replace")
    if rc == SGSF_ERR_INVALID:
        raise DimensionMismatch(f"{what}: {msg}")
    if rc == SGSF_ERR_SINGULAR:
        raise SingularKKT(f"{what}: {msg}")
    if rc == SGSF_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg}")


def launch_count() -> int:
    return int(load().sgsf_launch_count())


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream) -> int:
    return stream.cuda_stream if stream is not None else 0
