"""ctypes binding of ``libredve_b200.so`` (the C ABI in include/redve_b200.h).

This is the reference-side FFI binding for the hot path: the reference is
pure Python, so ctypes is the FFI it would use.  There is no fallback: if
the library is missing or no CUDA device is present, every compute call
raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libredve_b200.so")

REDVE_OK, E_VALUE, E_SHAPE, E_KERNEL, E_CUDA, E_NONFINITE, E_CG, E_UNSUPPORTED = range(8)
OP_BLUR, OP_BLUR_DOWNSAMPLE = 0, 1
DN_IDENTITY, DN_CONV, DN_MEDIAN3, DN_FILTERBANK, DN_PATCH, DN_EXTERNAL = range(6)
VE_CODES = {"mpe": 0, "rre": 1, "svdmpe": 2}
VE_NAMES = {v: k for k, v in VE_CODES.items()}
METHOD_FP, METHOD_FP_VE, METHOD_SD, METHOD_SD_VE, METHOD_NESTEROV = range(5)
METHOD_CODES = {"fp": METHOD_FP, "fp-ve": METHOD_FP_VE, "sd": METHOD_SD, "sd-ve": METHOD_SD_VE,
                "nesterov": METHOD_NESTEROV}
MAXKP1 = 12

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class OperatorDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("ksize", C.c_int), ("taps", _dp), ("factor", C.c_int)]


class DenoiserDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("ksize", C.c_int), ("taps", _dp),
        ("patch_radius", C.c_int), ("search_radius", C.c_int), ("balance_iters", C.c_int),
        ("h", C.c_double),
        ("n_filters", C.c_int), ("fsize", C.c_int), ("filters", _dp), ("scales", _dp),
        ("tau", C.c_double), ("weight_bits", C.c_int),
    ]


class SolveConfigC(C.Structure):
    _fields_ = [
        ("method", C.c_int), ("ve_method", C.c_int), ("m", C.c_int), ("kappa", C.c_int),
        ("max_inner_steps", C.c_int), ("tol", C.c_double), ("stabilization_iters", C.c_int),
        ("rank_tolerance", C.c_double), ("step_size", C.c_double),
    ]


class TraceC(C.Structure):
    _fields_ = [
        ("cap", C.c_int), ("ccap", C.c_int),
        ("n_records", _ip), ("step_norm", _dp), ("cost", _dp), ("psnr", _dp),
        ("gamma_abs_sum", _dp), ("elapsed_s", _dp), ("n_cycles", _ip), ("cycle_meta", _ip),
        ("cycle_stability", _dp), ("cycle_gamma", _dp), ("cycle_c", _dp), ("status", _ip),
        ("returned_best", _ip), ("cg_iters", _ip),
    ]


class VeResultC(C.Structure):
    _fields_ = [
        ("converged", C.c_int), ("extrapolated", C.c_int), ("kappa_used", C.c_int),
        ("method", C.c_int), ("fallback", C.c_int), ("stability_sum", C.c_double),
        ("gamma", C.c_double * 12), ("c", C.c_double * 12),
    ]


# The exported symbols, exactly the declarations of include/redve_b200.h.
SYMBOLS = {
    "redve_version": (C.c_char_p, []),
    "redve_kernel_launches": (C.c_uint64, []),
    "redve_release_cached_memory": (None, []),
    "redve_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "redve_profile_report": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, _dp, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int)]),
    "redve_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "redve_destroy": (None, [C.c_void_p]),
    "redve_last_error": (C.c_char_p, [C.c_void_p]),
    "redve_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "redve_synchronize": (C.c_int, [C.c_void_p]),
    "redve_denoise": (C.c_int, [C.c_void_p, C.POINTER(DenoiserDesc), C.c_int, C.c_int, C.c_int,
                                C.c_void_p, C.c_void_p]),
    "redve_patch_weight_maps": (C.c_int, [C.c_void_p, C.POINTER(DenoiserDesc), C.c_int, C.c_int,
                                          C.c_int, C.c_void_p, C.c_void_p]),
    "redve_operator_apply": (C.c_int, [C.c_void_p, C.POINTER(OperatorDesc), C.c_int, C.c_int,
                                       C.c_int, C.c_void_p, C.c_void_p]),
    "redve_operator_adjoint": (C.c_int, [C.c_void_p, C.POINTER(OperatorDesc), C.c_int, C.c_int,
                                         C.c_int, C.c_void_p, C.c_void_p]),
    "redve_problem_create": (C.c_int, [C.c_void_p, C.POINTER(OperatorDesc), C.POINTER(DenoiserDesc),
                                       C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_double,
                                       C.c_double, C.c_void_p, C.POINTER(C.c_void_p)]),
    "redve_problem_destroy": (None, [C.c_void_p]),
    "redve_problem_set_measurements": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "redve_problem_graph_captures": (C.c_uint64, [C.c_void_p]),
    "redve_fp_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "redve_fp_step_denoised": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "redve_gradient": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "redve_cost": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, _dp, _dp, _dp, _dp]),
    "redve_solve": (C.c_int, [C.c_void_p, C.POINTER(SolveConfigC), C.c_void_p, C.c_void_p,
                              C.POINTER(TraceC)]),
    "redve_sr_normal_matvec": (C.c_int, [C.c_void_p, C.POINTER(OperatorDesc), C.c_double, C.c_double,
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                         C.c_void_p]),
    "redve_vec_dot": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, _dp]),
    "redve_vec_dist2": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, _dp]),
    "redve_vec_axpby": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_double,
                                  C.c_void_p]),
    "redve_enable_peer_access": (C.c_int, [C.c_void_p, C.c_int]),
    "redve_halo_push": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "redve_sr_fidelity": (C.c_int, [C.c_void_p, C.POINTER(OperatorDesc), C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, _dp]),
    "redve_window_gram": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, _dp]),
    "redve_ve_decide": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_int, C.c_double,
                                  C.POINTER(VeResultC), _dp, C.POINTER(C.c_int)]),
    "redve_ve_decide_r": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_int, C.c_int,
                                    C.POINTER(VeResultC), _dp]),
    "redve_window_combine": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int, _dp,
                                       C.c_void_p]),
    "redve_extrapolate": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_int,
                                    C.c_double, C.c_void_p, C.POINTER(VeResultC)]),
}

_lib = None
_lock = threading.Lock()


def library():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(_LIB_PATH):
                    raise ImportError(
                        f"{_LIB_PATH} is missing: build it with `python __graft_entry__.py` "
                        "(there is no CPU fallback)")
                lib = C.CDLL(_LIB_PATH)
                for name, (res, args) in SYMBOLS.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_ctx = {}


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("redve_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch


def context(device: int | None = None):
    """Native context of (device, calling thread), bound to torch's current stream.

    A context is not thread-safe but distinct contexts run concurrently
    (include/redve_b200.h), so every host thread gets its own: that is what lets
    ``pipeline.solve_stream`` keep several batches in flight."""
    import threading

    torch = _torch()
    dev = torch.cuda.current_device() if device is None else int(device)
    lib = library()
    key = (dev, threading.get_ident())
    if key not in _ctx:
        h = C.c_void_p()
        rc = lib.redve_create(C.byref(h), dev)
        if rc != REDVE_OK:
            raise NativeError(rc, lib.redve_last_error(h).decode())
        _ctx[key] = h
    h = _ctx[key]
    lib.redve_set_stream(h, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    return h


def check(rc, ctx):
    if rc != REDVE_OK:
        msg = library().redve_last_error(ctx).decode()
        from . import errors

        raise errors.from_code(rc, msg)


def dptr(t):
    """Raw device pointer of a contiguous fp64 CUDA tensor (or None)."""
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return C.c_void_p(t.data_ptr())


def hptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


def profile(enable: bool, device: int | None = None):
    lib = library()
    lib.redve_profile(context(device), 1 if enable else 0)


def profile_report(device: int | None = None):
    """{kernel kind: (total_ms, launches)} since the last report (synchronises)."""
    lib = library()
    ctx = context(device)
    mx = 64
    names = C.create_string_buffer(32 * mx)
    tot = np.zeros(mx)
    cnt = np.zeros(mx, np.int64)
    n = C.c_int()
    check(lib.redve_profile_report(ctx, mx, names, hptr(tot), cnt.ctypes.data_as(
        C.POINTER(C.c_int64)), C.byref(n)), ctx)
    out = {}
    for k in range(n.value):
        nm = names.raw[32 * k: 32 * k + 32].split(b"\0")[0].decode()
        out[nm] = (float(tot[k]), int(cnt[k]))
    return out


def kernel_launches() -> int:
    return int(library().redve_kernel_launches())
