"""ctypes wrapper around ``lif_oracle.c`` (TEST INFRASTRUCTURE ONLY -- see __init__.py).

Marshalling only: every number is computed by the C file, in fp64, on the exact input
values the caller passes (fp32 / bf16 values are widened to float64 exactly).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lif_oracle.c")
_LIB = os.path.join(_HERE, "liblif_oracle.so")


def build_oracle(force: bool = False) -> str:
    """Compile lif_oracle.c with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("tau", ctypes.c_double),
        ("v_th", ctypes.c_double),
        ("v_reset", ctypes.c_double),
        ("soft_reset", ctypes.c_int),
        ("decay_input", ctypes.c_int),
        ("detach_reset", ctypes.c_int),
        ("surrogate", ctypes.c_int),
        ("alpha", ctypes.c_double),
        ("smoothed", ctypes.c_int),
    ]


@dataclass(frozen=True)
class OracleParams:
    """LIF hyper-parameters as the oracle reads them.

    ``tau``, ``v_th``, ``v_reset`` and ``alpha`` are taken as given; callers that
    compare against an fp32 kernel pass the same float32 values the kernel received
    (widened exactly to double), SURVEY R9.
    """
    tau: float = 1.25
    v_th: float = 0.3
    v_reset: float = 0.0
    soft_reset: bool = False
    decay_input: bool = False
    detach_reset: bool = False
    surrogate: str = "sigmoid"  # or "atan"
    alpha: float = 4.0
    smoothed: bool = False

    def _c(self) -> _Params:
        return _Params(float(self.tau), float(self.v_th), float(self.v_reset),
                       int(self.soft_reset), int(self.decay_input), int(self.detach_reset),
                       {"sigmoid": 0, "atan": 1}[self.surrogate], float(self.alpha),
                       int(self.smoothed))


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        P = ctypes.POINTER(_Params)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.lif_oracle_surrogate.argtypes = [P, ctypes.c_double]
        lib.lif_oracle_surrogate.restype = ctypes.c_double
        lib.lif_oracle_smooth_step.argtypes = [P, ctypes.c_double]
        lib.lif_oracle_smooth_step.restype = ctypes.c_double
        lib.lif_oracle_forward.argtypes = [P, ctypes.c_int64, ctypes.c_int64, dp, dp,
                                           dp, dp, dp, dp, dp]
        lib.lif_oracle_forward.restype = None
        lib.lif_oracle_backward.argtypes = [P, ctypes.c_int64, ctypes.c_int64, dp, dp, dp,
                                            dp, dp, dp, dp, dp]
        lib.lif_oracle_backward.restype = None
        i64 = ctypes.c_int64
        lib.lif_oracle_affine_input.argtypes = [i64, i64, dp, dp, dp, i64, i64, dp]
        lib.lif_oracle_affine_input.restype = None
        lib.lif_oracle_affine_residual_input.argtypes = [i64, i64, dp, dp, dp, dp, i64, i64, dp]
        lib.lif_oracle_affine_residual_input.restype = None
        lib.lif_oracle_affine_grads.argtypes = [i64, i64, dp, dp, dp, i64, i64, dp, dp, dp]
        lib.lif_oracle_affine_grads.restype = None
        _lib = lib
    return _lib


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def surrogate(p: OracleParams, u: float) -> float:
    """delta(u), u = H - V_th."""
    c = p._c()
    return _load().lif_oracle_surrogate(ctypes.byref(c), float(u))


def smooth_step(p: OracleParams, u: float) -> float:
    """The surrogate's primitive (sigma(alpha u) or 1/2 + arctan(.)/pi)."""
    c = p._c()
    return _load().lif_oracle_smooth_step(ctypes.byref(c), float(u))


def forward(p: OracleParams, x, v_init=None):
    """Forward over all T steps.  ``x``: [T, N] array-like.  Returns a dict with
    S (float64 0/1, or the smooth step), H, V (post-reset, every step) and v_final."""
    x = _f64(x)
    if x.ndim == 1:
        x = x[:, None]
    T, N = x.shape
    vi = None if v_init is None else _f64(v_init).reshape(N)
    S = np.empty((T, N)); H = np.empty((T, N)); V = np.empty((T, N))
    vf = np.empty(N); work = np.empty(N)
    c = p._c()
    _load().lif_oracle_forward(ctypes.byref(c), T, N, _dp(x), _dp(vi), _dp(S), _dp(H),
                               _dp(V), _dp(vf), _dp(work))
    return {"S": S, "H": H, "V": V, "v_final": vf}


def backward(p: OracleParams, gS, H, grad_v_final=None, return_terms=False):
    """Backward over t = T-1..0.  Returns (gX [T, N], grad_v_init [N]) and, with
    return_terms, also {"delta": [T, N], "dVdH": [T, N]} (for error bounds)."""
    gS = _f64(gS); H = _f64(H)
    if gS.ndim == 1:
        gS = gS[:, None]; H = H[:, None]
    T, N = gS.shape
    assert H.shape == (T, N)
    gvf = None if grad_v_final is None else _f64(grad_v_final).reshape(N)
    gX = np.empty((T, N)); gvi = np.empty(N); work = np.empty(N)
    d = np.empty((T, N)) if return_terms else None
    dv = np.empty((T, N)) if return_terms else None
    c = p._c()
    _load().lif_oracle_backward(ctypes.byref(c), T, N, _dp(gS), _dp(H), _dp(gvf), _dp(gX),
                                _dp(gvi), _dp(work), _dp(d), _dp(dv))
    if return_terms:
        return gX, gvi, {"delta": d, "dVdH": dv}
    return gX, gvi


def affine_input(x, scale, shift, C, HW, residual=None):
    """X'[t, n] = scale[c] X[t, n] + shift[c] (+ R[t, n]), c = (n / HW) % C.
    The gradient of the residual R is dL/dX' itself (lif_oracle_affine_residual_input)."""
    x = _f64(x); scale = _f64(scale); shift = _f64(shift)
    T, N = x.shape
    out = np.empty((T, N))
    if residual is None:
        _load().lif_oracle_affine_input(T, N, _dp(x), _dp(scale), _dp(shift), int(C), int(HW), _dp(out))
    else:
        r = _f64(residual)
        assert r.shape == x.shape
        _load().lif_oracle_affine_residual_input(T, N, _dp(x), _dp(scale), _dp(shift), _dp(r), int(C),
                                                 int(HW), _dp(out))
    return out


def affine_grads(x, gxp, scale, C, HW):
    """(dL/dX, dL/dscale [C], dL/dshift [C]) from dL/dX' through the affine prologue."""
    x = _f64(x); gxp = _f64(gxp); scale = _f64(scale)
    T, N = x.shape
    gx = np.empty((T, N)); gs = np.empty(int(C)); gb = np.empty(int(C))
    _load().lif_oracle_affine_grads(T, N, _dp(x), _dp(gxp), _dp(scale), int(C), int(HW), _dp(gx),
                                    _dp(gs), _dp(gb))
    return gx, gs, gb
