"""numpy-facing wrapper of the C oracle (streamstab_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this
module, and only as the checker / the timed CPU restatement of the reference.
The product package never imports it.

Every function mirrors the reference function of the same name
(/root/reference/pkg/src/streamstab/flow.py, consistency.py) on plain numpy
arrays; flows are passed as (uv float32 (H, W, 2), valid bool (H, W)).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libstreamstab_oracle.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile the oracle library in place (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Params(ctypes.Structure):
    _fields_ = [
        ("k1", ctypes.c_float),
        ("k2", ctypes.c_float),
        ("alpha", ctypes.c_float),
        ("lam", ctypes.c_float),
        ("eta", ctypes.c_float),
        ("kappa", ctypes.c_float),
        ("iterations", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "streamstab_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        c_int, vp = ctypes.c_int, ctypes.c_void_p
        L.orc_backward_warp.argtypes = [_f32p, c_int, c_int, c_int, _f32p, _u8p, _f32p, vp]
        L.orc_occlusion_mask.argtypes = [_f32p, _u8p, _f32p, _u8p, c_int, c_int, _f32p]
        L.orc_warp_weight.argtypes = [_f32p, _f32p, c_int, c_int, c_int, ctypes.c_float,
                                      ctypes.c_float, vp, _f32p]
        L.orc_local_blend.argtypes = [_f32p, _f32p, _f32p, _f32p, _f32p, c_int, c_int, c_int, _f32p]
        L.orc_adaptive_blend.argtypes = [_f32p, _f32p, _f32p, c_int, c_int, c_int, _f32p]
        L.orc_consistency_weight.argtypes = [_f32p, _f32p, c_int, c_int, c_int, ctypes.c_float,
                                             ctypes.c_float, _f32p]
        L.orc_laplacian.argtypes = [_f32p, c_int, c_int, c_int, _f32p]
        L.orc_numpy_pairwise_sum.argtypes = [_f32p, ctypes.c_ssize_t]
        L.orc_numpy_pairwise_sum.restype = ctypes.c_float
        L.orc_solve_screened_poisson.argtypes = [_f32p, _f32p, _f32p, c_int, c_int, c_int,
                                                 ctypes.POINTER(_Params), _f32p, _f32p,
                                                 ctypes.POINTER(ctypes.c_int)]
        L.orc_run_step.argtypes = [c_int, c_int, c_int, c_int, _f32p, _f32p, _f32p, _f32p, vp, vp,
                                   _f32p, _f32p, _u8p, vp, vp, ctypes.POINTER(_Params), _f32p,
                                   vp, vp, ctypes.POINTER(ctypes.c_int)]
        L.orc_num_threads.restype = c_int
        L.orc_set_num_threads.argtypes = [c_int]
        _lib = L
    return _lib


class OracleDivergence(Exception):
    def __init__(self, iteration: int):
        super().__init__(f"solver diverged at iteration {iteration}")
        self.iteration = iteration


@dataclass(frozen=True)
class Params:
    """Mirror of ConsistencyParams (consistency.py:37-51)."""

    k1: float = 0.3
    k2: float = 0.5
    alpha: float = 6.5e3
    lam: float = 2.0
    eta: float = 0.15
    kappa: float = 0.2
    iterations: int = 150

    def c(self) -> _Params:
        return _Params(self.k1, self.k2, self.alpha, self.lam, self.eta, self.kappa,
                       int(self.iterations))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _hwc(img):
    img = _f32(img)
    return img if img.ndim == 3 else img[:, :, None]


def _flow(uv, valid=None):
    uv = _f32(uv)
    if valid is None:
        valid = np.abs(uv).max(axis=2) <= 1e9  # imgio.py:172
    return uv, np.ascontiguousarray(valid, dtype=np.uint8)


def set_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def backward_warp(image, uv, valid=None):
    squeeze = np.asarray(image).ndim == 2
    img = _hwc(image)
    h, w, c = img.shape
    uv, vd = _flow(uv, valid)
    out = np.empty_like(img)
    mask = np.empty((h, w), np.float32)
    lib().orc_backward_warp(img, h, w, c, uv, vd, out, mask.ctypes.data)
    return (out[:, :, 0] if squeeze else out), mask


def occlusion_mask(fwd_uv, fwd_valid, bwd_uv, bwd_valid):
    fu, fv = _flow(fwd_uv, fwd_valid)
    bu, bv = _flow(bwd_uv, bwd_valid)
    h, w = fu.shape[:2]
    out = np.empty((h, w), np.float32)
    lib().orc_occlusion_mask(fu, fv, bu, bv, h, w, out)
    return out


def warp_weight(reference, warped, alpha, bound, validity=None):
    r, wv = _hwc(reference), _hwc(warped)
    h, w, c = r.shape
    out = np.empty((h, w), np.float32)
    vp = None
    if validity is not None:
        validity = _f32(validity)
        vp = validity.ctypes.data
    lib().orc_warp_weight(r, wv, h, w, c, np.float32(alpha), np.float32(bound), vp, out)
    return out


def local_blend(cur, prev, nxt, wp, wn):
    squeeze = np.asarray(cur).ndim == 2
    c0, p0, n0 = _hwc(cur), _hwc(prev), _hwc(nxt)
    h, w, c = c0.shape
    out = np.empty_like(c0)
    lib().orc_local_blend(c0, p0, n0, _f32(wp), _f32(wn), h, w, c, out)
    return out[:, :, 0] if squeeze else out


input_blend = local_blend


def adaptive_blend(g, l, wp):
    squeeze = np.asarray(g).ndim == 2
    g0, l0 = _hwc(g), _hwc(l)
    h, w, c = g0.shape
    out = np.empty_like(g0)
    lib().orc_adaptive_blend(g0, l0, _f32(wp), h, w, c, out)
    return out[:, :, 0] if squeeze else out


def consistency_weight(cur, blended, alpha, lam):
    c0, b0 = _hwc(cur), _hwc(blended)
    h, w, c = c0.shape
    out = np.empty((h, w), np.float32)
    lib().orc_consistency_weight(c0, b0, h, w, c, np.float32(alpha), np.float32(lam), out)
    return out


def laplacian(img):
    squeeze = np.asarray(img).ndim == 2
    i0 = _hwc(img)
    h, w, c = i0.shape
    out = np.empty_like(i0)
    lib().orc_laplacian(i0, h, w, c, out)
    return out[:, :, 0] if squeeze else out


def numpy_pairwise_sum(a) -> np.float32:
    a = _f32(a).ravel()
    return np.float32(lib().orc_numpy_pairwise_sum(a, a.size))


def solve_screened_poisson(P, A, wc, params: Params, init=None):
    squeeze = np.asarray(P).ndim == 2
    p0, a0 = _hwc(P), _hwc(A)
    i0 = a0 if init is None else _hwc(init)
    h, w, c = p0.shape
    out = np.empty_like(p0)
    it = ctypes.c_int(0)
    pr = params.c()
    st = lib().orc_solve_screened_poisson(p0, a0, _f32(wc), h, w, c, ctypes.byref(pr), i0, out,
                                          ctypes.byref(it))
    if st == 3:
        raise OracleDivergence(it.value)
    if st != 0:
        raise MemoryError("oracle allocation failed")
    return out[:, :, 0] if squeeze else out


def run_step(I_prev, P_prev, I_cur, P_cur, I_next, P_next, O_prev, flow_prev, flow_next,
             params: Params, want_intermediates: bool = False):
    """One _run_step (consistency.py:368-413) with the two flows given.

    flow_* are (uv, valid) pairs; I_next/P_next/flow_next are None at stream end.
    """
    ip, pp, ic, pc, op = (_hwc(x) for x in (I_prev, P_prev, I_cur, P_cur, O_prev))
    h, w, cin = ic.shape
    cp = pc.shape[2]
    fpu, fpv = _flow(*flow_prev)
    keep = []
    if I_next is not None:
        inx, pnx = _hwc(I_next), _hwc(P_next)
        fnu, fnv = _flow(*flow_next)
        keep += [inx, pnx, fnu, fnv]
        args_next = (inx.ctypes.data, pnx.ctypes.data)
        args_fn = (fnu.ctypes.data, fnv.ctypes.data)
    else:
        args_next = (None, None)
        args_fn = (None, None)
    out = np.empty((h, w, cp), np.float32)
    A = np.empty((h, w, cp), np.float32) if want_intermediates else None
    wc = np.empty((h, w), np.float32) if want_intermediates else None
    it = ctypes.c_int(0)
    pr = params.c()
    st = lib().orc_run_step(h, w, cin, cp, ip, pp, ic, pc, *args_next, op, fpu, fpv, *args_fn,
                            ctypes.byref(pr), out,
                            None if A is None else A.ctypes.data,
                            None if wc is None else wc.ctypes.data, ctypes.byref(it))
    if st == 3:
        raise OracleDivergence(it.value)
    if st != 0:
        raise MemoryError("oracle allocation failed")
    if want_intermediates:
        return out, A, wc
    return out


def constant_flow(h, w, u, v, steps):
    """ConstantFlow.flow_between (flow.py:406-425): (b - a) * (u, v) everywhere."""
    uv = np.empty((h, w, 2), np.float32)
    uv[:, :, 0] = float(u) * steps
    uv[:, :, 1] = float(v) * steps
    return uv, np.ones((h, w), bool)


def stabilize_stream(inputs, processed, params: Params, flow_fn):
    """stabilize_stream (consistency.py:416-433) over lists of frames.

    flow_fn(pos_a, frame_a, pos_b, frame_b) -> (uv, valid).  Yields (pos, O).
    """
    n = len(inputs)
    if n == 0:
        return
    prev_out = _hwc(processed[0])
    yield 1, prev_out
    for t in range(2, n + 1):
        with_next = t < n
        i_prev, p_prev = inputs[t - 2], processed[t - 2]
        i_cur, p_cur = inputs[t - 1], processed[t - 1]
        fprev = flow_fn(t, i_cur, t - 1, i_prev)
        if with_next:
            i_next, p_next = inputs[t], processed[t]
            fnext = flow_fn(t, i_cur, t + 1, i_next)
        else:
            i_next = p_next = fnext = None
        prev_out = run_step(i_prev, p_prev, i_cur, p_cur, i_next, p_next, prev_out, fprev, fnext,
                            params)
        yield t, prev_out
