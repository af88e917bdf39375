"""Adaptive local/global temporal consistency on B200 (reference: consistency.py).

Same public names, signatures, argument meaning and exceptions as
/root/reference/pkg/src/streamstab/consistency.py; the numpy bodies are
replaced by sm_100a kernels behind the C ABI (include/streamstab_b200.h):

* ``SessionState`` owns an ``ss_session``: the (t-1, t, t+1) ring, O_{t-1},
  flow slots and solver buffers live in HBM; the index logic runs natively.
* ``stabilize_step`` / ``stream_end_step`` = flows (provider seam) + K1 fused
  pre-solve + K2 temporally-blocked solver, one ``ss_step`` call.
* The functional ops (warp_weight, blends, consistency_weight, laplacian,
  solve_screened_poisson) accept numpy (returned as numpy) or CUDA tensors.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, fields, replace
from typing import Mapping

import numpy as np

from . import _dev, _lib
from ._dev import ResolutionMismatch, SolverDivergence
from .flow import FlowProvider, backward_warp
from .imgio import FlowField

__all__ = [
    "ConsistencyParams", "PRESETS", "preset", "SolverDivergence", "StepTiming", "SessionState",
    "stabilize_step", "stream_end_step", "stabilize_stream", "warp_weight", "local_blend",
    "input_blend", "global_warp", "adaptive_blend", "consistency_weight", "laplacian",
    "solve_screened_poisson",
]


@dataclass(frozen=True)
class ConsistencyParams:
    """consistency.py:37-95 -- the full user-tunable consistency state."""

    k1: float = 0.3
    k2: float = 0.5
    alpha: float = 6.5e3
    lam: float = 2.0
    eta: float = 0.15
    kappa: float = 0.2
    iterations: int = 150
    flow_downscale: int = 1

    def validate(self) -> None:
        if not (0.0 <= self.k1 < 1.0 and 0.0 <= self.k2 < 1.0):
            raise ValueError("k1 and k2 must lie in [0, 1)")
        if self.k1 + self.k2 <= 0.0:
            raise ValueError("k1+k2 must be > 0")
        if self.k1 + self.k2 >= 1.0:
            raise ValueError("k1+k2 must be < 1")
        if self.lam < 0.0:
            raise ValueError("lambda must be >= 0")
        if self.eta <= 0.0:
            raise ValueError("eta must be > 0")
        if not (0.0 <= self.kappa < 1.0):
            raise ValueError("kappa must be in [0, 1)")
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if self.flow_downscale not in (1, 2, 4):
            raise ValueError("flow_downscale must be 1, 2 or 4")

    def replace(self, **changes) -> "ConsistencyParams":
        updated = replace(self, **changes)
        updated.validate()
        return updated

    def to_dict(self) -> dict:
        d = {f.name: getattr(self, f.name) for f in fields(self)}
        d["lambda"] = d.pop("lam")
        return d

    @classmethod
    def from_dict(cls, payload: Mapping, base: "ConsistencyParams | None" = None):
        allowed = {f.name for f in fields(cls)}
        changes = {}
        for key, value in payload.items():
            name = "lam" if key == "lambda" else key
            if name not in allowed:
                raise ValueError(f"unknown parameter {key!r}")
            changes[name] = int(value) if name in ("iterations", "flow_downscale") else float(value)
        params = replace(base if base is not None else cls(), **changes)
        params.validate()
        return params


PRESETS: dict[str, ConsistencyParams] = {
    "default": ConsistencyParams(),
    "objective": ConsistencyParams(k1=0.3, k2=0.3, alpha=1.0e4, lam=0.7),
    "fast": ConsistencyParams(flow_downscale=2, iterations=50),
}


def preset(name: str) -> ConsistencyParams:
    try:
        return PRESETS[name]
    except KeyError:
        raise ValueError(f"unknown preset {name!r}; choose from {sorted(PRESETS)}") from None


def _shape_hw(a):
    return tuple(a.shape[:2])


def _check_same_shape(*arrays) -> None:
    shapes = {_shape_hw(a) for a in arrays}
    if len(shapes) != 1:
        raise ResolutionMismatch(f"resolution mismatch: {sorted(shapes)}")


def _check_same_images(*images) -> None:
    shapes = {tuple(img.shape) for img in images}
    if len(shapes) != 1:
        raise ResolutionMismatch(f"image shapes differ: {sorted(shapes)}")


def _hwc(x):
    """to CUDA float32 (H, W, C); returns (tensor, squeeze)"""
    t = _dev.to_dev(x)
    if t.ndim == 2:
        return t[:, :, None].contiguous(), True
    return t, False


# ---------------------------------------------------------------------------
def warp_weight(reference, warped, alpha: float, bound: float, validity=None):
    """consistency.py:133-154: min(bound, exp(-alpha ||ref - warped||^2)) * [validity > 0]."""
    _check_same_images(reference, warped)
    if not (0.0 <= bound < 1.0):
        raise ValueError("bound must lie in [0, 1)")
    host = not _dev.is_torch(reference)
    r, _ = _hwc(reference)
    wv, _ = _hwc(warped)
    h, w, c = r.shape
    vd = None
    if validity is not None:
        _check_same_shape(reference, validity)
        vd = _dev.to_dev(validity)
    t = _dev.torch()
    out = t.empty((h, w), device=r.device, dtype=t.float32)
    _dev.check(_lib.lib().ss_warp_weight(r.data_ptr(), wv.data_ptr(), h, w, c,
                                         np.float32(alpha), np.float32(bound), _dev.ptr(vd),
                                         out.data_ptr(), _dev.stream_ptr()))
    return _dev.out(host, out)


def local_blend(current, warped_prev, warped_next, w_p, w_n):
    """consistency.py:157-171: (1 - (wp + wn)) cur + wp prev + wn next."""
    _check_same_images(current, warped_prev, warped_next)
    _check_same_shape(current, w_p, w_n)
    host = not _dev.is_torch(current)
    cur, sq = _hwc(current)
    pv, _ = _hwc(warped_prev)
    nx, _ = _hwc(warped_next)
    wp, wn = _dev.to_dev(w_p), _dev.to_dev(w_n)
    h, w, c = cur.shape
    out = _dev.torch().empty_like(cur)
    _dev.check(_lib.lib().ss_local_blend(cur.data_ptr(), pv.data_ptr(), nx.data_ptr(),
                                         wp.data_ptr(), wn.data_ptr(), h, w, c, out.data_ptr(),
                                         _dev.stream_ptr()))
    return _dev.out(host, out[:, :, 0] if sq else out)


def input_blend(current_input, warped_input_prev, warped_input_next, w_p, w_n):
    """consistency.py:174-182: local_blend applied to the input frames."""
    return local_blend(current_input, warped_input_prev, warped_input_next, w_p, w_n)


def global_warp(prev_output, flow_to_prev: FlowField):
    """consistency.py:185-187."""
    return backward_warp(prev_output, flow_to_prev)


def adaptive_blend(global_image, local_image, w_p):
    """consistency.py:190-195: wp G + (1 - wp) L."""
    _check_same_images(global_image, local_image)
    _check_same_shape(global_image, w_p)
    host = not _dev.is_torch(global_image)
    g, sq = _hwc(global_image)
    l, _ = _hwc(local_image)
    wp = _dev.to_dev(w_p)
    h, w, c = g.shape
    out = _dev.torch().empty_like(g)
    _dev.check(_lib.lib().ss_adaptive_blend(g.data_ptr(), l.data_ptr(), wp.data_ptr(), h, w, c,
                                            out.data_ptr(), _dev.stream_ptr()))
    return _dev.out(host, out[:, :, 0] if sq else out)


def consistency_weight(current_input, blended_input, alpha: float, lam: float):
    """consistency.py:198-208: lam exp(-alpha ||I - blended I||^2)."""
    _check_same_images(current_input, blended_input)
    if lam < 0.0:
        raise ValueError("lambda must be >= 0")
    host = not _dev.is_torch(current_input)
    a, _ = _hwc(current_input)
    b, _ = _hwc(blended_input)
    h, w, c = a.shape
    t = _dev.torch()
    out = t.empty((h, w), device=a.device, dtype=t.float32)
    _dev.check(_lib.lib().ss_consistency_weight(a.data_ptr(), b.data_ptr(), h, w, c,
                                                np.float32(alpha), np.float32(lam),
                                                out.data_ptr(), _dev.stream_ptr()))
    return _dev.out(host, out)


def laplacian(image):
    """consistency.py:224-227: 5-point Laplacian, replicate boundaries."""
    host = not _dev.is_torch(image)
    img, sq = _hwc(image)
    h, w, c = img.shape
    out = _dev.torch().empty_like(img)
    _dev.check(_lib.lib().ss_laplacian(img.data_ptr(), h, w, c, out.data_ptr(),
                                       _dev.stream_ptr()))
    return _dev.out(host, out[:, :, 0] if sq else out)


def solve_screened_poisson(processed, target, w_c, params: ConsistencyParams, init):
    """consistency.py:253-295: ``params.iterations`` SGD-momentum updates from
    ``init``, clamp to [0, 1]; raises SolverDivergence(j + 1) like the reference."""
    _check_same_images(processed, target, init)
    _check_same_shape(processed, w_c)
    host = not _dev.is_torch(processed)
    p, sq = _hwc(processed)
    a, _ = _hwc(target)
    i0, _ = _hwc(init)
    wc = _dev.to_dev(w_c)
    h, w, c = p.shape
    out = _dev.torch().empty_like(p)
    it = ctypes.c_int(0)
    prm = _dev.params_struct(params)
    rc = _lib.lib().ss_solve_screened_poisson(p.data_ptr(), a.data_ptr(), wc.data_ptr(), h, w,
                                              c, ctypes.byref(prm), i0.data_ptr(), out.data_ptr(),
                                              ctypes.byref(it), _dev.stream_ptr())
    _dev.check(rc, it.value)
    return _dev.out(host, out[:, :, 0] if sq else out)


# ---------------------------------------------------------------------------
@dataclass
class StepTiming:
    """consistency.py:298-303 plus the device split of the step (CUDA events)."""

    flow_ms: float = 0.0
    solve_ms: float = 0.0
    warp_blend_ms: float = 0.0


class SessionState:
    """consistency.py:306-353 -- one-frame-latency stream state, device-resident.

    Push (input, processed) pairs in stream order; once three consecutive pairs
    are buffered ``stabilize_step`` solves the middle one.  The first output is
    pinned to the first processed frame.  ``pairs`` keeps the caller's frame
    references exactly like the reference; the frames themselves are copied
    into the session's HBM ring on push.
    """

    def __init__(self, params: ConsistencyParams, pairs=None, prev_output=None,
                 solved_through: int = 0, last_timing: StepTiming | None = None):
        self.params = params
        self.pairs: list = []
        self.last_timing = last_timing or StepTiming()
        self._handle = None
        self._shapes = None  # (input shape, processed shape)
        self._first_output = None
        self._out_cache = None
        self._squeeze = False
        self._flow0_for = None  # step whose flow t -> t-1 was started early
        self._inflight: list = []  # device push sources, alive until the next step
        # the reference's dataclass fields (consistency.py:305-319) may be set
        # at construction or assigned later (resume from a known O_{t-1}):
        # held here until the device session exists (first push)
        self._has_prev = prev_output is not None
        self._pending_prev = prev_output
        self._pending_st = int(solved_through)
        for pos, i, p in (pairs or []):
            # pre-filled pairs are buffered as given; prev_output /
            # solved_through stay what the caller passed (no pinning)
            self.push_pair(pos, i, p, _pin=False)

    # -- device session ------------------------------------------------------
    def _ensure_session(self, input_frame, processed_frame):
        if self._handle is not None:
            return
        _dev.device()
        h, w = _shape_hw(input_frame)
        ci = 1 if len(input_frame.shape) == 2 else int(input_frame.shape[2])
        cp = 1 if len(processed_frame.shape) == 2 else int(processed_frame.shape[2])
        handle = ctypes.c_void_p()
        _dev.check(_lib.lib().ss_session_create(h, w, ci, cp, ctypes.c_void_p(_dev.stream_ptr()),
                                                ctypes.byref(handle)))
        self._handle = handle
        self._squeeze = len(processed_frame.shape) == 2

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib.lib().ss_session_destroy(h)
            except Exception:
                pass
            self._handle = None

    @property
    def handle(self):
        return self._handle

    @property
    def solved_through(self) -> int:
        if self._handle is None:
            return self._pending_st
        return int(_lib.lib().ss_solved_through(self._handle))

    @solved_through.setter
    def solved_through(self, value: int) -> None:
        if self._handle is None:
            self._pending_st = int(value)
            return
        _dev.check(_lib.lib().ss_session_set_state(self._handle, _lib.SS_STATE_POSITION, int(value), None, 0, 0))
        self._flow0_for = None

    @property
    def prev_output(self):
        """O_{solved_through}: the pushed P_1 object itself until the first step
        (or the object assigned to it)."""
        if not self._has_prev:
            return None
        if self._handle is None:
            return self._pending_prev
        if self._first_output is not None:
            return self._first_output
        if self._out_cache is None:
            self._out_cache = self.output_host()
        return self._out_cache

    @prev_output.setter
    def prev_output(self, value) -> None:
        self._has_prev = value is not None
        self._out_cache = None
        self._first_output = None
        if self._handle is None:
            self._pending_prev = value
            return
        self._set_device_prev(value, self.solved_through)

    def _set_device_prev(self, value, solved_through: int) -> None:
        L = _lib.lib()
        self._flow0_for = None
        if value is None:
            _dev.check(L.ss_session_set_state(self._handle, _lib.SS_STATE_CLEAR, int(solved_through), None, 0, 0))
            return
        if tuple(value.shape) != tuple(self._shapes[1]):
            raise ResolutionMismatch("prev_output does not match the processed frames")
        if _dev.is_torch(value) and value.is_cuda:
            v = _dev.to_dev(value)
            _dev.check(L.ss_session_wait_stream(self._handle, _dev.stream_ptr()))
            _dev.check(L.ss_session_set_state(self._handle, _lib.SS_STATE_OUTPUT, int(solved_through),
                                              ctypes.c_void_p(v.data_ptr()), _lib.SS_F32, _lib.SS_DEVICE))
            self._inflight.append(v)
        else:
            v = np.ascontiguousarray(np.asarray(value), dtype=np.float32)
            _dev.check(L.ss_session_set_state(self._handle, _lib.SS_STATE_OUTPUT, int(solved_through),
                                              v.ctypes.data_as(ctypes.c_void_p), _lib.SS_F32, _lib.SS_HOST))
        self._first_output = value  # the reference keeps the assigned object

    def output_host(self) -> np.ndarray:
        h, w, c = self._out_shape()
        out = np.empty((h, w, c), np.float32)
        _dev.check(_lib.lib().ss_output(self._handle, out.ctypes.data, _lib.SS_F32, _lib.SS_HOST))
        return out[:, :, 0] if self._squeeze else out

    def output_u8(self) -> np.ndarray:
        """The current output quantized on the device as the reference's
        writers do: rint(clip(O, 0, 1) * 255) -> uint8 (imgio.py:132,
        service.py:101-102)."""
        h, w, c = self._out_shape()
        out = np.empty((h, w, c), np.uint8)
        _dev.check(_lib.lib().ss_output(self._handle, out.ctypes.data, _lib.SS_U8, _lib.SS_HOST))
        return out[:, :, 0] if self._squeeze else out

    def output_device(self):
        """The current output as a CUDA tensor (copy)."""
        t = _dev.torch()
        h, w, c = self._out_shape()
        out = t.empty((h, w, c), device=_dev.device(), dtype=t.float32)
        _dev.check(_lib.lib().ss_output(self._handle, out.data_ptr(), _lib.SS_F32,
                                        _lib.SS_DEVICE))
        return out[:, :, 0] if self._squeeze else out

    def _out_shape(self):
        ps = self._shapes[1]
        return ps[0], ps[1], (1 if len(ps) == 2 else ps[2])

    # -- consistency.py:321-340 ---------------------------------------------
    def push_pair(self, position: int, input_frame, processed_frame, _pin: bool = True) -> None:
        if _shape_hw(input_frame) != _shape_hw(processed_frame):
            raise ResolutionMismatch("input and processed frames differ in resolution")
        if self.pairs:
            if position != self.pairs[-1][0] + 1:
                raise ValueError(
                    f"non-consecutive frame position {position} after {self.pairs[-1][0]}")
            if tuple(input_frame.shape) != tuple(self.pairs[-1][1].shape):
                raise ResolutionMismatch("resolution drift mid-stream")
            if tuple(processed_frame.shape) != tuple(self.pairs[-1][2].shape):
                raise ResolutionMismatch("resolution drift mid-stream")
        elif self._shapes is not None and (
                tuple(input_frame.shape) != self._shapes[0]
                or tuple(processed_frame.shape) != self._shapes[1]):
            raise ResolutionMismatch("resolution drift mid-stream")
        created = self._handle is None
        self._ensure_session(input_frame, processed_frame)
        if self._shapes is None:
            self._shapes = (tuple(input_frame.shape), tuple(processed_frame.shape))
        if created:
            # state assigned before the session existed (consistency.py:305-319)
            if self._has_prev:
                self._set_device_prev(self._pending_prev, self._pending_st)
            elif self._pending_st:
                _dev.check(_lib.lib().ss_session_set_state(self._handle, _lib.SS_STATE_POSITION,
                                                           self._pending_st, None, 0, 0))
            self._pending_prev = None
        first = not self._has_prev
        self._push_device(position, input_frame, processed_frame)
        self.pairs.append((position, input_frame, processed_frame))
        if len(self.pairs) > 3:
            self.pairs.pop(0)
        if first and not _pin:
            # pre-filled pairs (constructor): the device pinned O to this pair
            # as a push does; the reference leaves prev_output / solved_through
            _dev.check(_lib.lib().ss_session_set_state(self._handle, _lib.SS_STATE_CLEAR, self._pending_st,
                                                       None, 0, 0))
        elif first:
            # the first output *is* the pushed P_1 object (consistency.py:338-340);
            # an 8-bit frame is stored as its float32 load (x / 255), read back
            self._has_prev = True
            self._first_output = None if _is_u8(processed_frame) else processed_frame

    def _push_device(self, position, input_frame, processed_frame):
        L = _lib.lib()
        if _is_u8(input_frame) and _is_u8(processed_frame):
            # 8-bit frames (the live path's decoded PNG/PPM bytes): the device
            # widens them exactly as imgio.load_frame does (uint8 / 255 in
            # float32, imgio.py:72) -- 4x less host->device traffic
            if _dev.is_torch(input_frame):
                i, p = input_frame.contiguous(), processed_frame.contiguous()
                where = _lib.SS_DEVICE if i.is_cuda else _lib.SS_HOST
                if where == _lib.SS_DEVICE:
                    _dev.check(L.ss_session_wait_stream(self._handle, _dev.stream_ptr()))
                    self._inflight.append((i, p))
                _dev.check(L.ss_push_pair(self._handle, position, i.data_ptr(), p.data_ptr(),
                                          _lib.SS_U8, where))
                if where == _lib.SS_HOST:  # pageable host copies complete before return
                    _dev.check(L.ss_session_signal_stream(self._handle, _dev.stream_ptr()))
            else:
                i = np.ascontiguousarray(input_frame)
                p = np.ascontiguousarray(processed_frame)
                _dev.check(L.ss_push_pair(self._handle, position, i.ctypes.data, p.ctypes.data,
                                          _lib.SS_U8, _lib.SS_HOST))
            return
        if _dev.is_torch(input_frame) and input_frame.is_cuda:
            i = _dev.to_dev(input_frame)
            p = _dev.to_dev(processed_frame)
            # the sources (and any converted temporaries) come from torch's
            # current stream: the session stream waits for it before copying
            _dev.check(L.ss_session_wait_stream(self._handle, _dev.stream_ptr()))
            _dev.check(L.ss_push_pair(self._handle, position, i.data_ptr(), p.data_ptr(),
                                      _lib.SS_F32, _lib.SS_DEVICE))
            # the copy is stream-ordered on the session stream: keep the
            # sources referenced until the next step, which waits for that
            # stream -- no host wait here
            self._inflight.append((i, p))
        else:
            i = np.ascontiguousarray(np.asarray(input_frame), dtype=np.float32)
            p = np.ascontiguousarray(np.asarray(processed_frame), dtype=np.float32)
            _dev.check(L.ss_push_pair(self._handle, position, i.ctypes.data, p.ctypes.data,
                                      _lib.SS_F32, _lib.SS_HOST))

    def _snippet(self, want_next: bool) -> int:
        if self._handle is None:
            raise ValueError("no buffered frames")
        t = ctypes.c_int64(0)
        _dev.check(_lib.lib().ss_check_step(self._handle, int(want_next), ctypes.byref(t)))
        return int(t.value)


def _is_u8(x) -> bool:
    dt = getattr(x, "dtype", None)
    return dt is not None and str(dt) in ("uint8", "torch.uint8")


def _provide_flow(state: SessionState, flow_backend, which: int, t: int, other: int):
    """FlowProvider.flow_between(t, I_t, other, I_other) into the session slot."""
    by_pos = {p: i for p, i, _ in state.pairs}
    if hasattr(flow_backend, "device_flow"):
        flow_backend.device_flow(state.handle, which, t, other)
        return
    f = flow_backend.flow_between(t, by_pos[t], other, by_pos[other])
    h, w = state._shapes[0][:2]
    if (f.height, f.width) != (h, w):
        raise ResolutionMismatch(f"flow {f.width}x{f.height} vs image {w}x{h}")
    L = _lib.lib()
    if getattr(f, "on_device", False):
        uv = f.uv.to(_dev.torch().float32).contiguous()
        vd = f.valid.to(_dev.torch().uint8).contiguous()
        # produced on torch's current stream: the session copies after it,
        # and torch's stream (which may reuse the temporaries once they are
        # dropped) continues only after the copies
        sp = _dev.stream_ptr()
        _dev.check(L.ss_session_wait_stream(state.handle, sp))
        _dev.check(L.ss_set_flow(state.handle, which, uv.data_ptr(), vd.data_ptr(),
                                 _lib.SS_DEVICE))
        _dev.check(L.ss_session_signal_stream(state.handle, sp))
    else:
        uv = np.ascontiguousarray(f.uv, dtype=np.float32)
        vd = np.ascontiguousarray(f.valid, dtype=np.uint8)
        _dev.check(L.ss_set_flow(state.handle, which, uv.ctypes.data, vd.ctypes.data,
                                 _lib.SS_HOST))


def _start_flow_to_prev(state: SessionState, flow_backend) -> None:
    """Start the pending step's flow t -> t-1 before the next pair is pushed.

    It needs only frames already buffered; with a device-native provider it
    runs on the session's side stream, so the host->device copy of the next
    pair overlaps it.  _run_step then skips it (pure scheduling: same flow).
    """
    if not hasattr(flow_backend, "device_flow") or state.handle is None:
        return
    t = state.solved_through + 1
    if not any(p == t - 1 for p, _, _ in state.pairs) or not any(p == t for p, _, _ in state.pairs):
        return
    _provide_flow(state, flow_backend, 0, t, t - 1)
    state._flow0_for = t


def _run_step(state: SessionState, flow_backend, with_next: bool, return_host: bool = True):
    t = state._snippet(want_next=with_next)
    params = state.params
    t0 = time.perf_counter()
    if state._flow0_for != t:
        _provide_flow(state, flow_backend, 0, t, t - 1)
    state._flow0_for = None
    if with_next:
        _provide_flow(state, flow_backend, 1, t, t + 1)
    flow_ms = (time.perf_counter() - t0) * 1e3
    it = ctypes.c_int(0)
    prm = _dev.params_struct(params)
    t1 = time.perf_counter()
    rc = _lib.lib().ss_step(state.handle, int(with_next), ctypes.byref(prm), ctypes.byref(it))
    state._inflight.clear()  # ss_step waited for the session stream (pushes included)
    _dev.check(rc, it.value)
    solve_ms = (time.perf_counter() - t1) * 1e3
    tm = _lib.SSTiming()
    _lib.lib().ss_last_timing(state.handle, ctypes.byref(tm))
    state._first_output = None
    state._out_cache = None
    # device (CUDA-event) times when available: the flow network's kernels
    # run asynchronously, so the host clock around the provider calls would
    # only see the launches
    state.last_timing = StepTiming(
        flow_ms=float(tm.flow_ms) if tm.flow_ms > 0 else flow_ms,
        solve_ms=float(tm.solve_ms) if tm.solve_ms > 0 else solve_ms,
        warp_blend_ms=float(tm.warp_blend_ms))
    if not return_host:
        return state.output_device()
    out = state.output_host()
    state._out_cache = out
    return out


def stabilize_step(state: SessionState, flow_backend: FlowProvider):
    """consistency.py:356-359: solve the next pending frame with both neighbours."""
    return _run_step(state, flow_backend, with_next=True)


def stream_end_step(state: SessionState, flow_backend: FlowProvider):
    """consistency.py:362-365: final frame; next-frame terms drop out."""
    return _run_step(state, flow_backend, with_next=False)


def stabilize_stream(pairs, params: ConsistencyParams, flow_backend: FlowProvider):
    """consistency.py:416-433: yields (position, stabilized frame), one-frame latency."""
    state = SessionState(params=params)
    position = 0
    for input_frame, processed_frame in pairs:
        position += 1
        if position >= 3:
            _start_flow_to_prev(state, flow_backend)
        state.push_pair(position, input_frame, processed_frame)
        if position == 1:
            yield 1, state.prev_output
        elif position >= 3:
            yield position - 1, stabilize_step(state, flow_backend)
    if position >= 2:
        yield position, stream_end_step(state, flow_backend)
