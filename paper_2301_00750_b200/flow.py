"""Flow-side API of the reference (flow.py), on B200.

backward_warp / occlusion_mask run the sm_100a kernels through the C ABI
(ss_backward_warp, ss_occlusion_mask) and accept numpy arrays (returned as
numpy) or torch CUDA tensors (returned as tensors).  Flow providers keep the
reference's FlowProvider seam (flow.py:353-358); providers that can write a
flow straight into a session's device slot implement ``device_flow``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol

import numpy as np

from . import _dev, _lib
from ._dev import ResolutionMismatch
from .imgio import FlowField

__all__ = [
    "ResolutionMismatch", "FlowProvider", "ConstantFlow", "ReplayFlow", "backward_warp",
    "occlusion_mask", "endpoint_error",
]


def _flow_dev(flow: FlowField):
    t = _dev.torch()
    return _dev.to_dev(flow.uv), _dev.to_dev(flow.valid, dtype=t.uint8)


def backward_warp(image, flow: FlowField):
    """flow.py:102-127: sample ``image`` at x + flow(x); returns (warped, mask).

    Bit-identical to the reference (bilinear taps, border clamp, inside & valid).
    """
    host = not _dev.is_torch(image)
    squeeze = len(image.shape) == 2
    img = _dev.to_dev(image)
    if squeeze:
        img = img[:, :, None].contiguous()
    h, w, c = img.shape
    if (flow.height, flow.width) != (h, w):
        raise ResolutionMismatch(f"flow {flow.width}x{flow.height} vs image {w}x{h}")
    uv, valid = _flow_dev(flow)
    t = _dev.torch()
    out = t.empty_like(img)
    mask = t.empty((h, w), device=img.device, dtype=t.float32)
    _dev.check(_lib.lib().ss_backward_warp(img.data_ptr(), h, w, c, uv.data_ptr(),
                                           valid.data_ptr(), out.data_ptr(), mask.data_ptr(),
                                           _dev.stream_ptr()))
    if squeeze:
        out = out[:, :, 0]
    return _dev.out(host, out), _dev.out(host, mask)


def occlusion_mask(forward: FlowField, backward: FlowField):
    """flow.py:130-153: forward-backward consistency mask (bit-exact)."""
    if (forward.height, forward.width) != (backward.height, backward.width):
        raise ResolutionMismatch("flow fields differ in resolution")
    host = not forward.on_device
    fu, fv = _flow_dev(forward)
    bu, bv = _flow_dev(backward)
    h, w = forward.height, forward.width
    t = _dev.torch()
    out = t.empty((h, w), device=fu.device, dtype=t.float32)
    _dev.check(_lib.lib().ss_occlusion_mask(fu.data_ptr(), fv.data_ptr(), bu.data_ptr(),
                                            bv.data_ptr(), h, w, out.data_ptr(),
                                            _dev.stream_ptr()))
    return _dev.out(host, out)


def endpoint_error(pred: FlowField, gt: FlowField) -> float:
    """flow.py:156-165: mean Euclidean distance over jointly valid pixels."""
    if (pred.height, pred.width) != (gt.height, gt.width):
        raise ResolutionMismatch("flow fields differ in resolution")
    p, g = pred.to_host(), gt.to_host()
    valid = p.valid & g.valid
    if not valid.any():
        raise ValueError("no valid pixels for endpoint error")
    diff = p.uv - g.uv
    return float(np.sqrt((diff ** 2).sum(axis=2))[valid].mean())


class FlowProvider(Protocol):
    """Supplies flow from frame at stream position ``pos_a`` to ``pos_b``."""

    def flow_between(self, pos_a: int, frame_a, pos_b: int, frame_b) -> FlowField: ...


class ConstantFlow:
    """flow.py:406-425: uniform flow (b - a) * (u, v).

    GPU-native: ``device_flow`` fills the session's flow slot on device.
    """

    def __init__(self, u: float, v: float):
        self.u = float(u)
        self.v = float(v)
        self.backend_id = f"constant({self.u},{self.v})"

    def flow_between(self, pos_a, frame_a, pos_b, frame_b) -> FlowField:
        h, w = frame_a.shape[:2]
        steps = pos_b - pos_a
        uv = np.empty((h, w, 2), dtype=np.float32)
        uv[:, :, 0] = self.u * steps
        uv[:, :, 1] = self.v * steps
        return FlowField(uv)

    def device_flow(self, session, which: int, pos_a: int, pos_b: int) -> None:
        _dev.check(_lib.lib().ss_set_constant_flow(session, which, self.u, self.v, pos_b - pos_a))


@dataclass(frozen=True)
class FlowOptions:
    """flow.py:27-42 -- tuning knobs of the built-in estimator."""

    levels: int = 5
    patch_size: int = 9
    iterations_per_level: int = 4
    downscale: int = 1

    def __post_init__(self):
        if self.levels < 1:
            raise ValueError("levels must be >= 1")
        if self.patch_size < 3 or self.patch_size % 2 == 0:
            raise ValueError("patch_size must be odd and >= 3")
        if self.downscale not in (1, 2, 4):
            raise ValueError("downscale must be 1, 2 or 4")


def estimate_flow(from_frame, to_frame, opts: FlowOptions = FlowOptions()) -> FlowField:
    """flow.py:168-189: DIS-style coarse-to-fine inverse-search flow from
    ``from_frame`` toward ``to_frame``, on the GPU (csrc/dis.cu)."""
    if tuple(from_frame.shape[:2]) != tuple(to_frame.shape[:2]):
        raise ResolutionMismatch(
            f"frames differ: {tuple(from_frame.shape[:2])} vs {tuple(to_frame.shape[:2])}")
    host = not _dev.is_torch(from_frame)
    a, b = _dev.to_dev(from_frame), _dev.to_dev(to_frame)
    if a.ndim == 2:
        a, b = a[:, :, None].contiguous(), b[:, :, None].contiguous()
    h, w, c = a.shape
    t = _dev.torch()
    uv = t.empty((h, w, 2), device=a.device, dtype=t.float32)
    valid = t.empty((h, w), device=a.device, dtype=t.uint8)
    _dev.check(_lib.lib().ss_dis_flow(a.data_ptr(), b.data_ptr(), h, w, c, opts.levels,
                                      opts.patch_size, opts.iterations_per_level, opts.downscale,
                                      uv.data_ptr(), valid.data_ptr(), _dev.stream_ptr()))
    if host:
        t.cuda.current_stream().synchronize()
        return FlowField(uv.cpu().numpy(), valid.cpu().numpy().astype(bool))
    return FlowField(uv, valid.bool())


class BuiltinFlow:
    """flow.py:361-369: the reference's default provider, on B200.  Inside a
    session the flow is written straight into the session's HBM flow slot."""

    def __init__(self, opts: FlowOptions = FlowOptions()):
        self.opts = opts
        self.backend_id = (f"builtin(levels={opts.levels},patch={opts.patch_size},"
                           f"downscale={opts.downscale})")

    def flow_between(self, pos_a, frame_a, pos_b, frame_b) -> FlowField:
        return estimate_flow(frame_a, frame_b, self.opts)

    def device_flow(self, session, which: int, pos_a: int, pos_b: int) -> None:
        o = self.opts
        _dev.check(_lib.lib().ss_session_compute_dis_flow(session, which, o.levels, o.patch_size,
                                                          o.iterations_per_level, o.downscale))


class ReplayFlow:
    """Returns recorded flows keyed by (pos_a, pos_b) -- the FloDirFlow seam
    (flow.py:372-385) without the disk; used to inject the reference's flows."""

    def __init__(self, table: dict):
        self.table = table
        self.backend_id = "replay"

    def flow_between(self, pos_a, frame_a, pos_b, frame_b) -> FlowField:
        f = self.table[(pos_a, pos_b)]
        return f if isinstance(f, FlowField) else FlowField(*f)
