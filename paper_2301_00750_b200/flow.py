"""Flow-side API of the reference (flow.py), on B200.

backward_warp / occlusion_mask run the sm_100a kernels through the C ABI
(ss_backward_warp, ss_occlusion_mask) and accept numpy arrays (returned as
numpy) or torch CUDA tensors (returned as tensors).  Flow providers keep the
reference's FlowProvider seam (flow.py:353-358); providers that can write a
flow straight into a session's device slot implement ``device_flow``.
"""

from __future__ import annotations

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


class ReplayFlow:
    """Returns recorded flows keyed by (pos_a, pos_b) -- the FloDirFlow seam
    (flow.py:372-385) without the disk; used to inject the reference's flows."""

    def __init__(self, table: dict):
        self.table = table
        self.backend_id = "replay"

    def flow_between(self, pos_a, frame_a, pos_b, frame_b) -> FlowField:
        f = self.table[(pos_a, pos_b)]
        return f if isinstance(f, FlowField) else FlowField(*f)
