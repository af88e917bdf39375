"""Evaluation metrics on B200 (reference: metrics.py) -- SURVEY §8(f3), (f4).

``warping_error_pair`` / ``warping_error`` (metrics.py:107-151): the
occlusion-masked temporal warping error E_warp, computed by one fused kernel
(occlusion mask + backward warp + masked channel-mean L1, float64 sums).
``ssim`` / ``ssim_report`` (metrics.py:75-104, :154-163): single-scale luma
SSIM in float64.  Same names, arguments, return values and errors as the
reference; frames may be numpy or CUDA tensors.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from ._dev import ResolutionMismatch

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5


@dataclass
class MetricReport:
    """metrics.py:28-66: per-frame values and their mean."""

    name: str
    per_frame: list
    skipped: list = field(default_factory=list)
    preset: str | None = None
    flow_backend: str | None = None

    @property
    def mean(self) -> float:
        if not self.per_frame:
            return math.nan
        return float(np.mean([v for _, v in self.per_frame]))

    @property
    def count(self) -> int:
        return len(self.per_frame)

    def summary(self) -> dict:
        return {"metric": self.name, "mean": self.mean, "count": self.count,
                "skipped": self.skipped, "preset": self.preset,
                "flow_backend": self.flow_backend}


def _frame(x):
    t = _dev.to_dev(x)
    return t[:, :, None].contiguous() if t.ndim == 2 else t


def _flow(f):
    t = _dev.torch()
    return _dev.to_dev(f.uv), _dev.to_dev(f.valid, dtype=t.uint8)


def warping_error_pair(frame_a, frame_b, pos_a: int, pos_b: int, flow_backend):
    """metrics.py:107-128: occlusion-masked mean L1 between frame a and warped
    frame b; None when every pixel is masked out."""
    forward = flow_backend.flow_between(pos_a, frame_a, pos_b, frame_b)
    backward = flow_backend.flow_between(pos_b, frame_b, pos_a, frame_a)
    if (forward.height, forward.width) != (backward.height, backward.width):
        raise ResolutionMismatch("flow fields differ in resolution")
    a, b = _frame(frame_a), _frame(frame_b)
    h, w, c = a.shape
    if (forward.height, forward.width) != (h, w):
        raise ResolutionMismatch(f"flow {forward.width}x{forward.height} vs image {w}x{h}")
    fu, fv = _flow(forward)
    bu, bv = _flow(backward)
    sums = (ctypes.c_double * 2)()
    _dev.check(_lib.lib().ss_warping_error_sums(a.data_ptr(), b.data_ptr(), h, w, c,
                                                fu.data_ptr(), fv.data_ptr(), bu.data_ptr(),
                                                bv.data_ptr(), sums, _dev.stream_ptr()))
    if sums[1] == 0.0:
        return None
    return float(sums[0] / sums[1])


def warping_error(frames, flow_backend) -> MetricReport:
    """metrics.py:131-151: E_warp over consecutive frames (indexed by the
    earlier frame's 1-based position)."""
    report = MetricReport(name="ewarp", per_frame=[],
                          flow_backend=getattr(flow_backend, "backend_id", None))
    prev = None
    pos = 0
    for frame in frames:
        pos += 1
        if prev is not None:
            value = warping_error_pair(prev, frame, pos - 1, pos, flow_backend)
            if value is None:
                report.skipped.append(pos - 1)
            else:
                report.per_frame.append((pos - 1, value))
        prev = frame
    if pos < 2:
        raise ValueError("warping error needs at least 2 frames")
    return report


def ssim(a, b) -> float:
    """metrics.py:75-104: luma SSIM, 11x11 Gaussian (sigma 1.5), reflect borders,
    half-window crop, float64."""
    if tuple(a.shape[:2]) != tuple(b.shape[:2]):
        raise ResolutionMismatch(f"{tuple(a.shape[:2])} vs {tuple(b.shape[:2])}")
    h, w = a.shape[:2]
    if h < SSIM_WINDOW or w < SSIM_WINDOW:
        raise ValueError(f"image {w}x{h} smaller than the {SSIM_WINDOW}x{SSIM_WINDOW} window")
    x, y = _frame(a), _frame(b)
    if x.shape[2] != y.shape[2]:
        raise ResolutionMismatch("channel counts differ")
    out = ctypes.c_double(0.0)
    _dev.check(_lib.lib().ss_ssim(x.data_ptr(), y.data_ptr(), h, w, x.shape[2],
                                  ctypes.byref(out), _dev.stream_ptr()))
    return float(out.value)


def ssim_report(candidate_frames, reference_frames) -> MetricReport:
    """metrics.py:154-163: per-frame SSIM of two aligned sequences."""
    report = MetricReport(name="ssim", per_frame=[])
    pos = 0
    for cand, ref in zip(candidate_frames, reference_frames, strict=True):
        pos += 1
        report.per_frame.append((pos, ssim(cand, ref)))
    if pos == 0:
        raise ValueError("empty sequences")
    return report
