"""Boundary data types of the reference (imgio.py:33-46, :154-192).

Frames are float32 (H, W, C), C in {1, 3}, values in [0, 1]; flow fields are
float32 (H, W, 2) with u horizontal and v vertical plus a boolean validity map
where |component| > 1e9 marks unknown flow (Middlebury convention).  A
FlowField here may hold numpy arrays (host) or torch CUDA tensors (device);
the device form never round-trips through the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FLO_INVALID_THRESHOLD = 1e9


def as_frame(data) -> np.ndarray:
    """imgio.as_frame (imgio.py:33-46): float32, (H, W, C), C in {1, 3}, read-only."""
    arr = np.asarray(data, dtype=np.float32)
    if arr.ndim == 2:
        arr = arr[:, :, None]
    if arr.ndim != 3 or arr.shape[2] not in (1, 3):
        raise ValueError(f"frame must be (H, W, 1|3), got shape {arr.shape}")
    if arr.shape[0] == 0 or arr.shape[1] == 0:
        raise ValueError("zero-sized frame")
    if not np.all(np.isfinite(arr)):
        raise ValueError("frame contains non-finite values")
    arr = np.clip(arr, 0.0, 1.0)
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class FlowField:
    """Dense displacement + validity (imgio.py:154-192).

    ``uv`` is (H, W, 2) float32, ``valid`` (H, W) bool.  Either both numpy
    (host) or both torch CUDA tensors (device).
    """

    uv: object
    valid: object = field(default=None)

    def __post_init__(self):
        uv = self.uv
        if _is_torch(uv):
            import torch

            uv = uv.to(torch.float32).contiguous()
            if uv.ndim != 3 or uv.shape[2] != 2:
                raise ValueError(f"flow must be (H, W, 2), got {tuple(uv.shape)}")
            valid = self.valid
            if valid is None:
                valid = uv.abs().amax(dim=2) <= FLO_INVALID_THRESHOLD
            valid = valid.to(device=uv.device, dtype=torch.bool).contiguous()
            if tuple(valid.shape) != tuple(uv.shape[:2]):
                raise ValueError("validity mask shape mismatch")
        else:
            uv = np.asarray(uv, dtype=np.float32)
            if uv.ndim != 3 or uv.shape[2] != 2:
                raise ValueError(f"flow must be (H, W, 2), got {uv.shape}")
            valid = self.valid
            if valid is None:
                valid = np.abs(uv).max(axis=2) <= FLO_INVALID_THRESHOLD
            valid = np.ascontiguousarray(valid, dtype=bool)
            if valid.shape != uv.shape[:2]:
                raise ValueError("validity mask shape mismatch")
            uv = np.ascontiguousarray(uv)
            uv.flags.writeable = False
            valid.flags.writeable = False
        object.__setattr__(self, "uv", uv)
        object.__setattr__(self, "valid", valid)

    @property
    def height(self) -> int:
        return int(self.uv.shape[0])

    @property
    def width(self) -> int:
        return int(self.uv.shape[1])

    @property
    def on_device(self) -> bool:
        return _is_torch(self.uv)

    @staticmethod
    def zero(height: int, width: int) -> "FlowField":
        return FlowField(np.zeros((height, width, 2), dtype=np.float32))

    def to_host(self) -> "FlowField":
        if not self.on_device:
            return self
        return FlowField(self.uv.cpu().numpy(), self.valid.cpu().numpy())


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")
