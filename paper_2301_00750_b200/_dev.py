"""Device plumbing: torch owns device memory and streams; the C ABI does the work."""

from __future__ import annotations

import numpy as np

from . import _lib


class ResolutionMismatch(Exception):
    """Inputs that must share a resolution do not (flow.py:23)."""


class SolverDivergence(Exception):
    """Non-finite iterate appeared during the solve (consistency.py:29-34)."""

    def __init__(self, iteration: int):
        super().__init__(f"solver diverged at iteration {iteration}")
        self.iteration = iteration


_torch = None
_initialised = set()


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2301_00750_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    dev = t.device("cuda", t.cuda.current_device())
    if dev.index not in _initialised:
        check(_lib.lib().ss_init(dev.index))
        _initialised.add(dev.index)
    return dev


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def check(rc: int, iteration: int = 0) -> None:
    if rc == _lib.SS_OK:
        return
    msg = _lib.last_error()
    if rc == _lib.SS_RESOLUTION_MISMATCH:
        raise ResolutionMismatch(msg)
    if rc == _lib.SS_VALUE_ERROR:
        raise ValueError(msg)
    if rc == _lib.SS_SOLVER_DIVERGENCE:
        raise SolverDivergence(iteration)
    if rc == _lib.SS_NO_MEMORY:
        raise MemoryError(msg)
    raise _lib.CudaError(f"{_lib.lib().ss_status_string(rc).decode()}: {msg}")


def is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def to_dev(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (float32 unless dtype given)."""
    t = torch()
    dtype = dtype or t.float32
    dev = device()
    if is_torch(x):
        return x.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(x)
    if not arr.flags.writeable:
        arr = arr.copy()
    return t.from_numpy(arr).to(device=dev, dtype=dtype, non_blocking=False).contiguous()


def ptr(x) -> int | None:
    return None if x is None else x.data_ptr()


def out(like_host: bool, tensor):
    """Return numpy when the caller passed numpy, else the device tensor."""
    if like_host:
        torch().cuda.current_stream().synchronize()
        return tensor.cpu().numpy()
    return tensor


def params_struct(params) -> _lib.SSParams:
    """ConsistencyParams -> ss_params with the reference's float32 casts."""
    return _lib.SSParams(
        np.float32(params.k1), np.float32(params.k2), np.float32(params.alpha),
        np.float32(params.lam), np.float32(params.eta), np.float32(params.kappa),
        int(params.iterations), int(getattr(params, "flow_downscale", 1)))
