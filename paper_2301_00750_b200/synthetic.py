"""Synthetic translating-texture streams (the reference's benchmark input recipe,
synthetic.py:19-75): a smoothed-noise texture that wraps while translating by
an integer (u, v) per frame, and a "stylized" stream = gamma 0.7 + channel mix
+ fresh Gaussian noise per frame (the flicker the stabilizer removes).

``translating_sequence`` builds host frames (numpy); ``DeviceSequence`` builds
the same kind of stream directly in HBM (torch on CUDA) for the benchmark, so
1080p/4K inputs never cross PCIe unless the e2e leg asks for it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_MIX = np.array([[0.7, 0.2, 0.1], [0.1, 0.7, 0.2], [0.2, 0.1, 0.7]], dtype=np.float32)


def _gauss_blur(img: np.ndarray, sigma: float) -> np.ndarray:
    from scipy import ndimage

    return ndimage.gaussian_filter(img, sigma)


def noise_texture(height: int, width: int, rng: np.random.Generator, smoothness: float = 1.5):
    planes = []
    for _ in range(3):
        base = rng.random((height, width)).astype(np.float32)
        s = _gauss_blur(base, smoothness)
        lo, hi = float(s.min()), float(s.max())
        planes.append((s - lo) / (hi - lo))
    return np.stack(planes, axis=2).astype(np.float32)


def stylize(frame: np.ndarray) -> np.ndarray:
    shaped = np.power(np.clip(frame, 0.0, 1.0), 0.7)
    return np.clip(0.1 + 0.8 * (shaped @ _MIX.T), 0.0, 1.0).astype(np.float32)


@dataclass(frozen=True)
class SyntheticSequence:
    inputs: list
    processed: list
    step_u: int
    step_v: int


def translating_sequence(frames: int, height: int = 96, width: int = 128,
                         step: tuple[int, int] = (2, 1), noise_sigma: float = 0.05,
                         seed: int = 0) -> SyntheticSequence:
    rng = np.random.default_rng(seed)
    base = noise_texture(height, width, rng)
    su, sv = step
    inputs, processed = [], []
    for t in range(frames):
        frame = np.roll(base, shift=(t * sv, t * su), axis=(0, 1))
        styled = stylize(frame)
        if noise_sigma > 0.0:
            styled = styled + rng.normal(0.0, noise_sigma, styled.shape).astype(np.float32)
        inputs.append(np.clip(frame, 0.0, 1.0).astype(np.float32))
        processed.append(np.clip(styled, 0.0, 1.0).astype(np.float32))
    return SyntheticSequence(inputs=inputs, processed=processed, step_u=su, step_v=sv)


class DeviceSequence:
    """The same stream generated on the GPU (torch), frame by frame on demand."""

    def __init__(self, height: int, width: int, step=(2, 1), noise_sigma: float = 0.05,
                 seed: int = 0, device=None):
        import torch

        self.torch = torch
        self.h, self.w = height, width
        self.step = step
        self.sigma = noise_sigma
        g = torch.Generator(device="cpu").manual_seed(seed)
        # smoothed noise built at low cost on device: box-blur twice ~ gaussian
        base = torch.rand((3, 1, height, width), generator=g)
        dev = device or torch.device("cuda")
        base = base.to(dev)
        k = torch.ones((1, 1, 5, 5), device=dev) / 25.0
        for _ in range(2):
            base = torch.nn.functional.conv2d(torch.nn.functional.pad(base, (2, 2, 2, 2),
                                                                      mode="circular"), k)
        base = base[:, 0]
        lo = base.amin(dim=(1, 2), keepdim=True)
        hi = base.amax(dim=(1, 2), keepdim=True)
        self.base = ((base - lo) / (hi - lo)).permute(1, 2, 0).contiguous()  # (H, W, 3)
        self.mix = torch.from_numpy(_MIX).to(dev)
        self.gen = torch.Generator(device=dev).manual_seed(seed + 1)
        self.device = dev

    def frame(self, t: int):
        """(input, processed) for stream position t (1-based), both (H, W, 3) f32."""
        torch = self.torch
        su, sv = self.step
        inp = torch.roll(self.base, shifts=((t - 1) * sv, (t - 1) * su), dims=(0, 1))
        styled = 0.1 + 0.8 * (inp.clamp(0, 1).pow(0.7) @ self.mix.T)
        if self.sigma > 0:
            styled = styled + self.sigma * torch.randn(styled.shape, device=self.device,
                                                       generator=self.gen)
        return inp.contiguous(), styled.clamp(0.0, 1.0).contiguous()
