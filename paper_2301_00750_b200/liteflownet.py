"""Lite optical-flow network ("our-4light-sepref", arXiv 2301.00750 sec. 3.3).

The reference package has no flow CNN (SPEC.md:14 puts it out of scope) and the
paper gives only the compression steps applied to PWC-Net (PAPER.md:506-510,
:847-851, :864-867, :1598-1611): DenseNet connections kept only in the last
two estimator layers ("light"), the quarter-resolution estimator removed
("4" estimators: 1/64 .. 1/8), and separable convolutions in the refinement
("sepref").  The concrete table below is this project's fixed choice, written
down once here and restated independently by the CPU checker:

Feature pyramid (shared by both frames), 3x3 convs + LeakyReLU(0.1):
    L1  8->16 s2, 16->16, 16->16          (input RGB - 0.5, zero channels 3..7)
    L2 16->32 s2, 32->32, 32->32
    L3 32->64 s2, 64->64, 64->64
    L4 64->96 s2, 96->96, 96->96
    L5 96->128 s2, 128->128, 128->128
    L6 128->192 s2, 192->192, 192->192   (PWC-Net uses 196; 192 keeps every width a multiple of 16)
Estimator at level l in (6, 5, 4, 3):
    up   = 2 * bilinear_x2(flow_{l+1})             (l < 6)
    w2   = bilinear warp of f2_l by up (zeros outside)
    x    = [LeakyReLU(corr(f1_l, w2)) 81 | 0 x7 | up 2 | 0 x6 | f1_l C_l]  (l = 6: corr | 0 x7)
    e1 = conv(x, 128); e2 = conv(e1, 128); e3 = conv(e2, 96); e4 = conv(e3, 64)
    e5 = conv([e4, e3], 32);  flow_l = conv([e5, e4], 2)  (no activation)
Refinement at level 3 (depthwise-separable, dilations 1 2 4 8 16 1):
    r_in = [flow_3 2 | 0 x6 | e5 32 | e4 64]
    sep(104->128,d1) sep(128->128,d2) sep(128->128,d4) sep(128->96,d8)
    sep(96->64,d16) sep(64->32,d1), conv3x3(32->2); flow_3 += r
Output: 8 * bilinear_x8(flow_3), cropped to the frame (network input is the
frame replicate-padded to a multiple of 64).  corr(a, b)[d] = sum_c a_c b_c(x+d)
/ C over the 9x9 displacements d in [-4, 4]^2 (row-major dy, dx), zeros
outside; bilinear sampling is at pixel centres (align_corners=False).

Channel groups are padded to multiples of 8 (zero weights), so a 16-byte chunk
of fp32 (4 ch) or bf16 (8 ch) activations never straddles a filter tap.  Weights are random-init (no checkpoint is
available offline) from a seeded generator; ``layer_table()`` fixes the order
in which they are flattened for the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as _lib_mod

PYR_CH = (16, 32, 64, 96, 128, 192)
EST_LEVELS = (6, 5, 4, 3)
MD = 4
N_DISP = (2 * MD + 1) ** 2
LEAKY = 0.1


def pad8(c: int) -> int:
    return (c + 7) // 8 * 8


def est_in_channels(level: int) -> int:
    """Padded channel count of the estimator input x at ``level``."""
    if level == 6:
        return pad8(N_DISP)  # 88
    return pad8(N_DISP) + 8 + PYR_CH[level - 1]


@dataclass(frozen=True)
class Layer:
    name: str
    kind: str          # "conv" (k x k, groups=1) or "dw" (depthwise 3x3)
    cin: int           # padded input channels read
    cout: int          # output channels written
    k: int = 3
    stride: int = 1
    dil: int = 1
    act: bool = True

    @property
    def n_weights(self) -> int:
        if self.kind == "dw":
            return 9 * self.cin
        return self.k * self.k * self.cin * self.cout

    @property
    def fan_in(self) -> int:
        return 9 if self.kind == "dw" else self.k * self.k * self.cin


def layer_table() -> list[Layer]:
    L = []
    cin = 8
    for lvl, c in enumerate(PYR_CH, start=1):
        L.append(Layer(f"pyr{lvl}a", "conv", cin, c, stride=2))
        L.append(Layer(f"pyr{lvl}b", "conv", c, c))
        L.append(Layer(f"pyr{lvl}c", "conv", c, c))
        cin = c
    for lvl in EST_LEVELS:
        x = est_in_channels(lvl)
        L.append(Layer(f"est{lvl}_1", "conv", x, 128))
        L.append(Layer(f"est{lvl}_2", "conv", 128, 128))
        L.append(Layer(f"est{lvl}_3", "conv", 128, 96))
        L.append(Layer(f"est{lvl}_4", "conv", 96, 64))
        L.append(Layer(f"est{lvl}_5", "conv", 64 + 96, 32))
        L.append(Layer(f"est{lvl}_6", "conv", 32 + 64, 2, act=False))
    sep = [(104, 128, 1), (128, 128, 2), (128, 128, 4), (128, 96, 8), (96, 64, 16), (64, 32, 1)]
    for i, (ci, co, d) in enumerate(sep, start=1):
        L.append(Layer(f"ref{i}_dw", "dw", ci, ci, dil=d, act=False))
        L.append(Layer(f"ref{i}_pw", "conv", ci, co, k=1))
    L.append(Layer("ref7", "conv", 32, 2, act=False))
    return L


# logical (unpadded) input channels of a layer's weight rows: rows for the
# zero-padding channels are kept at exactly zero
def _live_rows(layer: Layer) -> np.ndarray:
    live = np.ones(layer.cin, bool)
    n = layer.name
    if n == "pyr1a":
        live[3:] = False
    elif n.startswith("pyr") and n[-1] in "bc":
        live[PYR_CH[int(n[3]) - 1]:] = False
    elif n.startswith("pyr") and n[-1] == "a":
        live[PYR_CH[int(n[3]) - 2]:] = False
    elif n.endswith("_1"):
        live[N_DISP:pad8(N_DISP)] = False
        if n != "est6_1":
            live[pad8(N_DISP) + 2:pad8(N_DISP) + 8] = False
    elif n in ("ref1_dw", "ref1_pw"):
        live[2:8] = False
    return live


def make_weights(seed: int = 0) -> dict:
    """Seeded random init: conv W ~ U(+-sqrt(6 / fan_in)) (Kaiming-uniform for
    the leaky slope), biases U(+-0.01); at this scale the random network emits
    flows of about 0.5-3 pixels on the synthetic streams.  Returns {name: (W, b)} with W laid out
    (k, k, cin, cout) -- dw: (3, 3, cin) -- float32."""
    rng = np.random.default_rng(seed)
    out = {}
    for layer in layer_table():
        bound = np.sqrt(6.0 / layer.fan_in)
        if layer.kind == "dw":
            w = rng.uniform(-bound, bound, (3, 3, layer.cin))
            w[:, :, ~_live_rows(layer)] = 0.0
            b = np.zeros(layer.cin)
        else:
            w = rng.uniform(-bound, bound, (layer.k, layer.k, layer.cin, layer.cout))
            w[:, :, ~_live_rows(layer), :] = 0.0
            b = rng.uniform(-0.01, 0.01, layer.cout)
        out[layer.name] = (w.astype(np.float32), b.astype(np.float32))
    return out


def flatten_weights(weights: dict) -> np.ndarray:
    """Concatenate (W, b) per layer in layer_table() order -- the C ABI layout."""
    parts = []
    for layer in layer_table():
        w, b = weights[layer.name]
        parts.append(np.ascontiguousarray(w, np.float32).ravel())
        parts.append(np.ascontiguousarray(b, np.float32).ravel())
    return np.concatenate(parts)


def n_params() -> int:
    return sum(l.n_weights + (l.cin if l.kind == "dw" else l.cout) for l in layer_table())


class LiteFlowNet:
    """FlowProvider (flow.py:353-358) backed by the lite flow CNN on B200.

    Inside a session (``device_flow``) the network writes the step's flows
    straight into the session's HBM flow slots and caches each ring frame's
    feature pyramid, so a step computes one new pyramid and two estimator
    passes.  ``flow_between`` is the stateless form (FlowField out).
    precision: "fp32" (fp32-class products on tcgen05: split-bf16 -- each
    operand as hi + lo bf16, three products, fp32 accumulation -- on the 3x3
    stride-1 layers, 3xTF32 on the stride-2 and 1x1 ones) or "bf16" (bf16
    operands on tcgen05, fp32 accumulation).
    downscale: FlowOptions.downscale semantics (flow.py:34, :183-188) -- the
    network runs on ``box_downscale(frame, d)`` and the flow is
    ``resize_bilinear``'d back times d; callers pass the preset's
    ``flow_downscale`` (the fast preset: 2), as ``service.py:188`` does for
    the built-in provider.
    """

    def __init__(self, weights: dict | None = None, seed: int = 0, precision: str = "fp32",
                 downscale: int = 1):
        if precision not in ("fp32", "bf16"):
            raise ValueError("precision must be 'fp32' or 'bf16'")
        if downscale not in (1, 2, 4):
            raise ValueError("downscale must be 1, 2 or 4")
        self.weights = weights if weights is not None else make_weights(seed)
        self.precision = precision
        self.downscale = downscale
        self._flat = flatten_weights(self.weights)
        self._nets = {}
        self.backend_id = f"liteflownet(4light-sepref,{precision},downscale={downscale})"

    def handle(self):
        import ctypes

        from . import _dev, _lib

        dev = _dev.device()
        if dev.index not in self._nets:
            L = _lib.lib()
            if int(L.ss_flownet_num_params()) != self._flat.size:
                raise ValueError("weight table does not match the native network")
            h = ctypes.c_void_p()
            prec = _lib.SS_FLOW_FP32 if self.precision == "fp32" else _lib.SS_FLOW_BF16
            _dev.check(L.ss_flownet_create(self._flat.ctypes.data, self._flat.size, prec,
                                           ctypes.byref(h)))
            self._nets[dev.index] = h
            _dev.check(L.ss_flownet_set_downscale(h, self.downscale))
        return self._nets[dev.index]

    def __del__(self):
        lib = _lib_mod._lib
        if lib is None:
            return
        for h in getattr(self, "_nets", {}).values():
            try:
                lib.ss_flownet_destroy(h)
            except Exception:
                pass

    def device_flow(self, session, which: int, pos_a: int, pos_b: int) -> None:
        from . import _dev, _lib

        L = _lib.lib()
        _dev.check(L.ss_session_attach_flownet(session, self.handle()))
        _dev.check(L.ss_session_compute_flow(session, which))

    def flow_between(self, pos_a, frame_a, pos_b, frame_b):
        from . import _dev, _lib
        from .imgio import FlowField

        host = not _dev.is_torch(frame_a)
        a, b = _dev.to_dev(frame_a), _dev.to_dev(frame_b)
        if a.ndim == 2:
            a, b = a[:, :, None].contiguous(), b[:, :, None].contiguous()
        h, w, c = a.shape
        t = _dev.torch()
        uv = t.empty((h, w, 2), device=a.device, dtype=t.float32)
        valid = t.empty((h, w), device=a.device, dtype=t.uint8)
        _dev.check(_lib.lib().ss_flownet_flow(self.handle(), a.data_ptr(), b.data_ptr(), h, w, c,
                                              uv.data_ptr(), valid.data_ptr(), _dev.stream_ptr()))
        if host:
            t.cuda.current_stream().synchronize()
            return FlowField(uv.cpu().numpy(), valid.cpu().numpy().astype(bool))
        return FlowField(uv, valid.bool())
