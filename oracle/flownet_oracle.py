"""CPU restatement of the lite flow network -- TEST INFRASTRUCTURE ONLY.

Independent numpy restatement of the architecture documented in
paper_2301_00750_b200/liteflownet.py (the reference package has no flow CNN:
SPEC.md:14; paper PAPER.md:506-510, :847-867, :1598-1611).  It shares only the
weight dictionary with the product (weights are inputs, like frames).
Accumulation is float64, every layer output is rounded to float32 (the GPU
fp32 path's storage precision).  Parity for this path is therefore pinned to
this restatement, not to reference outputs ("parity unpinned" at the
reference).
"""

from __future__ import annotations

import numpy as np

PYR_CH = (16, 32, 64, 96, 128, 192)
MD = 4
LEAKY = 0.1


def _leaky(x):
    return np.where(x >= 0, x, LEAKY * x)


def prep(img):
    """(H, W, C) in [0, 1] -> (H64, W64, 8): RGB - 0.5, replicate pad, zero ch 3..7."""
    img = np.asarray(img, np.float32)
    if img.ndim == 2:
        img = img[:, :, None]
    if img.shape[2] == 1:
        img = np.repeat(img, 3, axis=2)
    h, w = img.shape[:2]
    H, W = -(-h // 64) * 64, -(-w // 64) * 64
    ys = np.minimum(np.arange(H), h - 1)
    xs = np.minimum(np.arange(W), w - 1)
    out = np.zeros((H, W, 8), np.float32)
    out[:, :, :3] = img[ys][:, xs] - np.float32(0.5)
    return out


def conv(x, w, b, stride=1, dil=1, act=True):
    """k x k conv, zero padding dil * (k // 2), float64 accumulation."""
    k = w.shape[0]
    H, W, C = x.shape
    pad = dil * (k // 2)
    Ho = (H + 2 * pad - dil * (k - 1) - 1) // stride + 1
    Wo = (W + 2 * pad - dil * (k - 1) - 1) // stride + 1
    xp = np.zeros((H + 2 * pad, W + 2 * pad, C), np.float64)
    xp[pad:pad + H, pad:pad + W] = x
    acc = np.zeros((Ho, Wo, w.shape[3]), np.float64) + b.astype(np.float64)
    for ky in range(k):
        for kx in range(k):
            sl = xp[ky * dil: ky * dil + stride * (Ho - 1) + 1: stride,
                    kx * dil: kx * dil + stride * (Wo - 1) + 1: stride]
            acc += (sl.reshape(-1, C) @ w[ky, kx].astype(np.float64)).reshape(Ho, Wo, -1)
    if act:
        acc = _leaky(acc)
    return acc.astype(np.float32)


def depthwise(x, w, dil):
    H, W, C = x.shape
    pad = dil
    xp = np.zeros((H + 2 * pad, W + 2 * pad, C), np.float64)
    xp[pad:pad + H, pad:pad + W] = x
    acc = np.zeros((H, W, C), np.float64)
    for ky in range(3):
        for kx in range(3):
            acc += xp[ky * dil: ky * dil + H, kx * dil: kx * dil + W] * w[ky, kx].astype(np.float64)
    return acc.astype(np.float32)


def corr(f1, f2):
    """[d] = sum_c f1 * f2(x + d) / C, d in [-4, 4]^2 (dy-major), zeros outside."""
    H, W, C = f1.shape
    p = np.zeros((H + 2 * MD, W + 2 * MD, C), np.float64)
    p[MD:MD + H, MD:MD + W] = f2
    out = np.empty((H, W, (2 * MD + 1) ** 2), np.float64)
    a = f1.astype(np.float64)
    i = 0
    for dy in range(-MD, MD + 1):
        for dx in range(-MD, MD + 1):
            out[:, :, i] = (a * p[MD + dy:MD + dy + H, MD + dx:MD + dx + W]).sum(axis=2) / C
            i += 1
    return out.astype(np.float32)


def _bilinear_resize(x, Ho, Wo):
    """align_corners=False bilinear, negative source coords clamped to 0."""
    H, W = x.shape[:2]
    sy = np.maximum((np.arange(Ho) + 0.5) * (H / Ho) - 0.5, 0.0)
    sx = np.maximum((np.arange(Wo) + 0.5) * (W / Wo) - 0.5, 0.0)
    y0 = np.floor(sy).astype(int)
    x0 = np.floor(sx).astype(int)
    y1 = np.minimum(y0 + 1, H - 1)
    x1 = np.minimum(x0 + 1, W - 1)
    fy = (sy - y0)[:, None, None]
    fx = (sx - x0)[None, :, None]
    x = x.astype(np.float64)
    top = x[y0][:, x0] * (1 - fx) + x[y0][:, x1] * fx
    bot = x[y1][:, x0] * (1 - fx) + x[y1][:, x1] * fx
    return top * (1 - fy) + bot * fy


def warp_zero(f, uv):
    """Bilinear sample f at (x + u, y + v); taps outside the grid contribute 0."""
    H, W, C = f.shape
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    sx = xx + uv[:, :, 0].astype(np.float64)
    sy = yy + uv[:, :, 1].astype(np.float64)
    x0 = np.floor(sx).astype(int)
    y0 = np.floor(sy).astype(int)
    fx = (sx - x0)[:, :, None]
    fy = (sy - y0)[:, :, None]
    out = np.zeros((H, W, C), np.float64)
    for dy, wy in ((0, 1 - fy), (1, fy)):
        for dx, wx in ((0, 1 - fx), (1, fx)):
            ty, tx = y0 + dy, x0 + dx
            ok = (ty >= 0) & (ty < H) & (tx >= 0) & (tx < W)
            v = f[np.clip(ty, 0, H - 1), np.clip(tx, 0, W - 1)].astype(np.float64)
            out += np.where(ok[:, :, None], v, 0.0) * wy * wx
    return out.astype(np.float32)


def pyramid(weights, img):
    x = prep(img)
    feats = []
    for lvl in range(1, 7):
        for s, tag in ((2, "a"), (1, "b"), (1, "c")):
            w, b = weights[f"pyr{lvl}{tag}"]
            x = conv(x, w, b, stride=s)
        feats.append(x)
    return feats  # index l-1 -> level l


def box_downscale(arr, f):
    """Restates reference flow.py:69-80: integer box average, remainder cropped."""
    arr = np.asarray(arr, np.float32)
    if f == 1:
        return arr
    h2, w2 = arr.shape[0] // f * f, arr.shape[1] // f * f
    c = arr[:h2, :w2]
    v = c.reshape(h2 // f, f, w2 // f, f, *c.shape[2:])
    return v.mean(axis=(1, 3), dtype=np.float32)


def resize_bilinear(arr, shape):
    """Restates reference flow.py:54-66 (+ _bilinear_gather :83-99): pixel
    centres, border clamp, float32."""
    arr = np.asarray(arr, np.float32)
    ih, iw = arr.shape[:2]
    oh, ow = shape
    if (ih, iw) == (oh, ow):
        return arr.copy()
    ys = (np.arange(oh, dtype=np.float32) + 0.5) * (ih / oh) - 0.5
    xs = (np.arange(ow, dtype=np.float32) + 0.5) * (iw / ow) - 0.5
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    yy = np.clip(yy, 0.0, ih - 1.0)
    xx = np.clip(xx, 0.0, iw - 1.0)
    y0, x0 = np.floor(yy).astype(np.intp), np.floor(xx).astype(np.intp)
    y1, x1 = np.minimum(y0 + 1, ih - 1), np.minimum(x0 + 1, iw - 1)
    fy = (yy - y0).astype(np.float32)[..., None]
    fx = (xx - x0).astype(np.float32)[..., None]
    top = arr[y0, x0] * (1 - fx) + arr[y0, x1] * fx
    bot = arr[y1, x0] * (1 - fx) + arr[y1, x1] * fx
    return (top * (1 - fy) + bot * fy).astype(np.float32)


def flow(weights, img1, img2, pyr1=None, pyr2=None, downscale=1):
    """Flow from img1 toward img2 (FlowProvider.flow_between(t, I_t, b, I_b)):
    (H, W, 2) float32, u horizontal, v vertical, in full-resolution pixels.
    downscale d: the network on box_downscale(frame, d), the flow resized back
    times d -- the provider-level FlowOptions.downscale of flow.py:183-188."""
    if downscale != 1:
        h, w = np.asarray(img1).shape[:2]
        small = flow(weights, box_downscale(img1, downscale), box_downscale(img2, downscale))
        return resize_bilinear(small, (h, w)) * np.float32(downscale)
    h, w = np.asarray(img1).shape[:2]
    p1 = pyr1 or pyramid(weights, img1)
    p2 = pyr2 or pyramid(weights, img2)
    fl = None
    for lvl in (6, 5, 4, 3):
        f1, f2 = p1[lvl - 1], p2[lvl - 1]
        H, W, C = f1.shape
        if lvl == 6:
            x = np.zeros((H, W, 88), np.float32)
            x[:, :, :81] = _leaky(corr(f1, f2))
        else:
            up = (2.0 * _bilinear_resize(fl, H, W)).astype(np.float32)
            w2 = warp_zero(f2, up)
            x = np.zeros((H, W, 96 + C), np.float32)
            x[:, :, :81] = _leaky(corr(f1, w2))
            x[:, :, 88:90] = up
            x[:, :, 96:] = f1
        e1 = conv(x, *weights[f"est{lvl}_1"])
        e2 = conv(e1, *weights[f"est{lvl}_2"])
        e3 = conv(e2, *weights[f"est{lvl}_3"])
        e4 = conv(e3, *weights[f"est{lvl}_4"])
        e5 = conv(np.concatenate([e4, e3], axis=2), *weights[f"est{lvl}_5"])
        w6, b6 = weights[f"est{lvl}_6"]
        fl = conv(np.concatenate([e5, e4], axis=2), w6, b6, act=False)
    # separable refinement at level 3
    r = np.concatenate([fl, np.zeros(fl.shape[:2] + (6,), np.float32), e5, e4], axis=2)
    for i, d in enumerate((1, 2, 4, 8, 16, 1), start=1):
        wd, _ = weights[f"ref{i}_dw"]
        r = depthwise(r, wd, d)
        r = conv(r, *weights[f"ref{i}_pw"])
    w7, b7 = weights["ref7"]
    fl = (fl.astype(np.float64) + conv(r, w7, b7, act=False)).astype(np.float32)
    H64, W64 = fl.shape[0] * 8, fl.shape[1] * 8
    full = (8.0 * _bilinear_resize(fl, H64, W64)).astype(np.float32)
    return np.ascontiguousarray(full[:h, :w])
