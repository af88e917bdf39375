"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container, where the reference is importable:

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference package is imported from $STREAMSTAB_REF_SRC (default
/root/reference/pkg/src).  Nothing on the GPU box reads the reference: the
committed .npz files are the pinned outputs.  Every array here is produced by
the reference's own public functions (flow.py / consistency.py); the inputs are
seeded so the script is reproducible.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("STREAMSTAB_REF_SRC", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import streamstab  # noqa: F401
    from streamstab import consistency, flow, imgio, synthetic

    return consistency, flow, imgio, synthetic


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def make_warp(flow, imgio):
    rng = np.random.default_rng(101)
    out = {}
    cases = [
        ("c3", rng.random((17, 23, 3)).astype(np.float32)),
        ("c1", rng.random((19, 13, 1)).astype(np.float32)),
        ("gray2d", rng.random((11, 16)).astype(np.float32)),
    ]
    for tag, img in cases:
        h, w = img.shape[:2]
        uv = rng.normal(0.0, 3.0, (h, w, 2)).astype(np.float32)
        # exact integer / half-integer displacements and border hits
        uv[0, :, :] = np.round(uv[0, :, :])
        uv[1, :, :] = np.round(uv[1, :, :] * 2) / 2
        uv[2, :3, 0] = 1e6   # far out of bounds -> clamped, masked
        uv[2, 3:5, 1] = -1e6
        uv[3, 0, :] = 2e9    # |uv| > 1e9 -> invalid (imgio.py:172)
        valid = np.abs(uv).max(axis=2) <= 1e9
        valid[4, :2] = False  # explicit invalid pixels
        field = imgio.FlowField(uv, valid)
        warped, mask = flow.backward_warp(img, field)
        out[f"{tag}_img"] = img
        out[f"{tag}_uv"] = uv
        out[f"{tag}_valid"] = valid
        out[f"{tag}_warped"] = warped
        out[f"{tag}_mask"] = mask
    _save("warp.npz", **out)


def make_occlusion(flow, imgio):
    rng = np.random.default_rng(202)
    out = {}
    for tag, (h, w), sigma in (("a", (21, 29), 2.0), ("b", (33, 17), 0.6), ("c", (40, 40), 6.0)):
        fu = rng.normal(0.0, sigma, (h, w, 2)).astype(np.float32)
        bu = (-fu + rng.normal(0.0, 0.4, (h, w, 2))).astype(np.float32)
        fu[::5, ::3, :] = np.round(fu[::5, ::3, :] * 2) / 2   # rint ties (half-even)
        bu[1::4, :, :] = np.round(bu[1::4, :, :])
        fv = np.ones((h, w), bool)
        bv = np.ones((h, w), bool)
        fv[rng.random((h, w)) < 0.05] = False
        bv[rng.random((h, w)) < 0.1] = False
        m = flow.occlusion_mask(imgio.FlowField(fu, fv), imgio.FlowField(bu, bv))
        out.update({f"{tag}_fuv": fu, f"{tag}_fvalid": fv, f"{tag}_buv": bu,
                    f"{tag}_bvalid": bv, f"{tag}_mask": m})
    _save("occlusion.npz", **out)


def make_weights(consistency):
    rng = np.random.default_rng(303)
    h, w = 14, 18
    out = {}
    for c in (3, 1):
        ref = rng.random((h, w, c)).astype(np.float32)
        warped = (ref + rng.normal(0, 0.02, (h, w, c))).astype(np.float32)
        validity = (rng.random((h, w)) > 0.2).astype(np.float32)
        wp = consistency.warp_weight(ref, warped, 6.5e3, 0.3, validity)
        wn = consistency.warp_weight(ref, warped[::-1].copy(), 1.0e3, 0.5, None)
        prev = rng.random((h, w, c)).astype(np.float32)
        nxt = rng.random((h, w, c)).astype(np.float32)
        L = consistency.local_blend(ref, prev, nxt, wp, wn)
        G = rng.random((h, w, c)).astype(np.float32)
        A = consistency.adaptive_blend(G, L, wp)
        wc = consistency.consistency_weight(ref, warped, 6.5e3, 2.0)
        lap = consistency.laplacian(ref)
        out.update({f"c{c}_ref": ref, f"c{c}_warped": warped, f"c{c}_validity": validity,
                    f"c{c}_wp": wp, f"c{c}_wn": wn, f"c{c}_prev": prev, f"c{c}_next": nxt,
                    f"c{c}_L": L, f"c{c}_G": G, f"c{c}_A": A, f"c{c}_wc": wc,
                    f"c{c}_lap": lap})
    _save("weights.npz", **out)


def make_solver(consistency):
    rng = np.random.default_rng(404)
    CP = consistency.ConsistencyParams
    out = {}
    cases = [
        ("default", (13, 11, 3), CP(), 2.0),
        ("gray", (9, 15, 1), CP(eta=0.2, kappa=0.5, iterations=37), 2.0),
        ("unscreened", (8, 8, 1), CP(iterations=300), 0.0),
        ("long", (16, 16, 3), CP(iterations=600), 2.0),
    ]
    for tag, shape, prm, wmax in cases:
        p = rng.random(shape).astype(np.float32)
        a = rng.random(shape).astype(np.float32)
        wc = rng.uniform(0.0, wmax, shape[:2]).astype(np.float32)
        o = consistency.solve_screened_poisson(p, a, wc, prm, init=a)
        out.update({f"{tag}_P": p, f"{tag}_A": a, f"{tag}_wc": wc, f"{tag}_O": o,
                    f"{tag}_params": np.array([prm.k1, prm.k2, prm.alpha, prm.lam, prm.eta,
                                               prm.kappa, prm.iterations], np.float64)})
    # divergence: the reference raises SolverDivergence(j+1) on a non-finite
    # np.sum of the update (consistency.py:292-293)
    div = []
    for i, (shape, wcv, iters) in enumerate((((8, 8), 100.0, 500), ((24, 20, 3), 40.0, 500),
                                              ((64, 48, 3), 15.0, 900))):
        p = rng.random(shape).astype(np.float32)
        a = rng.random(shape).astype(np.float32)
        wc = np.full(shape[:2], wcv, np.float32)
        try:
            with np.errstate(all="ignore"):
                consistency.solve_screened_poisson(p, a, wc, CP(iterations=iters), init=a)
            it = 0
        except consistency.SolverDivergence as e:
            it = e.iteration
        out.update({f"div{i}_P": p, f"div{i}_A": a, f"div{i}_wc": wc,
                    f"div{i}_iters": np.array(iters), f"div{i}_iteration": np.array(it)})
        div.append(it)
    print("divergence iterations", div)
    _save("solver.npz", **out)


class _Recorder:
    """Wraps a reference FlowProvider and records every flow it returns."""

    def __init__(self, inner):
        self.inner = inner
        self.log = {}

    def flow_between(self, pos_a, frame_a, pos_b, frame_b):
        f = self.inner.flow_between(pos_a, frame_a, pos_b, frame_b)
        self.log[(pos_a, pos_b)] = f
        return f


def make_streams(consistency, flow, synthetic):
    out = {}

    def run(tag, inputs, processed, provider, params_list=None):
        rec = _Recorder(provider)
        if params_list is None:
            outs = list(consistency.stabilize_stream(zip(inputs, processed), params_list_default,
                                                     rec))
        else:
            # interactive path: params swapped between frames (service.py:177-190)
            state = consistency.SessionState(params=params_list[0])
            outs = []
            n = len(inputs)
            for pos in range(1, n + 1):
                state.push_pair(pos, inputs[pos - 1], processed[pos - 1])
                if pos == 1:
                    outs.append((1, state.prev_output))
                elif pos >= 3:
                    state.params = params_list[pos - 2]
                    outs.append((pos - 1, consistency.stabilize_step(state, rec)))
            state.params = params_list[n - 1]
            outs.append((n, consistency.stream_end_step(state, rec)))
        out[f"{tag}_n"] = np.array(len(inputs))
        for i, (img, pr) in enumerate(zip(inputs, processed)):
            out[f"{tag}_I{i + 1}"] = np.asarray(img, np.float32)
            out[f"{tag}_P{i + 1}"] = np.asarray(pr, np.float32)
        for pos, o in outs:
            out[f"{tag}_O{pos}"] = np.asarray(o, np.float32)
        for (a, b), f in rec.log.items():
            out[f"{tag}_flow_{a}_{b}_uv"] = f.uv
            out[f"{tag}_flow_{a}_{b}_valid"] = f.valid
        if params_list is not None:
            out[f"{tag}_params"] = np.array(
                [[p.k1, p.k2, p.alpha, p.lam, p.eta, p.kappa, p.iterations] for p in params_list],
                np.float64)

    params_list_default = consistency.preset("default")
    seq = synthetic.translating_sequence(frames=5, height=48, width=64, step=(2, 1), seed=0)
    run("int", seq.inputs, seq.processed, flow.ConstantFlow(2, 1))
    run("subpix", seq.inputs, seq.processed, flow.ConstantFlow(2.37, 1.13))
    seq2 = synthetic.translating_sequence(frames=4, height=40, width=56, step=(3, -2), seed=7)
    run("dis", seq2.inputs, seq2.processed, flow.BuiltinFlow(flow.FlowOptions()))
    # gray input, color stylization (test_consistency.py:321-336)
    seq3 = synthetic.translating_sequence(frames=4, height=32, width=32, noise_sigma=0.0, seed=8)
    gray = [flow.luma(f)[:, :, None] for f in seq3.inputs]
    color = [synthetic.stylize(np.repeat(g, 3, axis=2)) for g in gray]
    run("gray", gray, color, flow.ConstantFlow(seq3.step_u, seq3.step_v))
    # two-frame stream: only the end step (test_consistency.py:271-273)
    run("two", seq.inputs[:2], seq.processed[:2], flow.ConstantFlow(2, 1))
    # interactive schedule: k1 in {0.3, 0.5}, lambda in {2.0, 0.5} per frame
    sched = [consistency.ConsistencyParams(k1=0.3 if i % 2 == 0 else 0.1,
                                           k2=0.5 if i % 2 == 0 else 0.3,
                                           lam=2.0 if i % 3 else 0.5)
             for i in range(5)]
    run("sched", seq.inputs, seq.processed, flow.ConstantFlow(2.37, 1.13), params_list=sched)
    _save("streams.npz", **out)


def make_metrics(flow, imgio, synthetic):
    from streamstab import metrics

    out = {}
    rng = np.random.default_rng(505)
    # E_warp pairs: translating texture with ground-truth flow, a sub-pixel
    # flow, and flows recorded from the reference's DIS estimator
    seq = synthetic.translating_sequence(frames=3, height=40, width=56, step=(2, 1), seed=5)
    cases = [("gt", seq.processed[0], seq.processed[1], flow.ConstantFlow(2, 1)),
             ("subpix", seq.processed[0], seq.processed[1], flow.ConstantFlow(1.37, -0.61)),
             ("dis", seq.inputs[1], seq.inputs[2], flow.BuiltinFlow(flow.FlowOptions()))]
    for tag, a, b, prov in cases:
        fw = prov.flow_between(1, a, 2, b)
        bw = prov.flow_between(2, b, 1, a)
        out[f"ew_{tag}_a"] = np.asarray(a, np.float32)
        out[f"ew_{tag}_b"] = np.asarray(b, np.float32)
        out[f"ew_{tag}_fuv"], out[f"ew_{tag}_fvalid"] = fw.uv, fw.valid
        out[f"ew_{tag}_buv"], out[f"ew_{tag}_bvalid"] = bw.uv, bw.valid
        rec = {(1, 2): fw, (2, 1): bw}

        class _P:
            def flow_between(self, pa, fa, pb, fb):
                return rec[(pa, pb)]

        v = metrics.warping_error_pair(a, b, 1, 2, _P())
        out[f"ew_{tag}_value"] = np.array(np.nan if v is None else v)
    # SSIM: random frames, a grey pair, and noisy-vs-clean stylized frames
    a = rng.random((23, 31, 3)).astype(np.float32)
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1).astype(np.float32)
    g1 = rng.random((16, 12, 1)).astype(np.float32)
    g2 = rng.random((16, 12, 1)).astype(np.float32)
    for tag, x, y in (("rgb", a, b), ("gray", g1, g2), ("seq", seq.processed[0], seq.inputs[0])):
        out[f"ssim_{tag}_a"], out[f"ssim_{tag}_b"] = x, y
        out[f"ssim_{tag}_value"] = np.array(metrics.ssim(x, y))
    _save("metrics.npz", **out)


def make_dis(flow, synthetic):
    """Reference DIS flows (estimate_flow, flow.py:168-325) for GPU parity."""
    out = {}
    rng = np.random.default_rng(606)
    tex = synthetic.noise_texture(128, 128, rng)
    tex2 = synthetic.noise_texture(128, 128, rng, smoothness=2.5)
    seq = synthetic.translating_sequence(frames=3, height=96, width=128, step=(2, 1), seed=12)
    gray = flow.luma(seq.inputs[0])[:, :, None]
    cases = [
        ("shift", tex, np.roll(tex, shift=(3, 5), axis=(0, 1)), flow.FlowOptions()),
        ("same", tex[:64, :64], tex[:64, :64], flow.FlowOptions()),
        ("down2", tex2, np.roll(tex2, shift=(2, 4), axis=(0, 1)), flow.FlowOptions(downscale=2)),
        ("seqprev", seq.inputs[1], seq.inputs[0], flow.FlowOptions()),
        ("seqnext", seq.inputs[1], seq.inputs[2], flow.FlowOptions()),
        ("gray", gray, np.roll(gray, shift=(1, -2), axis=(0, 1)), flow.FlowOptions(levels=3)),
        ("odd", seq.inputs[0][:77, :101], seq.inputs[1][:77, :101], flow.FlowOptions(patch_size=7)),
    ]
    for tag, a, b, opts in cases:
        f = flow.estimate_flow(a, b, opts)
        out[f"{tag}_a"] = np.asarray(a, np.float32)
        out[f"{tag}_b"] = np.asarray(b, np.float32)
        out[f"{tag}_uv"] = f.uv
        out[f"{tag}_opts"] = np.array([opts.levels, opts.patch_size, opts.iterations_per_level,
                                       opts.downscale])
    _save("dis.npz", **out)


def _sha(a) -> np.ndarray:
    import hashlib

    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


def make_dis_large(flow, synthetic):
    """Reference DIS flow at 960x540 (parity at >= 540p).  The
    frames are regenerated on the test side by the package's synthetic module
    (same recipe, same seed); their hashes pin that they are the same frames.
    The flow is pinned bit for bit by its sha256, plus a strided sample for
    diagnostics."""
    out = {}
    seq = synthetic.translating_sequence(frames=2, height=540, width=960, step=(2, 1), seed=31)
    for tag, opts in (("d1", flow.FlowOptions()), ("d2", flow.FlowOptions(downscale=2))):
        f = flow.estimate_flow(seq.inputs[1], seq.inputs[0], opts)
        out[f"{tag}_uv_sha"] = _sha(f.uv)
        out[f"{tag}_valid_sha"] = _sha(f.valid)
        out[f"{tag}_uv_sample"] = np.ascontiguousarray(f.uv[::7, ::7])
        out[f"{tag}_opts"] = np.array([opts.levels, opts.patch_size, opts.iterations_per_level,
                                       opts.downscale])
    out["a_sha"] = _sha(np.asarray(seq.inputs[1], np.float32))
    out["b_sha"] = _sha(np.asarray(seq.inputs[0], np.float32))
    out["shape"] = np.array([540, 960, 3])
    out["seed"] = np.array(31)
    _save("dis_large.npz", **out)


def make_imgio(consistency, flow, imgio, synthetic):
    """8-bit I/O of the live path: load = uint8 / 255 in float32
    (imgio.py:72 via a real PNG round trip), quantize = rint(clip(x)*255)
    (imgio.py:132, service.py:101-102), and a Session.solve_next-shaped u8
    stream (service.py:154-226): u8 frames loaded, stabilized with an integer
    ConstantFlow, outputs quantized."""
    import io
    import tempfile

    from PIL import Image

    from streamstab import service

    out = {}
    rng = np.random.default_rng(707)
    u8 = rng.integers(0, 256, (16, 24, 3), dtype=np.uint8)
    u8.reshape(-1)[:256] = np.arange(256, dtype=np.uint8)  # every code value
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "f.png")
        Image.fromarray(u8, mode="RGB").save(path)
        out["load_u8"] = u8
        out["load_f32"] = imgio.load_frame(path)
    # quantization: ties (k + 0.5) / 255, values just around them, outside [0, 1]
    k = np.arange(256, dtype=np.float64)
    vals = np.concatenate([(k + 0.5) / 255.0, k / 255.0,
                           np.nextafter(((k + 0.5) / 255.0).astype(np.float32), np.float32(0)),
                           np.nextafter(((k + 0.5) / 255.0).astype(np.float32), np.float32(1)),
                           [-1.0, -1e-7, 1.0 + 1e-7, 2.0, 0.5]]).astype(np.float32)
    vals = np.concatenate([vals, rng.random(4 * 256 * 3 - vals.size).astype(np.float32)])
    q = vals[: 16 * 64 * 3].reshape(16, 64, 3)
    png = service.encode_png(q)
    out["quant_f32"] = q
    out["quant_u8"] = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"), np.uint8)
    # u8 stream through the solve_next loop shape
    seq = synthetic.translating_sequence(frames=5, height=40, width=64, step=(2, 1), seed=41)
    ins = [np.rint(np.asarray(f) * 255).astype(np.uint8) for f in seq.inputs]
    prs = [np.rint(np.asarray(f) * 255).astype(np.uint8) for f in seq.processed]
    load = lambda a: imgio.as_frame(a.astype(np.float32) / 255.0)  # noqa: E731 (imgio.py:72)
    state = consistency.SessionState(params=consistency.preset("default"))
    prov = flow.ConstantFlow(2, 1)
    n = len(ins)
    state.push_pair(1, load(ins[0]), load(prs[0]))
    state.push_pair(2, load(ins[1]), load(prs[1]))
    loaded = 2
    outs = {1: np.rint(np.clip(state.prev_output, 0, 1) * 255.0).astype(np.uint8)}
    while state.solved_through < n:
        target = state.solved_through + 1
        if target < n:
            if loaded < target + 1:
                loaded += 1
                state.push_pair(loaded, load(ins[loaded - 1]), load(prs[loaded - 1]))
            o = consistency.stabilize_step(state, prov)
        else:
            o = consistency.stream_end_step(state, prov)
        outs[target] = np.rint(np.clip(o, 0.0, 1.0) * 255.0).astype(np.uint8)
    for i in range(n):
        out[f"stream_I{i + 1}"] = ins[i]
        out[f"stream_P{i + 1}"] = prs[i]
        out[f"stream_O{i + 1}"] = outs[i + 1]
    out["stream_n"] = np.array(n)
    _save("imgio.npz", **out)


def main():
    consistency, flow, imgio, synthetic = _import_ref()
    if len(sys.argv) > 1:  # regenerate only the named fixtures
        for name in sys.argv[1:]:
            {"dis_large": lambda: make_dis_large(flow, synthetic),
             "imgio": lambda: make_imgio(consistency, flow, imgio, synthetic)}[name]()
        return
    make_dis_large(flow, synthetic)
    make_imgio(consistency, flow, imgio, synthetic)
    make_dis(flow, synthetic)
    make_warp(flow, imgio)
    make_occlusion(flow, imgio)
    make_weights(consistency)
    make_solver(consistency)
    make_streams(consistency, flow, synthetic)
    make_metrics(flow, imgio, synthetic)


if __name__ == "__main__":
    main()
