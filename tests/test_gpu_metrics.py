"""GPU metrics (E_warp, SSIM) against the reference's own values
(tests/golden/metrics.npz), and the reference's release criteria
(test_acceptance.py:32-243) restated on the B200 path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_00750_b200 as m

    return m


class _Recorded:
    def __init__(self, ss, g, tag):
        self.t = {(1, 2): ss.FlowField(g[f"ew_{tag}_fuv"], g[f"ew_{tag}_fvalid"]),
                  (2, 1): ss.FlowField(g[f"ew_{tag}_buv"], g[f"ew_{tag}_bvalid"])}

    def flow_between(self, pa, fa, pb, fb):
        return self.t[(pa, pb)]


@pytest.mark.parametrize("tag", ["gt", "subpix", "dis"])
def test_warping_error_matches_reference(ss, golden, tag):
    g = golden("metrics.npz")
    v = ss.warping_error_pair(g[f"ew_{tag}_a"], g[f"ew_{tag}_b"], 1, 2, _Recorded(ss, g, tag))
    assert v == pytest.approx(float(g[f"ew_{tag}_value"]), rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("tag", ["rgb", "gray", "seq"])
def test_ssim_matches_reference(ss, golden, tag):
    g = golden("metrics.npz")
    v = ss.ssim(g[f"ssim_{tag}_a"], g[f"ssim_{tag}_b"])
    assert v == pytest.approx(float(g[f"ssim_{tag}_value"]), abs=1e-6)


def test_metric_edge_cases(ss):
    rng = np.random.default_rng(0)
    a = rng.random((8, 8, 3)).astype(np.float32)
    assert ss.warping_error_pair(a, a, 1, 2, ss.ConstantFlow(100.0, 0.0)) is None
    rep = ss.warping_error([a, a, a], ss.ConstantFlow(100.0, 0.0))
    assert rep.skipped == [1, 2] and rep.count == 0
    with pytest.raises(ValueError, match="2 frames"):
        ss.warping_error([a], ss.ConstantFlow(0, 0))
    f = [rng.random((16, 16, 3)).astype(np.float32) for _ in range(3)]
    assert [v for _, v in ss.ssim_report(f, f).per_frame] == pytest.approx([1.0] * 3)
    with pytest.raises(ValueError, match="window"):
        ss.ssim(a, a)


# ----------------------------------------------- release criteria, GPU path
def test_static_scene_identity(ss):
    """test_acceptance.py:69-81: 10 static frames, RMSE(O, P) <= 1e-3."""
    rng = np.random.default_rng(11)
    frame = rng.random((64, 64, 3)).astype(np.float32)
    styled = np.clip(frame * 0.75 + 0.15, 0.0, 1.0).astype(np.float32)
    outs = list(ss.stabilize_stream(iter([(frame, styled)] * 10), ss.preset("default"),
                                    ss.ConstantFlow(0, 0)))
    assert len(outs) == 10
    assert max(float(np.sqrt(np.mean((o - styled) ** 2))) for _, o in outs) <= 1e-3


def test_consistency_off_fidelity(ss):
    """test_acceptance.py:83-97: k1 = k2 = 1e-6, lambda = 0 -> SSIM(O, P) >= 0.99."""
    from paper_2301_00750_b200 import synthetic

    params = ss.ConsistencyParams(k1=1e-6, k2=1e-6, lam=0.0)
    worst = 1.0
    for seed, (h, w) in ((1, (48, 64)), (2, (64, 48)), (3, (56, 56))):
        seq = synthetic.translating_sequence(frames=5, height=h, width=w, seed=seed)
        for pos, out in ss.stabilize_stream(zip(seq.inputs, seq.processed), params,
                                            ss.ConstantFlow(seq.step_u, seq.step_v)):
            worst = min(worst, ss.ssim(out, seq.processed[pos - 1]))
    assert worst >= 0.99


def test_flicker_reduction_and_lambda_sweep(ss):
    """test_acceptance.py:99-129: E_warp ratio <= 0.7; E_warp non-increasing in lambda."""
    from paper_2301_00750_b200 import synthetic

    seq = synthetic.translating_sequence(frames=10, height=96, width=128, step=(2, 1), seed=0)
    gt = ss.ConstantFlow(seq.step_u, seq.step_v)
    base = ss.warping_error(seq.processed, gt).mean
    outs = [o for _, o in ss.stabilize_stream(zip(seq.inputs, seq.processed),
                                              ss.preset("default"), gt)]
    assert ss.warping_error(outs, gt).mean / base <= 0.7
    sweep = []
    for lam in (0.1, 1.0, 2.0, 5.0):
        p = ss.preset("default").replace(lam=lam)
        o = [x for _, x in ss.stabilize_stream(zip(seq.inputs, seq.processed), p, gt)]
        sweep.append(ss.warping_error(o, gt).mean)
    assert all(b <= a + 1e-9 for a, b in zip(sweep, sweep[1:]))


def test_deterministic_outputs(ss):
    """test_consistency.py:308-319 / test_acceptance.py:209-243: bitwise repeatable."""
    from paper_2301_00750_b200 import synthetic

    seq = synthetic.translating_sequence(frames=5, height=48, width=48, seed=9)
    net = ss.LiteFlowNet(seed=0)
    runs = [[o.tobytes() for _, o in ss.stabilize_stream(zip(seq.inputs, seq.processed),
                                                         ss.preset("default"), net)]
            for _ in range(2)]
    assert runs[0] == runs[1]
