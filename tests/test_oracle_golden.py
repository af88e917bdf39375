"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

Bit-exact for warp / mask / occlusion / laplacian / blends / solver (given the
same inputs) and for the divergence iteration; exp-derived weights within
2 ulp (numpy SIMD expf vs libm expf); full-step outputs within 1e-5.
"""

import numpy as np
import pytest

import oracle as orc
from conftest import stream_case

EXP_ULP_RTOL = 2.5e-7  # <= 2 ulp of float32 for values in (0, 2]


def ulp_close(a, b, ulps=2):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    gap = np.abs(a.astype(np.float64) - b.astype(np.float64))
    tol = ulps * np.spacing(np.maximum(np.abs(a), np.abs(b))).astype(np.float64)
    return bool(np.all(gap <= tol))


@pytest.mark.parametrize("tag", ["c3", "c1", "gray2d"])
def test_backward_warp_bitwise(golden, tag):
    g = golden("warp.npz")
    warped, mask = orc.backward_warp(g[f"{tag}_img"], g[f"{tag}_uv"], g[f"{tag}_valid"])
    assert np.array_equal(warped, g[f"{tag}_warped"])
    assert np.array_equal(mask, g[f"{tag}_mask"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_occlusion_mask_bitwise(golden, tag):
    g = golden("occlusion.npz")
    m = orc.occlusion_mask(g[f"{tag}_fuv"], g[f"{tag}_fvalid"], g[f"{tag}_buv"],
                           g[f"{tag}_bvalid"])
    assert np.array_equal(m, g[f"{tag}_mask"])
    assert 0 < m.sum() < m.size  # the case exercises both outcomes


@pytest.mark.parametrize("c", [3, 1])
def test_weights_and_blends(golden, c):
    g = golden("weights.npz")
    k = f"c{c}_"
    wp = orc.warp_weight(g[k + "ref"], g[k + "warped"], 6.5e3, 0.3, g[k + "validity"])
    assert ulp_close(wp, g[k + "wp"])
    wn = orc.warp_weight(g[k + "ref"], g[k + "warped"][::-1], 1.0e3, 0.5)
    assert ulp_close(wn, g[k + "wn"])
    # blends are exact given the same weights
    L = orc.local_blend(g[k + "ref"], g[k + "prev"], g[k + "next"], g[k + "wp"], g[k + "wn"])
    assert np.array_equal(L, g[k + "L"])
    A = orc.adaptive_blend(g[k + "G"], g[k + "L"], g[k + "wp"])
    assert np.array_equal(A, g[k + "A"])
    wc = orc.consistency_weight(g[k + "ref"], g[k + "warped"], 6.5e3, 2.0)
    assert ulp_close(wc, g[k + "wc"])
    assert np.array_equal(orc.laplacian(g[k + "ref"]), g[k + "lap"])


def _params(arr):
    k1, k2, alpha, lam, eta, kappa, iters = arr.tolist()
    return orc.Params(k1=k1, k2=k2, alpha=alpha, lam=lam, eta=eta, kappa=kappa,
                      iterations=int(iters))


@pytest.mark.parametrize("tag", ["default", "gray", "unscreened", "long"])
def test_solver_bitwise(golden, tag):
    g = golden("solver.npz")
    o = orc.solve_screened_poisson(g[f"{tag}_P"], g[f"{tag}_A"], g[f"{tag}_wc"],
                                   _params(g[f"{tag}_params"]))
    assert np.array_equal(o, g[f"{tag}_O"])


@pytest.mark.parametrize("i", [0, 1, 2])
def test_solver_divergence_iteration_exact(golden, i):
    g = golden("solver.npz")
    want = int(g[f"div{i}_iteration"])
    assert want >= 1
    with pytest.raises(orc.OracleDivergence) as err:
        orc.solve_screened_poisson(g[f"div{i}_P"], g[f"div{i}_A"], g[f"div{i}_wc"],
                                   orc.Params(iterations=int(g[f"div{i}_iters"])))
    assert err.value.iteration == want


def test_pairwise_sum_matches_numpy(rng):
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 4097, 100_003):
        a = (rng.standard_normal(n) * np.exp(rng.standard_normal(n) * 4)).astype(np.float32)
        assert orc.numpy_pairwise_sum(a) == np.sum(a)


@pytest.mark.parametrize("tag", ["int", "subpix", "dis", "gray", "two", "sched"])
def test_stream_outputs(golden, tag):
    g = golden("streams.npz")
    inputs, processed, outputs, flows, params = stream_case(g, tag)
    n = len(inputs)

    def flow_fn(a, fa, b, fb):
        return flows[(a, b)]

    if params is None:
        got = dict(orc.stabilize_stream(inputs, processed, orc.Params(), flow_fn))
    else:
        # per-frame params: frame t is solved with params[t-1]
        got = {1: processed[0]}
        prev = processed[0]
        for t in range(2, n + 1):
            fn = flows.get((t, t + 1))
            prev = orc.run_step(inputs[t - 2], processed[t - 2], inputs[t - 1], processed[t - 1],
                                inputs[t] if t < n else None, processed[t] if t < n else None,
                                prev, flows[(t, t - 1)], fn, _params(params[t - 1]))
            got[t] = prev
    assert sorted(got) == list(range(1, n + 1))
    assert np.array_equal(got[1], outputs[1])
    worst = max(float(np.abs(got[t] - outputs[t]).max()) for t in got)
    assert worst <= 1e-5, worst
