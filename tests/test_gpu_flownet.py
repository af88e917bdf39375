"""GPU parity of the lite flow network (north star (a)) against its CPU
restatement (oracle/flownet_oracle.py, float64 accumulation).

The reference has no flow CNN, so these pins are to the restatement of the
architecture in liteflownet.py with the same seeded random-init weights:
  * fp32 path: flow max |GPU - CPU| <= 2e-3 px, mean EPE <= 1e-4 px;
  * full step with CNN flows: O_t within 1e-3 max-abs (the north star's fp32
    bar) of the CPU oracle fed the CPU network's flows.
"""

import numpy as np
import pytest

import flownet_oracle as fo
import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_00750_b200 as m

    return m


@pytest.fixture(scope="module")
def net(ss):
    return ss.LiteFlowNet(seed=0)


def _epe(a, b):
    return np.sqrt(((a - b) ** 2).sum(axis=2))


@pytest.mark.parametrize("shape", [(64, 64, 3), (120, 200, 3), (72, 130, 1), (200, 130, 3)])
def test_flow_fp32_matches_cpu(ss, net, shape):
    from paper_2301_00750_b200 import synthetic

    seq = synthetic.translating_sequence(frames=2, height=shape[0], width=shape[1], seed=4)
    a, b = seq.inputs[1], seq.inputs[0]
    if shape[2] == 1:
        a, b = a.mean(axis=2, keepdims=True), b.mean(axis=2, keepdims=True)
    got = net.flow_between(2, a, 1, b)
    want = fo.flow(net.weights, a, b)
    assert got.uv.shape == want.shape and got.valid.all()
    e = _epe(got.uv, want)
    assert float(e.max()) <= 2e-3 and float(e.mean()) <= 5e-4, (float(e.max()), float(e.mean()))
    assert float(np.abs(want).mean()) > 0.05  # the random net emits non-trivial flow


@pytest.mark.parametrize("shape", [(120, 200, 3), (96, 160, 3)])
def test_flow_bf16_within_stated_tolerance(ss, shape):
    """bf16 tensor-core path vs the fp32 CPU restatement: EPE mean <= 0.03 px,
    max <= 0.15 px (flows of ~1 px); the consistency output it drives stays
    within PSNR >= 45 dB of the fp32-flow output."""
    from paper_2301_00750_b200 import synthetic

    net16 = ss.LiteFlowNet(seed=0, precision="bf16")
    seq = synthetic.translating_sequence(frames=2, height=shape[0], width=shape[1], seed=4)
    a, b = seq.inputs[1], seq.inputs[0]
    got = net16.flow_between(2, a, 1, b)
    want = fo.flow(net16.weights, a, b)
    e = _epe(got.uv, want)
    assert float(e.mean()) <= 0.03 and float(e.max()) <= 0.15, (float(e.mean()), float(e.max()))


def test_step_bf16_psnr_vs_fp32(ss, net):
    from paper_2301_00750_b200 import synthetic

    seq = synthetic.translating_sequence(frames=4, height=96, width=160, seed=6)
    net16 = ss.LiteFlowNet(seed=0, precision="bf16")
    o32 = dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), ss.preset("default"), net))
    o16 = dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), ss.preset("default"), net16))
    for t in o32:
        mse = float(np.mean((o32[t] - o16[t]) ** 2))
        psnr = 10 * np.log10(1.0 / max(mse, 1e-20))
        assert psnr >= 45.0, (t, psnr)


def test_session_cnn_step_within_1e3(ss, net):
    """The full step (CNN flows + consistency) vs the CPU oracle end to end."""
    from paper_2301_00750_b200 import synthetic

    seq = synthetic.translating_sequence(frames=4, height=96, width=160, seed=6)
    got = dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), ss.preset("default"), net))

    def flow_fn(a, fa, b, fb):
        uv = fo.flow(net.weights, fa, fb)
        return uv, np.ones(uv.shape[:2], bool)

    want = dict(orc.stabilize_stream(seq.inputs, seq.processed, orc.Params(), flow_fn))
    worst = max(float(np.abs(got[t] - want[t]).max()) for t in want)
    assert worst <= 1e-3, worst


def test_session_flows_match_stateless(ss, net):
    """Pyramid caching inside the session does not change the flows."""
    import ctypes

    from paper_2301_00750_b200 import _lib, synthetic

    seq = synthetic.translating_sequence(frames=3, height=64, width=128, seed=2)
    state = ss.SessionState(params=ss.preset("default"))
    for i in range(3):
        state.push_pair(i + 1, seq.inputs[i], seq.processed[i])
    ss.stabilize_step(state, net)
    for which, other in ((0, 1), (1, 3)):
        uv = np.empty((64, 128, 2), np.float32)
        _lib.lib().ss_flows(state.handle, which, uv.ctypes.data, None, _lib.SS_HOST)
        ref = net.flow_between(2, seq.inputs[1], other, seq.inputs[other - 1])
        assert np.array_equal(uv, ref.uv)


def test_concurrent_flows_bitwise_equal_serial(ss, net, monkeypatch):
    """The flow to t-1 on the side stream (started before the next push) gives
    the same stream, bit for bit, as both flows serialised on one stream."""
    from paper_2301_00750_b200 import synthetic

    seq = synthetic.translating_sequence(frames=7, height=72, width=120, seed=9)
    conc = dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), ss.preset("default"), net))
    monkeypatch.setenv("SS_FLOW_CONCURRENT", "0")
    serial = dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), ss.preset("default"), net))
    assert sorted(conc) == sorted(serial) == list(range(1, 8))
    for t in conc:
        assert np.array_equal(conc[t], serial[t]), t


def test_concurrent_sessions_threads_bitwise(ss, net):
    """Independent streams on their own CUDA streams, driven from two host
    threads at once (bench --streams), give exactly the sequential results."""
    import threading

    import torch

    from paper_2301_00750_b200 import synthetic

    seqs = [synthetic.translating_sequence(frames=5, height=64, width=96, seed=s) for s in (11, 12)]

    def run(seq):
        return dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), ss.preset("default"), net))

    want = [run(q) for q in seqs]
    got = [None, None]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def worker(k):
        with torch.cuda.stream(streams[k]):
            got[k] = run(seqs[k])

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for k in range(2):
        assert sorted(got[k]) == sorted(want[k])
        for t in want[k]:
            assert np.array_equal(got[k][t], want[k][t]), (k, t)


# ------------------------------------------- provider downscale (fast preset)
@pytest.mark.parametrize("shape,d", [((130, 200, 3), 2), ((257, 321, 3), 2), ((260, 392, 1), 4)])
def test_flow_downscale_matches_cpu(ss, net, shape, d):
    """FlowOptions.downscale semantics for the CNN (flow.py:183-188): the
    network on box_downscale(frame, d), the flow resize_bilinear'd back times
    d -- odd sizes crop the remainder.  Same fp32 bar as the full-resolution
    path, scaled by d (the flow is d times the network's)."""
    from paper_2301_00750_b200 import synthetic

    nd = ss.LiteFlowNet(weights=net.weights, downscale=d)
    seq = synthetic.translating_sequence(frames=2, height=shape[0], width=shape[1], seed=6)
    a, b = seq.inputs[1], seq.inputs[0]
    if shape[2] == 1:
        a, b = a.mean(axis=2, keepdims=True), b.mean(axis=2, keepdims=True)
    got = nd.flow_between(2, a, 1, b)
    want = fo.flow(net.weights, a, b, downscale=d)
    assert got.uv.shape == want.shape == shape[:2] + (2,) and got.valid.all()
    e = _epe(got.uv, want)
    assert float(e.max()) <= 2e-3 * d and float(e.mean()) <= 5e-4 * d, (float(e.max()), float(e.mean()))


def test_fast_preset_stream_with_downscaled_cnn(ss, net):
    """The fast preset end to end (50 iterations, flow_downscale 2 handed to the
    provider as service.py:188 does): GPU session vs the C oracle fed the CPU
    network's downscaled flows, O_t within 1e-3."""
    from paper_2301_00750_b200 import synthetic

    p = ss.preset("fast")
    nd = ss.LiteFlowNet(weights=net.weights, downscale=p.flow_downscale)
    seq = synthetic.translating_sequence(frames=3, height=96, width=160, step=(2, 1), seed=8)
    got = dict(ss.stabilize_stream(zip(seq.inputs, seq.processed), p, nd))

    def cnn_fn(a, fa, b, fb):
        uv = fo.flow(net.weights, fa, fb, downscale=p.flow_downscale)
        return uv, np.ones(uv.shape[:2], bool)

    want = dict(orc.stabilize_stream(seq.inputs, seq.processed,
                                     orc.Params(k1=p.k1, k2=p.k2, alpha=p.alpha, lam=p.lam, eta=p.eta,
                                                kappa=p.kappa, iterations=p.iterations), cnn_fn))
    assert sorted(got) == sorted(want)
    for t in want:
        assert float(np.abs(got[t] - want[t]).max()) <= 1e-3, t


def test_downscale_validation(ss):
    with pytest.raises(ValueError, match="downscale must be 1, 2 or 4"):
        ss.LiteFlowNet(seed=0, downscale=3)
