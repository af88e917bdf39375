"""Session I/O paths of the C ABI on the GPU: asynchronous output
(ss_output_async / ss_output_wait) returns exactly what ss_output returns,
for f32 and u8, while later steps run; the launch counter advances."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_00750_b200 import _lib

    L = _lib.lib()
    assert L.ss_init(0) == 0
    return _lib, L


def _params(_lib):
    from paper_2301_00750_b200._dev import params_struct
    from paper_2301_00750_b200.consistency import ConsistencyParams

    return params_struct(ConsistencyParams(iterations=20))


def test_output_async_matches_sync(lib):
    _lib, L = lib
    h, w = 48, 64
    rng = np.random.default_rng(3)
    frames = [rng.random((h, w, 3), dtype=np.float32) for _ in range(5)]
    sess = ctypes.c_void_p()
    assert L.ss_session_create(h, w, 3, 3, None, ctypes.byref(sess)) == 0
    n0 = L.ss_kernel_launches()
    prm = _params(_lib)
    it = ctypes.c_int(0)
    try:
        for pos in (1, 2):
            f = frames[pos - 1]
            assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
        pending = []
        for pos in (3, 4, 5):
            f = frames[pos - 1]
            assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
            assert L.ss_set_constant_flow(sess, 0, 1.0, 0.0, -1) == 0
            assert L.ss_set_constant_flow(sess, 1, 1.0, 0.0, 1) == 0
            assert L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)) == 0
            want = np.empty((h, w, 3), np.float32)
            assert L.ss_output(sess, want.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
            want8 = np.empty((h, w, 3), np.uint8)
            assert L.ss_output(sess, want8.ctypes.data, _lib.SS_U8, _lib.SS_HOST) == 0
            got = np.full((h, w, 3), np.nan, np.float32)
            assert L.ss_output_async(sess, got.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
            pending.append((got, want))
            assert L.ss_output_wait(sess) == 0
            got8 = np.zeros((h, w, 3), np.uint8)
            assert L.ss_output_async(sess, got8.ctypes.data, _lib.SS_U8, _lib.SS_HOST) == 0
            assert L.ss_output_wait(sess) == 0
            assert np.array_equal(got8, want8)
        for got, want in pending:
            assert np.array_equal(got, want)
    finally:
        L.ss_session_destroy(sess)
    assert L.ss_kernel_launches() > n0


def test_stage_pair_matches_push(lib):
    """A pair staged with ss_stage_pair and then pushed gives bit-identical
    steps to plain pushes (and a mismatched push still copies)."""
    _lib, L = lib
    h, w = 40, 56
    rng = np.random.default_rng(5)
    frames = [np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32)) for _ in range(6)]
    prm = _params(_lib)

    def run(stage):
        sess = ctypes.c_void_p()
        assert L.ss_session_create(h, w, 3, 3, None, ctypes.byref(sess)) == 0
        outs = []
        it = ctypes.c_int(0)
        try:
            for pos in range(1, 7):
                f = frames[pos - 1]
                assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                if stage and pos < 6:
                    g = frames[pos]
                    # stage the next pair; pos 3 stages a different pointer than it pushes
                    src = g if pos != 3 else g.copy()
                    assert L.ss_stage_pair(sess, pos + 1, src.ctypes.data, src.ctypes.data, _lib.SS_F32,
                                           _lib.SS_HOST) == 0
                if pos >= 3:
                    assert L.ss_set_constant_flow(sess, 0, 1.0, 1.0, -1) == 0
                    assert L.ss_set_constant_flow(sess, 1, 1.0, 1.0, 1) == 0
                    assert L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)) == 0
                    o = np.empty((h, w, 3), np.float32)
                    assert L.ss_output(sess, o.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                    outs.append(o)
        finally:
            L.ss_session_destroy(sess)
        return outs

    a, b = run(False), run(True)
    assert len(a) == len(b) == 4
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_pipelined_cnn_session_matches_plain(lib):
    """With the lite CNN attached, ss_step pre-launches the next step's flow to
    its previous frame and, when the pair after next is staged, that frame's
    pyramid.  Driving the session that way (flow 0 claimed, staged pushes, a
    re-staged position, a staged pointer the push does not use) gives outputs
    bit-identical to plain pushes with every flow computed on demand."""
    _lib, L = lib
    import paper_2301_00750_b200 as ss

    h, w = 72, 96
    rng = np.random.default_rng(11)
    frames = [np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32)) for _ in range(8)]
    alt = np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32))  # first staging of pos 6
    net = ss.LiteFlowNet(seed=0)
    prm = _params(_lib)

    def run(pipelined):
        sess = ctypes.c_void_p()
        assert L.ss_session_create(h, w, 3, 3, None, ctypes.byref(sess)) == 0
        assert L.ss_session_attach_flownet(sess, net.handle()) == 0
        outs = []
        it = ctypes.c_int(0)
        try:
            for pos in (1, 2):
                f = frames[pos - 1]
                assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
            for pos in range(3, 9):
                f = frames[pos - 1]
                if pipelined:
                    assert L.ss_session_compute_flow(sess, 0) == 0  # claims the pre-launched flow
                assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                if not pipelined:
                    assert L.ss_session_compute_flow(sess, 0) == 0
                assert L.ss_session_compute_flow(sess, 1) == 0
                if pipelined and pos < 8:
                    g = frames[pos]
                    # pos 6 is first staged with other data (re-staged after
                    # the step); pos 7's staged copy is not what gets pushed
                    src = alt if pos == 5 else (g.copy() if pos == 6 else g)
                    assert L.ss_stage_pair(sess, pos + 1, src.ctypes.data, src.ctypes.data, _lib.SS_F32,
                                           _lib.SS_HOST) == 0
                assert L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)) == 0
                if pipelined and pos == 5:
                    g = frames[pos]
                    assert L.ss_stage_pair(sess, pos + 1, g.ctypes.data, g.ctypes.data, _lib.SS_F32,
                                           _lib.SS_HOST) == 0
                o = np.empty((h, w, 3), np.float32)
                assert L.ss_output(sess, o.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                outs.append(o)
        finally:
            L.ss_session_destroy(sess)
        return outs

    a, b = run(False), run(True)
    assert len(a) == len(b) == 6
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_pipelined_cnn_session_divergence_retry(lib):
    """A step that diverges after its pre-launches (next flow t+1 -> t, staged
    pyramid) keeps its own flows: retrying it with sane params, then
    continuing the pipelined loop, matches a session that never diverged."""
    _lib, L = lib
    import paper_2301_00750_b200 as ss
    from paper_2301_00750_b200._dev import params_struct
    from paper_2301_00750_b200.consistency import ConsistencyParams

    h, w = 72, 96
    rng = np.random.default_rng(13)
    frames = [np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32)) for _ in range(7)]
    net = ss.LiteFlowNet(seed=0)
    good = _params(_lib)
    bad = params_struct(ConsistencyParams(eta=0.9999, lam=1e6, alpha=0.0, iterations=300, k1=0.1, k2=0.1))

    def run(diverge_at):
        sess = ctypes.c_void_p()
        assert L.ss_session_create(h, w, 3, 3, None, ctypes.byref(sess)) == 0
        assert L.ss_session_attach_flownet(sess, net.handle()) == 0
        outs = []
        it = ctypes.c_int(0)
        try:
            for pos in (1, 2):
                f = frames[pos - 1]
                assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
            for pos in range(3, 8):
                f = frames[pos - 1]
                assert L.ss_session_compute_flow(sess, 0) == 0
                assert L.ss_push_pair(sess, pos, f.ctypes.data, f.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                assert L.ss_session_compute_flow(sess, 1) == 0
                if pos < 7:
                    g = frames[pos]
                    assert L.ss_stage_pair(sess, pos + 1, g.ctypes.data, g.ctypes.data, _lib.SS_F32,
                                           _lib.SS_HOST) == 0
                if pos == diverge_at:
                    rc = L.ss_step(sess, 1, ctypes.byref(bad), ctypes.byref(it))
                    assert rc == _lib.SS_SOLVER_DIVERGENCE and it.value >= 1
                assert L.ss_step(sess, 1, ctypes.byref(good), ctypes.byref(it)) == 0
                o = np.empty((h, w, 3), np.float32)
                assert L.ss_output(sess, o.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                outs.append(o)
        finally:
            L.ss_session_destroy(sess)
        return outs

    a, b = run(None), run(4)
    assert len(a) == len(b) == 5
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_pipelined_dis_session_matches_stateless_flows(lib):
    """With the built-in DIS flow, ss_step pre-launches the next step's flow
    t+1 -> t on the side estimator and ss_session_compute_dis_flow(0) claims
    it.  That loop gives outputs bit-identical to flows computed by the
    stateless estimator and installed with ss_set_flow (no pre-launch)."""
    _lib, L = lib
    torch = pytest.importorskip("torch")
    h, w = 64, 96
    gen = torch.Generator(device="cpu").manual_seed(17)
    I = [torch.rand(h, w, 3, generator=gen).cuda().contiguous() for _ in range(7)]
    P = [torch.rand(h, w, 3, generator=gen).cuda().contiguous() for _ in range(7)]
    opts = (5, 9, 4, 1)  # levels, patch, iterations, downscale (FlowOptions defaults)
    prm = _params(_lib)

    def run(pipelined):
        sess = ctypes.c_void_p()
        assert L.ss_session_create(h, w, 3, 3, None, ctypes.byref(sess)) == 0
        uv = [torch.empty(h, w, 2, device="cuda") for _ in range(2)]
        vd = [torch.empty(h, w, dtype=torch.uint8, device="cuda") for _ in range(2)]
        outs = []
        it = ctypes.c_int(0)
        try:
            for pos in (1, 2):
                assert L.ss_push_pair(sess, pos, I[pos - 1].data_ptr(), P[pos - 1].data_ptr(), _lib.SS_F32,
                                      _lib.SS_DEVICE) == 0
            for pos in range(3, 8):
                t = pos - 1  # the step solved after pushing pos
                if pipelined:
                    assert L.ss_session_compute_dis_flow(sess, 0, *opts) == 0  # claims the pre-launch
                assert L.ss_push_pair(sess, pos, I[pos - 1].data_ptr(), P[pos - 1].data_ptr(), _lib.SS_F32,
                                      _lib.SS_DEVICE) == 0
                if pipelined:
                    assert L.ss_session_compute_dis_flow(sess, 1, *opts) == 0
                else:
                    for which, other in ((0, t - 1), (1, t + 1)):
                        assert L.ss_dis_flow(I[t - 1].data_ptr(), I[other - 1].data_ptr(), h, w, 3, *opts,
                                             uv[which].data_ptr(), vd[which].data_ptr(), None) == 0
                    torch.cuda.synchronize()
                    for which in (0, 1):
                        assert L.ss_set_flow(sess, which, uv[which].data_ptr(), vd[which].data_ptr(),
                                             _lib.SS_DEVICE) == 0
                assert L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)) == 0
                o = np.empty((h, w, 3), np.float32)
                assert L.ss_output(sess, o.ctypes.data, _lib.SS_F32, _lib.SS_HOST) == 0
                outs.append(o)
        finally:
            L.ss_session_destroy(sess)
        return outs

    a, b = run(False), run(True)
    assert len(a) == len(b) == 5
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
