"""INTEGRATION.md §2 executed ("the INTEGRATION.md stub itself is
never executed"): the ctypes binding a reference maintainer would add
(``streamstab/_b200.py``) is taken verbatim from INTEGRATION.md, loaded into
the reference package itself (baseline/_ref, installed from /root/reference),
and the two-line change INTEGRATION.md describes for ``push_pair`` /
``_run_step`` is applied; the reference's own ``stabilize_stream`` then runs
through the B200 library and matches the unmodified reference (<= 1e-5, the
exp-ulp bound of the golden streams).

Skipped when the reference is not installed in baseline/_ref.
"""

import importlib.util
import os
import re
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2. ctypes binding"):]
    m = re.search(r"```python\n(# streamstab/_b200.py.*?)```", sec, re.S)
    assert m, "INTEGRATION.md §2 has no _b200.py block"
    lib = os.path.join(ROOT, "paper_2301_00750_b200", "lib", "libstreamstab_b200.so")
    # the library path is deployment-specific; the stub names the bare soname
    return m.group(1).replace('"libstreamstab_b200.so"', repr(lib))


@pytest.fixture(scope="module")
def ref():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "streamstab")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    import streamstab
    from streamstab import consistency, flow, synthetic

    spec = importlib.util.spec_from_loader("streamstab._b200", loader=None)
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = "streamstab"
    exec(compile(_stub_source(), "INTEGRATION.md:_b200.py", "exec"), mod.__dict__)
    sys.modules["streamstab._b200"] = mod
    yield streamstab, consistency, flow, synthetic, mod
    sys.modules.pop("streamstab._b200", None)
    sys.path.remove(REF)


def _patched(consistency, b200):
    """INTEGRATION.md §2's change to consistency.py, as a maintainer would make it."""
    orig_push = consistency.SessionState.push_pair

    def push_pair(self, position, input_frame, processed_frame):
        orig_push(self, position, input_frame, processed_frame)  # the existing checks
        if getattr(self, "_dev", None) is None:
            ci = 1 if input_frame.ndim == 2 else input_frame.shape[2]
            cp = 1 if processed_frame.ndim == 2 else processed_frame.shape[2]
            self._dev = b200.Device(*input_frame.shape[:2], ci, cp)
        self._dev.push(position, input_frame, processed_frame)

    def _run_step(state, flow_backend, t, by_pos, with_next):
        params = state.params
        input_prev, _ = by_pos[t - 1]
        input_cur, _ = by_pos[t]
        t0 = time.perf_counter()
        flow_to_prev = flow_backend.flow_between(t, input_cur, t - 1, input_prev)
        flow_to_next = None
        if with_next:
            input_next, _ = by_pos[t + 1]
            flow_to_next = flow_backend.flow_between(t, input_cur, t + 1, input_next)
        flow_ms = (time.perf_counter() - t0) * 1e3
        t1 = time.perf_counter()
        output = state._dev.step(params, flow_to_prev, flow_to_next)  # replaces :387-407
        solve_ms = (time.perf_counter() - t1) * 1e3
        state.prev_output = output
        state.solved_through = t
        state.last_timing = consistency.StepTiming(flow_ms=flow_ms, solve_ms=solve_ms)
        return output

    return push_pair, _run_step


@pytest.mark.parametrize("flow_kind", ["int", "subpix", "builtin"])
def test_reference_runs_through_integration_stub(ref, monkeypatch, flow_kind):
    streamstab, consistency, flow, synthetic, b200 = ref
    seq = synthetic.translating_sequence(frames=5, height=48, width=64, step=(2, 1), seed=3)
    prov = {"int": flow.ConstantFlow(2, 1), "subpix": flow.ConstantFlow(2.37, 1.13),
            "builtin": flow.BuiltinFlow(flow.FlowOptions())}[flow_kind]
    prm = consistency.preset("default")
    want = dict(consistency.stabilize_stream(zip(seq.inputs, seq.processed), prm, prov))
    push_pair, run_step = _patched(consistency, b200)
    monkeypatch.setattr(consistency.SessionState, "push_pair", push_pair)
    monkeypatch.setattr(consistency, "_run_step", run_step)
    got = dict(consistency.stabilize_stream(zip(seq.inputs, seq.processed), prm, prov))
    assert sorted(got) == sorted(want) == list(range(1, 6))
    worst = max(float(np.abs(np.asarray(got[t]) - want[t]).max()) for t in want)
    assert worst <= 1e-5, worst
    if flow_kind == "int":
        assert all(np.array_equal(got[t], want[t]) for t in want)


def test_stub_maps_divergence(ref):
    """SolverDivergence through the stub carries the reference's own iteration."""
    streamstab, consistency, flow, synthetic, b200 = ref
    rng = np.random.default_rng(1)
    f = [rng.random((12, 12, 3)).astype(np.float32) for _ in range(3)]
    prm = consistency.ConsistencyParams(eta=0.9999, lam=1e6, alpha=0.0, iterations=300,
                                        k1=0.1, k2=0.1)
    prov = flow.ConstantFlow(0.5, 0)
    state = consistency.SessionState(params=prm)
    for i in range(3):
        state.push_pair(i + 1, f[i], f[(i + 2) % 3])
    with pytest.raises(consistency.SolverDivergence) as want:
        consistency.stabilize_step(state, prov)
    dev = b200.Device(12, 12, 3, 3)
    for i in range(3):
        dev.push(i + 1, f[i], f[(i + 2) % 3])
    with pytest.raises(consistency.SolverDivergence) as got:
        dev.step(prm, prov.flow_between(2, f[1], 1, f[0]), prov.flow_between(2, f[1], 3, f[2]))
    assert got.value.iteration == want.value.iteration >= 1
