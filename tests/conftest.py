import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture
def random_frame(rng):
    return rng.random((12, 10, 3)).astype(np.float32)


def stream_case(g, tag):
    """Unpack one stream case of streams.npz into lists + a replay flow table."""
    n = int(g[f"{tag}_n"])
    inputs = [g[f"{tag}_I{i}"] for i in range(1, n + 1)]
    processed = [g[f"{tag}_P{i}"] for i in range(1, n + 1)]
    outputs = {i: g[f"{tag}_O{i}"] for i in range(1, n + 1)}
    flows = {}
    prefix = f"{tag}_flow_"
    for k in g:
        if k.startswith(prefix) and k.endswith("_uv"):
            a, b = k[len(prefix):-3].split("_")
            flows[(int(a), int(b))] = (g[k], g[k[:-3] + "_valid"])
    params = g.get(f"{tag}_params")
    return inputs, processed, outputs, flows, params
