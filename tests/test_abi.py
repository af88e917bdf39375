"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/streamstab_b200.h declares, and its host-only entry points
(version, status strings, parameter validation) behave.  No device calls."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "streamstab_b200.h")


def _header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^SS_API\s+[\w\s\*]*?\b(ss_\w+)\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2301_00750_b200 import _lib

    _lib.build()
    return _lib.lib()


def test_header_and_binding_agree():
    from paper_2301_00750_b200 import _lib

    assert _header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_header_symbol(lib):
    from paper_2301_00750_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ss_\w+)$", out, flags=re.M))
    missing = set(_header_symbols()) - exported
    assert not missing, missing
    for name in _header_symbols():
        assert hasattr(lib, name)


def test_version_and_status_strings(lib):
    assert lib.ss_abi_version() == 1
    assert lib.ss_status_string(3) == b"solver divergence"
    assert lib.ss_status_string(1) == b"resolution mismatch"


@pytest.mark.parametrize("changes,msg", [
    (dict(k1=0.6, k2=0.5), b"k1+k2 must be < 1"),
    (dict(eta=0.0), b"eta must be > 0"),
    (dict(kappa=1.0), b"kappa must be in [0, 1)"),
    (dict(iterations=0), b"iterations must be >= 1"),
    (dict(lam=-0.1), b"lambda must be >= 0"),
    (dict(flow_downscale=3), b"flow_downscale must be 1, 2 or 4"),
    (dict(k1=0.0, k2=0.0), b"k1+k2 must be > 0"),
])
def test_params_validate_matches_reference_messages(lib, changes, msg):
    from paper_2301_00750_b200 import _lib
    from paper_2301_00750_b200.consistency import ConsistencyParams
    from paper_2301_00750_b200._dev import params_struct

    p = ConsistencyParams(**changes)
    assert lib.ss_params_validate(ctypes.byref(params_struct(p))) == _lib.SS_VALUE_ERROR
    assert lib.ss_last_error() == msg
    with pytest.raises(ValueError, match=re.escape(msg.decode())):
        p.validate()
    assert lib.ss_params_validate(ctypes.byref(params_struct(ConsistencyParams()))) == 0


def test_flownet_param_count_matches_layer_table(lib):
    from paper_2301_00750_b200 import liteflownet as lf

    w = lf.make_weights(0)
    assert lib.ss_flownet_num_params() == lf.n_params() == lf.flatten_weights(w).size
    # padding rows are exactly zero; live rows are not
    w1, _ = w["est5_1"]
    assert not w1[:, :, 81:88].any() and not w1[:, :, 90:96].any() and w1[:, :, 96:].any()
    assert w1[:, :, 88:90].any()


def test_flownet_oracle_shapes():
    import numpy as np

    import flownet_oracle as fo
    from paper_2301_00750_b200 import liteflownet as lf

    w = lf.make_weights(1)
    rng = np.random.default_rng(0)
    a = rng.random((40, 70, 3)).astype(np.float32)
    f = fo.flow(w, a, np.roll(a, 2, axis=1))
    assert f.shape == (40, 70, 2) and f.dtype == np.float32 and np.isfinite(f).all()
    assert 0.01 < float(np.abs(f).mean()) < 20.0


def test_product_has_no_oracle_dependency():
    """The shipped package never imports or links the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2301_00750_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", "Makefile")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in text.lower().replace("oracles", ""), f
