"""Host-side mirror of the reference interface (no device): parameters,
presets, FlowField semantics, and the synthetic stream recipe."""

import numpy as np
import pytest

from paper_2301_00750_b200.consistency import PRESETS, ConsistencyParams, preset
from paper_2301_00750_b200.imgio import FlowField, as_frame
from paper_2301_00750_b200 import synthetic


def test_presets_pin_published_values():
    d = PRESETS["default"]
    assert (d.k1, d.k2, d.alpha, d.lam) == (0.3, 0.5, 6.5e3, 2.0)
    assert (d.eta, d.kappa, d.iterations, d.flow_downscale) == (0.15, 0.2, 150, 1)
    o = PRESETS["objective"]
    assert (o.k1, o.k2, o.alpha, o.lam, o.iterations) == (0.3, 0.3, 1.0e4, 0.7, 150)
    f = PRESETS["fast"]
    assert f.iterations == 50 and f.flow_downscale == 2


def test_dict_roundtrip_uses_lambda_key():
    d = preset("default").to_dict()
    assert d["lambda"] == 2.0 and "lam" not in d
    assert ConsistencyParams.from_dict(d) == preset("default")
    with pytest.raises(ValueError, match="unknown parameter"):
        ConsistencyParams.from_dict({"gamma": 1})
    with pytest.raises(ValueError, match="unknown preset"):
        preset("speedy")


def test_validation_boundaries():
    # float sums are evaluated in double exactly like the reference
    with pytest.raises(ValueError, match="k1\\+k2 must be < 1"):
        ConsistencyParams(k1=0.3, k2=0.7).validate()
    ConsistencyParams(k1=0.3, k2=0.6999).validate()
    with pytest.raises(ValueError):
        ConsistencyParams(iterations=0).validate()


def test_flowfield_validity_convention():
    uv = np.zeros((3, 4, 2), np.float32)
    uv[1, 2, 0] = 2e9
    f = FlowField(uv)
    assert f.valid.sum() == 11 and not f.valid[1, 2]
    assert (f.height, f.width) == (3, 4)
    assert not f.uv.flags.writeable
    with pytest.raises(ValueError):
        FlowField(np.zeros((3, 4, 3), np.float32))


def test_as_frame_contract():
    fr = as_frame(np.full((2, 3), 1.5))
    assert fr.shape == (2, 3, 1) and fr.max() == 1.0 and not fr.flags.writeable
    with pytest.raises(ValueError):
        as_frame(np.zeros((2, 3, 2)))


def test_synthetic_translation_is_exact():
    seq = synthetic.translating_sequence(frames=3, height=20, width=24, step=(2, 1), seed=4)
    a, b = seq.inputs[0], seq.inputs[1]
    assert np.array_equal(np.roll(a, shift=(1, 2), axis=(0, 1)), b)
    assert all(p.min() >= 0 and p.max() <= 1 for p in seq.processed)
