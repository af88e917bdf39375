"""EPE of the lite CNN's fp32-class path at 1920x1080 against the CPU
restatement (float64 accumulation), for the implementation selected by
SS_FP32_IMPL (tf32x3 | bf16x2); prints one JSON line.

    SS_FP32_IMPL=bf16x2 python tools/fp32_epe.py [cache.npz]
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import flownet_oracle as fo
import paper_2301_00750_b200 as ss
from paper_2301_00750_b200 import liteflownet as lf, synthetic

cache = sys.argv[1] if len(sys.argv) > 1 else None
seq = synthetic.translating_sequence(frames=3, height=1080, width=1920, seed=4)
a, b = seq.inputs[1], seq.inputs[0]
if cache and os.path.exists(cache):
    want = np.load(cache)["uv"]
else:
    want = fo.flow(lf.make_weights(0), a, b)
    if cache:
        np.savez(cache, uv=want)
got = ss.LiteFlowNet(seed=0).flow_between(2, a, 1, b).uv
e = np.sqrt(((got.astype(np.float64) - want) ** 2).sum(axis=2))
print(json.dumps({"impl": os.environ.get("SS_FP32_IMPL", "tf32x3"), "epe_max": float(e.max()),
                  "epe_mean": float(e.mean()), "epe_p999": float(np.quantile(e, 0.999)),
                  "flow_mag_mean": float(np.abs(want).mean())}))
