"""bf16 flow-path accuracy at 1080p against the CPU restatement (diagnostic).

    python tools/bf16_epe.py            # heads in 3xTF32 (default)
    SS_BF16_HEADS=bf16 python tools/bf16_epe.py

Prints EPE mean / p99.9 / max of the bf16 path (and the fp32 path) against
oracle/flownet_oracle.py, and the PSNR of one consistency step driven by bf16
flows vs the same step driven by fp32 flows.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import flownet_oracle as fo  # noqa: E402

import paper_2301_00750_b200 as ss  # noqa: E402
from paper_2301_00750_b200 import liteflownet as lf, synthetic  # noqa: E402

h, w = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (1080, 1920)))
seq = synthetic.translating_sequence(frames=3, height=h, width=w, seed=4)
wts = lf.make_weights(0)
want = fo.flow(wts, seq.inputs[1], seq.inputs[0])
res = {"size": [h, w], "heads": os.environ.get("SS_BF16_HEADS", "tf32x3"),
       "mean_abs_flow": float(np.abs(want).mean())}
outs = {}
for prec in ("fp32", "bf16"):
    net = ss.LiteFlowNet(seed=0, precision=prec)
    got = np.asarray(net.flow_between(2, seq.inputs[1], 1, seq.inputs[0]).uv, np.float64)
    e = np.sqrt(((got - want) ** 2).sum(axis=2))
    res[prec] = {"epe_mean": float(e.mean()), "epe_p999": float(np.quantile(e, 0.999)),
                 "epe_max": float(e.max())}
    state = ss.SessionState(params=ss.preset("default"))
    for i in range(3):
        state.push_pair(i + 1, seq.inputs[i], seq.processed[i])
    outs[prec] = ss.stabilize_step(state, net)
mse = float(np.mean((outs["fp32"].astype(np.float64) - outs["bf16"]) ** 2))
res["step_psnr_bf16_vs_fp32"] = 10 * np.log10(1.0 / max(mse, 1e-30))
print(json.dumps(res))
