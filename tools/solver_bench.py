"""Device time of the 150-iteration solve at a given size (diagnostic).

    SS_SOLVER=tma|v2 python tools/solver_bench.py [H W] [steps]

Runs a device-resident session with ConstantFlow and prints the median
solver stage time (CUDA events on the session stream, ss_last_timing) and
the K1 time, as JSON.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2301_00750_b200 as ss  # noqa: E402
from paper_2301_00750_b200.synthetic import DeviceSequence  # noqa: E402

h, w = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (1080, 1920)))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
seq = DeviceSequence(h, w, step=(2, 1), seed=0)
pool = [seq.frame(k + 1) for k in range(8)]
torch.cuda.synchronize()
state = ss.SessionState(params=ss.preset("default"))
flow = ss.ConstantFlow(2.37, 1.13)
solve, blend = [], []
for k in range(steps + 2):
    i, p = pool[k % len(pool)]
    state.push_pair(k + 1, i, p)
    if k >= 2:
        ss.consistency._run_step(state, flow, with_next=True, return_host=False)
        solve.append(state.last_timing.solve_ms)
        blend.append(state.last_timing.warp_blend_ms)
solve = sorted(solve[3:])
blend = sorted(blend[3:])
print(json.dumps({"variant": os.environ.get("SS_SOLVER", "default"), "size": [h, w],
                  "solve_ms_median": solve[len(solve) // 2], "solve_ms_min": solve[0],
                  "k1_ms_median": blend[len(blend) // 2]}))
