"""Host-side phase times of the drop-in numpy API loop at 1080p (what the
bench's e2e_python_api measures): push_pair(numpy), the step until the
output array is returned, per step (median over 20 steps)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2301_00750_b200 as ss
from paper_2301_00750_b200.consistency import _start_flow_to_prev
from paper_2301_00750_b200.synthetic import DeviceSequence

h, w = 1080, 1920
seq = DeviceSequence(h, w, step=(2, 1), seed=7)
frames = [tuple(np.ascontiguousarray(x.cpu().numpy()) for x in seq.frame(k + 1)) for k in range(4)]
net = ss.LiteFlowNet(seed=0)
st = ss.SessionState(params=ss.preset("default"))
pos = [0]
def push():
    pos[0] += 1
    i, p = frames[(pos[0] - 1) % 4]
    st.push_pair(pos[0], i, p)
push(); push()
T = {"pre": [], "push": [], "step": [], "total": []}
for k in range(30):
    t0 = time.perf_counter()
    _start_flow_to_prev(st, net)
    t1 = time.perf_counter()
    push()
    t2 = time.perf_counter()
    out = ss.stabilize_step(st, net)
    t3 = time.perf_counter()
    if k >= 10:
        T["pre"].append(t1 - t0); T["push"].append(t2 - t1); T["step"].append(t3 - t2); T["total"].append(t3 - t0)
for k, v in T.items():
    print(f"{k:6s} median {1e3*np.median(v):.3f} ms")
