"""Diagnostics: lite flow net GPU paths (3xTF32 and bf16 tcgen05) vs the CPU
restatement, and 1080p flow timing.  Usage: python tools/flow_check.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch
import flownet_oracle as fo
import paper_2301_00750_b200 as ss
from paper_2301_00750_b200 import synthetic

seq = synthetic.translating_sequence(frames=2, height=120, width=200, seed=4)
a, b = seq.inputs[1], seq.inputs[0]
net32 = ss.LiteFlowNet(seed=0, precision="fp32")
net16 = ss.LiteFlowNet(seed=0, precision="bf16")
want = fo.flow(net32.weights, a, b)
for name, net in (("tf32x3", net32), ("bf16", net16)):
    got = net.flow_between(2, a, 1, b).uv
    e = np.sqrt(((got - want) ** 2).sum(axis=2))
    print(f"{name}: EPE mean {e.mean():.3g} max {e.max():.3g}  |flow| mean {np.abs(want).mean():.3g}", flush=True)
x = torch.rand(1080, 1920, 3, device="cuda"); y = torch.rand(1080, 1920, 3, device="cuda")
for name, net in (("tf32x3", net32), ("bf16", net16)):
    for _ in range(3):
        net.flow_between(1, x, 2, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        net.flow_between(1, x, 2, y)
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: stateless 1080p flow (2 pyramids + estimators) {e0.elapsed_time(e1)/10:.3f} ms", flush=True)
