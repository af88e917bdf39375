"""DIS parity stats vs the reference golden flows + 1080p timing."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2301_00750_b200.flow import FlowOptions, estimate_flow
g = np.load(os.path.join(ROOT, "tests/golden/dis.npz"))
for tag in ("shift", "same", "down2", "seqprev", "seqnext", "gray", "odd"):
    lv, ps, it, ds = (int(x) for x in g[f"{tag}_opts"])
    got = estimate_flow(g[f"{tag}_a"], g[f"{tag}_b"], FlowOptions(lv, ps, it, ds)).uv
    want = g[f"{tag}_uv"]
    e = np.sqrt(((got - want) ** 2).sum(axis=2))
    print(f"{tag}: bitwise-equal px {np.mean(np.all(got == want, axis=2)):.4f}  mean|d| {e.mean():.2e}  max|d| {e.max():.2e}")
x = torch.rand(1080, 1920, 3, device="cuda"); y = torch.roll(x, (1, 2), (0, 1))
for o in (FlowOptions(), FlowOptions(downscale=2)):
    for _ in range(3): estimate_flow(x, y, o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): estimate_flow(x, y, o)
    b.record(); torch.cuda.synchronize()
    print(f"1080p DIS flow downscale={o.downscale}: {a.elapsed_time(b)/10:.3f} ms")
