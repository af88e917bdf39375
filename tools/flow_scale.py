"""Device time of the lite flow network (1 pyramid + 1 flow, graph-launched)
against resolution: separates the per-layer fixed latency from the per-pixel
work.  Usage: flow_scale.py [fp32|bf16] [H W]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_00750_b200 as ss

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
sizes = [(64, 64), (128, 128), (192, 320), (360, 640), (540, 960), (720, 1280), (1080, 1920)]
if len(sys.argv) > 3:
    sizes = [(int(sys.argv[2]), int(sys.argv[3]))]
net = ss.LiteFlowNet(seed=0, precision=prec)
for h, w in sizes:
    frames = [torch.rand(h, w, 3, device="cuda") for _ in range(4)]
    pos = 0
    def run():
        global pos
        pos += 1
        # the previous call's second frame is cached: one new pyramid + one flow
        net.flow_between(pos + 1, frames[(pos + 1) % 4], pos, frames[pos % 4])
    for _ in range(6):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{h}x{w}: {ms:.3f} ms per pyramid + flow ({h * w / 1e6:.3f} Mpx)", flush=True)
