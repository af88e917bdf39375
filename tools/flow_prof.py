"""Per-layer device times of one 1080p flow (SS_FLOW_PROFILE=1 prints them)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_00750_b200 as ss
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
net = ss.LiteFlowNet(seed=0, precision=prec)
x = torch.rand(1080, 1920, 3, device="cuda"); y = torch.rand(1080, 1920, 3, device="cuda")
for _ in range(2):
    net.flow_between(1, x, 2, y)
torch.cuda.synchronize()
print("---- measured call ----", file=sys.stderr, flush=True)
net.flow_between(1, x, 2, y)
torch.cuda.synchronize()
