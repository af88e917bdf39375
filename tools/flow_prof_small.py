"""Per-layer device times of one flow at a small size (SS_FLOW_PROFILE=1): the
network's per-kernel fixed latency when every layer is tiny."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_00750_b200 as ss
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
H = int(sys.argv[2]) if len(sys.argv) > 2 else 128
W = int(sys.argv[3]) if len(sys.argv) > 3 else 128
net = ss.LiteFlowNet(seed=0, precision=prec)
x = torch.rand(H, W, 3, device="cuda"); y = torch.rand(H, W, 3, device="cuda")
for _ in range(2):
    net.flow_between(1, x, 2, y)
torch.cuda.synchronize()
print("---- measured call ----", file=sys.stderr, flush=True)
net.flow_between(1, x, 2, y)
torch.cuda.synchronize()
