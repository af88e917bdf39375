"""Launch ONLY the flow network's est3_1 conv (the heaviest layer, 1/8-res
3x3, 152 -> 128 channels) a few times on a 1080p session's buffers, for an
ncu capture that cannot pick the wrong layer (the round-1 capture
labelled est3_1 was ref3_pw).  The first k_conv_tc3 launches of this process
are est3_1: ss_session_time_conv runs one warm-up + `reps` launches before
any pyramid or flow.

    python tools/conv_probe.py fp32|bf16
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2301_00750_b200 as ss  # noqa: E402
from paper_2301_00750_b200 import _lib  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
L = _lib.lib()
net = ss.LiteFlowNet(seed=0, precision=prec)
st = ss.SessionState(params=ss.preset("default"))
x = torch.rand(1080, 1920, 3, device="cuda")
st.push_pair(1, x, x)
st.push_pair(2, x, x)
assert L.ss_session_attach_flownet(st.handle, net.handle()) == 0, L.ss_last_error()
ms, fl = ctypes.c_float(0), ctypes.c_double(0)
assert L.ss_session_time_conv(st.handle, 3, 4, ctypes.byref(ms), ctypes.byref(fl)) == 0
torch.cuda.synchronize()
print(f"est3_1 {prec}: {ms.value * 1e3:.1f} us, {fl.value / 1e9:.2f} GFLOP algorithmic, "
      f"{fl.value / ms.value / 1e9:.1f} TFLOP/s")
