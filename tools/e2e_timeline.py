"""Host-side timeline of the e2e loop (bench.run_e2e_abi order): wall time spent in
each C-ABI call per step, to locate host blocking.  Usage: e2e_timeline.py fp32"""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_00750_b200 as ss
from paper_2301_00750_b200 import _lib
from paper_2301_00750_b200._dev import params_struct
from paper_2301_00750_b200.consistency import ConsistencyParams
from paper_2301_00750_b200.synthetic import DeviceSequence

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
mode = sys.argv[2] if len(sys.argv) > 2 else "full"  # full | nostage | noout | devpush
h, w = 1080, 1920
L = _lib.lib()
seq = DeviceSequence(h, w, step=(2, 1), seed=0)
pool = [seq.frame(k + 1) for k in range(4)]
host_i = [p[0].cpu().pin_memory() for p in pool]
host_p = [p[1].cpu().pin_memory() for p in pool]
outs = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
douts = [torch.empty((h, w, 3), dtype=torch.float32, device="cuda") for _ in range(2)]
outs8 = [torch.empty((h, w, 3), dtype=torch.uint8).pin_memory() for _ in range(2)]
net = ss.LiteFlowNet(seed=0, precision=prec)
if os.environ.get("E2E_OWN_STREAM"):
    _strm = torch.cuda.Stream()
    torch.cuda.set_stream(_strm)
st = ss.SessionState(params=ConsistencyParams())
st.push_pair(1, pool[0][0], pool[0][1])
st.push_pair(2, pool[1][0], pool[1][1])
sess = st.handle
L.ss_session_attach_flownet(sess, net.handle())
pos = 2
acc = {}
def tcall(name, f):
    t0 = time.perf_counter(); rc = f(); acc.setdefault(name, []).append(time.perf_counter() - t0)
    assert rc == 0, (name, L.ss_last_error())
for k in range(30):
    pos += 1
    tcall("flow0", lambda: L.ss_session_compute_flow(sess, 0))
    if mode == "devpush":
        tcall("push", lambda: L.ss_push_pair(sess, pos, pool[k % 4][0].data_ptr(), pool[k % 4][1].data_ptr(), 0, 1))
    else:
        tcall("push", lambda: L.ss_push_pair(sess, pos, host_i[k % 4].data_ptr(), host_p[k % 4].data_ptr(), 0, 0))
    tcall("flow1", lambda: L.ss_session_compute_flow(sess, 1))
    if mode in ("full", "noout"):
        tcall("stage", lambda: L.ss_stage_pair(sess, pos + 1, host_i[(k + 1) % 4].data_ptr(), host_p[(k + 1) % 4].data_ptr(), 0, 0))
    if os.environ.get("E2E_INTERACTIVE"):  # bench.py's per-frame schedule
        prm = params_struct(ConsistencyParams(k1=0.3, k2=0.5, lam=2.0) if k % 2 == 0 else
                            ConsistencyParams(k1=0.5, k2=0.3, lam=0.5))
    else:
        prm = params_struct(ConsistencyParams())
    it = ctypes.c_int(0)
    tcall("step", lambda: L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)))
    if mode == "outdev":
        tcall("out", lambda: L.ss_output_async(sess, douts[k % 2].data_ptr(), 0, 1))
    elif mode == "outu8":
        tcall("out", lambda: L.ss_output_async(sess, outs8[k % 2].data_ptr(), 1, 0))
    elif mode != "noout" and mode != "devpush":
        tcall("out", lambda: L.ss_output_async(sess, outs[k % 2].data_ptr(), 0, 0))
torch.cuda.synchronize()
for n, v in acc.items():
    v = v[10:]
    print(f"{n:6s} mean {1e3 * sum(v) / len(v):7.3f} ms  max {1e3 * max(v):7.3f}")
print(mode, "total per step", sum(1e3 * sum(v[10:]) / len(v[10:]) for v in acc.values()))
