"""GPU-side kernel timeline of the device-resident step (CUPTI via
torch.profiler): per-kernel start / duration / stream for one step, plus the
idle gaps on the critical stream.  Graph-replayed kernels are included.

Usage: gpu_timeline.py [fp32|bf16] [H W] [out.json]
"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2301_00750_b200 as ss
from paper_2301_00750_b200 import _lib
from paper_2301_00750_b200._dev import params_struct
from paper_2301_00750_b200.consistency import ConsistencyParams
from paper_2301_00750_b200.synthetic import DeviceSequence

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
E2E = os.environ.get("TL_E2E") is not None  # bench.py's e2e loop: pinned host staging + async output
h = int(sys.argv[2]) if len(sys.argv) > 2 else 1080
w = int(sys.argv[3]) if len(sys.argv) > 3 else 1920
out_path = sys.argv[4] if len(sys.argv) > 4 else None
L = _lib.lib()
seq = DeviceSequence(h, w, step=(2, 1), seed=0)
pool = [seq.frame(k + 1) for k in range(4)]
net = ss.LiteFlowNet(seed=0, precision=prec)
st = ss.SessionState(params=ConsistencyParams())
st.push_pair(1, pool[0][0], pool[0][1])
st.push_pair(2, pool[1][0], pool[1][1])
sess = st.handle
L.ss_session_attach_flownet(sess, net.handle())
pos = 2
host = [(p[0].cpu().pin_memory(), p[1].cpu().pin_memory()) for p in pool]
outs = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]


def step_e2e(k):
    global pos
    pos += 1
    for name, rc in (("flow0", L.ss_session_compute_flow(sess, 0)),
                     ("push", L.ss_push_pair(sess, pos, host[k % 4][0].data_ptr(), host[k % 4][1].data_ptr(), 0, 0)),
                     ("flow1", L.ss_session_compute_flow(sess, 1)),
                     ("stage", L.ss_stage_pair(sess, pos + 1, host[(k + 1) % 4][0].data_ptr(),
                                               host[(k + 1) % 4][1].data_ptr(), 0, 0))):
        assert rc == 0, (name, L.ss_last_error())
    prm = params_struct(ConsistencyParams())
    it = ctypes.c_int(0)
    assert L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)) == 0, L.ss_last_error()
    assert L.ss_output_async(sess, outs[k % 2].data_ptr(), 0, 0) == 0


def step(k):
    if E2E:
        return step_e2e(k)
    # bench.py's order: flow 0 (claims the pre-launched one), push (swaps the
    # staged pair in), flow 1, stage the pair after next, step
    global pos
    pos += 1
    for name, rc in (("flow0", L.ss_session_compute_flow(sess, 0)),
                     ("push", L.ss_push_pair(sess, pos, pool[k % 4][0].data_ptr(), pool[k % 4][1].data_ptr(), 0, 1)),
                     ("flow1", L.ss_session_compute_flow(sess, 1)),
                     ("stage", L.ss_stage_pair(sess, pos + 1, pool[(k + 1) % 4][0].data_ptr(),
                                               pool[(k + 1) % 4][1].data_ptr(), 0, 1))):
        assert rc == 0, (name, L.ss_last_error())
    prm = params_struct(ConsistencyParams())
    it = ctypes.c_int(0)
    assert L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)) == 0, L.ss_last_error()


for k in range(8):
    step(k)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for k in range(8, 11):
        step(k)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = []
for e in evs:
    ks.append({"name": e.name, "start": e.time_range.start, "end": e.time_range.end,
               "stream": getattr(e, "device_resource_id", -1)})
ks.sort(key=lambda r: r["start"])
# the last full step: from the previous step's final kernel (the solver's
# per-pass maxima readback, k_copy_u32) to the last one
marks = [r["start"] for r in ks if "k_copy_u32" in r["name"]]
t_from = marks[-2] if len(marks) >= 2 else ks[0]["start"]
last = [r for r in ks if r["start"] >= t_from]
base = last[0]["start"]
print(f"{len(ks)} kernels in 3 steps; last step {len(last)} kernels, {last[-1]['end'] - base:.1f} us")
busy = 0.0
cur_end = base
for r in last:
    gap = r["start"] - cur_end
    if gap > 0:
        busy += 0
    print(f"{r['start'] - base:9.1f} {r['end'] - r['start']:8.1f} s{r['stream']:<3} gap{max(0.0, r['start'] - cur_end):6.1f}  {r['name'][:80]}")
    cur_end = max(cur_end, r["end"])
# union of busy intervals
iv = sorted((r["start"], r["end"]) for r in last)
tot = 0.0
cs, ce = iv[0]
for s_, e_ in iv[1:]:
    if s_ > ce:
        tot += ce - cs
        cs, ce = s_, e_
    else:
        ce = max(ce, e_)
tot += ce - cs
print(f"busy (any kernel running) {tot:.1f} us of {last[-1]['end'] - base:.1f} us")
if out_path:
    json.dump(last, open(out_path, "w"))
# host-side runtime API calls (CUPTI) over the same window
api = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")]
api.sort(key=lambda e: e.time_range.start)
print("---- host runtime calls (last step window) ----")
for e in api:
    if e.time_range.start >= base - 200:
        print(f"{e.time_range.start - base:9.1f} dur{e.time_range.end - e.time_range.start:7.1f}  {e.name}")
