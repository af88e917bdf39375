#!/usr/bin/env python
"""Benchmark: 1080p frames/s of the per-frame temporal-consistency step
(flow + warp + blend + solve), BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--flow fp32|bf16|constant] [--height H --width W]

One process per GPU (torchrun for N > 1).  Streams are independent (SURVEY
§8(e)): every rank runs its own 1080p stream; torch.distributed is used only
for the timing barrier and the max over ranks, never on the data path ->
"scaling": "weak".

A step = one stabilize_step of a 1920x1080 RGB stream with the lite flow CNN
(BASELINE config 2: fp32 flow, interactive local/global blend): push the next
(input, processed) pair; the network computes the new frame's feature pyramid
and the two flows t->t-1, t->t+1 into the session's flow slots; the fused
warp/weights/blend pass (K1); the 150-iteration screened-Poisson solve (K2);
commit.  The consistency params alternate per frame (k1/k2 0.3/0.5 <-> 0.5/0.3,
lambda 2.0 <-> 0.5).

`value` is device-timed (one CUDA event pair on the session stream around the
K steps; no L2 flush -- each step touches several times the L2) with the
frames already in HBM; `e2e` is the same step
through the C ABI from pinned host buffers (H2D of the pair and D2H of O_t in
the timed region).  `--impl reference` times the CPU restatement of the
reference step (oracle/, all host threads) on a bounded sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W = 1080, 1920
METRIC = "1080p frames/s (flow+warp+blend), per stream and box aggregate at 1/2/4/8 GPU"
SOLVER_K = 8  # iterations per temporally-blocked solver pass (csrc/solver.cu)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--flow", default="fp32", choices=["fp32", "bf16", "dis", "constant"])
    ap.add_argument("--height", type=int, default=H)
    ap.add_argument("--width", type=int, default=W)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=1,
                    help="concurrent independent video streams per GPU (BASELINE configs[4]); "
                         "each has its own session on its own CUDA stream, driven by its own "
                         "host thread")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def params_for(t):
    from paper_2301_00750_b200.consistency import ConsistencyParams

    if t % 2 == 0:
        return ConsistencyParams(k1=0.3, k2=0.5, lam=2.0)
    return ConsistencyParams(k1=0.5, k2=0.3, lam=0.5)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU restatement (oracle/): the reference arm and the cpu_baseline leg
def _cpu_step_seconds(h, w, flow_kind, budget_s):
    """Seconds per full step of the CPU restatement on all host threads:
    consistency step (C, OpenMP) timed in full; the flow CNN (numpy restatement)
    timed on a 1/16-area crop and scaled by pixel count (one new pyramid + two
    estimator passes per step, like the GPU step)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import flownet_oracle as fo
    import oracle as orc
    from paper_2301_00750_b200 import liteflownet as lf
    from paper_2301_00750_b200 import synthetic

    orc.build()
    cores = os.cpu_count() or 1
    orc.set_threads(cores)
    seq = synthetic.translating_sequence(frames=3, height=h, width=w, step=(2, 1), seed=0)
    fp = orc.constant_flow(h, w, 2, 1, -1)
    fn = orc.constant_flow(h, w, 2, 1, 1)
    cons = []
    while not cons or (sum(cons) < budget_s and len(cons) < 3):
        t0 = time.perf_counter()
        orc.run_step(seq.inputs[0], seq.processed[0], seq.inputs[1], seq.processed[1],
                     seq.inputs[2], seq.processed[2], seq.processed[0], fp, fn, orc.Params())
        cons.append(time.perf_counter() - t0)
    t_cons = sum(cons) / len(cons)
    t_flow = 0.0
    sample = f"{len(cons)} full {w}x{h} consistency steps (oracle/streamstab_oracle.c, {cores} threads)"
    if flow_kind == "dis":
        sample += " (DIS flow not included: no CPU restatement of it on the box)"
    if flow_kind in ("fp32", "bf16"):
        ch, cw = max(64, h // 4), max(64, w // 4)
        scale = (math.ceil(h / 64) * math.ceil(w / 64)) / (math.ceil(ch / 64) * math.ceil(cw / 64))
        wts = lf.make_weights(0)
        a = np.ascontiguousarray(seq.inputs[1][:ch, :cw])
        b = np.ascontiguousarray(seq.inputs[0][:ch, :cw])
        t0 = time.perf_counter()
        pa = fo.pyramid(wts, a)
        t_pyr = time.perf_counter() - t0
        pb = fo.pyramid(wts, b)
        t0 = time.perf_counter()
        fo.flow(wts, a, b, pyr1=pa, pyr2=pb)
        t_est = time.perf_counter() - t0
        t_flow = scale * (t_pyr + 2 * t_est)
        sample += (f" + flow CNN restatement (oracle/flownet_oracle.py, numpy) timed on a "
                   f"{cw}x{ch} crop and scaled x{scale:.1f} by area")
    return t_cons + t_flow, cores, sample


def run_reference(args, rank, world):
    if rank != 0:
        return
    h, w = args.height, args.width
    steps = max(1, min(args.steps, 3))
    warm = 1 if args.warmup > 0 else 0  # one untimed sample (each is ~4 s of CPU work)
    for _ in range(warm):
        _cpu_step_seconds(h, w, args.flow, budget_s=10.0)
    secs, cores, sample = [], 0, ""
    for _ in range(steps):
        s, cores, sample = _cpu_step_seconds(h, w, args.flow, budget_s=10.0)
        secs.append(s)
    sec = sum(secs) / len(secs)
    fps = 1.0 / sec
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(fps, 5), "unit": "frames/s",
        "n_gpus": world, "steps": len(secs), "warmup": warm, "ms_per_step": round(sec * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{w}x{h} single stream, default preset, 150 iterations, "
                               f"flow={args.flow}"},
        "cpu_baseline": {"value": round(fps, 5), "unit": "frames/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(fps, 5), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2301_00750_b200 as ss
    from paper_2301_00750_b200 import _lib
    from paper_2301_00750_b200.consistency import _run_step, _start_flow_to_prev
    from paper_2301_00750_b200.synthetic import DeviceSequence

    h, w = args.height, args.width
    L = _lib.lib()
    seq = DeviceSequence(h, w, step=(2, 1), seed=rank)
    if args.flow == "constant":
        flow = ss.ConstantFlow(2, 1)
    elif args.flow == "dis":
        from paper_2301_00750_b200.flow import BuiltinFlow

        flow = BuiltinFlow()  # the reference's default provider (flow.py:361-369)
    else:
        flow = ss.LiteFlowNet(seed=0, precision=args.flow)
    # frames are generated in HBM before any timed region (a pool cycled by
    # position; the consistency step never sees the generator)
    pool_n = 16
    pool = [seq.frame(k + 1) for k in range(pool_n)]
    torch.cuda.synchronize()
    if args.streams > 1:
        run_multi(args, torch, dist, rank, world, local, L, ss, flow, pool)
        return
    state = ss.SessionState(params=params_for(0))
    stream = torch.cuda.current_stream()
    pos = 0

    def push():
        nonlocal pos
        pos += 1
        i, p = pool[(pos - 1) % pool_n]
        state.push_pair(pos, i, p)

    push()
    push()

    def step():
        _start_flow_to_prev(state, flow)  # stabilize_stream's order
        push()
        # stage the next pair (device -> device on the session's upload
        # stream, overlapping this step): ss_step then also computes its
        # pyramid behind the solver, and the next push swaps it in
        i2, p2 = pool[pos % pool_n]
        _check(L.ss_stage_pair(state.handle, pos + 1, i2.data_ptr(), p2.data_ptr(), _lib.SS_F32,
                               _lib.SS_DEVICE), L)
        state.params = params_for(pos)
        _run_step(state, flow, with_next=True, return_host=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-timed region -------------------------------------------------
    sampler = ClockSampler(local)
    # one event pair around all K steps: ss_step pre-launches the next step's
    # pyramid and flow t+1 -> t behind its solver, so per-step intervals would
    # miss the work between one step's end and the next one's start.  The
    # region ends with the session's internal streams joined, so it holds
    # exactly K pre-launched pyramids and flows (the first ones ran during
    # warm-up).  No L2 flush: each step touches > 0.5 GB (ring frames, both
    # flows' activations, solver iterates), several times the 126 MB L2.
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_end = torch.cuda.Event(enable_timing=True)
    flow_ms, blend_ms, solve_ms = [], [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    launches0 = int(L.ss_kernel_launches())
    ev_start.record(stream)
    for k in range(args.steps):
        step()
        tm = state.last_timing
        flow_ms.append(tm.flow_ms)
        blend_ms.append(tm.warp_blend_ms)
        solve_ms.append(tm.solve_ms)
    _check(L.ss_session_join(state.handle), L)
    ev_end.record(stream)
    torch.cuda.synchronize()
    launches = int(L.ss_kernel_launches()) - launches0  # this library's kernels, timed steps
    clocks = sampler.stop()
    total_ms = ev_start.elapsed_time(ev_end)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * 1e3 / ms_per_step  # frames/s over all ranks (one stream each)

    e2e = None if args.no_e2e else run_e2e(args, L, state, pool, flow, torch, dist)

    # ---- roofline: stage times are CUDA events on the session stream ----------
    med = lambda xs: sorted(xs)[len(xs) // 2]  # noqa: E731
    med_flow, med_blend, med_solve = med(flow_ms), med(blend_ms), med(solve_ms)
    n_pass = math.ceil(150 / SOLVER_K)
    per_pass_ms = med_solve / n_pass
    flops_per_pass = 14.0 * h * w * 3 * SOLVER_K  # algorithmic FP32 ops, SURVEY 8(d)
    fp32_peak = 148 * 128 * 1.965e9 / 1e12
    achieved = flops_per_pass / (per_pass_ms * 1e-3) / 1e12
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    bf16_peak = float(peaks.get("bf16_tflops_sustained", 1412.7))
    k1_gbs = 130.0 * h * w / (med_blend * 1e-3) / 1e9
    traffic = _traffic_table()
    solver_line = {
        "kernel": f"k_sgd_tma<{SOLVER_K}> (solver pass = {SOLVER_K} SGD-momentum iterations)",
        "bound": "fp32", "achieved": round(achieved, 3), "peak": round(fp32_peak, 2),
        "unit": "TFLOP/s", "frac": round(achieved / fp32_peak, 4),
        "traffic": traffic.get("k_sgd_tma<8> solver pass") if SOLVER_K == 8 else None,
        "peak_source": "derived: 148 SMs x 128 FP32 lanes x 1965 MHz non-FMA op rate "
                       "(MEASURED_PEAKS.json has no FP32 entry)",
        "launch_ms": round(per_pass_ms, 5), "stage_ms": round(med_solve, 4)}
    k1_line = {
        "kernel": "k_presolve (K1 fused warp+weights+blend)", "bound": "hbm",
        "achieved": round(k1_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(k1_gbs / hbm_peak, 4), "traffic": traffic.get("k_presolve K1"),
        "launch_ms": round(med_blend, 5),
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"}
    if args.flow in ("constant", "dis"):
        roofline = dict(solver_line, secondary=[k1_line])
    else:
        # the flow network is the largest stage; its heaviest kernel is the
        # 1/8-resolution first estimator conv, timed live on the session's
        # buffers (CUDA events, 20 launches)
        cms, cfl = ctypes.c_float(0.0), ctypes.c_double(0.0)
        _check(L.ss_session_time_conv(state.handle, 3, 20, ctypes.byref(cms), ctypes.byref(cfl)), L)
        conv_tf = cfl.value / (cms.value * 1e-3) / 1e12
        # 3xTF32: tf32 runs at half the bf16 rate and each fp32 product is 3 MMAs
        conv_peak = bf16_peak if args.flow == "bf16" else bf16_peak / 6.0
        roofline = {
            "kernel": "k_conv_tc3<%d,1,0> est3_1 (1/8-res 3x3 conv, 147 live -> 128 ch; TMA halo tiles, "
                      "tcgen05/TMEM, %s)" % ((0, "bf16 operands") if args.flow == "bf16" else (1, "3xTF32")),
            "bound": "tensor", "achieved": round(conv_tf, 2), "peak": round(conv_peak, 1),
            "unit": "TFLOP/s", "frac": round(conv_tf / conv_peak, 4),
            "traffic": traffic.get("k_conv_tc3 est3_1 " + ("bf16" if args.flow == "bf16" else "fp32")),
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained" if args.flow == "bf16"
                            else "derived: MEASURED_PEAKS bf16 sustained / 2 (tf32 rate) / 3 "
                                 "(3xTF32 MMAs per fp32 product)"),
            "launch_ms": round(cms.value, 5),
            "flow_stage": {"ms": round(med_flow, 4), "gflop": 131.0,
                           "achieved_tflops": round(131.0 / med_flow, 2)},
            "secondary": [solver_line, k1_line],
        }
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, cores, sample = _cpu_step_seconds(h, w, args.flow, budget_s=10.0)
        cpu = {"value": round(1.0 / sec, 5), "unit": "frames/s", "cores": cores, "kind": "port",
               "sample": sample}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{w}x{h} single stream per GPU, flow={args.flow} + "
                               "default preset with per-frame interactive k1/k2/lambda schedule, "
                               "150 solver iterations",
                   "flow": {"fp32": "lite flow CNN, fp32-class (3xTF32 tcgen05 convs, fp32 "
                                    "activations), random-init seeded weights",
                            "bf16": "lite flow CNN, bf16 tcgen05 convs, random-init seeded "
                                    "weights",
                            "dis": "reference built-in DIS flow (BuiltinFlow, FlowOptions()) on "
                                   "GPU, bit-identical to flow.py on the golden cases",
                            "constant": "ConstantFlow(2,1) on device"}[args.flow],
                   "streams_per_gpu": 1,
                   "l2": "not flushed: each step touches > 0.5 GB (frames, two flows' activations, solver iterates) >> 126 MB L2",
                   "stage_ms_median": {"flow": round(med_flow, 4), "warp_blend": round(med_blend, 4),
                                       "solve": round(med_solve, 4)}},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_multi(args, torch, dist, rank, world, local, L, ss, flow, pool):
    """S independent streams per GPU (BASELINE configs[4]): one session per
    stream, each on its own CUDA stream and driven by its own host thread
    (the C ABI releases the GIL), so their kernels overlap on the GPU.  Device
    time = earliest start event to latest end event over the streams (CUDA
    events), max over ranks; the streams' working set (S x 0.6 GB) is far
    larger than L2, so no flush is needed between steps."""
    from paper_2301_00750_b200.consistency import _run_step, _start_flow_to_prev

    S = args.streams
    pool_n = len(pool)
    streams = [torch.cuda.Stream() for _ in range(S)]
    states, pos = [], [0] * S
    for s_ in range(S):
        with torch.cuda.stream(streams[s_]):
            states.append(ss.SessionState(params=params_for(0)))

    def step(s_):
        st = states[s_]
        _start_flow_to_prev(st, flow)
        pos[s_] += 1
        i, p = pool[(pos[s_] + 3 * s_ - 1) % pool_n]
        st.push_pair(pos[s_], i, p)
        st.params = params_for(pos[s_])
        _run_step(st, flow, with_next=True, return_host=False)

    for s_ in range(S):  # prime + warm up serially (one-time setup, graph capture)
        with torch.cuda.stream(streams[s_]):
            for _ in range(2):
                pos[s_] += 1
                i, p = pool[(pos[s_] + 3 * s_ - 1) % pool_n]
                states[s_].push_pair(pos[s_], i, p)
            for _ in range(args.warmup):
                step(s_)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(S)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(S)]
    gate = threading.Barrier(S)
    errors = []

    def worker(s_):
        try:
            with torch.cuda.stream(streams[s_]):
                gate.wait()
                ev0[s_].record(streams[s_])
                for _ in range(args.steps):
                    step(s_)
                _check(L.ss_session_join(states[s_].handle), L)
                ev1[s_].record(streams[s_])
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ref = torch.cuda.Event(enable_timing=True)
    ref.record()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = int(L.ss_kernel_launches())
    threads = [threading.Thread(target=worker, args=(s_,)) for s_ in range(S)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    launches = int(L.ss_kernel_launches()) - launches0
    clocks = sampler.stop()
    if errors:
        raise errors[0]
    total_ms = (max(ref.elapsed_time(e) for e in ev1) - min(ref.elapsed_time(e) for e in ev0))
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    frames = world * S * args.steps
    value = frames / (total_ms * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.flow != "bf16" else "bf16", "data": "synthetic",
        "config": {"workload": f"{args.width}x{args.height}, {S} concurrent streams per GPU "
                               f"(configs[4]), flow={args.flow}, default preset with per-frame "
                               "interactive schedule, 150 solver iterations",
                   "streams_per_gpu": S, "per_stream_fps": round(value / (world * S), 3),
                   "l2": "not flushed: working set of the concurrent streams >> L2"},
        "e2e": None, "gpu_launches": launches, "clocks": clocks,
        "roofline": None, "cpu_baseline": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_e2e(args, L, state, pool, flow, torch, dist):
    """The same step through the C ABI from pinned host memory."""
    from paper_2301_00750_b200 import _lib
    from paper_2301_00750_b200._dev import params_struct

    h, w = args.height, args.width
    n_host = 4
    host_i = [pool[k][0].cpu().pin_memory() for k in range(n_host)]
    host_p = [pool[k][1].cpu().pin_memory() for k in range(n_host)]
    # two pinned result buffers: each step's result is read back with
    # ss_output_async, overlapping the next step (one copy in flight)
    outs = [torch.empty((h, w, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    sess = state.handle
    pos = [int(L.ss_solved_through(sess)) + 1]  # last pushed position
    use_cnn = args.flow in ("fp32", "bf16")
    if use_cnn:
        _check(L.ss_session_attach_flownet(sess, flow.handle()), L)

    def step(k):
        pos[0] += 1
        if use_cnn:
            # flow t -> t-1 needs only buffered frames: start it on the side
            # stream first so the host->device copy of frame t+1 overlaps it
            # (the order consistency.stabilize_stream uses)
            _check(L.ss_session_compute_flow(sess, 0), L)
        _check(L.ss_push_pair(sess, pos[0], host_i[k % n_host].data_ptr(),
                              host_p[k % n_host].data_ptr(), _lib.SS_F32, _lib.SS_HOST), L)
        t = int(L.ss_solved_through(sess)) + 1
        if use_cnn:
            _check(L.ss_session_compute_flow(sess, 1), L)
        elif args.flow == "dis":
            for which in (0, 1):
                _check(L.ss_session_compute_dis_flow(sess, which, 5, 9, 4, 1), L)
        else:
            _check(L.ss_set_constant_flow(sess, 0, 2.0, 1.0, -1), L)
            _check(L.ss_set_constant_flow(sess, 1, 2.0, 1.0, 1), L)
        # the next pair's upload overlaps this step (ss_push_pair swaps it in)
        _check(L.ss_stage_pair(sess, pos[0] + 1, host_i[(k + 1) % n_host].data_ptr(),
                               host_p[(k + 1) % n_host].data_ptr(), _lib.SS_F32, _lib.SS_HOST), L)
        prm = params_struct(params_for(t))
        it = ctypes.c_int(0)
        _check(L.ss_step(sess, 1, ctypes.byref(prm), ctypes.byref(it)), L)
        _check(L.ss_output_async(sess, outs[k % 2].data_ptr(), _lib.SS_F32, _lib.SS_HOST), L)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    # three back-to-back windows of K steps (host wall clock, device
    # synchronised at both ends of each); the median window is reported --
    # a single window of a host-driven loop is sensitive to host jitter
    dts, k0 = [], args.warmup
    for _ in range(3):
        t0 = time.perf_counter()
        for k in range(k0, k0 + args.steps):
            step(k)
        _check(L.ss_output_wait(sess), L)
        torch.cuda.synchronize()
        dts.append(time.perf_counter() - t0)
        k0 += args.steps
    dt = sorted(dts)[1]
    if dist:
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    world = dist.get_world_size() if dist else 1
    return {"value": round(world * args.steps / dt, 3), "unit": "frames/s",
            "windows_fps": [round(world * args.steps / x, 2) for x in dts],
            "h2d_bytes_per_step": 2 * h * w * 3 * 4, "d2h_bytes_per_step": h * w * 3 * 4,
            "path": "C ABI per step: ss_session_compute_flow(0) + ss_push_pair (pair staged from "
                    "pinned host f32 by the previous step's ss_stage_pair: its upload overlaps that "
                    "step) + ss_session_compute_flow(1) + ss_stage_pair(next pair) + ss_step + "
                    "ss_output_async (pinned, double-buffered: the result copy overlaps the next step)",
            "timer": "host wall clock around K steps, device synchronised at both ends; median of "
                     "3 consecutive windows"}


def _traffic_table():
    """DRAM bytes per launch of the roofline kernels, from the committed ncu
    --set full captures (profiles/r01_traffic.json; tools/profile_round.sh)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            tab = json.load(f)["kernels"]
    except (OSError, KeyError, ValueError):
        return {}
    return {k: v["traffic_bytes"] for k, v in tab.items()}


def _check(rc, L):
    if rc != 0:
        raise RuntimeError(f"streamstab_b200 error {rc}: {L.ss_last_error().decode()}")


if __name__ == "__main__":
    main()
