#!/usr/bin/env python
"""AERO-MPPI plan-cycle benchmark (BASELINE.json metric: rollout-steps/s and
p50 plan-cycle latency).

Default workload = config C5 (the largest single-GPU config): 4096
independent synthetic scenes (forest / verticals / inclines, 20k LiDAR points
each), every scene planned with 4x2 anchors x 256 samples x 30 steps.  A
"step" is one full plan cycle (build_snapshot + plan_step) for every scene.
Under torchrun every rank plans its own --scenes scenes (scene ids
rank*S .. rank*S+S-1): weak scaling, no data-path collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value  : rollout-steps/s with inputs resident in HBM (amppi_cycle_batch_device)
e2e    : same metric through the host-pointer API amppi_cycle_batch (pinned
         host inputs copied in and results copied out every step)
latency: p50 / p99 of host-to-host amppi_snapshot + amppi_plan on a C1 cycle
roofline / cpu_baseline / clocks / gpu_launches: see DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rollout-steps/s (anchors×samples×horizon); p50 plan-cycle latency ms"
FLOPS_PER_STEP = 440  # algorithmic FP32 flops per rollout-step (FMA = 2)
TRAFFIC_BYTES_PER_LAUNCH = 193.6e6  # bound + main screening pass DRAM bytes, profiles/r01_c5_full.md
ISSUE_ACTIVE_FRAC = 0.722  # main screening pass issue-slot utilisation, same capture


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c4", "c2"],
                    help="c5: batched scenes (default, the driver's line); c4: 64x8192x50 ensemble, samples "
                         "sharded over the ranks with NCCL; c2: 200-cycle closed loop on the device")
    ap.add_argument("--scenes", type=int, default=4096)
    ap.add_argument("--points", type=int, default=20000)
    ap.add_argument("--latency-cycles", type=int, default=1000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
def cpu_baseline(data: dict, cfg, scene_ids, seconds: float) -> dict:
    """Oracle restatement (oracle/, the reference's parallel_for threading with
    hardware_concurrency workers) on a time-bounded sample of the workload."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    from oracle_py import Oracle

    orc = Oracle()
    cores = os.cpu_count() or 1
    orc.set_workers(cores)
    ocfg = orc.config(cfg)
    off = data["offsets"]
    done, t0 = 0, time.perf_counter()
    for s in scene_ids:
        pts = data["xyz"][off[s]:off[s + 1]].astype(np.float64)
        snap = orc.snapshot(pts, data["poses"][s], cfg.r_max)
        g = data["goals"][s]
        orc.plan(snap, ocfg, data["states"][s], g[0:3], g[3:6], g[6:10], None, data["last"][s],
                 int(data["cycles"][s]), int(data["seeds"][s]))
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    steps = done * cfg.grid.count() * cfg.mppi.rollouts * cfg.mppi.horizon * cfg.mppi.iterations
    return {"value": steps / dt, "unit": "rollout-steps/s", "cores": cores, "kind": "port",
            "sample": f"{done} scenes of the workload (build_snapshot + plan_step each), {dt:.1f} s, "
                      f"oracle/ restatement, parallel_for over {cores} threads"}


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path (the
    oracle restatement; the reference itself cannot be built here, SURVEY.md
    §0) on this box's host cores, same config / metric, bounded samples."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    from oracle_py import Oracle

    from paper_2509_17340_b200.workloads import plan_config, rollout_steps

    cfg = plan_config()
    orc = Oracle()
    cores = os.cpu_count() or 1
    orc.set_workers(cores)
    ocfg = orc.config(cfg)
    # inputs from the oracle's own simulator: C5 scene family, 20k points each
    n_sample = 3
    scenes = []
    for s in range(n_sample):
        sc = orc.scene(1 + s % 3, s + 1)
        rng = np.random.default_rng(12345 + s)
        start = np.array([rng.uniform(1.0, 30.0), rng.uniform(-8.0, 8.0), 2.0])
        frames, pose = [], None
        for f in range(20):
            pose = np.concatenate([start + [0.06 * f, 0, 0], [1, 0, 0, 0], [3.0, 0, 0]])
            frames.append(sc.lidar(pose, 1000 * s + f))
        pts = np.concatenate(frames)[: args.points]
        scenes.append((pts, pose))
    goal_q = np.array([1.0, 0, 0, 0])

    def step(i):
        for pts, pose in scenes:
            snap = orc.snapshot(pts, pose, cfg.r_max)
            orc.plan(snap, ocfg, pose, [45.0, 0, 2.0], [0, 0, 0], goal_q, None, [9.81, 0, 0, 0], 100 + i, 1)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = rollout_steps(cfg, n_sample) * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": "rollout-steps/s", "impl": "reference", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C5 sample: forest/verticals/inclines scenes x (4x2 anchors x 256 samples x 30 "
                                   "steps), 20k points each", "scenes_per_step": n_sample,
                       "anchors": cfg.grid.count(), "samples": cfg.mppi.rollouts, "horizon": cfg.mppi.horizon},
            "cpu_baseline": {"value": value, "unit": "rollout-steps/s", "cores": cores, "kind": "port",
                             "sample": f"{n_sample} scenes per step, oracle/ restatement of build_snapshot + "
                                       f"plan_step (reference not buildable: Eigen/vendor absent)"},
            "e2e": {"value": value, "unit": "rollout-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_b200(args):
    import numpy as np
    import torch

    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State, load
    from paper_2509_17340_b200.workloads import plan_config, rollout_steps, scenes

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # a dedicated (non-default) stream: the planner launches on it and the
    # timing events are recorded on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    cfg = plan_config()
    S = args.scenes  # per rank (weak scaling)
    S_total = S * ws
    first = rank * S
    data = scenes(S, points=args.points, frames=20, first=first, device=local)
    P = int(data["offsets"][-1])
    planner = Planner(cfg, device=local, precision=32, max_scenes=S, max_points=max(P, 1 << 16), profile=True,
                      stream=stream.cuda_stream)

    def tens(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a).view(dt) if a.dtype != dt else np.ascontiguousarray(a))

    dvals = {
        "xyz": torch.from_numpy(data["xyz"]).to(dev),
        "offsets": torch.from_numpy(data["offsets"]).to(dev),
        "poses": torch.from_numpy(data["poses"]).to(dev),
        "states": torch.from_numpy(data["states"]).to(dev),
        "goals": torch.from_numpy(data["goals"]).to(dev),
        "last": torch.from_numpy(data["last"]).to(dev),
        "cycles": torch.from_numpy(data["cycles"].view(np.int64)).to(dev),
        "seeds": torch.from_numpy(data["seeds"].view(np.int64)).to(dev),
    }
    N, M = cfg.mppi.horizon, cfg.grid.count()
    dout = {"status": torch.zeros(S, dtype=torch.int32, device=dev), "winner": torch.zeros(S, dtype=torch.int32, device=dev),
            "control": torch.zeros(S, 4, dtype=torch.float64, device=dev),
            "winner_nominal": torch.zeros(S, N, 4, dtype=torch.float64, device=dev),
            "stage2": torch.zeros(S, M, dtype=torch.float64, device=dev),
            "breakdown": torch.zeros(S, 5, dtype=torch.float64, device=dev)}
    dptr = {k: v.data_ptr() for k, v in dvals.items()}
    optr = {k: v.data_ptr() for k, v in dout.items()}

    def step():
        dvals["cycles"].add_(1)  # fresh perturbation streams every cycle
        planner.cycle_batch_device(dptr, optr, S, cfg.r_max)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    planner.kernel_times_reset()
    sampler = ClockSampler(local)
    sampler.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    planner.synchronize()
    ktimes = planner.kernel_times()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_steps = rollout_steps(cfg, S_total) * args.steps
    value = total_steps / (ms_max / 1e3)
    n_ok = int((dout["status"] == 0).sum().item())
    launches = sum(v[1] for v in ktimes.values())
    # Per-kernel times for the roofline and the `kernels` table: a short extra
    # pass with the whole batch as one chunk.  (The timed steps above split it
    # into chunks on concurrent streams, where a kernel's events also span the
    # other streams' kernels.)
    planner.set_schedule(device_chunks=1)
    step()
    torch.cuda.synchronize(dev)
    planner.kernel_times_reset()
    for _ in range(min(args.steps, 5)):
        step()
    planner.synchronize()
    ktimes = planner.kernel_times()
    planner.set_schedule(device_chunks=0)

    # roofline of the dominant kernel (FP32 stage-I rollouts)
    lib = load()
    import ctypes

    peak = ctypes.c_double()
    pms = ctypes.c_double()
    lib.amppi_probe_fp32_peak(local, ctypes.byref(peak), ctypes.byref(pms))
    # the FP32 stage-I screening = bound pass (first 32 samples per instance)
    # + main pass (the rest): together one evaluation of every rollout-step
    k_ms, k_n = ktimes.get("k_stage1_f32", (float("nan"), 1))
    b_ms = ktimes.get("k_stage1_f32_bound", (0.0, 1))[0]
    per_launch_flops = FLOPS_PER_STEP * rollout_steps(cfg, S) / cfg.mppi.iterations
    screen_ms = (k_ms + b_ms) / k_n
    achieved = per_launch_flops / (screen_ms / 1e3) / 1e12
    share = (k_ms + b_ms) / sum(v[0] for v in ktimes.values())

    # e2e through the host-pointer API
    e2e = None
    if not args.no_e2e:
        # the user-facing call, without the per-kernel timing events of the
        # device-resident measurement above
        planner.close()
        planner = Planner(cfg, device=local, precision=32, max_scenes=S, max_points=max(P, 1 << 16),
                          stream=stream.cuda_stream)
        pinned_xyz = torch.from_numpy(data["xyz"]).pin_memory()  # keep alive while in use
        host = {k: data[k] for k in ("offsets", "poses", "states", "goals", "last", "cycles", "seeds")}
        host["xyz"] = pinned_xyz.numpy()
        for i in range(max(1, args.warmup)):
            planner.cycle_batch(host["offsets"], host["xyz"], host["poses"], host["states"], host["goals"],
                                host["last"], host["cycles"] + i, host["seeds"])
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for i in range(args.steps):
            planner.cycle_batch(host["offsets"], host["xyz"], host["poses"], host["states"], host["goals"],
                                host["last"], host["cycles"] + 1000 + i, host["seeds"])
        el = time.perf_counter() - t0
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
        h2d = (data["xyz"].nbytes + data["offsets"].nbytes + data["poses"].nbytes + data["states"].nbytes +
               data["goals"].nbytes + data["last"].nbytes + data["cycles"].nbytes + data["seeds"].nbytes)
        d2h = S * (4 + 4 + 8 * 4 + 8 * N * 4 + 8 * M + 8 * 5)
        e2e = {"value": total_steps / el, "unit": "rollout-steps/s", "h2d_bytes_per_step": int(h2d) * ws,
               "d2h_bytes_per_step": int(d2h) * ws, "ms_per_step": 1000 * el / args.steps}

    latency = None
    cpu = None
    if rank == 0:
        # p50 plan-cycle latency: C1 single scene, host-to-host through the C
        # ABI (amppi_snapshot + amppi_plan with caller-owned result buffers, as
        # a C++ caller of the shim does), and through the Python wrapper
        import ctypes

        from paper_2509_17340_b200 import _abi

        one = scenes(1, points=args.points, frames=20, first=0, kinds=1, device=local)
        lp = Planner(cfg, device=local, precision=32, max_scenes=1, max_points=1 << 16)
        pts = np.ascontiguousarray(one["xyz"], dtype=np.float32)
        x = State.from_array(one["states"][0])
        goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
        la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
        M1, N1 = cfg.grid.count(), cfg.mppi.horizon
        xs, gs, lc = x.to_c(), goal.to_c(), la.to_c()
        res = _abi.PlanResult()
        nominal = np.zeros((M1, N1, 4))
        res.nominal = nominal.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        prev = np.zeros((N1, 4))
        prev_p = prev.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        pts_p = pts.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        lib_c = lp.lib

        def c_abi_cycle(i, prev_len):
            rc = lib_c.amppi_snapshot(lp._h, pts_p, len(pts), ctypes.byref(xs), ctypes.c_double(cfg.r_max))
            rc |= lib_c.amppi_plan(lp._h, ctypes.byref(xs), ctypes.byref(gs), prev_p, prev_len, ctypes.byref(lc),
                                   ctypes.c_uint64(100 + i), ctypes.c_uint64(1), None, ctypes.byref(res))
            return rc

        lat, prev_len = [], 0
        for i in range(100 + args.latency_cycles):
            t0 = time.perf_counter()
            rc = c_abi_cycle(i, prev_len)
            t1 = time.perf_counter()
            if rc != 0:
                raise RuntimeError(f"C1 cycle failed ({rc})")
            prev[:] = nominal[res.winner]
            prev_len = N1
            if i >= 100:
                lat.append(1000 * (t1 - t0))
        lat_py, prevn = [], None
        for i in range(100 + args.latency_cycles // 2):
            t0 = time.perf_counter()
            snap = lp.build_snapshot(pts, x, cfg.r_max)
            r = lp.plan_step(x, goal, snap, prevn, la, 100 + i, 1, want_rollout=False)
            t1 = time.perf_counter()
            prevn = r.per_instance[r.winner].nominal
            if i >= 100:
                lat_py.append(1000 * (t1 - t0))
        lp.close()
        lat.sort()
        lat_py.sort()
        latency = {"workload": "C1: one forest scene, 20k float32 points (pageable host buffer), 4x2 anchors x 256 x "
                               "30, host-to-host amppi_snapshot + amppi_plan through the C ABI, warm nominal",
                   "p50_ms": lat[len(lat) // 2], "p99_ms": lat[int(0.99 * len(lat))], "cycles": len(lat),
                   "p50_ms_python_api": lat_py[len(lat_py) // 2],
                   "rollout_steps_per_s_at_p50": rollout_steps(cfg, 1) / (lat[len(lat) // 2] / 1e3)}
        # the paper's default ensemble (M = 15 = 5x3 anchors, K = 256, N = 25), whose full pipeline runs
        # at 500 Hz (2.0 ms per cycle) on an RTX 4080 SUPER, same scene, Python API
        pcfg = plan_config(5, 3, K=256, N=25)
        pp = Planner(pcfg, device=local, precision=32, max_scenes=1, max_points=1 << 16)
        lat_p, prevp = [], None
        for i in range(100 + args.latency_cycles // 2):
            t0 = time.perf_counter()
            snap = pp.build_snapshot(pts, x, pcfg.r_max)
            r = pp.plan_step(x, goal, snap, prevp, la, 100 + i, 1, want_rollout=False)
            t1 = time.perf_counter()
            prevp = r.per_instance[r.winner].nominal
            if i >= 100:
                lat_p.append(1000 * (t1 - t0))
        pp.close()
        lat_p.sort()
        latency["paper_default"] = {"config": "5x3 anchors x 256 samples x 25 steps, same C1 scene, Python API "
                                              "(the paper: 500 Hz = 2.0 ms per cycle on an RTX 4080 SUPER)",
                                    "p50_ms": lat_p[len(lat_p) // 2], "p99_ms": lat_p[int(0.99 * len(lat_p))]}
        cpu = cpu_baseline(data, cfg, range(S), args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 stage-I screening / f64 keys, anchors, update, "
                                                             "stage II", "data": "synthetic",
            "config": {"workload": "C5: independent synthetic scenes (forest/verticals/inclines, GPU LiDAR, "
                                   f"{args.points} points each) x (4x2 anchors x 256 samples x 30 steps), one full "
                                   "plan cycle (snapshot + plan) per scene per step",
                       "scenes": S_total, "scenes_per_gpu": S, "anchors": M, "samples": cfg.mppi.rollouts, "horizon": N,
                       "iterations": cfg.mppi.iterations, "points_total": int(P) * ws,
                       "parallelism": f"scene-sharded x{ws} (weak: {S} scenes per GPU)",
                       "l2": "inputs larger than L2 (points alone %.0f MB vs 126 MB)" % (data["xyz"].nbytes / 1e6),
                       "planned_ok": n_ok},
            "latency": latency,
            "e2e": e2e,
            "roofline": {"bound": "fp32", "kernel": "k_stage1_f32_bound + k_stage1_f32 (FP32 stage-I screening)",
                         "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s", "frac": achieved / peak.value,
                         "traffic": TRAFFIC_BYTES_PER_LAUNCH,
                         "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of both kernels, ncu --set "
                                           "full, profiles/r01_c5_full.md",
                         "peak_source": "measured FFMA probe (amppi_probe_fp32_peak) in this run; CUDA-core FP32, "
                                        "not a tensor-core path",
                         "algorithmic_flops_per_launch": per_launch_flops,
                         "kernel_ms_per_launch": screen_ms, "kernel_share_of_step": share,
                         # what actually bounds it (ncu, profiles/r01_c5_full.md): warp-instruction issue;
                         # most issued instructions are the exact collision query, outside the 440 flops
                         "issue_active_frac": ISSUE_ACTIVE_FRAC,
                         "issue_source": "smsp__issue_active.avg.pct_of_peak_sustained_active of the main "
                                         "pass, ncu --set full, profiles/r01_c5_full.md"},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": int(launches),
            "kernels": {k: {"ms_total": v[0], "launches": v[1]} for k, v in sorted(ktimes.items())},
        }
        print(json.dumps(line), flush=True)
    planner.close()
    if dist:
        dist.destroy_process_group()


def run_c4(args):
    """Config C4: one forest scene, 8x8 anchors x 8192 samples x 50 steps; the
    samples of every instance are split over the ranks (global sample index in
    the RNG key) and merged with one all-reduce MIN + one all-gather per
    iteration (sharding.plan_step_sharded).  value = rollout-steps/s of the
    whole job, device time max over ranks; scaling: strong (fixed ensemble)."""
    import numpy as np
    import torch

    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State
    from paper_2509_17340_b200.sharding import TorchComm, plan_step_sharded
    from paper_2509_17340_b200.workloads import plan_config, rollout_steps, scenes

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    import torch.distributed as dist

    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    cfg = plan_config(m_h=8, m_v=8, K=8192, N=50)
    one = scenes(1, points=args.points, frames=20, first=0, kinds=1, device=local)
    planner = Planner(cfg, device=local, precision=32, max_points=1 << 16, profile=True, stream=stream.cuda_stream)
    x = State.from_array(one["states"][0])
    goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
    la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
    snap = planner.build_snapshot(one["xyz"], x, cfg.r_max)
    prev = None

    class _Single:  # one rank: the collectives are identities
        rank, world = 0, 1

        @staticmethod
        def allreduce_min(t):
            pass

        @staticmethod
        def allgather(out, t):
            out.copy_(t)

    comm = TorchComm() if ws > 1 else _Single()

    def step(i):
        nonlocal prev
        r = plan_step_sharded(planner, x, goal, snap, prev, la, 100 + i, 1, comm, want_rollout=False)
        prev = r.per_instance[r.winner].nominal
        return r

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    planner.kernel_times_reset()
    sampler = ClockSampler(local)
    sampler.start()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    kt = planner.kernel_times()
    value = rollout_steps(cfg, 1) * args.steps / (ms / 1e3)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 screening / f64 support, update, stage II", "data": "synthetic",
            "config": {"workload": "C4: one forest scene (GPU LiDAR, 20k points), 8x8 anchors x 8192 samples x "
                                   "50 steps, samples sharded over the ranks (NCCL all-reduce MIN + all-gather "
                                   "of the softmin partials per iteration); host-to-host plan_step per step",
                       "anchors": 64, "samples": 8192, "horizon": 50, "parallelism": f"sample-sharded x{ws}"},
            "clocks": clocks, "gpu_launches": int(sum(v[1] for v in kt.values())),
            "kernels": {k: {"ms_total": v[0], "launches": v[1]} for k, v in sorted(kt.items())},
        }), flush=True)
    planner.close()
    if ws > 1:
        dist.destroy_process_group()


def run_c2(args):
    """Config C2: the 200-cycle closed-loop forest flight (speed cap 7 m/s,
    4x2 anchors x 256 x 30) run entirely on the device (amppi_loop_*: LiDAR,
    point-cloud ring, snapshot, plan, vehicle step); one step = one episode of
    200 cycles.  value = rollout-steps/s of the planning inside the loop;
    cpu_baseline = the oracle's execute_cycle loop on the host cores."""
    import torch

    from paper_2509_17340_b200 import ClosedLoop, Planner
    from paper_2509_17340_b200.planner import apply_velocity_cap
    from paper_2509_17340_b200.workloads import plan_config, rollout_steps

    ws, rank, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    cfg = apply_velocity_cap(plan_config(), 7.0)
    cycles = 200
    planner = Planner(cfg, device=local, precision=32, max_points=10 * 7200)

    def episode(i):
        lp = ClosedLoop(planner, 1, 1, 31 + i, buffer_capacity=10, max_cycles=cycles)
        t0 = time.perf_counter()
        ran = lp.run(cycles)
        dt = time.perf_counter() - t0
        lp.close()
        return ran, dt

    for i in range(args.warmup):
        episode(i)
    sampler = ClockSampler(local)
    sampler.start()
    total_cycles, total_t = 0, 0.0
    for i in range(args.steps):
        ran, dt = episode(args.warmup + i)
        total_cycles += ran
        total_t += dt
    clocks = sampler.stop()
    planner.close()
    ms_cycle = 1e3 * total_t / max(total_cycles, 1)
    value = rollout_steps(cfg, 1) * total_cycles / total_t
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_py import Oracle

    orc = Oracle()
    orc.set_workers(os.cpu_count() or 1)
    lo = orc.loop(1, 1, orc.config(cfg), 31, capacity=10)
    t0 = time.perf_counter()
    n_cpu = lo.run(50)
    t_cpu = time.perf_counter() - t0
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
        "scaling": "replicas", "vs_baseline": None, "dtype": "f32 screening / f64 plan, LiDAR and vehicle",
        "data": "synthetic",
        "config": {"workload": "C2: 200-cycle closed-loop forest flight (seed 1), speed cap 7 m/s, 4x2 anchors x 256 "
                               "x 30, LiDAR + point-cloud ring + snapshot + plan + vehicle step on the device "
                               "(amppi_loop_run, one CUDA graph per cycle); one step = one episode",
                   "cycles_per_episode": cycles, "ms_per_cycle": ms_cycle},
        "cpu_baseline": {"value": rollout_steps(cfg, 1) * n_cpu / t_cpu, "unit": "rollout-steps/s",
                         "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{n_cpu} cycles of the oracle's execute_cycle loop ({1e3 * t_cpu / n_cpu:.2f} "
                                   f"ms/cycle)"},
        "clocks": clocks,
    }), flush=True)


def main():
    args = parse()
    if args.impl == "b200" and args.workload == "c4":
        run_c4(args)
    elif args.impl == "b200" and args.workload == "c2":
        run_c2(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
