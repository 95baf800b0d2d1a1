#!/usr/bin/env python
"""AERO-MPPI plan-cycle benchmark (BASELINE.json metric: rollout-steps/s and
p50 plan-cycle latency).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload c5|c4|c3|c2]

Workloads (BASELINE.json configs; one "step" = one pass of the plan path):
  c5 (default) one batch of --scenes (4096) independent synthetic scenes
     (forest / verticals / inclines, 20k LiDAR points each), every scene
     planned with 4x2 anchors x 256 samples x 30 steps (snapshot + plan).
     With N GPUs the batch is split by scene (rank r plans scenes
     [r*S/N, (r+1)*S/N)): strong scaling, no data-path collective.
  c4 one forest scene, 8x8 anchors x 8192 samples x 50 steps, the samples of
     every instance sharded over the ranks (NCCL all-reduce MIN + all-gather
     of the softmin partials, issued by the library: amppi_plan_sharded).
  c3 one ~1M-point accumulated verticals scan, snapshot + plan at C1 sizes
     (replicas across ranks).
  c2 the 200-cycle closed-loop forest flight on the device (replicas).

With --gpus N > 1 and no torchrun environment, bench.py relaunches itself
under torch.distributed.run with N ranks (one per GPU, 127.0.0.1).

value  : rollout-steps/s of the whole job, inputs resident in HBM, device
         time (CUDA events on the planner's stream) max over ranks
e2e    : the same metric through the host-pointer C ABI (inputs copied in,
         results copied out inside the timed region)
latency: (c5, rank 0) p50 / p99 of host-to-host amppi_snapshot + amppi_plan on
         the reference's own latency protocol (acceptance.cpp:339-377), with
         the oracle's p50 on the same inputs beside it
roofline / cpu_baseline / clocks / gpu_launches: see DESIGN.md §5.
--impl reference: the reference's CPU path (the oracle restatement; the
reference itself cannot be built here) on the host cores, same workload
bytes (the host twin of the input generator), same config / metric.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rollout-steps/s (anchors×samples×horizon); p50 plan-cycle latency ms"
FLOPS_PER_STEP = 440  # algorithmic FP32 flops per rollout-step (FMA = 2)
BYTES_PER_POINT = 12  # FP32 xyz read once by the keying pass
# ncu --set full of the FP32 screening kernels (bound + main pass) on the C5
# batch as one chunk: DRAM read+write per step and the main pass's issue-slot
# use (profiles/r02_c5_full.md)
TRAFFIC_BYTES_PER_LAUNCH = 195.4e6
TRAFFIC_SOURCE = "profiles/r02_c5_full.md"
ISSUE_ACTIVE_FRAC = 0.7225
# FP32 flops the two screening kernels executed in one C5 launch, counted by ncu on the SASS page
# (FFMA 2, FADD/FMUL 1, FFMA2 4, FADD2/FMUL2 2 per predicated-on thread instruction; the collision
# queries' distance arithmetic included): main pass 2.109e11 + bound pass 5.552e10
# (tools/ncu_lines.py <rep> --ops <kernel>, profiles/r02_c5_full.md)
EXECUTED_FLOPS_PER_LAUNCH = 2.109e11 + 5.552e10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c4", "c3", "c2"])
    ap.add_argument("--scenes", type=int, default=4096, help="c5: scenes in the batch (split over the ranks)")
    ap.add_argument("--points", type=int, default=20000)
    ap.add_argument("--latency-cycles", type=int, default=1000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--device-chunks", type=int, default=0, help="c5: concurrent chunks (0 = automatic)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N local ranks; returns its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Dist:
    """Rank bookkeeping and the control-plane collectives of the bench
    (barrier, max over ranks, object broadcast).  NCCL when every rank owns a
    GPU; gloo when ranks share one (a functional run on a 1-GPU box)."""

    def __init__(self):
        import torch

        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = max(1, torch.cuda.device_count())
        self.device = self.local % ndev
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(self.world)))
        self.shared_gpu = local_world > ndev
        self.dist = None
        self.backend = None
        torch.cuda.set_device(self.device)
        if self.world > 1:
            import torch.distributed as dist

            self.backend = "gloo" if self.shared_gpu else "nccl"
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            else:
                dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not self.dist:
            return v
        import torch

        dev = torch.device("cuda", self.device) if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.dist:
            return v
        import torch

        dev = torch.device("cuda", self.device) if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def broadcast(self, obj):
        if not self.dist:
            return obj
        lst = [obj]
        self.dist.broadcast_object_list(lst, src=0)
        return lst[0]

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


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
            t0 = time.time()  # sampling is live before the timed region starts
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        # one more sample after the timed region, so a region shorter than the
        # 200 ms sampling period is still bracketed by samples
        n0, t0 = len(self.lines), time.time()
        while len(self.lines) <= n0 and time.time() - t0 < 1.0:
            time.sleep(0.01)
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


def oracle():
    """The CPU oracle restatement (test infrastructure; only the CPU legs of
    the bench load it, after and outside the device-timed regions)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_py import Oracle

    orc = Oracle()
    orc.set_workers(os.cpu_count() or 1)
    return orc


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p))["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "fallback 6.65 TB/s of /opt/skills/guides/B200_PROFILING.md"


# ---------------------------------------------------------------------------
# workload definitions shared by both arms (same config dict, same bytes)
# ---------------------------------------------------------------------------
def c5_config(args, ws):
    from paper_2509_17340_b200.workloads import plan_config

    cfg = plan_config()
    conf = {"workload": "C5: one batch of independent synthetic scenes (forest/verticals/inclines, "
                        f"{args.points} LiDAR points each) x (4x2 anchors x 256 samples x 30 steps); one step = one "
                        "full plan cycle (snapshot + plan) of every scene",
            "scenes": args.scenes, "anchors": cfg.grid.count(), "samples": cfg.mppi.rollouts,
            "horizon": cfg.mppi.horizon, "iterations": cfg.mppi.iterations, "points_per_scene": args.points,
            "parallelism": f"scene-sharded x{ws} (strong: {args.scenes} scenes split over {ws} GPU(s))",
            "l2": "inputs larger than L2 (the batch's points alone are ~%.0f MB vs 126 MB)"
                  % (args.scenes * args.points * 12 / 1e6)}
    return cfg, conf


def c4_config(ws):
    from paper_2509_17340_b200.workloads import plan_config

    cfg = plan_config(m_h=8, m_v=8, K=8192, N=50)
    conf = {"workload": "C4: one forest scene (20k LiDAR points), 8x8 anchors x 8192 samples x 50 steps; one step = "
                        "one build_snapshot + plan_step, samples sharded over the ranks (amppi_plan_sharded: NCCL "
                        "all-reduce MIN + all-gather of the softmin partials per iteration)",
            "anchors": 64, "samples": 8192, "horizon": 50, "iterations": 1,
            "parallelism": f"sample-sharded x{ws} (strong)"}
    return cfg, conf


def c3_config():
    from paper_2509_17340_b200.workloads import plan_config

    cfg = plan_config()
    conf = {"workload": "C3: one ~1M-point accumulated verticals scan (scene seed 8), snapshot + plan at C1 sizes "
                        "(4x2 anchors x 256 samples x 30 steps); one step = one plan cycle",
            "points": 1_000_000, "anchors": 8, "samples": 256, "horizon": 30, "parallelism": "replicas"}
    return cfg, conf


def c4_scene(host: bool, device: int = 0):
    from paper_2509_17340_b200.workloads import scenes

    return scenes(1, points=20000, frames=20, first=0, kinds=1, device=device, host=host)


def c3_scene(host: bool, device: int = 0):
    from paper_2509_17340_b200.workloads import scenes

    # ~1M points: a slowly advancing vehicle accumulating ~330 frames
    return scenes(1, points=1_000_000, frames=600, first=7, kinds=2, device=device, host=host, frame_step=0.004)


# ---------------------------------------------------------------------------
# CPU legs (oracle)
# ---------------------------------------------------------------------------
def cpu_plan_scenes(orc, cfg, data, scene_ids, seconds: float):
    """build_snapshot + plan_step of the given scenes with the oracle until
    `seconds` pass; returns (scenes planned, elapsed s)."""
    import numpy as np

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
    return done, time.perf_counter() - t0


def latency_inputs(orc, cfg):
    """The reference's latency protocol (acceptance.cpp:339-377): the forest
    seed-1 closed loop flown 100 cycles into the clutter, then 50 plan cycles;
    the oracle's loop records the exact inputs of those 50 cycles."""
    lo = orc.loop(1, 1, orc.config(cfg), 1, capacity=20)
    lo.run(150)
    recs = lo.records()
    return recs[100:150], lo.goal()


# ---------------------------------------------------------------------------
# b200 arm
# ---------------------------------------------------------------------------
def kernel_summary(ktimes):
    return {k: {"ms_total": v[0], "launches": v[1]} for k, v in sorted(ktimes.items())}


def fp32_peak(device: int) -> float:
    from paper_2509_17340_b200 import load

    lib = load()
    peak, pms = ctypes.c_double(), ctypes.c_double()
    lib.amppi_probe_fp32_peak(device, ctypes.byref(peak), ctypes.byref(pms))
    return peak.value


def screening_roofline(ktimes, rollout_steps_per_launch: float, peak: float, total_ms: float,
                       executed_flops: float | None = None) -> dict:
    k_ms, k_n = ktimes.get("k_stage1_f32", (float("nan"), 1))
    b_ms = ktimes.get("k_stage1_f32_bound", (0.0, 1))[0]
    per_launch_flops = FLOPS_PER_STEP * rollout_steps_per_launch
    screen_ms = (k_ms + b_ms) / k_n
    achieved = per_launch_flops / (screen_ms / 1e3) / 1e12
    return {"bound": "fp32", "kernel": "k_stage1_f32_bound + k_stage1_f32 (FP32 stage-I screening)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": TRAFFIC_BYTES_PER_LAUNCH,
            "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of both kernels, ncu --set full, "
                              + TRAFFIC_SOURCE,
            "peak_source": "measured FFMA probe (amppi_probe_fp32_peak) in this run; CUDA-core FP32 (MEASURED_PEAKS"
                           ".json has no FP32 entry; its bf16 figure is a tensor-core number)",
            "algorithmic_flops_per_launch": per_launch_flops,
            "achieved_note": "effective rate: 440 flop x every rollout-step of the launch, including the steps the "
                             "abort bound proves outside the softmin support and never integrates",
            **({} if executed_flops is None else {
                "executed_flops_per_launch": executed_flops,
                "executed_tflops": executed_flops / (screen_ms / 1e3) / 1e12,
                "executed_frac": executed_flops / (screen_ms / 1e3) / 1e12 / peak,
                "executed_note": "FP32 flops the screening kernels executed in one C5 launch (ncu SASS counts, "
                                 "collision-query distance arithmetic included, " + TRAFFIC_SOURCE
                                 + ") over this run's kernel time"}),
            "kernel_ms_per_launch": screen_ms, "kernel_share_of_step": (k_ms + b_ms) / total_ms,
            "issue_active_frac": ISSUE_ACTIVE_FRAC,
            "issue_source": "smsp__issue_active.avg.pct_of_peak_sustained_active of the main pass, ncu --set full, "
                            + TRAFFIC_SOURCE}


def run_c5(args, D: Dist):
    import numpy as np
    import torch

    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.sharding import shard_ranges
    from paper_2509_17340_b200.workloads import rollout_steps, scenes

    ws, rank, device = D.world, D.rank, D.device
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(dev)  # the planner launches on it; the timing events are recorded on it
    torch.cuda.set_stream(stream)
    cfg, conf = c5_config(args, ws)
    first, S = shard_ranges(args.scenes, ws)[rank]
    data = scenes(S, points=args.points, frames=20, first=first, device=device)
    P = int(data["offsets"][-1])
    sched = {"device_chunks": args.device_chunks} if args.device_chunks else {}
    planner = Planner(cfg, device=device, precision=32, max_scenes=S, max_points=max(P, 1 << 16), profile=True,
                      stream=stream.cuda_stream, **sched)
    dvals = {
        "xyz": torch.from_numpy(data["xyz"]).to(dev), "offsets": torch.from_numpy(data["offsets"]).to(dev),
        "poses": torch.from_numpy(data["poses"]).to(dev), "states": torch.from_numpy(data["states"]).to(dev),
        "goals": torch.from_numpy(data["goals"]).to(dev), "last": torch.from_numpy(data["last"]).to(dev),
        "cycles": torch.from_numpy(data["cycles"].view(np.int64)).to(dev),
        "seeds": torch.from_numpy(data["seeds"].view(np.int64)).to(dev),
    }
    N, M = cfg.mppi.horizon, cfg.grid.count()
    dout = {"status": torch.zeros(S, dtype=torch.int32, device=dev),
            "winner": torch.zeros(S, dtype=torch.int32, device=dev),
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
    sampler = ClockSampler(device)
    sampler.start()
    D.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    D.barrier()
    clocks = sampler.stop()
    planner.synchronize()
    ms_max = D.max(e0.elapsed_time(e1))
    launches = sum(v[1] for v in planner.kernel_times().values())
    total_steps = rollout_steps(cfg, args.scenes) * args.steps
    value = total_steps / (ms_max / 1e3)
    n_ok = int((dout["status"] == 0).sum().item())
    n_ok_all = int(D.sum(float(n_ok)))
    # Per-kernel times for the roofline and the `kernels` table: a short extra
    # pass with the rank's batch as one chunk (in the timed steps chunks run on
    # concurrent streams, where a kernel's events also span other streams' work).
    planner.set_schedule(device_chunks=1)
    step()
    torch.cuda.synchronize(dev)
    planner.kernel_times_reset()
    for _ in range(min(args.steps, 5)):
        step()
    planner.synchronize()
    ktimes = planner.kernel_times()
    planner.set_schedule(device_chunks=args.device_chunks)
    roof = screening_roofline(ktimes, rollout_steps(cfg, S) / cfg.mppi.iterations, fp32_peak(device),
                              sum(v[0] for v in ktimes.values()),
                              executed_flops=EXECUTED_FLOPS_PER_LAUNCH * S / 4096)  # profiled on 4096 scenes

    e2e = None
    if not args.no_e2e:
        # the user-facing call: host-pointer batches from pinned buffers,
        # results copied out, no per-kernel timing events
        planner.close()
        planner = Planner(cfg, device=device, precision=32, max_scenes=S, max_points=max(P, 1 << 16),
                          stream=stream.cuda_stream)
        pinned_xyz = torch.from_numpy(data["xyz"]).pin_memory()  # keep alive while in use
        host = {k: data[k] for k in ("offsets", "poses", "states", "goals", "last", "cycles", "seeds")}
        host["xyz"] = pinned_xyz.numpy()
        def submit(c):
            return planner.cycle_batch_submit(host["offsets"], host["xyz"], host["poses"], host["states"],
                                              host["goals"], host["last"], host["cycles"] + c, host["seeds"])

        for i in range(max(1, args.warmup)):
            planner.cycle_batch_wait(submit(i))
        D.barrier()
        torch.cuda.synchronize(dev)
        # streaming: steps i+1 and i+2 are submitted before step i's results are
        # read, so step i+1's upload starts as soon as the copy engine is free
        # and runs under step i's planning; every step still uploads its inputs
        # and reads its results back inside the timed region
        t0 = time.perf_counter()
        pending = [submit(1000 + i) for i in range(min(2, args.steps))]
        for i in range(args.steps):
            if i + 2 < args.steps:
                pending.append(submit(1000 + i + 2))
            planner.cycle_batch_wait(pending.pop(0))
        el = D.max(time.perf_counter() - t0)
        h2d = sum(data[k].nbytes for k in ("xyz", "offsets", "poses", "states", "goals", "last", "cycles", "seeds"))
        d2h = S * (4 + 4 + 8 * 4 + 8 * N * 4 + 8 * M + 8 * 5)
        e2e = {"value": total_steps / el, "unit": "rollout-steps/s",
               "h2d_bytes_per_step": int(D.sum(float(h2d))), "d2h_bytes_per_step": int(D.sum(float(d2h))),
               "ms_per_step": 1000 * el / args.steps,
               "api": "amppi_cycle_batch_submit / _wait (host pointers, pinned xyz; up to three batches in flight)"}
    planner.close()

    latency = cpu = None
    if rank == 0:
        orc = oracle()
        if not args.no_latency:
            latency = latency_block(args, orc, device)
        done, secs = cpu_plan_scenes(orc, cfg, data, range(S), args.cpu_seconds)
        cores = os.cpu_count() or 1
        cpu = {"value": rollout_steps(cfg, done) / secs, "unit": "rollout-steps/s", "cores": cores, "kind": "port",
               "sample": f"{done} scenes of this workload (scene ids {first}..{first + done - 1}: build_snapshot + "
                         f"plan_step each), {secs:.1f} s, oracle/ restatement, parallel_for over {cores} threads "
                         f"({cpu_model()})"}
        line = {
            "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 stage-I screening / f64 keys, anchors, softmin support, update, stage II",
            "data": "synthetic (reference scenario families; GPU LiDAR, bytes equal to its host twin)", "config": conf,
            "workload_stats": {"scenes_rank0": S, "points_rank0": P, "planned_ok": n_ok_all,
                               "dist_backend": D.backend, "ranks_share_a_gpu": D.shared_gpu},
            "latency": latency, "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": int(launches), "kernels": kernel_summary(ktimes),
        }
        print(json.dumps(line), flush=True)


def latency_block(args, orc, device):
    """p50 / p99 of host-to-host amppi_snapshot_f64 + amppi_plan (C ABI,
    caller-owned result buffers, warm nominal) over the 50 inputs of the
    reference's latency protocol, replayed to args.latency_cycles samples
    after 100 warm-up cycles; the oracle's build_snapshot + plan_step p50 on
    the same 50 inputs beside it (acceptance.cpp:351-372)."""
    import numpy as np

    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State, _abi
    from paper_2509_17340_b200.workloads import plan_config, rollout_steps

    cfg = plan_config()
    recs, (gp, gv, gq) = latency_inputs(orc, cfg)
    lp = Planner(cfg, device=device, precision=32, max_scenes=1, max_points=1 << 17)
    M, N = cfg.grid.count(), cfg.mppi.horizon
    res = _abi.PlanResult()
    nominal = np.zeros((M, N, 4))
    res.nominal = nominal.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    goal = _abi.Goal()
    goal.p_goal[:], goal.v_goal[:], goal.q_goal[:] = list(gp), list(gv), list(gq)
    ins = []
    for r in recs:
        st = _abi.State()
        st.p[:], st.q[:], st.v[:] = list(r["x"][0:3]), list(r["x"][3:7]), list(r["x"][7:10])
        la = _abi.Control()
        la.thrust, la.omega[:] = r["last_applied"][0], list(r["last_applied"][1:4])
        cloud = np.ascontiguousarray(r["cloud"], dtype=np.float64)
        prev = np.ascontiguousarray(r["prev"], dtype=np.float64)
        ins.append((st, la, cloud, prev, r["prev_len"], r["cycle"]))
    lib = lp.lib

    def c_abi_cycle(k):
        st, la, cloud, prev, plen, cyc = ins[k % len(ins)]
        rc = lib.amppi_snapshot_f64(lp._h, cloud.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(cloud),
                                    ctypes.byref(st), ctypes.c_double(cfg.r_max))
        rc |= lib.amppi_plan(lp._h, ctypes.byref(st), ctypes.byref(goal),
                             prev.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if plen else None, plen,
                             ctypes.byref(la), ctypes.c_uint64(cyc), ctypes.c_uint64(1), None, ctypes.byref(res))
        return rc

    lat, winners = [], [None] * len(ins)
    for i in range(100 + args.latency_cycles):
        t0 = time.perf_counter()
        rc = c_abi_cycle(i)
        t1 = time.perf_counter()
        if rc != 0:
            raise RuntimeError(f"C1 cycle failed ({rc})")
        if i >= 100:
            lat.append(1000 * (t1 - t0))
        winners[i % len(ins)] = int(res.winner)
    lp.close()
    lat.sort()
    # the oracle on the same inputs: acceptance.cpp's median of 50 cycles
    ocfg = orc.config(cfg)
    lat_cpu, same = [], 0
    for k, r in enumerate(recs):
        t0 = time.perf_counter()
        snap = orc.snapshot(r["cloud"], r["x"], cfg.r_max)
        o = orc.plan(snap, ocfg, r["x"], gp, gv, gq, r["prev"] if r["prev_len"] else None, r["last_applied"],
                     r["cycle"], 1)
        lat_cpu.append(1000 * (time.perf_counter() - t0))
        same += int(o["winner"] == winners[k])
    lat_cpu.sort()
    # the paper's default ensemble (5x3 anchors x 256 x 25; 2.0 ms per cycle on an RTX 4080 SUPER)
    pcfg = plan_config(5, 3, K=256, N=25)
    pp = Planner(pcfg, device=device, precision=32, max_scenes=1, max_points=1 << 17)
    pgoal = GoalSpec(tuple(gp), tuple(gv), tuple(gq))
    lat_p, prevp = [], None
    for i in range(100 + args.latency_cycles // 2):
        r = recs[i % len(recs)]
        x = State.from_array(r["x"])
        t0 = time.perf_counter()
        snap = pp.build_snapshot(r["cloud"], x, pcfg.r_max, f64=True)
        res_p = pp.plan_step(x, pgoal, snap, prevp, ControlInput(r["last_applied"][0], tuple(r["last_applied"][1:])),
                             r["cycle"], 1, want_rollout=False)
        t1 = time.perf_counter()
        prevp = res_p.per_instance[res_p.winner].nominal
        if i >= 100:
            lat_p.append(1000 * (t1 - t0))
    pp.close()
    lat_p.sort()
    pts = [len(r["cloud"]) for r in recs]
    return {"workload": "C1 latency protocol of acceptance.cpp:339-377: forest seed 1 flown 100 cycles into the "
                        "clutter by the oracle's execute_cycle loop (buffer 20 frames), then the recorded inputs of "
                        "the next 50 plan cycles; host-to-host amppi_snapshot_f64 + amppi_plan through the C ABI, "
                        "4x2 anchors x 256 x 30, warm nominal",
            "points_per_cycle": [min(pts), max(pts)],
            "p50_ms": lat[len(lat) // 2], "p99_ms": lat[int(0.99 * len(lat))], "cycles": len(lat),
            "cpu_p50_ms": lat_cpu[len(lat_cpu) // 2], "cpu_cycles": len(lat_cpu),
            "cpu": f"oracle build_snapshot + plan_step, parallel_for over {os.cpu_count()} threads ({cpu_model()})",
            "winners_equal_to_oracle": f"{same}/{len(recs)}",
            "rollout_steps_per_s_at_p50": rollout_steps(cfg, 1) / (lat[len(lat) // 2] / 1e3),
            "paper_default": {"config": "5x3 anchors x 256 samples x 25 steps, same inputs, Python API (the paper: "
                                        "500 Hz = 2.0 ms per cycle on an RTX 4080 SUPER)",
                              "p50_ms": lat_p[len(lat_p) // 2], "p99_ms": lat_p[int(0.99 * len(lat_p))]}}


def run_c4(args, D: Dist):
    import numpy as np
    import torch

    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State
    from paper_2509_17340_b200.sharding import NcclComm, TorchComm, plan_step_sharded, plan_step_sharded_native
    from paper_2509_17340_b200.workloads import rollout_steps

    ws, rank, device = D.world, D.rank, D.device
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    cfg, conf = c4_config(ws)
    one = c4_scene(False, device)
    planner = Planner(cfg, device=device, precision=32, max_points=1 << 16, profile=True, stream=stream.cuda_stream)
    x = State.from_array(one["states"][0])
    goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
    la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
    pts = np.ascontiguousarray(one["xyz"])
    # the library's own NCCL path when every rank owns a GPU; torch
    # collectives over gloo when ranks share one (functional run)
    comm, native = None, False
    if not D.shared_gpu:
        try:
            uid = D.broadcast(NcclComm.unique_id() if rank == 0 else None)
            comm, native = NcclComm(uid, rank, ws, device), True
        except RuntimeError:
            comm = None
    if comm is None and ws > 1:
        comm = TorchComm()
    prev = None

    def step(i):
        nonlocal prev
        snap = planner.build_snapshot(pts, x, cfg.r_max)
        if native:
            r = plan_step_sharded_native(planner, comm, x, goal, snap, prev, la, 100 + i, 1, want_rollout=False)
        elif comm is not None:
            r = plan_step_sharded(planner, x, goal, snap, prev, la, 100 + i, 1, comm, want_rollout=False)
        else:
            r = planner.plan_step(x, goal, snap, prev, la, 100 + i, 1, want_rollout=False)
        prev = r.per_instance[r.winner].nominal
        return r

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    planner.kernel_times_reset()
    sampler = ClockSampler(device)
    sampler.start()
    D.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    wall = D.max(time.perf_counter() - t0)
    clocks = sampler.stop()
    ms = D.max(e0.elapsed_time(e1))
    kt = planner.kernel_times()
    value = rollout_steps(cfg, 1) * args.steps / (ms / 1e3)
    k_rank = cfg.mppi.rollouts // ws  # samples per instance on this rank
    roof = screening_roofline(kt, cfg.grid.count() * k_rank * cfg.mppi.horizon, fp32_peak(device),
                              sum(v[0] for v in kt.values()))
    roof["traffic"] = None
    roof["traffic_source"] = "not captured for C4 (profiles/ holds the C5 capture)"
    planner.close()
    if native:
        comm.close()
    if rank == 0:
        orc = oracle()
        ocfg = orc.config(cfg)
        t0c = time.perf_counter()
        osnap = orc.snapshot(pts.astype(np.float64), one["poses"][0], cfg.r_max)
        orc.plan(osnap, ocfg, one["states"][0], goal.p_goal, goal.v_goal, goal.q_goal, None, one["last"][0], 100, 1)
        secs = time.perf_counter() - t0c
        cpu = {"value": rollout_steps(cfg, 1) / secs, "unit": "rollout-steps/s", "cores": os.cpu_count(),
               "kind": "port", "sample": f"one C4 plan cycle (build_snapshot + plan_step, 26.2 M rollout-steps) on "
                                         f"the same scene bytes, {secs:.1f} s, oracle/ restatement over "
                                         f"{os.cpu_count()} threads ({cpu_model()})"}
        h2d = pts.nbytes + 4 * 8 * 10 + 50 * 4 * 8
        d2h = 64 * (8 * 3 + 1 + 50 * 4 * 8 + 8 * 13 + 4 * 2 + 18 * 8)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 screening / f64 support, update, stage II", "data": "synthetic",
            "config": conf,
            "e2e": {"value": rollout_steps(cfg, 1) * args.steps / wall, "unit": "rollout-steps/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": 1000 * wall / args.steps,
                    "api": "build_snapshot + plan_step (sharded) host-to-host, wall clock max over ranks"},
            "collectives": "amppi_plan_sharded (library NCCL)" if native else (
                "torch.distributed (gloo, ranks share a GPU)" if comm is not None else "none (1 rank)"),
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": int(sum(v[1] for v in kt.values())), "kernels": kernel_summary(kt),
        }), flush=True)


def run_c3(args, D: Dist):
    import numpy as np
    import torch

    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State, _abi
    from paper_2509_17340_b200.workloads import rollout_steps

    device = D.device
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    cfg, conf = c3_config()
    one = c3_scene(False, device)
    pts = np.ascontiguousarray(one["xyz"])
    P = pts.shape[0]
    x = State.from_array(one["states"][0])
    goal = GoalSpec((45.0, 0.0, 2.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
    la = ControlInput(one["last"][0][0], (0.0, 0.0, 0.0))
    d_pts = torch.from_numpy(pts).to(dev)
    planner = Planner(cfg, device=device, precision=32, max_points=P + 1024, profile=True, stream=stream.cuda_stream)
    lib = planner.lib
    xs, gs, lc = x.to_c(), goal.to_c(), la.to_c()
    res = _abi.PlanResult()

    def device_cycle(i):
        # device-resident points: the snapshot reads them straight from HBM
        rc = lib.amppi_snapshot_device(planner._h, ctypes.cast(ctypes.c_void_p(d_pts.data_ptr()), _abi.c_float_p), P,
                                       ctypes.byref(xs), ctypes.c_double(cfg.r_max))
        rc |= lib.amppi_plan(planner._h, ctypes.byref(xs), ctypes.byref(gs), None, 0, ctypes.byref(lc),
                             ctypes.c_uint64(100 + i), ctypes.c_uint64(1), None, ctypes.byref(res))
        if rc:
            raise RuntimeError(f"C3 cycle failed ({rc})")

    for i in range(args.warmup):
        device_cycle(i)
    torch.cuda.synchronize(dev)
    planner.kernel_times_reset()
    sampler = ClockSampler(device)
    sampler.start()
    D.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        device_cycle(args.warmup + i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    ms = D.max(e0.elapsed_time(e1))
    kt = planner.kernel_times()
    # e2e: host points (pinned, as a LiDAR driver's DMA buffer would be) through
    # build_snapshot (amppi_snapshot) + plan_step
    pinned = torch.from_numpy(pts).pin_memory()
    hpts = pinned.numpy()
    t0 = time.perf_counter()
    for i in range(args.steps):
        snap = planner.build_snapshot(hpts, x, cfg.r_max)
        planner.plan_step(x, goal, snap, None, la, 200 + i, 1, want_rollout=False)
    wall = D.max(time.perf_counter() - t0)
    planner.close()
    ws = D.world
    value = rollout_steps(cfg, 1) * ws * args.steps / (ms / 1e3)
    key_ms, key_n = kt.get("k_key_points", (float("nan"), 1))
    snap_ms = sum(kt.get(k, (0.0, 0))[0] for k in ("k_key_points", "k_resolve_ties", "k_finalize_scene")) / key_n
    achieved = BYTES_PER_POINT * P / (key_ms / key_n / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    if D.rank == 0:
        orc = oracle()
        ocfg = orc.config(cfg)
        t0c = time.perf_counter()
        osnap = orc.snapshot(pts.astype(np.float64), one["poses"][0], cfg.r_max)
        t_snap = time.perf_counter() - t0c
        orc.plan(osnap, ocfg, one["states"][0], goal.p_goal, goal.v_goal, goal.q_goal, None, one["last"][0], 100, 1)
        secs = time.perf_counter() - t0c
        cpu = {"value": rollout_steps(cfg, 1) / secs, "unit": "rollout-steps/s", "cores": os.cpu_count(),
               "kind": "port", "build_snapshot_ms": 1000 * t_snap,
               "sample": f"one C3 plan cycle on the same 1M points: build_snapshot {1000 * t_snap:.0f} ms (serial, "
                         f"as the reference) + plan_step, {secs:.2f} s, oracle/ restatement ({cpu_model()})"}
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "replicas",
            "vs_baseline": None, "dtype": "f32 screening / f64 keys, plan", "data": "synthetic", "config": conf,
            "snapshot_ms": snap_ms,
            "e2e": {"value": rollout_steps(cfg, 1) * ws * args.steps / wall, "unit": "rollout-steps/s",
                    "h2d_bytes_per_step": int(pts.nbytes), "d2h_bytes_per_step": 64 * 8 * 200,
                    "ms_per_step": 1000 * wall / args.steps,
                    "api": "Planner.build_snapshot (pinned host points) + plan_step, host to host"},
            "roofline": {"bound": "hbm", "kernel": "k_key_points (keying: every point read once)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "algorithmic_bytes_per_launch": BYTES_PER_POINT * P,
                         "kernel_ms_per_launch": key_ms / key_n, "peak_source": peak_src},
            "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": int(sum(v[1] for v in kt.values())), "kernels": kernel_summary(kt),
        }), flush=True)


def run_c2(args, D: Dist):
    from paper_2509_17340_b200 import ClosedLoop, Planner
    from paper_2509_17340_b200.planner import apply_velocity_cap
    from paper_2509_17340_b200.workloads import plan_config, rollout_steps

    if D.rank != 0:
        return
    device = D.device
    cfg = apply_velocity_cap(plan_config(), 7.0)
    cycles = 200
    planner = Planner(cfg, device=device, precision=32, max_points=10 * 7200)

    def episode(i):
        lp = ClosedLoop(planner, 1, 1, 31 + i, buffer_capacity=10, max_cycles=cycles)
        t0 = time.perf_counter()
        ran = lp.run(cycles)
        dt = time.perf_counter() - t0
        lp.close()
        return ran, dt

    for i in range(args.warmup):
        episode(i)
    sampler = ClockSampler(device)
    sampler.start()
    total_cycles, total_t = 0, 0.0
    for i in range(args.steps):
        ran, dt = episode(args.warmup + i)
        total_cycles += ran
        total_t += dt
    clocks = sampler.stop()
    planner.close()
    orc = oracle()
    lo = orc.loop(1, 1, orc.config(cfg), 31, capacity=10)
    t0 = time.perf_counter()
    n_cpu = lo.run(50)
    t_cpu = time.perf_counter() - t0
    value = rollout_steps(cfg, 1) * total_cycles / total_t
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "rollout-steps/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
        "scaling": "replicas", "vs_baseline": None, "dtype": "f32 screening / f64 plan, LiDAR and vehicle",
        "data": "synthetic",
        "config": {"workload": "C2: 200-cycle closed-loop forest flight (seed 1), speed cap 7 m/s, 4x2 anchors x 256 "
                               "x 30, LiDAR + point-cloud ring + snapshot + plan + vehicle step on the device "
                               "(amppi_loop_run, one CUDA graph per cycle); one step = one episode",
                   "cycles_per_episode": cycles, "ms_per_cycle": 1e3 * total_t / max(total_cycles, 1)},
        "e2e": {"value": value, "unit": "rollout-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8,
                "note": "the loop is device-resident: per episode the host reads back only the cycle counter"},
        "cpu_baseline": {"value": rollout_steps(cfg, 1) * n_cpu / t_cpu, "unit": "rollout-steps/s",
                         "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{n_cpu} cycles of the oracle's execute_cycle loop ({1e3 * t_cpu / n_cpu:.2f} "
                                   f"ms/cycle)"},
        "clocks": clocks,
    }), flush=True)


# ---------------------------------------------------------------------------
# reference arm: the oracle on the host cores, same config and input bytes
# ---------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path (the
    oracle restatement; the reference itself cannot be built here, DESIGN.md
    §8) with all host threads, on the b200 arm's config, metric and input
    bytes (scenes regenerated by the host twin of the input generator,
    amppi_sim_scan_host); each step is a bounded sample of the workload."""
    ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from paper_2509_17340_b200.workloads import rollout_steps, scenes

    orc = oracle()
    cores = os.cpu_count() or 1
    if args.workload == "c5":
        cfg, conf = c5_config(args, ws)
        n_sample = 4
        data = scenes(n_sample * (args.steps + args.warmup), points=args.points, frames=20, first=0, host=True)
        units = rollout_steps(cfg, n_sample)
        sample = (f"{n_sample} scenes per step (scene ids 0.. of the same batch; bytes identical to the b200 arm's: "
                  f"host twin of the GPU LiDAR), build_snapshot + plan_step each")

        def step(i):
            cpu_plan_scenes(orc, cfg, data, range(i * n_sample, (i + 1) * n_sample), 1e9)
    elif args.workload in ("c4", "c3"):
        cfg, conf = c4_config(ws) if args.workload == "c4" else c3_config()
        one = c4_scene(True) if args.workload == "c4" else c3_scene(True)
        ocfg = orc.config(cfg)
        pts = one["xyz"].astype(np.float64)
        units = rollout_steps(cfg, 1)
        sample = ("one C4 plan cycle per step (26.2 M rollout-steps)" if args.workload == "c4" else
                  "one C3 plan cycle per step (build_snapshot of the 1M points, serial, + plan_step)") + \
            ", same scene bytes as the b200 arm"

        def step(i):
            snap = orc.snapshot(pts, one["poses"][0], cfg.r_max)
            orc.plan(snap, ocfg, one["states"][0], [45.0, 0, 2.0], [0, 0, 0], [1.0, 0, 0, 0], None, one["last"][0],
                     100 + i, 1)
    else:
        from paper_2509_17340_b200.planner import apply_velocity_cap
        from paper_2509_17340_b200.workloads import plan_config

        cfg = apply_velocity_cap(plan_config(), 7.0)
        conf = {"workload": "C2: 200-cycle closed-loop forest flight (seed 1), speed cap 7 m/s, 4x2 anchors x 256 "
                            "x 30 (the oracle's execute_cycle loop)"}
        units = rollout_steps(cfg, 20)
        sample = "20 cycles of the oracle's execute_cycle loop per step"
        lo = orc.loop(1, 1, orc.config(cfg), 31, capacity=10)

        def step(i):
            lo.run(20)
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = units * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": "rollout-steps/s", "impl": "reference", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.workload in ("c5", "c4") else "replicas",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": conf,
            "cpu_baseline": {"value": value, "unit": "rollout-steps/s", "cores": cores, "kind": "port",
                             "sample": sample + f"; oracle/ restatement, parallel_for over {cores} threads "
                                                f"({cpu_model()}); the reference itself is not buildable here "
                                                f"(Eigen / vendor/ absent)"},
            "e2e": {"value": value, "unit": "rollout-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rc = relaunch(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
        return
    D = Dist()
    try:
        {"c5": run_c5, "c4": run_c4, "c3": run_c3, "c2": run_c2}[args.workload](args, D)
    finally:
        D.close()


if __name__ == "__main__":
    main()
