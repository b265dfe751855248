"""Benchmark: SF-projected feasible swarm samples/s (16 drones, H=100) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One "step" = one pass of the hot path over one batch: the persistent SF kernel
solves every sample of the batch to tol 1e-3 (or max_iters), then the fused
feasibility verdict (and, for N > 1, the NCCL gather of the projected
trajectories, iterations and verdicts).  Workload = BASELINE config 2: seeded
16-robot H=100 scenario (paper_2501_19042_b200.scenarios, seed 2), 1000
proposals per GPU from the reference's Gaussian sampler (seed 0), boundary-
projected start, degree 10, rho 1, max_iters 500 (this scenario needs
~290-380 iterations; none converge within 200).  Weak scaling: each rank
solves its own contiguous 1000-sample shard of one global seeded batch.

`value` is device-timed (CUDA events, inputs resident in HBM, L2 flushed
between steps, max over ranks); `e2e` is the same metric through the public
API with pinned host buffers, H2D and D2H inside the timed region.
`--impl reference` times the CPU oracle port of the reference algorithm
(oracle/sf_oracle.py: trig projection + dense LU, the reference's own
arithmetic) on the host cores with a process pool, on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SF-projected feasible swarm samples/sec (16 drones, H=100); ms per 1k batch"
BATCH_PER_GPU = 1000
MAX_ITERS = 500


def flop_per_si(n: int, S: int, m1: int) -> int:
    """Algorithmic FLOPs per sample-iteration."""
    P = n * (n - 1) // 2
    return 33 * P * S + 30 * n * S + 12 * n * S * m1 + 12 * n * m1 * m1 + 42 * n * m1


def workload(rank: int, world: int, batch: int):
    from paper_2501_19042_b200 import SolverConfig, sample_proposals
    from paper_2501_19042_b200.basis import build_basis
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(2)
    basis = build_basis(prob.duration, degree=10, samples=prob.horizon_samples)
    props = sample_proposals(prob, basis, batch * world, seed=0).proposals
    shard = props[rank * batch:(rank + 1) * batch]
    return prob, shard, SolverConfig(max_iters=MAX_ITERS, svars=False)


# ----------------------------------------------------------------------------- CPU legs
def _oracle_worker(args):
    from threadpoolctl import threadpool_limits
    doc, xb, max_iters = args
    with threadpool_limits(limits=1):
        from oracle import sf_oracle
        prob = sf_oracle.make_problem(doc, degree=10)
        t0 = time.perf_counter()
        r = sf_oracle.solve(prob, xb, max_iters=max_iters)
        dt = time.perf_counter() - t0
        return r.iterations, sf_oracle.feasible(prob, r), dt


def cpu_sample(doc, props, budget_s: float, max_samples: int | None = None):
    """Run the oracle port over as many proposals as fit ~budget_s on all host cores."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    done, feas, its, t_start = 0, 0, 0, time.perf_counter()
    with ctx.Pool(cores) as pool:
        while True:
            chunk = props[done:done + cores]
            if max_samples is not None:
                chunk = chunk[:max(0, max_samples - done)]
            if len(chunk) == 0:
                break
            for it, fe, _ in pool.map(_oracle_worker, [(doc, x, MAX_ITERS) for x in chunk]):
                its += it
                feas += int(fe)
            done += len(chunk)
            if time.perf_counter() - t_start >= budget_s:
                break
    wall = time.perf_counter() - t_start
    return {"samples": done, "feasible": feas, "sample_iterations": its, "wall_s": wall, "cores": cores}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """`nvidia-smi -lms 100` into a CSV.  Started before the warm-up (its start-up queries the driver and
    must not overlap the timed steps); `mark()` brackets the timed region and the summary uses those rows."""

    def __init__(self, path: Path):
        self.path = path
        self.proc = None
        self.marks = []

    def lines(self) -> int:
        try:
            with open(self.path) as fh:
                return sum(1 for _ in fh)
        except OSError:
            return 0

    def wait_first(self, timeout_s: float = 5.0) -> None:
        t0 = time.perf_counter()
        while self.proc is not None and self.lines() == 0 and time.perf_counter() - t0 < timeout_s:
            time.sleep(0.05)

    def mark(self) -> None:
        self.marks.append(self.lines())

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self, device_index: int) -> dict:
        rows = []
        try:
            lines = open(self.path).read().splitlines()
        except OSError:
            lines = []
        if len(self.marks) == 2 and self.marks[1] > self.marks[0]:
            lines = lines[self.marks[0]:self.marks[1] + 1]   # the timed region (+ the sample just after it)
        for line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9 and f[0] == str(device_index):
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    prob, shard, cfg = workload(0, 1, BATCH_PER_GPU)
    doc = prob.to_doc()
    steps = []
    total_feas = total_samples = 0
    # per-step CPU budget: --ref-budget, or ~150 s over the timed steps (1.5-12 s each: at least one
    # round of proposals per core), so the whole --steps K --warmup W run stays within a few minutes
    budget = args.ref_budget if args.ref_budget is not None else min(12.0, max(1.5, 150.0 / max(1, args.steps)))
    for _ in range(args.warmup):
        cpu_sample(doc, shard, budget_s=0.0, max_samples=os.cpu_count() or 1)
    for k in range(args.steps):
        off = (k * (os.cpu_count() or 1)) % len(shard)
        r = cpu_sample(doc, list(shard[off:]) + list(shard[:off]), budget_s=budget)
        steps.append(r)
        total_feas += r["feasible"]
        total_samples += r["samples"]
    wall = sum(s["wall_s"] for s in steps)
    value = total_feas / wall if wall > 0 else 0.0
    cores = steps[0]["cores"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "feasible samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scenario + reference Gaussian sampler)",
        "config": {"workload": "BASELINE config 2: 16 drones, H=100, SF to 1e-3 (max_iters 500); "
                               "each step a bounded sample of the 1000-proposal batch",
                   "n": 16, "H": 100, "batch": BATCH_PER_GPU, "max_iters": MAX_ITERS},
        "ms_per_1k_batch": 1e3 * 1000 / value if value > 0 else None,
        "cpu_baseline": {"value": value, "unit": "feasible samples/s", "cores": cores, "kind": "port",
                         "sample": f"{total_samples} proposals over {args.steps} steps, all iterations, "
                                   f"process pool on {cores} cores ({cpu_model()}), BLAS 1 thread/process"},
        "e2e": {"value": value, "unit": "feasible samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2501_19042_b200 import SafetyFilter, native
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    prob, shard, cfg = workload(rank, world, args.batch)
    if args.precision != "lean":
        from paper_2501_19042_b200 import SolverConfig
        cfg = SolverConfig(max_iters=MAX_ITERS, svars=False, precision=args.precision)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    n, S, m1 = prob.n, prob.horizon_samples, 11
    xb_host = torch.from_numpy(shard).pin_memory()
    xb = xb_host.to(dev)
    dim = xb.shape[1]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    peak_tflops = ctypes_peak(native)

    def gather(out):
        if world == 1:
            return
        for t in (out.coeffs, out.iterations, out.feasible, out.residual_inf):
            buf = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
            dist.all_gather_into_tensor(buf, t.contiguous())

    def step(timing=None):
        out = sf.solve_batched(xb, config=cfg, timing=timing)
        gather(out)
        return out

    clocks = ClockSampler(ROOT / "gpurun_out" / f"clocks_rank{rank}.csv") if rank == 0 else None
    if clocks:
        (ROOT / "gpurun_out").mkdir(exist_ok=True)
        clocks.__enter__()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if clocks:
        clocks.wait_first()

    # ---- device-timed region: inputs resident in HBM
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    feas_counts, its_total = [], []
    launches0 = native.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.mark()
    outs = []
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record()
        out = step(timing=kev[k])
        ev[k][1].record()
        outs.append((out.feasible, out.iterations))   # the rest is freed: the next step reuses its blocks
        del out
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if clocks:
        time.sleep(0.15)   # one more sample after the last step
        clocks.mark()
        clocks.__exit__()
    launches = native.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    for feas, its in outs:
        feas_counts.append(int(feas.sum().item()))
        its_total.append(int(its.sum().item()))
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms, float(sum(feas_counts))], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        total_ms_max, feas_all = float(tmax[0]), float(t[1])
    else:
        total_ms_max, feas_all = total_ms, float(t[1])
    value = feas_all / (total_ms_max * 1e-3)

    # ---- end-to-end through the public API: pinned host in, host out
    h_coeffs = torch.empty((xb.shape[0], dim), dtype=torch.float64).pin_memory()
    h_its = torch.empty(xb.shape[0], dtype=torch.int32).pin_memory()
    h_feas = torch.empty(xb.shape[0], dtype=torch.uint8).pin_memory()
    e2e_ms = []
    for k in range(args.steps + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        xd = xb_host.to(dev, non_blocking=True)
        out = sf.solve_batched(xd, config=cfg)
        gather(out)
        h_coeffs.copy_(out.coeffs, non_blocking=True)
        h_its.copy_(out.iterations, non_blocking=True)
        h_feas.copy_(out.feasible, non_blocking=True)
        b.record()
        b.synchronize()
        if k:   # first one is a warm-up
            e2e_ms.append(a.elapsed_time(b))
    e2e_feas = int(h_feas.numpy().sum())
    te = torch.tensor([sum(e2e_ms), float(e2e_feas * len(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        temax = te.clone()
        dist.all_reduce(temax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(te[1:], op=dist.ReduceOp.SUM)
        e2e_value = float(te[1]) / (float(temax[0]) * 1e-3)
    else:
        e2e_value = float(te[1]) / (float(te[0]) * 1e-3)
    h2d = xb_host.numel() * 8
    d2h = h_coeffs.numel() * 8 + h_its.numel() * 4 + h_feas.numel()

    if rank != 0:
        return
    # ---- roofline of the dominant kernel (persistent SF kernel)
    fps = flop_per_si(n, S, m1)
    flops_per_launch = statistics.mean(its_total) * fps
    kern_avg_ms = statistics.mean(kern_ms)
    achieved = flops_per_launch / (kern_avg_ms * 1e-3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "feasible samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": total_ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"lean": "f32 terms + f64 state", "hybrid": "f32 screening + f64 values", "strict": "f64"}[args.precision],
        "data": "synthetic (seeded 16-robot scenario, reference Gaussian sampler proposals)",
        "config": {"workload": "BASELINE config 2: 16 drones, H=100, batch 1000 per GPU, SF to 1e-3 "
                               "(max_iters 500), boundary-projected start",
                   "n": n, "H": S - 1, "degree": 10, "batch_per_gpu": int(xb.shape[0]), "max_iters": MAX_ITERS,
                   "rho": 1.0, "precision": args.precision, "l2_flush": "256 MB write between steps",
                   "parallelism": f"dp{world} (contiguous sample shards, NCCL all_gather of outputs)"},
        "ms_per_1k_batch": (total_ms_max / args.steps) * 1000.0 / xb.shape[0],
        "feasible_fraction": feas_all / (args.steps * xb.shape[0] * world),
        "mean_iterations": statistics.mean(its_total) / xb.shape[0],
        "gpu_launches": int(round(launches / args.steps)),
        "e2e": {"value": e2e_value, "unit": "feasible samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": {"bound": "fp32_cuda_core", "achieved": achieved, "peak": peak_tflops,
                     "unit": "TFLOP/s", "frac": achieved / peak_tflops if peak_tflops else None,
                     "traffic": traffic, "kernel": "sf_persistent_kernel<float,16>",
                     "kernel_ms": kern_avg_ms, "flop_per_si": fps,
                     "peak_source": "FFMA microbenchmark (sgsf_fp32_peak) run live in this process; "
                                    "MEASURED_PEAKS.json has no FP32 figure"},
        "clocks": clocks.summary(local_rank) if clocks else None,
    }
    if args.cpu_baseline and world == 1:
        cb = cpu_sample(prob.to_doc(), shard, budget_s=args.ref_budget if args.ref_budget is not None else 12.0)
        v = cb["feasible"] / cb["wall_s"]
        line["cpu_baseline"] = {"value": v, "unit": "feasible samples/s", "cores": cb["cores"], "kind": "port",
                                "sample": f"{cb['samples']} proposals of this batch, all iterations "
                                          f"({cb['sample_iterations']} sample-iterations) in {cb['wall_s']:.1f} s, "
                                          f"oracle/sf_oracle.py process pool on {cb['cores']} cores "
                                          f"({cpu_model()})"}
    print(json.dumps(line), flush=True)


def ctypes_peak(native) -> float:
    import ctypes
    tf, ms = ctypes.c_double(), ctypes.c_double()
    import torch
    native.check(native.load().sgsf_fp32_peak(ctypes.byref(tf), ctypes.byref(ms),
                                              torch.cuda.current_stream().cuda_stream), "sgsf_fp32_peak")
    return float(tf.value)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH_PER_GPU)
    ap.add_argument("--precision", default="lean", choices=["lean", "strict", "hybrid"])
    ap.add_argument("--ref-budget", type=float, default=None,
                    help="seconds of CPU work per reference step (default: 12 s for the cpu_baseline leg; "
                         "150 s / steps, within 1.5-12 s, for --impl reference)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
