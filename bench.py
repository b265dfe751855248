"""Benchmark: SF-projected feasible swarm samples/s (16 drones, H=100) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 2|3|4]
                    [--precision hybrid|lean|strict]

One "step" = one pass of the hot path over one batch: the persistent SF kernel solves every sample of the
batch to tol 1e-3 (or max_iters), the feasible verdict runs behind it, and for N > 1 the per-sample outputs
(coefficients, multipliers, residual histories, iterations, verdicts, displacement, status) are all-gathered
over NCCL.  The headline is BASELINE config 2 (`--config 2`, default): a seeded 16-robot H=100 scenario,
1000 proposals per GPU from the reference's Gaussian sampler (seed 0), boundary-projected start, degree 10,
rho 1, max_iters 500 -- weak scaling over N GPUs.  `--config 3` (32 robots, H=100, 4096 samples) and
`--config 4` (64 robots, H=150, 8192 samples) strong-scale one batch over the N GPUs, as BASELINE states them.

Precision (default "hybrid"): FP32 screening with guard bands, FP64 targets/residuals/state and an FP64
re-evaluation of the stop decision near tol -- the precision whose iteration counts and verdicts equal the
reference's on all 1000 headline samples (tests/test_gpu_batch_parity.py).  At N = 1 the line also carries
device-timed numbers of "lean" (FP32 terms) and "strict" (FP64 everywhere) from the same run.

`value` is device-timed (CUDA events, inputs resident in HBM, max over ranks) over K batches submitted with
two in flight (`SafetyFilter.solve_pipelined`: the next batch starts on the SMs the previous batch's tail
frees); `pipelining.batch_latency_ms` times the same K batches one after another, and the roofline takes the
kernel's per-launch time from that run.  The steps' inputs rotate over device copies of the batch totalling
>= 256 MB (inputs larger than L2: no step finds its proposals cached).  `e2e` is the same metric through the
public API with pinned host buffers, the H2D copy of the proposals and the D2H copy of every per-sample output
of each batch on its own stream inside the timed region.  At N = 1 two more end-to-end
numbers: `e2e_dropin` (the reference-compatible `SafetyFilter.batch_solve` on a list of numpy proposals at its
defaults, plus `feasible_results`) and `pipeline` (config 2 as BASELINE states it: CVAE samples -> boundary QP
-> init-network warm start -> SF -> verdict, all on the device).

`--impl reference` (and the `cpu_baseline` leg) time the reference's own CPU solver on the host cores: the
compiled reference built into oracle/_ref by oracle/build_ref.sh (`kind: "reference"`), or, where that is
missing, the numpy port oracle/sf_oracle.py (`kind: "port"`).  One persistent process pool (BLAS pinned to 1
thread per process) streams the batch's proposals; each timed step counts the samples the pool completes in
its time slice, so the rate is the pool's steady-state throughput.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SF-projected feasible swarm samples/sec (16 drones, H=100); ms per 1k batch"
MAX_ITERS = 500
# per BASELINE config: (robots, horizon, batch, scaling, max_iters); config 2's batch is per GPU (weak scaling).
# Config 4 states "SF to 1e-3 residual" with no cap; its 64-robot swarm needs ~1000 iterations
CONFIGS = {2: (16, 100, 1000, "weak", 500), 3: (32, 100, 4096, "strong", 500), 4: (64, 150, 8192, "strong", 1000)}
REF_DIR = ROOT / "oracle" / "_ref"


def flop_per_si(n: int, S: int, m1: int) -> int:
    """Algorithmic FLOPs per sample-iteration."""
    P = n * (n - 1) // 2
    return 33 * P * S + 30 * n * S + 12 * n * S * m1 + 12 * n * m1 * m1 + 42 * n * m1


def max_iters_of(config: int) -> int:
    return CONFIGS[config][4]


def global_batch(config: int, world: int, batch: int | None) -> int:
    n, H, b, scaling, _ = CONFIGS[config]
    b = batch or b
    return b * world if scaling == "weak" else b


def workload(config: int, rank: int, world: int, batch: int | None = None):
    """(problem, this rank's proposal shard, global batch): one global seeded batch, contiguous shards."""
    from paper_2501_19042_b200 import sample_proposals
    from paper_2501_19042_b200.basis import build_basis
    from paper_2501_19042_b200.distributed import shard_range
    from paper_2501_19042_b200.scenarios import config_problem
    prob = config_problem(config)
    basis = build_basis(prob.duration, degree=10, samples=prob.horizon_samples)
    B = global_batch(config, world, batch)
    props = sample_proposals(prob, basis, B, seed=0).proposals
    lo, hi = shard_range(B, world, rank)
    return prob, props[lo:hi], B


def config2_case(batch: int = 1000, precision: str = "lean"):
    """(problem, proposals, SolverConfig) of the headline workload on one GPU (tools and tests)."""
    from paper_2501_19042_b200 import SolverConfig
    prob, shard, _ = workload(2, 0, 1, batch)
    return prob, shard, SolverConfig(max_iters=MAX_ITERS, svars=False, precision=precision)


def config_label(config: int, B: int, world: int) -> str:
    n, H, _, scaling, mi = CONFIGS[config]
    what = {2: "CVAE-shaped Gaussian proposals", 3: "VQ-VAE-shaped Gaussian proposals", 4: "Gaussian proposals"}
    per = f"{B // world} per GPU" if scaling == "weak" else f"{B} strong-scaled over {world} GPU(s)"
    return (f"BASELINE config {config}: {n} drones, H={H}, batch {per}, SF to 1e-3 (max_iters {mi}), "
            f"boundary-projected start; {what[config]}")


# ----------------------------------------------------------------------------- CPU legs (reference solver)
_W = {}


def _pool_init(doc, use_ref, max_iters):
    os.environ["OPENBLAS_NUM_THREADS"] = os.environ["OMP_NUM_THREADS"] = os.environ["MKL_NUM_THREADS"] = "1"
    if use_ref:
        sys.path.insert(0, str(REF_DIR))
        import swarmfilter as sfm
        prob = sfm.load_problem(doc)
        _W.update(kind="reference", sfm=sfm, prob=prob,
                  filt=sfm.SafetyFilter(prob, degree=10, config=sfm.SolverConfig(max_iters=max_iters)))
    else:
        from oracle import sf_oracle
        _W.update(kind="port", mod=sf_oracle, prob=sf_oracle.make_problem(doc, degree=10), max_iters=max_iters)


def _pool_solve(x):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        if _W["kind"] == "reference":
            sfm = _W["sfm"]
            r = _W["filt"].solve(x)
            feas = len(sfm.metrics.feasible_results([r], _W["prob"])) == 1   # the headline's own numerator
            its = r.iterations
        else:
            r = _W["mod"].solve(_W["prob"], x, max_iters=_W["max_iters"])
            feas, its = _W["mod"].feasible(_W["prob"], r), r.iterations
        return its, bool(feas), time.perf_counter() - t0


def reference_available() -> bool:
    if not (REF_DIR / "swarmfilter").is_dir():
        return False
    code = ("import sys; sys.path.insert(0, %r); from swarmfilter import kernels; "
            "assert kernels.active_backend() == 'compiled'" % str(REF_DIR))
    return subprocess.run([sys.executable, "-c", code], capture_output=True).returncode == 0


class CpuStream:
    """One persistent fork pool streaming the proposals (cyclically) through the reference solver, 2 tasks per
    core in flight; `take(s)` counts what completes in the next s seconds: the pool's steady-state throughput,
    with no per-step pool start-up and no straggler wave at the end of a step."""

    def __init__(self, doc, props, max_iters=MAX_ITERS, cores=None):
        import itertools
        import multiprocessing as mp
        import queue
        self.use_ref = reference_available()
        self.kind = "reference" if self.use_ref else "port"
        self.cores = cores or os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_pool_init,
                                                  initargs=(doc, self.use_ref, max_iters))
        self.cyc = itertools.cycle(list(props))
        self.done = queue.Queue()
        for _ in range(2 * self.cores):
            self._submit()

    def _submit(self):
        self.pool.apply_async(_pool_solve, (next(self.cyc),), callback=self.done.put, error_callback=self.done.put)

    def take(self, seconds: float, min_samples: int = 0) -> dict:
        n = feas = its = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds or n < min_samples:
            r = self.done.get()
            if isinstance(r, BaseException):
                raise r
            self._submit()
            i, f, _ = r
            n, feas, its = n + 1, feas + int(f), its + i
        return {"samples": n, "feasible": feas, "sample_iterations": its, "wall_s": time.perf_counter() - t0}

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_desc(stream: CpuStream, r: dict, what: str) -> str:
    src = ("compiled reference (oracle/_ref: swarmfilter with its Cython kernel, SafetyFilter.solve + "
           "metrics.feasible_results)" if stream.kind == "reference" else "numpy port oracle/sf_oracle.py")
    return (f"{what}: {r['samples']} proposals of this batch, all iterations ({r['sample_iterations']} sample-"
            f"iterations) in {r['wall_s']:.1f} s, {src}, persistent process pool on {stream.cores} cores "
            f"({cpu_model()}), BLAS 1 thread/process")


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
    prob, shard, B = workload(args.config, 0, 1, args.batch)
    stream = CpuStream(prob.to_doc(), shard, max_iters_of(args.config))
    # per-step CPU time slice: --ref-budget, or ~150 s over the timed steps (2-12 s each), so the whole
    # --steps K --warmup W run stays within a few minutes
    budget = args.ref_budget if args.ref_budget is not None else min(12.0, max(2.0, 150.0 / max(1, args.steps)))
    try:
        # warm-up: fill the pool's pipeline (workers import the solver and start their first samples)
        for _ in range(max(1, args.warmup)):
            stream.take(min(budget, 3.0))
        steps = [stream.take(budget) for _ in range(args.steps)]
    finally:
        stream.close()
    wall = sum(s["wall_s"] for s in steps)
    feas = sum(s["feasible"] for s in steps)
    done = sum(s["samples"] for s in steps)
    value = feas / wall if wall > 0 else 0.0
    tot = {"samples": done, "sample_iterations": sum(s["sample_iterations"] for s in steps), "wall_s": wall}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "feasible samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True,
        "scaling": CONFIGS[args.config][3], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded scenario + reference Gaussian sampler)",
        "config": {"workload": config_label(args.config, B, 1) + "; each step a time slice of the batch",
                   "n": prob.n, "H": prob.horizon_samples - 1, "batch": B, "max_iters": max_iters_of(args.config)},
        "ms_per_1k_batch": 1e3 * 1000 / value if value > 0 else None,
        "feasible_fraction": feas / done if done else None,
        "cpu_baseline": {"value": value, "unit": "feasible samples/s", "cores": stream.cores, "kind": stream.kind,
                         "sample": cpu_desc(stream, tot, f"{args.steps} steps of {budget:.1f} s")},
        "e2e": {"value": value, "unit": "feasible samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def _timed(fn, reps: int = 1):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        r = fn()
    b.record()
    b.synchronize()
    return r, a.elapsed_time(b) / reps


def side_precisions(sf, ring, cfg, steps: int = 3) -> dict:
    """Device-timed step of the other precisions on the same batch (N = 1 only; one batch at a time, the
    inputs rotating over the copies in `ring`)."""
    import torch
    from dataclasses import replace
    out = {}
    for prec in ("hybrid", "lean", "strict"):
        if prec == cfg.precision:
            continue
        c = replace(cfg, precision=prec)
        xb = ring[0]
        sf.solve_batched(xb, config=c)
        torch.cuda.synchronize()
        step_ms, kern_ms, feas, its = [], [], 0, 0
        for k in range(steps):
            xb = ring[(k + 1) % len(ring)]
            kev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            o, ms = _timed(lambda: sf.solve_batched(xb, config=c, timing=kev))
            step_ms.append(ms)
            kern_ms.append(kev[0].elapsed_time(kev[1]))
            feas, its = int(o.feasible.sum().item()), int(o.iterations.sum().item())
        ms = statistics.median(step_ms)
        out[prec] = {"value": feas / (ms * 1e-3), "ms_per_step": ms, "ms_per_1k_batch": ms * 1000 / xb.shape[0],
                     "kernel_ms": statistics.median(kern_ms), "step_ms_all": step_ms, "feasible": feas,
                     "mean_iterations": its / xb.shape[0]}
    return out


def dropin_e2e(prob, shard, reps: int = 3) -> dict:
    """The reference-compatible call: SafetyFilter.batch_solve(list of numpy proposals) at its defaults
    (svars on) + metrics.feasible_results -- numpy in, SolveResults out (solver.py:368-407, metrics.py:57-69)."""
    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, feasible_results
    sf = SafetyFilter(prob, degree=10, config=SolverConfig(max_iters=MAX_ITERS))
    props = [x.copy() for x in shard]
    feasible_results(sf.batch_solve(props).results, prob)   # warm-up: handles, pinned staging buffers
    times, feas = [], 0
    for _ in range(reps):
        t0 = time.perf_counter()
        res = sf.batch_solve(props)
        feas = len(feasible_results(res.results, prob))
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": feas / t, "unit": "feasible samples/s", "ms_per_batch": 1e3 * t, "feasible": feas,
            "precision": sf.config.precision, "svars": True,
            "what": "SafetyFilter.batch_solve(list of numpy proposals) + feasible_results, host wall clock"}


def pipeline_e2e(prob, batch: int, reps: int = 8) -> dict:
    """BASELINE config 2 as stated: CVAE samples -> QP layer -> init-network warm start -> SF -> verdict."""
    import torch

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig
    from paper_2501_19042_b200.generative import FusedDecoder, calibrate_batchnorm, decode_proposals, make_decoder
    from paper_2501_19042_b200.initnet import FoldedInitNet, InitNet, initial_states
    from paper_2501_19042_b200.unrolled import device_constants_of
    torch.manual_seed(0)
    sf = SafetyFilter(prob, degree=10, config=SolverConfig(max_iters=MAX_ITERS, svars=False))
    dec = calibrate_batchnorm(sf, make_decoder("cvae", prob.n).cuda()).eval()
    fused = FusedDecoder(dec)   # K4: the decoder's forward pass as one sm_100a kernel
    net = InitNet(prob.n, sf.coeff_dim).cuda().eval()
    net = FoldedInitNet(net, device_constants_of(sf, "cuda")["context"][None])   # per-problem folded GEMMs
    gen = torch.Generator(device="cuda").manual_seed(0)
    # one warm-up pass, then `reps` passes enqueued back to back (no host sync between them) so the
    # stage times are the device's, not the host's launch latency after a synchronize
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps + 1)]
    acc = [0.0, 0.0, 0.0]
    out = None
    for r in range(reps + 1):
        with torch.no_grad():
            ev[r][0].record()
            xb = decode_proposals(sf, dec, dec.sample_latent(batch, gen, "cuda"), fused)
            ev[r][1].record()
            xi0, lam0 = initial_states(sf, xb, "initnet", net)
            ev[r][2].record()
            out = sf.solve_batched(xb, xi0=xi0, lam0=lam0)
            ev[r][3].record()
        if r == 0:
            ev[0][3].synchronize()
    ev[reps][3].synchronize()
    for r in range(1, reps + 1):
        for i in range(3):
            acc[i] += ev[r][i].elapsed_time(ev[r][i + 1]) / reps
    total = sum(acc)
    feas = int(out.feasible.sum().item())
    return {"value": feas / (total * 1e-3), "unit": "feasible samples/s", "decode_qp_ms": acc[0],
            "initnet_ms": acc[1], "sf_verdict_ms": acc[2], "total_ms": total, "feasible": feas,
            "mean_iterations": float(out.iterations.double().mean()),
            "note": "random-init CVAE decoder (kernel K4) and init network (no trained weights offline), device-timed"}


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, native
    from paper_2501_19042_b200.distributed import GATHERED_FIELDS, gather_outputs, gather_outputs_async
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    prob, shard, B = workload(args.config, rank, world, args.batch)
    cfg = SolverConfig(max_iters=max_iters_of(args.config), svars=False, precision=args.precision)
    sf = SafetyFilter(prob, degree=10, config=cfg)
    n, S, m1 = prob.n, prob.horizon_samples, 11
    xb_host = torch.from_numpy(shard).pin_memory()
    xb = xb_host.to(dev)
    dim = xb.shape[1]
    # inputs larger than L2 instead of a flush: the steps rotate over R device copies of the batch, >= 256 MB
    # in all (2x the 126 MB L2), so no step finds its proposals L2-resident from an earlier step
    ring = [xb] + [xb.clone() for _ in range(max(2, -(-256 * 2**20 // max(1, xb.numel() * 8))) - 1)]
    peak_tflops = ctypes_peak(native)

    def step(x, timing=None):
        out = sf.solve_batched(x, config=cfg, timing=timing)
        full = gather_outputs(out, B) if world > 1 else None
        return out, full

    clocks = ClockSampler(ROOT / "gpurun_out" / f"clocks_rank{rank}.csv") if rank == 0 else None
    if clocks:
        (ROOT / "gpurun_out").mkdir(exist_ok=True)
        clocks.__enter__()
    for _ in range(max(3, args.warmup)):
        step(xb)
    # (and the two-in-flight submission: its side streams and their allocator pools, outside the timed region)
    sf.solve_pipelined((ring[k % len(ring)] for k in range(max(4, args.warmup))), config=cfg,
                       finish=(lambda k, out: gather_outputs(out, B)) if world > 1 else None, keep=False)
    torch.cuda.synchronize()
    if clocks:
        clocks.wait_first()

    # ---- device-timed region (the headline value): inputs resident in HBM, K batches with two in flight
    # (SafetyFilter.solve_pipelined: batch k on side stream k % 2, so the next batch's CTAs start on the SMs
    # the previous batch's tail frees); each batch is still its own launch with its own outputs
    # each step's verdicts and counts are copied aside (device-to-device copies: copy engines, not SMs) and its
    # outputs dropped, so the caching allocator reuses their blocks (keeping K batches' outputs alive made the
    # first timed run allocate); a kernel here would wait for an SM behind the other stream's batch
    nb = int(xb.shape[0])
    feas_k = torch.empty((args.steps, nb), dtype=torch.uint8, device=dev)
    its_k = torch.empty((args.steps, nb), dtype=torch.int32, device=dev)

    pend = []   # N > 1: the NCCL gathers of the steps' outputs, asynchronous (finished after the loop, in the timing)

    def gather(k, out):
        if world > 1:
            pend.append(gather_outputs_async(out, B))
        feas_k[k].copy_(out.feasible, non_blocking=True)
        its_k[k].copy_(out.iterations, non_blocking=True)

    launches0 = native.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.mark()
    a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    sf.solve_pipelined((ring[k % len(ring)] for k in range(args.steps)), config=cfg, finish=gather, keep=False)
    for fin in pend:
        fin()
    pend.clear()
    b0.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = native.launch_count() - launches0
    pipe_ms = a0.elapsed_time(b0)
    pfeas = int(feas_k.sum().item())
    pits = int(its_k.to(torch.int64).sum().item())

    # ---- the same K batches one after another (one stream): the per-batch latency and the per-launch
    # kernel time of the roofline (the kernel alone on the GPU)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    outs = []
    for k in range(args.steps):
        ev[k][0].record()
        out, full = step(ring[k % len(ring)], timing=kev[k])
        ev[k][1].record()
        outs.append((out.feasible, out.iterations))   # the rest is freed: the next step reuses its blocks
        del out, full
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if clocks:
        time.sleep(0.15)   # one more sample after the last step
        clocks.mark()
        clocks.__exit__()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    feas_counts = [int(f.sum().item()) for f, _ in outs]
    its_total = [int(i.sum().item()) for _, i in outs]
    if pfeas != sum(feas_counts) or pits != sum(its_total):
        raise SystemExit(f"pipelined batches disagree with the sequential ones: {pfeas} vs {sum(feas_counts)} feasible")
    t = torch.tensor([pipe_ms, sum(step_ms), float(pfeas), float(pits)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax[:2], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[2:], op=dist.ReduceOp.SUM)
        total_ms_max, seq_ms_max = float(tmax[0]), float(tmax[1])
    else:
        total_ms_max, seq_ms_max = float(t[0]), float(t[1])
    feas_all, its_all = float(t[2]), float(t[3])
    value = feas_all / (total_ms_max * 1e-3)

    # ---- end to end through the public API: pinned host proposals in, every per-sample output out, the
    # same two-in-flight submission (H2D, solve, D2H of batch k on its stream; no host sync between batches)
    probe, _ = step(xb)
    host = [{}, {}]
    for k in GATHERED_FIELDS + ("eq_err",):
        v = getattr(probe, k, None)
        if v is not None:
            for hb in host:
                hb[k] = torch.empty(tuple(v.shape), dtype=v.dtype).pin_memory()
    del probe

    def h2d(k, _):
        return xb_host.to(dev, non_blocking=True)

    def d2h(k, out):
        for key, h in host[k % 2].items():
            h.copy_(getattr(out, key), non_blocking=True)

    e2e_ms = []
    for rep in range(2):   # the first one is a warm-up
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sf.solve_pipelined(range(args.steps), config=cfg, prepare=h2d, finish=d2h, keep=False)
        b.record()
        b.synchronize()
        if rep:
            e2e_ms.append(a.elapsed_time(b))
    e2e_feas = int(host[(args.steps - 1) % 2]["feasible"].numpy().sum())
    te = torch.tensor([sum(e2e_ms), float(e2e_feas * args.steps)], dtype=torch.float64, device=dev)
    if world > 1:
        temax = te.clone()
        dist.all_reduce(temax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(te[1:], op=dist.ReduceOp.SUM)
        e2e_value = float(te[1]) / (float(temax[0]) * 1e-3)
    else:
        e2e_value = float(te[1]) / (float(te[0]) * 1e-3)
    h2d_bytes = xb_host.numel() * 8
    d2h_bytes = sum(h.numel() * h.element_size() for h in host[0].values())

    if rank != 0:
        return
    # ---- roofline of the dominant kernel (persistent SF kernel, this rank)
    fps = flop_per_si(n, S, m1)
    flops_per_launch = statistics.mean(its_total) * fps
    kern_avg_ms = statistics.mean(kern_ms)
    achieved = flops_per_launch / (kern_avg_ms * 1e-3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            traffic = tj.get(f"config{args.config}_{args.precision}", {}).get("dram_bytes_per_launch")
        except (ValueError, OSError, AttributeError):
            traffic = None
    kname = {16: "sf_persistent_kernel<float,16> (tcgen05 positions)", 32: "sf_persistent_kernel<32, two lanes>",
             64: "sf_large_kernel<64>"}.get(n, "sf_persistent_kernel")
    line = {
        "metric": METRIC, "value": value, "unit": "feasible samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": total_ms_max / args.steps,
        "higher_is_better": True, "scaling": CONFIGS[args.config][3], "vs_baseline": None,
        "dtype": {"lean": "f32 terms + f64 state", "hybrid": "f32 screening + f64 values",
                  "strict": "f64"}[args.precision],
        "data": "synthetic (seeded scenario, reference Gaussian sampler proposals)",
        "config": {"workload": config_label(args.config, B, world), "n": n, "H": S - 1, "degree": 10,
                   "batch": B, "batch_per_gpu": int(xb.shape[0]), "max_iters": cfg.max_iters, "rho": 1.0,
                   "precision": args.precision, "l2_flush": f"no flush kernel: inputs larger than L2 (the steps rotate over {len(ring)} device copies of the batch, {len(ring) * xb.numel() * 8 / 2**20:.0f} MB)",
                   "parallelism": f"dp{world} (contiguous sample shards"
                                  + (", NCCL all_gather of every per-sample output in the step)" if world > 1 else ")")},
        "ms_per_1k_batch": (total_ms_max / args.steps) * 1000.0 / B,
        "feasible_fraction": feas_all / (args.steps * B),
        "mean_iterations": its_all / (args.steps * B),
        "gpu_launches": int(round(launches / args.steps)),
        "e2e": {"value": e2e_value, "unit": "feasible samples/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes, "outputs": sorted(host[0])},
        "pipelining": {"batches_in_flight": 2, "batch_latency_ms": seq_ms_max / args.steps,
                       "sequential_value": feas_all / (seq_ms_max * 1e-3),
                       "note": "value / ms_per_step: the K batches submitted with two in flight "
                               "(SafetyFilter.solve_pipelined); batch_latency_ms / sequential_value: the same "
                               "K batches one after another; roofline: per-launch kernel time of the latter"},
        "roofline": {"bound": "fp32_cuda_core", "achieved": achieved, "peak": peak_tflops,
                     "unit": "TFLOP/s", "frac": achieved / peak_tflops if peak_tflops else None,
                     # the same algorithmic FLOPs over the two-in-flight region (the tail's idle SMs filled)
                     "frac_pipelined": (pits * fps / (pipe_ms * 1e-3) / 1e12) / peak_tflops if peak_tflops else None,
                     "traffic": traffic, "kernel": kname, "kernel_ms": kern_avg_ms, "flop_per_si": fps,
                     "peak_source": "FFMA microbenchmark (sgsf_fp32_peak) run live in this process; "
                                    "MEASURED_PEAKS.json has no FP32 figure"},
        "clocks": clocks.summary(local_rank) if clocks else None,
    }
    if world == 1 and not args.quick:
        line["precisions"] = side_precisions(sf, ring, cfg)
        if args.config == 2:
            line["e2e_dropin"] = dropin_e2e(prob, shard)
            line["pipeline"] = pipeline_e2e(prob, int(xb.shape[0]))
    if args.cpu_baseline and world == 1:
        stream = CpuStream(prob.to_doc(), shard, cfg.max_iters)
        budget = args.ref_budget if args.ref_budget is not None else 12.0
        try:
            if prob.n > 32:
                # 64 robots: one sample takes ~95 s on a core, so a 12 s slice after a warm-up would count one
                # straggler.  Count from the pool's start until every core has finished a sample instead.
                r = stream.take(budget, min_samples=stream.cores)
            else:
                stream.take(3.0)   # pool start-up and the first wave
                r = stream.take(budget)
        finally:
            stream.close()
        si_rate = r["sample_iterations"] / r["wall_s"]
        line["cpu_baseline"] = {"value": r["feasible"] / r["wall_s"], "unit": "feasible samples/s",
                                "cores": stream.cores, "kind": stream.kind,
                                "sample": cpu_desc(stream, r, "one 12 s time slice" if prob.n <= 32 else
                                                   "from the pool's start until every core finished a sample"),
                                "sample_iterations_per_s": si_rate,
                                # a slice of a few slow samples (config 4: ~95 s each on one core) says little
                                # about the feasible rate; this is the CPU's iteration rate times the batch's own
                                # feasible samples per sample-iteration (the GPU run's, equal to the
                                # reference's by the parity tests)
                                "value_from_iteration_rate": si_rate * line["feasible_fraction"] / max(
                                    line["mean_iterations"], 1e-9)}
    print(json.dumps(line), flush=True)


def run_stub(args, rank: int, world: int) -> None:
    """`--stub` (CPU, gloo): the launcher, sharding, output gather and max-over-ranks reduction of the real
    arm with the solve replaced by row-identifying fake outputs -- for tests/test_bench_launcher.py."""
    import torch
    import torch.distributed as dist

    from paper_2501_19042_b200.distributed import gather_outputs, shard_range
    prob, shard, B = workload(args.config, rank, world, args.batch)
    lo, hi = shard_range(B, world, rank)
    steps_ms, feas = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rows = torch.arange(lo, hi, dtype=torch.float64)
        out = {"coeffs": torch.from_numpy(shard).clone(), "iterations": (rows % 7).to(torch.int32),
               "feasible": (rows.to(torch.int64) % 3 == 0).to(torch.uint8)}
        full = gather_outputs(out, B) if world > 1 else out
        assert full["coeffs"].shape[0] == B
        feas = int(full["feasible"].sum())
        steps_ms.append(1e3 * (time.perf_counter() - t0))
    t = torch.tensor([sum(steps_ms)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": feas * args.steps / (float(t[0]) * 1e-3), "unit": "feasible samples/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(t[0]) / args.steps,
                          "scaling": CONFIGS[args.config][3], "stub": True, "feasible_per_step": feas,
                          "config": {"workload": config_label(args.config, B, world), "batch": B,
                                     "batch_per_gpu": hi - lo}}), flush=True)


def ctypes_peak(native) -> float:
    import ctypes

    import torch
    tf, ms = ctypes.c_double(), ctypes.c_double()
    native.check(native.load().sgsf_fp32_peak(ctypes.byref(tf), ctypes.byref(ms),
                                              torch.cuda.current_stream().cuda_stream), "sgsf_fp32_peak")
    return float(tf.value)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: re-run this command as N ranks (one process per GPU, NCCL)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=None, help="batch (per GPU for config 2; global for 3/4)")
    ap.add_argument("--precision", default="hybrid", choices=["hybrid", "lean", "strict"])
    ap.add_argument("--ref-budget", type=float, default=None,
                    help="seconds of CPU time slice per reference step (default: 12 s for the cpu_baseline leg; "
                         "150 s / steps, within 2-12 s, for --impl reference)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--quick", action="store_true", help="skip the side precisions, drop-in and pipeline numbers")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)   # CPU/gloo launcher test (no GPU)
    return ap.parse_args(argv)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(launch_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.stub:
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
        try:
            run_stub(args, rank, world)
        finally:
            if world > 1:
                dist.destroy_process_group()
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
