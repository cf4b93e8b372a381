#!/usr/bin/env python
"""Benchmark: complex DD/QD polynomial system + Jacobian evaluations per second on B200
(BASELINE.json metric: "complex DD/QD system+Jacobian evals/sec; achieved % of B200 FP64 peak").

One "step" = one pass of the whole hot path (power table, Speelpenning monomial stage,
coefficient product, reductions, writes of F and J: SURVEY.md §8(a) rows a1-a8) over one batch
of synthetic points resident in HBM.

Default workload: BASELINE.json configs[4] "large" as its 4,096-point batch (n = m = 256,
k = 32, D = 8, complex QD -- the paper's tracking precision), the largest
configuration that fits one GPU.  At N = 1 the same JSON line also carries nested records for
the large single point ("large_single": median of >= 200 calls, L2 flushed before each) and for
the DD batch config ("batch_dd": configs[3], 65,536 points), each with its own clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

Multi-GPU (SURVEY.md §8(e), strong scaling of ONE fixed batch):
  * under torchrun (WORLD_SIZE = N, one process per GPU): rank r evaluates the contiguous
    shard [rP/N, (r+1)P/N) of the batch through phc_eval_jacobian_batch_range and its kernels
    store F and J straight into rank 0's buffers, mapped with CUDA IPC -- the final gather is
    fused into the evaluation (NVLink stores), no collective on the data path; NCCL
    point-to-point copies are the fallback when IPC is refused;
  * without torchrun, --gpus N > 1 runs one process calling phc_eval_jacobian_batch with the
    device list 0..N-1 (the library's own sharded call, fused peer stores).
  Timed region: barrier + synchronize on both sides, max over ranks of the device time.

`--impl reference` times the CPU oracle (oracle/, the plain definition in exact rationals or
mpmath at 512 bits) on the same workload, a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "large_batch"
METRIC = "complex DD/QD system+Jacobian evals/sec"
DATA = "synthetic (seeded unit-circle systems and points, BASELINE.json recipe; DESIGN.md §5)"
# SURVEY.md §8(d) frozen model (paper-faithful op counts, standard DD costs): reported beside
# the executed count, not the roofline numerator
MODEL_FLOPS = {2: dict(cm=80, ca=40), 4: dict(cm=800, ca=200)}
# nominal FP64 peak derived from the unit counts and the clock:
# 148 SMs x 64 FP64 FMA/clk/SM x 2 flops x 1.965 GHz (clocks.max.sm)
SMS, FMA_PER_SM_CLK, SM_MAX_MHZ = 148, 64, 1965.0


def nominal_fp64_tflops(sm_mhz=SM_MAX_MHZ):
    return SMS * FMA_PER_SM_CLK * 2 * sm_mhz * 1e6 / 1e12


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: 10, batch DD 20)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--points", type=int, default=None, help="override the batch size")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--single-calls", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nested", action="store_true", help="skip the nested large_single / batch_dd records")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=None, help="reference arm: rows per step (QD configs)")
    ap.add_argument("--verify", action="store_true",
                    help="torchrun mode: rank 0 re-evaluates the whole batch alone and checks the gathered F, J bitwise")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------------------
# host-side plumbing (CPU-testable with gloo: tests/test_dist.py)
# ---------------------------------------------------------------------------------------

def shard_range(rank, world, P):
    """The batch call's sharding rule (include/phc.h): contiguous ranges [rP/N, (r+1)P/N)."""
    return rank * P // world, (rank + 1) * P // world


def max_over_ranks(value, world, device=None):
    """The timing rule: the slowest rank defines the time (all_reduce MAX)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(points_total, steps, ms_max):
    """Whole-job throughput: every point of the batch, all steps, over the max-over-ranks time."""
    return points_total * steps / (ms_max * 1e-3)


def share_handles(rank, world, payload):
    """Rank 0's IPC handles (bytes) to every rank (broadcast_object_list)."""
    import torch.distributed as dist
    obj = [payload if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]


def gather_to_rank0(rank, world, full, shard_rows):
    """Fallback gather without IPC: rank r sends rows [p0, p1) of `full` to rank 0 (point to
    point; NCCL on GPUs, gloo in the CPU test).  `full` has the batch as its leading axis."""
    import torch.distributed as dist
    if world <= 1:
        return
    if rank == 0:
        for r in range(1, world):
            a, b = shard_rows(r)
            dist.recv(full[a:b], src=r)
    else:
        a, b = shard_rows(rank)
        dist.send(full[a:b].contiguous(), dst=0)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_dict(name, c, P, flush, parallelism):
    return {
        "workload": name,
        "seed": 1,
        "n": c["n"], "m": c["m"], "k": c["k"], "D": c["D"],
        "precision": "complex DD" if c["limbs"] == 2 else "complex QD",
        "points": P,
        "l2": "flushed before every timed step (256 MiB write)" if flush else "not flushed",
        "parallelism": parallelism,
    }


def model_counts(s, st):
    """CM = T(6k-5) + n(D-2), CA = n(m-1) + T k - nnz(J) (paper-faithful)."""
    import numpy as np
    k = np.diff(s.term_ptr)
    cm = int(np.sum(np.where(k >= 1, 6 * k - 5, 0))) + s.n_var * max(0, int(st["D"]) - 2)
    m = np.diff(s.poly_ptr)
    ca = int(np.sum(np.maximum(m - 1, 0))) + int(k.sum()) - int(st["nnz_J"])
    return cm, ca


def latency_kernel_name(st):
    return f"poly_seg_kernel<4,{st['latency_G']}>" if st["latency_kernel"] == 2 else "poly_scan_kernel"


def latency_path_name(st):
    if st["latency_kernel"] == 2:
        return f"latency (segmented: {st['latency_G']} lanes per term, power table + kernel)"
    return "latency (one warp per term)"


def launches_per_call(st, points):
    """kernel launches of one eval call with `points` points (phc_system_stats)"""
    return int(st["latency_launches"] if latency_regime(st, points) else st["launches"])


def latency_regime(st, points):
    """True when a call with `points` points takes the latency path (phc.h: n_points * n_terms
    <= the bound in phc_system_stats out[13])."""
    return st["latency_bound"] > 0 and points * st["n_terms"] <= st["latency_bound"]


def exec_flops_per_point(st, points):
    """Executed FP64 flops per point of the kernels' useful work, as counted by the library
    (phc_system_stats; per-op costs from arith.cuh, checked against ncu)."""
    if latency_regime(st, points):
        return int(st["latency_exec_flops_per_point"])
    return int(st["exec_flops_per_point"])


def traffic_per_point(workload):
    """DRAM bytes per point of the dominant kernel from the committed ncu capture (profiles/traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[workload]["bytes_per_point"]
    except (OSError, KeyError, ValueError):
        return None


class ClockSampler:
    """nvidia-smi clocks during a timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        try:
            for line in open(self.f.name):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        finally:
            os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[4 + j].lower() == "active"})
        loaded = sorted(x for x in sm if x > 500) or sorted(sm)
        med = loaded[len(loaded) // 2] if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands
# ---------------------------------------------------------------------------------------

def sample_rows(s, rows, terms_per_row):
    """A bounded sample of the workload for the oracle: the first `terms_per_row` terms of each
    polynomial in `rows`, as a system of len(rows) polynomials over the same n_var variables
    (the same terms, so the same work per term as the full evaluation)."""
    import numpy as np
    from synthetic import SystemArrays
    tsel = []
    for i in rows:
        a, b = int(s.poly_ptr[i]), int(s.poly_ptr[i + 1])
        tsel.extend(range(a, min(b, a + terms_per_row)))
    pp = [0]
    for i in rows:
        a, b = int(s.poly_ptr[i]), int(s.poly_ptr[i + 1])
        pp.append(pp[-1] + min(b - a, terms_per_row))
    tp = [0]
    vi, ex = [], []
    for t in tsel:
        a, b = int(s.term_ptr[t]), int(s.term_ptr[t + 1])
        vi.extend(s.var_idx[a:b].tolist())
        ex.extend(s.exponent[a:b].tolist())
        tp.append(len(vi))
    return SystemArrays(n_eq=len(rows), n_var=s.n_var, limbs=s.limbs, poly_ptr=np.array(pp, np.int64),
                        term_ptr=np.array(tp, np.int64), var_idx=np.array(vi, np.int32),
                        exponent=np.array(ex, np.int32), coeff=np.ascontiguousarray(s.coeff[tsel])), len(tsel)


def run_reference(args):
    """--impl reference: the oracle (naive evaluator; exact rationals for the DD configs and c3,
    mpmath 512 bits for the large QD config) on the host cores, a bounded sample per step: one
    whole point for n <= 64; for the large config `cores` polynomials x 32 of their terms (one
    polynomial per process), the value scaled by the fraction of the point's terms evaluated."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import evaluate_rows
    from synthetic import CONFIGS, config_system
    c = CONFIGS[args.workload]
    npts = max(args.steps_eff + args.warmup, 1)
    s, X = config_system(args.workload, seed=1, points=min(npts, c["points"]))
    small = c["n"] <= 64
    arith = "exact" if small else "mp"
    cores = host_cores()
    tpr = 32
    nrows = min(args.ref_rows or cores, s.n_eq)

    def one(i):
        if small:
            evaluate_rows(s, X[i % X.shape[0]], None, arith)
            return 1.0
        rows = [(i * nrows + r) % s.n_eq for r in range(nrows)]
        sub, nt = sample_rows(s, rows, tpr)
        evaluate_rows(sub, X[i % X.shape[0]], None, arith)
        return nt / s.n_terms

    for w in range(args.warmup):
        one(w)
    t = 0.0
    work = 0.0
    for i in range(args.steps_eff):
        t0 = time.perf_counter()
        work += one(args.warmup + i)
        t += time.perf_counter() - t0
    v = work / t
    sample = (f"each step = one full point ({arith} arithmetic, rows over {cores} processes)" if small else
              f"each step = {tpr} terms of each of {nrows} polynomials of one point ({nrows * tpr} of "
              f"{s.n_terms} terms, full Jacobian rows; mpmath 512 bits, one polynomial per process on "
              f"{cores} processes); evals/s = evaluated fraction of the point / time")
    out = {
        "metric": METRIC, "value": v, "unit": "evals/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps_eff, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps_eff,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (exact / mp512 oracle)",
        "data": DATA,
        "config": config_dict(args.workload, c, c["points"], False, "host cores (oracle)"),
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "cpu": cpu_model(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


def cpu_baseline(workload, steps=2):
    """The oracle timed on this host's cores on a bounded sample (rank 0, N = 1 only): the
    reference arm itself, run in a fresh subprocess (its process pool then forks from a
    process without CUDA state, so the figure equals the --impl reference arm's)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
           "--steps", str(steps), "--warmup", "0"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    for line in r.stdout.splitlines()[::-1]:
        if line.startswith("{"):
            cb = json.loads(line)["cpu_baseline"]
            cb["sample"] = f"{steps} steps of the reference arm: " + cb["sample"]
            return cb
    return {"value": None, "unit": "evals/s", "cores": host_cores(), "kind": "oracle",
            "sample": f"reference arm failed: {r.stderr[-300:]}"}


# ---------------------------------------------------------------------------------------
# GPU measurements
# ---------------------------------------------------------------------------------------

def roofline(exec_pp, points_per_launch, ms_per_launch, peak_run, workload, kernel):
    achieved = exec_pp * points_per_launch / (ms_per_launch * 1e-3) / 1e12 if ms_per_launch > 0 else 0.0
    nominal = nominal_fp64_tflops()
    tpp = traffic_per_point(workload)
    return {
        "bound": "alu",
        "kernel": kernel,
        "achieved": achieved,
        "peak": nominal,
        "unit": "TFLOP/s",
        "frac": achieved / nominal,
        "traffic": tpp * points_per_launch if tpp else None,
        "peak_source": (f"nominal FP64: {SMS} SMs x {FMA_PER_SM_CLK} FMA/clk x 2 x {SM_MAX_MHZ:.0f} MHz "
                        "(DESIGN.md §4; MEASURED_PEAKS.json has no FP64 entry)"),
        "peak_measured_in_run": peak_run,
        "frac_of_measured": achieved / peak_run if peak_run else None,
        "peak_measured_source": "phc_fp64_peak: independent DFMA chains on this GPU in this run",
        "flops": "executed FP64 flops (DADD = DMUL = 1, DFMA = 2) of the kernel's useful work per launch",
        "traffic_source": "profiles/traffic.json (ncu --set full: dram read+write bytes per point x points)",
    }


def measure_batch(phc, h, Xd, F, J, steps, warmup, stream, scrub, local, devices=None):
    """Per-step CUDA-event times of eval_batch (after `warmup` steps), the library's per-class
    kernel times over the timed region, and the clocks during it."""
    import torch
    for _ in range(max(warmup, 0)):
        h.eval_batch(Xd, F, J, devices=devices, stream=stream)
    torch.cuda.synchronize()
    phc.phc_profile_enable(h._h, True)
    phc.phc_profile_read(h._h, reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(steps):
            if scrub is not None:
                scrub.fill_(i & 0xFF)
            ev[i][0].record(stream)
            h.eval_batch(Xd, F, J, devices=devices, stream=stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    kms, kn = phc.phc_profile_read(h._h, reset=True)
    phc.phc_profile_enable(h._h, False)
    return [a.elapsed_time(b) for a, b in ev], kms, kn, clk.summary()


def measure_e2e(h, X, steps, devices=None):
    """End to end through the host-pointer C-ABI call (phc_eval_jacobian_batch_host): pinned
    host X in, pinned host F and J out, H2D + evaluation + D2H inside the timed region."""
    import torch
    P = X.shape[0]
    Xh = torch.from_numpy(X).pin_memory()
    Fh = torch.empty((P, h.n_eq, 2, h.limbs), dtype=torch.float64).pin_memory()
    Jh = torch.empty((P, h.n_eq, h.n_var, 2, h.limbs), dtype=torch.float64).pin_memory()
    h.eval_batch_host(Xh.numpy(), Fh.numpy(), Jh.numpy(), devices=devices)  # warm-up (allocates staging)
    t0 = time.perf_counter()
    for _ in range(steps):
        h.eval_batch_host(Xh.numpy(), Fh.numpy(), Jh.numpy(), devices=devices)
    dt = time.perf_counter() - t0
    bi, bo = Xh.numel() * 8, (Fh.numel() + Jh.numel()) * 8
    del Xh, Fh, Jh
    return dt, bi, bo


def measure_single(phc, h, x, calls, local, flush=True):
    """Single-point latency: `calls` timed calls of phc_eval_jacobian (after 10 warm-ups), each
    preceded by an L2 flush (256 MiB write) and bracketed by its own CUDA events; median."""
    import torch
    dev = x.device
    f = torch.empty((h.n_eq, 2, h.limbs), dtype=torch.float64, device=dev)
    j = torch.empty((h.n_eq, h.n_var, 2, h.limbs), dtype=torch.float64, device=dev)
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    stream = torch.cuda.current_stream(dev)
    for _ in range(10):
        h.eval(x, f, j, stream=stream)
    torch.cuda.synchronize()
    phc.phc_profile_enable(h._h, True)
    phc.phc_profile_read(h._h, reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(calls)]
    with ClockSampler(local) as clk:
        for i in range(calls):
            if scrub is not None:
                scrub.fill_(i & 0xFF)
            ev[i][0].record(stream)
            h.eval(x, f, j, stream=stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    _, kn = phc.phc_profile_read(h._h, reset=True)
    phc.phc_profile_enable(h._h, False)
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    st = h.stats
    nl = max(int(sum(kn)), launches_per_call(st, 1) * calls)
    return us, clk.summary(), nl, f.cpu().numpy(), j.cpu().numpy()


def _exact_ints(limbs, scale=1300):
    """[N][2][L] float64 limbs -> (re, im) exact integer multiples of 2^-scale (Python ints)."""
    out = []
    for v in limbs:
        parts = []
        for part in v:
            acc = 0
            for d in part:
                num, den = float(d).as_integer_ratio()
                acc += num << (scale - (den.bit_length() - 1))
            parts.append(acc)
        out.append(parts)
    return out


def _golden_err(gpu, ref):
    """max(||d||_inf / ||ref||_inf, ||d||_F / ||ref||_F), entries as complex moduli, from exact
    squared moduli (integers); only the final ratio is rounded.  gpu [..][2][L], ref [..][2][10]."""
    import numpy as np
    from fractions import Fraction
    a = _exact_ints(np.asarray(gpu).reshape(-1, 2, np.asarray(gpu).shape[-1]))
    b = _exact_ints(np.asarray(ref).reshape(-1, 2, np.asarray(ref).shape[-1]))
    if len(a) != len(b):
        raise ValueError(f"{len(a)} GPU values against {len(b)} oracle values")
    d2 = [(x[0] - y[0]) ** 2 + (x[1] - y[1]) ** 2 for x, y in zip(a, b)]
    r2 = [y[0] ** 2 + y[1] ** 2 for y in b]
    if max(r2) == 0:
        return 0.0 if max(d2) == 0 else float("inf")
    return float(max(Fraction(max(d2), max(r2)), Fraction(sum(d2), sum(r2)))) ** 0.5


def parity_vs_golden(f, j):
    """Normwise relative errors (reading C9) of the large point 0's F and J against the
    committed oracle values (tests/golden/large_seed1.npz, written by tools/make_golden_large.py
    from the mp512 oracle): exact integer arithmetic on the limbs, no oracle code executed."""
    import numpy as np
    g = np.load(os.path.join(ROOT, "tests", "golden", "large_seed1.npz"))

    return {"err_F": _golden_err(f, g["F0"]), "err_J": _golden_err(j, g["J0"]), "tolerance": 1e-60,
            "checked": f"all {f.shape[0]} F and {j.shape[0] * j.shape[1]} J entries of point 0 against the "
                       "committed mp512 oracle values (tests/golden/large_seed1.npz)"}


def parity_batch(workload, F, J):
    """The batch line's own parity: GPU rows at the committed oracle points (batch: every entry
    of 16 points, exact-rational oracle; large_batch: 8 rows at each of 8 points, mp512 oracle)
    against tests/golden/*_seed1.npz, normwise per point (reading C9); the worst point reported."""
    import numpy as np
    if workload == "batch":
        g = np.load(os.path.join(ROOT, "tests", "golden", "batch_seed1.npz"))
        pts = [int(p) for p in g["points"]]
        cases = [(F[p].cpu().numpy(), J[p].cpu().numpy(), g["F"][q], g["J"][q]) for q, p in enumerate(pts)]
        what, tol = f"every entry of F and J at {len(pts)} points (first and last of each 8-way shard)", 1e-28
    elif workload == "large_batch":
        g = np.load(os.path.join(ROOT, "tests", "golden", "large_seed1.npz"))
        pts = [int(p) for p in g["batch_points"]]
        cases = []
        for q, p in enumerate(pts):
            rows = [int(r) for r in g["batch_rows"][q]]
            cases.append((F[p].cpu().numpy()[rows], J[p].cpu().numpy()[rows], g["Fb"][q], g["Jb"][q]))
        what, tol = f"8 rows of F and J at each of {len(pts)} points", 1e-60
    else:
        return None
    ef = ej = 0.0
    for f, j, gf, gj in cases:
        ef = max(ef, _golden_err(f, gf))
        ej = max(ej, _golden_err(j, gj))
    return {"err_F": ef, "err_J": ej, "tolerance": tol,
            "checked": what + f" against the committed oracle values (tests/golden/, {workload})"}


def built_points(workload):
    """The full batch size of a workload (the golden points index into it)."""
    from synthetic import CONFIGS
    return CONFIGS[workload]["points"]


def build_workload(workload, P, device):
    import paper_1109_0545_b200 as phc
    from synthetic import CONFIGS, config_system
    c = CONFIGS[workload]
    P = P or c["points"]
    s, X = config_system(workload, seed=1, points=P)
    return c, s, X, phc.System(s, device=device)


def batch_record(phc, workload, P, steps, warmup, flush, local, e2e_steps, peak_run, devices=None, label=None,
                 built=None):
    """One batch workload on this process's device(s): the throughput line fields."""
    import torch
    dev = torch.device("cuda", local)
    c, s, X, h = built or build_workload(workload, P, local)
    P = X.shape[0]
    st = h.stats
    Xd = torch.from_numpy(X).to(dev)
    F = torch.empty((P, s.n_eq, 2, s.limbs), dtype=torch.float64, device=dev)
    J = torch.empty((P, s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    ms_list, kms, kn, clocks = measure_batch(phc, h, Xd, F, J, steps, warmup, stream, scrub, local, devices)
    ms = sum(ms_list)
    ok = bool(torch.isfinite(F).all().item()) and bool(torch.isfinite(J).all().item())
    parity = parity_batch(workload, F, J) if P == built_points(workload) else None
    del Xd, F, J, scrub
    torch.cuda.empty_cache()
    e2e_s, bi, bo = measure_e2e(h, X, e2e_steps, devices)
    cm_model, ca_model = model_counts(s, st)
    mf = MODEL_FLOPS[s.limbs]
    model_pp = cm_model * mf["cm"] + ca_model * mf["ca"]
    exec_pp = exec_flops_per_point(st, P)
    names = ["power_table", "term", "reduce", latency_kernel_name(st) if latency_regime(st, P) else "fused_block"]
    dom = max(range(4), key=lambda i: kms[i])
    dom_ms = kms[dom] / max(kn[dom], 1)
    launches_dom_per_step = max(kn[dom] / steps, 1)
    kernel = {3: f"block_kernel<{s.limbs},{st['K']},{st['layout']},0>" if not latency_regime(st, P)
              else latency_kernel_name(st)}.get(dom, names[dom])
    step_s = ms / steps * 1e-3
    multi = devices is not None and len(devices) > 1
    rl = roofline(exec_pp, P / launches_dom_per_step, dom_ms, peak_run, workload, kernel)
    if multi:
        rl["note"] = "kernel time of the home device's shard only; the step time covers every device"
    rec = {
        "value": aggregate_value(P, steps, ms),
        "ms_per_step": ms / steps,
        "ms_per_step_median": statistics.median(ms_list),
        "config": config_dict(workload, c, P, flush,
                              f"points sharded over devices {list(devices)} (one process)" if multi else "one GPU"),
        "path": latency_path_name(st) if latency_regime(st, P) else "batch kernels",
        "roofline": rl,
        "fp64": {
            "step_exec_tflops": exec_pp * P / step_s / 1e12,
            "step_exec_frac": exec_pp * P / step_s / 1e12 / nominal_fp64_tflops(),
            "step_model_tflops": model_pp * P / step_s / 1e12,
            "model": "SURVEY.md §8(d): CM=T(6k-5)+n(D-2), CA=n(m-1)+Tk-nnz(J); DD 80/40, QD 800/200 flops per op",
            "exec_flops_per_point": exec_pp,
            "model_flops_per_point": model_pp,
        },
        "kernels_ms_per_step": {names[i]: kms[i] / steps for i in range(4) if kn[i]},
        "clocks": clocks,
        "e2e": {
            "value": aggregate_value(P, e2e_steps, e2e_s * 1e3),
            "unit": "evals/s",
            "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo,
            "api": "phc_eval_jacobian_batch_host (pinned host buffers; H2D, evaluation, D2H timed)",
        },
        # the profile records the block kernel; the power-table kernel of layout 0 (a
        # programmatic dependent launch) is counted from the plan's launches per call
        "gpu_launches": max(int(sum(kn)), launches_per_call(st, P) * steps),
        "outputs_finite": ok,
    }
    if parity:
        rec["parity"] = parity
    if label:
        rec["label"] = label
    return rec, h, X


def run_one_process(args):
    """N = 1 (or --gpus N > 1 without torchrun: the library's device-list call)."""
    import torch

    import paper_1109_0545_b200 as phc
    local = 0
    torch.cuda.set_device(local)
    ngpu = args.gpus
    devices = None
    if ngpu > 1:
        have = torch.cuda.device_count()
        if have < ngpu:
            raise SystemExit(f"--gpus {ngpu} but only {have} CUDA device(s) visible")
        devices = list(range(ngpu))
    peak_run = phc.phc_fp64_peak(local, 300.0)
    flush = not args.no_flush
    built = build_workload(args.workload, args.points, local)
    rec, h, X = batch_record(phc, args.workload, args.points, args.steps_eff, args.warmup, flush, local,
                             args.e2e_steps, peak_run, devices, built=built)
    out = {"metric": METRIC, "value": rec.pop("value"), "unit": "evals/s", "n_gpus": ngpu, "steps": args.steps_eff,
           "warmup": args.warmup, "ms_per_step": rec.pop("ms_per_step"), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA}
    out.update(rec)
    if ngpu == 1 and not args.no_nested and args.workload == "large_batch":
        # the large single point (the same system; point 0 of the batch), L2 flushed per call
        x0 = torch.from_numpy(X[0]).cuda(local)
        us, clk, nl, f0, j0 = measure_single(phc, h, x0, args.single_calls, local, flush=True)
        st = h.stats
        exec_pp = exec_flops_per_point(st, 1)
        med = statistics.median(us)
        tf = exec_pp / (med * 1e-6) / 1e12
        out["large_single"] = {
            "config": "BASELINE.json configs[4] large, single point (phc_eval_jacobian), point 0 of the batch",
            "us_median": med, "us_p10": us[len(us) // 10], "us_p90": us[(9 * len(us)) // 10],
            "calls": len(us), "evals_per_s": 1e6 / med, "l2": "flushed before every call (256 MiB write)",
            "exec_flops_per_point": exec_pp, "exec_tflops": tf,
            "frac": tf / nominal_fp64_tflops(), "frac_of_measured": tf / peak_run, "clocks": clk,
            "gpu_launches": nl,
            "parity": parity_vs_golden(f0, j0),
        }
        del x0
    if ngpu == 1 and not args.no_nested and args.workload != "batch":
        del h
        torch.cuda.empty_cache()
        rb, hb, _ = batch_record(phc, "batch", None, max(args.steps_eff, 10), max(args.warmup, 3), flush, local,
                                 args.e2e_steps, peak_run, label="BASELINE.json configs[3] batch, complex DD")
        out["batch_dd"] = rb
    if ngpu == 1 and not args.no_nested:
        # the three small single-point configs (BASELINE.json configs[0..2]): latency-bound
        # calls, reported as the median of single calls with the L2 flushed before each
        small = {}
        for name in ("tiny", "c2", "c3"):
            _, ss, Xs, hs = build_workload(name, None, local)
            xs = torch.from_numpy(Xs[0]).cuda(local)
            us, clk, nl, _, _ = measure_single(phc, hs, xs, args.single_calls, local, flush=True)
            st = hs.stats
            med = statistics.median(us)
            small[name] = {"us_median": med, "us_p10": us[len(us) // 10], "us_p90": us[(9 * len(us)) // 10],
                           "evals_per_s": 1e6 / med, "calls": len(us),
                           "path": latency_path_name(st) if latency_regime(st, 1) else "batch kernels",
                           "gpu_launches": nl, "clocks": clk}
            del hs, xs
        out["small_single"] = small
    if ngpu == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.workload)
    print(json.dumps(out), flush=True)


def run_multiprocess(args):
    """torchrun, one process per GPU: rank r evaluates its shard of ONE batch (strong scaling)
    and its kernels store F, J into rank 0's buffers (CUDA IPC mapping, fused gather)."""
    import torch
    import torch.distributed as dist

    import paper_1109_0545_b200 as phc
    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    local = local % max(ndev, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # NCCL needs one GPU per rank; ranks sharing a GPU (a test of the IPC path on a one-GPU
    # box) use gloo for the control plane (barriers, handle broadcast, timing reductions) --
    # the data path is the same IPC-mapped stores either way
    backend = "nccl" if ndev >= world else "gloo"
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    cdev = dev if backend == "nccl" else None
    flush = not args.no_flush
    # rank 0 draws the batch and broadcasts it (every rank evaluates part of the SAME batch;
    # the system itself is cheap to draw and identical on every rank)
    import numpy as np
    from synthetic import CONFIGS, config_system
    c = CONFIGS[args.workload]
    P = args.points or c["points"]
    if rank == 0:
        s, X = config_system(args.workload, seed=1, points=P)
    else:
        s, _ = config_system(args.workload, seed=1, points=1)
        X = np.empty((P, s.n_var, 2, s.limbs), dtype=np.float64)
    Xt = torch.from_numpy(X).to(dev) if backend == "nccl" else torch.from_numpy(X)
    dist.broadcast(Xt, src=0)
    X = Xt.cpu().numpy() if backend == "nccl" else Xt.numpy()
    del Xt
    h = phc.System(s, device=local)
    st = h.stats
    p0, p1 = shard_range(rank, world, P)
    Xd = torch.from_numpy(X).to(dev)  # inputs resident in HBM before the timed region
    F = J = None
    if rank == 0:
        F = torch.empty((P, s.n_eq, 2, s.limbs), dtype=torch.float64, device=dev)
        J = torch.empty((P, s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device=dev)
    # rank 0 exports its F and J; every other rank maps them
    gather = "fused NVLink stores into rank 0's IPC-mapped F/J"
    payload = None
    if rank == 0:
        try:
            payload = [phc.phc_ipc_get_handle(F.data_ptr()), phc.phc_ipc_get_handle(J.data_ptr())]
        except Exception as e:  # noqa: BLE001
            payload = ("error", str(e))
    payload = share_handles(rank, world, payload)
    fptr = jptr = None
    bases = []
    if rank == 0:
        fptr, jptr = F.data_ptr(), J.data_ptr()
    if isinstance(payload, tuple):
        gather = f"NCCL point-to-point copies to rank 0 (IPC refused: {payload[1][:120]})"
    elif rank != 0:
        try:
            for (hnd, off) in payload:
                base = phc.phc_ipc_open(hnd, local)
                bases.append(base)
            fptr, jptr = bases[0] + payload[0][1], bases[1] + payload[1][1]
        except Exception as e:  # noqa: BLE001
            gather = f"NCCL point-to-point copies to rank 0 (IPC open failed: {str(e)[:120]})"
    ok_flags = torch.tensor([1 if (fptr is not None or rank == 0) else 0], device=cdev)
    dist.all_reduce(ok_flags, op=dist.ReduceOp.MIN)
    use_ipc = bool(ok_flags.item()) and not gather.startswith("NCCL")
    if not use_ipc:
        if backend != "nccl":
            raise SystemExit(f"ranks share a GPU and IPC failed ({gather}); no NCCL fallback")
        gather = gather if gather.startswith("NCCL") else "NCCL point-to-point copies to rank 0"
        if rank != 0:
            F = torch.empty((P, s.n_eq, 2, s.limbs), dtype=torch.float64, device=dev)
            J = torch.empty((P, s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device=dev)
        fptr, jptr = F.data_ptr(), J.data_ptr()
    stream = torch.cuda.current_stream(dev)
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    def step():
        h.eval_batch_range(Xd, p0, p1, fptr, jptr, stream=stream)
        if not use_ipc:
            gather_to_rank0(rank, world, F, lambda r: shard_range(r, world, P))
            gather_to_rank0(rank, world, J, lambda r: shard_range(r, world, P))

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    phc.phc_profile_enable(h._h, True)
    phc.phc_profile_read(h._h, reset=True)
    steps = args.steps_eff
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(steps):
            if scrub is not None:
                scrub.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ms_local = sum(a.elapsed_time(b) for a, b in ev)
    kms, kn = phc.phc_profile_read(h._h, reset=True)
    phc.phc_profile_enable(h._h, False)
    ms = max_over_ranks(ms_local, world, cdev)
    kernel_ms = max_over_ranks(kms[3] / steps, world, cdev)
    launches = int(max_over_ranks(st["launches"] * steps, world, cdev)) * world
    clocks = clk.summary()
    # end to end: each rank copies its shard of X from pinned host memory, evaluates it into
    # rank 0's buffers, and rank 0 reads F and J back to pinned host memory
    Xh = torch.from_numpy(X[p0:p1]).pin_memory()
    if rank == 0:
        Fh = torch.empty(tuple(F.shape), dtype=torch.float64).pin_memory()
        Jh = torch.empty(tuple(J.shape), dtype=torch.float64).pin_memory()
    e2e_steps = args.e2e_steps
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        Xd[p0:p1].copy_(Xh, non_blocking=True)
        step()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            Fh.copy_(F, non_blocking=True)
            Jh.copy_(J, non_blocking=True)
            torch.cuda.synchronize()
        dist.barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world, cdev)
    ok = True
    verified = None
    if rank == 0:
        ok = bool(torch.isfinite(F).all().item()) and bool(torch.isfinite(J).all().item())
        if args.verify:
            Fv, Jv = h.eval_batch(Xd)
            torch.cuda.synchronize()
            verified = bool(torch.equal(Fv, F)) and bool(torch.equal(Jv, J))
            del Fv, Jv
        exec_pp = exec_flops_per_point(st, P)
        step_s = ms / steps * 1e-3
        fj_bytes = (F.numel() + J.numel()) * 8
        shard_pts = p1 - p0
        out = {
            "metric": METRIC, "value": aggregate_value(P, steps, ms), "unit": "evals/s", "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": dict(config_dict(args.workload, c, P, flush, f"points sharded over {world} processes / GPUs"),
                           gather=gather, control_plane=backend,
                           gpus_visible=ndev),
            "roofline": roofline(exec_pp, shard_pts, kernel_ms, None, args.workload,
                                 f"block_kernel<{s.limbs},{st['K']},{st['layout']},0>"),
            "multi_gpu": {
                "step_ms_max_over_ranks": ms / steps,
                "kernel_ms_max_over_ranks": kernel_ms,
                "gather_bytes_per_step": fj_bytes * (world - 1) // world,
                "home_ingress_gbs": fj_bytes * (world - 1) / world / step_s / 1e9,
                "home_ingress_reference_gbs": 770.0,
                "shard_points": [shard_range(r, world, P) for r in range(world)],
            },
            "fp64": {"step_exec_tflops": exec_pp * P / step_s / 1e12,
                     "step_exec_frac_of_n_gpus_nominal": exec_pp * P / step_s / 1e12 / (world * nominal_fp64_tflops())},
            "clocks": clocks,
            "e2e": {"value": aggregate_value(P, e2e_steps, e2e_s * 1e3), "unit": "evals/s",
                    "h2d_bytes_per_step": X.nbytes, "d2h_bytes_per_step": fj_bytes,
                    "api": "per rank: H2D of its shard of X, phc_eval_jacobian_batch_range into rank 0's F/J; "
                           "rank 0: D2H of F and J (pinned)"},
            "gpu_launches": launches,
            "outputs_finite": ok,
        }
        if verified is not None:
            out["verified_bitwise_vs_one_process"] = verified
        print(json.dumps(out), flush=True)
    dist.barrier()
    for b in bases:
        phc.phc_ipc_close(b, local)
    dist.destroy_process_group()


def main(argv=None):
    args = parse(argv)
    args.steps_eff = args.steps if args.steps is not None else 10
    if args.impl == "reference":
        run_reference(args)
        return
    _, world, _ = dist_env()
    if world > 1:
        run_multiprocess(args)
    else:
        run_one_process(args)


if __name__ == "__main__":
    main()
