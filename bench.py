#!/usr/bin/env python
"""Benchmark: complex DD/QD polynomial system + Jacobian evaluations per second on B200.

One "step" = one pass of the whole hot path (power table, Speelpenning monomial stage,
coefficient product, reductions: SURVEY.md §8(a) rows a1-a8) over one batch of
synthetic points resident in HBM.  Default workload: BASELINE.json configs[3]
("batch": n=32, m=32, k=16, D=4, complex DD, 65,536 unit-circle points per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): every rank evaluates its own 65,536-point
batch (weak scaling, no data-path collective); the timed region is bracketed by a
barrier + synchronize and the max over ranks is taken.  `--impl reference` times the
CPU oracle (oracle/, exact arithmetic) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# SURVEY.md §8(d) frozen model (paper-faithful op counts, standard DD costs)
MODEL_FLOPS = {2: dict(cm=80, ca=40), 4: dict(cm=800, ca=200)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="batch")
    ap.add_argument("--points", type=int, default=None, help="override points per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def traffic_per_launch(workload, points):
    """roofline.traffic: DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[workload]
        return t["bytes_per_point"] * points
    except (OSError, KeyError, ValueError):
        return None


def rank_seed(rank):
    """Weak scaling: every rank evaluates its own batch of the workload, drawn with seed 1 + rank."""
    return 1 + rank


def max_over_ranks(value, world, device=None):
    """The timing rule: the slowest rank defines the step time (all_reduce MAX)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(world, points_per_rank, steps, ms_max):
    """Whole-job throughput: the units all ranks processed / the max-over-ranks time."""
    return world * points_per_rank * steps / (ms_max * 1e-3)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def config_dict(name, c, P, flush):
    return {
        "workload": name,
        "n": c["n"], "m": c["m"], "k": c["k"], "D": c["D"],
        "precision": "complex DD" if c["limbs"] == 2 else "complex QD",
        "points_per_gpu": P,
        "l2": "flushed between timed steps (256 MiB write)" if flush else "outputs > L2",
    }


def model_counts(s, st):
    """CM = T(6k-5) + n(D-2), CA = n(m-1) + T k - nnz(J) (paper-faithful)."""
    import numpy as np
    k = np.diff(s.term_ptr)
    T = len(k)
    cm = int(np.sum(np.where(k >= 1, 6 * k - 5, 0))) + s.n_var * max(0, int(st["D"]) - 2)
    m = np.diff(s.poly_ptr)
    ca = int(np.sum(np.maximum(m - 1, 0))) + int(k.sum()) - int(st["nnz_J"])
    return cm, ca


def latency_regime(st, points):
    """True when a call with `points` points takes the latency path (phc.h: n_points * n_terms
    <= the bound in phc_system_stats out[13])."""
    return st["latency_bound"] > 0 and points * st["n_terms"] <= st["latency_bound"]


def exec_flops_per_point(s, st, points=None):
    """Executed FP64 flops per point of the kernels' useful work, as counted by the library
    (phc_system_stats out[8], or out[12] for the latency path; per-op costs from arith.cuh,
    checked against ncu)."""
    if points is not None and latency_regime(st, points):
        return int(st["latency_exec_flops_per_point"])
    return int(st["exec_flops_per_point"])


class ClockSampler:
    """nvidia-smi clocks during the timed region (B200_PROFILING.md clocks line)."""

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
                                       "--format=csv,noheader,nounits", "-lms", "200"],
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


def run_reference(args):
    """--impl reference: the CPU oracle (exact arithmetic, all host cores over rows), as it stands."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import evaluate_system
    from synthetic import CONFIGS, config_system
    c = CONFIGS[args.workload]
    s, X = config_system(args.workload, seed=1, points=max(args.steps + args.warmup, 1))
    arith = "exact" if c["limbs"] == 2 or c["n"] <= 64 else "mp"
    cores = host_cores()
    for w in range(args.warmup):
        evaluate_system(s, X[w % X.shape[0]], arith)
    t = 0.0
    for i in range(args.steps):
        t0 = time.perf_counter()
        evaluate_system(s, X[(args.warmup + i) % X.shape[0]], arith)
        t += time.perf_counter() - t0
    v = args.steps / t
    out = {
        "metric": "complex DD/QD system+Jacobian evals/sec", "value": v, "unit": "evals/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded unit-circle systems and points, BASELINE.json recipe)",
        "config": dict(config_dict(args.workload, c, c["points"], False),
                       sample=f"each step = 1 point of the workload (oracle, {arith} arithmetic)"),
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "kind": "oracle",
                         "sample": f"1 point per step, {args.steps} steps, {arith} arithmetic, rows over {cores} processes"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


def cpu_baseline(workload, budget_s=15.0):
    """The oracle timed on this host's cores on a bounded sample (rank 0, N=1 only)."""
    from oracle import evaluate_rows
    from synthetic import CONFIGS, config_system
    c = CONFIGS[workload]
    s, X = config_system(workload, seed=1, points=min(c["points"], 64))
    cores = host_cores()
    arith = "exact" if c["limbs"] == 2 or c["n"] <= 64 else "mp"
    if c["n"] <= 64:
        t0 = time.perf_counter()
        npts = 0
        while time.perf_counter() - t0 < budget_s and npts < X.shape[0]:
            evaluate_rows(s, X[npts], None, arith)
            npts += 1
        dt = time.perf_counter() - t0
        return {"value": npts / dt, "unit": "evals/s", "cores": cores, "kind": "oracle",
                "sample": f"{npts} full points of '{workload}' ({arith} arithmetic, rows over {cores} processes) in {dt:.1f} s"}
    rows = list(range(min(cores, s.n_eq)))
    t0 = time.perf_counter()
    evaluate_rows(s, X[0], rows, arith)
    dt = time.perf_counter() - t0
    per_point = dt * s.n_eq / len(rows)
    return {"value": 1.0 / per_point, "unit": "evals/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(rows)} of {s.n_eq} rows of one point ({arith}, 512 bits) in {dt:.1f} s, extrapolated to a full point"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1109_0545_b200 as phc
    from synthetic import CONFIGS, config_system

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = CONFIGS[args.workload]
    P = args.points or c["points"]
    s, X = config_system(args.workload, seed=rank_seed(rank), points=P)
    h = phc.System(s, device=local)
    st = h.stats
    Xd = torch.from_numpy(X).to(dev)
    F = torch.empty((P, s.n_eq, 2, s.limbs), dtype=torch.float64, device=dev)
    J = torch.empty((P, s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = not args.no_flush
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    peak_now = phc.phc_fp64_peak(local, 300.0)

    for _ in range(max(args.warmup, 0)):
        h.eval_batch(Xd, F, J, stream=stream)
    torch.cuda.synchronize()
    phc.phc_profile_enable(h._h, True)
    phc.phc_profile_read(h._h, reset=True)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush:
                scrub.fill_(i & 0xFF)
            ev[i][0].record(stream)
            h.eval_batch(Xd, F, J, stream=stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    kms, kn = phc.phc_profile_read(h._h, reset=True)
    phc.phc_profile_enable(h._h, False)
    ms = max_over_ranks(ms, world, dev)
    clocks = clk.summary()

    # end to end through the C-ABI host call: pinned host buffers, H2D + eval + D2H every step
    Xh = torch.from_numpy(X).pin_memory()
    Fh = torch.empty((P, s.n_eq, 2, s.limbs), dtype=torch.float64).pin_memory()
    Jh = torch.empty((P, s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64).pin_memory()
    h.eval_batch_host(Xh.numpy(), Fh.numpy(), Jh.numpy())  # warm-up (allocates staging)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        h.eval_batch_host(Xh.numpy(), Fh.numpy(), Jh.numpy())
    e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s, world, dev)
    ok = bool(torch.isfinite(F).all().item()) and bool(torch.isfinite(J).all().item())

    if rank == 0:
        cm_model, ca_model = model_counts(s, st)
        mf = MODEL_FLOPS[s.limbs]
        model_flops_pp = cm_model * mf["cm"] + ca_model * mf["ca"]
        exec_pp = exec_flops_per_point(s, st, P)
        value = aggregate_value(world, P, args.steps, ms)
        peak = peak_now
        # dominant kernel (largest summed time among the classes)
        names = ["power_table", "term", "reduce", "poly_scan" if latency_regime(st, P) else "fused_block"]
        dom = max(range(4), key=lambda i: kms[i])
        dom_ms = kms[dom] / max(kn[dom], 1)
        # the dominant kernel does (nearly) all of the step's FP64 work: the fused block
        # kernel all of it, the generic term kernel all but the power table and sums
        dom_flops = exec_pp * P / max(kn[dom] / args.steps, 1) if dom in (1, 3) else 0.0
        achieved = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else 0.0
        step_exec_tflops = exec_pp * P / (ms / args.steps * 1e-3) / 1e12
        step_model_tflops = model_flops_pp * P / (ms / args.steps * 1e-3) / 1e12
        launches = int(sum(kn))
        bytes_in = X.nbytes
        bytes_out = Fh.numel() * 8 + Jh.numel() * 8
        out = {
            "metric": "complex DD/QD system+Jacobian evals/sec",
            "value": value,
            "unit": "evals/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded unit-circle systems and points, BASELINE.json recipe)",
            "config": dict(config_dict(args.workload, c, P, flush), parallelism=f"dp{world} (points)",
                           path="latency (one warp per term)" if latency_regime(st, P) else "batch kernels"),
            "roofline": {
                "bound": "alu",
                "kernel": names[dom],
                "achieved": achieved,
                "peak": peak,
                "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None,
                "traffic": traffic_per_launch(args.workload, P / max(kn[dom] / args.steps, 1)),
                "traffic_source": "profiles/traffic.json (ncu --set full, dram read+write per point x points per launch)",
                "flops": "executed FP64 flops (DADD=DMUL=1, DFMA=2) per launch from the kernel op counts",
                "peak_source": "phc_fp64_peak: DFMA chains measured in this run (profiles/fp64_peak_r01.jsonl: 34.2 sustained)",
            },
            "fp64": {
                "step_exec_tflops": step_exec_tflops,
                "step_exec_frac": step_exec_tflops / peak,
                "step_model_tflops": step_model_tflops,
                "step_model_frac": step_model_tflops / peak,
                "model": "SURVEY.md §8(d): CM=T(6k-5)+n(D-2), CA=n(m-1)+Tk-nnz(J); DD 80/40, QD 800/200 flops",
                "exec_flops_per_point": exec_pp,
                "model_flops_per_point": model_flops_pp,
            },
            "kernels_ms_per_step": {names[i]: kms[i] / args.steps for i in range(4) if kn[i]},
            "clocks": clocks,
            "e2e": {
                "value": aggregate_value(world, P, args.e2e_steps, e2e_s * 1e3),
                "unit": "evals/s",
                "h2d_bytes_per_step": bytes_in,
                "d2h_bytes_per_step": bytes_out,
                "api": "phc_eval_jacobian_batch_host (pinned host buffers)",
            },
            "gpu_launches": launches,
            "outputs_finite": ok,
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args.workload)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
