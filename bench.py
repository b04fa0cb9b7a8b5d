#!/usr/bin/env python
"""Benchmark of the CPA singular-value shrinkage hot path on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun
for N > 1) prints ONE JSON line on rank 0.  A "step" is one full pass of the
hot path -- one ``cpa_svt_apply`` call: Gram, Lambda_max power iteration,
coefficients, recurrence init and the K-2 fused recurrence steps -- over one
synthetic input resident in HBM.  The default workload is BASELINE.json
configs[1] (``c2``: 1024 x 1024 fp64, soft tau = 0.05 sigma_max_hat, K = 30,
T = 300); at N > 1 every rank runs its own independent problem (replicas,
weak scaling, no data-path collective: DESIGN.md §Multi-GPU).

Metric (BASELINE.json): GFLOP/s of algorithmic work, F = s(s+1)L (Gram) +
(K-1) 2 s^2 L (recurrence products), s = min(m,n), L = max(m,n).

``--impl reference`` times the CPU oracle (oracle/, fp64 numpy) on the same
config on this host's cores; it is the only other place bench.py executes the
oracle besides the ``cpu_baseline`` leg.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402  (seeded generators only; no arithmetic of the method)


def dense_flops(m, n, K, T):
    s, L = min(m, n), max(m, n)
    return {"gram": s * (s + 1) * L, "recurrence": (K - 1) * 2 * s * s * L,
            "power": T * (2 * s * s + 3 * s), "epilogue": (K - 1) * 5 * s * L,
            "step_gemm": 2 * s * s * L}


def dense_executed_flops(m, n, K, form):
    """Algorithmic flops of the form that ran (what the kernels must do)."""
    s, L = min(m, n), max(m, n)
    gram = s * (s + 1) * L
    if form == 1:
        return gram + (K - 1) * 2 * s * s * L
    if form == 2:
        return gram + max(K - 2, 0) * s * s * (s + 1) + 2 * s * s * L
    return gram + max(K - 2, 0) * 2 * s ** 3 + 2 * s * s * L


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


class Clocks:
    """nvidia-smi sampling during the timed region (recipe in B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, r[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank number over the torch.distributed world (identity when not initialised)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def oracle_step(cfg, X):
    """One oracle pass over the workload (cpu_baseline / --impl reference legs only)."""
    import oracle as O
    return O.cpa_shrink(X, O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, X, F, budget_s=10.0):
    t0 = time.perf_counter()
    runs = 0
    while True:
        oracle_step(cfg, X)
        runs += 1
        el = time.perf_counter() - t0
        if el >= budget_s or runs >= 50:
            break
    per = el / runs
    return {"value": F / per / 1e9, "unit": "GFLOP/s", "cores": blas_threads(), "kind": "oracle",
            "sample": f"{runs} full oracle run(s) of {cfg['name']} (numpy fp64, Alg. 1 literal form), "
                      f"{per:.3f} s each", "ms_per_step": per * 1e3}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    X = cfg["gen"](0)
    F = cfg["F"]
    for _ in range(args.warmup):
        oracle_step(cfg, X)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(cfg, X)
    t = (time.perf_counter() - t0) / args.steps
    v = F / t / 1e9
    line = {"impl": "reference", "metric": cfg["metric"], "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": cfg["config"],
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": blas_threads(), "kind": "oracle",
                             "sample": f"{args.steps} full oracle runs of {cfg['name']} on host cores"},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def make_cfg(name):
    c = dict(W.CONFIGS[name])
    c["name"] = name
    if name == "c2":
        c["gen"] = lambda seed: W.gen_c2(seed)
    elif name == "c1":
        c["gen"] = lambda seed: W.gen_c1(seed)
    else:
        raise SystemExit(f"bench.py: config {name} is a parity case, not a bench line (DESIGN.md §Measurement)")
    fl = dense_flops(c["m"], c["n"], c["K"], c["T"])
    c["flops"] = fl
    c["F"] = fl["gram"] + fl["recurrence"]
    c["metric"] = "CPA shrinkage GFLOP/s & % of FP64/HBM roofline; ms per SVT at 1/2/4/8 GPUs"
    c["config"] = {"workload": f"{name}: {c['m']}x{c['n']} fp64 (BASELINE configs[1]) rank-20 + 0.1 noise, "
                               f"soft tau={c['kernel']['tau']} sigma_max_hat, K={c['K']}, T={c['T']} power steps",
                   "m": c["m"], "n": c["n"], "K": c["K"], "T": c["T"], "side": "left" if c["m"] <= c["n"] else "right",
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "flops_per_step": c["F"],
                   "flop_count": "value = F / time with F = s(s+1)L + (K-1) 2 s^2 L, the Gram plus the apply-to-X "
                                 "recurrence (the north star's formulation), fixed per workload; the symmetric "
                                 "s x s form that runs does fewer flops (algorithmic_gflop_executed), so value is "
                                 "an effective rate -- ms_per_step is the time",
                   "parallelism": "replicas (independent problem per rank)"}
    c["dtype"] = "f64"
    return c


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import numpy as np

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1705_07112_b200 as P

    X = cfg["gen"](rank)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    Yd = torch.empty_like(Xd)
    h = P.Handle(local)
    kern, K, T = cfg["kernel"], cfg["K"], cfg["T"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        h.apply(Xd, kern, K, T=T, Y=Yd)
    _, info0 = h.apply(Xd, kern, K, T=T, Y=Yd, info=True)
    form = info0["form"]
    torch.cuda.synchronize()
    # ---------------- timed region: device-resident inputs ----------------
    clocks = Clocks(local)
    launches0 = h.launches
    h.profile(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)                 # evict X, G, W from L2 (untimed)
        ev[i][0].record(stream)
        h.apply(Xd, kern, K, T=T, Y=Yd)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    prof = h.profile_read()
    h.profile(False)
    gpu_launches = h.launches - launches0
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps, torch.device("cuda", local))
    value = world * cfg["F"] / (ms * 1e-3) / 1e9

    # ---------------- e2e: C-ABI call with HOST buffers ----------------
    Xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    for _ in range(max(3, args.warmup)):
        h.apply_host(Xh, Yh, kern, K, T=T)
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ee[i][0].record(stream)
        h.apply_host(Xh, Yh, kern, K, T=T)
        ee[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max_over_ranks(sum(a.elapsed_time(b) for a, b in ee) / args.steps, torch.device("cuda", local))
    nbytes = X.size * 8

    # ---------------- roofline of the dominant kernel (fused step) ----------------
    # form 2 (auto for K > 2): k_cheb_sym_tma (k_cheb_sym for odd s) -- all K-2 steps of the symmetric s x s form in ONE
    # persistent launch, algorithmic work s^2 (s+1) flops per step (lower-triangle elements,
    # 2s flops each).  form 1: k_cheb_flow -- init + K-2 steps of apply-to-X, 2 s^2 L per product.
    s_, L_ = min(cfg["m"], cfg["n"]), max(cfg["m"], cfg["n"])
    step_ms, step_n = prof["step"]
    avg = step_ms / max(step_n, 1)
    if form == 4:   # (c1-sized problems: the whole SVT in one thread block)
        kname = "k_small_f64 (all of Alg. 1 in one thread block, shared memory, DFMA)"
        flops_per_launch = dense_executed_flops(cfg["m"], cfg["n"], K, 3) * args.steps / max(step_n, 1)
    elif form == 2:
        kname = ("k_cheb_sym_tma (symmetric s x s recurrence: K-2 fused steps in one persistent launch, "
                 "TMA-fed DMMA)" if s_ % 2 == 0 else
                 "k_cheb_sym (symmetric s x s recurrence: K-2 fused steps in one persistent launch, cp.async-fed DMMA)")
        flops_per_launch = (K - 2) * s_ * s_ * (s_ + 1) * args.steps / max(step_n, 1)
    else:
        products = (K - 1) if prof["init"][1] == 0 else (K - 2)
        kname = ("k_cheb_flow (fused recurrence: init + K-2 steps, DMMA)" if prof["init"][1] == 0
                 else "k_dmma_gemm<EPI_STEP> (fused recurrence step)")
        flops_per_launch = cfg["flops"]["step_gemm"] * products * args.steps / max(step_n, 1)
    peaks = load_json(os.path.join(ROOT, "profiles", "r01_peaks.json")) or {}
    peak = peaks.get("fp64_dmma_tflops")
    achieved = flops_per_launch / (avg * 1e-3) / 1e12 if avg > 0 else None
    traffic = None
    tr = load_json(os.path.join(ROOT, "profiles", "traffic.json"))
    if tr and tr.get("config") == cfg["name"] and tr.get("form", 1) == form:
        traffic = tr.get("dram_bytes_per_launch")
    phase_share = {k: round(v[0] / max(1e-9, sum(x[0] for x in prof.values())), 4) for k, v in prof.items() if v[1]}
    executed = dense_executed_flops(cfg["m"], cfg["n"], K, form)
    line = {
        "metric": cfg["metric"], "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (workloads.gen_c2, seed = rank)",
        "config": cfg["config"],
        "roofline": {"bound": "tensor", "kernel": kname,
                     "flops_per_launch": flops_per_launch,
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
                     "peak_source": "measured FP64 DMMA loop, profiles/r01_peaks.json (MEASURED_PEAKS.json has no fp64)",
                     "launch_ms": avg, "phase_share": phase_share,
                     "phase_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]}},
        "form": {1: "apply-to-X", 2: "Alg. 1 s x s form, symmetric tiles", 3: "s x s form, full tiles",
                 4: "Alg. 1 s x s form in one thread block"}[form],
        "algorithmic_gflop_executed": executed / 1e9,
        "gflops_executed": world * executed / (ms * 1e-3) / 1e9,
        "e2e": {"value": world * cfg["F"] / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes},
        "gpu_launches": gpu_launches, "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, X, cfg["F"], args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    cfg = make_cfg(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
