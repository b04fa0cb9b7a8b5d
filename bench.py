#!/usr/bin/env python
"""Benchmark of the CPA singular-value shrinkage hot path on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun
for N > 1) prints ONE JSON line on rank 0.  A "step" is one full pass of the
hot path -- one ``cpa_svt_apply`` call: Gram, Lambda_max power iteration,
coefficients, the K-2 fused recurrence steps and line 12 -- over one synthetic
input resident in HBM.

Workloads: at N = 1 the default is BASELINE.json configs[1] (``c2``: 1024 x 1024
fp64, soft tau = 0.05 sigma_max_hat, K = 30, T = 300), the config the metric is
quoted on that fits one GPU.  At N > 1 the default is configs[4] (``c5``: 16384 x
65536, column-sharded over the N ranks through the library's NCCL path -- the
north star's multi-GPU split, strong scaling); ``--config c5`` runs that at N = 1
too (one-rank communicator), so ``--config c5 --gpus 1/2/4/8`` is the "ms per SVT
at 1/2/4/8 GPUs" series.  ``--math 3xtf32`` gives the fp32 tensor-core variant.

Metric (BASELINE.json): GFLOP/s of the algorithmic work of the form that ran,
each flop counted once for the whole job, and ms per SVT.

``--impl reference`` times the CPU oracle (oracle/, fp64 numpy) on the same
config (c5: the same recipe at a reduced shape) on this host's cores; it is the
only other place bench.py executes the oracle besides the ``cpu_baseline`` leg.
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


def cpu_baseline(cfg, budget_s=10.0):
    X = cfg["oracle_X"]()
    F = cfg["oracle_F"]
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
            "sample": f"{runs} x {cfg['oracle_sample']}, {per:.3f} s each; value = the same algorithmic "
                      f"flop count as the GPU line / oracle time", "ms_per_step": per * 1e3}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    X = cfg["oracle_X"]()
    F = cfg["oracle_F"]
    for _ in range(args.warmup):
        oracle_step(cfg, X)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(cfg, X)
    t = (time.perf_counter() - t0) / args.steps
    v = F / t / 1e9
    line = {"impl": "reference", "metric": cfg["metric"], "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": cfg["config"],
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": blas_threads(), "kind": "oracle",
                             "sample": cfg["oracle_sample"]},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


METRIC = "CPA shrinkage GFLOP/s & % of FP64/HBM roofline; ms per SVT at 1/2/4/8 GPUs"


def make_cfg(name, world, math):
    if name not in ("c1", "c2", "c5"):
        raise SystemExit(f"bench.py: config {name} is a parity case, not a bench line (DESIGN.md §Measurement)")
    c = dict(W.CONFIGS[name])
    c["name"] = name
    c["math"] = math
    m, n, K, T = c["m"], c["n"], c["K"], c["T"]
    c["metric"] = METRIC
    c["dtype"] = "f64" if math == "native" else "f32"
    sharded = name == "c5"
    c["sharded"] = sharded
    c["scaling"] = "strong" if sharded else "weak"
    which = {"c1": "configs[0]", "c2": "configs[1]", "c5": "configs[4]"}[name]
    c["config"] = {"workload": f"{name} ({which}): {m}x{n} {c['dtype']}"
                               + (f" [{math}]" if math != "native" else "")
                               + f", soft tau={c['kernel']['tau']}{' sigma_max_hat' if c['kernel']['tau_relative'] else ''}"
                               f", K={K}, T={T} power steps",
                   "m": m, "n": n, "K": K, "T": T, "side": "left" if m <= n else "right",
                   "l2": "flushed between timed steps (256 MiB write, untimed)" if not sharded else
                         "inputs larger than L2 (X block >= 1 GiB per rank)",
                   "flop_count": "value = algorithmic flops of the form that ran, each counted once for the whole "
                                 "job (Gram s(s+1)L + (K-2) s^2 (s+1) symmetric s x s steps + 2 s^2 L line 12), "
                                 "divided by the max-over-ranks time; never above the hardware peak",
                   "parallelism": (f"column shards over {world} rank(s): NCCL all-reduce of the s x s Gram, "
                                   "series broadcast, each rank applies H_hat to its block" if sharded
                                   else "replicas (independent problem per rank)")}
    # oracle legs (cpu_baseline / --impl reference): the full problem where it finishes in seconds,
    # else the same recipe at a reduced shape
    if name == "c5":
        om, on = 1024, 4096
        c["oracle_X"] = lambda: W.gen_c5(m=om, n=on)
        c["oracle_sample"] = f"full oracle SVTs of the c5 recipe at {om}x{on} (numpy fp64, Alg. 1 literal form)"
    else:
        om, on = m, n
        c["oracle_X"] = (lambda: W.gen_c1()) if name == "c1" else (lambda: W.gen_c2())
        c["oracle_sample"] = f"full oracle SVTs of {name} (numpy fp64, Alg. 1 literal form)"
    c["oracle_F"] = dense_executed_flops(om, on, K, 2)
    return c


def gen_block_device(cfg, rank, world, dtype):
    """This rank's input on the device.  c1/c2: the numpy recipe (seed = rank, replicas).
    c5: column block [b, e) of a c5-recipe matrix drawn on the device (torch Philox; the
    factor A shared by all ranks, B and the noise per rank) -- statistically the c5 recipe,
    not its numpy stream (parity tests use the numpy stream)."""
    import numpy as np
    import torch
    if not cfg["sharded"]:
        X = cfg["oracle_X"]() if rank == 0 else (W.gen_c1(rank) if cfg["name"] == "c1" else W.gen_c2(rank))
        return torch.from_numpy(np.ascontiguousarray(X)).cuda().to(dtype)
    from paper_1705_07112_b200 import dist as D
    m, n = cfg["m"], cfg["n"]
    b, e = D.shard_range(n, world, rank)
    sd = (50 ** -0.5) ** 0.5
    g = torch.Generator(device="cuda").manual_seed(12345)
    A = torch.randn(m, 50, dtype=torch.float64, device="cuda", generator=g) * sd
    g.manual_seed(1000 + rank)
    X = torch.empty((m, e - b), dtype=dtype, device="cuda")
    step = 4096
    for c0 in range(0, e - b, step):
        c1 = min(e - b, c0 + step)
        B = torch.randn(c1 - c0, 50, dtype=torch.float64, device="cuda", generator=g) * sd
        E = torch.randn(m, c1 - c0, dtype=torch.float64, device="cuda", generator=g)
        X[:, c0:c1] = (A @ B.T + 0.01 * E).to(dtype)
    return X


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1705_07112_b200 as P
    from paper_1705_07112_b200 import dist as D

    dtype = torch.float64 if cfg["math"] == "native" else torch.float32
    esize = 8 if dtype == torch.float64 else 4
    Xd = gen_block_device(cfg, rank, world, dtype)
    Yd = torch.empty_like(Xd)
    m_g, n_g = cfg["m"], cfg["n"]
    if cfg["sharded"]:
        h = D.make_handle(local)            # library-owned NCCL communicator, any world size
        call = lambda X, Y, **kw: D.apply_sharded(h, X, m_g, n_g, kern, K, T=T, Y=Y, math=cfg["math"], **kw)
    else:
        h = P.Handle(local)
        call = lambda X, Y, **kw: h.apply(X, kern, K, T=T, Y=Y, math=cfg["math"], **kw)
    kern, K, T = cfg["kernel"], cfg["K"], cfg["T"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    warm = max(3, args.warmup)
    for _ in range(warm):
        call(Xd, Yd)
    _, info0 = call(Xd, Yd, info=True)
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
        if not cfg["sharded"]:
            flush.fill_(i & 0xFF)             # evict X, G, W from L2 (untimed)
        ev[i][0].record(stream)
        call(Xd, Yd)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    prof = h.profile_read()
    h.profile(False)
    gpu_launches = (h.launches - launches0) // args.steps
    dev = torch.device("cuda", local)
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps, dev)
    s_, L_ = min(m_g, n_g), max(m_g, n_g)
    executed = dense_executed_flops(m_g, n_g, K, form)       # one SVT of the whole problem, counted once
    job_flops = executed * (1 if cfg["sharded"] else world)
    value = job_flops / (ms * 1e-3) / 1e9

    # ---------------- e2e: through the public API with HOST buffers ----------------
    Xh = Xd.cpu().pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    if cfg["sharded"]:
        Xe, Ye = torch.empty_like(Xd), torch.empty_like(Yd)

        def e2e_call():
            Xe.copy_(Xh, non_blocking=True)           # H2D of this step's input
            call(Xe, Ye)
            Yh.copy_(Ye, non_blocking=True)           # D2H of the step's result
        e2e_api = "paper_1705_07112_b200.dist.apply_sharded with pinned-host H2D / D2H copies on the stream"
    else:
        def e2e_call():
            h.apply_host(Xh, Yh, kern, K, T=T, math=cfg["math"])
        e2e_api = "cpa_svt_apply_host (C ABI, pinned host X and Y)"
    for _ in range(warm):
        e2e_call()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        if not cfg["sharded"]:
            flush.fill_(i & 0xFF)
        ee[i][0].record(stream)
        e2e_call()
        ee[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max_over_ranks(sum(a.elapsed_time(b) for a, b in ee) / args.steps, dev)
    nbytes = Xd.numel() * esize

    # ---------------- roofline of the dominant kernel ----------------
    step_ms, step_n = prof["step"]
    avg = step_ms / max(step_n, 1)
    if form == 4:   # (c1-sized problems: the whole SVT in one thread block)
        kname = "k_small_f64 (all of Alg. 1 in one thread block, shared memory, DMMA)"
        s1, L1 = min(m_g, n_g), max(m_g, n_g)
        # (K - 3 products with the two chains and Psi_2 from the squaring, readings R28/R29)
        nprod = info0.get("rec_products") or (K - 2)
        rec_flops = s1 * (s1 + 1) * L1 + nprod * 2 * s1 ** 3 + 2 * s1 * s1 * L1
    elif form == 2:
        kname = ("k_cheb_sym_tma (symmetric s x s recurrence, TMA-fed DMMA)" if cfg["math"] == "native"
                 else "k_tc_gemm (symmetric s x s recurrence step, tcgen05 " + cfg["math"] + ")")
        # (K - 3 products when Psi_2 came from the power iteration's squaring, reading R29)
        nprod = info0.get("rec_products") or (K - 2)
        rec_flops = nprod * s_ * s_ * (s_ + 1) * (3 if cfg["math"] == "3xtf32" else 1)
        if info0.get("line12_in_recurrence"):   # line 12 (2 s^2 L) ran inside the same launch
            rec_flops += 2 * s_ * s_ * L_
    else:
        kname = "k_cheb_flow (fused apply-to-X recurrence, DMMA)"
        rec_flops = (K - 1) * 2 * s_ * s_ * (n_g // world if cfg["sharded"] else L_)
    rec_flops *= float(info0.get("rec_share", 1.0))
    flops_per_launch = rec_flops * args.steps / max(step_n, 1)
    peaks = load_json(os.path.join(ROOT, "profiles", "r01_peaks.json")) or {}
    mp_ = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    if cfg["math"] == "native":
        peak = peaks.get("fp64_dmma_tflops")
        peak_src = "measured FP64 DMMA loop, profiles/r01_peaks.json (MEASURED_PEAKS.json has no fp64)"
    else:
        # the recurrence runs for seconds under the power cap: the SUSTAINED figure applies
        peak = (mp_.get("bf16_tflops_sustained") or mp_.get("bf16_tflops") or 0) / 2 or None
        peak_src = ("MEASURED_PEAKS.json bf16 sustained / 2 (nominal TF32:BF16 ratio; the kernel runs inside a "
                    "seconds-long step); 3xTF32 counts its 3 MMAs")
    achieved = flops_per_launch / (avg * 1e-3) / 1e12 if avg > 0 else None
    traffic = None
    tr = load_json(os.path.join(ROOT, "profiles", "traffic.json"))
    if tr and tr.get("config") == cfg["name"] and tr.get("form", 1) == form:
        traffic = tr.get("dram_bytes_per_launch")
    phase_share = {k: round(v[0] / max(1e-9, sum(x[0] for x in prof.values())), 4) for k, v in prof.items() if v[1]}
    line = {
        "metric": cfg["metric"], "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": ms, "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": cfg["dtype"],
        "data": ("synthetic (workloads.gen_" + cfg["name"] + ", seed = rank)") if not cfg["sharded"] else
                "synthetic (c5 recipe drawn on the device per column block)",
        "config": cfg["config"],
        "ms_per_svt": ms,
        "roofline": {"bound": "tensor", "kernel": kname,
                     "flops_per_launch": flops_per_launch,
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
                     "peak_source": peak_src, "launch_ms": avg, "phase_share": phase_share,
                     "phase_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]}},
        "form": {1: "apply-to-X", 2: "Alg. 1 s x s form, symmetric tiles", 3: "s x s form, full tiles",
                 4: "Alg. 1 s x s form in one thread block"}[form],
        "algorithmic_gflop_per_svt": executed / 1e9,
        "e2e": {"value": job_flops / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "api": e2e_api},
        "gpu_launches": gpu_launches, "clocks": clk,
    }
    if cfg["math"] == "native" and peak:
        assert value <= world * peak * 1e3 * 1.02, "executed-flop rate above the hardware peak"
    if cfg["sharded"]:
        nr, rk = h.comm_info()             # the library's own communicator, as NCCL reports it
        line["nccl"] = {"comm_nranks": nr, "comm_rank": rk, "comm_nranks_ok": nr == world and rk == rank}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_budget)
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return line if rank == 0 else None


class _StdoutToStderr:
    """Route fd 1 to stderr while the benchmark runs (NCCL and CUDA libraries print to the C-level
    stdout, e.g. "NCCL version ..."), so the only thing on stdout is the JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def emit(line: dict):
    """The one JSON line on the real stdout."""
    sys.stdout.flush()
    os.write(1, (json.dumps(line) + "\n").encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c2 (default at N = 1), c5 (default at N > 1), c1")
    ap.add_argument("--math", default="native", choices=["native", "3xtf32", "tf32"],
                    help="native = fp64 DMMA; 3xtf32 / tf32 = the fp32 tensor-core variant")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    name = args.config or ("c2" if world == 1 and args.gpus <= 1 else "c5")
    cfg = make_cfg(name, world, args.math)
    with _StdoutToStderr():
        if args.impl == "reference":
            line = run_reference(args, cfg)
        else:
            line = run_ours(args, cfg)
    if line is not None:
        emit(line)
    return 0


if __name__ == "__main__":
    sys.exit(main())
