"""Projected c5 (16384 x 65536) SVT time at P = 1 / 2 / 4 / 8 GPUs from measured per-rank work on ONE
B200 (this run has one GPU): rank 0's column block (65536 / P columns, c5 recipe) goes through the
library's multi-GPU path with a one-rank communicator and CPA_SVT_PANEL_SIM = P, which runs the P
ranks' panel launches one after another on this GPU -- so each phase's time is P x one rank's
(panel steps, row-sharded power products) or exactly one rank's (local Gram, unpack, line 12).
Per-rank time = gram + power / P + step / P + unpack + final, plus the collectives modelled at
the measured NVLink references of the profiling guide (8-rank all-reduce bus bandwidth 725 GB/s,
all-gather payload at the same bus rate, 20 us per small all-gather).  fp64 (default) or --math 3xtf32.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1705_07112_b200 import dist as D  # noqa: E402

BUS = 725e9
SMALL_AG_S = 20e-6
math = sys.argv[sys.argv.index("--math") + 1] if "--math" in sys.argv else "native"
dt = torch.float64 if math == "native" else torch.float32
es = 8 if math == "native" else 4
m, n, K, T = 16384, 65536, 40, 300
kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
h = D.make_handle(0)
for P in (1, 2, 4, 8):
    nb = n // P
    g = torch.Generator(device="cuda").manual_seed(12345)
    sd = (50 ** -0.5) ** 0.5
    A = torch.randn(m, 50, dtype=torch.float64, device="cuda", generator=g) * sd
    g.manual_seed(1000)
    X = torch.empty((m, nb), dtype=dt, device="cuda")
    for c0 in range(0, nb, 4096):
        c1 = min(nb, c0 + 4096)
        B = torch.randn(c1 - c0, 50, dtype=torch.float64, device="cuda", generator=g) * sd
        X[:, c0:c1] = (A @ B.T + 0.01 * torch.randn(m, c1 - c0, dtype=torch.float64, device="cuda", generator=g)).to(dt)
    if P > 1:
        os.environ["CPA_SVT_PANEL_SIM"] = str(P)
    try:
        D.apply_sharded(h, X, m, n, kern, K, T=T, math=math)   # warm-up
        torch.cuda.synchronize()
        h.profile(True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        D.apply_sharded(h, X, m, n, kern, K, T=T, math=math)
        ev1.record()
        torch.cuda.synchronize()
        prof = h.profile_read()
        h.profile(False)
    finally:
        os.environ.pop("CPA_SVT_PANEL_SIM", None)
    ms = {k: v[0] for k, v in prof.items() if v[1]}
    gram = ms.get("gram", 0.0)
    power = ms.get("power", 0.0) / P
    step = ms.get("step", 0.0) / P
    unpack = ms.get("exchange", 0.0)
    final = ms.get("final", 0.0) + ms.get("init", 0.0)
    G_bytes = m * m * es
    ar = 0.0 if P == 1 else 2 * (P - 1) / P * G_bytes / BUS * 1e3
    tri = m * (m + 64) / 2 * es                       # the packed lower triangle exchanged per step
    ag_steps = 0.0 if P == 1 else (K - 2) * ((P - 1) / P * tri / BUS * 1e3)
    ag_power = 0.0 if P == 1 else T * SMALL_AG_S * 1e3
    total = gram + ar + power + ag_power + step + unpack + ag_steps + final
    r = {"P": P, "math": math, "measured_one_gpu_ms": ev0.elapsed_time(ev1),
         "per_rank_ms": {"gram": gram, "power": power, "step": step, "unpack": unpack, "final+init": final},
         "modelled_collectives_ms": {"allreduce_G": ar, "allgather_power": ag_power, "allgather_steps": ag_steps},
         "projected_ms_per_svt": total}
    print(json.dumps(r), flush=True)
    del X
    torch.cuda.empty_cache()
h.close()
