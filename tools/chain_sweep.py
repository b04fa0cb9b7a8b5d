"""Sweep of the two-chain recurrence (CPA_SVT_SYM_CHAIN, CPA_SVT_CHAIN_SPLIT) against the one-chain
kernel on the c2 recipe at several s: median ms per SVT over `reps` L2-flushed calls and the
recurrence phase (profile).  python tools/chain_sweep.py [reps] [s,s,...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("PKG_DIR"):   # (A/B against another build of the package)
    sys.path.insert(0, os.environ["PKG_DIR"])
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sizes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1024, 2048, 4096]
kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for s in sizes:
    X = torch.from_numpy(W.gen_c2(m=s, n=s)).cuda()
    Y = torch.empty_like(X)
    ref = None
    grid = [("0", "")] + [(m, str(q)) for m in ("2", "3") for q in (0, 1, 2, 3, 4, 6)]
    for chain, split in ([("0", "")] if os.environ.get("SWEEP_ONECHAIN") else grid):
        os.environ["CPA_SVT_SYM_CHAIN"] = chain
        if split and split != "0":
            os.environ["CPA_SVT_CHAIN_SPLIT"] = split
        else:
            os.environ.pop("CPA_SVT_CHAIN_SPLIT", None)
        h = P.Handle(0)
        h.set_form("poly")
        for _ in range(3):
            h.apply(X, kern, 30, T=300, Y=Y)
        h.profile(True)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for i in range(reps):
            flush.fill_(i & 255)
            ev[i][0].record()
            h.apply(X, kern, 30, T=300, Y=Y)
            ev[i][1].record()
        torch.cuda.synchronize()
        prof = h.profile_read()
        h.close()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        if ref is None:
            ref = Y.clone()
            d = 0.0
        else:
            d = float(torch.linalg.norm(Y - ref) / torch.linalg.norm(ref))
        step = prof.get("step", prof.get("recurrence", [0, 0]))
        print(f"s={s} chain={chain} split={split or 'auto'} median={ms[len(ms) // 2]:.4f} ms "
              f"step={step[0] / reps:.4f} ms  rel_vs_onechain={d:.2e}", flush=True)
