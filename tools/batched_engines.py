"""c3 with both batched engines: time (CUDA events) and parity on 256 sampled matrices."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W, oracle as O
cfg = W.CONFIGS["c3"]
Xb = W.gen_c3()
Xd = torch.from_numpy(Xb).cuda()
idx = np.random.default_rng(0).choice(Xb.shape[0], 128, replace=False)
Yo, lo = O.cpa_shrink_batched(Xb[idx].astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
for eng in ("ffma", "tc"):
    h = P.Handle(0)
    h.set_batched_engine(eng)
    Y = torch.empty_like(Xd)
    lam = torch.empty(Xb.shape[0], dtype=torch.float32, device="cuda")
    for _ in range(2):
        h.apply_batched(Xd, cfg["kernel"], cfg["K"], T=cfg["T"], Y=Y, lambda_out=lam)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(5):
        h.apply_batched(Xd, cfg["kernel"], cfg["K"], T=cfg["T"], Y=Y, lambda_out=lam)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 5
    Ys = Y[torch.from_numpy(idx).cuda()].cpu().numpy().astype(np.float64)
    err = O.rel_fro(Ys, Yo)
    lerr = float(np.max(np.abs(lam.cpu().numpy()[idx] - lo) / lo))
    print(json.dumps({"engine": eng, "ms": ms, "rel_fro": err, "lambda_rel_err": lerr}), flush=True)
    h.close()
