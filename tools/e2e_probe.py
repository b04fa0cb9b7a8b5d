"""Where does the e2e time of cpa_svt_apply_host go (c2)?"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W
cfg = W.CONFIGS["c2"]
X = W.gen_c2()
Xh = torch.from_numpy(X).pin_memory(); Yh = torch.empty_like(Xh).pin_memory()
Xd = Xh.cuda(); Yd = torch.empty_like(Xd)
h = P.Handle(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, n=10, fl=False):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(n):
        if fl: flush.fill_(i & 255)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(); fn(); e[1].record(); torch.cuda.synchronize()
        tot += e[0].elapsed_time(e[1])
    return tot / n
for fl in (False, True):
    print("flush", fl, "device apply   %.3f ms" % t(lambda: h.apply(Xd, cfg["kernel"], cfg["K"], T=cfg["T"], Y=Yd), fl=fl))
    print("flush", fl, "apply_host     %.3f ms" % t(lambda: h.apply_host(Xh, Yh, cfg["kernel"], cfg["K"], T=cfg["T"]), fl=fl))
print("h2d+d2h torch  %.3f ms" % t(lambda: (Xd.copy_(Xh, non_blocking=True), Yh.copy_(Yd, non_blocking=True))))
import time
for _ in range(3): h.apply_host(Xh, Yh, cfg["kernel"], cfg["K"], T=cfg["T"])
t0 = time.perf_counter()
for _ in range(10): h.apply_host(Xh, Yh, cfg["kernel"], cfg["K"], T=cfg["T"])
print("apply_host wall %.3f ms" % ((time.perf_counter() - t0) / 10 * 1e3))
