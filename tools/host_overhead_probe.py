"""Host-side cost of one c2 call (the part an apply_host e2e number cannot hide): wall time of the
binding + C ABI call for a device-resident (asynchronous) apply, and of apply_host (synchronous)
next to its device-timed span.   python tools/host_overhead_probe.py   (GPU box)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

c = W.CONFIGS["c2"]
X = torch.from_numpy(np.ascontiguousarray(W.gen_c2())).cuda()
Y = torch.empty_like(X)
h = P.Handle(0)
for _ in range(5):
    h.apply(X, c["kernel"], c["K"], T=c["T"], Y=Y)
torch.cuda.synchronize()
# asynchronous calls: the host returns long before the GPU is done (queue depth 30 << limits)
t = []
for _ in range(30):
    t0 = time.perf_counter()
    h.apply(X, c["kernel"], c["K"], T=c["T"], Y=Y)
    t.append(time.perf_counter() - t0)
torch.cuda.synchronize()
t.sort()
print(f"device-resident apply: host time per call median {1e6 * t[len(t) // 2]:.1f} us (min {1e6 * t[0]:.1f})")
# the raw C call (no binding): same arguments
import ctypes  # noqa: E402
k = P.kernel_from_dict(c["kernel"])
lam = P.Lambda(c["T"], 0, 1.01, 0.0, 0.0)
t = []
for _ in range(30):
    t0 = time.perf_counter()
    P.lib.cpa_svt_apply(h._h, 0, 0, 1024, 1024, 0, 0, X.data_ptr(), 1024, Y.data_ptr(), 1024, ctypes.byref(k),
                        c["K"], None, ctypes.byref(lam), None)
    t.append(time.perf_counter() - t0)
torch.cuda.synchronize()
t.sort()
print(f"raw cpa_svt_apply: host time per call median {1e6 * t[len(t) // 2]:.1f} us (min {1e6 * t[0]:.1f})")
Xh = X.cpu().pin_memory()
Yh = torch.empty_like(Xh).pin_memory()
for _ in range(5):
    h.apply_host(Xh, Yh, c["kernel"], c["K"], T=c["T"])
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
wall, dev = [], []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    h.apply_host(Xh, Yh, c["kernel"], c["K"], T=c["T"])
    ev[1].record()
    torch.cuda.synchronize()
    wall.append(time.perf_counter() - t0)
    dev.append(ev[0].elapsed_time(ev[1]) * 1e-3)
wall.sort(); dev.sort()
print(f"apply_host: wall median {1e6 * wall[10]:.1f} us, event span median {1e6 * dev[10]:.1f} us")
