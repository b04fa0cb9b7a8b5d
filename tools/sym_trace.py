"""Timeline of the c2 symmetric recurrence (trace build of the library: CPA_SYM_TRACE).
Per unit: claim, claim broadcast, dependency satisfied, mainloop end, epilogue end (globaltimer, ns).
Prints where the CTA time goes and how the steps overlap.
  python paper_1705_07112_b200/build.py --variant trace CPA_SYM_TRACE=1
  CPA_SVT_LIB=paper_1705_07112_b200/libcpasvt_trace.so python tools/sym_trace.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

assert "trace" in P.LIB_PATH, "set CPA_SVT_LIB to the trace build"
P.lib.cpa_svt_debug_sym_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
X = torch.from_numpy(W.gen_c2()).cuda()
h = P.Handle(0)
kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
for _ in range(3):
    h.apply(X, kern, 30, T=300)
torch.cuda.synchronize()
h.apply(X, kern, 30, T=300)
torch.cuda.synchronize()
T, K = 16, 30
S = int(os.environ.get("TRACE_S", "6"))   # the k-splits of the launch (two chains at c2: 3)
units = (K - 2) * T * (T + 1) // 2 * S
buf = np.zeros(units * 6, dtype=np.uint64)
assert P.lib.cpa_svt_debug_sym_trace(buf.ctypes.data, units) == 0
tr = buf.reshape(units, 6).astype(np.int64)
t0 = tr[:, 0].min()
tc, tb, td, tm, te = [(tr[:, i] - t0) / 1e3 for i in range(5)]   # us
sm = tr[:, 5] & 0xFFFF
cta = tr[:, 5] >> 16
per_step = T * (T + 1) // 2 * S
step = np.arange(units) // per_step
q = np.arange(units) % S
total = te.max()
res = {"kernel_us": total,
       "mean_us": {"claim_atomic": float((tb - tc).mean()), "dep_wait": float((td - tb).mean()),
                   "mainloop": float((tm - td).mean()), "epilogue": float((te - tm).mean()),
                   "epilogue_reducer": float((te - tm)[q == S - 1].mean()),
                   "epilogue_publisher": float((te - tm)[q < S - 1].mean())}}
# per-CTA busy fractions and the gaps between a CTA's units
ncta = int(cta.max()) + 1
frac = {"claim": 0.0, "dep": 0.0, "main": 0.0, "epi": 0.0}
gaps = []
for c in range(ncta):
    idx = np.where(cta == c)[0]
    idx = idx[np.argsort(tc[idx])]
    frac["claim"] += float((tb[idx] - tc[idx]).sum())
    frac["dep"] += float((td[idx] - tb[idx]).sum())
    frac["main"] += float((tm[idx] - td[idx]).sum())
    frac["epi"] += float((te[idx] - tm[idx]).sum())
    gaps += list(tc[idx][1:] - te[idx][:-1])
tot_cta = ncta * total
res["cta_time_fraction"] = {k: v / tot_cta for k, v in frac.items()}
res["cta_time_fraction"]["between_units"] = float(np.sum(gaps)) / tot_cta
res["steps"] = [{"k": int(k + 2), "first_claim": float(tc[step == k].min()), "last_end": float(te[step == k].max()),
                 "median_end": float(np.median(te[step == k]))} for k in range(K - 2)]
per_step_dur = np.diff([s_["last_end"] for s_ in res["steps"]])
res["mean_step_spacing_us"] = float(per_step_dur.mean())
# the (15, 15) corner tile's units per step (the chain the wavefront cannot overlap)
corner = T * (T + 1) // 2 - 1
res["corner_tile_ends"] = [float(te[(step == k) & (np.arange(units) % per_step // S == corner)].max())
                           for k in range(K - 2)]
print(json.dumps(res))
