"""Device timeline of c2 SVTs (torch.profiler / CUPTI): every kernel and memset of one
cpa_svt_apply call with its start, duration and the idle gap before it -- what the launch
sequence costs beyond the kernels themselves.

    python tools/gap_trace.py [config=c2] [reps=5]   (GPU box)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    c = W.CONFIGS[name]
    X = torch.from_numpy(np.ascontiguousarray(W.gen_c2() if name == "c2" else W.gen_c1())).cuda()
    Y = torch.empty_like(X)
    h = P.Handle(0)
    for _ in range(5):
        h.apply(X, c["kernel"], c["K"], T=c["T"], Y=Y)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(20):
        h.apply(X, c["kernel"], c["K"], T=c["T"], Y=Y)
    ev[1].record()
    torch.cuda.synchronize()
    per = ev[0].elapsed_time(ev[1]) / 20
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            h.apply(X, c["kernel"], c["K"], T=c["T"], Y=Y)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    rows = [(e.name, e.time_range.start, e.time_range.end - e.time_range.start) for e in evs]
    # one SVT = the ops between consecutive first-kernel occurrences
    first = rows[0][0]
    starts = [i for i, r in enumerate(rows) if r[0] == first]
    out = []
    for a, b in zip(starts, starts[1:] + [len(rows)]):
        seg = rows[a:b]
        t0 = seg[0][1]
        end = seg[-1][1] + seg[-1][2]
        busy = sum(r[2] for r in seg)
        gaps = [seg[i][1] - (seg[i - 1][1] + seg[i - 1][2]) for i in range(1, len(seg))]
        out.append({"span_us": end - t0, "busy_us": busy, "gap_us": sum(gaps),
                    "ops": [(r[0][:60], round(r[2], 1), round(g, 1)) for r, g in zip(seg, [0.0] + gaps)]})
    print(json.dumps({"config": name, "event_ms_per_svt": per, "svts": out[1:]}, indent=1))


if __name__ == "__main__":
    main()
