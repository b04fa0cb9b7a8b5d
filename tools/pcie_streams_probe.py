"""H2D bandwidth of 8 MiB from pinned memory: one stream vs the same bytes split over 2 / 4
streams (separate copy engines), the question behind cpa_svt_apply_host's copy pipeline."""
import torch
N = 1024 * 1024
x = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    def run():
        ev = torch.cuda.Event()
        ev.record()
        for i, s in enumerate(ss):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                lo, hi = i * N // ns, (i + 1) * N // ns
                d[lo:hi].copy_(x[lo:hi], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
    for _ in range(5): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("h2d %d stream(s): %.3f ms for 8 MiB -> %.1f GB/s" % (ns, ms, 8.388608e6 / ms / 1e6))
