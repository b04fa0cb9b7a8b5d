import torch, time
x = torch.empty(1024*1024, dtype=torch.float64).pin_memory()
y = torch.empty(1024*1024, dtype=torch.float64).pin_memory()
d = torch.empty(1024*1024, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    d.copy_(x, non_blocking=True); y.copy_(d, non_blocking=True)
torch.cuda.synchronize()
for name, fn in [("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: y.copy_(d, non_blocking=True))]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(name, "%.3f ms for 8 MiB -> %.1f GB/s" % (ms, 8.388608e6 / ms / 1e6))
