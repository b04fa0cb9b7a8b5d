"""cuBLAS fp64 / tf32 / fp32 GEMM throughput on this B200 (roofline context)."""
import json, torch
r = {}
torch.backends.cuda.matmul.allow_tf32 = False
for name, dt, n, tf32 in [("dgemm", torch.float64, 8192, False), ("sgemm", torch.float32, 8192, False),
                          ("tf32gemm", torch.float32, 8192, True)]:
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    r[name + "_tflops"] = 2 * n**3 / best / 1e9
# 1024^2 dgemm (config-2 step size)
torch.backends.cuda.matmul.allow_tf32 = False
a = torch.randn(1024, 1024, device="cuda", dtype=torch.float64); b = torch.randn_like(a)
for _ in range(10): a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(100): a @ b
e1.record(); torch.cuda.synchronize()
r["dgemm1024_us"] = e0.elapsed_time(e1) * 10
r["dgemm1024_tflops"] = 2 * 1024**3 / (e0.elapsed_time(e1) / 100) / 1e9
print(json.dumps(r))
