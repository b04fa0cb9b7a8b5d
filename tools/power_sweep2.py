"""Power-phase time vs T at large s (fp64 and fp32 Gram), the streaming product."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W
h = P.Handle(0)
for s, dt, math in [(4096, torch.float64, "native"), (16384, torch.float64, "native"), (16384, torch.float32, "tf32")]:
    X = torch.randn(s, s + 64, dtype=torch.float64, device="cuda").to(dt)
    Y = torch.empty_like(X)
    kern = W.CONFIGS["c2"]["kernel"]
    for T in [1, 11, 101, 300]:
        for _ in range(1): h.apply(X, kern, 3, T=T, Y=Y, math=math)
        torch.cuda.synchronize()
        h.profile(True)
        for _ in range(3): h.apply(X, kern, 3, T=T, Y=Y, math=math)
        pr = h.profile_read(); h.profile(False)
        print(s, dt, T, "power ms %.3f" % (pr["power"][0] / 3), flush=True)
