"""Per-product cost of the power iteration: power-phase time vs T, with and without squaring."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W
h = P.Handle(0)
for s in [1024, 4096]:
    X = torch.from_numpy(W.gen_c2(m=s, n=s)).cuda()
    Y = torch.empty_like(X)
    kern = W.CONFIGS["c2"]["kernel"]
    for T in [1, 2, 8, 15, 16, 60, 120, 300, 1000]:
        for _ in range(2): h.apply(X, kern, 3, T=T, Y=Y)
        torch.cuda.synchronize()
        h.profile(True)
        for _ in range(5): h.apply(X, kern, 3, T=T, Y=Y)
        pr = h.profile_read(); h.profile(False)
        print(s, T, "power ms %.4f" % (pr["power"][0] / 5), "gram ms %.4f" % (pr["gram"][0] / 5), flush=True)
