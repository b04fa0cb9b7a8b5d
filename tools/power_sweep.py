import sys, torch, json
sys.path.insert(0, "/root/repo")
import paper_1705_07112_b200 as P, workloads as W
h = P.Handle(0)
X = torch.from_numpy(W.gen_c2()).cuda()
Y = torch.empty_like(X)
kern = W.CONFIGS["c2"]["kernel"]
for T in [1, 2, 15, 16, 60, 120, 300]:
    for _ in range(2): h.apply(X, kern, 3, T=T, Y=Y)
    torch.cuda.synchronize()
    h.profile(True)
    for _ in range(5): h.apply(X, kern, 3, T=T, Y=Y)
    pr = h.profile_read(); h.profile(False)
    print(T, "power ms", pr["power"][0] / 5, "gram ms", pr["gram"][0] / 5)
