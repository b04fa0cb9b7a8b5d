import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_1705_07112_b200 as P, workloads as W
h = P.Handle(0)
X = torch.from_numpy(W.gen_c2()).cuda()
h.apply(X, W.CONFIGS["c2"]["kernel"], 3, T=10)
torch.cuda.synchronize()
