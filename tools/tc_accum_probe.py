"""How accurate is the tcgen05 fp32 accumulation over a long K?  C = A A^T (3xTF32)
for A = (c5 recipe rows) at K = 1024..65536, against fp64."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W
h = P.Handle(0)
X = W.gen_c5(m=256, n=65536, dtype=np.float32)
for K in [1024, 4096, 16384, 65536]:
    A = np.ascontiguousarray(X[:, :K])
    C = h.debug_gemm_tf32(torch.from_numpy(A).cuda(), torch.from_numpy(A).cuda(), False, 3).cpu().numpy().astype(np.float64)
    R = A.astype(np.float64) @ A.astype(np.float64).T
    d = np.diag(C) / np.diag(R) - 1
    e = np.abs(C - R).max() / np.abs(R).max()
    # plain fp32 sequential-ish reference error for scale
    R32 = (A @ A.T).astype(np.float64)
    print(K, "diag rel err mean %.2e max %.2e" % (d.mean(), np.abs(d).max()), "max err %.2e" % e,
          "| numpy fp32 %.2e" % (np.abs(R32 - R).max() / np.abs(R).max()), flush=True)
ones = np.ones((128, 65536), dtype=np.float32) * np.float32(1 + 2 ** -11)
C = h.debug_gemm_tf32(torch.from_numpy(ones).cuda(), torch.from_numpy(ones).cuda(), False, 3).cpu().numpy()
print("const (1+2^-11)^2 * 65536: got %.9g want %.9g" % (C[0, 0], 65536 * (1 + 2 ** -11) ** 2))
