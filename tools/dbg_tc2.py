import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_1705_07112_b200 as P
torch.manual_seed(0)
for (M, N, K) in [(128, 128, 32), (128, 128, 64), (256, 384, 100)]:
    A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda")
    ref = (A.double() @ B.double()).float()
    for lbo, sbo in [(4096, 512), (512, 4096), (4096, 1024), (1024, 4096)]:
        os.environ["CPA_SVT_DBG_LBO"] = str(lbo); os.environ["CPA_SVT_DBG_SBO"] = str(sbo)
        h = P.Handle(0)
        C = h.debug_gemm_tf32(A, B, True, 3)
        err = float((C - ref).norm() / ref.norm())
        print(M, N, K, lbo, sbo, "err", err, "nz", float((C != 0).float().mean()), flush=True)
        h.close()
