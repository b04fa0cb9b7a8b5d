import torch, numpy as np, sys
sys.path.insert(0, "/root/repo")
import paper_1705_07112_b200 as P
h = P.Handle(0)
torch.manual_seed(0)
for (M, N, K, bmn) in [(128, 128, 32, False), (128, 128, 32, True), (128, 128, 64, True), (200, 130, 100, True)]:
    A = torch.randn(M, (K + 3)//4*4, device="cuda")[:, :K].contiguous() if K % 4 == 0 else None
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")
    C = h.debug_gemm_tf32(A, B, bmn, 3)
    ref = (A.double() @ (B.double() if bmn else B.double().T)).float()
    err = (C - ref).norm() / ref.norm()
    print(M, N, K, bmn, "rel err", float(err), "C[0,:4]", C[0, :4].tolist(), "ref", ref[0, :4].tolist())
    nz = (C != 0).float().mean().item()
    print("   nonzero frac", nz, "C max", C.abs().max().item())
    if err > 1e-3:
        # try to identify structure: compare C with ref transposed / permuted
        r = ref.cpu().numpy(); c = C.cpu().numpy()
        for name, cand in [("T", r.T if r.shape[0]==r.shape[1] else None)]:
            if cand is not None: print("   vs", name, np.linalg.norm(c-cand)/np.linalg.norm(cand))
        # row/col nonzero pattern
        print("   nonzero rows", np.nonzero(np.abs(c).sum(1))[0][:20], "cols", np.nonzero(np.abs(c).sum(0))[0][:20])
