import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1705_07112_b200 as P, oracle as O, workloads as W
h = P.Handle(0)
def run(X, kern, K, math, **kw):
    Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    Y, info = h.apply(Xd, kern, K, math=math, info=True, **kw)
    return Y.cpu().numpy().astype(np.float64), info
for shape in [(128, 256), (200, 333), (257, 1030)]:
    X = W.random_dense(*shape, seed=shape[0] + shape[1]).astype(np.float32).astype(np.float64)
    lam = 2.0 * float(np.linalg.norm(X, 2)) ** 2
    for math in ("3xtf32", "tf32"):
        Y, _ = run(X, None, 4, math, lambda_max=lam, coeffs=[lam, lam / 2, 0.0, 0.0])
        print("raw", shape, math, O.rel_fro(Y, X @ X.T @ X))
    # same chain in fp32 numpy for scale
    Xf = X.astype(np.float32)
    print("   numpy fp32 chain", O.rel_fro((Xf @ Xf.T @ Xf).astype(np.float64), X @ X.T @ X))
for shape, K in [((512, 2048), 40), ((700, 300), 12), ((300, 700), 20)]:
    X = W.gen_c2(m=shape[0], n=shape[1], seed=5).astype(np.float32).astype(np.float64)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=300, return_info=True)
    for math in ("3xtf32", "tf32"):
        Y, info = run(X, kern, K, math, T=300)
        print("parity", shape, K, math, O.rel_fro(Y, Yo), "lam rel", abs(info["lambda_hat"] - io["lambda_hat"]) / io["lambda_hat"])
    # same with the oracle's lambda given
    for math in ("3xtf32",):
        Y, info = run(X, kern, K, math, T=300, lambda_max=io["lambda_max"])
        print("   with oracle lambda", math, O.rel_fro(Y, Yo))
