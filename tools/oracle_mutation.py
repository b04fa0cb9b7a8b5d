"""Mutation check of the oracle's pins: each mutation below changes one piece of the oracle's
arithmetic (a dropped term, a wrong sign, scale, index, start vector or step count -- the kinds of
mistake the pins exist to catch); the CPU suite (`pytest -m "not gpu"`) must fail for every one.
Runs on a copy of the repository in a temporary directory; the repository is never modified.

    python tools/oracle_mutation.py          # prints KILLED / SURVIVED per mutation, exit 1 if any survive
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTS = [
 ("wsoft sqrt->id", "w = kernel.w_c / (math.sqrt(max(x - kernel.w_shift, 0.0)) + kernel.w_eps)", "w = kernel.w_c / (max(x - kernel.w_shift, 0.0) + kernel.w_eps)"),
 ("wsoft 2w", "return (r - w) / r if r > w else 0.0", "return (r - 2*w) / r if r > 2*w else 0.0"),
 ("soft tau sign", "return (r - tau) / r if r > tau else 0.0", "return (r + tau) / r if r > tau else 0.0"),
 ("hard >=", "return 1.0 if r > tau else 0.0", "return 1.0 if r >= 0.9*tau else 0.0"),
 ("theta l", "theta = [math.pi * (l - 0.5) / K for l in range(1, K + 1)]", "theta = [math.pi * (l - 0.4) / K for l in range(1, K + 1)]"),
 ("2/K", "c.append(2.0 / K * acc)", "c.append(1.0 / K * acc)"),
 ("c0/2 series", "acc = 0.5 * c[0]", "acc = 1.0 * c[0]"),
 ("c0/2 alg1", "H = 0.5 * c[0] * Psi_km2\n    if Kc > 1:", "H = 1.0 * c[0] * Psi_km2\n    if Kc > 1:"),
 ("Bh scale", "Bh = (2.0 / lam) * Phi_ - Id", "Bh = (2.0 / lam) * Phi_ - Id * 1.0001"),
 ("recurrence sign", "Psi_k = 2.0 * (Bh @ Psi_km1) - Psi_km2\n        H = H + c[k] * Psi_k", "Psi_k = 2.0 * (Bh @ Psi_km1) + Psi_km2\n        H = H + c[k] * Psi_k"),
 ("line12 scale", "return B @ H, info", "return (B @ H) * 1.0000001, info"),
 ("sigma from Lambda", "return lam, lam_hat, math.sqrt(max(lam_hat, 0.0))", "return lam, lam_hat, math.sqrt(max(lam, 0.0))"),
 ("power v0", "v = np.full(s, 1.0 / math.sqrt(s))\n    hist = []", "v = np.full(s, 1.0 / math.sqrt(s)); v[0] *= 2\n    hist = []"),
 ("power T-1", "    for _ in range(T):\n        u = apply_phi(v)", "    for _ in range(max(T - 1, 1)):\n        u = apply_phi(v)"),
 ("safety", "DEFAULT_SAFETY = 1.01", "DEFAULT_SAFETY = 1.02"),
 ("vec bhat sign", "return (2.0 / lam) * apply_phi(W) - W", "return (2.0 / lam) * apply_phi(W) + 0.0001 * W - W"),
 ("vec recurrence", "w_k = 2.0 * bhat(w_km1) - w_km2", "w_k = 2.0 * bhat(w_km1) - 1.0001 * w_km2"),
 ("vec c0/2", "out = 0.5 * c[0] * w_km2", "out = 0.5001 * c[0] * w_km2"),
 ("vec c1", "out = out + c[1] * w_km1", "out = out + 1.0001 * c[1] * w_km1"),
 ("sparse power n-side", "return power_iteration(lambda v: Xs @ (Xs.T @ v), m, T)", "return power_iteration(lambda v: Xs.T @ (Xs @ v), Xs.shape[1], T)"),
 ("sparse phi", "        return Xs.T @ (Xs @ W)\n\n    return cpa_apply_vectors", "        return 1.0001 * (Xs.T @ (Xs @ W))\n\n    return cpa_apply_vectors"),
 ("columns lam", "    lam_, lam_hat, sig = _lam_from_gram_side(apply_phi, m, T, safety, lam)", "    lam_, lam_hat, sig = _lam_from_gram_side(apply_phi, m, T + 1, safety, lam)"),
 ("rows lam", "    lam_, lam_hat, sig = _lam_from_gram_side(apply_phi, n, T, safety, lam)", "    lam_, lam_hat, sig = _lam_from_gram_side(apply_phi, n, T + 1, safety, lam)"),
 ("batched safety", "Y[b], info = cpa_shrink(Xb[b], kernel, K, T=T, safety=safety, return_info=True)", "Y[b], info = cpa_shrink(Xb[b], kernel, K, T=T, safety=safety * 1.001, return_info=True)"),
 ("alg1 T+1", "        lambda: power_iteration(lambda v: Phi_ @ v, n, T)[0], lam_override, safety)", "        lambda: power_iteration(lambda v: Phi_ @ v, n, T + 1)[0], lam_override, safety)"),
 ("sparse T+1", "return power_iteration(lambda v: Xs @ (Xs.T @ v), m, T)", "return power_iteration(lambda v: Xs @ (Xs.T @ v), m, T + 1)"),
 ("haar high sign", "        T[nl + i, 2 * i + 1] = -r", "        T[nl + i, 2 * i + 1] = r"),
 ("haar odd tail", "        T[nl - 1, n - 1] = 1.0", "        T[nl - 1, n - 1] = r"),
 ("dct a0", "    C[0, :] = math.sqrt(1.0 / n)", "    C[0, :] = math.sqrt(2.0 / n)"),
 ("dct phase", "    C = np.cos(np.pi * (2 * j + 1) * k / (2 * n)) * math.sqrt(2.0 / n)", "    C = np.cos(np.pi * (2 * j) * k / (2 * n)) * math.sqrt(2.0 / n)"),
 ("block dct size", "def dct2_block_matrix(n: int, b: int = 8) -> np.ndarray:", "def dct2_block_matrix(n: int, b: int = 4) -> np.ndarray:"),
 ("haar highpass kept", "        Phi_[nl:, :] = 0.0\n        Phi_[:, nl:] = 0.0", "        Phi_[nl:, :] = 0.0"),
 ("threshold >", "    return np.where(A >= thr, Phi, 0.0), thr", "    return np.where(A > thr, Phi, 0.0), thr"),
 ("topk index", "        thr = float(flat[min(max(k, 1), flat.size) - 1])", "        thr = float(flat[min(max(k, 1), flat.size - 1)])"),
 ("transform line12", "    Y = B @ Tm.T @ H @ Tm\n", "    Y = B @ Tm @ H @ Tm.T\n"),
 ("eps schedule El", "    frac = 0.5e-4 if E > 0.3e-1 else (1.5e-4 if E > 6e-4 else 0.5e-3)", "    frac = 0.5e-4 if E > 0.3e-2 else (1.5e-4 if E > 6e-4 else 0.5e-3)"),
 ("synthetic D", "        D[b * p:(b + 1) * p, b * p:(b + 1) * p] -= 0.5", "        D[b * p:(b + 1) * p, b * p:(b + 1) * p] -= 0.25"),
 ("admm l update", "    return (zu1 + psit(zu2) + w * zu3 + zu4) / (3.0 + w)", "    return (zu1 + psit(zu2) + w * zu3 + zu4) / (4.0 + w)"),
 ("admm l no inverse DCT", "    return (zu1 + psit(zu2) + w * zu3 + zu4) / (3.0 + w)", "    return (zu1 + zu2 + w * zu3 + zu4) / (3.0 + w)"),
 ("admm z2 threshold", "    return np.sign(v) * np.maximum(np.abs(v) - eta / rho, 0.0)", "    return np.sign(v) * np.maximum(np.abs(v) - eta * rho, 0.0)"),
 ("admm z4 clip", "    return np.clip(v, 0.0, 1.0)", "    return np.clip(v, 0.0, 2.0)"),
 ("jacobi rotation sign", "                    A[:, i], A[:, j] = c * ai - s * aj, s * ai + c * aj", "                    A[:, i], A[:, j] = c * ai + s * aj, s * ai + c * aj"),
 ("jacobi V update", "                    V[:, i], V[:, j] = c * vi - s * vj, s * vi + c * vj", "                    V[:, i], V[:, j] = c * vi - s * vj, s * vi - c * vj"),
 ("jacobi sweeps", "def jacobi_svd(A, max_sweeps: int = 80, tol: float = 1e-15):", "def jacobi_svd(A, max_sweeps: int = 1, tol: float = 1e-15):"),
 ("jacobi transposed", "    if transposed:\n        U, V = V, U\n    return U, sigma, V", "    return U, sigma, V"),
 ("exact shrink g", "    gs = np.array([g_response(kernel, float(si), tau) for si in s])", "    gs = np.array([g_response(kernel, float(si), 0.9 * tau) for si in s])"),
 ("svd char", "    d = np.array([float(si) * series_eval(c, lam, float(si) ** 2) if si > 1e-300 else 0.0 for si in s])", "    d = np.array([float(si) * series_eval(c, lam, float(si)) if si > 1e-300 else 0.0 for si in s])"),
 ("rel_fro den", "    den = float(np.linalg.norm(B))", "    den = float(np.linalg.norm(A))"),
]


def main():
    src = open(os.path.join(ROOT, "oracle", "cpa_oracle.py")).read()
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    for d in ("tests", "oracle", "workloads", "paper_1705_07112_b200", "include", "examples"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d), ignore=shutil.ignore_patterns("build", "build_*"))
    for f in ("pytest.ini", "bench.py", "__graft_entry__.py"):
        shutil.copy(os.path.join(ROOT, f), tmp)
    survived = 0
    try:
        for name, a, b in MUTS:
            assert a in src, f"mutation target of {name!r} not found"
            open(os.path.join(tmp, "oracle", "cpa_oracle.py"), "w").write(src.replace(a, b, 1))
            # the oracle's pins first (most mutations fail there within seconds), then the rest of the
            # CPU suite (pytest drops the duplicate collection of the pins file)
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "tests", "-m", "not gpu",
                                "-x", "-q", "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
            last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
            # a kill is a FAILED test; a collection error would "kill" every mutation and prove nothing
            killed = r.returncode != 0 and " failed" in last and " error" not in last
            survived += not killed
            print(f"{name:22s} {'KILLED' if killed else 'SURVIVED'}  {last[:90]}", flush=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print(f"{len(MUTS) - survived} of {len(MUTS)} mutations killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
