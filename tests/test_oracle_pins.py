"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the SURVEY.md §8c pin (P1..P17) and the PAPER.md passage.
None re-types the oracle's own formula: they check closed forms, invariants,
brute force, or independent library routines (numpy.linalg.svd / eigvalsh).
"""

import json
import math
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _orth(n, rng):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


# --- P1: coefficient exactness -----------------------

@pytest.mark.parametrize("K", [2, 3, 8, 20, 41])
def test_p1_constant_and_linear(K):
    lam = 7.25
    c = O.chebyshev_coefficients(lambda x: 1.0, K, lam)
    assert abs(c[0] - 2.0) < 1e-14 and max(abs(v) for v in c[1:] or [0]) < 1e-14
    c = O.chebyshev_coefficients(lambda x: 2 * x / lam - 1.0, K, lam)
    want = [0.0] * K
    want[1] = 1.0
    assert max(abs(a - b) for a, b in zip(c, want)) < 1e-14


@pytest.mark.parametrize("K,j", [(8, 3), (8, 7), (20, 11), (30, 0)])
def test_p1_polynomial_reproduced(K, j):
    # h(x) = cos(j arccos(2x/lam - 1)) is psi_j of the shifted variable;
    # discrete orthogonality over the K first-kind nodes gives c = 2 e_j (j=0) / e_j.
    lam = 3.0
    h = lambda x: math.cos(j * math.acos(max(-1.0, min(1.0, 2 * x / lam - 1.0))))
    c = O.chebyshev_coefficients(h, K, lam)
    want = [0.0] * K
    want[j] = 2.0 if j == 0 else 1.0
    assert max(abs(a - b) for a, b in zip(c, want)) < 1e-13


# --- P2: interpolation at the nodes --------------------------------------------

@pytest.mark.parametrize("kind", ["soft", "hard", "wsoft"])
def test_p2_interpolates_at_nodes(kind):
    K, lam = 17, 50.0
    k = O.Kernel(kind, tau=3.1, w_c=9.0, w_eps=1e-6)
    c = O.kernel_coefficients(k, K, lam, 1.0)
    for l in range(1, K + 1):
        x = lam / 2 * (math.cos(math.pi * (l - 0.5) / K) + 1)
        assert abs(O.series_eval(c, lam, x) - O.h_response(k, x, 3.1)) < 1e-13


# --- P3: recurrence == closed form -----------------------------------------------

def test_p3_psi_recurrence_closed_form():
    for k in range(65):
        for th in [0.0, math.pi / 7, math.pi / 3, math.pi / 2, 2.5, math.pi, 0.123]:
            assert abs(O.chebyshev_psi_recurrence(k, math.cos(th)) - math.cos(k * th)) < 1e-12
            assert abs(O.chebyshev_psi(k, math.cos(th)) - math.cos(k * th)) < 1e-12


# --- golden: kernel values (SPEC examples) ----------------------------------------

def test_golden_kernel_eval():
    for e in GOLDEN["kernel_eval"]:
        assert O.h_response(O.Kernel(e["kind"], tau=e["tau"]), e["x"], e["tau"]) == e["h"], e["cite"]


def test_golden_power_iteration():
    for e in GOLDEN["power_iteration"]:
        G = np.diag(e["diag"])
        lam, _ = O.power_iteration(lambda v: G @ v, len(e["diag"]), 200)
        assert abs(lam - e["lambda"]) < 1e-12, e["cite"]


def test_golden_exact_shrink():
    e = GOLDEN["exact_shrink"][0]
    Y = O.exact_shrink(np.array(e["X"]), O.Kernel(e["kind"], tau=e["tau"]), e["tau"])
    s = np.linalg.svd(Y, compute_uv=False)
    assert np.allclose(s, e["singular_values"], atol=1e-14), e["cite"]
    e = GOLDEN["exact_shrink"][1]
    Y = O.exact_shrink(np.array(e["X"], float), O.Kernel(e["kind"], tau=e["tau"]), e["tau"])
    assert np.allclose(Y, e["Y_diag"] * np.eye(4), atol=1e-15), e["cite"]


# --- P4: diagonal X -------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(9, 6), (6, 9), (7, 7)])
def test_p4_diagonal(shape):
    m, n = shape
    d = np.array([5.0, 3.0, 2.5, 1.0, 0.5, 0.25, 4.0][:min(m, n)])
    X = np.zeros(shape)
    X[np.arange(len(d)), np.arange(len(d))] = d
    k = O.Kernel("soft", tau=1.1)
    Y, info = O.cpa_shrink(X, k, 12, T=400, return_info=True)
    want = np.zeros(shape)
    for i, di in enumerate(d):
        want[i, i] = di * O.series_eval(info["coeffs"], info["lambda_max"], di * di)
    assert np.abs(Y - want).max() <= 1e-13 * np.abs(want).max()
    off = Y.copy()
    off[np.arange(len(d)), np.arange(len(d))] = 0
    assert np.abs(off).max() == 0.0


# --- P5: node-exact shrinkage vs the TRUE g ----------------------------------------------

@pytest.mark.parametrize("kind", ["soft", "hard", "wsoft"])
def test_p5_node_exact(kind):
    rng = np.random.default_rng(5)
    K, lam, m, n = 10, 100.0, 14, 10
    nodes = [lam / 2 * (math.cos(math.pi * (l - 0.5) / K) + 1) for l in range(1, K + 1)]
    d = np.sqrt(np.array(nodes))
    U, V = _orth(m, rng)[:, :n], _orth(n, rng)
    X = (U * d) @ V.T
    k = O.Kernel(kind, tau=4.0, w_c=20.0, w_eps=1e-6)
    Y = O.cpa_shrink(X, k, K, lam=lam)
    want = (U * np.array([O.g_response(k, di, 4.0) for di in d])) @ V.T
    assert O.rel_fro(Y, want) < 1e-12


# --- P6: orthogonal X ---------------------------------------------------------------------

def test_p6_orthogonal():
    rng = np.random.default_rng(6)
    a = 3.0
    Q = _orth(12, rng)
    Y, info = O.cpa_shrink(a * Q, O.Kernel("soft", tau=1.0), 15, T=30, return_info=True)
    assert abs(info["lambda_hat"] - a * a) < 1e-13 * a * a
    f = a * O.series_eval(info["coeffs"], info["lambda_max"], a * a)
    assert O.rel_fro(Y, f * Q) < 1e-13


# --- P7: rank one ---------------------------------------------------------------------------

def test_p7_rank_one():
    rng = np.random.default_rng(7)
    u = rng.standard_normal(20); u /= np.linalg.norm(u)
    v = rng.standard_normal(13); v /= np.linalg.norm(v)
    sig = 6.5
    X = sig * np.outer(u, v)
    Y, info = O.cpa_shrink(X, O.Kernel("soft", tau=2.0), 20, T=50, return_info=True)
    assert abs(info["lambda_hat"] - sig ** 2) < 1e-12 * sig ** 2
    f = sig * O.series_eval(info["coeffs"], info["lambda_max"], sig ** 2)
    assert O.rel_fro(Y, f * np.outer(u, v)) < 1e-13


# --- P8: raw coefficients ----------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(11, 7), (7, 11)])
def test_p8_raw_coefficients(shape):
    rng = np.random.default_rng(8)
    X = rng.standard_normal(shape)
    lam = 2.0 * np.linalg.norm(X, 2) ** 2
    assert O.rel_fro(O.cpa_shrink(X, None, 4, lam=lam, coeffs=[2.0, 0, 0, 0]), X) < 1e-15
    G_side = X @ X.T @ X  # (XX^T)X == X(X^T X)
    assert O.rel_fro(O.cpa_shrink(X, None, 4, lam=lam, coeffs=[lam, lam / 2, 0, 0]), G_side) < 1e-13
    # e_k -> Psi_k(B_hat) applied to X, compared with a plain GEMM chain of the closed form
    m, n = shape
    left = m <= n
    G = X @ X.T if left else X.T @ X
    s = G.shape[0]
    Bh = 2.0 / lam * G - np.eye(s)
    # Psi_k via the eigen-decomposition closed form: P diag(cos k theta_i) P^T
    ev, P = np.linalg.eigh(Bh)
    for kk in [2, 3, 5]:
        c = [0.0] * 6
        c[kk] = 1.0
        Psi = (P * np.cos(kk * np.arccos(np.clip(ev, -1, 1)))) @ P.T
        want = Psi @ X if left else X @ Psi
        assert O.rel_fro(O.cpa_shrink(X, None, 6, lam=lam, coeffs=c), want) < 1e-12


# --- P9: SVD characterization (+ Jacobi pinned to numpy SVD, P16) ------------------------

@pytest.mark.parametrize("shape,kind", [((64, 48), "soft"), ((30, 40), "hard"), ((25, 25), "wsoft")])
def test_p9_svd_characterization(shape, kind):
    X = W.random_dense(*shape, seed=9)
    k = O.Kernel(kind, tau=3.0, w_c=15.0, w_eps=1e-6)
    Y, info = O.cpa_shrink(X, k, 20, T=60, return_info=True)
    Z = O.svd_characterization(X, info["coeffs"], info["lambda_max"])
    assert O.rel_fro(Y, Z) < 1e-12


def test_p16_jacobi_svd():
    for shape in [(64, 48), (48, 64), (10, 10), (1, 5), (5, 1)]:
        X = W.random_dense(*shape, seed=16)
        U, s, V = O.jacobi_svd(X)
        assert np.linalg.norm(X - (U * s) @ V.T) <= 1e-13 * np.linalg.norm(X)
        assert np.abs(U.T @ U - np.eye(len(s))).max() < 1e-13
        assert np.abs(V.T @ V - np.eye(len(s))).max() < 1e-13
        assert np.allclose(s, np.linalg.svd(X, compute_uv=False), rtol=1e-13, atol=1e-13)
    # diagonal / rank-1 exact
    U, s, V = O.jacobi_svd(np.diag([1.0, 4.0, 2.0]))
    assert list(s) == [4.0, 2.0, 1.0]


# --- P10: error vs exact shrinkage decreases with K on config 1 -----------------------------

def test_p10_c1_vs_exact_decreasing():
    X = W.gen_c1()
    cfg = W.CONFIGS["c1"]
    k = O.Kernel(**cfg["kernel"])
    exact = O.exact_shrink(X, k, 2.0)
    errs = [O.rel_fro(O.cpa_shrink(X, k, K, T=30), exact) for K in (5, 10, 20, 40)]
    assert all(a > b for a, b in zip(errs, errs[1:])), errs
    assert errs[2] <= 2e-2


# --- P11: hard with tau = 0 returns X ------------------------------------------------------------

def test_p11_hard_zero_tau_identity():
    X = W.random_dense(15, 9, seed=11)
    Y, info = O.cpa_shrink(X, O.Kernel("hard", tau=0.0), 25, T=30, return_info=True)
    assert info["coeffs"][0] == 2.0 and all(abs(v) < 1e-14 for v in info["coeffs"][1:])
    assert O.rel_fro(Y, X) < 1e-14


# --- P12: singular vectors preserved (YX^T, X^T Y symmetric) -----------------------------------

def test_p12_symmetry():
    X = W.gen_c1()
    Y = O.cpa_shrink(X, O.Kernel("soft", tau=2.0), 20, T=30)
    for M in (Y @ X.T, X.T @ Y):
        assert np.linalg.norm(M - M.T) <= 1e-12 * np.linalg.norm(M)


# --- P13: transpose covariance ---------------------------------------------------------------------

def test_p13_transpose():
    X = W.random_dense(13, 21, seed=13)
    k = O.Kernel("soft", tau=1.5)
    lam = 1.01 * np.linalg.norm(X, 2) ** 2
    assert O.rel_fro(O.cpa_shrink(X.T, k, 18, lam=lam), O.cpa_shrink(X, k, 18, lam=lam).T) < 1e-13


# --- P14: power-of-two scaling is bitwise --------------------------------------------------------------

def test_p14_pow2_bitwise():
    X = W.random_dense(20, 12, seed=14)
    a = O.cpa_shrink(X, O.Kernel("soft", tau=1.0), 15, T=30)
    b = O.cpa_shrink(2 * X, O.Kernel("soft", tau=2.0), 15, T=30)
    assert np.array_equal(2 * a, b)


# --- P15: power iteration ---------------------------------------------------------------------------

def test_p15_power_iteration():
    rng = np.random.default_rng(15)
    A = rng.standard_normal((40, 25))
    G = A.T @ A
    lam, hist = O.power_iteration(lambda v: G @ v, 25, 2000)
    assert abs(lam - np.linalg.eigvalsh(G)[-1]) < 1e-12 * lam
    assert all(b >= a * (1 - 1e-15) for a, b in zip(hist, hist[1:]))  # non-decreasing
    assert O.power_iteration(lambda v: 0 * v, 5, 10)[0] == 0.0


def test_p15b_power_iteration_finite_T_closed_form():
    """Every iterate, not only the converged value: for Phi = diag(a) and v_0 = 1_s / sqrt(s)
    (reading R6), v_{t-1} is proportional to Phi^{t-1} 1, so
    lambda_t = ||Phi v_{t-1}|| = sqrt(sum a_i^{2t} / sum a_i^{2t-2}) exactly (sum a_i^0 = s).
    Pins the start vector and the product count T (a v_0 or an off-by-one in T changes
    lambda_T); the reference values are exact rationals (fractions), not the oracle's arithmetic.
    Hand values for SPEC.md:61's diag(1, 2, 3): lambda_1 = sqrt(14/3), lambda_2 = sqrt(7)."""
    from fractions import Fraction
    lam1, _ = O.power_iteration(lambda v: np.diag([1.0, 2.0, 3.0]) @ v, 3, 1)
    assert abs(lam1 - math.sqrt(14.0 / 3.0)) <= 1e-15 * lam1
    lam2, hist2 = O.power_iteration(lambda v: np.diag([1.0, 2.0, 3.0]) @ v, 3, 2)
    assert abs(lam2 - math.sqrt(7.0)) <= 1e-15 * lam2 and len(hist2) == 2
    for a, T in (([1, 2, 3], 7), ([5, 1, 4, 4, 2], 12), ([3, 3, 1], 30), ([7, 6, 1, 2, 2, 5, 6], 40)):
        G = np.diag(np.array(a, dtype=np.float64))
        lam, hist = O.power_iteration(lambda v: G @ v, len(a), T)
        assert len(hist) == T
        for t, got in enumerate(hist, start=1):
            want = math.sqrt(Fraction(sum(x ** (2 * t) for x in a), sum(x ** (2 * t - 2) for x in a)))
            assert abs(got - want) <= 4e-15 * want, (a, t, got, want)
        assert lam == hist[-1]


# --- P17: the paper's block-diagonal D, closed form ------------------------------------------------------

@pytest.mark.parametrize("N,nb,copies", [(1000, 10, 1), (200, 4, 1), (120, 6, 4)])
def test_p17_block_diagonal(N, nb, copies):
    D = W.block_diag_D(N, nb, copies)
    p = N // nb
    s1, s2 = math.sqrt(copies) * (N - p / 2), math.sqrt(copies) * (p / 2)
    sv = np.linalg.svd(D, compute_uv=False)
    assert abs(sv[0] - s1) < 1e-9 * s1 and np.allclose(sv[1:nb], s2, rtol=1e-9) and sv[nb] < 1e-9 * s1
    k = O.Kernel("soft", tau=0.3, tau_relative=True)
    Y, info = O.cpa_shrink(D, k, 16, T=30, return_info=True)
    assert abs(info["lambda_hat"] - s1 ** 2) < 1e-12 * s1 ** 2  # exact after one step from 1/sqrt(s)
    lam, c = info["lambda_max"], info["coeffs"]
    q = np.ones(N) / math.sqrt(N)
    Pb = np.zeros((N, N))
    for b in range(nb):
        Pb[b * p:(b + 1) * p, b * p:(b + 1) * p] = 1.0 / p
    f1 = s1 * O.series_eval(c, lam, s1 ** 2)
    f2 = s2 * O.series_eval(c, lam, s2 ** 2)
    # D = sqrt(copies) [ (N - p/2) q q^T - (p/2)(P_b - q q^T) ] R with R the row-orthonormal copy map
    R = np.concatenate([np.eye(N)] * copies, axis=1) / math.sqrt(copies)
    want = (f1 * np.outer(q, q) - f2 * (Pb - np.outer(q, q))) @ R
    assert O.rel_fro(Y, want) < 1e-12
    for e in GOLDEN["block_diag_D"]:
        sv = np.linalg.svd(W.block_diag_D(e["N"], e["nblocks"]), compute_uv=False)
        assert abs(sv[0] - e["sigma"][0]) < 1e-9 and np.allclose(sv[1:e["rank"]], e["sigma"][1]), e["cite"]


# --- vector / sparse forms agree with Alg. 1 ---------------------------------------------------------------

def test_vector_forms_match_alg1():
    import scipy.sparse as sp
    k = O.Kernel("hard", tau=0.5, tau_relative=True)
    Xw = W.random_dense(12, 30, seed=21)
    Y = O.cpa_shrink(Xw, k, 14, T=100)
    Yc, _ = O.cpa_shrink_columns(Xw, [0, 7, 29], k, 14, T=100)
    assert O.rel_fro(Yc, Y[:, [0, 7, 29]]) < 1e-12
    Xt = Xw.T.copy()
    Yr, _ = O.cpa_shrink_rows(Xt, [3, 4], k, 14, T=100)
    assert O.rel_fro(Yr, Y.T[[3, 4], :]) < 1e-12
    # unconverged power iterations (T = 3, 7): the vector forms run the same T products from the
    # same 1/sqrt(s) on the same (Gram) side as Alg. 1, so lambda_hat and the columns still agree
    for T in (3, 7):
        Yt, it = O.cpa_shrink(Xw, k, 14, T=T, return_info=True)
        Yc, ic = O.cpa_shrink_columns(Xw, [0, 7, 29], k, 14, T=T)
        Yr, ir = O.cpa_shrink_rows(Xt, [3, 4], k, 14, T=T)
        for inf in (ic, ir):
            assert abs(inf["lambda_hat"] - it["lambda_hat"]) <= 1e-13 * it["lambda_hat"], (T, inf, it)
        assert O.rel_fro(Yc, Yt[:, [0, 7, 29]]) < 1e-12 and O.rel_fro(Yr, Yt.T[[3, 4], :]) < 1e-12
    # sparse: lambda from the m-side (XX^T) power iteration; use a given lambda to compare forms
    row_ptr, col, val = W.gen_c4(m=40, n=400, nnz=800)
    Xs = sp.csr_matrix((val, col, row_ptr), shape=(40, 400))
    lam = 1.01 * np.linalg.norm(Xs.toarray(), 2) ** 2
    Yd = O.cpa_shrink(Xs.toarray(), k, 14, lam=lam)
    Ys, _ = O.cpa_shrink_sparse_rows(Xs, [0, 5, 39], k, 14, lam=lam)
    assert O.rel_fro(Ys, Yd[[0, 5, 39], :]) < 1e-12
    # sparse power iteration on the m-side equals the dense one on the same side
    l1, _ = O.sparse_power_iteration(Xs, 50)
    Xd = Xs.toarray()
    l2, _ = O.power_iteration(lambda v: Xd @ (Xd.T @ v), 40, 50)
    assert abs(l1 - l2) < 1e-12 * l2


def test_degenerate_zero():
    Y, info = O.cpa_shrink(np.zeros((5, 3)), O.Kernel("soft", tau=1.0), 10, return_info=True)
    assert info["degenerate"] and not Y.any()


def test_generators_deterministic():
    assert np.array_equal(W.gen_c1(), W.gen_c1())
    X = W.gen_c1()
    assert X.shape == (64, 48)
    s = np.linalg.svd(X, compute_uv=False)
    assert s[4] > 10 and s[5] < 2  # rank-5 signal over 0.1 noise
    r, c, v = W.gen_c4(m=50, n=500, nnz=250)
    assert r[-1] == 250 and len(set(zip(np.repeat(np.arange(50), np.diff(r)), c))) == 250
    Xb = W.gen_c3(batch=4)
    assert Xb.dtype == np.float32 and Xb.shape == (4, 64, 64)


# ---- NEXT-2: Alg. 1 with the one-level Haar DWT (reading R22)

@pytest.mark.parametrize("n", [1, 2, 7, 8, 33])
def test_haar1_orthogonal(n):
    T = O.haar1_matrix(n)
    assert np.allclose(T @ T.T, np.eye(n), atol=1e-15) and np.allclose(T.T @ T, np.eye(n), atol=1e-15)
    # low-pass rows average adjacent pairs, high-pass rows difference them
    y = np.arange(n, dtype=float)
    t = T @ y
    nh = n // 2
    assert np.allclose(t[:nh], (y[0:2 * nh:2] + y[1:2 * nh:2]) / np.sqrt(2))
    assert np.allclose(t[n - nh:], (y[0:2 * nh:2] - y[1:2 * nh:2]) / np.sqrt(2))


@pytest.mark.parametrize("shape", [(20, 40), (40, 26), (31, 60)])
def test_transform_lowpass_signal_equals_identity_transform(shape):
    """A signal with no high-frequency content along the Gram index (pairwise equal rows /
    columns) has Phi_ = Phi = T G T^T exactly, and T^T H(T G T^T) T = H(G) for orthogonal T:
    the transform variant reduces to plain Alg. 1 (T = I)."""
    m, n = shape
    rng = np.random.default_rng(m * n)
    left = m <= n
    s = m if left else n
    base = rng.standard_normal(((s + 1) // 2, n if left else m))
    full = np.repeat(base, 2, axis=0)[:s]
    X = full if left else full.T
    kern = O.Kernel(kind="soft", tau=0.2, tau_relative=True)
    # the power iterations start from 1/sqrt(s) in different bases (T^T 1 != 1), so fix
    # Lambda to compare the series itself; lambda_hat then agrees to its convergence
    lam = 1.01 * float(np.linalg.eigvalsh(X @ X.T if left else X.T @ X)[-1])
    Yt = O.cpa_shrink_transform(X, kern, 12, lam=lam)
    Yi = O.cpa_shrink(X, kern, 12, lam=lam)
    assert O.rel_fro(Yt, Yi) <= 1e-12
    _, it = O.cpa_shrink_transform(X, kern, 12, T=300, return_info=True)
    assert abs(it["lambda_hat"] * 1.01 / lam - 1) <= 1e-9


@pytest.mark.parametrize("shape", [(16, 30), (30, 17), (9, 9)])
def test_transform_block_structure(shape):
    """In the transform basis Phi_ = blockdiag(G_L, 0) with G_L the Gram of the low-pass
    half A_L = T_L A, so H_hat(Phi_) = blockdiag(H_hat(G_L), h_hat(0) I): the result equals
    T_L^T H_hat(G_L) A_L + h_hat(0) T_H^T A_H, with h_hat(0) = c_0/2 + sum_k c_k (-1)^k
    (psi_k(-1) = (-1)^k)."""
    X = np.random.default_rng(5).standard_normal(shape)
    m, n = shape
    left = m <= n
    A = X if left else X.T
    s = A.shape[0]
    Tm = O.haar1_matrix(s)
    nl = s - s // 2
    AL, AH = Tm[:nl] @ A, Tm[nl:] @ A
    kern = O.Kernel(kind="soft", tau=0.3, tau_relative=True)
    K = 9
    Y, info = O.cpa_shrink_transform(X, kern, K, T=80, return_info=True)
    c = info["coeffs"]
    lam = info["lambda_max"]
    # H_hat(G_L) A_L by the vector form at the same Lambda and coefficients
    GL = AL @ AL.T
    YL = O.cpa_apply_vectors(lambda V: GL @ V, AL, c, lam)
    h0 = 0.5 * c[0] + sum(c[k] * (-1) ** k for k in range(1, K))
    want = Tm[:nl].T @ YL + h0 * (Tm[nl:].T @ AH)
    want = want if left else want.T
    assert O.rel_fro(Y, want) <= 1e-12
    assert abs(O.series_eval(c, lam, 0.0) - h0) <= 1e-12 * max(1.0, abs(h0))


# ---- NEXT-3: ADMM recovery (synthetic D of PAPER.md:1095-1100)

@pytest.mark.parametrize("n", [1, 2, 5, 16])
def test_dct2_orthonormal(n):
    C = O.dct2_matrix(n)
    assert np.allclose(C @ C.T, np.eye(n), atol=1e-14)
    # DCT of a constant vector is concentrated in the DC coefficient
    y = np.full(n, 3.0)
    assert np.allclose((C @ y)[1:], 0.0, atol=1e-13) and abs((C @ y)[0] - 3.0 * np.sqrt(n)) < 1e-12


def test_synthetic_D_spectrum():
    # sigma_1 = N - p/2, sigma_2..rank = p/2, rank exactly `rank`
    N, r = 120, 6
    p = N // r
    s = np.linalg.svd(O.synthetic_D(N, r), compute_uv=False)
    assert abs(s[0] - (N - p / 2)) < 1e-9 and np.allclose(s[1:r], p / 2, atol=1e-9) and s[r] < 1e-9


def _svd_soft(X, tau):
    U, sv, Vt = np.linalg.svd(X, full_matrices=False)
    return (U * np.maximum(sv - tau, 0.0)) @ Vt


def test_admm_exact_shrink_recovers_full_observation():
    """With every entry observed and tiny weights, the ADMM fixed point is the data itself:
    z3 pins l to D on all entries."""
    D = O.synthetic_D(60, 5)
    mask = np.ones_like(D)
    kern = O.Kernel(kind="soft", tau=0.05, tau_relative=False)
    L = O.admm_recover(D, mask, kern, 10, 30, rho=20.0, eta=0.0, max_iter=400, tol=1e-9,
                       shrink=lambda X: _svd_soft(X, 0.05))
    assert O.rel_fro(L, D) <= 1e-3


def test_admm_cpa_tracks_exact_on_corrupted_D():
    """10% of D zeroed: the CPA-ADMM recovery is close to the exact-shrinkage
    ADMM recovery and much closer to D than the corrupted input (the paper's Fig. 9 claim)."""
    rng = np.random.default_rng(0)
    D = O.synthetic_D(80, 4)
    mask = (rng.random(D.shape) >= 0.10).astype(float)
    Dobs = D * mask
    kern = O.Kernel(kind="soft", tau=1.0, tau_relative=False)
    Lc = O.admm_recover(Dobs, mask, kern, 20, 30, rho=1.0, eta=0.01, max_iter=300, tol=1e-4)
    Le = O.admm_recover(Dobs, mask, kern, 20, 30, rho=1.0, eta=0.01, max_iter=300, tol=1e-4,
                        shrink=lambda X: _svd_soft(X, 1.0))
    assert O.rel_fro(Lc, D) < 0.5 * O.rel_fro(Dobs, D)
    assert O.rel_fro(Lc, Le) < 0.05


# ---- NEXT-2 DCT + epsilon thresholding

def test_threshold_components_topk_and_abs():
    Phi = np.array([[4.0, -3.0, 0.5], [-3.0, 2.0, -1.0], [0.5, -1.0, 1.5]])
    P1, t1 = O.threshold_components(Phi, "topk", 4)      # |.| sorted: 4, 3, 3, 2, 1.5, 1, 1, .5, .5
    assert t1 == 2.0 and np.count_nonzero(P1) == 4 and np.array_equal(P1, P1.T)
    P2, t2 = O.threshold_components(Phi, "abs", 1.0)
    assert t2 == 1.0 and np.count_nonzero(P2) == 7 and P2[0, 2] == 0.0
    P3, _ = O.threshold_components(Phi, None)
    assert P3 is Phi


@pytest.mark.parametrize("shape", [(24, 40), (40, 24)])
def test_dct_keep_all_equals_identity_transform(shape):
    """T orthogonal and nothing thresholded: T^T H(T G T^T) T = H(G), so the DCT variant
    reduces to plain Alg. 1 at a fixed Lambda."""
    X = np.random.default_rng(9).standard_normal(shape)
    m, n = shape
    kern = O.Kernel(kind="soft", tau=0.3, tau_relative=True)
    lam = 1.01 * float(np.linalg.eigvalsh(X @ X.T if m <= n else X.T @ X)[-1])
    Yd = O.cpa_shrink_transform(X, kern, 10, lam=lam, transform="dct")
    Yi = O.cpa_shrink(X, kern, 10, lam=lam)
    assert O.rel_fro(Yd, Yi) <= 1e-12


def test_dct_thresholded_is_exact_shrink_of_the_thresholded_gram():
    """With components thresholded the method is Alg. 1 on Phi_ exactly: its result equals
    T^T H_hat(Phi_) T applied to B, where H_hat(Phi_) is evaluated spectrally (eigh of Phi_,
    the series at each eigenvalue) -- an independent route to the same quantity."""
    X = np.random.default_rng(4).standard_normal((30, 50))
    kern = O.Kernel(kind="hard", tau=0.4, tau_relative=True)
    K = 11
    Y, info = O.cpa_shrink_transform(X, kern, K, T=200, return_info=True, transform="dct",
                                      eps_mode="topk", eps=120)
    Tm = O.dct2_matrix(30)
    Phi_, _ = O.threshold_components(Tm @ (X @ X.T) @ Tm.T, "topk", 120)
    w, V = np.linalg.eigh(Phi_)
    hh = np.array([O.series_eval(info["coeffs"], info["lambda_max"], x) for x in w])
    H = (V * hh) @ V.T
    assert O.rel_fro(Y, Tm.T @ H @ Tm @ X) <= 1e-11
    assert info["nnz"] >= 120


# ---- NEXT-2 block DCT (block diagonal DCT with 8 x 8 blocks; reading R24)

@pytest.mark.parametrize("n", [1, 5, 8, 16, 21])
def test_block_dct_structure(n):
    T = O.dct2_block_matrix(n)
    assert np.allclose(T @ T.T, np.eye(n), atol=1e-14)
    for i0 in range(0, n, 8):            # each diagonal block is the DCT-II of its size...
        w = min(8, n - i0)
        assert np.array_equal(T[i0:i0 + w, i0:i0 + w], O.dct2_matrix(w))
        T[i0:i0 + w, i0:i0 + w] = 0.0
    assert not T.any()                   # ...and nothing couples two blocks
    # an 8-periodic signal constant on every block has only DC coefficients per block
    y = np.repeat(np.arange(1.0, 4.0), 8)
    c = O.dct2_block_matrix(24) @ y
    assert np.allclose(np.delete(c, [0, 8, 16]), 0.0, atol=1e-13)


@pytest.mark.parametrize("shape", [(20, 44), (44, 20)])
def test_block_dct_keep_all_equals_identity_transform(shape):
    X = np.random.default_rng(2).standard_normal(shape)
    m, n = shape
    kern = O.Kernel(kind="soft", tau=0.3, tau_relative=True)
    lam = 1.01 * float(np.linalg.eigvalsh(X @ X.T if m <= n else X.T @ X)[-1])
    Yb = O.cpa_shrink_transform(X, kern, 10, lam=lam, transform="dct8")
    assert O.rel_fro(Yb, O.cpa_shrink(X, kern, 10, lam=lam)) <= 1e-12


def test_block_dct_thresholded_is_exact_shrink_of_the_thresholded_gram():
    X = np.random.default_rng(6).standard_normal((28, 45))
    kern = O.Kernel(kind="soft", tau=0.2, tau_relative=True)
    K = 9
    Y, info = O.cpa_shrink_transform(X, kern, K, T=200, return_info=True, transform="dct8",
                                      eps_mode="abs", eps=1.5)
    Tm = O.dct2_block_matrix(28)
    Phi_, _ = O.threshold_components(Tm @ (X @ X.T) @ Tm.T, "abs", 1.5)
    w, V = np.linalg.eigh(Phi_)
    hh = np.array([O.series_eval(info["coeffs"], info["lambda_max"], x) for x in w])
    assert O.rel_fro(Y, Tm.T @ ((V * hh) @ V.T) @ Tm @ X) <= 1e-11
    assert 0 < info["nnz"] < 28 * 28


# ---- NEXT-2 adaptive epsilon of the ADMM (eq. recommendation_epsilon)

def test_epsilon_schedule_k_breakpoints():
    n = 1000                                     # k1..k3 of PAPER.md:1074-1076 at n = 1000
    assert O.epsilon_schedule_k(float("inf"), n) == 50
    assert O.epsilon_schedule_k(0.031, n) == 50
    assert O.epsilon_schedule_k(0.03, n) == 150   # E_l >= E > E_m
    assert O.epsilon_schedule_k(6.01e-4, n) == 150
    assert O.epsilon_schedule_k(6e-4, n) == 500   # otherwise
    assert O.epsilon_schedule_k(0.0, n) == 500
    assert O.epsilon_schedule_k(1.0, 10) == 1     # never below one component


def test_admm_adaptive_eps_uses_the_schedule(monkeypatch):
    """The adaptive ADMM thresholds iteration t's shrinkage at the schedule's k for the error of
    iteration t - 1 (E = inf first): the k passed to every shrink call is recorded and checked
    against the returned error history."""
    from oracle import cpa_oracle as CO
    rng = np.random.default_rng(3)
    D = O.synthetic_D(200, 4)
    mask = (rng.random(D.shape) >= 0.1).astype(float)
    kern = O.Kernel(kind="soft", tau=1.0, tau_relative=False)
    seen = []
    real = CO.cpa_shrink_transform
    def spy(X, *a, **kw):
        seen.append((kw.get("eps_mode"), kw.get("eps"), kw.get("transform")))
        return real(X, *a, **kw)
    monkeypatch.setattr(CO, "cpa_shrink_transform", spy)
    L, hist = O.admm_recover(D * mask, mask, kern, 8, 30, rho=1.0, eta=0.01, max_iter=5, tol=0.0,
                             transform="dct", adaptive_eps=True, return_history=True)
    assert len(seen) == len(hist) == 5
    want = [O.epsilon_schedule_k(E, 200) for E in [float("inf")] + hist[:-1]]
    assert [k for _, k, _ in seen] == want
    assert all(mode == "topk" and tr == "dct" for mode, _, tr in seen)
    assert want[0] == 2 and np.isfinite(L).all()


# --- weighted soft (BASELINE configs[2]) and relative tau: pins independent of h_response -----

def test_golden_wsoft_eval():
    # hand-computed values of eq. filter_response_ours, weighted-soft member
    for e in GOLDEN["wsoft_eval"]:
        k = O.Kernel("wsoft", w_c=e["w_c"], w_shift=e["w_shift"], w_eps=e["w_eps"])
        assert abs(O.h_response(k, e["x"], 0.0) - e["h"]) <= 1e-15, e["cite"]
        assert abs(O.g_response(k, math.sqrt(e["x"]), 0.0) - e["g"]) <= 1e-14 * max(1.0, e["g"]), e["cite"]


def test_wsoft_constant_weight_is_soft():
    # With w_shift >= every Gram eigenvalue the weight is the constant w_c / w_eps (the paper's
    # constant-weight case, Fig. 3(b)/(d) captions), so weighted soft must be soft
    # shrinkage with tau = w_c / w_eps -- bitwise, every coefficient and output.
    X = W.random_dense(23, 17, seed=31)
    soft = O.Kernel("soft", tau=3.0)
    wsoft = O.Kernel("wsoft", w_c=3.0, w_shift=1e12, w_eps=1.0)
    Ys, i1 = O.cpa_shrink(X, soft, 18, T=60, return_info=True)
    Yw, i2 = O.cpa_shrink(X, wsoft, 18, T=60, return_info=True)
    assert i1["coeffs"] == i2["coeffs"]
    assert np.array_equal(Ys, Yw)
    # and the batched loop (c3's engine in the oracle) agrees with it
    Xb = np.stack([X[:16, :16], 2 * X[:16, :16]])
    Yb, _ = O.cpa_shrink_batched(Xb, wsoft, 18, T=60)
    for b in range(2):
        assert np.array_equal(Yb[b], O.cpa_shrink(Xb[b], soft, 18, T=60))


def test_p5_node_exact_wsoft_closed_form():
    # Singular values at the Chebyshev nodes: the K-point rule interpolates h exactly there
    # (PAPER.md:233), so Y = U g(Sigma) V^T with the closed form of the weighted-soft singular-value
    # response g(sigma) = max(sigma - w_c/(sigma + w_eps), 0) (w_shift = 0; PAPER.md:510-512, 520:
    # g(sqrt x) = sqrt(x) h(x)) -- built here without h_response.
    rng = np.random.default_rng(55)
    K, lam, m, n = 12, 144.0, 17, 12
    nodes = [lam / 2 * (math.cos(math.pi * (l - 0.5) / K) + 1) for l in range(1, K + 1)]
    d = np.sqrt(np.array(nodes))
    U, V = _orth(m, rng)[:, :n], _orth(n, rng)
    X = (U * d) @ V.T
    w_c, w_eps = 22.4, 1e-6
    g = np.array([max(s - w_c / (s + w_eps), 0.0) for s in d])
    assert (g == 0).sum() >= 3 and (g > 0).sum() >= 3      # both branches exercised
    want = (U * g) @ V.T
    Y = O.cpa_shrink(X, O.Kernel("wsoft", w_c=w_c, w_eps=w_eps), K, lam=lam)
    assert O.rel_fro(Y, want) < 1e-12


def test_relative_tau_is_tau_times_sigma_max():
    # Reading R7: a relative threshold is tau * sigma_max_hat with sigma_max_hat = sqrt(lambda_hat)
    # (before the 1.01 safety factor).  At a converged power iteration lambda_hat = sigma_1(X)^2,
    # so the threshold must equal tau * sigma_1 from an independent SVD (numpy LAPACK).
    rng = np.random.default_rng(71)
    U, V = _orth(30, rng)[:, :20], _orth(20, rng)
    sv = np.linspace(10.0, 1.0, 20)
    X = (U * sv) @ V.T
    for kind in ("soft", "hard"):
        k = O.Kernel(kind, tau=0.37, tau_relative=True)
        Y, info = O.cpa_shrink(X, k, 16, T=400, return_info=True)
        s1 = np.linalg.svd(X, compute_uv=False)[0]
        assert abs(info["tau"] - 0.37 * s1) <= 1e-12 * s1
        assert abs(info["sigma_max_hat"] - s1) <= 1e-12 * s1
        assert abs(info["lambda_max"] - 1.01 * s1 * s1) <= 1e-12 * s1 * s1
        # the output equals the absolute-tau shrinkage at that threshold and Lambda_max
        Ya = O.cpa_shrink(X, O.Kernel(kind, tau=0.37 * s1), 16, lam=1.01 * s1 * s1)
        assert O.rel_fro(Y, Ya) < 1e-12
    # scale invariance of a relative threshold: shrink(a X) = a shrink(X)
    k = O.Kernel("soft", tau=0.37, tau_relative=True)
    assert O.rel_fro(O.cpa_shrink(3.0 * X, k, 16, T=400), 3.0 * O.cpa_shrink(X, k, 16, T=400)) < 1e-12


# ---- NEXT-3 ADMM steps against their definitions (eq. admm_algorithm_inp)

def test_admm_steps_match_their_definitions():
    """Each ADMM sub-step against what defines it, computed another way:
    z2 = prox of (eta/rho)|.| -- argmin_z eta |z| + rho/2 (z - v)^2 by bounded scalar minimisation;
    z4 = Euclidean projection onto [0, 1] -- argmin over [0, 1] the same way;
    l  = least-squares solution of K l = z - u with K = [I; Psi; diag(mask); I] assembled as an
         explicit matrix (Psi = C_m (.) C_n^T on the row-major vec: kron(C_m, C_n)) -- numpy lstsq."""
    from scipy.optimize import minimize_scalar
    rng = np.random.default_rng(11)
    eta, rho = 0.7, 2.5                                  # eta / rho = 0.28, eta * rho = 1.75
    v = rng.uniform(-2.0, 2.0, 40)
    z2 = O.admm_z2_step(v, eta, rho)
    for vi, zi in zip(v, z2):
        r = minimize_scalar(lambda z: eta * abs(z) + 0.5 * rho * (z - vi) ** 2, bounds=(-3, 3), method="bounded",
                            options={"xatol": 1e-12})
        assert abs(zi - r.x) < 1e-7, (vi, zi, r.x)
    v4 = rng.uniform(-1.0, 2.0, 40)
    z4 = O.admm_z4_step(v4)
    for vi, zi in zip(v4, z4):
        r = minimize_scalar(lambda z: (z - vi) ** 2, bounds=(0.0, 1.0), method="bounded", options={"xatol": 1e-12})
        assert abs(zi - r.x) < 1e-6, (vi, zi, r.x)
    m, n = 3, 4
    Cm, Cn = O.dct2_matrix(m), O.dct2_matrix(n)
    w = (rng.random((m, n)) < 0.6).astype(float)
    zu = [rng.standard_normal((m, n)) for _ in range(4)]
    Kmat = np.vstack([np.eye(m * n), np.kron(Cm, Cn), np.diag(w.ravel()), np.eye(m * n)])
    rhs = np.concatenate([z.ravel() for z in zu])
    l_ls = np.linalg.lstsq(Kmat, rhs, rcond=None)[0].reshape(m, n)
    l = O.admm_l_step(zu[0], zu[1], zu[2], zu[3], w, lambda S: Cm.T @ S @ Cn)
    assert np.allclose(l, l_ls, atol=1e-12), np.abs(l - l_ls).max()


def test_rel_fro_is_relative_to_the_reference():
    """The parity metric (reading R16): ||A - B||_F / ||B||_F, B the oracle's output -- hand values."""
    assert abs(O.rel_fro(np.array([[3.0, 4.0]]), np.array([[0.0, 5.0]])) - math.sqrt(10.0) / 5.0) < 1e-15
    assert O.rel_fro(np.array([2.0]), np.array([1.0])) == 1.0
    assert O.rel_fro(np.array([1.0]), np.array([0.0])) == 1.0     # zero reference: the absolute norm
