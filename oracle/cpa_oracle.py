"""Plain fp64 CPU oracle of CPA singular-value shrinkage (arXiv 1705.07112).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Nothing in the product
path imports this file.

Notation follows the paper: K is the approximation order alpha (number of
coefficients c_0..c_{K-1}), h is the eigenvalue response, g the singular-value
response with h(x) = g(sqrt(x))/sqrt(x), Lambda_max the bound on
the Gram spectrum.  The transform T of Alg. 1 is the identity and the
component threshold epsilon is 0 on this path (reading R5).

Library primitives used as single steps (allowed by the task): numpy matmul,
numpy vector norms, scipy.sparse matrix-vector products.  Everything else is
written out in the paper's order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Kernel", "h_response", "g_response", "resolve_tau", "chebyshev_psi",
    "chebyshev_psi_recurrence", "chebyshev_coefficients", "kernel_coefficients",
    "series_eval", "gram", "power_iteration", "cpa_shrink", "cpa_apply_vectors",
    "cpa_shrink_columns", "cpa_shrink_rows", "cpa_shrink_batched",
    "sparse_power_iteration", "cpa_shrink_sparse_rows", "jacobi_svd",
    "exact_shrink", "svd_characterization", "rel_fro", "haar1_matrix", "cpa_shrink_transform",
    "dct2_matrix", "dct2_block_matrix", "synthetic_D", "admm_recover", "threshold_components",
    "epsilon_schedule_k", "admm_l_step", "admm_z2_step", "admm_z4_step",
    "DEFAULT_SAFETY", "DEGENERATE_LAMBDA",
]

# Lambda_max safety factor (reading R6): power
# iteration approaches lambda_max from below, and psi_k grows outside [-1,1]
# (PAPER.md:230), so the bound actually used is 1.01 * lambda_hat.
DEFAULT_SAFETY = 1.01
# A Gram with lambda_hat at or below this is the zero matrix: Y = 0
# (reading R17).
DEGENERATE_LAMBDA = 1e-300


# ---------------------------------------------------------------------------
# Shrinkage responses  (PAPER.md:454-463 eq. ideal_filter_response,
#                       PAPER.md:496-519 eq. filter_response_ours)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Kernel:
    """One member of the paper's generic response family h(x; w(x)/rho, tau).

    kind = "hard":  h(x; 0, tau)          -> keep sigma > tau unchanged.
    kind = "soft":  h(x; 1/rho, 1/rho)    -> g(sigma) = max(sigma - tau, 0), tau = 1/rho.
    kind = "wsoft": h(x; w(x)/rho, w(x)/rho) with the weight
                    w(x) = w_c / (sqrt(max(x - w_shift, 0)) + w_eps)   (reading R10).
    tau_relative: tau is a multiple of the power-iteration estimate of sigma_max
    (BASELINE configs 2, 4, 5; reading R7).
    """

    kind: str
    tau: float = 0.0
    tau_relative: bool = False
    w_c: float = 0.0
    w_shift: float = 0.0
    w_eps: float = 0.0


def resolve_tau(kernel: Kernel, sigma_max_hat: float) -> float:
    """Absolute threshold: tau * sigma_max_hat if relative (reading R7)."""
    return kernel.tau * sigma_max_hat if kernel.tau_relative else kernel.tau


def h_response(kernel: Kernel, x: float, tau: float) -> float:
    """h(x) of PAPER.md:497-502, evaluated at one Gram eigenvalue x >= 0.

    The zero branch is tested first so sqrt(x) = 0 never divides
    (reading R8: the comparison is strict, sqrt(x) = tau -> 0).
    """
    r = math.sqrt(x)
    if kernel.kind == "hard":            # h(x; 0, tau_hard)
        return 1.0 if r > tau else 0.0
    if kernel.kind == "soft":            # h(x; 1/rho, 1/rho)
        return (r - tau) / r if r > tau else 0.0
    if kernel.kind == "wsoft":           # h(x; w(x)/rho, w(x)/rho)
        w = kernel.w_c / (math.sqrt(max(x - kernel.w_shift, 0.0)) + kernel.w_eps)
        return (r - w) / r if r > w else 0.0
    raise ValueError(f"unknown kernel kind {kernel.kind!r}")


def g_response(kernel: Kernel, sigma: float, tau: float) -> float:
    """g(sigma) = sigma * h(sigma^2), g(0) = 0."""
    if sigma <= 0.0:
        return 0.0
    return sigma * h_response(kernel, sigma * sigma, tau)


# ---------------------------------------------------------------------------
# Chebyshev machinery
# ---------------------------------------------------------------------------

def chebyshev_psi(k: int, x: float) -> float:
    """psi_k(x) = cos(k arccos x), PAPER.md:158 eq. chebychev_polynomial."""
    return math.cos(k * math.acos(x))


def chebyshev_psi_recurrence(k: int, x: float) -> float:
    """psi_k by the three-term recurrence, PAPER.md:164-165 eq. chebyche2."""
    if k == 0:
        return 1.0
    p_prev, p = 1.0, x
    for _ in range(2, k + 1):
        p_prev, p = p, 2.0 * x * p - p_prev
    return p


def chebyshev_coefficients(h, K: int, lam: float) -> list:
    """c_k of PAPER.md:233 eq. chebychev_coeff_shifted, k = 0..K-1.

    c_k = (2/K) sum_{l=1}^{K} cos(k theta(l)) h( (lam/2)(cos theta(l) + 1) ),
    theta(l) = pi (l - 1/2) / K.   ``h`` is any callable.
    """
    if K < 1:
        raise ValueError("K must be >= 1")
    theta = [math.pi * (l - 0.5) / K for l in range(1, K + 1)]
    hv = [h(lam / 2.0 * (math.cos(t) + 1.0)) for t in theta]
    c = []
    for k in range(K):
        acc = 0.0
        for l in range(K):
            acc += math.cos(k * theta[l]) * hv[l]
        c.append(2.0 / K * acc)
    return c


def kernel_coefficients(kernel: Kernel, K: int, lam: float, sigma_max_hat: float) -> list:
    """Alg. 1 line 4 for one of the paper's kernels."""
    tau = resolve_tau(kernel, sigma_max_hat)
    return chebyshev_coefficients(lambda x: h_response(kernel, x, tau), K, lam)


def series_eval(c, lam: float, x: float) -> float:
    """h_hat(x) = c_0/2 + sum_{k>=1} c_k psi_k(2x/lam - 1)."""
    xh = 2.0 * x / lam - 1.0
    acc = 0.5 * c[0]
    for k in range(1, len(c)):
        acc += c[k] * chebyshev_psi_recurrence(k, xh)
    return acc


# ---------------------------------------------------------------------------
# Gram and Lambda_max  (Alg. 1 lines 1-3)
# ---------------------------------------------------------------------------

def gram(B: np.ndarray) -> np.ndarray:
    """Phi = B^T B (Alg. 1 line 1 with T = I)."""
    B = np.asarray(B, dtype=np.float64)
    return B.T @ B


def power_iteration(apply_phi, s: int, T: int):
    """Power iteration for Lambda_max (Alg. 1 line 3; reading R6).

    v_0 = 1_s / sqrt(s); for t = 1..T: u_t = Phi v_{t-1}, lam_t = ||u_t||_2,
    v_t = u_t / lam_t.  Returns (lam_T, [lam_1..lam_T]).  A zero Gram stops
    early with lam = 0.
    """
    v = np.full(s, 1.0 / math.sqrt(s))
    hist = []
    lam = 0.0
    for _ in range(T):
        u = apply_phi(v)
        lam = float(np.linalg.norm(u))
        hist.append(lam)
        if lam <= DEGENERATE_LAMBDA:
            return 0.0, hist
        v = u / lam
    return lam, hist


def _lambda_and_sigma(lam_hat_fn, lam_override, safety):
    """Lambda_max = safety * lambda_hat; sigma_max_hat = sqrt(lambda_hat) (reading R7).

    With an override Lambda_max given, lambda_hat := Lambda_max / safety.
    """
    if lam_override is not None and lam_override > 0:
        lam = float(lam_override)
        lam_hat = lam / safety
    else:
        lam_hat = lam_hat_fn()
        lam = safety * lam_hat
    return lam, lam_hat, math.sqrt(max(lam_hat, 0.0))


# ---------------------------------------------------------------------------
# Algorithm 1 with T = I, epsilon = 0
# ---------------------------------------------------------------------------

def cpa_shrink(X, kernel: Kernel | None, K: int, T: int = 30, safety: float = DEFAULT_SAFETY,
               lam: float | None = None, coeffs=None, return_info: bool = False):
    """CPA-based singular value shrinkage G_hat(X), Algorithm 1 of PAPER.md:354-373.

    The paper states Alg. 1 for B in R^{m x n} with m > n and
    the Gram B^T B.  For a wide X (m <= n) the oracle runs Alg. 1 on B = X^T and
    returns the transpose, i.e. the Gram is always on the
    smaller side (reading R3).  ``coeffs`` overrides line 4 (raw-coefficient
    pins); ``lam`` overrides line 3.
    """
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError("X must be 2-D")
    m, n = X.shape
    if m <= n:
        Yt, info = _alg1(X.T, kernel, K, T, safety, lam, coeffs)
        info["side"] = "left"
        Y = Yt.T
    else:
        Y, info = _alg1(X, kernel, K, T, safety, lam, coeffs)
        info["side"] = "right"
    return (Y, info) if return_info else Y


def _alg1(B, kernel, K, T, safety, lam_override, coeffs):
    if K < 2 and coeffs is None:
        raise ValueError("K must be >= 2")
    n = B.shape[1]
    # line 1: Phi <- T B^T B T^T with T = I
    Phi = gram(B)
    # line 2: Phi_ <- Phi thresholded at epsilon = 0: |Phi_ij| >= 0 keeps all
    Phi_ = Phi
    # line 3: Lambda_max of Phi_
    lam, lam_hat, sig_hat = _lambda_and_sigma(
        lambda: power_iteration(lambda v: Phi_ @ v, n, T)[0], lam_override, safety)
    info = {"lambda_hat": lam_hat, "lambda_max": lam, "sigma_max_hat": sig_hat, "degenerate": False}
    if lam_hat <= DEGENERATE_LAMBDA:
        info["degenerate"] = True
        return np.zeros_like(B), info
    # line 4: coefficients
    if coeffs is None:
        c = kernel_coefficients(kernel, K, lam, sig_hat)
        info["tau"] = resolve_tau(kernel, sig_hat)
    else:
        c = [float(v) for v in coeffs]
    info["coeffs"] = c
    Kc = len(c)
    # line 5: B_hat <- (2 / Lambda_max) Phi_ - Id
    Id = np.eye(n)
    Bh = (2.0 / lam) * Phi_ - Id
    # line 6: Psi_0 <- Id, Psi_1 <- B_hat
    Psi_km2, Psi_km1 = Id, Bh
    # line 7: H <- c_0/2 Psi_0 + c_1 Psi_1
    H = 0.5 * c[0] * Psi_km2
    if Kc > 1:
        H = H + c[1] * Psi_km1
    # lines 8-11
    for k in range(2, Kc):
        Psi_k = 2.0 * (Bh @ Psi_km1) - Psi_km2
        H = H + c[k] * Psi_k
        Psi_km2, Psi_km1 = Psi_km1, Psi_k
    # line 12: G_hat(B) <- B T^T H T with T = I
    return B @ H, info


# ---------------------------------------------------------------------------
# Alg. 1 with a sparsifying transform T (NEXT-2 / reading R22)
# ---------------------------------------------------------------------------

def haar1_matrix(n: int) -> np.ndarray:
    """One-level Haar DWT as an n x n orthogonal matrix T (forward transform y -> T y,
    PAPER.md:321-322, 628-630).  Rows 0..ceil(n/2)-1 are the low-pass (scaling)
    coefficients (y_{2i} + y_{2i+1})/sqrt 2 -- for odd n the last sample is its own
    low-pass coefficient -- and the remaining floor(n/2) rows the high-pass (wavelet)
    coefficients (y_{2i} - y_{2i+1})/sqrt 2."""
    nh = n // 2
    nl = n - nh
    T = np.zeros((n, n))
    r = 1.0 / math.sqrt(2.0)
    for i in range(nh):
        T[i, 2 * i] = r
        T[i, 2 * i + 1] = r
        T[nl + i, 2 * i] = r
        T[nl + i, 2 * i + 1] = -r
    if nl > nh:
        T[nl - 1, n - 1] = 1.0
    return T


def threshold_components(Phi, eps_mode=None, eps=0.0):
    """Line 2 of Alg. 1, eq. threshold_components: keep Phi_ij with
    |Phi_ij| >= epsilon, zero the rest.  eps_mode None keeps all; "abs": epsilon = eps;
    "topk": epsilon = K(|Phi|, k), the k-th largest |Phi_ij|, k = int(eps)
    (every entry tied with the k-th largest is kept).  Returns (Phi_, epsilon)."""
    if eps_mode is None:
        return Phi, 0.0
    A = np.abs(Phi)
    if eps_mode == "abs":
        thr = float(eps)
    elif eps_mode == "topk":
        k = int(eps)
        flat = np.sort(A.ravel())[::-1]
        thr = float(flat[min(max(k, 1), flat.size) - 1])
    else:
        raise ValueError(eps_mode)
    return np.where(A >= thr, Phi, 0.0), thr


def cpa_shrink_transform(X, kernel: Kernel, K: int, T: int = 30, safety: float = DEFAULT_SAFETY,
                         lam: float | None = None, return_info: bool = False, transform: str = "haar1",
                         eps_mode=None, eps: float = 0.0):
    """Algorithm 1 with a sparsifying orthogonal transform T of the Gram
    index:

      line 1  Phi  <- T B^T B T^T
      line 2  Phi_ <- Phi thresholded (eq. threshold_components); for the
              one-level Haar DWT the high-frequency rows and columns are zeroed first
              (reading R22)
      lines 3-11 as in cpa_shrink, on Phi_ (s x s; Psi_0 = Id over the whole index space)
      line 12 G_hat(B) <- B T^T H_hat(Phi_) T

    transform: "haar1" (haar1_matrix), "dct" (dct2_matrix, orthonormal DCT-II) or "dct8"
    (dct2_block_matrix: the 8 x 8 block DCT of PAPER.md:947).
    Orientation as cpa_shrink: a wide X (m <= n) runs on B = X^T (Gram X X^T)."""
    X = np.asarray(X, dtype=np.float64)
    m, n = X.shape
    B = X.T if m <= n else X
    s = B.shape[1]
    Tm = {"haar1": haar1_matrix, "dct": dct2_matrix, "dct8": dct2_block_matrix}[transform](s)
    # line 1
    Phi = Tm @ gram(B) @ Tm.T
    # line 2
    Phi_ = Phi.copy()
    if transform == "haar1":
        nl = s - s // 2
        Phi_[nl:, :] = 0.0
        Phi_[:, nl:] = 0.0
    Phi_, thr = threshold_components(Phi_, eps_mode, eps)
    # line 3
    lam_, lam_hat, sig_hat = _lambda_and_sigma(
        lambda: power_iteration(lambda v: Phi_ @ v, s, T)[0], lam, safety)
    info = {"lambda_hat": lam_hat, "lambda_max": lam_, "sigma_max_hat": sig_hat, "degenerate": False,
            "epsilon": thr, "nnz": int(np.count_nonzero(Phi_))}
    if lam_hat <= DEGENERATE_LAMBDA:
        info["degenerate"] = True
        return (np.zeros_like(X), info) if return_info else np.zeros_like(X)
    # line 4
    c = kernel_coefficients(kernel, K, lam_, sig_hat)
    info["tau"] = resolve_tau(kernel, sig_hat)
    info["coeffs"] = c
    # lines 5-11
    Id = np.eye(s)
    Bh = (2.0 / lam_) * Phi_ - Id
    Psi_km2, Psi_km1 = Id, Bh
    H = 0.5 * c[0] * Psi_km2 + c[1] * Psi_km1
    for k in range(2, K):
        Psi_k = 2.0 * (Bh @ Psi_km1) - Psi_km2
        H = H + c[k] * Psi_k
        Psi_km2, Psi_km1 = Psi_km1, Psi_k
    # line 12
    Y = B @ Tm.T @ H @ Tm
    Y = Y.T if m <= n else Y
    return (Y, info) if return_info else Y


# ---------------------------------------------------------------------------
# NEXT-3: ADMM recovery with CPA shrinkage as the nuclear-norm prox
# (PAPER.md:657-692 ADMM, 1193-1214 eq. admm_algorithm_inp, 1095-1100 synthetic data)
# ---------------------------------------------------------------------------

def dct2_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II matrix C (C y = DCT of y; PAPER.md:1185 uses DCT matrices T1, T2):
    C[k, j] = a_k cos(pi (2j + 1) k / (2n)), a_0 = sqrt(1/n), a_k = sqrt(2/n)."""
    k = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    C = np.cos(np.pi * (2 * j + 1) * k / (2 * n)) * math.sqrt(2.0 / n)
    C[0, :] = math.sqrt(1.0 / n)
    return C


def dct2_block_matrix(n: int, b: int = 8) -> np.ndarray:
    """Block DCT ("the block diagonal forms of the DCT (block DCT) whose block
    size was 8x8"): T = blockdiag(C_b, ..., C_b, C_r) with C_b = dct2_matrix(b) and, when b does
    not divide n, a last block C_r = dct2_matrix(n mod b) (reading R24)."""
    T = np.zeros((n, n))
    for i0 in range(0, n, b):
        w = min(b, n - i0)
        T[i0:i0 + w, i0:i0 + w] = dct2_matrix(w)
    return T


def synthetic_D(N: int, rank: int) -> np.ndarray:
    """The paper's synthetic matrix: D = J - blkdiag(0.5 1 1^T, rank), N x N."""
    p = N // rank
    D = np.ones((N, N))
    for b in range(rank):
        D[b * p:(b + 1) * p, b * p:(b + 1) * p] -= 0.5
    return D


def epsilon_schedule_k(E: float, n: int) -> int:
    """The recommended threshold of eq. recommendation_epsilon: epsilon(E_t)
    = the k-th largest |Phi_|, k = (0.5e-4) n^2 if E_t > E_l, (1.5e-4) n^2 if E_l >= E_t > E_m,
    (0.5e-3) n^2 otherwise, E_l = 0.3e-1, E_m = 6e-4, n x n the size of Phi_.
    k = max(1, floor(.)) (reading R25)."""
    frac = 0.5e-4 if E > 0.3e-1 else (1.5e-4 if E > 6e-4 else 0.5e-3)
    return max(1, int(frac * n * n))


def admm_l_step(zu1, zu2, zu3, zu4, w, psit):
    """l-update of the ADMM (eq. admm_algorithm_inp): the least-squares
    solution l = (K^T K)^-1 K^T (z - u) of K l = z - u for K l = [l; Psi l; Omega l; l] (Psi the
    orthonormal 2-D DCT, so Psi^T Psi = I; Omega = diag(mask), mask in {0, 1}): K^T K = (3 + mask) I
    elementwise.  zu_i = z_i - u_i."""
    return (zu1 + psit(zu2) + w * zu3 + zu4) / (3.0 + w)


def admm_z2_step(v, eta: float, rho: float):
    """z2-update: prox of (eta / rho) ||.||_1 at v, the elementwise soft threshold at eta / rho
    (PAPER.md:1193-1214)."""
    return np.sign(v) * np.maximum(np.abs(v) - eta / rho, 0.0)


def admm_z4_step(v):
    """z4-update: Euclidean projection onto the box [0, 1] (Pi_D)."""
    return np.clip(v, 0.0, 1.0)


def admm_recover(D_obs, mask, kernel: Kernel, K: int, T: int, rho: float, eta: float,
                 max_iter: int = 300, tol: float = 1e-4, shrink=None, return_history: bool = False,
                 transform: str | None = None, adaptive_eps: bool = False):
    """ADMM of PAPER.md:1193-1214 (eq. admm_algorithm_inp) for the synthetic experiment
    (PAPER.md:1095-1100): the average-term constraint z^(5) is dropped, so
    K l = [l; Psi l; Omega l; l] with Psi = 2-D orthonormal DCT (C_m L C_n^T) and Omega the
    observed-entry selector (mask = 1 on observed entries).  K^T K = (3 + mask) I elementwise.

      l   <- (K^T K)^-1 K^T (z - u)
      z1  <- prox_{1/rho ||.||_*}(l + u1)      -- CPA shrinkage (or `shrink`)
      z2  <- soft(Psi l + u2, eta / rho)
      z3  <- D_obs on the observed entries     (Pi_I keeps the assigned values)
      z4  <- clip(l + u4, 0, 1)                (Pi_D)
      u   <- u + K l - z
    stopping: ||l_{t+1} - l_t|| / ||l_{t+1}|| < tol (PAPER.md:694 footnote).  z, u start at 0.
    transform: the shrinkage runs cpa_shrink_transform with this T ("dct" / "dct8" / "haar1");
    adaptive_eps: its components are thresholded at epsilon(E) of epsilon_schedule_k with E the
    previous iteration's ||dl|| / ||l|| (the first iteration: E = inf; reading R25)."""
    D_obs = np.asarray(D_obs, dtype=np.float64)
    w = np.asarray(mask, dtype=np.float64)
    m, n = D_obs.shape
    Cm, Cn = dct2_matrix(m), dct2_matrix(n)
    psi = lambda X: Cm @ X @ Cn.T
    psit = lambda S: Cm.T @ S @ Cn
    E_prev = [math.inf]
    if shrink is None and transform is not None:
        def shrink(X):
            s_ = min(X.shape)
            if adaptive_eps:
                return cpa_shrink_transform(X, kernel, K, T=T, transform=transform, eps_mode="topk",
                                            eps=epsilon_schedule_k(E_prev[0], s_))
            return cpa_shrink_transform(X, kernel, K, T=T, transform=transform)
    if shrink is None:
        shrink = lambda X: cpa_shrink(X, kernel, K, T=T)
    z1 = np.zeros((m, n)); z2 = np.zeros((m, n)); z4 = np.zeros((m, n))
    z3 = w * D_obs
    u1 = np.zeros((m, n)); u2 = np.zeros((m, n)); u3 = np.zeros((m, n)); u4 = np.zeros((m, n))
    l = np.zeros((m, n))
    hist = []
    for it in range(max_iter):
        l_prev = l
        l = admm_l_step(z1 - u1, z2 - u2, z3 - u3, z4 - u4, w, psit)
        pl = psi(l)
        z1 = shrink(l + u1)
        z2 = admm_z2_step(pl + u2, eta, rho)
        z4 = admm_z4_step(l + u4)
        u1 = u1 + l - z1
        u2 = u2 + pl - z2
        u3 = u3 + w * l - z3
        u4 = u4 + l - z4
        rel = float(np.linalg.norm(l - l_prev) / max(np.linalg.norm(l), 1e-300))
        hist.append(rel)
        E_prev[0] = rel
        if rel < tol:
            break
    return (l, hist) if return_history else l


def cpa_apply_vectors(apply_phi, V, c, lam: float):
    """H_hat(Phi) V by the vector form of the recurrence (eq. 310).

    Each column v of V: w_0 = v, w_1 = B_hat v, w_k = 2 B_hat w_{k-1} - w_{k-2},
    result = c_0/2 w_0 + c_1 w_1 + sum_k c_k w_k, with B_hat w = (2/lam) Phi w - w
    (PAPER.md:364, 401-409).  ``apply_phi`` maps an (s x r) block to Phi times it.
    """
    V = np.asarray(V, dtype=np.float64)

    def bhat(W):
        return (2.0 / lam) * apply_phi(W) - W

    w_km2 = V
    out = 0.5 * c[0] * w_km2
    if len(c) > 1:
        w_km1 = bhat(w_km2)
        out = out + c[1] * w_km1
        for k in range(2, len(c)):
            w_k = 2.0 * bhat(w_km1) - w_km2
            out = out + c[k] * w_k
            w_km2, w_km1 = w_km1, w_k
    return out


def _lam_from_gram_side(apply_phi, s, T, safety, lam):
    return _lambda_and_sigma(lambda: power_iteration(apply_phi, s, T)[0], lam, safety)


def cpa_shrink_columns(X, cols, kernel: Kernel, K: int, T: int = 30, safety: float = DEFAULT_SAFETY,
                       lam: float | None = None):
    """Selected columns of G_hat(X) for a wide X (m <= n), never forming the Gram.

    Y = H_hat(X X^T) X, so Y[:, j] = H_hat(XX^T) x_j  (vector form, PAPER.md:310
    applied to X^T).  Phi w = X (X^T w).  Returns (Y[:, cols], info).
    """
    X = np.asarray(X, dtype=np.float64)
    m, n = X.shape
    assert m <= n

    def apply_phi(W):
        return X @ (X.T @ W)

    lam_, lam_hat, sig = _lam_from_gram_side(apply_phi, m, T, safety, lam)
    info = {"lambda_hat": lam_hat, "lambda_max": lam_, "sigma_max_hat": sig}
    if lam_hat <= DEGENERATE_LAMBDA:
        return np.zeros((m, len(cols))), info
    c = kernel_coefficients(kernel, K, lam_, sig)
    info["coeffs"] = c
    return cpa_apply_vectors(apply_phi, X[:, cols], c, lam_), info


def cpa_shrink_rows(X, rows, kernel: Kernel, K: int, T: int = 30, safety: float = DEFAULT_SAFETY,
                    lam: float | None = None):
    """Selected rows of G_hat(X) for a tall X (m > n): Y[i, :] = (H_hat(X^T X) x_i^T)^T."""
    X = np.asarray(X, dtype=np.float64)
    m, n = X.shape
    assert m > n

    def apply_phi(W):
        return X.T @ (X @ W)

    lam_, lam_hat, sig = _lam_from_gram_side(apply_phi, n, T, safety, lam)
    info = {"lambda_hat": lam_hat, "lambda_max": lam_, "sigma_max_hat": sig}
    if lam_hat <= DEGENERATE_LAMBDA:
        return np.zeros((len(rows), n)), info
    c = kernel_coefficients(kernel, K, lam_, sig)
    info["coeffs"] = c
    return cpa_apply_vectors(apply_phi, X[rows, :].T, c, lam_).T, info


def cpa_shrink_batched(Xb, kernel: Kernel, K: int, T: int = 30, safety: float = DEFAULT_SAFETY):
    """Independent Alg. 1 per matrix of a [batch, m, n] stack (fp64 of the given values)."""
    Xb = np.asarray(Xb, dtype=np.float64)
    Y = np.empty_like(Xb)
    lams = np.empty(Xb.shape[0])
    for b in range(Xb.shape[0]):
        Y[b], info = cpa_shrink(Xb[b], kernel, K, T=T, safety=safety, return_info=True)
        lams[b] = info["lambda_max"]
    return Y, lams


# ---------------------------------------------------------------------------
# Sparse X (BASELINE config 4): right form, Gram never formed
# ---------------------------------------------------------------------------

def sparse_power_iteration(Xs, T: int):
    """Lambda_max of X^T X via the m x m side: v -> X (X^T v), v_0 = 1_m/sqrt(m) (reading R4)."""
    m = Xs.shape[0]
    return power_iteration(lambda v: Xs @ (Xs.T @ v), m, T)


def cpa_shrink_sparse_rows(Xs, rows, kernel: Kernel, K: int, T: int = 300,
                           safety: float = DEFAULT_SAFETY, lam: float | None = None):
    """Selected rows of G_hat(X) = X H_hat(X^T X) for a scipy.sparse CSR X.

    Row i: H_hat(X^T X) x_i^T by the vector recurrence, Phi w = X^T (X w).
    """
    lam_, lam_hat, sig = _lambda_and_sigma(lambda: sparse_power_iteration(Xs, T)[0], lam, safety)
    info = {"lambda_hat": lam_hat, "lambda_max": lam_, "sigma_max_hat": sig}
    n = Xs.shape[1]
    if lam_hat <= DEGENERATE_LAMBDA:
        return np.zeros((len(rows), n)), info
    c = kernel_coefficients(kernel, K, lam_, sig)
    info["coeffs"] = c
    V = np.asarray(Xs[rows, :].todense(), dtype=np.float64).T

    def apply_phi(W):
        return Xs.T @ (Xs @ W)

    return cpa_apply_vectors(apply_phi, V, c, lam_).T, info


# ---------------------------------------------------------------------------
# Exact shrinkage (PAPER.md:264-276 eq. sing_shrink_exact) via one-sided Jacobi
# ---------------------------------------------------------------------------

def jacobi_svd(A, max_sweeps: int = 80, tol: float = 1e-15):
    """Textbook one-sided (Hestenes) Jacobi SVD of A (any shape).

    Returns U (m x r), sigma (r), V (n x r), r = min(m, n), with A = U diag(sigma) V^T.
    Works on the tall orientation; for each column pair (i, j):
    alpha = |a_i|^2, beta = |a_j|^2, gamma = a_i . a_j; if |gamma| > tol sqrt(alpha beta)
    rotate with zeta = (beta - alpha)/(2 gamma), t = sign(zeta)/(|zeta| + sqrt(1 + zeta^2)),
    c = 1/sqrt(1 + t^2), s = c t.  Sweeps repeat until no pair rotates.
    """
    A = np.array(A, dtype=np.float64)
    transposed = A.shape[0] < A.shape[1]
    if transposed:
        A = A.T.copy()
    m, n = A.shape
    V = np.eye(n)
    for _ in range(max_sweeps):
        rotated = False
        for i in range(n - 1):
            for j in range(i + 1, n):
                ai, aj = A[:, i], A[:, j]
                alpha = float(ai @ ai)
                beta = float(aj @ aj)
                gamma = float(ai @ aj)
                if abs(gamma) > tol * math.sqrt(alpha * beta) and gamma != 0.0:
                    rotated = True
                    zeta = (beta - alpha) / (2.0 * gamma)
                    t = (1.0 if zeta >= 0 else -1.0) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                    c = 1.0 / math.sqrt(1.0 + t * t)
                    s = c * t
                    A[:, i], A[:, j] = c * ai - s * aj, s * ai + c * aj
                    vi, vj = V[:, i].copy(), V[:, j].copy()
                    V[:, i], V[:, j] = c * vi - s * vj, s * vi + c * vj
        if not rotated:
            break
    sigma = np.sqrt(np.einsum("ij,ij->j", A, A))
    U = np.zeros_like(A)
    nz = sigma > 1e-300
    U[:, nz] = A[:, nz] / sigma[nz]
    order = np.argsort(-sigma, kind="stable")
    U, sigma, V = U[:, order], sigma[order], V[:, order]
    if transposed:
        U, V = V, U
    return U, sigma, V


def exact_shrink(X, kernel: Kernel, tau: float):
    """G(X) = U g(Sigma) V^T with the true g."""
    U, s, V = jacobi_svd(X)
    gs = np.array([g_response(kernel, float(si), tau) for si in s])
    return (U * gs) @ V.T


def svd_characterization(X, c, lam: float):
    """Y = U diag(sigma_i h_hat(sigma_i^2)) V^T  (PAPER.md:331 eq. ATA_eig_fil, 374-397)."""
    U, s, V = jacobi_svd(X)
    d = np.array([float(si) * series_eval(c, lam, float(si) ** 2) if si > 1e-300 else 0.0 for si in s])
    return (U * d) @ V.T


def rel_fro(A, B) -> float:
    """||A - B||_F / ||B||_F in fp64 (reading R16)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    den = float(np.linalg.norm(B))
    num = float(np.linalg.norm(A - B))
    return num / den if den > 0 else num
