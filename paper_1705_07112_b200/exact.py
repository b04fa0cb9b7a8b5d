"""NEXT-4: the paper's exact EVD-based singular-value shrinkage, the baseline its
Tables I-II time CPA against ("the EVD-based method ... eigendecomposition of
B^T B"), on the same B200 through cuSOLVER / cuBLAS (torch.linalg.eigh, matmul).

This is a COMPARISON baseline built on library routines -- not the CPA product path (which is
libcpasvt's kernels, paper_1705_07112_b200.Handle).  It exists so the speed and the approximation
error of CPA can be measured beside the exact method on the same device.

  G = X X^T (m <= n) or X^T X;  (lambda_i, v_i) = eigh(G);
  Y = V diag(h(lambda)) V^T X   (or X V diag(h(lambda)) V^T),
with h the response of PAPER.md:496-519 (hard / soft / weighted soft, the same kernel dict the
library takes), i.e. Y = U g(Sigma) V^T with g(sigma) = sigma h(sigma^2).
A relative tau resolves against the exact sigma_max = sqrt(lambda_max(G)).
"""

from __future__ import annotations


def h_exact(lam, kernel: dict, tau: float):
    """h(lambda) of PAPER.md:496-519 on a tensor of Gram eigenvalues (clamped at 0)."""
    import torch
    x = torch.clamp(lam, min=0.0)
    r = torch.sqrt(x)
    safe = torch.where(r > 0, r, torch.ones_like(r))
    kind = kernel["kind"]
    if kind == "hard":
        return (r > tau).to(lam.dtype)
    if kind == "soft":
        return torch.where(r > tau, (r - tau) / safe, torch.zeros_like(r))
    if kind == "wsoft":
        w = kernel["w_c"] / (torch.sqrt(torch.clamp(x - kernel.get("w_shift", 0.0), min=0.0)) + kernel["w_eps"])
        return torch.where(r > w, (r - w) / safe, torch.zeros_like(r))
    raise ValueError(f"unknown kernel kind {kind!r}")


def exact_shrink(X, kernel: dict, tau: float | None = None):
    """Exact shrinkage of a 2-D (CUDA) tensor by the EVD of its smaller Gram.  `tau` overrides the
    kernel's threshold (absolute); otherwise kernel['tau'] (x sigma_max if tau_relative)."""
    import torch
    m, n = X.shape
    left = m <= n
    G = X @ X.T if left else X.T @ X
    lam, V = torch.linalg.eigh(G)
    if tau is None:
        tau = float(kernel.get("tau", 0.0))
        if kernel.get("tau_relative"):
            tau *= float(torch.sqrt(torch.clamp(lam[-1], min=0.0)))
    Hm = (V * h_exact(lam, kernel, tau)) @ V.T
    return Hm @ X if left else X @ Hm
