"""Callers of the tall-and-skinny multiply named by the paper: ABFT checksum
encoding and k-means distance computation, on device-resident column-major torch tensors.

Both reduce to one TSM2R / TSM2L call through :func:`paper_2002_03258_b200.gemm` (the sm_100a
kernels; no CPU path) plus O(m·n) torch elementwise glue:

* :func:`abft_encode` — checksum columns of A: ``A @ W`` with ``W = [1, 1..k]`` (plain and
  weighted checksum vectors, Huang-Abraham ABFT), a TSM2R with n = 2.
* :func:`kmeans_distances` / :func:`kmeans_assign` — squared distances of m points (rows of X,
  m × d) to c ≤ 16 centroids: ``|x|² − 2·X·Cᵀ + |c|²``; X·Cᵀ is TSM2L when d is small and
  TSM2R when d is large.
"""

from __future__ import annotations

from .kernels import colmajor_empty, gemm


def _colmajor_copy(T):
    out = colmajor_empty(T.shape[0], T.shape[1], T.dtype, T.device)
    out.copy_(T)
    return out


def abft_encode(A, weighted: bool = True):
    """Checksum columns of a column-major CUDA tensor A (m × k): returns the m × 2 (or m × 1)
    column-major tensor ``A @ [1, (1..k)]`` computed by the TSM2R kernel."""
    import torch
    m, k = A.shape
    n = 2 if weighted else 1
    W = colmajor_empty(k, n, A.dtype, A.device)
    W[:, 0] = 1
    if weighted:
        W[:, 1] = torch.arange(1, k + 1, device=A.device, dtype=A.dtype)
    C = colmajor_empty(m, n, A.dtype, A.device)
    C.zero_()
    return gemm(A, W, C, variant="l-opt2" if k <= 64 else "v3", c_is_zero=True)


def abft_check(A, checksums, rtol: float = None):
    """Recomputes the checksums of A and returns the row indices whose checksums disagree with
    ``checksums`` beyond ``rtol`` (relative to the row's |A| @ W) — an ABFT verification pass."""
    import torch
    weighted = checksums.shape[1] == 2
    fresh = abft_encode(A, weighted)
    if rtol is None:
        rtol = 1e-10 if A.dtype == torch.float64 else 1e-4
    scale = abft_encode(A.abs(), weighted).abs() + torch.finfo(A.dtype).tiny
    bad = ((fresh - checksums).abs() > rtol * scale).any(dim=1)
    return torch.nonzero(bad).flatten()


def kmeans_distances(X, centroids):
    """Squared Euclidean distances (m × c, column-major) of the rows of X (m × d, CUDA) to the
    rows of ``centroids`` (c × d, c ≤ 16 per pass), with X·Cᵀ on the TSM2 kernels."""
    import torch
    m, d = X.shape
    c = centroids.shape[0]
    if centroids.shape[1] != d:
        raise ValueError(f"dimension mismatch: X {m}x{d}, centroids {c}x{centroids.shape[1]}")
    Xc = X if X.stride(0) == 1 else _colmajor_copy(X)
    Ct = colmajor_empty(d, c, X.dtype, X.device)
    Ct.copy_(centroids.t())
    G = colmajor_empty(m, c, X.dtype, X.device)
    G.zero_()
    gemm(Xc, Ct, G, variant="l-opt2" if d <= 64 else "v3", c_is_zero=True)
    xn = (Xc * Xc).sum(dim=1, keepdim=True)
    cn = (centroids * centroids).sum(dim=1).unsqueeze(0)
    return (xn - 2 * G + cn).clamp_min_(0)


def kmeans_assign(X, centroids):
    """Index of the nearest centroid for every row of X (one k-means assignment step)."""
    return kmeans_distances(X, centroids).argmin(dim=1)
