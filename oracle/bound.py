"""The tighter spectral-norm bound of Algorithm 2, line 1 in float64.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Theorem 2: for A symmetric, eigenvalues lambda_n <= ... <= lambda_1 of A^2,
sigma real with lambda_1 the eigenvalue of A^2 nearest sigma, and any unit q,

    ||A||_2 <= sqrt(sigma + ||A^2 q - sigma q||_2).

P:L724: (sigma, q) is "the largest Ritz value produced by a 20-step Lanczos run on A^2
together with its Ritz vector".  Here, step by step:

    A0 = X / ||X||_F                                   (the chain's normalisation, R4)
    v_0 = h / ||h||                                    (start vector: the counter hash below)
    for k = 0 .. m-1  (m = min(steps, n)):             (Lanczos, Parlett ch. 13, with full
        w = A0 (A0 v_k)                                 re-orthogonalisation: two classical
        for pass in 1, 2:                               Gram-Schmidt passes)
            c = V_k^T w;  w = w - V_k c;  alpha_k += c_k
        beta_k = ||w||;  v_{k+1} = w / beta_k  (0 if beta_k == 0)
    T_m = tridiag(beta, alpha, beta);  (theta, y) = largest eigenpair of T_m (numpy eigh)
    q = V_m y;  sigma = theta
    lambda~ = ||X||_F * min(1, sqrt(sigma + ||A0^2 q - sigma q||) * safety)

Readings (R21): the Krylov run is on X / ||X||_F (any positive scaling gives the same
Ritz vectors); ``min(1, .)`` keeps the bound no looser than Frobenius; ``safety`` multiplies
the bound (1 = the paper's).  The start vector is not given by the paper: both sides use the
same counter-based hash (the task's rule for random numbers a method draws).
"""
import numpy as np

from .chain import symmetric_from_upper


def start_vector(n):
    """h_j = 0.5 + (H(j) & 0xFFFF) / 65536 with H the 32-bit multiplicative hash below."""
    j = np.arange(n, dtype=np.uint64)
    M = np.uint64(0xFFFFFFFF)
    h = (j * np.uint64(2654435761) + np.uint64(0x9E3779B9)) & M
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(2246822519)) & M
    h ^= h >> np.uint64(13)
    return 0.5 + (h & np.uint64(0xFFFF)).astype(np.float64) / 65536.0


def lanczos_ritz(A, steps):
    """Largest Ritz pair (theta, q) of a ``steps``-step Lanczos run on the symmetric A
    (full re-orthogonalisation), started from ``start_vector``."""
    n = A.shape[0]
    m = min(steps, n)
    V = np.zeros((m + 1, n))
    h = start_vector(n)
    V[0] = h / np.linalg.norm(h)
    alpha = np.zeros(m)
    beta = np.zeros(m)
    for k in range(m):
        w = A @ V[k]
        for _ in range(2):
            c = V[: k + 1] @ w
            w = w - V[: k + 1].T @ c
            alpha[k] += c[k]
        beta[k] = np.linalg.norm(w)
        V[k + 1] = w / beta[k] if beta[k] > 0 else 0.0
    T = np.diag(alpha) + np.diag(beta[: m - 1], 1) + np.diag(beta[: m - 1], -1)
    theta, Y = np.linalg.eigh(T)
    y = Y[:, -1]
    return float(theta[-1]), V[:m].T @ y


def theorem2_bound(A, sigma, q):
    """sqrt(sigma + ||A^2 q - sigma q||) for unit q (Eq. comp:upper-bound)."""
    q = q / np.linalg.norm(q)
    r = A @ (A @ q) - sigma * q
    return float(np.sqrt(sigma + np.linalg.norm(r)))


def lanczos_bound(X, steps=20, safety=1.0):
    """lambda~ of Algorithm 2 line 1 for the upper-triangle symmetric X."""
    Xs = symmetric_from_upper(X)
    lamF = float(np.sqrt(np.sum(Xs * Xs)))
    if lamF == 0.0 or not np.isfinite(lamF):
        return lamF
    A0 = Xs / lamF
    theta, q = lanczos_ritz(A0 @ A0, steps)
    f = theorem2_bound(A0, theta, q) * safety
    return lamF * min(1.0, f)
