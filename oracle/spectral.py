"""Spectral references for the oracle.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* ``eig_project``  -- Higham's closed form Pi(X) = Q max(Lambda, 0) Q^T (Eq.
  intro:closed-form) with numpy ``eigh`` as the library primitive.
* ``spectral_apply`` -- the spectral operator F(X) = Q diag(f(lambda)) Q^T
  (Eq. spectral-operator); with f = the composite ReLU approximant it
  equals Algorithm 2's output exactly, which pins the matrix chain.
* ``hadamard`` / ``structured_project`` -- exact large-n reference: for an
  orthogonal H, p(H B H^T) = H p(B) H^T (same identity), so with
  B block-diagonal the projection costs blockwise chains plus two fast
  Walsh-Hadamard transforms.  Used for parity at n = 4096 and 16384 where the
  dense O(G n^3) oracle would take minutes to hours (SURVEY.md [chk-9]).
"""
import numpy as np

from . import chain


def eig_project(X):
    """Pi_{S+}(X) = Q diag(max(lambda_i, 0)) Q^T."""
    Xs = chain.symmetric_from_upper(X)
    lam, Q = np.linalg.eigh(Xs)
    return (Q * np.maximum(lam, 0.0)) @ Q.T


def spectral_apply(X, f):
    """F(X) = Q diag(f(lambda_1..n)) Q^T."""
    Xs = chain.symmetric_from_upper(X)
    lam, Q = np.linalg.eigh(Xs)
    return (Q * f(lam)) @ Q.T


def fwht_rows(A):
    """A @ H for the normalised Sylvester-Hadamard H (n = 2^k), H = H^T, H H = I."""
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[-1]
    assert n & (n - 1) == 0, "n must be a power of two"
    h = 1
    while h < n:
        A = A.reshape(A.shape[:-1] + (n // (2 * h), 2, h))
        a0 = A[..., 0, :].copy()
        a1 = A[..., 1, :]
        A[..., 0, :] = a0 + a1
        A[..., 1, :] = a0 - a1
        A = A.reshape(A.shape[:-3] + (n,))
        h *= 2
    return A / np.sqrt(n)


def hadamard_conjugate(B):
    """H B H^T for the normalised Hadamard H (both transforms fast)."""
    return fwht_rows(fwht_rows(B).T).T


def blockdiag(blocks):
    n = sum(b.shape[0] for b in blocks)
    out = np.zeros((n, n))
    i = 0
    for b in blocks:
        k = b.shape[0]
        out[i:i + k, i:i + k] = b
        i += k
    return out


def structured_project(blocks, stages, kappas, lam):
    """P(H B H^T) = H P(B) H^T with P(B) computed blockwise by Algorithm 2
    (``chain.project`` with the SAME lambda~ for every block)."""
    pb = [chain.project(b, stages, kappas, lam=lam)[0] for b in blocks]
    return hadamard_conjugate(blockdiag(pb))


def structured_project_rows(blocks, stages, kappas, lam, rows):
    """Rows `rows` of P(H B H^T) = H P(B) H^T without forming the n x n matrix: row i is
    (H e_i)^T P(B) H (H symmetric), i.e. the Hadamard transform of h_i^T blockdiag(P(B)) with
    h_i = H e_i -- O(n log n) per row (for the n = 16384 checks)."""
    pb = [chain.project(b, stages, kappas, lam=lam)[0] for b in blocks]
    n = sum(b.shape[0] for b in blocks)
    E = np.zeros((len(rows), n))
    E[np.arange(len(rows)), list(rows)] = 1.0
    Hr = fwht_rows(E)                               # rows of H (H = H^T)
    U = np.empty_like(Hr)
    i = 0
    for b in pb:
        k = b.shape[0]
        U[:, i:i + k] = Hr[:, i:i + k] @ b
        i += k
    return fwht_rows(U)


def structured_sign(blocks, stages, kappas, lam):
    sb = [chain.sign(b, stages, kappas, lam=lam)[0] for b in blocks]
    return hadamard_conjugate(blockdiag(sb))


def jacobi_eigvals(X, sweeps=100, tol=1e-15):
    """Cyclic Jacobi eigenvalues for tiny symmetric X (textbook; independent of LAPACK)."""
    A = np.array(chain.symmetric_from_upper(X), dtype=np.float64)
    n = A.shape[0]
    for _ in range(sweeps):
        off = np.sqrt(np.sum(A * A) - np.sum(np.diag(A) ** 2))
        if off <= tol * np.sqrt(np.sum(A * A)):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                if A[p, q] == 0.0:
                    continue
                theta = (A[q, q] - A[p, p]) / (2.0 * A[p, q])
                t = np.sign(theta) / (abs(theta) + np.sqrt(theta * theta + 1.0)) if theta != 0 else 1.0
                c = 1.0 / np.sqrt(t * t + 1.0)
                s = t * c
                J = np.eye(n)
                J[p, p] = c
                J[q, q] = c
                J[p, q] = s
                J[q, p] = -s
                A = J.T @ A @ J
    return np.sort(np.diag(A))


def rel_error(A_plus, Pi):
    """||A_+ - Pi||_F / ||Pi||_F, computed in fp64; reading R12: if
    ||Pi||_F == 0 the absolute error ||A_+||_F is returned."""
    A_plus = np.asarray(A_plus, dtype=np.float64)
    Pi = np.asarray(Pi, dtype=np.float64)
    den = np.linalg.norm(Pi)
    num = np.linalg.norm(A_plus - Pi)
    return float(num / den) if den > 0 else float(num)
