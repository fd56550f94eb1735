"""Algorithm 2 of arXiv 2507.09165 in plain float64 (the parity oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Algorithm 2 "Run-time projection algorithm":

    lambda~ <- upper bound of ||X||_2
    X_0     <- X / lambda~
    for t = 1..T:  X_t <- f~*_t(X_{t-1})
    return lambda~ * 1/2 * X_0 (I_n + X_T)

with f_t(x) = sum_j c_{t,j} x^{2j+1} an odd polynomial and the
stabilisation rescale X <- kappa_t X at the end of stage t (reading R1).

Readings:
  R4  the bound is the Frobenius norm ||X||_F unless ``lam`` is given;
  R10 only the upper triangle of X is read (X_ij := X_min(i,j),max(i,j));
  R14 the returned matrix is symmetrised 1/2 (P + P^T).

Every matrix power here is a plain float64 matrix product (``matmul``: numpy's BLAS product by
default for speed; ``naive_matmul`` is the textbook i-k-j triple loop, and the pins check that the
two agree on small inputs); f_t(Z) is evaluated as the monomial sum of its definition, not by
Horner, not fused.
"""
import numpy as np


def naive_matmul(A, B):
    """C = A B by the textbook i-k-j triple loop, float64 (the north star's "naive matmuls")."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    n, k = A.shape
    k2, m = B.shape
    assert k == k2
    C = [[0.0] * m for _ in range(n)]
    Bl = B.tolist()
    for i in range(n):
        Ci = C[i]
        Ai = A[i].tolist()
        for kk in range(k):
            a = Ai[kk]
            if a == 0.0:
                continue
            Bk = Bl[kk]
            for j in range(m):
                Ci[j] += a * Bk[j]
    return np.array(C, dtype=np.float64)


def blas_matmul(A, B):
    return np.asarray(A, dtype=np.float64) @ np.asarray(B, dtype=np.float64)


matmul = blas_matmul        # module-level hook: tests swap in naive_matmul


def symmetric_from_upper(X):
    """X_ij := X_{min(i,j), max(i,j)} (reading R10, LAPACK uplo='U')."""
    X = np.asarray(X, dtype=np.float64)
    U = np.triu(X)
    return U + np.triu(X, 1).T


def frobenius_bound(X):
    """lambda~ = ||X||_F >= ||X||_2 of the upper-triangle symmetric X."""
    Xs = symmetric_from_upper(X)
    return float(np.sqrt(np.sum(Xs * Xs)))


def odd_poly_matrix(Z, coeffs):
    """f(Z) = sum_{j=0}^{p} c_j Z^{2j+1}   (P:L57 odd monomials; P:L395-399 powers as products)."""
    Z = np.asarray(Z, dtype=np.float64)
    out = coeffs[0] * Z
    if len(coeffs) == 1:
        return out
    Z2 = matmul(Z, Z)
    power = Z                        # Z^{2j+1}, starting at j = 0
    for j in range(1, len(coeffs)):
        power = matmul(power, Z2)    # Z^{2j+1} = Z^{2j-1} Z^2
        out = out + coeffs[j] * power
    return out


def sign_chain(X0, stages, kappas=None):
    """X_T = f_T o ... o f_1 (X_0), f_1 applied first.

    ``kappas[t]`` (if given) multiplies the iterate at the end of stage t
    (P:L727 stabilisation, applied literally, never folded).
    """
    Z = np.asarray(X0, dtype=np.float64)
    for t, c in enumerate(stages):
        Z = odd_poly_matrix(Z, c)
        if kappas is not None:
            Z = kappas[t] * Z
    return Z


def project(X, stages, kappas=None, lam=None):
    """Algorithm 2.  Returns (P, lambda~).

    ``lam`` overrides the bound (the GPU exports the lambda~ it used, so parity
    never depends on the bound; reading R4).  lambda~ == 0 returns 0.
    """
    Xs = symmetric_from_upper(X)
    n = Xs.shape[0]
    if lam is None:
        lam = frobenius_bound(Xs)
    lam = float(lam)
    if lam == 0.0:
        return np.zeros_like(Xs), 0.0
    X0 = Xs / lam
    S = sign_chain(X0, stages, kappas)
    P = lam * 0.5 * matmul(X0, np.eye(n) + S)
    return 0.5 * (P + P.T), lam                              # R14


def sign(X, stages, kappas=None, lam=None):
    """The matrix-sign output S = X_T of the same chain (psd_sign)."""
    Xs = symmetric_from_upper(X)
    if lam is None:
        lam = frobenius_bound(Xs)
    lam = float(lam)
    if lam == 0.0:
        return np.zeros_like(Xs), 0.0
    S = sign_chain(Xs / lam, stages, kappas)
    return 0.5 * (S + S.T), lam


def project_batch(Xb, stages, kappas=None, lams=None):
    """Algorithm 2 applied independently to each matrix of a batch."""
    Xb = np.asarray(Xb, dtype=np.float64)
    out = np.empty_like(Xb)
    used = np.empty(Xb.shape[0])
    for b in range(Xb.shape[0]):
        out[b], used[b] = project(Xb[b], stages, kappas, None if lams is None else lams[b])
    return out, used


# ---------------------------------------------------------------- scalar chain

def odd_poly_scalar(x, coeffs):
    """f(x) = sum_j c_j x^{2j+1} on scalars / arrays."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    for j, c in enumerate(coeffs):
        out = out + c * x ** (2 * j + 1)
    return out


def scalar_chain(x, stages, kappas=None):
    """s(x) = f_T o ... o f_1 (x) with kappa_t after stage t."""
    z = np.asarray(x, dtype=np.float64)
    for t, c in enumerate(stages):
        z = odd_poly_scalar(z, c)
        if kappas is not None:
            z = kappas[t] * z
    return z


def relu_approx(x, stages, kappas=None):
    """f(x) = 1/2 x (1 + s(x))  (Eq. comp:fstar; Eq. comp:sign P:L517)."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + scalar_chain(x, stages, kappas))


def gemm_count(degrees, reconstruction=True):
    """GEMMs Algorithm 2 needs: sum_t (d_t+1)/2 (+1 for the return line).

    Reading R6: P:L598 (31 for T=10, d=5) and P:L647 (22 for T=7, d=5) fix the
    count; the "sum d_i" at P:L416 is loose.  A degree-1 stage is a scalar (0).
    """
    g = sum((d + 1) // 2 if d > 1 else 0 for d in degrees)
    return g + (1 if reconstruction else 0)
