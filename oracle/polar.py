"""The polar factor by the same composite odd filter, in plain float64 (the parity oracle of
``psd_polar``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper builds its filters for the matrix sign and names the polar factor as its
generalisation (composite odd polynomials "approximate the polar factor (a
generalization of matrix sign function)"); SURVEY 8(f)#4 asks for ``psd_sign`` as a matrix-sign /
polar primitive, where "nonsymmetric polar needs X^T X products".  For a general square A with
singular value decomposition A = W diag(sigma) V^T, an odd polynomial f(x) = sum_j c_j x^{2j+1}
 acts on the singular values:

    f(A) := W diag(f(sigma)) V^T = sum_j c_j A (A^T A)^j

and the composite chain f_T o ... o f_1 applied to A_0 = A / lambda~ (lambda~ >= ||A||_2; the
Frobenius norm by default) maps every singular value in [eps, 1] to within the chain's
sign error of 1, i.e. approximates the orthogonal polar factor W V^T.

Written as that definition: A_t = f_t(A_{t-1}) with (A^T A)^j as plain float64 matrix products
(``chain.matmul``) and the kappa_t rescale applied literally after stage t (reading R1).
"""
import numpy as np

from oracle import chain


def frobenius(A):
    """||A||_F >= ||A||_2 of a general matrix (the Frobenius bound)."""
    A = np.asarray(A, dtype=np.float64)
    return float(np.sqrt(np.sum(A * A)))


def odd_poly_general(Z, coeffs):
    """f(Z) = sum_{j=0}^{p} c_j Z (Z^T Z)^j -- the odd polynomial on the singular values of Z."""
    Z = np.asarray(Z, dtype=np.float64)
    out = coeffs[0] * Z
    if len(coeffs) == 1:
        return out
    G = chain.matmul(Z.T, Z)             # Z^T Z
    power = Z                            # Z (Z^T Z)^j, starting at j = 0
    for j in range(1, len(coeffs)):
        power = chain.matmul(power, G)
        out = out + coeffs[j] * power
    return out


def polar_chain(A0, stages, kappas=None):
    """A_T = f_T o ... o f_1 (A_0), f_1 applied first, kappa_t after stage t."""
    Z = np.asarray(A0, dtype=np.float64)
    for t, c in enumerate(stages):
        Z = odd_poly_general(Z, c)
        if kappas is not None:
            Z = kappas[t] * Z
    return Z


def polar(A, stages, kappas=None, lam=None):
    """The filter's polar iterate of a general square A.  Returns (U, lambda~).

    ``lam`` overrides the bound (the GPU exports the lambda~ it used); lambda~ == 0 returns 0."""
    A = np.asarray(A, dtype=np.float64)
    if lam is None:
        lam = frobenius(A)
    lam = float(lam)
    if lam == 0.0:
        return np.zeros_like(A), 0.0
    return polar_chain(A / lam, stages, kappas), lam
