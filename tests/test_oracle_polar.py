"""Pins of the polar oracle (oracle/polar.py) against what the mathematics fixes: the singular-value
closed form with known orthogonal factors, numpy's SVD, the symmetric special case (the sign chain),
scaling and transpose invariants, and the certified distance to the true polar factor.  No value here
comes from the CUDA path."""
import numpy as np
import pytest

from oracle import chain, polar, tables


def _orth(n, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return q * np.sign(np.diag(r))


HALF = (tables.F_HALF_REFINED, tables.half_kappas(7))


def test_singular_value_closed_form():
    """A = W diag(sigma) V^T with known W, V: polar(A) = W diag(s(sigma / ||A||_F)) V^T, s the scalar
    chain evaluated on scalars (chain.scalar_chain: a separate code path, monomials on floats)."""
    n = 12
    W, V = _orth(n, 1), _orth(n, 2)
    sigma = np.geomspace(1.0, 2e-3, n)
    A = W @ np.diag(sigma) @ V.T
    st, kap = HALF
    U, lam = polar.polar(A, st, kap)
    assert abs(lam - np.sqrt(np.sum(sigma ** 2))) < 1e-12 * lam
    ref = W @ np.diag(chain.scalar_chain(sigma / lam, st, kap)) @ V.T
    assert np.max(np.abs(U - ref)) < 1e-12


def test_matches_numpy_svd_on_random_input():
    """Brute force on a random (non-normal) 9 x 9 input: the definition through np.linalg.svd."""
    A = np.random.default_rng(3).standard_normal((9, 9))
    st, kap = HALF
    U, lam = polar.polar(A, st, kap)
    w, s, vt = np.linalg.svd(A)
    ref = w @ np.diag(chain.scalar_chain(s / lam, st, kap)) @ vt
    assert np.linalg.norm(U - ref) / np.linalg.norm(ref) < 1e-12


def test_symmetric_input_is_the_sign_chain():
    """For symmetric A, Z^T Z = Z^2 at every stage: polar(A) equals the matrix-sign oracle."""
    B = np.random.default_rng(4).standard_normal((10, 10))
    X = 0.5 * (B + B.T)
    st, kap = HALF
    U, lam = polar.polar(X, st, kap)
    S, lam2 = chain.sign(X, st, kap)
    assert lam == pytest.approx(lam2, rel=1e-15)
    assert np.max(np.abs(U - S)) < 1e-12


def test_transpose_and_scale_invariance():
    """polar(A^T) = polar(A)^T; polar(2^k A) = polar(A) with the Frobenius bound (exact scaling)."""
    A = np.random.default_rng(5).standard_normal((8, 8))
    st, kap = HALF
    U, _ = polar.polar(A, st, kap)
    Ut, _ = polar.polar(A.T, st, kap)
    assert np.max(np.abs(Ut - U.T)) < 1e-12
    U8, _ = polar.polar(8.0 * A, st, kap)
    assert np.array_equal(U8, U)


def test_certified_distance_to_the_polar_factor():
    """Singular values in [eps, 1] after the scaling: ||polar(A) - W V^T||_2 <= the chain's sign error
    on [eps, 1] (1 - a_{T+1}, the interval recursion of f*_half, eps = 1e-3)."""
    n = 16
    W, V = _orth(n, 6), _orth(n, 7)
    sigma = np.geomspace(1.0, 1.5e-3, n)
    sigma = sigma / np.sqrt(np.sum(sigma ** 2))            # ||A||_F = 1: A_0 = A
    A = W @ np.diag(sigma) @ V.T
    st = tables.F_HALF
    a = 1e-3
    for c in st:
        a = float(chain.odd_poly_scalar(a, c))
    sign_err = 1.0 - a
    U, lam = polar.polar(A, st, lam=1.0)
    assert np.linalg.norm(U - W @ V.T, 2) <= sign_err * (1 + 1e-9)
    assert sign_err < 1e-8


def test_zero_and_degree_one():
    st, kap = HALF
    U, lam = polar.polar(np.zeros((5, 5)), st, kap)
    assert lam == 0.0 and not U.any()
    A = np.random.default_rng(8).standard_normal((6, 6))
    U, lam = polar.polar(A, [[2.0]])                         # a degree-1 stage is a scalar (R7)
    assert np.array_equal(U, 2.0 * (A / lam))


def test_naive_and_blas_products_agree():
    """The oracle's products through the textbook loop (chain.naive_matmul) match BLAS."""
    A = np.random.default_rng(9).standard_normal((7, 7))
    st, kap = HALF
    U1, _ = polar.polar(A, st, kap)
    old = chain.matmul
    try:
        chain.matmul = chain.naive_matmul
        U2, _ = polar.polar(A, st, kap)
    finally:
        chain.matmul = old
    assert np.max(np.abs(U1 - U2)) < 1e-13


@pytest.mark.parametrize("rows,cols", [(11, 5), (4, 9)])
def test_rectangular_matches_svd(rows, cols):
    """Tall and wide A: the same definition, f(A) = W diag(s(sigma / lambda~)) V^T with the thin SVD."""
    A = np.random.default_rng(10 + rows).standard_normal((rows, cols))
    st, kap = HALF
    U, lam = polar.polar(A, st, kap)
    assert U.shape == (rows, cols)
    w, s, vt = np.linalg.svd(A, full_matrices=False)
    ref = w @ np.diag(chain.scalar_chain(s / lam, st, kap)) @ vt
    assert np.linalg.norm(U - ref) / np.linalg.norm(ref) < 1e-12
