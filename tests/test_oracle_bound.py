"""Pins of the Lanczos / Theorem-2 bound oracle (oracle/bound.py).

Each check ties the oracle to something other than itself: numpy's 2-norm (a library SVD),
closed forms (rank one, identity, full Krylov space), the theorem's inequality on random
Ritz-free inputs, and invariances the definition implies.
"""
import numpy as np
import pytest

from oracle import bound
from synth import goe, haar, sdp_shaped


def _py_hash(j):
    h = (j * 2654435761 + 0x9E3779B9) % 2**32
    h ^= h >> 15
    h = (h * 2246822519) % 2**32
    h ^= h >> 13
    return 0.5 + (h & 0xFFFF) / 65536.0


def test_start_vector_matches_integer_hash():
    v = bound.start_vector(1000)
    assert all(v[j] == _py_hash(j) for j in (0, 1, 2, 17, 999))
    assert v.min() >= 0.5 and v.max() < 1.5


def test_full_krylov_space_gives_the_exact_norm():
    # n <= steps: the Krylov space is all of R^n, the top Ritz pair is the top eigenpair and
    # the residual vanishes -> lambda~ = ||X||_2 (P:L709-711 with equality)
    rng = np.random.default_rng(5)
    A = rng.standard_normal((12, 12))
    X = A + A.T
    lam = bound.lanczos_bound(X, steps=20, safety=1.0)
    assert lam == pytest.approx(np.linalg.norm(X, 2), rel=1e-10)


@pytest.mark.parametrize("name,X", [("goe", goe(400, seed=1)), ("haar", haar(300, seed=2)),
                                    ("sdp", sdp_shaped(512, seed=3))])
def test_valid_and_tight_on_paper_spectra(name, X):
    # the 20-step heuristic yields a valid upper bound in practice; it is far below
    # the Frobenius bound (the point of the tighter bound)
    s2 = np.linalg.norm(X, 2)
    lam = bound.lanczos_bound(X, steps=20, safety=1.0)
    assert s2 * (1 - 1e-12) <= lam <= 1.01 * s2
    assert lam < 0.2 * np.linalg.norm(X)


def test_rank_one_closed_form():
    rng = np.random.default_rng(7)
    u = rng.standard_normal(300)
    X = np.outer(u, u)
    assert bound.lanczos_bound(X, 20, 1.0) == pytest.approx(u @ u, rel=1e-12)


def test_identity_start_vector_is_an_eigenvector():
    # every vector is an eigenvector: beta_0 = 0, theta = 1, residual 0 -> lambda~ = 1 * safety
    X = np.eye(50)
    assert bound.lanczos_bound(X, 20, 1.0) == pytest.approx(1.0, rel=1e-14)
    assert bound.lanczos_bound(X, 20, 1.01) == pytest.approx(1.01, rel=1e-14)


def test_never_looser_than_frobenius_and_invariances():
    X = goe(200, seed=9)
    F = np.linalg.norm(X)
    assert bound.lanczos_bound(X, 1, 2.0) <= F
    lam = bound.lanczos_bound(X, 20, 1.0)
    assert bound.lanczos_bound(-X, 20, 1.0) == pytest.approx(lam, rel=1e-12)
    assert bound.lanczos_bound(3.5 * X, 20, 1.0) == pytest.approx(3.5 * lam, rel=1e-12)
    assert bound.lanczos_bound(np.zeros((8, 8)), 20, 1.0) == 0.0


def test_theorem2_inequality_on_random_vectors():
    # Theorem 2 with sigma at the top of A^2's spectrum side: for sigma >= the
    # midpoint of lambda_1 and lambda_2 of A^2, lambda_1 is the nearest eigenvalue and the
    # bound must hold for every unit q; at the top eigenvector it is an equality
    rng = np.random.default_rng(11)
    X = goe(60, seed=12)
    ev = np.linalg.eigvalsh(X @ X)
    s2 = np.sqrt(ev[-1])
    for _ in range(50):
        q = rng.standard_normal(60)
        sigma = rng.uniform(0.5 * (ev[-1] + ev[-2]), 2 * ev[-1])
        assert bound.theorem2_bound(X, sigma, q) >= s2 * (1 - 1e-12)
    w, V = np.linalg.eigh(X @ X)
    assert bound.theorem2_bound(X, w[-1], V[:, -1]) == pytest.approx(s2, rel=1e-10)


def test_more_steps_is_tighter():
    X = goe(600, seed=13)
    s2 = np.linalg.norm(X, 2)
    gaps = [bound.lanczos_bound(X, k, 1.0) / s2 - 1 for k in (5, 20, 40)]
    assert gaps[0] > gaps[1] > gaps[2] >= -1e-12
