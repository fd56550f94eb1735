"""Pins of oracle/admm.py (the SDP consumer, Eq. exp:admm-three-step) against the
mathematics, independent of the formula it types: the ADMM fixed point at a KKT pair, the
Moreau decomposition of the exact projection, the certified filter bound carried through the
update, and convergence of the whole iteration on a small max-cut SDP."""
import numpy as np

import synth
from oracle import admm, certify, chain, spectral, tables


def _rand_orth(n, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def test_kkt_point_is_a_fixed_point():
    """If S* >= 0, X* >= 0, S* X* = 0 and C = A* y* + S*, then Pi(C - A*y* - X*/sigma) = S*
    (the two parts are orthogonal PSD / NSD pieces) and the X line returns X*: the exact ADMM
    step is stationary at a KKT point (a plausible sign or term error in either line breaks it)."""
    n, k = 24, 7
    Q = _rand_orth(n, 3)
    rng = np.random.default_rng(4)
    s = np.concatenate([rng.uniform(0.5, 2.0, k), np.zeros(n - k)])
    x = np.concatenate([np.zeros(k), rng.uniform(0.5, 2.0, n - k)])
    S_star = Q @ np.diag(s) @ Q.T
    X_star = Q @ np.diag(x) @ Q.T
    y_star = rng.standard_normal(n)
    C = np.diag(y_star) + S_star
    for sigma in (0.3, 1.0, 4.0):
        S, X, _ = admm.s_update(C, X_star, y_star, sigma, None, exact=True)
        assert np.allclose(S, S_star, atol=1e-11), sigma
        assert np.allclose(X, X_star, atol=1e-11), sigma


def test_moreau_decomposition_of_the_update():
    """With the exact projection: S >= 0, X_next >= 0, <S, X_next> = 0 and S - X_next / sigma = M
    (Moreau: M = Pi_+(M) + Pi_-(M), X_next = -sigma Pi_-(M))."""
    n, sigma = 80, 1.7
    C, Xk, y = synth.maxcut_admm(n, synth.SEED_BASE + 91)
    S, X, _ = admm.s_update(C, Xk, y, sigma, None, exact=True)
    M = admm.form_argument(C, Xk, y, sigma)
    scale = np.linalg.norm(M)
    assert np.linalg.eigvalsh(S).min() >= -1e-12 * scale
    assert np.linalg.eigvalsh(X).min() >= -1e-12 * scale * sigma
    assert abs(np.sum(S * X)) <= 1e-10 * scale * scale * sigma
    assert np.allclose(S - X / sigma, M, atol=1e-12 * scale)


def test_filter_update_within_certified_bound():
    """With the composite filter as Pi: ||S - Pi(M)||_2 <= lam~ relu_err (the certified
    scalar bound) and ||X_next - X_exact||_2 <= sigma lam~ relu_err."""
    n, sigma = 96, 2.0
    C, Xk, y = synth.maxcut_admm(n, synth.SEED_BASE + 92)
    st, kap = tables.F_HALF_REFINED, tables.half_kappas(7)
    e, _, _ = certify.relu_err(st, kap)
    S, X, lam = admm.s_update(C, Xk, y, sigma, st, kap)
    Se, Xe, _ = admm.s_update(C, Xk, y, sigma, None, exact=True)
    assert lam == chain.frobenius_bound(admm.form_argument(C, Xk, y, sigma))
    assert np.linalg.norm(S - Se, 2) <= lam * e * (1 + 1e-9)
    assert np.linalg.norm(X - Xe, 2) <= sigma * lam * e * (1 + 1e-9)


def test_admm_converges_on_small_maxcut():
    """The whole iteration (A A* = I for max-cut) reaches the paper's stopping rule
    eta < 1e-4 with the exact projection, and the filter-based iteration reaches the paper's
    warm-start switch level 1e-2; the exact solution is primal/dual feasible."""
    n = 40
    C, _, _ = synth.maxcut_admm(n, synth.SEED_BASE + 93)
    X, y, S, etas = admm.solve(C, sigma=3.0, iters=400, exact=True)
    assert min(etas) < 1e-4, min(etas)
    assert np.allclose(np.diag(X), 1.0, atol=1e-3)
    assert np.linalg.eigvalsh(X).min() >= -1e-6 and np.linalg.eigvalsh(S).min() >= -1e-6
    st, kap = tables.F_HALF_REFINED, tables.half_kappas(7)
    _, _, _, etas_f = admm.solve(C, sigma=3.0, iters=100, stages=st, kappas=kap)
    assert min(etas_f) < 1e-2, min(etas_f)
