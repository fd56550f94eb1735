"""The SDP consumer of the projection: three-step ADMM (Eq. exp:admm-three-step)
in plain float64, with the PSD-cone projection replaced by the composite filter.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

For the primal/dual pair of Eq. (exp:sdp) with constraint matrices A_i:

    y^{k+1} = (A A*)^{-1} ( b / sigma - A( X^k / sigma + S^k - C ) )
    S^{k+1} = Pi( C - A* y^{k+1} - X^k / sigma )
    X^{k+1} = X^k + sigma ( S^{k+1} + A* y^{k+1} - C )

Here the constraints are diagonal (max-cut, A_i = e_i e_i^T, b = 1): A X = diag(X),
A* y = Diag(y), A A* = I.  ``s_update`` is the fused GPU step (psd_admm_update): the S and
X lines for a given y; ``solve`` runs the whole iteration for the pins.  The KKT residual
eta follows P:L942-948.
"""
import numpy as np

from . import chain, spectral


def form_argument(C, Xk, y, sigma):
    """M = C - A* y - X^k / sigma  (the argument of Pi), A* y = Diag(y)."""
    C = chain.symmetric_from_upper(C)
    Xk = chain.symmetric_from_upper(Xk)
    return C - np.diag(np.asarray(y, dtype=np.float64)) - Xk / sigma


def s_update(C, Xk, y, sigma, stages, kappas=None, lam=None, exact=False):
    """(S^{k+1}, X^{k+1}, lambda~): the S line with Pi = the composite filter (Algorithm 2,
    ``chain.project``; ``exact=True``: the Higham closed form, ``spectral.eig_project``) and
    the X line, literally as printed."""
    M = form_argument(C, Xk, y, sigma)
    if exact:
        S, lam = spectral.eig_project(M), None
    else:
        S, lam = chain.project(M, stages, kappas, lam=lam)
    X_next = chain.symmetric_from_upper(Xk) + sigma * (S + np.diag(np.asarray(y, dtype=np.float64))
                                                       - chain.symmetric_from_upper(C))
    return S, X_next, lam


def y_update(C, Xk, Sk, sigma, b):
    """y^{k+1} = (A A*)^{-1} (b / sigma - A(X^k / sigma + S^k - C)) with A = diag(.), A A* = I."""
    return b / sigma - np.diag(Xk / sigma + Sk - C)


def kkt_residual(C, X, y, S, b):
    """The KKT surrogate the paper monitors while the filter runs: max of the primal,
    dual and duality-gap terms of eta."""
    pr = np.linalg.norm(np.diag(X) - b) / (1.0 + np.linalg.norm(b))
    du = np.linalg.norm(np.diag(y) + S - C) / (1.0 + np.linalg.norm(C))
    co = abs(np.sum(C * X) - b @ y) / (1.0 + abs(np.sum(C * X)) + abs(b @ y))
    return max(pr, du, co)


def solve(C, sigma, iters, stages=None, kappas=None, exact=False, X0=None, S0=None):
    """Run ``iters`` ADMM iterations from X = S = 0 (or the given start); returns
    (X, y, S, [eta_k]).  b = 1 (max-cut: diag(X) = 1)."""
    n = C.shape[0]
    b = np.ones(n)
    X = np.zeros((n, n)) if X0 is None else X0.copy()
    S = np.zeros((n, n)) if S0 is None else S0.copy()
    etas = []
    y = np.zeros(n)
    for _ in range(iters):
        y = y_update(C, X, S, sigma, b)
        S, X, _ = s_update(C, X, y, sigma, stages, kappas, exact=exact)
        etas.append(kkt_residual(C, X, y, S, b))
    return X, y, S, etas
