"""Sequential Remez (Algorithm 1) with the Remez exchange of
Appendix A (Algorithm app:remez).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Used offline to make
coefficient sets the paper does not print (config c2's T=4, d=7 filter; see
``tools/make_coeffs.py``) and pinned by reproducing Table 2.

Notation follows the paper: target g = f_sign = 1 on [a, b] (Eq. comp:remez-1,
P:L535), basis Phi = {x, x^3, ..., x^d} (odd, d = 2p+1, m = p+1 functions),
m+1 alternation points.
"""
import numpy as np
from scipy.optimize import brentq


def _basis(x, m):
    x = np.asarray(x, dtype=np.float64)
    return np.stack([x ** (2 * l + 1) for l in range(m)], axis=-1)


def _err(c, x):
    """Residual e(x) = sum_l c_l phi_l(x) - g(x), g = 1 (App. A step (2))."""
    return _basis(x, len(c)) @ c - 1.0


def _critical_points(c, lo, hi):
    """Zeros of e'(x) = sum_l (2l+1) c_l x^{2l} in (lo, hi), via the polynomial in u = x^2."""
    m = len(c)
    if m < 2:
        return []
    # e'(u) coefficients, highest degree first for np.roots
    poly = [(2 * l + 1) * c[l] for l in range(m)][::-1]
    out = []
    for u in np.roots(poly):
        if abs(u.imag) > 1e-12 * max(1.0, abs(u.real)) or u.real <= 0:
            continue
        x = np.sqrt(u.real)
        if lo < x < hi:
            out.append(float(x))
    return out


def remez(a, b, d, tol=1e-14, maxit=200):
    """Minimax odd polynomial of degree d for g = 1 on [a, b] (Algorithm app:remez).

    Returns (c, E): c[l] multiplies x^{2l+1}; |E| is the equioscillation level.
    """
    m = (d + 1) // 2
    n_pts = m + 1
    # Initialization: m+1 Chebyshev nodes on [a, b].
    k = np.arange(n_pts)
    x = np.sort((a + b) / 2 + (b - a) / 2 * np.cos(np.pi * (2 * k + 1) / (2 * n_pts)))
    c = None
    E = 0.0
    for _ in range(maxit):
        # (1) alternation system: sum_l c_l phi_l(x_i) - g(x_i) = (-1)^i E
        A = np.zeros((n_pts, m + 1))
        A[:, :m] = _basis(x, m)
        A[:, m] = -((-1.0) ** np.arange(n_pts))
        sol = np.linalg.solve(A, np.ones(n_pts))
        c, E = sol[:m], sol[m]
        # (2) roots z_l of e between consecutive x_i
        z = [a]
        for i in range(n_pts - 1):
            z.append(brentq(lambda t: float(_err(c, t)), x[i], x[i + 1], xtol=1e-300, rtol=1e-15, maxiter=500))
        z.append(b)
        # (3) extremal point of e on each [z_{i-1}, z_i]: max if e(x_i) > 0, min otherwise
        y = np.empty(n_pts)
        for i in range(n_pts):
            lo, hi = z[i], z[i + 1]
            cands = [lo, hi] + _critical_points(c, lo, hi)
            vals = np.array([float(_err(c, t)) for t in cands])
            s = np.sign(float(_err(c, x[i])))
            y[i] = cands[int(np.argmax(s * vals))]
        # (4) convergence
        done = np.max(np.abs(y - x)) <= tol * (b - a) + 1e-300
        x = y
        if done:
            break
    return c, abs(E)


def flat_polynomial(d):
    """Limit of the minimax polynomial when [a, b] collapses to {1}: the odd degree-d
    polynomial with f(1) = 1 and f^{(k)}(1) = 0 for k = 1..p (d=5: 15/8, -10/8, 3/8).
    Table 1 prints it for stages 9-10."""
    m = (d + 1) // 2
    A = np.zeros((m, m))
    for k in range(m):                       # k-th derivative at x = 1
        for l in range(m):
            e = 2 * l + 1
            v = 1.0
            for q in range(k):
                v *= (e - q)
            A[k, l] = v if e >= k else 0.0
    rhs = np.zeros(m)
    rhs[0] = 1.0
    return np.linalg.solve(A, rhs)


def image(c, a, b):
    """[min, max] of f on [a, b] (Eq. comp:update-interval)."""
    cands = [a, b] + _critical_points(np.asarray(c), a, b)
    vals = [float(_basis(t, len(c)) @ np.asarray(c)) for t in cands]
    return min(vals), max(vals)


def sequential_remez(eps, degrees, degenerate_width=1e-7):
    """Algorithm 1: returns (stages, intervals).

    intervals[t] = [a_t, b_t] before stage t, plus the final image [a_{T+1}, b_{T+1}].
    When the interval has collapsed to width < ``degenerate_width`` the Remez system
    is singular; the stage is the flat limit polynomial (see ``flat_polynomial``).
    """
    a, b = float(eps), 1.0
    stages, intervals = [], [(a, b)]
    for d in degrees:
        if b - a < degenerate_width:
            c = flat_polynomial(d)
        else:
            c, _ = remez(a, b, d)
        stages.append(tuple(float(v) for v in c))
        a, b = image(c, a, b)
        intervals.append((a, b))
    return stages, intervals
