"""Pins of the float64 oracle against what the paper and mathematics fix.

Each test names the passage it pins and is chosen so that a plausible mistake
(dropped term, wrong sign/index, wrong composition order, wrong kappa placement)
fails at least one of them.  No value here comes from the CUDA path.
"""
import numpy as np
import pytest

import synth
from oracle import certify, chain, remez, spectral, tables


# ----------------------------------------------------------- paper tables (data)

def test_tables_match_golden(golden):
    """oracle/tables.py transcribes Tables 1-2 exactly as the golden file."""
    g = golden["paper"]
    for name, tab in [("f_single", tables.F_SINGLE), ("f_single_refined", tables.F_SINGLE_REFINED),
                      ("f_half", tables.F_HALF), ("f_half_refined", tables.F_HALF_REFINED)]:
        assert np.array_equal(np.array(g[name]["stages"]), np.array(tab))
    assert g["n_float_in_unit_interval"]["value"] == 2 * 0x3F800000 + 1


def test_remez_reproduces_table2():
    """Algorithm 1 with eps=1e-3, T=7, d=5 reproduces Table 2 f*_half."""
    st, _ = remez.sequential_remez(1e-3, [5] * 7)
    got, ref = np.array(st), np.array(tables.F_HALF)
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-9


def test_remez_reproduces_table1_with_eps_1e4():
    """Reading R2: Table 1 f*_single is the eps=1e-4 sequential-Remez output."""
    st, _ = remez.sequential_remez(1e-4, [5] * 10)
    got, ref = np.array(st), np.array(tables.F_SINGLE)
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 2e-7
    st3, _ = remez.sequential_remez(1e-3, [5] * 10)
    assert np.max(np.abs(np.array(st3) - ref) / np.abs(ref)) > 0.1   # eps=1e-3 does NOT match


def test_remez_equioscillation_and_flat_limit():
    """App. A: the minimax error equioscillates m+1 times; the flat
    limit 15/8, -10/8, 3/8 is what Table 1 prints for stages 9-10."""
    c, E = remez.remez(0.1, 1.0, 5)
    xs = np.linspace(0.1, 1.0, 200001)
    e = chain.odd_poly_scalar(xs, c) - 1.0
    assert abs(np.max(np.abs(e)) - E) < 1e-9
    assert np.allclose(remez.flat_polynomial(5), [1.875, -1.25, 0.375], atol=1e-15)
    assert np.allclose(np.array(tables.F_SINGLE[8]), remez.flat_polynomial(5), atol=1e-12)
    # Newton-Schulz is the flat limit of degree 3
    assert np.allclose(remez.flat_polynomial(3), tables.NEWTON_SCHULZ_STAGE, atol=1e-15)


def test_interval_identities_draft_theorem():
    """Draft Theorem eq:10-11: a_{t+1} = p_t(a_t), b_{t+1} = 2 - a_{t+1},
    sign error = 1 - a_{T+1}; checked on Table 2 f*_half with the oracle's scalar chain."""
    st = tables.F_HALF
    a = 1e-3
    for c in st:
        a_next = float(chain.odd_poly_scalar(a, c))
        lo, hi = remez.image(c, a, 2 - a if a != 1e-3 else 1.0)
        assert abs(lo - a_next) < 1e-9           # printed coefficients carry 10 digits
        assert abs(hi - (2 - a_next)) < 1e-7
        a = a_next
    xs = np.linspace(1e-3, 1.0, 2_000_001)
    err = np.max(np.abs(chain.scalar_chain(xs, st) - 1.0))
    assert abs(err - (1.0 - a)) < 1e-9
    assert 0 < 1 - a < 1e-9        # [chk-1]: 1 - a_8 = 5.8e-10


# --------------------------------------------------------------- certificate

@pytest.mark.parametrize("name,stages", [("f_half", tables.F_HALF),
                                         ("f_half_refined", tables.F_HALF_REFINED),
                                         ("f_single_refined", tables.F_SINGLE_REFINED)])
def test_e_float_matches_printed(name, stages):
    """e_float printed under Tables 1-2 is 2 x relu_err (reading R3), within 0.5%."""
    e, _, count = certify.relu_err(stages)
    assert count == tables.N_FLOAT_IN_UNIT_INTERVAL
    printed = tables.E_FLOAT_PRINTED[name]
    assert abs(2 * e - printed) / printed < 5e-3


def test_e_float_single_belongs_to_eps1e3_chain():
    """Reading R2: Table 1's printed f*_single e_float (1.1092e-5) is that of the eps=1e-3,
    T=10 chain = f*_half stages 1-7 + 3 flat stages."""
    st = list(tables.F_HALF) + [tuple(remez.flat_polynomial(5))] * 3
    assert abs(certify.paper_convention(st) - 1.1092e-5) / 1.1092e-5 < 5e-3


def test_certificate_kappa_after_last_stage_closed_form():
    """Reading R1: kappa after the LAST stage too makes s -> 1/1.01 on [eps,1], so the ReLU
    error -> 1/2 (1 - 1/1.01) = 4.95e-3 at x = 1 (closed form); kappa on t < T keeps ~1e-4."""
    T = 7
    all_k = [tables.KAPPA_HALF] * T
    e_all, am, _ = certify.relu_err(tables.F_HALF_REFINED, all_k)
    assert abs(e_all - 0.5 * (1 - 1 / 1.01)) < 2e-4 and am > 0.9
    e_r1, _, _ = certify.relu_err(tables.F_HALF_REFINED, tables.half_kappas(T))
    assert e_r1 < 1e-4


def test_certificate_consistent_with_python_scalar_chain():
    """The C certificate's maximiser evaluates to the same error through chain.relu_approx."""
    e, am, _ = certify.relu_err(tables.F_HALF)
    v = abs(float(chain.relu_approx(am, tables.F_HALF)) - max(am, 0.0))
    assert abs(v - e) <= 1e-15
    xs = np.float32(np.linspace(0, 1, 1_000_001)).astype(np.float64)
    grid = np.max(np.abs(chain.relu_approx(xs, tables.F_HALF) - np.maximum(xs, 0)))
    assert grid <= e * (1 + 1e-12)


# --------------------------------------------------------------- matrix chain

def _g(stages, kappas, lam):
    return lambda l: lam * chain.relu_approx(l / lam, stages, kappas)


@pytest.mark.parametrize("n,family,stages,kappas", [
    (8, "goe", tables.F_HALF[:3], None),                           # config c1
    (48, "haar", tables.F_HALF_REFINED, tables.half_kappas(7)),
    (40, "sdp_shaped", tables.F_SINGLE_REFINED, tables.single_kappas(10)),
    (33, "dominant", tables.F_HALF, None),
])
def test_matrix_chain_equals_spectral_operator(n, family, stages, kappas):
    """Algorithm 2 output = Q diag(lam~ f(lambda/lam~)) Q^T, f = 1/2 x(1+s(x))."""
    X = synth.make(family, n, synth.SEED_BASE + n)
    P, lam = chain.project(X, stages, kappas)
    ref = spectral.spectral_apply(X, _g(stages, kappas, lam))
    assert np.linalg.norm(P - ref) <= 1e-12 * max(1.0, np.linalg.norm(ref))
    S, _ = chain.sign(X, stages, kappas)
    refS = spectral.spectral_apply(X, lambda l: chain.scalar_chain(l / lam, stages, kappas))
    assert np.linalg.norm(S - refS) <= 1e-11 * np.sqrt(n)


def test_c1_spectral_identity_vs_jacobi():
    """Config c1 (8x8, T=3 d=5 eps=1e-3): ||P - Pi(X)||_F = sqrt(sum (g(l_i) - relu(l_i))^2)
    with eigenvalues from a textbook Jacobi sweep (independent of LAPACK)."""
    X = synth.goe(8, synth.SEED_BASE + 1)
    st = tables.F_HALF[:3]
    P, lam = chain.project(X, st)
    lj = spectral.jacobi_eigvals(X)
    assert np.allclose(lj, np.linalg.eigvalsh(X), atol=1e-12)
    g = _g(st, None, lam)
    lhs = np.linalg.norm(P - spectral.eig_project(X))
    rhs = np.sqrt(np.sum((g(lj) - np.maximum(lj, 0)) ** 2))
    assert abs(lhs - rhs) < 1e-12 * max(1, rhs)


def test_diagonal_input_equals_scalar_chain(golden):
    """Diagonal X: the matrix chain acts entrywise; SPEC S:L398 example."""
    ex = golden["spec"]["diag_sign"]
    X0 = np.array(ex["X0"])
    S = chain.sign_chain(X0, tables.F_HALF)
    assert np.allclose(np.diag(S), ex["S_diag"], atol=ex["tol"])
    d = np.array([0.9, -0.3, 1e-3, 0.0, -1.0, 0.5])
    S = chain.sign_chain(np.diag(d), tables.F_HALF_REFINED, tables.half_kappas())
    assert np.allclose(np.diag(S), chain.scalar_chain(d, tables.F_HALF_REFINED, tables.half_kappas()), rtol=1e-14, atol=1e-15)
    assert np.count_nonzero(S - np.diag(np.diag(S))) == 0


def test_closed_form_examples(golden):
    for ex in golden["spec"]["eig_project"]:
        assert np.allclose(spectral.eig_project(np.array(ex["X"], float)), ex["P"], atol=1e-14)
    ex = golden["spec"]["rel_error"]
    P = spectral.eig_project(np.array(ex["X"], float))
    assert abs(spectral.rel_error(np.array(ex["cand"]), P) - ex["value"]) < 1e-12


def test_zero_and_degenerate_inputs():
    """lambda~ = 0 -> 0; degree-1 stage = scalar; X0 = 0 stays 0 (oddness)."""
    P, lam = chain.project(np.zeros((5, 5)), tables.F_HALF)
    assert lam == 0 and not P.any()
    X = synth.goe(6, 3)
    S1, lam = chain.sign(X, [(2.0,), (1.5, -0.5)])
    S2, _ = chain.sign(2.0 * X, [(1.5, -0.5)], lam=lam)
    assert np.allclose(S1, S2, rtol=1e-15, atol=1e-16)


def test_gemm_counts(golden):
    for degrees, g in golden["paper"]["gemm_counts"]["cases"]:
        assert chain.gemm_count(degrees) == g


def test_invariants():
    """S(-X) = -S(X) bitwise; P(X) - P(-X) = X; P(2^k X) = 2^k P(X) bitwise (Frobenius lam~)."""
    X = synth.goe(32, 11)
    st, k = tables.F_HALF_REFINED, tables.half_kappas()
    S, _ = chain.sign(X, st, k)
    Sm, _ = chain.sign(-X, st, k)
    assert np.array_equal(Sm, -S)
    P, _ = chain.project(X, st, k)
    Pm, _ = chain.project(-X, st, k)
    assert np.max(np.abs(P - Pm - X)) < 1e-13 * np.max(np.abs(X))
    P8, _ = chain.project(8.0 * X, st, k)
    assert np.array_equal(P8, 8.0 * P)
    assert np.array_equal(P, P.T)


def test_zero_padding_exact():
    """Odd chains map 0 to 0, so padding X with zero rows/cols pads P with zeros."""
    X = synth.goe(20, 5)
    st = tables.F_HALF
    P, lam = chain.project(X, st)
    Xp = np.zeros((28, 28))
    Xp[:20, :20] = X
    Pp, lamp = chain.project(Xp, st)
    assert lam == lamp
    assert np.allclose(Pp[:20, :20], P, rtol=0, atol=1e-14 * np.abs(P).max())
    assert not Pp[20:, :].any() and not Pp[:, 20:].any()


def test_certified_error_bound_and_near_psd():
    """||P - Pi(X)||_2 <= lam~ relu_err, and P >= -lam~ relu_err I."""
    st, k = tables.F_HALF_REFINED, tables.half_kappas()
    e, _, _ = certify.relu_err(st, k)
    for fam in ["goe", "haar", "sdp_shaped"]:
        X = synth.make(fam, 64, 99)
        P, lam = chain.project(X, st, k)
        D = P - spectral.eig_project(X)
        assert np.linalg.norm(D, 2) <= 1.01 * lam * e
        assert np.linalg.eigvalsh(P).min() >= -1.01 * lam * e


def test_structured_oracle_matches_dense():
    """p(H B H^T) = H p(B) H^T for the normalised Hadamard H."""
    n = 256
    X, blocks = synth.structured(n, 42, block=64)
    st, k = tables.F_HALF_REFINED, tables.half_kappas()
    lam = chain.frobenius_bound(X)
    P, _ = chain.project(X, st, k, lam=lam)
    Ps = spectral.structured_project(blocks, st, k, lam)
    assert np.linalg.norm(P - Ps) / np.linalg.norm(P) < 1e-6      # fp32 rounding of X only
    H = spectral.hadamard_conjugate(np.eye(8))
    assert np.allclose(H @ H, np.eye(8), atol=1e-15) and np.allclose(H, H.T)
    # the row-sampled form (used at n = 16384) against the dense conjugation and Algorithm 2 itself
    rows = [0, 1, 77, 128, 255]
    Pr = spectral.structured_project_rows(blocks, st, k, lam, rows)
    assert np.allclose(Pr, Ps[rows], atol=1e-13 * np.abs(Ps).max())
    assert np.linalg.norm(P[rows] - Pr) / np.linalg.norm(P[rows]) < 1e-6


def test_bound_is_upper_bound():
    """||X||_2 <= ||X||_F on every family; upper-triangle read (R10)."""
    for fam in ["goe", "haar", "sdp_shaped", "dominant"]:
        X = synth.make(fam, 50, 7)
        assert np.abs(np.linalg.eigvalsh(X)).max() <= chain.frobenius_bound(X)
    A = synth.rng(1).standard_normal((6, 6))
    assert chain.frobenius_bound(A) == chain.frobenius_bound(np.triu(A) + np.triu(A, 1).T)


# ------------------------------------------------------- pins added in round 2

def _c2_stages():
    """Config c2's T = 4, d = 7 Remez chain (data/remez_filters.json, written by tools/make_coeffs.py
    from oracle/remez.py only)."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "remez_filters.json")
    with open(path) as f:
        return [tuple(c) for c in json.load(f)["c2_T4_d7_eps1e-3"]["stages"]]


@pytest.mark.parametrize("which,eps,rtol,chk10", [
    ("c1", 1e-3, 1e-6, 0.860),      # f*_half stages 1-3 (config c1)
    ("c2", 1e-3, 1e-9, 0.137),      # config c2 (T = 4, d = 7)
    ("c3", 1e-3, 1e-4, 9.16e-4),    # f*_half stages 1-6 (config c3)
    ("half", 1e-3, 2e-3, 5.8e-10),  # f*_half (Table 2, T = 7)
])
def test_sign_err_closed_form(which, eps, rtol, chk10):
    """certify.sign_err (max over float32 x in [eps, 1] of |s(x) - 1|) equals the draft Theorem's
    closed form 1 - a_{T+1} with a_1 = eps, a_{t+1} = f_t(a_t) (eq:10-11): for a
    sequential-Remez chain (Algorithm 1) each stage maps [a_t, 2 - a_t] onto
    [a_{t+1}, 2 - a_{t+1}], so the worst sign error sits at the interval ends.  SURVEY [chk-10]
    values to 3 digits.  rtol follows the printed 10-digit coefficients (the T = 6, 7 chains are
    flat to 1e-4 / 1e-9 and inherit the coefficient rounding)."""
    st = {"c1": tables.F_HALF[:3], "c2": _c2_stages(), "c3": tables.F_HALF[:6], "half": tables.F_HALF}[which]
    a = eps
    for c in st:                           # a_{t+1} = f_t(a_t), the odd monomial sum written out
        a = sum(cj * a ** (2 * j + 1) for j, cj in enumerate(c))
    closed = 1.0 - a
    e, am = certify.sign_err(st, eps)
    assert abs(e - closed) <= rtol * closed, (e, closed)
    assert abs(closed - chk10) <= 5e-3 * chk10 + 1e-12
    assert eps <= am <= 1.0
    assert e >= abs(float(chain.scalar_chain(np.float32(0.5), st)) - 1.0)   # a maximum over [eps, 1]


def test_sign_err_window():
    """sign_err only looks at [eps, 1]: below eps s(x) -> 0 (s is odd, s(0) = 0), so a window that
    started at 0 would report ~1; a larger eps can only shrink the maximum (nested windows)."""
    st = tables.F_HALF
    e3, _ = certify.sign_err(st, 1e-3)
    e2, _ = certify.sign_err(st, 1e-2)
    e_tiny, am = certify.sign_err(st, 1e-6)
    assert e2 <= e3 < 1e-8
    assert e_tiny > 0.99 and am < 1e-3


@pytest.mark.parametrize("X,expected", [
    ([[3.0, 0.0], [0.0, 4.0]], 5.0),                          # diag(3, 4): the 3-4-5 triangle
    ([[1.0, 2.0], [2.0, 1.0]], np.sqrt(10.0)),               # off-diagonal counted twice
    ([[1.0, 2.0], [99.0, 1.0]], np.sqrt(10.0)),              # lower triangle never read (R10)
    ([[2.0, 1.0, 2.0], [0.0, 2.0, 1.0], [0.0, 0.0, 2.0]], np.sqrt(24.0)),
    ([[0.0]], 0.0),
])
def test_frobenius_bound_exact(X, expected):
    """lambda~ = ||X||_F = sqrt(sum_ij x_ij^2) of the upper-triangle symmetric X (R10),
    exact small-integer cases: a missing sqrt, an upper-triangle-only sum or a read of the lower
    triangle each fails one of them."""
    assert chain.frobenius_bound(np.array(X)) == expected


@pytest.mark.parametrize("family,which", [("goe", "half"), ("haar", "half"), ("sdp_shaped", "single"),
                                          ("goe", "c1"), ("dominant", "half")])
def test_idempotence_bound(family, which):
    """Idempotence error bound (BASELINE north star): with e = relu_err (Eq. comp:error-approx,
    P:L583-590), P(X) = Q g(L) Q^T and g(l) >= -lam~ e, and P(P(X)) = Q g'(g(L)) Q^T with
    |g'(m) - relu(m)| <= lam~' e (lam~' = ||P(X)||_F bounds its spectrum), so eigenvalue-wise
    |g'(g(l)) - g(l)| <= lam~' e + lam~ e:
        ||P(P(X)) - P(X)||_2 <= (lam~ + lam~') e,   ||.||_F <= sqrt(n) (lam~ + lam~') e.
    (SURVEY.md's 2 sqrt(n) lam~' e assumes lam~ <= lam~'; the bound above needs no assumption.)
    The exact projection is idempotent; a dropped 1/2 in the return line (P = 2 relu, P(P) = 4 relu)
    or the stabilisation applied after the last stage too (s -> 1/1.01) breaks the bound.  (A
    flipped reconstruction sign, min(X, 0), is idempotent as well: the spectral-operator pins above
    catch that one.)"""
    st, k = {"half": (tables.F_HALF_REFINED, tables.half_kappas()), "single": (tables.F_SINGLE_REFINED,
             tables.single_kappas(10)), "c1": (tables.F_HALF[:3], None)}[which]
    e, _, _ = certify.relu_err(st, k)
    n = 72
    X = synth.make(family, n, synth.SEED_BASE + 71)
    P, lam = chain.project(X, st, k)
    PP, lam2 = chain.project(P, st, k)
    assert lam2 == chain.frobenius_bound(P)
    D = PP - P
    assert np.linalg.norm(D, 2) <= 1.01 * (lam + lam2) * e
    assert np.linalg.norm(D) <= 1.01 * np.sqrt(n) * (lam + lam2) * e
    # and the method really is (nearly) idempotent at the paper's filter accuracy
    if which != "c1":
        assert np.linalg.norm(D) <= 1e-3 * np.linalg.norm(P)


def test_naive_matmul_oracle_agrees_with_blas():
    """The oracle's matrix products are plain float64 matmuls; with the textbook i-k-j triple loop
    swapped in (the north star's "naive matmuls") Algorithm 2 gives the same P on the c1 input and on
    a 24 x 24 GOE matrix with the half filter, to summation-order rounding."""
    from oracle import chain as ch
    X1 = synth.goe(8, synth.SEED_BASE + 1)
    X2 = synth.goe(24, 5)
    cases = [(X1, tables.F_HALF[:3], None), (X2, tables.F_HALF_REFINED, tables.half_kappas(7))]
    ref = [ch.project(X, st, kap)[0] for X, st, kap in cases]
    saved = ch.matmul
    try:
        ch.matmul = ch.naive_matmul
        got = [ch.project(X, st, kap)[0] for X, st, kap in cases]
    finally:
        ch.matmul = saved
    for r, g in zip(ref, got):
        assert np.max(np.abs(r - g)) <= 1e-13 * np.max(np.abs(r))
    A = np.arange(6.0).reshape(2, 3)
    B = np.arange(12.0).reshape(3, 4) - 5.0
    assert np.array_equal(ch.naive_matmul(A, B), A @ B)     # exact on small integers
