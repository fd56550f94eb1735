"""psd_polar (the filter's polar iterate of a general square matrix) against the
float64 polar oracle (oracle/polar.py) with the lambda~ the GPU used; properties at sizes the oracle
does not reach."""
import numpy as np
import pytest

import synth
from oracle import chain, polar, tables

pytestmark = pytest.mark.gpu

HALF = (tables.F_HALF_REFINED, tables.half_kappas(7))
SINGLE = (tables.F_SINGLE_REFINED, tables.single_kappas(10))
TOL = {"fp16": 5e-3, "bf16": 3e-2, "tf32": 5e-3, "fp16x3": 1e-5, "tf32x3": 1e-5}


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2507_09165_b200 as p
    p.load()
    return p


def _run(pkg, A, prec, bound="frobenius", lam_in=None):
    import torch
    single = prec.endswith("x3")
    f = pkg.Filter(pkg.filters.single_filter() if single else pkg.filters.half_filter(), precision=prec, bound=bound)
    Ad = torch.tensor(A, dtype=torch.float32, device="cuda")
    lam = torch.zeros(A.shape[0], dtype=torch.float64, device="cuda")
    li = None if lam_in is None else torch.tensor(lam_in, dtype=torch.float64, device="cuda")
    out = f.polar(Ad, lambda_in=li, lambda_out=lam)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), lam.cpu().numpy(), f


@pytest.mark.parametrize("n,batch,prec", [
    (40, 3, "fp16"),        # A zero-padded to m = 128 (H is 256 x 256)
    (100, 2, "fp16"),
    (257, 1, "bf16"),       # m = 384: three 128-tile rows per block
    (300, 2, "tf32"),
    (160, 2, "fp16x3"),     # FP32-class
    (512, 2, "fp16"),       # m = 512: 128 x 64 tiles (few-tile BN) in both block modes
    (512, 1, "tf32x3"),     # FP32-class with a K range of one accumulation run
    (2048, 2, "fp16"),      # m = 2048: the CTA-pair kernel on its polar tile lists, K ranges of 2048
    (1024, 4, "fp16x3"),    # CTA-pair kernel, split path: K range of two accumulation chunks
    (1024, 4, "tf32"),      # CTA-pair kernel with full (mirrored) operand storage
])
def test_polar_parity(pkg, n, batch, prec):
    A = np.stack([synth.ginibre(n, 7 * n + b) for b in range(batch)])
    U, lam, f = _run(pkg, A, prec)
    assert f.status() == "PSD_OK"
    st, kap = SINGLE if prec.endswith("x3") else HALF
    for b in range(batch):
        assert lam[b] == pytest.approx(polar.frobenius(A[b]), rel=1e-12)
        ref, _ = polar.polar(A[b], st, kap, lam=float(lam[b]))
        err = np.linalg.norm(U[b] - ref) / np.linalg.norm(ref)
        assert err < TOL[prec], (b, err)


def test_polar_of_symmetric_input_matches_sign(pkg):
    """For symmetric A the polar iterate is the sign chain: psd_polar(X) ~ psd_sign(X)."""
    import torch
    X = synth.batch("goe", 200, 2, 41)
    U, lam, f = _run(pkg, X, "fp16")
    S = f.sign(torch.tensor(X, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    for b in range(2):
        assert np.linalg.norm(U[b] - S[b]) / np.linalg.norm(S[b]) < 2 * TOL["fp16"]


@pytest.mark.parametrize("prec", ["fp16", "fp16x3"])
def test_polar_factor_property_large(pkg, prec):
    """n = 1536 with known factors and singular values in [0.05, 1]: the output is within the
    filter's error (sign error ~1e-9 at eps = 1e-3 after the Frobenius scaling puts sigma_min / ||A||_F
    above eps) plus the arithmetic's of the orthogonal polar factor W V^T."""
    n = 1536
    sigma = np.geomspace(1.0, 0.05, n)
    A, W, V = synth.svd_known(n, 5, sigma)
    U, lam, _ = _run(pkg, A[None], prec)
    assert sigma.min() / lam[0] > 1e-3
    Q = W @ V.T
    err = np.linalg.norm(U[0] - Q) / np.sqrt(n)
    assert err < (2e-3 if prec == "fp16" else 1e-5), err


def test_polar_zero_nonfinite_and_user_bound(pkg):
    import torch
    U, lam, f = _run(pkg, np.zeros((1, 64, 64)), "fp16")
    assert lam[0] == 0.0 and not U.any() and f.status() == "PSD_OK"
    A = synth.ginibre(96, 3)[None].copy()
    A[0, 5, 7] = np.nan
    _, _, f = _run(pkg, A, "fp16")
    assert f.status() == "PSD_ENONFINITE"
    A = synth.ginibre(96, 4)[None]
    lam_user = np.array([2.0 * polar.frobenius(A[0])])
    U, lam, f = _run(pkg, A, "fp16", bound="user", lam_in=lam_user)
    assert lam[0] == lam_user[0]
    ref, _ = polar.polar(A[0], *HALF, lam=float(lam_user[0]))
    assert np.linalg.norm(U[0] - ref) / np.linalg.norm(ref) < TOL["fp16"]


def test_polar_lanczos_bound(pkg):
    """PSD_BOUND_LANCZOS: the Theorem-2 bound of H (||H||_2 = ||A||_2) -- a valid bound, tighter than
    ||A||_F, and the output is the oracle's polar iterate with that lambda~."""
    A = np.stack([synth.ginibre(300, 21 + b) for b in range(2)])
    U, lam, f = _run(pkg, A, "fp16", bound="lanczos")
    assert f.status() == "PSD_OK"
    for b in range(2):
        s_max = np.linalg.norm(A[b], 2)
        assert s_max <= lam[b] <= polar.frobenius(A[b]) * (1 + 1e-12)
        assert lam[b] < 0.5 * polar.frobenius(A[b])                 # ~2 sigma_max / ||A||_F for Ginibre
        ref, _ = polar.polar(A[b], *HALF, lam=float(lam[b]))
        assert np.linalg.norm(U[b] - ref) / np.linalg.norm(ref) < TOL["fp16"]


@pytest.mark.parametrize("rows,cols,batch", [(300, 120, 2), (100, 257, 1), (1000, 130, 1),
                                             (600, 1100, 2)])   # wide on the CTA-pair kernel (top-left tiles)
def test_polar_rectangular(pkg, rows, cols, batch):
    """Tall and wide A (psd_polar_rect): parity against the oracle's rectangular definition."""
    import torch
    A = np.stack([np.asarray(synth.ginibre(max(rows, cols), 3 + b), dtype=np.float64)[:rows, :cols]
                  for b in range(batch)])
    f = pkg.Filter(pkg.filters.half_filter())
    lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
    U = f.polar(torch.tensor(A, dtype=torch.float32, device="cuda"), lambda_out=lam).double().cpu().numpy()
    assert f.status() == "PSD_OK" and U.shape == A.shape
    for b in range(batch):
        ref, lam_o = polar.polar(A[b], *HALF)
        assert float(lam[b]) == pytest.approx(lam_o, rel=1e-12)
        assert np.linalg.norm(U[b] - ref) / np.linalg.norm(ref) < TOL["fp16"]


def test_polar_tall_then_wide_same_handle(pkg):
    """One handle, a tall and then a wide input of the same padded edge (the cached runs on H are
    rebuilt for the other Gram side): both match the oracle."""
    import torch
    f = pkg.Filter(pkg.filters.half_filter())
    for rows, cols in [(300, 120), (120, 300), (300, 120)]:
        A = np.asarray(synth.ginibre(300, rows + 2 * cols), dtype=np.float64)[:rows, :cols][None]
        U = f.polar(torch.tensor(A, dtype=torch.float32, device="cuda")).double().cpu().numpy()
        ref, _ = polar.polar(A[0], *HALF)
        assert np.linalg.norm(U[0] - ref) / np.linalg.norm(ref) < TOL["fp16"], (rows, cols)


def test_polar_lanczos_bound_pair_kernel(pkg):
    """The Lanczos bound of H on the CTA-pair path (n = 1024, batch 8: 2m = 2048, 288 tiles)."""
    A = np.stack([synth.ginibre(1024, 61 + b) for b in range(8)])
    U, lam, f = _run(pkg, A, "fp16", bound="lanczos")
    assert f.status() == "PSD_OK"
    for b in (0, 7):
        assert np.linalg.norm(A[b], 2) <= lam[b] <= polar.frobenius(A[b]) * (1 + 1e-12)
        ref, _ = polar.polar(A[b], *HALF, lam=float(lam[b]))
        assert np.linalg.norm(U[b] - ref) / np.linalg.norm(ref) < TOL["fp16"]
