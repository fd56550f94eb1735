"""GPU parity of the fused ADMM S/X update (psd_admm_update; Eq. exp:admm-three-step,
P:L926-937) against the float64 oracle (oracle/admm.py), through the C ABI.

Tolerances as tests/test_gpu_parity.py (relative Frobenius error of S vs the oracle with the
GPU's lambda~); X_next = sigma (S - M) carries sigma times the error of S.  The GPU forms M in
fp32 (R22), the oracle in float64: lambda~ agrees to 1e-6 relative, far inside the bars.
"""
import numpy as np
import pytest

import synth
from oracle import admm, chain, tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"fp16": 5e-3, "fp16x3": 1e-5, "tf32": 5e-3, "bf16": 3e-2}
HALF = (tables.F_HALF_REFINED, tables.half_kappas(7))
SINGLE = (tables.F_SINGLE_REFINED, tables.single_kappas(10))


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_09165_b200 as p
    p.load()
    return p


def _inputs(n, batch, seed):
    Cs, Ks, ys = zip(*(synth.maxcut_admm(n, seed + 7 * b) for b in range(batch)))
    return np.stack(Cs), np.stack(Ks), np.stack(ys)


def _dev(a):
    return torch.tensor(a, dtype=torch.float32, device="cuda").contiguous()


def _m32(C, K, y, sigma):
    """M in the fp32 formation of the ABI (R22): (C - K * fl(1/sigma)) - y_i on the diagonal."""
    C32, K32, y32 = (np.asarray(a, dtype=np.float32) for a in (C, K, y))
    M = C32 - K32 * np.float32(1.0 / sigma)
    i = np.arange(C.shape[-1])
    M[..., i, i] -= y32
    return M


@pytest.mark.parametrize("n,batch,prec,sigma", [
    (64, 5, "fp16x3", 1.0),       # batched small-n kernel
    (37, 3, "fp16", 1.3),         # small-n kernel: rows not a multiple of 4 (scalar loads), odd batch
    (200, 2, "fp16", 2.0),        # ragged n, 1-CTA product kernel
    (512, 3, "fp16x3", 0.5),
    (1024, 8, "fp16", 1.0),       # CTA-pair kernel
])
def test_admm_update_parity(pkg, n, batch, prec, sigma):
    C, K, y = _inputs(n, batch, synth.SEED_BASE + 300 + n)
    st = pkg.filters.single_filter() if prec.endswith("x3") else pkg.filters.half_filter()
    ost = SINGLE if prec.endswith("x3") else HALF
    f = pkg.Filter(st, precision=prec)
    S, X = f.admm_update(_dev(C), _dev(K), _dev(y), sigma)
    torch.cuda.synchronize()
    assert f.status() == "PSD_OK"
    S, X = S.double().cpu().numpy(), X.double().cpu().numpy()
    for b in sorted({0, batch - 1}):
        M = admm.form_argument(C[b], K[b], y[b], sigma)
        lam = chain.frobenius_bound(M)
        Sr, Xr, _ = admm.s_update(C[b], K[b], y[b], sigma, *ost, lam=lam)
        e = np.linalg.norm(S[b] - Sr) / np.linalg.norm(Sr)
        assert e <= TOL[prec], (b, e)
        ex = np.linalg.norm(X[b] - Xr) / (sigma * np.linalg.norm(Sr))
        assert ex <= 2 * TOL[prec], (b, ex)
        assert np.array_equal(S[b], S[b].T) and np.array_equal(X[b], X[b].T)


@pytest.mark.parametrize("n,prec", [(64, "fp16"), (37, "fp16x3"), (384, "fp16"), (1024, "fp16")])
def test_admm_update_equals_projection_of_formed_argument(pkg, n, prec):
    """S is bitwise psd_project(M) of the fp32-formed M, and X_next is bitwise fl(sigma) (S - M):
    the fused formation in the bound, scale and epilogue stages changes nothing else; in place
    (S_out = C, X_out = Xk) gives the same bits."""
    batch, sigma = (2 if n < 1024 else 8), 1.5
    C, K, y = _inputs(n, batch, synth.SEED_BASE + 400 + n)
    f = pkg.Filter(pkg.filters.half_filter(), precision=prec)
    S, X = f.admm_update(_dev(C), _dev(K), _dev(y), sigma)
    M32 = _m32(C, K, y, sigma)
    P = f.project(_dev(M32))
    torch.cuda.synchronize()
    S, X, P = (t.cpu().numpy() for t in (S, X, P))
    assert np.array_equal(S, P)
    Mfull = np.stack([np.triu(m) + np.triu(m, 1).transpose() for m in M32])
    assert np.array_equal(X, np.float32(sigma) * (S - Mfull))
    Cd, Kd = _dev(C), _dev(K)
    S2, X2 = f.admm_update(Cd, Kd, _dev(y), sigma, S_out=Cd, X_out=Kd)
    torch.cuda.synchronize()
    assert np.array_equal(S2.cpu().numpy(), S) and np.array_equal(X2.cpu().numpy(), X)


def test_admm_update_arguments(pkg):
    f = pkg.Filter(pkg.filters.half_filter())
    C = _dev(np.eye(128))
    with pytest.raises(pkg.PsdError):
        f.admm_update(C, C.clone(), None, -1.0)
    S, X = f.admm_update(C, torch.zeros_like(C), None, 1.0)      # y = 0, X_k = 0: M = C = I
    torch.cuda.synchronize()
    Sn, Xn = S.cpu().numpy(), X.cpu().numpy()
    P = f.project(C).cpu().numpy()
    assert np.array_equal(Sn, P) and np.array_equal(Xn, np.float32(1.0) * (P - np.eye(128, dtype=np.float32)))


def test_admm_iteration_on_gpu_reaches_warm_start_level(pkg):
    """The paper's use: the three-step ADMM on a max-cut SDP with the S/X
    lines on the GPU (the y line is an n-vector update done with torch here) reaches the
    surrogate KKT level 1e-2 at which the paper switches to the FP64 projection, tracking the
    float64 oracle iteration with the same filter."""
    n, sigma, iters = 256, 3.0, 40
    C, _, _ = synth.maxcut_admm(n, synth.SEED_BASE + 500)
    f = pkg.Filter(pkg.filters.single_filter(), precision="fp16x3")
    Cd = _dev(C)
    X = torch.zeros_like(Cd)
    S = torch.zeros_like(Cd)
    b = torch.ones(n, dtype=torch.float32, device="cuda")
    etas = []
    for _ in range(iters):
        y = (b / sigma - torch.diagonal(X / sigma + S - Cd)).contiguous()       # P:L930, A A* = I
        S, X = f.admm_update(Cd, X, y, sigma, X_out=X)
        torch.cuda.synchronize()
        etas.append(admm.kkt_residual(C, X.double().cpu().numpy(), y.double().cpu().numpy(),
                                      S.double().cpu().numpy(), np.ones(n)))
    _, _, _, etas_o = admm.solve(C, sigma, iters, *SINGLE)
    assert min(etas) < 1e-2, min(etas)
    assert abs(np.log10(etas[-1]) - np.log10(etas_o[-1])) < 0.5, (etas[-1], etas_o[-1])
