"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle.

Tolerances: relative Frobenius error ||P_gpu - P_orc||_F /
||P_orc||_F with the SAME coefficients and the SAME lambda~ (exported by the GPU):
  fp16 <= 5e-3 (BASELINE.json north_star 16-bit bar), bf16 <= 3e-2 (u = 2^-8: the
  5e-3 bar is infeasible for plain bf16, reading R17), tf32 <= 5e-3 (u = 2^-11).
The oracle gets the paper's raw tables with the literal kappa rescale; the GPU gets the
product-side folded coefficients -- the two sides share nothing but the inputs.
"""
import numpy as np
import pytest

import synth
from oracle import chain, spectral, tables

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"fp16": 5e-3, "bf16": 3e-2, "tf32": 5e-3}
# n < 64: a handful of eigenvalues dominate ||P||_F and the fp16 rounding model of this very
# algorithm (operands RN to fp16, fp32 accumulate) reaches 1.6e-2 on 8x8 inputs (DESIGN.md
# "Tolerances"); the 5e-3 bar applies from n = 64 on.
TOL_SMALL_N = {"fp16": 2e-2, "bf16": 8e-2, "tf32": 2e-2}


def tol(prec, n, which="half"):
    if which == "c2" and n < 256:
        # the d=7 Remez filter of config c2 (large alternating coefficients, 11.8/-69.5/128.8/-71)
        # amplifies fp16 operand rounding to ~1.1e-2 at n = 64 in the rounding model of this
        # algorithm; the split-precision small-n path is what meets 5e-3 there.
        return 2 * TOL_SMALL_N[prec]
    return TOL[prec] if n >= 64 else TOL_SMALL_N[prec]


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_09165_b200 as p
    p.load()
    return p


def _lam(X, lam_gpu):
    """The oracle's own bound; the GPU's exported lambda~ must agree with it."""
    lo = chain.frobenius_bound(X)
    assert abs(lam_gpu - lo) <= 1e-9 * max(lo, 1e-300), (lam_gpu, lo)
    return lo


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _gpu(pkg, stages, X, precision, sign=False, inplace=False):
    f = pkg.Filter(stages, precision=precision)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    lam = torch.zeros(X.shape[0], dtype=torch.float64, device="cuda")
    if inplace:
        out = Xd
    else:
        out = torch.full_like(Xd, float("nan"))
    (f.sign if sign else f.project)(Xd, out=out, lambda_out=lam)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), lam.cpu().numpy(), f


HALF = (tables.F_HALF_REFINED, tables.half_kappas(7))
SINGLE = (tables.F_SINGLE_REFINED, tables.single_kappas(10))


def _product_filter(which, pkg):
    return {"half": pkg.filters.half_filter(), "single": pkg.filters.single_filter(),
            "c1": pkg.filters.remez_half_prefix(3), "c3": pkg.filters.remez_half_prefix(6),
            "c2": pkg.filters.c2_filter()}[which]


def _oracle_filter(which):
    from paper_2507_09165_b200 import filters as pf   # c2 coefficients are a data file (inputs)
    return {"half": HALF, "single": SINGLE, "c1": (tables.F_HALF[:3], None), "c3": (tables.F_HALF[:6], None),
            "c2": (pf.c2_filter(), None)}[which]


@pytest.mark.parametrize("n,batch,family,which,prec", [
    (8, 1, "goe", "c1", "fp16"),              # config c1
    (64, 5, "goe", "c2", "fp16"),             # config c2 shape, small batch
    (128, 2, "sdp_shaped", "half", "fp16"),
    (200, 3, "goe", "half", "fp16"),          # ragged: pads to 256
    (300, 2, "haar", "half", "bf16"),
    (257, 1, "dominant", "half", "fp16"),     # one past a tile boundary
    (384, 2, "goe", "single", "tf32"),
    (1024, 1, "goe", "c3", "fp16"),           # config c3
    (1024, 1, "goe", "c3", "bf16"),
])
def test_project_parity(pkg, n, batch, family, which, prec):
    X = synth.batch(family, n, batch, synth.SEED_BASE + n)
    P, lam, f = _gpu(pkg, _product_filter(which, pkg), X, prec)
    assert f.status() == "PSD_OK"
    st, kap = _oracle_filter(which)
    for b in range(batch):
        ref, _ = chain.project(X[b], st, kap, lam=_lam(X[b], lam[b]))
        err = _rel(P[b], ref)
        assert err <= tol(prec, n, which), f"b={b} err={err:.3e}"
        assert np.array_equal(P[b], P[b].T)


@pytest.mark.parametrize("n,prec,batch", [(200, "fp16", 2), (256, "tf32", 2), (1024, "fp16", 8), (1024, "bf16x3", 8)])
def test_sign_parity(pkg, n, prec, batch):
    """psd_sign (S = X_T) on the 1-CTA and the CTA-pair kernels (upper-only operand storage on
    the 16-bit paths) vs the oracle."""
    X = synth.batch("goe", n, batch, 7)
    S, lam, _ = _gpu(pkg, _product_filter("half", pkg), X, prec, sign=True)
    bar = TOL_X3[prec] * 10 if prec in TOL_X3 else tol(prec, n)     # bf16x3: half filter, 1e-3 bar
    for b in sorted({0, batch - 1}):
        ref, _ = chain.sign(X[b], *HALF, lam=_lam(X[b], lam[b]))
        # sign chain output has ||S||_F ~ sqrt(n); relative bar as for P
        assert _rel(S[b], ref) <= bar, _rel(S[b], ref)
        assert np.array_equal(S[b], S[b].T)


def test_sym_product_parity(pkg):
    """One fused product C = alpha A B + beta D (A, B commuting symmetric) vs fp64."""
    n = 320
    X = synth.goe(n, 3) / np.sqrt(n)
    A = X
    B = X @ X
    B = 0.5 * (B + B.T)
    D = synth.goe(n, 4)
    f = pkg.Filter(pkg.filters.half_filter())
    t = lambda M: torch.tensor(M[None], dtype=torch.float32, device="cuda")
    C = f.sym_product(t(A), t(B), t(D), alpha=0.75, beta=-0.5).double().cpu().numpy()[0]
    A32, B32, D32 = (M.astype(np.float32).astype(np.float64) for M in (A, B, D))
    ref = 0.75 * (A32 @ B32) - 0.5 * D32
    ref = np.triu(ref) + np.triu(ref, 1).T          # upper computed, mirrored
    assert _rel(C, ref) < 2e-3
    assert np.array_equal(C, C.T)


@pytest.mark.parametrize("n,prec,which", [
    (192, "fp16", "half"),      # 1-CTA product kernel
    (64, "fp16", "c2"),         # batched small-n kernel: positions 0 and 3 are the two halves of a pair
    (64, "fp16x3", "c2"),
    (33, "fp16", "half"),       # small-n kernel, rows not a multiple of 4 (scalar loads)
])
def test_batch_position_determinism_and_inplace(pkg, n, prec, which):
    """The same matrix at different batch positions gives bitwise-equal output; out == X works
    and equals the out-of-place result bitwise."""
    x = synth.goe(n, 11)
    X = np.stack([x, synth.goe(n, 12), synth.goe(n, 13), x])
    P, _, _ = _gpu(pkg, _product_filter(which, pkg), X, prec)
    assert np.array_equal(P[0], P[3])
    Pi, _, _ = _gpu(pkg, _product_filter(which, pkg), X, prec, inplace=True)
    assert np.array_equal(Pi, P)


@pytest.mark.parametrize("prec", ["fp16", "bf16", "fp16x3", "tf32x3"])
def test_split_k_cluster_matches_single_cta_runs(pkg, prec):
    """n = 1024 on the 1-CTA kernel: batch 1 runs as a CTA pair per 128 x 64 tile (cluster split-K,
    KS = 2: each CTA accumulates one 512-wide K chunk, the st.async push reduction adds the two),
    batch 3 as one CTA per 128 x 128 tile summing its two K runs in TMEM -- on the split precisions
    (R23's chunks) and on the single-pass ones (K halves, product_kchunk).  Same arithmetic
    (sym_gemm_split_k): bitwise-equal products and projections."""
    x = synth.goe(1024, 21)
    X3 = np.stack([synth.goe(1024, 22), x, synth.goe(1024, 23)])
    P1, _, _ = _gpu(pkg, _product_filter("c3", pkg), x[None], prec)
    P3, _, _ = _gpu(pkg, _product_filter("c3", pkg), X3, prec)
    assert np.array_equal(P1[0], P3[1])
    f = pkg.Filter(pkg.filters.half_filter(), precision=prec)
    t1 = torch.tensor(x[None], dtype=torch.float32, device="cuda")
    t3 = torch.tensor(X3, dtype=torch.float32, device="cuda")
    C1 = f.sym_product(t1, t1).cpu().numpy()
    C3 = f.sym_product(t3, t3).cpu().numpy()
    assert np.array_equal(C1[0], C3[1])


def test_zero_nan_and_upper_triangle(pkg):
    """lambda~ = 0 gives 0; a NaN input sets PSD_ENONFINITE; only the upper
    triangle of X is read (reading R10)."""
    X = np.zeros((2, 96, 96))
    X[1] = synth.goe(96, 5)
    P, lam, f = _gpu(pkg, _product_filter("half", pkg), X, "fp16")
    assert lam[0] == 0 and not P[0].any()
    assert f.status() == "PSD_OK"
    Xn = X.copy()
    Xn[1, 3, 7] = np.nan
    _, lam, f = _gpu(pkg, _product_filter("half", pkg), Xn, "fp16")
    assert f.status() == "PSD_ENONFINITE" and np.isnan(lam[1]) and lam[0] == 0
    Xl = X.copy()
    Xl[1][np.tril_indices(96, -1)] = 123.0           # garbage below the diagonal
    Pl, _, _ = _gpu(pkg, _product_filter("half", pkg), Xl, "fp16")
    assert np.array_equal(Pl, P)


@pytest.mark.parametrize("n,batch,prec", [(60, 3, "fp16x3"), (300, 2, "fp16"), (1024, 8, "fp16"), (640, 2, "tf32")])
def test_lower_triangle_never_read(pkg, n, batch, prec):
    """Reading R10 on every kernel path: NaN / Inf below the diagonal changes nothing, bitwise
    (the host pipeline relies on it: it copies only the upper panels host-to-device)."""
    X = synth.batch("goe", n, batch, synth.SEED_BASE + 21 * n)
    P, lam, f = _gpu(pkg, _product_filter("half", pkg), X, prec)
    Xg = X.copy()
    il = np.tril_indices(n, -1)
    for b in range(batch):
        Xg[b][il] = np.where(np.arange(il[0].size) % 2, np.nan, np.inf)
    Pg, lamg, fg = _gpu(pkg, _product_filter("half", pkg), Xg, prec)
    assert fg.status() == "PSD_OK" and np.array_equal(lam, lamg)
    assert np.array_equal(P, Pg)


def test_psd_and_exact_projection_accuracy(pkg):
    """Method accuracy vs the exact Pi(X) (Higham) at n=512 fp16 is at the
    level the paper reports for FP16 (~1e-3, Table 3) on GOE."""
    X = synth.batch("goe", 512, 1, 99)
    P, lam, _ = _gpu(pkg, _product_filter("half", pkg), X, "fp16")
    err = spectral.rel_error(P[0], spectral.eig_project(X[0]))
    assert err < 5e-3


@pytest.mark.parametrize("n,batch,family,prec", [
    (1024, 8, "goe", "fp16"),          # 80 pair tiles: CTA-pair (cta_group::2) kernel
    (2048, 3, "sdp_shaped", "fp16"),   # 108 pair tiles
    (1280, 6, "haar", "bf16"),         # ragged for 256-tiles (1280 = 5 x 256), bf16
    (1024, 8, "goe", "tf32"),
])
def test_pair_kernel_parity(pkg, n, batch, family, prec):
    """Large-n path (persistent CTA-pair kernel, 256x256 tiles): sampled matrices vs oracle."""
    X = synth.batch(family, n, batch, synth.SEED_BASE + 3 * n)
    P, lam, f = _gpu(pkg, _product_filter("half", pkg), X, prec)
    assert f.status() == "PSD_OK"
    for b in sorted({0, batch - 1}):
        ref, _ = chain.project(X[b], *HALF, lam=_lam(X[b], lam[b]))
        assert _rel(P[b], ref) <= tol(prec, n), (b, _rel(P[b], ref))
    for b in range(batch):
        assert np.array_equal(P[b], P[b].T)


def test_c4_full_size_structured(pkg):
    """Config c4 in bench.py's launch configuration (batch 32 x n=4096, fp16, f~*_half+kappa):
    every output exactly symmetric; sampled outputs vs the exact structured oracle
    P(H B H^T) = H P(B) H^T (oracle/spectral.py) with the GPU's lambda~."""
    n, batch = 4096, 32
    mats, blocks = [], []
    for b in range(batch):
        Xb, bl = synth.structured(n, synth.SEED_BASE + 17 * b, block=64, family="goe" if b % 2 else "sdp_shaped")
        mats.append(Xb)
        blocks.append(bl)
    X = np.stack(mats)
    P, lam, f = _gpu(pkg, _product_filter("half", pkg), X, "fp16")
    assert f.status() == "PSD_OK"
    for b in range(batch):
        assert np.array_equal(P[b], P[b].T)
    for b in [0, 1, 17, 31]:
        ref = spectral.structured_project(blocks[b], *HALF, _lam(X[b], lam[b]))
        assert _rel(P[b], ref) <= TOL["fp16"], (b, _rel(P[b], ref))


# FP32-class split path (3 tcgen05 passes hi*hi + hi*lo + lo*hi): BASELINE north star bar 1e-5.
# bf16x3 carries 2 x 8 significand bits (u ~ 2^-16): bar 1e-4.
TOL_X3 = {"fp16x3": 1e-5, "tf32x3": 1e-5, "bf16x3": 1e-4}


@pytest.mark.parametrize("n,batch,family,which,prec", [
    (8, 1, "goe", "c1", "fp16x3"),            # config c1 on the FP32-class path
    (64, 6, "goe", "c2", "fp16x3"),           # config c2 filter meets 5e-3 (and 1e-5) here
    (256, 2, "sdp_shaped", "single", "fp16x3"),
    (256, 2, "haar", "single", "tf32x3"),
    (300, 1, "goe", "half", "bf16x3"),
    (1024, 8, "goe", "single", "fp16x3"),     # CTA-pair kernel, split
    (1024, 8, "sdp_shaped", "single", "tf32x3"),
    (1024, 1, "goe", "c3", "fp16x3"),         # config c3, FP32-class (cluster split-K)
    (1024, 1, "goe", "c3", "tf32x3"),
])
def test_split_precision_parity(pkg, n, batch, family, which, prec):
    X = synth.batch(family, n, batch, synth.SEED_BASE + 5 * n)
    P, lam, f = _gpu(pkg, _product_filter(which, pkg), X, prec)
    assert f.status() == "PSD_OK"
    st, kap = _oracle_filter(which)
    for b in sorted({0, batch - 1}):
        ref, _ = chain.project(X[b], st, kap, lam=_lam(X[b], lam[b]))
        err = _rel(P[b], ref)
        # the coarse Remez sets (c1: T=3, sign error 0.86; c2: d=7, coefficients up to 128.8)
        # amplify fp32 accumulation rounding: model with sgemm-style fp32 accumulation 6-9e-6
        # at n=64
        bar = 5e-5 if which in ("c1", "c2") else TOL_X3[prec]
        assert err <= bar, f"b={b} err={err:.3e}"
        assert np.array_equal(P[b], P[b].T)


def test_split_sign_parity(pkg):
    X = synth.batch("goe", 512, 2, 77)
    S, lam, _ = _gpu(pkg, _product_filter("single", pkg), X, "fp16x3", sign=True)
    for b in range(2):
        ref, _ = chain.sign(X[b], *SINGLE, lam=_lam(X[b], lam[b]))
        assert _rel(S[b], ref) <= 1e-5


@pytest.mark.parametrize("n,batch,family,which,prec", [
    (64, 4096, "goe", "c2", "fp16x3"),        # config c2, bench launch configuration
    (64, 4096, "goe", "c2", "fp16"),
    (8, 3, "goe", "c1", "fp16x3"),            # config c1 through the small path, odd batch
    (33, 7, "sdp_shaped", "half", "fp16x3"),  # ragged n (zero padded to 64)
    (50, 5, "haar", "single", "fp16"),
])
def test_small_batch_parity(pkg, n, batch, family, which, prec):
    """Batched small-n kernel (n <= 64): whole chain on-chip; sampled matrices vs oracle,
    every output exactly symmetric."""
    X = synth.batch(family, n, batch, synth.SEED_BASE + 11 * n) if batch <= 64 else \
        np.stack([synth.goe(n, synth.SEED_BASE + 7 * b) for b in range(batch)])
    P, lam, f = _gpu(pkg, _product_filter(which, pkg), X, prec)
    assert f.status() == "PSD_OK"
    st, kap = _oracle_filter(which)
    bar = (5e-5 if which in ("c1", "c2") else 1e-5) if prec == "fp16x3" else tol(prec, n, which)
    for b in sorted({0, 1, batch // 2, batch - 1}):
        ref, _ = chain.project(X[b], st, kap, lam=_lam(X[b], lam[b]))
        err = _rel(P[b], ref)
        assert err <= bar, f"b={b} err={err:.3e}"
    assert all(np.array_equal(P[b], P[b].T) for b in range(0, batch, max(1, batch // 64)))


def test_small_batch_sign_and_nonfinite(pkg):
    X = synth.batch("goe", 40, 4, 123)
    S, lam, f = _gpu(pkg, _product_filter("half", pkg), X, "fp16x3", sign=True)
    for b in range(4):
        ref, _ = chain.sign(X[b], *HALF, lam=_lam(X[b], lam[b]))
        assert _rel(S[b], ref) <= 1e-5
        assert np.array_equal(S[b], S[b].T)
    Xn = X.copy()
    Xn[2, 5, 9] = np.inf
    _, lam, f = _gpu(pkg, _product_filter("half", pkg), Xn, "fp16")
    assert f.status() == "PSD_ENONFINITE" and np.isnan(lam[2])


def test_project_host_pipeline(pkg):
    """psd_project_host (chunked H2D / project / D2H on three streams) equals psd_project bitwise,
    including a ragged last chunk and in-place output."""
    X = synth.batch("goe", 384, 7, 31)
    f = pkg.Filter(pkg.filters.half_filter())
    Xh = torch.tensor(X, dtype=torch.float32).pin_memory()
    out = f.project_host(Xh, chunks=3)
    torch.cuda.synchronize()
    ref = f.project(Xh.cuda()).cpu()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    Xh2 = Xh.clone().pin_memory()
    f.project_host(Xh2, Xh2, chunks=2)
    torch.cuda.synchronize()
    assert torch.equal(Xh2, ref)


@pytest.mark.parametrize("n,batch,chunks", [(256, 7, 7), (128, 9, 4), (128, 13, 5), (96, 30, 7)])
def test_project_host_chunking(pkg, n, batch, chunks):
    """Chunk plans of psd_project_host (half-size first / last chunks, more chunks than the 6 chunk
    buffers: a chunk's host-to-device copy waits for the device-to-host copy of the chunk that last
    used its buffer) -- results bitwise equal to psd_project.  (9, 4) and (13, 5) are chunk plans
    whose tail fix-up once produced a chunk larger than the buffers."""
    X = synth.batch("goe", n, batch, 37 + batch)
    f = pkg.Filter(pkg.filters.half_filter())
    Xh = torch.tensor(X, dtype=torch.float32).pin_memory()
    ref = f.project(Xh.cuda()).cpu()
    for _ in range(2):
        out = f.project_host(Xh, chunks=chunks)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


# Lanczos bound (Algorithm 2 line 1 + Theorem 2; reading R21).  The GPU runs the
# Krylov iteration on the operand copy of X / ||X||_F in fp32 vectors: lambda~ agrees with the
# float64 oracle (oracle/bound.py) to the operand rounding (fp16: u = 2^-11 per entry; tf32 op
# copies are exact fp32) plus fp32 Lanczos rounding.
LZ_TOL = {"fp16": 2e-3, "tf32": 1e-4, "bf16": 1e-2}


@pytest.mark.parametrize("n,batch,family,prec", [
    (10, 2, "goe", "tf32"),            # n < steps: the Krylov space is all of R^n
    (200, 3, "goe", "fp16"),           # ragged
    (512, 2, "sdp_shaped", "fp16"),
    (384, 2, "haar", "tf32"),
    (256, 2, "goe", "bf16"),
])
def test_lanczos_bound_parity(pkg, n, batch, family, prec):
    from oracle import bound
    X = synth.batch(family, n, batch, synth.SEED_BASE + 3 * n)
    f = pkg.Filter(pkg.filters.half_filter(), precision=prec, bound="lanczos")
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
    P = f.project(Xd, lambda_out=lam)
    torch.cuda.synchronize()
    assert f.status() == "PSD_OK"
    lam = lam.cpu().numpy()
    P = P.double().cpu().numpy()
    for b in range(batch):
        lo = bound.lanczos_bound(X[b], steps=20, safety=1.01)
        assert abs(lam[b] - lo) <= LZ_TOL[prec] * lo, (b, lam[b], lo)
        s2 = np.linalg.norm(X[b], 2)
        assert s2 <= lam[b] <= 1.03 * s2                 # valid and ~sqrt(n)/2 x tighter than ||X||_F
        ref, _ = chain.project(X[b], *HALF, lam=lo)
        assert _rel(P[b], ref) <= tol(prec, n) + 4 * LZ_TOL[prec], (b, _rel(P[b], ref))
        assert np.array_equal(P[b], P[b].T)


def test_lanczos_bound_accuracy_gain(pkg):
    """The tighter bound moves the spectrum of X_0 out of the filter's transition
    region: in float64 the half filter's method error vs the exact projection drops ~2x on GOE
    n = 768 (oracle: 6.3e-5 -> 3.5e-5).  fp16/tf32 rounding (~1e-3) hides that, so the check runs
    on the FP32-class split path, whose rounding (~1e-6) is below the method error."""
    X = synth.batch("goe", 768, 1, 31)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    exact = spectral.eig_project(X[0])
    errs = {}
    for bnd in ("frobenius", "lanczos"):
        f = pkg.Filter(pkg.filters.half_filter(), precision="fp16x3", bound=bnd)
        P = f.project(Xd).double().cpu().numpy()[0]
        errs[bnd] = spectral.rel_error(P, exact)
    assert errs["lanczos"] < 0.75 * errs["frobenius"], errs


def test_lanczos_bound_edge_cases(pkg):
    """Zero matrix keeps lambda~ = 0; rank one gives ||u||^2; identity gives 1 -- up to the
    operand rounding: the Krylov run sees the operand copy of X / ||X||_F, whose entries carry
    u = 2^-11 (fp16 and tf32 both keep 10 fraction bits); for I / sqrt(n) every entry rounds
    the same way, so the deficit is that rounding itself (reading R21; the default safety
    1.01 covers it)."""
    n = 160
    u = synth.goe(n, 1)[0]
    X = np.stack([np.zeros((n, n)), np.outer(u, u), np.eye(n)]).astype(np.float32).astype(np.float64)
    f = pkg.Filter(pkg.filters.half_filter(), precision="tf32", bound="lanczos", lanczos_safety=1.0)
    lam = torch.zeros(3, dtype=torch.float64, device="cuda")
    P = f.project(torch.tensor(X, dtype=torch.float32, device="cuda"), lambda_out=lam).double().cpu().numpy()
    lam = lam.cpu().numpy()
    assert lam[0] == 0 and not P[0].any()
    assert lam[1] == pytest.approx(np.linalg.norm(X[1], 2), rel=1e-5)
    assert abs(lam[2] - 1.0) <= 2.0 ** -11


@pytest.fixture(scope="module")
def c5_input(pkg):
    """One n = 16384 structured input on the GPU (synth.structured_torch), its blocks and the
    oracle's Frobenius bound, shared by the c5 full-size tests."""
    n = 16384
    Xd, blocks = synth.structured_torch(n, synth.SEED_BASE + 16384, block=64, family="goe")
    lam = chain.frobenius_bound(Xd.cpu().numpy())
    return Xd, blocks, lam


@pytest.mark.parametrize("mode", ["single_gpu", "p2p_virtual_8"])
def test_c5_full_size_structured(pkg, c5_input, mode):
    """Config c5 at its full size (one n = 16384 matrix, fp16, f~*_half+kappa): on one GPU through
    the CTA-pair kernel, and in the launch configuration of the 8-GPU bench -- 8 row-panel ranks of
    the peer-memory path, all regions on this GPU.  Sampled rows vs the exact structured oracle
    P(H B H^T) = H P(B) H^T (oracle/spectral.py, row-sampled form); output exactly symmetric on a
    sampled block."""
    Xd, blocks, lam = c5_input
    f = pkg.Filter(_product_filter("half", pkg), precision="fp16")
    if mode == "single_gpu":
        lam_d = torch.zeros(1, dtype=torch.float64, device="cuda")
        P = f.project(Xd[None], lambda_out=lam_d)[0]
        torch.cuda.synchronize()
        assert abs(float(lam_d[0]) - lam) <= 1e-9 * lam
    else:
        P = f.project_rowpanel_p2p_virtual(Xd, 8)
        torch.cuda.synchronize()
    assert f.status() == "PSD_OK"
    rows = [0, 1, 2047, 2048, 5000, 8191, 12345, 16383]
    Pr = P[rows].double().cpu().numpy()
    ref = spectral.structured_project_rows(blocks, *HALF, lam, rows)
    assert _rel(Pr, ref) <= TOL["fp16"], _rel(Pr, ref)
    blk = P[8000:8200, 3000:3200].cpu().numpy()
    assert np.array_equal(blk, P[3000:3200, 8000:8200].cpu().numpy().T)


@pytest.mark.parametrize("which", ["half", "single", "c2", "c3"])
def test_certificate_on_device(pkg, which):
    """psd_filter_certificate (every float32 in [0, 1] on the device, fp64, the folded chain the
    handle holds) vs the oracle's C certificate (raw tables, literal kappa; oracle/certify.c)."""
    from oracle import certify
    st, kap = _oracle_filter(which)
    f = pkg.Filter(_product_filter(which, pkg), eps=1e-3)
    c = f.certificate()
    e, am, _ = certify.relu_err(st, kap)
    s, sam = certify.sign_err(st, 1e-3, kap)
    assert abs(c["relu_err"] - e) <= 1e-9 * e, (c["relu_err"], e)
    assert abs(c["sign_err"] - s) <= 1e-9 * s, (c["sign_err"], s)
    assert 0.0 < c["relu_argmax"] <= 1.0 and 1e-3 <= c["sign_argmax"] <= 1.0


@pytest.mark.parametrize("n", [1, 2, 3, 63, 64, 65, 127, 128, 129, 255, 256, 1023, 1025])
def test_boundary_sizes(pkg, n):
    """Every padding / path boundary: n = 1..3 and around 64 (small-n kernel / tile kernels), 128
    and 256 (tile multiples) and 1024 (CTA-pair threshold): parity, exact symmetry, and a
    positive-semidefinite result up to the certified error."""
    batch = 3
    X = synth.batch("goe", n, batch, synth.SEED_BASE + 7 * n)
    P, lam, f = _gpu(pkg, _product_filter("half", pkg), X, "fp16x3")
    assert f.status() == "PSD_OK"
    for b in range(batch):
        lo = _lam(X[b], lam[b])
        ref, _ = chain.project(X[b], *HALF, lam=lo)
        # error on the problem's own scale lambda~ = ||X||_F: for n = 1, 2 every eigenvalue can be
        # negative, and then ||P|| itself is filter-error sized (1/2 x (1 - s(1))) and a relative
        # error says nothing
        err = np.linalg.norm(P[b] - ref) / lo
        assert err <= 1e-5, (b, err)
        assert np.array_equal(P[b], P[b].T)
        if n == 1:                                     # the scalar case: P = relu(x) up to the filter error
            assert abs(P[b][0, 0] - max(X[b][0, 0], 0.0)) <= 1e-2 * abs(X[b][0, 0])


# FP32-class bar at the north-star sizes.  The tensor cores' fp32 accumulator loses ~2^-24 relative
# per accumulating MMA (one n = 4096 product: 1.7e-5, profiles/r1s3_accumulation_error.txt); the
# split path accumulates K in independent runs of 512 summed round-to-nearest (reading R23).
@pytest.mark.parametrize("n,batch,family,prec", [
    (2048, 1, "dominant", "fp16x3"),   # 1-CTA kernel (36 tiles): 4 K runs in separate TMEM columns
    (2048, 1, "goe", "tf32x3"),
    (2048, 3, "dominant", "fp16x3"),   # CTA-pair kernel (108 tiles): K chunks folded by the epilogue
    (2048, 3, "goe", "tf32x3"),
    (2560, 2, "sdp_shaped", "fp16x3"), # ragged for 256-tiles? (2560 = 10 x 256), pair kernel
])
def test_split_fp32_bar_large_n(pkg, n, batch, family, prec):
    """The north-star FP32 bar (1e-5) at n >= 2048, incl. the paper's failure family."""
    X = synth.batch(family, n, batch, 2948 + n)
    P, lam, f = _gpu(pkg, pkg.filters.single_filter(), X, prec)
    assert f.status() == "PSD_OK"
    for b in sorted({0, batch - 1}):
        ref, _ = chain.project(X[b], tables.F_SINGLE_REFINED, tables.single_kappas(10), lam=_lam(X[b], lam[b]))
        assert _rel(P[b], ref) <= TOL_X3[prec], (b, _rel(P[b], ref))
        assert np.array_equal(P[b], P[b].T)


@pytest.mark.parametrize("n,batch", [(2048, 1), (4096, 1)])
def test_split_accumulation_runs(pkg, n, batch):
    """One split product C = X X with fp16-exact symmetric X (operand conversion exact, so only the
    accumulation errs): K runs of 512 bring the relative error under 3e-6 on both product kernels
    (n = 2048 batch 1: 1-CTA kernel; n = 4096: CTA-pair kernel), while one hardware accumulation over
    K = n (kchunk 0) is ~4e-9 n (reading R23)."""
    rng = np.random.default_rng(5)
    G = rng.standard_normal((n, n))
    X = ((G + G.T) / 2).astype(np.float16).astype(np.float64)
    ref = X @ X
    iu = np.triu_indices(n)
    t = torch.tensor(X[None], dtype=torch.float32, device="cuda")
    errs = {}
    for kc in (0, 512):
        f = pkg.Filter(pkg.filters.half_filter(), precision="fp16x3", accum_chunk=kc)
        C = f.sym_product(t, t).double().cpu().numpy()[0]
        errs[kc] = np.linalg.norm((C - ref)[iu]) / np.linalg.norm(ref[iu])
        assert np.array_equal(C, C.T)
    assert errs[512] <= 3e-6, errs
    assert errs[0] >= 2e-9 * n, errs        # the hardware effect the runs remove (documents R23)


@pytest.mark.parametrize("prec", ["fp16x3", "tf32x3"])
def test_c4_full_size_structured_fp32(pkg, prec):
    """Config c4 on the FP32-class path in bench.py's launch configuration: batch 32 x n = 4096,
    f~*_single + kappa (T = 10, 31 products), sampled outputs vs the exact structured oracle at the
    north-star 1e-5 bar; every output exactly symmetric."""
    n, batch = 4096, 32
    mats, blocks = [], []
    for b in range(batch):
        Xb, bl = synth.structured(n, synth.SEED_BASE + 19 * b, block=64,
                                  family=("goe", "sdp_shaped", "dominant")[b % 3])
        mats.append(Xb)
        blocks.append(bl)
    X = np.stack(mats)
    P, lam, f = _gpu(pkg, _product_filter("single", pkg), X, prec)
    assert f.status() == "PSD_OK"
    for b in range(batch):
        assert np.array_equal(P[b], P[b].T)
    for b in [0, 1, 2, 17, 31]:
        ref = spectral.structured_project(blocks[b], *SINGLE, _lam(X[b], lam[b]))
        assert _rel(P[b], ref) <= TOL_X3[prec], (b, _rel(P[b], ref))


def test_c5_full_size_structured_fp32(pkg, c5_input):
    """Config c5 (one n = 16384) on the FP32-class path (fp16x3, f~*_single + kappa): sampled rows
    vs the exact structured oracle at the 1e-5 bar."""
    Xd, blocks, lam = c5_input
    f = pkg.Filter(_product_filter("single", pkg), precision="fp16x3")
    lam_d = torch.zeros(1, dtype=torch.float64, device="cuda")
    P = f.project(Xd[None], lambda_out=lam_d)[0]
    torch.cuda.synchronize()
    assert f.status() == "PSD_OK"
    assert abs(float(lam_d[0]) - lam) <= 1e-9 * lam
    rows = [0, 1, 2047, 2048, 5000, 8191, 12345, 16383]
    Pr = P[rows].double().cpu().numpy()
    ref = spectral.structured_project_rows(blocks, *SINGLE, lam, rows)
    assert _rel(Pr, ref) <= TOL_X3["fp16x3"], _rel(Pr, ref)


# Baseline filters through the same path: Newton-Schulz g(x) = 1/2 x (3 - x^2)
# (10 / 15 iterations = 21 / 31 GEMMs) -- degree-3 stages take the p = 1
# plan branch (Z' = c_0 Z + c_1 Z Y, two products per stage) -- and chains with degree-1 stages
# (reading R7: a scalar, folded into the neighbouring products).
NS = (1.5, -0.5)
DEG1_CHAIN = [(2.0,), NS, NS, (0.9,), NS, NS, NS, (1.1,)]      # leading, inner and trailing degree-1 stages


@pytest.mark.parametrize("n,batch,iters,prec", [
    (64, 40, 10, "fp16"),        # small-n kernel
    (64, 40, 15, "fp16x3"),
    (256, 2, 10, "fp16"),        # 1-CTA kernel
    (256, 2, 15, "fp16x3"),
    (1024, 8, 10, "fp16"),       # CTA-pair kernel
    (1024, 8, 15, "fp16x3"),
    (640, 3, 10, "tf32"),
])
def test_newton_schulz_parity(pkg, n, batch, iters, prec):
    X = synth.batch("goe", n, batch, synth.SEED_BASE + 23 * n + iters)
    f = pkg.Filter(pkg.filters.newton_schulz(iters), precision=prec)
    assert f.gemm_count(True) == 2 * iters + 1                   # 21 / 31
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
    P = f.project(Xd, lambda_out=lam).double().cpu().numpy()
    S = f.sign(Xd).double().cpu().numpy()
    assert f.status() == "PSD_OK"
    bar = TOL_X3.get(prec) or tol(prec, n)
    for b in sorted({0, batch - 1}):
        lo = _lam(X[b], float(lam[b]))
        ref, _ = chain.project(X[b], [tables.NEWTON_SCHULZ_STAGE] * iters, lam=lo)
        assert _rel(P[b], ref) <= bar, (b, _rel(P[b], ref))
        refS, _ = chain.sign(X[b], [tables.NEWTON_SCHULZ_STAGE] * iters, lam=lo)
        assert _rel(S[b], refS) <= bar, (b, _rel(S[b], refS))
        assert np.array_equal(P[b], P[b].T)


@pytest.mark.parametrize("n,batch,prec", [(48, 9, "fp16x3"), (300, 2, "fp16"), (1024, 8, "fp16x3"), (256, 1, "tf32")])
def test_degree1_stages_parity(pkg, n, batch, prec):
    """Degree-1 stages (scalars, 0 products) before, between and after degree-3 stages."""
    X = synth.batch("haar", n, batch, synth.SEED_BASE + 29 * n)
    f = pkg.Filter(DEG1_CHAIN, precision=prec)
    assert f.gemm_count(True) == 2 * 5 + 1
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
    P = f.project(Xd, lambda_out=lam).double().cpu().numpy()
    S = f.sign(Xd).double().cpu().numpy()
    bar = TOL_X3.get(prec) or tol(prec, n)
    for b in sorted({0, batch - 1}):
        lo = _lam(X[b], float(lam[b]))
        ref, _ = chain.project(X[b], DEG1_CHAIN, lam=lo)
        assert _rel(P[b], ref) <= bar, (b, _rel(P[b], ref))
        refS, _ = chain.sign(X[b], DEG1_CHAIN, lam=lo)
        assert _rel(S[b], refS) <= bar, (b, _rel(S[b], refS))


def test_coefficient_file_roundtrip(pkg, tmp_path):
    """A coefficient file (SPEC S:L213 JSON: epsilon, T, degrees, stages, provenance; optional
    stabilisation kappas folded offline, reading R1) gives the same projection as the coefficient
    tuples it holds."""
    import json
    path = tmp_path / "half.json"
    json.dump({"epsilon": 1e-3, "T": 7, "degrees": [5] * 7, "stages": [list(c) for c in pkg.filters.HALF_REFINED],
               "kappas": [1 / 1.01] * 6 + [1.0], "provenance": "Table 2 right column (P:L671-677)"},
              open(path, "w"))
    X = torch.tensor(synth.batch("goe", 300, 2, 5), dtype=torch.float32, device="cuda")
    a = pkg.Filter.from_file(str(path)).project(X)
    b = pkg.Filter(pkg.filters.half_filter()).project(X)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
