"""Seeded synthetic symmetric inputs shared by the tests, the oracle legs and bench.py.

This module holds NONE of the method's arithmetic (no bound, no polynomial, no
projection): it only draws matrices.  Both the CUDA path and the oracle consume
its output; neither is imported here.

Families (the paper's datasets are symmetrised
Matrix-Depot matrices, A_sym = 1/2 (A + A^T), which are not
available offline, so these seeded families stand in for them):

* ``goe``        A ~ N(0,1)^{n x n}, X = 1/2 (A + A^T)          (the P:L777 symmetrisation)
* ``haar``       X = Q diag(lambda) Q^T, Q Haar, lambda_i uniform on [-1,-eps] U [eps, 1]
* ``sdp_shaped`` ADMM S-update argument M = C - A*(y) - X^k / sigma (Eq. exp:admm-three-step,
                 P:L926-937) for a max-cut-like SDP: C = -L/4 of a sparse random graph
                 (average degree 8), A*(y) = diag(y), X^k low-rank PSD (rank n/20), sigma = 1
* ``dominant``   one eigenvalue 1, the rest uniform in [-1e-3, 1e-3] (the paper's failure
                 family, "one dominant extremal eigenvalue")
* ``structured`` X = H B H^T with H the normalised Hadamard matrix (n = 2^k) and B
                 block-diagonal with blocks drawn from one of the families above; the
                 oracle projects it exactly in O(n^2 log n) (oracle/spectral.py).

All generators return float64 numpy arrays that are already rounded to float32
values (the device input is fp32; the oracle then sees exactly the same numbers).
"""
import numpy as np

SEED_BASE = 20250712


def rng(seed):
    return np.random.default_rng(seed)


def _f32(X):
    return np.asarray(X, dtype=np.float32).astype(np.float64)


def goe(n, seed):
    A = rng(seed).standard_normal((n, n))
    return _f32(0.5 * (A + A.T))


def ginibre(n, seed):
    """A general (nonsymmetric) square Gaussian matrix: the input of the polar path (psd_polar)."""
    return _f32(rng(seed + 31337).standard_normal((n, n)))


def svd_known(n, seed, sigma):
    """A = W diag(sigma) V^T with Haar W, V: a general matrix whose polar factor W V^T is known."""
    W = haar_orthogonal(n, seed)
    V = haar_orthogonal(n, seed + 1)
    return _f32((W * np.asarray(sigma)) @ V.T), W, V


def haar_orthogonal(n, seed):
    g = rng(seed).standard_normal((n, n))
    Q, R = np.linalg.qr(g)
    return Q * np.sign(np.diag(R))


def haar(n, seed, eps=1e-3, spectrum=None):
    r = rng(seed + 7919)
    if spectrum is None:
        mag = r.uniform(eps, 1.0, n)
        spectrum = mag * np.where(r.random(n) < 0.5, -1.0, 1.0)
    Q = haar_orthogonal(n, seed)
    X = (Q * np.asarray(spectrum)) @ Q.T
    return _f32(0.5 * (X + X.T))


def dominant(n, seed):
    r = rng(seed + 104729)
    spec = r.uniform(-1e-3, 1e-3, n)
    spec[0] = 1.0
    return haar(n, seed, spectrum=spec)


def sdp_shaped(n, seed, avg_degree=8, rank=None, sigma=1.0):
    r = rng(seed)
    m = int(round(avg_degree * n / 2))
    i = r.integers(0, n, m)
    j = r.integers(0, n, m)
    keep = i != j
    i, j = i[keep], j[keep]
    W = np.zeros((n, n))
    W[i, j] = 1.0
    W[j, i] = 1.0
    deg = W.sum(axis=1)
    y = r.standard_normal(n) - 0.25 * avg_degree
    rank = max(1, n // 20) if rank is None else rank
    V = r.standard_normal((n, rank)) * np.sqrt(avg_degree / (4.0 * n))
    # M = C - diag(y) - X^k / sigma with C = -L/4 = (W - diag(deg)) / 4
    M = V @ V.T
    M *= -1.0 / sigma
    W *= 0.25
    M += W
    del W
    M[np.diag_indices(n)] += -0.25 * deg - y
    M += M.T.copy()
    M *= 0.5
    return _f32(M)


def maxcut_admm(n, seed, avg_degree=8, rank=None):
    """Inputs of one ADMM S-update on a max-cut-like SDP: C = -L/4 of a random
    graph with average degree ``avg_degree`` (as in ``sdp_shaped``), a low-rank PSD iterate X^k
    (rank n/20, the paper's solution ranks) and a dual vector y.  Returns
    (C, Xk, y), fp32-representable float64 arrays.  Holds none of the method's arithmetic."""
    r = rng(seed)
    m = int(round(avg_degree * n / 2))
    i = r.integers(0, n, m)
    j = r.integers(0, n, m)
    keep = i != j
    i, j = i[keep], j[keep]
    W = np.zeros((n, n))
    W[i, j] = 1.0
    W[j, i] = 1.0
    C = 0.25 * (W - np.diag(W.sum(axis=1)))
    rank = max(1, n // 20) if rank is None else rank
    V = r.standard_normal((n, rank)) * np.sqrt(avg_degree / (4.0 * n))
    Xk = V @ V.T
    y = r.standard_normal(n) - 0.25 * avg_degree
    return _f32(C), _f32(0.5 * (Xk + Xk.T)), _f32(y)


def structured_torch(n, seed, block=64, family="goe", device="cuda"):
    """``structured`` computed with torch on `device` (same blocks, same butterflies in the same
    order in float64, so the same fp32 values) -- for n = 16384, where the numpy transform takes
    minutes.  Returns (X as an fp32 torch tensor on `device`, blocks)."""
    import torch
    assert n & (n - 1) == 0 and n % block == 0
    blocks = [make(family, block, seed + 31 * k) for k in range(n // block)]
    B = torch.zeros((n, n), dtype=torch.float64, device=device)
    for k, b in enumerate(blocks):
        B[k * block:(k + 1) * block, k * block:(k + 1) * block] = torch.from_numpy(b)

    def fwht_rows(A):
        h = 1
        while h < n:
            A = A.reshape(n, n // (2 * h), 2, h)
            a0 = A[:, :, 0, :].clone()
            a1 = A[:, :, 1, :]
            A[:, :, 0, :] = a0 + a1
            A[:, :, 1, :] = a0 - a1
            A = A.reshape(n, n)
            h *= 2
        return A / np.sqrt(n)

    X = fwht_rows(fwht_rows(B).T.contiguous()).T.contiguous()
    del B
    X = (0.5 * (X + X.T)).to(torch.float32)
    return X, blocks


FAMILIES = {"goe": goe, "haar": haar, "sdp_shaped": sdp_shaped, "dominant": dominant}


def make(family, n, seed):
    return FAMILIES[family](n, seed)


def batch(family, n, count, seed):
    return np.stack([make(family, n, seed + 1000 * b) for b in range(count)])


# ------------------------------------------------------------- structured (large n)

def _fwht_rows(A):
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[-1]
    h = 1
    while h < n:
        A = A.reshape(A.shape[:-1] + (n // (2 * h), 2, h))
        a0 = A[..., 0, :].copy()
        a1 = A[..., 1, :]
        A[..., 0, :] = a0 + a1
        A[..., 1, :] = a0 - a1
        A = A.reshape(A.shape[:-3] + (n,))
        h *= 2
    return A / np.sqrt(n)


def structured(n, seed, block=64, family="goe"):
    """Returns (X, blocks): X = H blockdiag(blocks) H^T rounded to fp32 values, and the
    blocks such that X is (up to the fp32 rounding of X) exactly that conjugation.

    The fp32 rounding is moved into the blocks' frame is NOT possible, so the caller's
    reference must be computed from X itself where bit-level input identity matters;
    the structured oracle is used with tolerances far above fp32 input rounding.
    """
    assert n & (n - 1) == 0 and n % block == 0
    blocks = [make(family, block, seed + 31 * k) for k in range(n // block)]
    B = np.zeros((n, n))
    for k, b in enumerate(blocks):
        B[k * block:(k + 1) * block, k * block:(k + 1) * block] = b
    X = _fwht_rows(_fwht_rows(B).T).T
    return _f32(0.5 * (X + X.T)), blocks
