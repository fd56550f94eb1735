"""B200-native PSD-cone projection by composite polynomial filtering (arXiv 2507.09165).

Thin Python binding over the C ABI of ``include/psd_filter.h`` (libpsdfilter.so).
PyTorch supplies device memory and streams only; every step of the projection --
the Frobenius bound, the scale/convert, the T-stage chain of fused symmetric
products and the reconstruction -- runs in this package's sm_100a kernels.

    import torch
    from paper_2507_09165_b200 import Filter, filters
    f = Filter(filters.half_filter(), precision="fp16")
    P = f.project(X)            # X: (n, n) or (batch, n, n) float32 CUDA tensor

Names follow the paper: ``project`` is Algorithm 2, ``sign`` returns
X_T (the matrix-sign approximation), ``gemm_count`` the GEMM budget.
"""
import ctypes

from . import dist, filters  # noqa: F401
from ._lib import BOUNDS, PRECISIONS, PsdError, check, load  # noqa: F401

__all__ = ["Filter", "filters", "PsdError", "version"]


def version():
    return load().psd_version().decode()


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check_matrix(X):
    import torch
    if not isinstance(X, torch.Tensor) or not X.is_cuda or X.dtype != torch.float32:
        raise TypeError("X must be a float32 CUDA tensor")
    if X.dim() == 2:
        Xb = X.unsqueeze(0)
    elif X.dim() == 3:
        Xb = X
    else:
        raise ValueError("X must be (n, n) or (batch, n, n)")
    if Xb.shape[-1] != Xb.shape[-2]:
        raise ValueError("X must be square")
    if not Xb.is_contiguous():
        raise ValueError("X must be contiguous")
    return Xb


class Filter:
    """A composite polynomial filter f_T o ... o f_1 (Eq. composite-polynomial-filter).

    stages    sequence of coefficient tuples (c_{t,0}, c_{t,1}, ...) of x, x^3, ...;
              stabilisation factors already folded (see ``filters``).
    precision 'fp16' (default, the paper's half path), 'bf16', 'tf32', 'tf32x3'.
    bound     'frobenius' (lambda~ = ||X||_F on device), 'lanczos' (Algorithm 2 line 1:
              Theorem 2 bound from a ``lanczos_steps``-step Lanczos run on X^2, times
              ``lanczos_safety``; never looser than Frobenius) or 'user'
              (pass lambda_in).
    """

    def __init__(self, stages, eps=1e-3, precision="fp16", bound="frobenius", lanczos_steps=20, lanczos_safety=1.01,
                 accum_chunk=None):
        self._lib = load()
        self.stages = [tuple(float(v) for v in c) for c in stages]
        degrees, coeffs = filters.flatten(self.stages)
        self.degrees = degrees
        d = (ctypes.c_int * len(degrees))(*degrees)
        c = (ctypes.c_double * len(coeffs))(*coeffs)
        h = ctypes.c_void_p()
        check(self._lib.psd_filter_create(len(degrees), d, c, float(eps), ctypes.byref(h)), "psd_filter_create")
        self._h = h
        self.precision = precision
        self.bound = bound
        check(self._lib.psd_filter_set_precision(self._h, PRECISIONS[precision]), "psd_filter_set_precision")
        check(self._lib.psd_filter_set_bound(self._h, BOUNDS[bound]), "psd_filter_set_bound")
        check(self._lib.psd_filter_set_lanczos(self._h, int(lanczos_steps), float(lanczos_safety)), "psd_filter_set_lanczos")
        if accum_chunk is not None:
            self.set_accum_chunk(accum_chunk)

    @classmethod
    def from_file(cls, path, **kw):
        """A filter from a coefficient file (``filters.load_coefficient_file``: SPEC S:L213 JSON)."""
        stages, eps, _ = filters.load_coefficient_file(path)
        return cls(stages, eps=kw.pop("eps", eps), **kw)

    def set_accum_chunk(self, kchunk):
        """Split (x3) precisions: K elements per independent accumulation run (0 = one run)."""
        check(self._lib.psd_filter_set_accum_chunk(self._h, int(kchunk)), "psd_filter_set_accum_chunk")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.psd_filter_destroy(h)
            self._h = None

    def gemm_count(self, for_project=True):
        return self._lib.psd_filter_gemm_count(self._h, 1 if for_project else 0)

    def workspace_bytes(self, n, batch=1):
        return self._lib.psd_workspace_bytes(self._h, n, batch)

    def _run(self, X, out, lambda_in, lambda_out, want_sign, stream):
        import torch
        Xb = _check_matrix(X)
        if out is None:
            out = torch.empty_like(X)
        outb = _check_matrix(out)
        if outb.shape != Xb.shape:
            raise ValueError("out shape mismatch")
        B, n = Xb.shape[0], Xb.shape[-1]
        for name, lam in (("lambda_in", lambda_in), ("lambda_out", lambda_out)):
            if lam is not None and not (isinstance(lam, torch.Tensor) and lam.is_cuda and lam.dtype == torch.float64
                                        and lam.is_contiguous() and lam.numel() == B):
                raise ValueError(f"{name} must be a contiguous float64 CUDA tensor of batch elements")
        li = ctypes.c_void_p(lambda_in.data_ptr()) if lambda_in is not None else None
        lo = ctypes.c_void_p(lambda_out.data_ptr()) if lambda_out is not None else None
        check(self._lib.psd_project_ex(self._h, ctypes.c_void_p(Xb.data_ptr()), n, B,
                                       ctypes.c_void_p(outb.data_ptr()), li, lo, 1 if want_sign else 0,
                                       _stream_ptr(stream)), "psd_project_ex")
        return out

    def project(self, X, out=None, lambda_in=None, lambda_out=None, stream=None):
        """P = lambda~ 1/2 X_0 (I + X_T)  (Algorithm 2).  ``lambda_out`` (float64
        CUDA tensor of length batch) receives the lambda~ used; ``lambda_in`` is required
        with bound='user'."""
        return self._run(X, out, lambda_in, lambda_out, False, stream)

    def sign(self, X, out=None, lambda_in=None, lambda_out=None, stream=None):
        """S = X_T = f_T o ... o f_1 (X / lambda~)."""
        return self._run(X, out, lambda_in, lambda_out, True, stream)

    def polar(self, A, out=None, lambda_in=None, lambda_out=None, stream=None):
        """The filter's polar iterate of a general (rows, cols) or (batch, rows, cols) A:
        f_T o ... o f_1 (A / lambda~) with f_t(Z) = sum_j c_j Z (Z^T Z)^j, i.e. W diag(s(sigma / lambda~)) V^T
        for A = W diag(sigma) V^T (psd_polar_rect; all of A is read)."""
        import torch
        if not isinstance(A, torch.Tensor) or not A.is_cuda or A.dtype != torch.float32:
            raise TypeError("A must be a float32 CUDA tensor")
        if A.dim() not in (2, 3):
            raise ValueError("A must be (rows, cols) or (batch, rows, cols)")
        Ab = A.unsqueeze(0) if A.dim() == 2 else A
        if not Ab.is_contiguous():
            raise ValueError("A must be contiguous")
        out = torch.empty_like(A) if out is None else out
        if not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or not out.is_cuda or \
                out.shape != A.shape or not out.is_contiguous():
            raise ValueError("out must be a contiguous float32 CUDA tensor shaped like A")
        B, rows, cols = Ab.shape
        for name, lam in (("lambda_in", lambda_in), ("lambda_out", lambda_out)):
            if lam is not None and not (isinstance(lam, torch.Tensor) and lam.is_cuda and lam.dtype == torch.float64
                                        and lam.is_contiguous() and lam.numel() == B):
                raise ValueError(f"{name} must be a contiguous float64 CUDA tensor of batch elements")
        li = ctypes.c_void_p(lambda_in.data_ptr()) if lambda_in is not None else None
        lo = ctypes.c_void_p(lambda_out.data_ptr()) if lambda_out is not None else None
        check(self._lib.psd_polar_rect(self._h, ctypes.c_void_p(Ab.data_ptr()), rows, cols, B,
                                       ctypes.c_void_p(out.data_ptr()), li, lo, _stream_ptr(stream)), "psd_polar_rect")
        return out

    def admm_update(self, C, Xk, y, sigma, S_out=None, X_out=None, stream=None):
        """One fused ADMM S/X update (Eq. exp:admm-three-step) for diagonal
        constraints (A* y = Diag(y)): S = P(C - Diag(y) - Xk / sigma) by this filter and
        X_next = Xk + sigma (S + Diag(y) - C).  ``y``: (batch, n) or (n,) float32 CUDA tensor or
        None.  Returns (S_out, X_out); X_out may be Xk (in place)."""
        import torch
        Cb, Kb = _check_matrix(C), _check_matrix(Xk)
        if Kb.shape != Cb.shape:
            raise ValueError("Xk shape mismatch")
        B, n = Cb.shape[0], Cb.shape[-1]
        if y is not None:
            if not (isinstance(y, torch.Tensor) and y.is_cuda and y.dtype == torch.float32 and y.is_contiguous()
                    and y.numel() == B * n):
                raise ValueError("y must be a contiguous float32 CUDA tensor of batch * n elements")
        S_out = torch.empty_like(C) if S_out is None else S_out
        X_out = torch.empty_like(Xk) if X_out is None else X_out
        Sb, Ob = _check_matrix(S_out), _check_matrix(X_out)
        if Sb.shape != Cb.shape or Ob.shape != Cb.shape:
            raise ValueError("output shape mismatch")
        check(self._lib.psd_admm_update(self._h, ctypes.c_void_p(Cb.data_ptr()), ctypes.c_void_p(Kb.data_ptr()),
                                        ctypes.c_void_p(y.data_ptr()) if y is not None else None, float(sigma), n, B,
                                        ctypes.c_void_p(Sb.data_ptr()), ctypes.c_void_p(Ob.data_ptr()),
                                        _stream_ptr(stream)), "psd_admm_update")
        return S_out, X_out

    def certificate(self):
        """{'relu_err', 'relu_argmax', 'sign_err', 'sign_argmax'}: the scalar worst cases of this
        chain over every float32 in [0, 1], computed on the device (psd_filter_certificate)."""
        v = [ctypes.c_double() for _ in range(4)]
        check(self._lib.psd_filter_certificate(self._h, *(ctypes.byref(x) for x in v)), "psd_filter_certificate")
        return {"sign_err": v[0].value, "relu_err": v[1].value, "sign_argmax": v[2].value, "relu_argmax": v[3].value}

    def status(self, stream=None):
        """Synchronise and return 'PSD_OK' or 'PSD_ENONFINITE' (device numeric status)."""
        from ._lib import STATUS_NAMES
        code = self._lib.psd_status(self._h, _stream_ptr(stream))
        if code not in (0, 5, 7):
            check(code, "psd_status")
        return STATUS_NAMES[code]

    def profile(self, enable=True):
        """Record device time of the product kernels of later calls (see psd_profile)."""
        check(self._lib.psd_profile(self._h, 1 if enable else 0), "psd_profile")

    def profile_read(self):
        """(product_ms, product_launches, kernel_launches) since the last read; synchronises."""
        ms = ctypes.c_double()
        pl = ctypes.c_int64()
        kl = ctypes.c_int64()
        check(self._lib.psd_profile_read(self._h, ctypes.byref(ms), ctypes.byref(pl), ctypes.byref(kl)),
              "psd_profile_read")
        return ms.value, pl.value, kl.value

    def project_host(self, X, out=None, chunks=4, stream=None):
        """End-to-end projection of a PINNED host float32 tensor (batch, n, n): chunked so the
        host-to-device copies, the projections and the device-to-host copies overlap
        (psd_project_host).  Returns `out` (pinned host); valid after the stream synchronises."""
        import torch
        if not isinstance(X, torch.Tensor) or X.is_cuda or X.dtype != torch.float32 or not X.is_pinned():
            raise TypeError("X must be a pinned host float32 tensor")
        Xb = X.unsqueeze(0) if X.dim() == 2 else X
        if out is None:
            out = torch.empty_like(X, pin_memory=True)
        ob = out.unsqueeze(0) if out.dim() == 2 else out
        if not (Xb.is_contiguous() and ob.is_contiguous() and ob.shape == Xb.shape and ob.is_pinned()):
            raise ValueError("out must be a pinned contiguous tensor shaped like X")
        check(self._lib.psd_project_host(self._h, ctypes.c_void_p(Xb.data_ptr()), Xb.shape[-1], Xb.shape[0],
                                         ctypes.c_void_p(ob.data_ptr()), int(chunks), _stream_ptr(stream)),
              "psd_project_host")
        return out

    def project_rowpanel_virtual(self, X, nranks, out=None, sign=False, stream=None):
        """Row-panel projection of one n x n matrix with `nranks` virtual ranks on this GPU (the
        per-rank code of the multi-GPU path; see dist.RowPanelProjector for real ranks)."""
        import torch
        Xb = _check_matrix(X)
        if Xb.shape[0] != 1:
            raise ValueError("row panels project one matrix")
        if out is None:
            out = torch.empty_like(X)
        n = Xb.shape[-1]
        check(self._lib.psd_project_rowpanel_virtual(self._h, ctypes.c_void_p(Xb.data_ptr()), n, int(nranks),
                                                     ctypes.c_void_p(_check_matrix(out).data_ptr()),
                                                     1 if sign else 0, _stream_ptr(stream)),
              "psd_project_rowpanel_virtual")
        return out

    def project_rowpanel_p2p_virtual(self, X, nranks, out=None, sign=False, stream=None):
        """Peer-memory row-panel projection (the product kernels store their tiles into every rank's
        operand region, no collective) with `nranks` virtual ranks whose regions all live on this GPU."""
        import torch
        Xb = _check_matrix(X)
        if Xb.shape[0] != 1:
            raise ValueError("row panels project one matrix")
        if out is None:
            out = torch.empty_like(X)
        check(self._lib.psd_project_rowpanel_p2p_virtual(self._h, ctypes.c_void_p(Xb.data_ptr()), Xb.shape[-1],
                                                         int(nranks), ctypes.c_void_p(_check_matrix(out).data_ptr()),
                                                         1 if sign else 0, _stream_ptr(stream)),
              "psd_project_rowpanel_p2p_virtual")
        return out

    def sym_product(self, A, B, D=None, alpha=1.0, beta=0.0, out=None, stream=None):
        """C = alpha (A B) + beta D for commuting symmetric A, B (upper triangles read)."""
        import torch
        Ab, Bb = _check_matrix(A), _check_matrix(B)
        if out is None:
            out = torch.empty_like(A)
        outb = _check_matrix(out)
        Db = _check_matrix(D) if D is not None else None
        nb, n = Ab.shape[0], Ab.shape[-1]
        check(self._lib.psd_sym_product(self._h, ctypes.c_void_p(Ab.data_ptr()), ctypes.c_void_p(Bb.data_ptr()),
                                        ctypes.c_void_p(Db.data_ptr()) if Db is not None else None,
                                        float(alpha), float(beta), n, nb, ctypes.c_void_p(outb.data_ptr()),
                                        _stream_ptr(stream)), "psd_sym_product")
        return out
