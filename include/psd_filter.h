/*
 * psd_filter.h -- C ABI of the B200 (sm_100a) PSD-cone projection library
 * (libpsdfilter.so) implementing the hot path of arXiv 2507.09165.
 *
 * Citations: "P:L<n>" is line n of the paper text (PAPER.md; Doc C, lines 337-1205,
 * is the authority).  DESIGN.md lists every reading R<k> of the paper used here.
 *
 * The method (Algorithm 2, "Run-time projection algorithm"):
 *     lambda~ = upper bound of ||X||_2          (here ||X||_F; reading R4)
 *     X_0     = X / lambda~
 *     X_t     = f_t(X_{t-1}),  t = 1..T
 *     P       = lambda~ * 1/2 * X_0 (I + X_T)
 * with f_t(x) = sum_{j=0}^{p_t} c_{t,j} x^{2j+1} odd of degree d_t = 2 p_t + 1
 * (Eq. comp:minimax-sign P:L502-508; odd monomials P:L57).  Every stage is a chain of
 * dense symmetric products: Y = X X; Horner in Y; one multiply by X.
 * GEMM count = sum_t (d_t + 1)/2 (+1 for the reconstruction), P:L598 / P:L647.
 *
 * Conventions common to every entry point
 *   - Matrices are dense, row-major, fp32, n x n, `batch` of them contiguous
 *     (matrix b starts at b*n*n).  Only the UPPER triangle of X is read
 *     (X_ij := X_min(i,j),max(i,j); reading R10).  Outputs are fully written and
 *     exactly symmetric (mirrored stores).
 *   - Device pointers: X, out, lambda_* live in device memory of the current
 *     device; they are caller-owned and must be 16-byte aligned.  out == X
 *     (in place) is allowed.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All device work is stream-ordered and asynchronous; the host never syncs
 *     except in psd_status().
 *   - Synchronous argument errors return PSD_EINVAL (etc.) immediately and set a
 *     thread-local message readable through psd_last_error().  Numeric problems
 *     found on the device (non-finite input) set the handle's status word;
 *     psd_status() reports them.
 *   - A handle owns its copied coefficients and a lazily grown device workspace.
 *     One handle may be used from one host thread at a time; distinct handles are
 *     independent.
 */
#ifndef PSD_FILTER_H
#define PSD_FILTER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psd_filter_s* psd_filter_t;

typedef enum {
    PSD_OK = 0,
    PSD_EINVAL = 1,        /* bad argument (message in psd_last_error) */
    PSD_ENOMEM = 2,        /* device workspace allocation failed */
    PSD_ECUDA = 3,         /* a CUDA runtime/driver call failed */
    PSD_ENCCL = 4,         /* reserved for the row-panel multi-GPU path */
    PSD_ENONFINITE = 5,    /* device found a non-finite input (output is NaN) */
    PSD_EUNSUPPORTED = 6,  /* configuration not supported by this build / device */
    PSD_ETIMEOUT = 7       /* peer row panels: a peer never reached a barrier (result invalid) */
} psd_status_t;

/* Operand precision of the tensor-core products; accumulation is always fp32.
 * FP16: the paper's half-precision path.  BF16: same kernel, bf16 operands.
 * TF32: kind::tf32 single pass.
 * *X3 (split precision, the FP32-class path standing in for the paper's FP32 /
 * BF16x9-emulated products): every operand is stored as hi + lo in the
 * operand type (fp16 with a per-buffer power-of-two scale that keeps lo in the normal
 * range) and each product is hi*hi + hi*lo + lo*hi, three tcgen05.mma passes into fp32
 * accumulators.  The tensor cores' fp32 accumulator loses ~2^-24 relative per accumulating
 * MMA (error linear in K: 1.7e-5 for one n = 4096 product), so the split precisions
 * accumulate K in runs of psd_filter_set_accum_chunk elements (default 512), each from zero,
 * summed with round-to-nearest fp32 adds (reading R23).  FP16X3 runs at the fp16 rate
 * (3 passes), TF32X3 at the tf32 rate.  Readings R11, R17, R19, R23 in DESIGN.md. */
typedef enum {
    PSD_PREC_FP16 = 0,
    PSD_PREC_BF16 = 1,
    PSD_PREC_TF32 = 2,
    PSD_PREC_TF32X3 = 3,
    PSD_PREC_FP16X3 = 4,
    PSD_PREC_BF16X3 = 5
} psd_precision_t;

/* FROBENIUS: lambda~ = ||X||_F computed on the device (default).
 * USER: lambda~ taken from psd_project_ex's lambda_in (device, one double per matrix).
 * LANCZOS: Algorithm 2 line 1 with Theorem 2: on X0 = X / ||X||_F (in the
 *   operand precision: the matrix the chain actually filters), a k-step Lanczos run on X0^2
 *   (k = 20 by default, the paper's; full re-orthogonalisation) gives the largest Ritz pair
 *   (sigma, q); lambda~ = ||X||_F * min(1, sqrt(sigma + ||X0^2 q - sigma q||) * safety).
 *   Theorem 2 assumes lambda_1(X^2) is the eigenvalue nearest sigma, which the paper finds
 *   to hold in practice; `safety` (default 1.01) absorbs the operand rounding.  Never
 *   looser than FROBENIUS.  Costs 2k + 2 matrix-vector passes over the operand copy.
 *   n <= 51200.  Reading R21. */
typedef enum {
    PSD_BOUND_FROBENIUS = 0,
    PSD_BOUND_USER = 1,
    PSD_BOUND_LANCZOS = 2
} psd_bound_t;

/* Library version string, e.g. "psdfilter 0.1 sm_100a". Never NULL. Host only. */
const char* psd_version(void);

/* Thread-local message for the last synchronous error on this thread ("" if none). */
const char* psd_last_error(void);

/* Create a composite filter (Eq. composite-polynomial-filter).
 *   T       number of stages, 1 <= T <= 64.
 *   degrees T odd degrees d_t, 1 <= d_t <= 15; stage t is applied t-th (f_1 first).
 *   coeffs  sum_t (d_t+1)/2 doubles, stage-major; within a stage c_{t,0} (of x) first,
 *           then x^3, x^5, ...  Stabilisation factors must already be folded in
 *           by the caller (python: paper_2507_09165_b200.filters).  All finite.
 *   eps     design epsilon of Eq. comp:minimax-sign (0 < eps < 1); recorded only, it
 *           does not change the map X -> P (reading R15).
 *   out     receives the handle.
 * Copies its inputs; makes no CUDA call (host only).  Degree-1 stages are scalar
 * multiplies folded into the neighbouring products (0 GEMMs, reading R7).
 * Returns PSD_EINVAL on bad arguments. */
psd_status_t psd_filter_create(int T, const int* degrees, const double* coeffs, double eps,
                               psd_filter_t* out);

/* Frees the handle and its device workspace (synchronises the device first). NULL-safe. */
void psd_filter_destroy(psd_filter_t h);

/* Operand precision (default PSD_PREC_FP16). Host only. */
psd_status_t psd_filter_set_precision(psd_filter_t h, psd_precision_t prec);

/* Bound used to normalise X (default PSD_BOUND_FROBENIUS). Host only. */
psd_status_t psd_filter_set_bound(psd_filter_t h, psd_bound_t bound);

/* PSD_BOUND_LANCZOS parameters: steps in [1, 64] (default 20; min(steps, n) are
 * run), safety in [1, 2] (default 1.01).  Host only; PSD_EINVAL outside the ranges. */
psd_status_t psd_filter_set_lanczos(psd_filter_t h, int steps, double safety);

/* Split (*X3) precisions only: accumulate each product's K range in independent runs of
 * `kchunk` elements (a multiple of 64, at least 64), summed round-to-nearest in fp32 by the
 * epilogue (reading R23); 0 = one hardware accumulation over the whole K (the
 * pre-R23 behaviour, error ~4e-9 * n).  The 1-CTA product kernel (few-tile problems) splits K
 * into at most 512 / tile-width runs of equal length instead.  Default 512.  Host only;
 * PSD_EINVAL for other values. */
psd_status_t psd_filter_set_accum_chunk(psd_filter_t h, int64_t kchunk);

/* Number of tensor-core products one matrix costs: sum_t (d_t+1)/2 over stages with
 * d_t > 1, plus 1 if `for_project` (the reconstruction of P:L757).  Host only.
 * Returns -1 for a NULL handle. */
int psd_filter_gemm_count(psd_filter_t h, int for_project);

/* Algorithm 2: out[b] = P(X[b]) for b < batch, n >= 1, batch >= 1.
 * X, out: device fp32, see conventions.  Returns PSD_OK once all work is enqueued. */
psd_status_t psd_project(psd_filter_t h, const float* X, int64_t n, int64_t batch,
                         float* out, void* stream);

/* Matrix sign output of the same chain: out[b] = X_T = f_T o ... o f_1 (X[b]/lambda~)
 * (Eq. matrix-sign; the loop of Algorithm 2). */
psd_status_t psd_sign(psd_filter_t h, const float* X, int64_t n, int64_t batch,
                      float* out, void* stream);

/* psd_project with explicit bounds.
 *   lambda_in   device, `batch` doubles; used iff the bound is PSD_BOUND_USER (else may be NULL).
 *   lambda_out  device, `batch` doubles receiving the lambda~ actually used; may be NULL.
 *   want_sign   0: out = P (psd_project); 1: out = X_T (psd_sign). */
psd_status_t psd_project_ex(psd_filter_t h, const float* X, int64_t n, int64_t batch,
                            float* out, const double* lambda_in, double* lambda_out,
                            int want_sign, void* stream);

/* Polar iterate of a general square matrix by the same composite filter (the
 * polar factor generalises the matrix sign): with A = W diag(sigma) V^T,
 *     out[b] = W diag(s(sigma / lambda~)) V^T = f_T o ... o f_1 (A[b] / lambda~),
 *     f_t(Z) = sum_j c_{t,j} Z (Z^T Z)^j,
 * which approaches the orthogonal polar factor W V^T for singular values in [eps, 1] * lambda~.
 * Computed through the symmetric path: the upper triangle of H = [[0, A'], [A'^T, 0]] (2m x 2m, A'
 * = A zero-padded to m = n rounded up to 128) is written to a handle-owned workspace and the sign
 * chain runs on H (f(H) = [[0, f(A')], [f(A')^T, 0]]) with every product restricted to its nonzero
 * block and K half -- the Gram product Z^T Z, the Horner products and the general product Z U of a
 * direct nonsymmetric chain (reading R25); the top-right block is copied to `out`.
 *   A, out : device, batch x n x n fp32 row-major (all of A is read; out fully written; out == A
 *            allowed), 16-byte aligned.
 *   lambda~: ||A||_F (>= ||A||_2 = ||H||_2; fp64, deterministic) with PSD_BOUND_FROBENIUS, the
 *            Lanczos/Theorem-2 bound of H with PSD_BOUND_LANCZOS, lambda_in with PSD_BOUND_USER.
 *   lambda_in  device, `batch` doubles, used iff the bound is PSD_BOUND_USER (else may be NULL).
 *   lambda_out device, `batch` doubles receiving the lambda~ used; may be NULL.
 * Workspace: 2 x batch x (2m)^2 fp32 (m = n rounded up to 128) beside the product workspace of n' = 2m.  Non-finite input
 * sets PSD_ENONFINITE (psd_status).  Errors: PSD_EINVAL for NULL pointers, n < 1, batch < 1. */
psd_status_t psd_polar(psd_filter_t h, const float* A, int64_t n, int64_t batch, float* out,
                       const double* lambda_in, double* lambda_out, void* stream);

/* psd_polar for a rectangular rows x cols A (batch x rows x cols fp32 in and out): the same
 * iterate f(A) = sum_j c_j A (A^T A)^j per stage; A is zero-padded to a square edge (zero singular
 * values map to 0).  psd_polar(h, A, n, ...) is psd_polar_rect(h, A, n, n, ...). */
psd_status_t psd_polar_rect(psd_filter_t h, const float* A, int64_t rows, int64_t cols, int64_t batch,
                            float* out, const double* lambda_in, double* lambda_out, void* stream);

/* One fused S- and X-update of the three-step ADMM for the SDP pair of Eq. (exp:sdp)
 * (Eq. exp:admm-three-step), for diagonal constraint operators (max-cut:
 * A_i = e_i e_i^T, so A* y = Diag(y)):
 *     M      = C - Diag(y) - X_k / sigma          formed on the fly by the bound and scale kernels
 *     S_out  = P(M)                               the composite-filter projection (psd_project of M)
 *     X_out  = X_k + sigma (S_out + Diag(y) - C)  = sigma (S_out - M), fused into the
 *                                                 reconstruction epilogue (one extra fp32 store)
 * M is formed in fp32 with one rounding per operation, (C - X_k * fl(1/sigma)) - y_i on the
 * diagonal (reading R22); S_out is what psd_project returns for that M.
 *   C, Xk : device, batch x n x n fp32 (upper triangles read), 16-byte aligned.
 *   y     : device, batch x n fp32 (the diagonal of A* y per matrix), or NULL (y = 0).
 *   sigma : ADMM penalty, finite and > 0.
 *   S_out, X_out : device, batch x n x n fp32, fully written, exactly symmetric.  S_out == C and
 *           X_out == Xk (in place) are allowed; S_out == X_out is not (PSD_EINVAL).
 * Not with bound USER (PSD_EUNSUPPORTED).  Stream-ordered; not graph-cached (sigma and the extra
 * pointers are kernel arguments).  Errors as psd_project. */
psd_status_t psd_admm_update(psd_filter_t h, const float* C, const float* Xk, const float* y, double sigma,
                             int64_t n, int64_t batch, float* S_out, float* X_out, void* stream);

/* The filter's certificate, computed on the device over EVERY float32 in [0, 1] (s is odd, so
 * [-1, 1] reduces to [0, 1]), in fp64, for the chain s = f_T o ... o f_1 this handle holds:
 *   relu_err = max 1/2 x |1 - s(x)|   (Eq. comp:error-approx; the paper prints
 *              2 x relu_err under Tables 1-2, reading R3),
 *   sign_err = max over x in [eps, 1] of |s(x) - 1|   (Eq. comp:minimax-sign; eps of
 *              psd_filter_create -- its only use, reading R15),
 * and the maximising x of each (ties: the smaller x).  Any pointer may be NULL.  Synchronous
 * (about 2 x 1.07e9 chain evaluations, a few ms); deterministic. */
psd_status_t psd_filter_certificate(psd_filter_t h, double* sign_err, double* relu_err, double* sign_argmax,
                                    double* relu_argmax);

/* Synchronises `stream`, then returns and clears the handle's device status word:
 * PSD_OK or PSD_ENONFINITE (some input had a non-finite entry). */
psd_status_t psd_status(psd_filter_t h, void* stream);

/* Bytes of device workspace the handle would hold for (n, batch) at its precision. */
int64_t psd_workspace_bytes(psd_filter_t h, int64_t n, int64_t batch);

/* One symmetric product with the fused epilogue, exposed as a building block and
 * for kernel-level tests (the products of P:L395-399 whose output is symmetric):
 *   C = alpha * (A B) + beta * D,   A, B symmetric with A B = B A, n x n, `batch` of them.
 *   A, B  device fp32 (upper triangle read), converted to the handle's precision first.
 *   D     device fp32 or NULL (beta ignored); upper triangle read.
 *   C     device fp32, fully written, mirrored from the computed upper triangle.
 * Uses the handle's workspace; stream-ordered. */
psd_status_t psd_sym_product(psd_filter_t h, const float* A, const float* B, const float* D,
                             double alpha, double beta, int64_t n, int64_t batch, float* C,
                             void* stream);

/* Profiling of the product chain (measurement support for bench.py).
 * psd_profile(h, 1): every later psd_project, psd_project_ex or psd_sign call records a CUDA event pair on its
 * stream around its contiguous run of product kernels.  psd_profile(h, 0) stops recording.
 * psd_profile_read: synchronises on the recorded events, returns the summed device time of
 * the product runs (ms), the number of product kernels they contained, and the number of
 * kernels the handle launched in total since the last read (always counted); then resets.
 * Any out pointer may be NULL. */
psd_status_t psd_profile(psd_filter_t h, int enable);
psd_status_t psd_profile_read(psd_filter_t h, double* product_ms, int64_t* product_launches,
                              int64_t* kernel_launches);

/* End-to-end projection of HOST matrices: X_host and out_host are pinned host buffers
 * (cudaMallocHost / cudaHostRegister), batch x n x n fp32.  The batch is processed in `chunks`
 * pieces on three internal streams so the host-to-device copy of chunk c+1, the projection of
 * chunk c and the device-to-host copy of chunk c-1 overlap (PCIe is full duplex).  Stream-ordered
 * with respect to `stream` (it waits for prior work and later work waits for the result).
 * out_host == X_host is allowed. */
psd_status_t psd_project_host(psd_filter_t h, const float* X_host, int64_t n, int64_t batch, float* out_host,
                              int chunks, void* stream);

/* ---------------------------------------------------------------- multi-GPU (row panels)
 * One large n over P GPUs, one process per GPU.  Every
 * product of the chain is split over the ranks by upper 256-tiles (rank r computes a balanced,
 * disjoint share), the packed tiles are all-gathered over NCCL (NVLink / NVSwitch) and every
 * rank rebuilds the exactly symmetric full operand; the input rows are all-gathered once.
 * NCCL is the library torch already loaded (libnccl.so.2), resolved at run time. */

/* Fills id[128] with a new NCCL unique id (call on one rank, broadcast the bytes). */
psd_status_t psd_nccl_unique_id(char id[128]);
/* Creates this rank's NCCL communicator (collective over the nranks processes). */
psd_status_t psd_nccl_comm_create(const char id[128], int nranks, int rank, void** comm);
psd_status_t psd_nccl_comm_destroy(void* comm);

/* Row-panel projection: rank `rank` of `nranks` passes rows [rank*n/nranks, (rank+1)*n/nranks)
 * of X (device fp32, row-major, n columns; the full X must be symmetric -- its upper triangle is
 * what is used) and receives the same rows of P (or of S when want_sign).  n % nranks == 0.
 * Precisions FP16, BF16, TF32.  Collective: every rank must call it with the same filter and n. */
psd_status_t psd_project_rowpanel(psd_filter_t h, const float* X_rows, int64_t n, int rank, int nranks,
                                  float* out_rows, int want_sign, void* comm, void* stream);

/* The same per-rank code with `nranks` virtual ranks in this process on this GPU (the
 * all-gather becomes shared memory): X and out are the full n x n matrices. Test path. */
psd_status_t psd_project_rowpanel_virtual(psd_filter_t h, const float* X, int64_t n, int nranks, float* out,
                                          int want_sign, void* stream);

/* Peer-memory row panels (SURVEY section 8(f) NEXT #3, config c5 without a collective on the data
 * path): the product and its all-gather are ONE kernel.  Every rank holds a device region with
 * the full operand buffers; each product kernel computes this rank's share of the upper 256-tiles
 * (round robin, psd_rowpanel_tiles) and its epilogue stores every tile and its mirror straight
 * into every rank's region through peer pointers (NVLink / NVSwitch), overlapping the transfer
 * with the next tiles' MMAs; a cross-rank epoch barrier (system-scope release/acquire flags in
 * the regions) separates consecutive products.  The final product stores each fp32 32-row block
 * to the rank that owns those rows.  FP16 / BF16 / TF32, Frobenius bound; n % nranks == 0,
 * (n / nranks) % 32 == 0, nranks <= 8.
 *
 * Setup (once per (n, nranks), every rank):
 *   psd_rowpanel_p2p_region(h, n, nranks, rank, handle)   allocate this rank's region
 *       (~ 6 n^2 operand bytes + 8 n^2) and return its CUDA IPC handle (64 bytes);
 *   exchange the handles (e.g. torch.distributed all_gather_object), then
 *   psd_rowpanel_p2p_attach(h, handles)                    handles: nranks x 64 bytes in rank
 *       order; opens the peers' regions (cudaIpcOpenMemHandle, lazy peer access).
 * Run: psd_project_rowpanel_p2p(h, X_rows, n, rank, nranks, out_rows, want_sign, stream): X_rows,
 *   out_rows = this rank's rows [rank*n/nranks, +n/nranks) x n fp32 (device).  Every rank must
 *   call it (collective) and the ranks should pass a host barrier between attach and the first
 *   call (dist.PeerRowPanelProjector does); a rank that never arrives makes the others give up
 *   after the timeout (default 10 s): psd_status then returns PSD_ETIMEOUT and out_rows is invalid
 *   -- the context is never trapped or hung.
 * psd_rowpanel_p2p_timeout(h, seconds): that barrier timeout, (0, 3600] s.
 * psd_project_rowpanel_p2p_virtual(h, X, n, nranks, out, want_sign, stream): all nranks regions
 *   local to this device and every rank's kernels run here (tests of the per-rank code on one
 *   GPU); X, out full n x n.
 * psd_rowpanel_p2p_release(h): close / free the regions (also done by psd_filter_destroy). */
psd_status_t psd_rowpanel_p2p_region(psd_filter_t h, int64_t n, int nranks, int rank, char handle[64]);
psd_status_t psd_rowpanel_p2p_attach(psd_filter_t h, const char* handles);
psd_status_t psd_project_rowpanel_p2p(psd_filter_t h, const float* X_rows, int64_t n, int rank, int nranks,
                                      float* out_rows, int want_sign, void* stream);
psd_status_t psd_project_rowpanel_p2p_virtual(psd_filter_t h, const float* X, int64_t n, int nranks, float* out,
                                              int want_sign, void* stream);
psd_status_t psd_rowpanel_p2p_timeout(psd_filter_t h, double seconds);
void psd_rowpanel_p2p_release(psd_filter_t h);

/* Host helper: the upper 256-tiles rank `rank` computes, as (I << 16) | J codes in its packed
 * order, padded with 0xFFFFFFFF to the common per-rank count.  Returns the real count (codes ==
 * NULL: returns the padded per-rank count). */
int psd_rowpanel_tiles(int64_t n, int nranks, int rank, uint32_t* codes, int cap);

#ifdef __cplusplus
}
#endif

#endif /* PSD_FILTER_H */
