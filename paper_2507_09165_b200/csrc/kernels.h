// kernels.h -- internal launch interface between the C-ABI driver (psd_api.cu) and the
// sm_100a kernels.  Not part of the public ABI (include/psd_filter.h is).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>

namespace psd {

// Experiment / A-B switches and phase stamps exist only in the debug build (-DPSD_DEBUG,
// libpsdfilter_dbg.so): the production library never reads the environment and its kernels
// carry no stamp code (every `if (kDebug && ...)` folds away).
#ifdef PSD_DEBUG
constexpr bool kDebug = true;
inline const char* debug_env(const char* name) { return std::getenv(name); }
#else
constexpr bool kDebug = false;
inline const char* debug_env(const char*) { return nullptr; }
#endif

enum class OpType : int { F16 = 0, BF16 = 1, TF32 = 2 };

// Square output tile of the symmetric product kernel and its K block (bytes of one
// operand row slice = one 128B swizzle atom).
constexpr int kTile = 128;
constexpr int kBlockKBytes = 128;
constexpr int kPadTo = 128;   // padded matrix dimension multiple

constexpr int kMaxPeers = 8;   // ranks of the peer-memory row-panel path

// Epilogue of one symmetric product C = alpha_eff * (A B) + beta * D over the upper
// tiles (I <= J) of each matrix; see sym_gemm.cu for which elements go where.
struct EpiParams {
    float alpha;              // host factor (already divided by the operands' scales)
    const double* alpha_dev;  // optional per-matrix factor (lambda~), multiplies alpha
    float beta;               // (already divided by the addend's scale)
    const void* Dop;          // optional addend in operand precision, upper triangle, ld npad
    const void* Dop_lo;       // split precision: low part of the addend (added to Dop)
    void* out_lo;             // split precision: low part of the output copy
    float out_scale;          // the output copy stores v * out_scale (power of two)
    const float* Df;          // optional fp32 addend (the input X), upper triangle read
    int64_t ldDf, strideDf;   // row stride / matrix stride (elements)
    int nDf;                  // rows/cols of Df that exist (mask)
    void* out_op;             // operand-precision copy, full mirrored, ld = npad (or NULL)
    float* outF;              // final fp32 output, full mirrored, masked to nF (or NULL)
    int64_t ldF, strideF;
    int nF;
    // Row-panel (multi-GPU) mode, CTA-pair kernel only: instead of the mirrored stores, tile slot
    // t of the launch is written, unmirrored and row-major, at packed + t * 256 * 256 (elements):
    // operand precision (out_op ignored) or fp32 when packed_f32.
    void* packed;
    int packed_f32;
    // debug: CTA 0 thread 0 stores %globaltimer at kernel phases (NULL in production)
    unsigned long long* dbg;
    unsigned long long* dbg_all;   // debug build: per-CTA %globaltimer stamps (PSD_DEBUG_TIMELINE, 1-CTA kernel)
    int dbg_nostore;          // debug experiment (PSD_DEBUG_NOSTORE): skip the epilogue's stores
    int upper_only;           // store off-diagonal tiles of the operand copy without their mirror
    // Peer-memory row-panel mode (the product and its all-gather in one kernel): the operand copy
    // goes to out_peers[0..npeers) -- the same buffer of every rank, mapped into this process --
    // and fp32 output row r to outF_peers[r / peer_rows] (its owner rank's buffer, ld ldF).
    void* out_peers[kMaxPeers];
    float* outF_peers[kMaxPeers];
    int npeers;
    int peer_rows;
    // Fused ADMM update (psd_admm_update): the fp32 addend is formed on the fly as
    // m = Df + df2_scale * Df2 - Diag(ddiag) (C - X_k / sigma - Diag(y); Df2 shares Df's layout,
    // ddiag is batch x nDf), and outF2 = outF2_scale * (v - m) = sigma (S - M) is stored like outF.
    const float* Df2;
    float df2_scale;
    const float* ddiag;
    float* outF2;
    float outF2_scale;
};

// The input of the bound / scale kernels: X itself, or the ADMM argument formed on the fly,
// M = X - inv_sigma * Xk - Diag(y)  (X = C; Xk, y as in psd_admm_update; Xk == NULL: plain X).
struct InputForm {
    const float* Xk = nullptr;
    const float* y = nullptr;          // batch x n (NULL: no diagonal term)
    float inv_sigma = 0.0f;
};

struct GemmShape {
    int npad;                 // padded n (multiple of kTile)
    int batch;
    const uint32_t* tiles;    // CTA-pair kernel: upper-tile visiting order, (I << 16) | J, one matrix
    int tiles_per_matrix;     // = nt (nt + 1) / 2 for nt = npad / 256
    int* counter;             // CTA-pair kernel: zeroed global tile counter (dynamic scheduler)
    // CTA-pair kernel, 16-bit operands: the operands hold only their upper 256-tiles (+ the full
    // diagonal tiles); the part of a row panel left of its diagonal tile is loaded transposed
    // (MN-major) from the stored upper tile, and the epilogue skips the mirrored stores of
    // off-diagonal tiles (half the operand stores and DRAM writes)
    int upper_only;
    // K-chunked accumulation (split / FP32-class precisions): the tensor cores' fp32 accumulator
    // loses ~2^-24 relative per accumulating MMA (error linear in K, profiles/r1s3_accumulation_error.txt),
    // so each run of `kchunk` K elements is accumulated from zero and the runs are summed with
    // round-to-nearest fp32 adds in the epilogue warps.  0: one accumulation over the whole K.
    int kchunk;
    // 1-CTA kernel only (psd_polar's block-structured products on H = [[0, A], [A^T, 0]], R25):
    // sub_mode 0 = the upper tiles of the whole npad matrix; 1 / 3 = the upper tiles of the sub_m x sub_m
    // bottom-right / top-left block; 2 = every tile of the sub_m x sub_m top-right block.  K runs over
    // [k_begin, k_end) (k_end 0: npad).  Zero-initialised = the symmetric product.
    int sub_mode;
    int sub_m;
    int k_begin, k_end;
};

// Visiting order of the upper 256-tiles of one matrix (host side), by name:
// "row" (row-major), "col" (column-major), "grouped<G>" (G x G super-tiles, row-major).
void make_tile_order(int nt, const char* order, uint32_t* out);

// Host-side TMA descriptor for an operand buffer [batch*npad rows][npad cols].
bool make_operand_tmap(CUtensorMap* map, const void* base, OpType t, int npad, int batch, int box_rows = kTile);
// 1-CTA product kernel tile width for (npad, batch): 128, or 64 for few-tile problems; its split-K.
int sym_gemm_bn(int npad, int batch);
int sym_gemm_split_k(int npad, int batch, OpType t, bool split, int kchunk);

// Operand tensor maps of one product: A, B (high parts) and, for split precision, their
// low parts (A*B ~= Ahi Bhi + Ahi Blo + Alo Bhi, three tcgen05.mma passes, one accumulator).
struct OperandMaps {
    CUtensorMap a, b, a_lo, b_lo;
    // 64 x 64 boxes of A and B (and their low parts): the transposed (MN-major) loads of the
    // upper-only storage mode
    CUtensorMap a_t, b_t, a_lo_t, b_lo_t;
};

// C = alpha*(A B) + beta*D on the upper tiles.
cudaError_t launch_sym_gemm(OpType t, bool split, const OperandMaps& m, const GemmShape& s, const EpiParams& e,
                            cudaStream_t stream);

// Same product, persistent CTA-pair kernel with 256 x 256 tiles (npad multiple of 256).
cudaError_t launch_sym_gemm_2cta(OpType t, bool split, const OperandMaps& m, const GemmShape& s,
                                 const EpiParams& e, cudaStream_t stream);
// Whether (n, batch) runs on the CTA-pair kernel, and the padded size it needs.
bool use_pair_kernel(int64_t n, int64_t batch);
int64_t padded_n(int64_t n, int64_t batch);

// Batched small-n path (n <= 64), the whole chain in one kernel (small_batch.cu).
struct SmallStep {
    int slot_a, slot_b;       // byte offsets of the operand slots within a matrix's smem region
    int slot_d;               // addend slot (-1: none; the fp32 X of a final_mode-1 step is implicit)
    int slot_out;             // output slot (final_mode 0)
    float alpha, beta, out_scale;
    int final_mode;           // 0: chain product; 1: P = lambda~ alpha acc + beta X; 2: S = alpha acc + beta D
    int reload_x0;            // restage X_0 into the Y slot before this product
    int mirror;               // make the output exactly symmetric (stage outputs Z; reading R20)
};
struct SmallPlan {
    int nsteps;
    float s_x0;               // operand scale of X_0
    InputForm form;           // ADMM: the input is M = X - inv_sigma Xk - Diag(y) (form.Xk != NULL)
    float* out2;              // ADMM: X_next = sigma2 (P - M), stored like out
    float sigma2;
    unsigned long long* dbg;  // debug: per-phase clock totals of CTA 0 (NULL in production)
    int split_commit;         // chain products: one MMA commit per matrix, each matrix's epilogue starts on its own
    SmallStep steps[40];
};
int small_slot_offset(bool split, int slot);   // slot 0 Z, 1 Y, 2 U
cudaError_t launch_small_batch(bool split, const float* X, float* out, int n, int batch, double* lambda_out,
                               unsigned* status, const SmallPlan& plan, cudaStream_t stream);

// The filter's scalar worst-case errors over every float32 in [0, 1] (certificate.cu): relu_err =
// max 1/2 x |1 - s(x)|, sign_err = max over x >= eps of |s(x) - 1| (synchronous, fp64).
cudaError_t certify_chain(const std::vector<std::vector<double>>& coeffs, double eps, double* relu_err,
                          double* relu_argmax, double* sign_err, double* sign_argmax);

// Row-panel multi-GPU path (rowpanel.cu).
cudaError_t launch_unpack_tiles(int elem_bytes, const void* packed, const uint32_t* codes, int ntiles, void* full,
                                int64_t ld, cudaStream_t stream, bool mirror = true);
int rowpanel_tiles(int nt, int nranks, int rank, uint32_t* codes, int cap);
// Cross-rank epoch barrier of the peer-memory path: signal stores `epoch` into slot `rank` of every
// rank's flag array (system-scope release after a system fence); wait spins until every slot of
// this rank's flags reaches `epoch` (system-scope acquire); after timeout_ns it sets bit 1 of
// *status (psd_status: PSD_ETIMEOUT) and returns instead of hanging.
cudaError_t launch_peer_signal(unsigned long long* const* flags_dev, int nranks, int rank, unsigned long long epoch,
                               cudaStream_t stream);
cudaError_t launch_peer_wait(const unsigned long long* my_flags, int nranks, unsigned long long epoch,
                             unsigned long long timeout_ns, unsigned* status, cudaStream_t stream);

// Frobenius partial sums: partial[b*nblk + k] = sum over rows i == k (mod nblk) of
// x_ii^2 + 2 sum_{j>i} x_ij^2 (upper triangle of matrix b), fp64.
int bound_blocks_per_matrix(int n, int batch);
// psd_polar (polar.cu): the upper triangle of H = [[0, A], [A^T, 0]] (2n x 2n) from a general A, with
// per-block fp64 partial sums of a^2 (finalised by launch_finalize_bound into lambda~ = ||A||_F),
// and the top-right n x n block of the 2n x 2n sign output
int polar_blocks_per_matrix(int m, int batch);
cudaError_t launch_polar_embed(const float* A, int rows, int cols, int m, int batch, float* H, double* partial,
                               int nblk, cudaStream_t stream);
cudaError_t launch_polar_extract(const float* S, int rows, int cols, int m, int batch, float* out, cudaStream_t stream);
cudaError_t launch_frobenius_partials(const float* X, int n, int batch, double* partial, int nblk,
                                      cudaStream_t stream, const InputForm& form = InputForm());

// lambda[b] = sqrt(sum_k partial[b*nblk+k]) (fixed order); status |= 1 if non-finite.
cudaError_t launch_finalize_bound(const double* partial, int nblk, int batch, double* lambda,
                                  double* lambda_out, unsigned* status, cudaStream_t stream);

// X0 = sym_upper(X) / lambda[b] (or * scale when lambda == NULL), written as
//   op copy (full, mirrored, zero padded, ld npad)  -- if out_op
//   fp32 master (upper 32-tiles, zero padded)       -- if out32
//   fp32 final (full, mirrored, ld n)               -- if outF (scaled by post)
// With out_lo (split precision): out_op = cvt(x0 * op_scale), out_lo = cvt(x0 * op_scale - out_op).
// Lanczos bound (Algorithm 2 line 1 + Theorem 2) on the operand copy X0 (scale s0) of
// X / lambda_F: overwrites lambda[b] (and lambda_out) with lambda_F * min(1, sqrt(sigma + r) / s0 *
// safety).  `scratch`: lanczos_scratch_bytes(npad, batch, steps) bytes of device memory.
size_t lanczos_scratch_bytes(int npad, int batch, int steps);
cudaError_t launch_lanczos_bound(OpType t, const void* X0, double s0, int n, int npad, int batch, int steps,
                                 double safety, void* scratch, double* lambda, double* lambda_out, cudaStream_t stream);
int lanczos_launches(int steps, int n);
void lanczos_prepare();   // kernel attributes (call once, outside graph capture)

cudaError_t launch_scale_convert(OpType t, const float* X, int n, int npad, int batch,
                                 const double* lambda, double scale, void* out_op, void* out_lo,
                                 double op_scale, float* outF, double post, cudaStream_t stream,
                                 const InputForm& form = InputForm(), int mirror_block = 0);

}  // namespace psd
