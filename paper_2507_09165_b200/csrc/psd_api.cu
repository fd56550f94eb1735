// psd_api.cu -- the C ABI of include/psd_filter.h: argument validation, the stage
// planner (Algorithm 2 as a list of fused symmetric products), the device workspace
// and the stream-ordered launches.  Host code; kernels live in sym_gemm.cu and
// bound_scale.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <dlfcn.h>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/psd_filter.h"
#include "kernels.h"

using namespace psd;

namespace {

thread_local std::string g_last_error;

psd_status_t fail(psd_status_t st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

psd_status_t cuda_fail(cudaError_t e, const char* where) {
    return fail(PSD_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Operand buffers of the chain (operand precision, full mirrored, [batch][npad][npad]).
enum Buf { B_XA = 0, B_XB, B_X0, B_Y, B_UA, B_UB, B_COUNT };
// Addend sources: an operand buffer (>= 0), none, or the fp32 input X.
enum Addend { D_NONE = -1, D_XIN = -2 };

struct Step {
    int A, B;            // operand buffers
    double alpha;        // host factor
    bool alpha_lambda;   // multiply alpha by lambda~[b] on the device
    double beta;
    int D;               // addend: operand buffer id, D_NONE or D_XIN
    int out_op;          // operand buffer written (-1: none)
    bool outF;           // final fp32 output
};

struct Workspace {
    int npad = 0, batch = 0;
    OpType op = OpType::F16;
    bool split = false;
    void* op_buf[2 * B_COUNT] = {};          // [B_COUNT..2 B_COUNT): low parts (split precision)
    double* partial = nullptr;
    double* lambda = nullptr;
    unsigned* status = nullptr;
    CUtensorMap tmap[2 * B_COUNT];
    CUtensorMap tmap64[2 * B_COUNT];        // 64-row boxes: B operand of the 128 x 64 tiles, transposed loads
    int nblk = 0;
    uint32_t* tiles = nullptr;     // CTA-pair tile visiting order (device)
    int tiles_per_matrix = 0;
    int* counters = nullptr;       // per-product tile counters of the dynamic scheduler
    void* lz_scratch = nullptr;    // Lanczos-bound scratch (allocated on first use)
    size_t lz_bytes = 0;
};

constexpr int kMaxSteps = 1024;
constexpr int kRowPanelChunks = 4;   // all-gathers per product on the NCCL row-panel path


int op_bytes(OpType t) { return t == OpType::TF32 ? 4 : 2; }

}  // namespace

struct psd_filter_s {
    std::vector<int> degrees;
    std::vector<std::vector<double>> coeffs;
    double eps = 1e-3;
    psd_precision_t prec = PSD_PREC_FP16;
    psd_bound_t bound = PSD_BOUND_FROBENIUS;
    int lz_steps = 20;             // PSD_BOUND_LANCZOS: Lanczos steps on X^2 and safety factor
    double lz_safety = 1.01;
    Workspace ws;
    // power-of-two operand scales of the fp16 split path: Z iterates, Y = Z^2, Horner U
    double s_z = 1.0, s_y = 1.0, s_u = 1.0;
    // row-panel (multi-GPU) workspace
    struct RowPanel {
        int npad = 0, nranks = 0, per = 0, n = 0;
        OpType op = OpType::F16;
        float* xg = nullptr;            // gathered X, n x n fp32
        float* pfull = nullptr;         // unpacked final product, npad x npad fp32
        void* packed_op = nullptr;      // [chunks][nranks][ct][256 * 256] operand precision
        float* packed_f32 = nullptr;    // [chunks][nranks][ct][256 * 256] fp32 (final product)
        uint32_t* codes = nullptr;      // [nranks][per] tile codes (each rank's list, compute order)
        uint32_t* codes_g = nullptr;    // [chunks][nranks][ct] tile codes in gathered-buffer order
        int chunks = 1, ct = 0;         // gathers per product, tiles per rank per chunk
        cudaStream_t cs = nullptr;      // communication stream (chunk c's all-gather under chunk c+1's MMAs)
        std::vector<int> counts;        // real tiles per rank
    } rp;
    // peer-memory row-panel path (multi-GPU without a collective on the data path): every rank
    // holds a region with the full operand buffers; each product kernel stores its tiles into
    // every rank's region (peer pointers over NVLink), an epoch barrier separates the products
    struct PeerPath {
        int n = 0, npad = 0, nranks = 0, rank = 0;
        bool is_virtual = false, attached = false;
        OpType op = OpType::F16;
        size_t region_bytes = 0, op_bytes_buf = 0, pfull_off = 0, xg_off = 0, flags_off = 0;
        std::vector<uint8_t*> base;          // [nranks]: own (cudaMalloc), peers (IPC-mapped) or all local (virtual)
        std::vector<char> ipc_opened;        // which bases were opened with cudaIpcOpenMemHandle
        std::vector<std::vector<CUtensorMap>> tmaps;   // [local region][B_COUNT]
        unsigned long long** flags_dev = nullptr;       // device array [nranks] of the flag arrays
        unsigned long long epoch = 0;
        uint32_t* codes = nullptr;           // [nranks][per] upper-tile codes
        std::vector<int> counts;
        int per = 0;
    } pp;
    unsigned long long peer_timeout_ns = 10000000000ull;   // peer barrier wait (psd_rowpanel_p2p_timeout)
    // CUDA-graph cache of whole psd_project sequences (host launch overhead dominates small n)
    struct GraphEntry {
        const void* X;
        const void* out;
        const void* lin;
        const void* lout;
        int64_t n, batch;
        int want_sign, prec, bound;
        cudaGraphExec_t exec;
        int64_t kernels, products;
        uint64_t last_use;
        // the captured graph (kept: its event-record nodes bracket the product run, so profiling
        // times the product kernels alone, not the whole sequence) and the nodes' own events
        cudaGraph_t graph;
        cudaGraphNode_t ev_node[2];
        cudaEvent_t own[2];
        bool borrowed;             // the nodes currently record profiling events from the pool
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_clock = 0;
    bool use_graphs = debug_env("PSD_NO_GRAPH") == nullptr;
    // K-chunked accumulation of the split (FP32-class) precisions, K elements per chunk
    // (psd_filter_set_accum_chunk; 0 = one accumulation over the whole K)
    int kchunk = 512;
    cudaStream_t capture_stream = nullptr;
    bool capturing = false;
    cudaEvent_t cap_ev[2] = {nullptr, nullptr};   // during capture: record nodes around the product run
    // pipelined host-buffer projection (psd_project_host)
    struct HostPipe {
        cudaStream_t s[3] = {nullptr, nullptr, nullptr};   // h2d, compute, d2h
        static constexpr int kMaxSlots = 8;      // chunk buffers in flight (H2D / project / D2H)
        float* dx[kMaxSlots] = {};
        float* dout[kMaxSlots] = {};
        int nslots = 0;
        size_t chunk_bytes = 0;
    } hp;
    // profiling / launch accounting
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pairs;
    int64_t product_launches_profiled = 0;
    int64_t kernel_launches = 0;
    int64_t last_products = 0;     // product-carrying launches of the last run_body (graph accounting)
    // psd_polar in progress: the block edge m of H = [[0, A], [A^T, 0]] (2m x 2m); the product loop
    // then restricts every product to its nonzero block and K range (GemmShape::sub_mode, R25)
    int polar_m = 0;
    bool polar_wide = false;       // rows < cols: the Gram products on the A A^T side (top-left block)
    // psd_polar: the 2n x 2n embedding H, the sign output on it, lambda~ and the norm partials
    struct Polar {
        float* H = nullptr;
        float* S = nullptr;
        double* lam = nullptr;
        double* part = nullptr;
        int64_t n = 0, batch = 0;
        bool wide = false;         // the plan the cached graphs on H were captured with
        // CTA-pair kernel (block edge a multiple of 256): its 256-tile lists per block product --
        // upper tiles of the top-left / bottom-right block, every tile of the top-right block
        uint32_t* tiles = nullptr;         // [tl: nsym][br: nsym][tr: ntr]
        int nsym = 0, ntr = 0;
    } pol;
};

namespace {

OpType op_of(psd_precision_t p) {
    switch (p) {
        case PSD_PREC_BF16:
        case PSD_PREC_BF16X3: return OpType::BF16;
        case PSD_PREC_TF32:
        case PSD_PREC_TF32X3: return OpType::TF32;
        default: return OpType::F16;
    }
}

bool split_of(psd_precision_t p) {
    return p == PSD_PREC_TF32X3 || p == PSD_PREC_FP16X3 || p == PSD_PREC_BF16X3;
}

// Bounds of |Z|, |Y|, |U| over the whole chain for spectra in [-1, 1] (||X_0||_2 <= 1 by the
// Frobenius normalisation; matrix entries are bounded by the spectral norm), evaluated on the
// scalar chain exactly as the planner folds it; each scale puts 1.25 x bound at <= 2^14.
void compute_scales(psd_filter_s* h) {
    const int N = 40001;
    std::vector<double> z(N);
    for (int i = 0; i < N; ++i) z[i] = -1.0 + 2.0 * i / (N - 1);
    double bz = 1.0, by = 0.0, bu = 0.0, s = 1.0;
    for (const auto& c : h->coeffs) {
        const int p = static_cast<int>(c.size()) - 1;
        if (p == 0) { s *= c[0]; continue; }
        std::vector<double> cs(c.size());
        for (int j = 0; j <= p; ++j) cs[j] = c[j] * std::pow(s, 2 * j + 1);
        s = 1.0;
        for (int i = 0; i < N; ++i) {
            const double y = z[i] * z[i];
            by = std::max(by, std::fabs(y));
            double u;
            if (p == 1) {
                u = cs[1] * y;
            } else {
                u = cs[p] * y * y + cs[p - 1] * y;
                bu = std::max(bu, std::fabs(u));
                for (int j = p - 2; j >= 1; --j) {
                    u = y * u + cs[j] * y;
                    bu = std::max(bu, std::fabs(u));
                }
            }
            z[i] = cs[0] * z[i] + z[i] * u;
            bz = std::max(bz, std::fabs(z[i]));
        }
    }
    auto scale_for = [](double b) {
        if (!(b > 0.0) || !std::isfinite(b)) return 1.0;
        return std::pow(2.0, std::floor(std::log2(16384.0 / (1.25 * b))));
    };
    h->s_z = scale_for(bz);
    h->s_y = scale_for(by);
    h->s_u = scale_for(bu);
}

void free_ws(Workspace& ws) {
    for (int i = B_COUNT; i < 2 * B_COUNT; ++i) { if (ws.op_buf[i]) cudaFree(ws.op_buf[i]); ws.op_buf[i] = nullptr; }
    for (auto& p : ws.op_buf) { if (p) cudaFree(p); p = nullptr; }
    if (ws.partial) cudaFree(ws.partial);
    if (ws.lambda) cudaFree(ws.lambda);
    if (ws.status) cudaFree(ws.status);
    if (ws.tiles) cudaFree(ws.tiles);
    if (ws.counters) cudaFree(ws.counters);
    if (ws.lz_scratch) cudaFree(ws.lz_scratch);
    ws.lz_scratch = nullptr;
    ws.lz_bytes = 0;
    ws.tiles = nullptr;
    ws.counters = nullptr;
    ws.partial = nullptr;
    ws.lambda = nullptr;
    ws.status = nullptr;
    ws.npad = ws.batch = 0;
}

int64_t ws_bytes(OpType op, bool split, int64_t npad, int64_t batch) {
    const int64_t mat = npad * npad * batch;
    return (split ? 2 : 1) * B_COUNT * mat * op_bytes(op) + batch * 256 * 8 + batch * 8 + 64;
}

void free_graphs(psd_filter_s* h);
void free_peerpath(psd_filter_s* h);

// Lanczos-bound scratch, grown on demand (never inside a graph capture)
psd_status_t ensure_lz(psd_filter_s* h, int npad, int batch) {
    Workspace& ws = h->ws;
    const size_t need = lanczos_scratch_bytes(npad, batch, h->lz_steps);
    if (ws.lz_bytes >= need) return PSD_OK;
    if (h->capturing) return fail(PSD_ECUDA, "Lanczos scratch must exist before capture");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
    free_graphs(h);          // captured Lanczos launches point into the old scratch
    if (ws.lz_scratch) cudaFree(ws.lz_scratch);
    ws.lz_scratch = nullptr;
    ws.lz_bytes = 0;
    if (cudaMalloc(&ws.lz_scratch, need) != cudaSuccess) return fail(PSD_ENOMEM, "cudaMalloc Lanczos scratch failed");
    ws.lz_bytes = need;
    lanczos_prepare();
    return PSD_OK;
}

psd_status_t ensure_ws(psd_filter_s* h, int npad, int batch) {
    Workspace& ws = h->ws;
    const OpType op = op_of(h->prec);
    const bool split = split_of(h->prec);
    if (ws.npad == npad && ws.batch >= batch && ws.op == op && ws.split == split && ws.status) return PSD_OK;
    if (ws.status) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
    }
    free_graphs(h);          // captured sequences point into the old workspace
    free_ws(ws);
    const size_t mat = static_cast<size_t>(npad) * npad * batch;
    for (int i = 0; i < (split ? 2 : 1) * B_COUNT; ++i) {
        if (cudaMalloc(&ws.op_buf[i], mat * op_bytes(op)) != cudaSuccess) {
            free_ws(ws);
            return fail(PSD_ENOMEM, "cudaMalloc operand workspace failed");
        }
    }
    ws.nblk = 256;
    if (cudaMalloc(&ws.partial, static_cast<size_t>(batch) * ws.nblk * 8) != cudaSuccess ||
        cudaMalloc(&ws.lambda, static_cast<size_t>(batch) * 8) != cudaSuccess ||
        cudaMalloc(&ws.status, 64) != cudaSuccess) {
        free_ws(ws);
        return fail(PSD_ENOMEM, "cudaMalloc small workspace failed");
    }
    cudaMemset(ws.status, 0, 64);
    // Zero everything once: padded rows/cols of every operand buffer must read as 0.
    for (int i = 0; i < (split ? 2 : 1) * B_COUNT; ++i) cudaMemset(ws.op_buf[i], 0, mat * op_bytes(op));
    for (int i = 0; i < (split ? 2 : 1) * B_COUNT; ++i) {
        if (!make_operand_tmap(&ws.tmap[i], ws.op_buf[i], op, npad, batch) ||
            !make_operand_tmap(&ws.tmap64[i], ws.op_buf[i], op, npad, batch, 64)) {
            free_ws(ws);
            return fail(PSD_ECUDA, "cuTensorMapEncodeTiled failed");
        }
    }
    {
        const int nt = npad / 256;
        ws.tiles_per_matrix = nt * (nt + 1) / 2;
        if (ws.tiles_per_matrix > 0) {
            std::vector<uint32_t> order(ws.tiles_per_matrix);
            // visiting order of the upper 256-tiles: row-major up to 16 tile rows (n <= 4096: the
            // panels in flight fit L2 either way), 8 x 8 super-tiles beyond (n = 16384: 79-82 vs
            // 91-97 ms per projection, tools/gemm_probe.py); PSD_TILE_ORDER overrides
            const char* env_order = debug_env("PSD_TILE_ORDER");
            make_tile_order(nt, env_order ? env_order : (nt > 16 ? "grouped8" : "row"), order.data());
            if (cudaMalloc(&ws.tiles, order.size() * 4) != cudaSuccess) {
                free_ws(ws);
                return fail(PSD_ENOMEM, "cudaMalloc tile order failed");
            }
            cudaMemcpy(ws.tiles, order.data(), order.size() * 4, cudaMemcpyHostToDevice);
        }
        if (cudaMalloc(&ws.counters, kMaxSteps * sizeof(int)) != cudaSuccess) {
            free_ws(ws);
            return fail(PSD_ENOMEM, "cudaMalloc counters failed");
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        free_ws(ws);
        return cuda_fail(e, "workspace init");
    }
    ws.npad = npad;
    ws.batch = batch;
    ws.op = op;
    ws.split = split;
    return PSD_OK;
}

// Algorithm 2's loop + return line as fused products.
// Stage t with coefficients c_0..c_p (p >= 1) on the iterate Z (operand buffer `cur`):
//   Y = Z Z
//   p == 1: Z' = c_0 Z + c_1 (Z Y)
//   p >= 2: U  = c_p (Y Y) + c_{p-1} Y ;  U <- Y U + c_j Y (j = p-2..1) ;  Z' = c_0 Z + Z U
// (identity-free Horner in Y = Z^2: no c*I term ever enters a low-precision operand).  The
// addends c_j Y and c_0 Z are read from the SAME rounded operand copies the tensor cores
// multiply, so every stage is exactly f_t of one rounded Z (DESIGN.md "consistent rounding":
// fp32 masters of Z, Y measured 2x less accurate in the rounding model).
// Degree-1 stages (p = 0) and trailing scalars are carried as a pending factor s and
// folded into the next products (f(sZ) = sum c_j s^{2j+1} Z^{2j+1}).
std::vector<Step> build_plan(const psd_filter_s* h, bool want_sign, double* sign_only_scale) {
    std::vector<Step> steps;
    double s = 1.0;
    int cur = B_X0;
    int last_gemm_stage = -1;
    for (size_t t = 0; t < h->coeffs.size(); ++t)
        if (h->coeffs[t].size() > 1) last_gemm_stage = static_cast<int>(t);
    double trailing = 1.0;
    for (size_t t = last_gemm_stage + 1; t < h->coeffs.size(); ++t) trailing *= h->coeffs[t][0];

    for (int t = 0; t <= last_gemm_stage; ++t) {
        const std::vector<double>& c = h->coeffs[t];
        const int p = static_cast<int>(c.size()) - 1;
        if (p == 0) { s *= c[0]; continue; }
        std::vector<double> cs(c.size());
        for (int j = 0; j <= p; ++j) cs[j] = c[j] * std::pow(s, 2 * j + 1);
        s = 1.0;
        const int nxt = (cur == B_XA) ? B_XB : B_XA;
        const bool last = (t == last_gemm_stage);
        steps.push_back({cur, cur, 1.0, false, 0.0, D_NONE, B_Y, false});
        Step fin;
        if (p == 1) {
            fin = {cur, B_Y, cs[1], false, cs[0], cur, nxt, false};
        } else {
            int u = B_UA;
            steps.push_back({B_Y, B_Y, cs[p], false, cs[p - 1], B_Y, u, false});
            for (int j = p - 2; j >= 1; --j) {
                const int un = (u == B_UA) ? B_UB : B_UA;
                steps.push_back({B_Y, u, 1.0, false, cs[j], B_Y, un, false});
                u = un;
            }
            fin = {cur, u, 1.0, false, cs[0], cur, nxt, false};
        }
        if (last && want_sign) {
            fin.alpha *= trailing;
            fin.beta *= trailing;
            fin.out_op = -1;
            fin.outF = true;
        }
        steps.push_back(fin);
        cur = nxt;
    }
    *sign_only_scale = 0.0;
    if (last_gemm_stage < 0) {
        // no products in the chain: S = s * X0 with s = prod of all degree-1 coefficients
        if (want_sign) {
            *sign_only_scale = trailing;
        } else {
            steps.push_back({B_X0, B_X0, 0.5 * trailing, true, 0.5, D_XIN, -1, true});
        }
        return steps;
    }
    if (!want_sign) {
        // P = 1/2 X + 1/2 lambda~ (X_0 S)  ==  lambda~ 1/2 X_0 (I + X_T)   (reading R5)
        steps.push_back({B_X0, cur, 0.5 * trailing, true, 0.5, D_XIN, -1, true});
    }
    return steps;
}

// Whether the per-product launches of run_body keep the operand copies upper-only (see
// GemmShape::upper_only): 16-bit operands, on the CTA-pair kernel and on the 1-CTA kernel (with or
// without cluster split-K).
// K accumulation chunk of the product kernels: the split precisions restart the accumulator every
// h->kchunk K elements (R23); single-pass products on the 1-CTA kernel at npad == 2 kchunk (c3,
// n = 1024) accumulate the two K halves separately, the arithmetic of the KS = 2 cluster launch
// (sym_gemm_split_k) -- faster at batch 1, and every batch size computes the same bits.
int product_kchunk(const psd_filter_s* h, bool split, int n, int npad, int batch) {
    if (split) return h->kchunk;
    const bool pair = npad % 256 == 0 && use_pair_kernel(n, batch);
    return (!pair && h->kchunk > 0 && npad == 2 * h->kchunk) ? h->kchunk : 0;
}

bool upper_only_mode(const psd_filter_s* h, int n, int batch, int npad) {
    if (op_of(h->prec) == OpType::TF32 || debug_env("PSD_NO_UPPER_ONLY")) return false;
    (void)h; (void)n; (void)batch; (void)npad;
    return true;
}

psd_status_t check_args(psd_filter_t h, const void* X, int64_t n, int64_t batch, const void* out) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (!X || !out) return fail(PSD_EINVAL, "null X or out");
    if (n < 1 || batch < 1) return fail(PSD_EINVAL, "n and batch must be >= 1");
    if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
        return fail(PSD_EINVAL, "X and out must be 16-byte aligned");
    if (n > 65536) return fail(PSD_EUNSUPPORTED, "n > 65536");
    return PSD_OK;
}

cudaEvent_t take_event(psd_filter_s* h) {
    if (!h->ev_pool.empty()) {
        cudaEvent_t e = h->ev_pool.back();
        h->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// psd_admm_update: the input is M = X - X_k / sigma - Diag(y) (X = C), formed on the fly, and the
// reconstruction also writes X_next = sigma (S - M)
struct AdmmArgs {
    InputForm form;
    float sigma;
    float* x_out;
};

psd_status_t run_body(psd_filter_t h, const float* X, int64_t n64, int64_t batch64, float* out,
                      const double* lambda_in, double* lambda_out, bool want_sign, cudaStream_t st,
                      const AdmmArgs* admm = nullptr) {
    const InputForm form = admm ? admm->form : InputForm();
    psd_status_t rc = check_args(h, X, n64, batch64, out);
    if (rc != PSD_OK) return rc;
    if (h->bound == PSD_BOUND_USER && !lambda_in) return fail(PSD_EINVAL, "PSD_BOUND_USER needs lambda_in");
    const int n = static_cast<int>(n64), batch = static_cast<int>(batch64);
    const int npad = static_cast<int>(padded_n(n, batch));
    rc = ensure_ws(h, npad, batch);
    if (rc != PSD_OK) return rc;
    Workspace& ws = h->ws;
    cudaError_t e;

    double sign_only = 0.0;
    std::vector<Step> steps = build_plan(h, want_sign, &sign_only);
    if (n <= 64 && h->bound == PSD_BOUND_FROBENIUS && ws.op == OpType::F16 && !steps.empty() &&
        steps.size() <= 40) {
        // batched small-n path: the whole chain in one kernel, operands resident in smem
        const bool sp = ws.split;
        const double sz = sp ? h->s_z : 1.0, sy = sp ? h->s_y : 1.0, su = sp ? h->s_u : 1.0;
        auto slot_of = [](int buf) { return buf == B_Y ? 1 : ((buf == B_UA || buf == B_UB) ? 2 : 0); };
        const double sc_slot[3] = {sz, sy, su};
        SmallPlan sp_plan{};
        sp_plan.nsteps = static_cast<int>(steps.size());
        if (admm) {
            sp_plan.form = admm->form;
            sp_plan.out2 = admm->x_out;
            sp_plan.sigma2 = admm->sigma;
        }
        sp_plan.s_x0 = static_cast<float>(sz);
        // one MMA commit per matrix in the chain products (c2: 146 -> 135 us fp16, 295 -> 273 us fp16x3 in the
        // debug build, profiles/r2s3/c2_split_commit/); PSD_SMALL_SPLIT_COMMIT=0 (debug build) for the A/B
        sp_plan.split_commit = debug_env("PSD_SMALL_SPLIT_COMMIT") ? std::atoi(debug_env("PSD_SMALL_SPLIT_COMMIT")) : 1;
        for (size_t i = 0; i < steps.size(); ++i) {
            const Step& s = steps[i];
            SmallStep& q = sp_plan.steps[i];
            int sa = slot_of(s.A), sb = slot_of(s.B);
            double scale_a = sc_slot[sa], scale_b = sc_slot[sb];
            q.reload_x0 = 0;
            q.mirror = 0;
            q.slot_d = -1;
            q.beta = static_cast<float>(s.beta);
            q.out_scale = 1.0f;
            q.slot_out = 0;
            if (s.outF && s.D == D_XIN) {              // reconstruction: X_0 restaged in the Y slot
                q.reload_x0 = 1;
                sa = 1;
                scale_a = sz;
                q.final_mode = 1;
            } else if (s.outF) {
                q.final_mode = 2;
            } else {
                q.final_mode = 0;
                q.slot_out = small_slot_offset(sp, slot_of(s.out_op));
                q.out_scale = static_cast<float>(sc_slot[slot_of(s.out_op)]);
                q.mirror = slot_of(s.out_op) == 0 ? 1 : 0;
            }
            if (s.D >= 0) {
                q.slot_d = small_slot_offset(sp, slot_of(s.D));
                q.beta = static_cast<float>(s.beta / sc_slot[slot_of(s.D)]);
            }
            q.slot_a = small_slot_offset(sp, sa);
            q.slot_b = small_slot_offset(sp, sb);
            q.alpha = static_cast<float>(s.alpha / (scale_a * scale_b));
        }
        std::pair<cudaEvent_t, cudaEvent_t> evs{nullptr, nullptr};
        if (h->profiling && !h->capturing) {
            evs = {take_event(h), take_event(h)};
            cudaEventRecord(evs.first, st);
        } else if (h->capturing && h->cap_ev[0]) {
            cudaEventRecordWithFlags(h->cap_ev[0], st, cudaEventRecordExternal);
        }
        const bool dbg = !h->capturing && debug_env("PSD_DEBUG_STAMPS") != nullptr;
        if (dbg) {
            sp_plan.dbg = reinterpret_cast<unsigned long long*>(ws.partial);
            cudaMemsetAsync(ws.partial, 0, 128, st);   // 16 counters
        }
        h->last_products = 1;
        e = launch_small_batch(sp, X, out, n, batch, lambda_out, ws.status, sp_plan, st);
        if (e != cudaSuccess) return cuda_fail(e, "small_batch");
        if (dbg) {
            unsigned long long t[16] = {};
            cudaStreamSynchronize(st);
            cudaMemcpy(t, sp_plan.dbg, sizeof(t), cudaMemcpyDeviceToHost);
            if (t[3]) std::fprintf(stderr, "psd small stamps (cycles/step, CTA 0, %llu steps): mma issue %.0f, mma wait + barrier %.0f, epilogue %.0f, fences + barrier %.0f\n",
                                   t[3], double(t[0]) / t[3], double(t[1]) / t[3], double(t[2]) / t[3], double(t[4]) / t[3]);
            if (t[7]) std::fprintf(stderr, "psd small stamps (cycles/pair, CTA 0, %llu pairs): load + bound + X_0 %.0f (loads %.0f, bound %.0f, X_0 %.0f), final product %.0f\n",
                                   t[7], double(t[5]) / t[7], double(t[8]) / t[7], double(t[9]) / t[7], double(t[10]) / t[7], double(t[6]) / t[7]);
            std::fprintf(stderr, "psd small stamps: first pair loads %llu cycles\n", t[11]);
        }
        h->kernel_launches += 1;
        if (evs.first) {
            cudaEventRecord(evs.second, st);
            h->ev_pairs.push_back(evs);
            h->product_launches_profiled += 1;     // one launch carries the whole chain
        } else if (h->capturing && h->cap_ev[1]) {
            cudaEventRecordWithFlags(h->cap_ev[1], st, cudaEventRecordExternal);
        }
        return PSD_OK;
    }
    // (a1) bound
    const double* lam = nullptr;
    if (h->bound == PSD_BOUND_FROBENIUS || h->bound == PSD_BOUND_LANCZOS) {
        const int nblk = bound_blocks_per_matrix(n, batch);
        e = launch_frobenius_partials(X, n, batch, ws.partial, nblk, st, form);
        if (e != cudaSuccess) return cuda_fail(e, "frobenius_partials");
        h->kernel_launches += 2;
        e = launch_finalize_bound(ws.partial, nblk, batch, ws.lambda, lambda_out, ws.status, st);
        if (e != cudaSuccess) return cuda_fail(e, "finalize_bound");
        lam = ws.lambda;
    } else {
        lam = lambda_in;
        if (lambda_out && lambda_out != lambda_in) {
            e = cudaMemcpyAsync(lambda_out, lambda_in, batch * sizeof(double), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "lambda copy");
        }
    }
    const bool split = ws.split;
    double sc[B_COUNT];
    for (int i = 0; i < B_COUNT; ++i) sc[i] = 1.0;
    if (split && ws.op == OpType::F16) {
        sc[B_X0] = sc[B_XA] = sc[B_XB] = h->s_z;
        sc[B_Y] = h->s_y;
        sc[B_UA] = sc[B_UB] = h->s_u;
    }
    // upper-only operand storage: X0's lower triangle is read only inside the diagonal tiles (at most
    // 256 x 256), so the scale pass writes the mirrored 64-tiles there alone
    const int x0_mirror_block = upper_only_mode(h, n, batch, npad) ? 256 : 0;
    if (h->bound == PSD_BOUND_LANCZOS) {
        // X / lambda_F into the operand buffer, Lanczos on its square, then lambda~ <- the
        // Theorem-2 bound (never looser than lambda_F); the real scale below uses it
        rc = ensure_lz(h, npad, batch);
        if (rc != PSD_OK) return rc;
        e = launch_scale_convert(ws.op, X, n, npad, batch, lam, 1.0, ws.op_buf[B_X0], nullptr, sc[B_X0], nullptr, 0.0, st,
                                 form, x0_mirror_block);
        if (e != cudaSuccess) return cuda_fail(e, "scale_convert (Lanczos bound)");
        e = launch_lanczos_bound(ws.op, ws.op_buf[B_X0], sc[B_X0], n, npad, batch, h->lz_steps, h->lz_safety,
                                 ws.lz_scratch, ws.lambda, lambda_out, st);
        if (e != cudaSuccess) return cuda_fail(e, "Lanczos bound");
        h->kernel_launches += 1 + lanczos_launches(h->lz_steps, n);
    }
    // psd_polar's block-restricted products run on the 1-CTA kernel (tile sub-blocks, K ranges)
    const bool pair_ok = npad % 256 == 0 && use_pair_kernel(n, batch) && (h->polar_m == 0 || h->pol.tiles);
    const bool bn64 = !pair_ok && sym_gemm_bn(npad, batch) == 64;
    const CUtensorMap* bmaps = bn64 ? ws.tmap64 : ws.tmap;
    auto maps = [&](int A, int B) {
        OperandMaps m;
        m.a = ws.tmap[A];
        m.b = bmaps[B];
        m.a_lo = ws.tmap[split ? A + B_COUNT : A];
        m.b_lo = bmaps[split ? B + B_COUNT : B];
        m.a_t = ws.tmap64[A];
        m.b_t = ws.tmap64[B];
        m.a_lo_t = ws.tmap64[split ? A + B_COUNT : A];
        m.b_lo_t = ws.tmap64[split ? B + B_COUNT : B];
        return m;
    };
    // (a2) scale + convert; the products-free sign chain finishes here
    e = launch_scale_convert(ws.op, X, n, npad, batch, lam, 1.0, ws.op_buf[B_X0],
                             split ? ws.op_buf[B_X0 + B_COUNT] : nullptr, sc[B_X0],
                             (want_sign && steps.empty()) ? out : nullptr, sign_only, st, form, x0_mirror_block);
    if (e != cudaSuccess) return cuda_fail(e, "scale_convert");
    h->kernel_launches += 1;
    // (a3-a6) products
    if (steps.size() > static_cast<size_t>(kMaxSteps)) return fail(PSD_EUNSUPPORTED, "too many products");
    e = cudaMemsetAsync(ws.counters, 0, steps.size() * sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "counter reset");
    GemmShape shape{npad, batch, ws.tiles, ws.tiles_per_matrix, ws.counters};
    shape.kchunk = product_kchunk(h, split, n, npad, batch);
    std::pair<cudaEvent_t, cudaEvent_t> evp{nullptr, nullptr};
    if (h->profiling && !h->capturing && !steps.empty()) {
        evp = {take_event(h), take_event(h)};
        cudaEventRecord(evp.first, st);
    } else if (h->capturing && h->cap_ev[0] && !steps.empty()) {
        cudaEventRecordWithFlags(h->cap_ev[0], st, cudaEventRecordExternal);
    }
    const bool pair = pair_ok;
    // the chain's operand copies hold only their upper tiles (16-bit operands)
    const bool upper_only = upper_only_mode(h, n, batch, npad);
    shape.upper_only = upper_only ? 1 : 0;
    auto make_ep = [&](const Step& s) {
        EpiParams ep{};
        ep.alpha = static_cast<float>(s.alpha / (sc[s.A] * sc[s.B]));
        ep.alpha_dev = s.alpha_lambda ? lam : nullptr;
        ep.beta = static_cast<float>(s.D >= 0 ? s.beta / sc[s.D] : s.beta);
        ep.out_scale = s.out_op >= 0 ? static_cast<float>(sc[s.out_op]) : 1.0f;
        if (s.D >= 0) {
            ep.Dop = ws.op_buf[s.D];
            ep.Dop_lo = split ? ws.op_buf[s.D + B_COUNT] : nullptr;
        } else if (s.D == D_XIN) {
            ep.Df = X;
            ep.ldDf = n;
            ep.strideDf = static_cast<int64_t>(n) * n;
            ep.nDf = n;
            if (admm) {           // ADMM: the addend is M, and X_next = sigma (S - M) is written too
                ep.Df2 = admm->form.Xk;
                ep.df2_scale = admm->form.inv_sigma;
                ep.ddiag = admm->form.y;
                ep.outF2 = admm->x_out;
                ep.outF2_scale = admm->sigma;
            }
        }
        ep.out_op = s.out_op >= 0 ? ws.op_buf[s.out_op] : nullptr;
        ep.out_lo = (s.out_op >= 0 && split) ? ws.op_buf[s.out_op + B_COUNT] : nullptr;
        if (s.outF) {
            ep.outF = out;
            ep.ldF = n;
            ep.strideF = static_cast<int64_t>(n) * n;
            ep.nF = n;
        }
        ep.dbg_nostore = debug_env("PSD_DEBUG_NOSTORE") != nullptr ? 1 : 0;   // debug build only
        ep.upper_only = upper_only ? 1 : 0;
        return ep;
    };
    h->last_products = static_cast<int64_t>(steps.size());
    for (size_t si = 0; si < steps.size(); ++si) {
        const Step& s = steps[si];
        shape.counter = ws.counters + si;
        Step sw = steps[si];
        if (h->polar_m) {
            // H = [[0, A], [A^T, 0]]: every iterate is block off-diagonal, Y = Z Z and the Horner
            // products block diagonal; only one diagonal block of Y / U -- the Gram side of the
            // smaller dimension: A^T A (bottom-right) for rows >= cols, A A^T (top-left) for wide A,
            // whose other side is numerically rank-deficient -- and the top-right block of Z' are
            // needed, each over the one nonzero K half
            const int m = h->polar_m;
            const bool wide = h->polar_wide;
            if (s.out_op == B_Y && s.A == s.B) {          // Y = Z Z: Z_BL Z_TR (K [0, m)) or Z_TR Z_BL (K [m, 2m))
                shape.sub_mode = wide ? 3 : 1;
                shape.k_begin = wide ? m : 0;
                shape.k_end = wide ? 2 * m : m;
            } else if (s.out_op == B_UA || s.out_op == B_UB) {   // U in the Y block
                shape.sub_mode = wide ? 3 : 1;
                shape.k_begin = wide ? 0 : m;
                shape.k_end = wide ? m : 2 * m;
            } else {                                      // Z'_TR = c0 Z_TR + Z_TR U_BR  or  + U_TL Z_TR
                shape.sub_mode = 2;
                shape.k_begin = wide ? 0 : m;
                shape.k_end = wide ? m : 2 * m;
                if (wide) std::swap(sw.A, sw.B);          // Z U = U Z (polynomials in H commute)
            }
            shape.sub_m = m;
            if (pair) {                                   // the CTA-pair kernel takes tile lists
                const auto& pl = h->pol;
                shape.tiles = shape.sub_mode == 2 ? pl.tiles + 2 * pl.nsym : pl.tiles + (shape.sub_mode == 1 ? pl.nsym : 0);
                shape.tiles_per_matrix = shape.sub_mode == 2 ? pl.ntr : pl.nsym;
            }
        }
        EpiParams ep = make_ep(s);
        const bool dbg = pair && !h->capturing && debug_env("PSD_DEBUG_STAMPS") != nullptr;
        if (dbg) {
            ep.dbg = reinterpret_cast<unsigned long long*>(ws.partial + batch * 128);
            cudaMemsetAsync(ep.dbg, 0, 128, st);
            cudaMemsetAsync(ep.dbg + 8, 0xFF, 8, st);
            cudaMemsetAsync(ep.dbg + 11, 0xFF, 8, st);
        }
        // debug build: every CTA's phase stamps of the 1-CTA kernel (PSD_DEBUG_TIMELINE; synchronous)
        static unsigned long long* tl_buf = nullptr;
        constexpr int kTlSlots = 1 << 16;
        const bool tl = !pair && !h->capturing && debug_env("PSD_DEBUG_TIMELINE") != nullptr;
        if (tl) {
            if (!tl_buf && cudaMalloc(&tl_buf, kTlSlots * sizeof(unsigned long long)) != cudaSuccess) tl_buf = nullptr;
            if (tl_buf) {
                cudaMemsetAsync(tl_buf, 0, kTlSlots * sizeof(unsigned long long), st);
                ep.dbg_all = tl_buf;
            }
        }
        e = pair ? launch_sym_gemm_2cta(ws.op, split, maps(sw.A, sw.B), shape, ep, st)
                 : launch_sym_gemm(ws.op, split, maps(sw.A, sw.B), shape, ep, st);
        if (e != cudaSuccess) return cuda_fail(e, "sym_gemm");
        h->kernel_launches += 1;
        if (dbg) {           // debug only: per-product phase counters of the pair kernel
            unsigned long long t[13] = {};
            cudaStreamSynchronize(st);
            cudaMemcpy(t, ep.dbg, sizeof(t), cudaMemcpyDeviceToHost);
            const double tiles = t[4] ? double(t[4]) : 1.0;
            std::fprintf(stderr, "psd step %zu (D %d, out %s): loop %.0f = tile %.0f + acc %.0f + operand %.0f + issue; "
                         "epilogue acc-wait %.0f work %.0f cycles/tile; %llu clusters (tiles %llu..%llu), starts "
                         "spread %.1f us, last end %.1f us after first start\n", si, s.D, s.outF ? "fp32" : "op",
                         t[3] / tiles, t[0] / tiles, t[1] / tiles, t[2] / tiles, t[5] / (2 * tiles), t[6] / (2 * tiles),
                         t[7], t[11], t[12], (t[9] - t[8]) * 1e-3, (t[10] - t[8]) * 1e-3);
        }
        if (tl && tl_buf) {
            std::vector<unsigned long long> t(kTlSlots);
            cudaStreamSynchronize(st);
            cudaMemcpy(t.data(), tl_buf, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            std::vector<double> wait, loop, epi, pre, chunk, post, addend;
            unsigned long long t0 = ~0ull, s_max = 0, e_max = 0;
            int ctas = 0;
            for (int c = 0; c < kTlSlots / 8 && t[8 * c + 3]; ++c, ++ctas) {
                const unsigned long long* u = &t[8 * c];
                t0 = std::min(t0, u[0]);
                s_max = std::max(s_max, u[0]);
                e_max = std::max(e_max, u[3]);
                wait.push_back(double(u[1] - u[0]));
                loop.push_back(double(u[2] - u[1]));
                epi.push_back(double(u[3] - u[2]));
                if (u[4] && u[5]) {
                    pre.push_back(double(u[4] - u[2]));      // accumulator ready -> first chunk's epilogue
                    chunk.push_back(double(u[5] - u[4]));    // one epilogue_chunk
                    post.push_back(double(u[6] - u[5]));     // -> final barrier passed
                    if (u[7] > u[4]) addend.push_back(double(u[7] - u[4]));   // chunk start -> addend added
                }
            }
            auto med = [](std::vector<double> v) {
                if (v.empty()) return 0.0;
                std::sort(v.begin(), v.end());
                return v[v.size() / 2] * 1e-3;
            };
            auto mx = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()) * 1e-3; };
            if (ctas)
                std::fprintf(stderr, "psd timeline step %zu: %d CTAs, starts spread %.2f us, prologue+wait med %.2f us, "
                             "mainloop med %.2f max %.2f us, epilogue+exit med %.2f max %.2f us (acc->chunk %.2f, "
                             "chunk %.2f of which addend %.2f, chunk->barrier %.2f), first start -> last end %.2f us\n", si,
                             ctas, (s_max - t0) * 1e-3, med(wait), med(loop), mx(loop), med(epi), mx(epi), med(pre),
                             med(chunk), med(addend), med(post), (e_max - t0) * 1e-3);
        }
    }
    if (evp.first) {
        cudaEventRecord(evp.second, st);
        h->ev_pairs.push_back(evp);
        h->product_launches_profiled += static_cast<int64_t>(steps.size());
    } else if (h->capturing && h->cap_ev[1] && !steps.empty()) {
        cudaEventRecordWithFlags(h->cap_ev[1], st, cudaEventRecordExternal);
    }
    return PSD_OK;
}

void free_graph_entry(psd_filter_s::GraphEntry& g) {
    cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    for (auto e : g.own)
        if (e) cudaEventDestroy(e);
}

void free_graphs(psd_filter_s* h) {
    for (auto& g : h->graphs) free_graph_entry(g);
    h->graphs.clear();
}

// psd_project through the graph cache: the first call with a given (pointers, shape, mode) key is
// captured (thread-local capture mode, internal stream) and instantiated; every call then costs
// one cudaGraphLaunch on the caller's stream.  Workspace growth happens before capture.
psd_status_t run(psd_filter_t h, const float* X, int64_t n64, int64_t batch64, float* out,
                 const double* lambda_in, double* lambda_out, bool want_sign, cudaStream_t st) {
    if (!h || !h->use_graphs || h->capturing) return run_body(h, X, n64, batch64, out, lambda_in, lambda_out, want_sign, st);
    psd_status_t rc = check_args(h, X, n64, batch64, out);
    if (rc != PSD_OK) return rc;
    const int64_t key_prec = h->prec, key_bound = h->bound;
    psd_filter_s::GraphEntry* hit = nullptr;
    for (auto& g : h->graphs)
        if (g.X == X && g.out == out && g.lin == lambda_in && g.lout == lambda_out && g.n == n64 && g.batch == batch64 &&
            g.want_sign == static_cast<int>(want_sign) && g.prec == key_prec && g.bound == key_bound) {
            hit = &g;
            break;
        }
    if (!hit) {
        // make sure every allocation exists, then capture
        rc = ensure_ws(h, static_cast<int>(padded_n(n64, batch64)), static_cast<int>(batch64));
        if (rc != PSD_OK) return rc;
        if (h->bound == PSD_BOUND_LANCZOS) {
            rc = ensure_lz(h, static_cast<int>(padded_n(n64, batch64)), static_cast<int>(batch64));
            if (rc != PSD_OK) return rc;
        }
        if (!h->capture_stream) {
            cudaError_t e = cudaStreamCreateWithFlags(&h->capture_stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
        const int64_t k0 = h->kernel_launches, p0 = h->product_launches_profiled;
        cudaEvent_t own[2] = {nullptr, nullptr};
        if (cudaEventCreate(&own[0]) != cudaSuccess || cudaEventCreate(&own[1]) != cudaSuccess) {
            for (auto x : own)
                if (x) cudaEventDestroy(x);
            return fail(PSD_ECUDA, "cudaEventCreate");
        }
        cudaError_t e = cudaStreamBeginCapture(h->capture_stream, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamBeginCapture");
        h->capturing = true;
        h->cap_ev[0] = own[0];
        h->cap_ev[1] = own[1];
        rc = run_body(h, X, n64, batch64, out, lambda_in, lambda_out, want_sign, h->capture_stream);
        h->capturing = false;
        h->cap_ev[0] = h->cap_ev[1] = nullptr;
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(h->capture_stream, &graph);
        auto drop = [&]() {
            if (graph) cudaGraphDestroy(graph);
            for (auto x : own) cudaEventDestroy(x);
        };
        if (rc != PSD_OK) {
            drop();
            return rc;
        }
        if (e != cudaSuccess) {
            drop();
            return cuda_fail(e, "cudaStreamEndCapture");
        }
        // the event-record nodes bracketing the product run (absent for a product-free chain)
        cudaGraphNode_t ev_node[2] = {nullptr, nullptr};
        {
            size_t count = 0;
            cudaGraphGetNodes(graph, nullptr, &count);
            std::vector<cudaGraphNode_t> nodes(count);
            if (count) cudaGraphGetNodes(graph, nodes.data(), &count);
            for (auto nd : nodes) {
                cudaGraphNodeType ty;
                if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeEventRecord) continue;
                cudaEvent_t ev = nullptr;
                cudaGraphEventRecordNodeGetEvent(nd, &ev);
                for (int i = 0; i < 2; ++i)
                    if (ev == own[i]) ev_node[i] = nd;
            }
        }
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        if (e != cudaSuccess) {
            drop();
            return cuda_fail(e, "cudaGraphInstantiate");
        }
        if (h->graphs.size() >= 8) {       // evict the least recently used
            size_t lru = 0;
            for (size_t i = 1; i < h->graphs.size(); ++i)
                if (h->graphs[i].last_use < h->graphs[lru].last_use) lru = i;
            free_graph_entry(h->graphs[lru]);
            h->graphs.erase(h->graphs.begin() + lru);
        }
        psd_filter_s::GraphEntry g{X, out, lambda_in, lambda_out, n64, batch64, static_cast<int>(want_sign), static_cast<int>(key_prec),
                     static_cast<int>(key_bound), exec, h->kernel_launches - k0, 0, 0, graph,
                     {ev_node[0], ev_node[1]}, {own[0], own[1]}, false};
        if (!(ev_node[0] && ev_node[1])) g.ev_node[0] = g.ev_node[1] = nullptr;
        // the product count of the sequence (for profiling) = its number of product kernels
        g.products = h->last_products;
        h->kernel_launches = k0;
        h->product_launches_profiled = p0;
        h->graphs.push_back(g);
        hit = &h->graphs.back();
    }
    hit->last_use = ++h->graph_clock;
    // profiling: the graph's own record nodes around the product run are pointed at a fresh event
    // pair for this launch, so the interval is the product kernels only (bound, scale, counter
    // reset excluded)
    std::pair<cudaEvent_t, cudaEvent_t> evp{nullptr, nullptr};
    cudaError_t e;
    if (h->profiling && hit->ev_node[0]) {
        evp = {take_event(h), take_event(h)};
        if ((e = cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[0], evp.first)) != cudaSuccess ||
            (e = cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[1], evp.second)) != cudaSuccess)
            return cuda_fail(e, "cudaGraphExecEventRecordNodeSetEvent");
        hit->borrowed = true;
    } else if (hit->borrowed) {
        // back to the graph's own events (the pool's may be reused elsewhere)
        if ((e = cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[0], hit->own[0])) != cudaSuccess ||
            (e = cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[1], hit->own[1])) != cudaSuccess)
            return cuda_fail(e, "cudaGraphExecEventRecordNodeSetEvent");
        hit->borrowed = false;
    }
    e = cudaGraphLaunch(hit->exec, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
    h->kernel_launches += hit->kernels;
    if (evp.first) {
        h->ev_pairs.push_back(evp);
        h->product_launches_profiled += hit->products;
    }
    return PSD_OK;
}

// ---------------------------------------------------------------- NCCL (resolved at run time)
struct NcclUniqueId {          // ncclUniqueId: passed BY VALUE to ncclCommInitRank
    char internal[128];
};

struct NcclApi {
    using GetUniqueId = int (*)(void*);
    using CommInitRank = int (*)(void**, int, NcclUniqueId, int);
    using AllGather = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
    using CommDestroy = int (*)(void*);
    using GetErrorString = const char* (*)(int);
    GetUniqueId get_unique_id = nullptr;
    CommInitRank comm_init_rank = nullptr;
    AllGather all_gather = nullptr;
    CommDestroy comm_destroy = nullptr;
    GetErrorString error_string = nullptr;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy torch loaded
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (lib) {
            api.get_unique_id = reinterpret_cast<NcclApi::GetUniqueId>(dlsym(lib, "ncclGetUniqueId"));
            api.comm_init_rank = reinterpret_cast<NcclApi::CommInitRank>(dlsym(lib, "ncclCommInitRank"));
            api.all_gather = reinterpret_cast<NcclApi::AllGather>(dlsym(lib, "ncclAllGather"));
            api.comm_destroy = reinterpret_cast<NcclApi::CommDestroy>(dlsym(lib, "ncclCommDestroy"));
            api.error_string = reinterpret_cast<NcclApi::GetErrorString>(dlsym(lib, "ncclGetErrorString"));
            api.ok = api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy;
        }
    }
    return api;
}

constexpr int kNcclInt8 = 0;   // byte-count all-gathers: ncclInt8

psd_status_t nccl_fail(int rc, const char* where) {
    const char* m = nccl().error_string ? nccl().error_string(rc) : "?";
    return fail(PSD_ENCCL, std::string(where) + ": " + m);
}

void free_rowpanel_ws(psd_filter_s::RowPanel& rp) {
    if (rp.xg) cudaFree(rp.xg);
    if (rp.pfull) cudaFree(rp.pfull);
    if (rp.packed_op) cudaFree(rp.packed_op);
    if (rp.packed_f32) cudaFree(rp.packed_f32);
    if (rp.codes) cudaFree(rp.codes);
    if (rp.codes_g) cudaFree(rp.codes_g);
    if (rp.cs) cudaStreamDestroy(rp.cs);
    rp = psd_filter_s::RowPanel();
}

void free_hostpipe(psd_filter_s* h) {
    auto& hp = h->hp;
    if (hp.s[0]) cudaDeviceSynchronize();
    for (auto& p : hp.dx) { if (p) cudaFree(p); p = nullptr; }
    for (auto& p : hp.dout) { if (p) cudaFree(p); p = nullptr; }
    for (auto& q : hp.s) { if (q) cudaStreamDestroy(q); q = nullptr; }
    hp.chunk_bytes = 0;
    hp.nslots = 0;
}

void free_rowpanel(psd_filter_s* h) {
    if (h->rp.codes) {
        cudaDeviceSynchronize();
        free_rowpanel_ws(h->rp);
    }
}

psd_status_t ensure_rowpanel(psd_filter_s* h, int n, int nranks) {
    auto& rp = h->rp;
    const int npad = (n + 255) / 256 * 256;
    const OpType op = op_of(h->prec);
    if (rp.npad == npad && rp.n == n && rp.nranks == nranks && rp.op == op && rp.codes) return PSD_OK;
    if (rp.codes) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
    }
    free_rowpanel_ws(rp);
    const int nt = npad / 256;
    const int per = rowpanel_tiles(nt, nranks, 0, nullptr, 0);
    std::vector<uint32_t> codes(static_cast<size_t>(nranks) * per);
    rp.counts.resize(nranks);
    for (int r = 0; r < nranks; ++r) rp.counts[r] = rowpanel_tiles(nt, nranks, r, codes.data() + r * per, per);
    // each product's tiles are gathered in `chunks` all-gathers (SURVEY 8(e) "Overlap"): chunk c
    // of every rank's list is computed, then gathered on the communication stream while chunk c+1
    // is computed; the gathered buffer is [chunk][rank][ct] and codes_g maps it to tile codes
    const int chunks = std::max(1, std::min(kRowPanelChunks, per));
    const int ct = (per + chunks - 1) / chunks;
    std::vector<uint32_t> codes_g(static_cast<size_t>(chunks) * nranks * ct, 0xFFFFFFFFu);
    for (int c = 0; c < chunks; ++c)
        for (int r = 0; r < nranks; ++r)
            for (int i = 0; i < ct && c * ct + i < per; ++i)
                codes_g[(static_cast<size_t>(c) * nranks + r) * ct + i] = codes[static_cast<size_t>(r) * per + c * ct + i];
    const size_t tiles = codes_g.size();
    if (cudaMalloc(&rp.xg, static_cast<size_t>(n) * n * 4) != cudaSuccess ||
        cudaMalloc(&rp.pfull, static_cast<size_t>(npad) * npad * 4) != cudaSuccess ||
        cudaMalloc(&rp.packed_op, tiles * 65536 * op_bytes(op)) != cudaSuccess ||
        cudaMalloc(&rp.packed_f32, tiles * 65536 * 4) != cudaSuccess ||
        cudaMalloc(&rp.codes, codes.size() * 4) != cudaSuccess ||
        cudaMalloc(&rp.codes_g, codes_g.size() * 4) != cudaSuccess) {
        free_rowpanel_ws(rp);
        return fail(PSD_ENOMEM, "cudaMalloc row-panel workspace failed");
    }
    cudaError_t se = cudaStreamCreateWithFlags(&rp.cs, cudaStreamNonBlocking);
    if (se != cudaSuccess) {
        free_rowpanel_ws(rp);
        return cuda_fail(se, "cudaStreamCreate");
    }
    cudaMemcpy(rp.codes, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(rp.codes_g, codes_g.data(), codes_g.size() * 4, cudaMemcpyHostToDevice);
    rp.chunks = chunks;
    rp.ct = ct;
    cudaMemset(rp.pfull, 0, static_cast<size_t>(npad) * npad * 4);
    rp.npad = npad;
    rp.n = n;
    rp.nranks = nranks;
    rp.per = per;
    rp.op = op;
    return PSD_OK;
}

// Row-panel Algorithm 2.  comm == nullptr: `nranks` virtual ranks in this process (X, out full).
psd_status_t run_rowpanel(psd_filter_s* h, const float* X, int64_t n64, int rank, int nranks, float* out,
                          bool want_sign, void* comm, cudaStream_t st) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (!X || !out) return fail(PSD_EINVAL, "null X or out");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PSD_EINVAL, "bad rank / nranks");
    if (n64 < 256 || n64 > 65536 || n64 % nranks) return fail(PSD_EINVAL, "row panels need 256 <= n, n % nranks == 0");
    if (split_of(h->prec)) return fail(PSD_EUNSUPPORTED, "row panels: FP16, BF16, TF32 only");
    if (h->bound != PSD_BOUND_FROBENIUS) return fail(PSD_EUNSUPPORTED, "row panels: Frobenius bound only");
    if (comm && !nccl().ok) return fail(PSD_ENCCL, "libnccl.so.2 not available");
    const int n = static_cast<int>(n64);
    const int npad = (n + 255) / 256 * 256;
    psd_status_t rc = ensure_ws(h, npad, 1);
    if (rc != PSD_OK) return rc;
    rc = ensure_rowpanel(h, n, nranks);
    if (rc != PSD_OK) return rc;
    Workspace& ws = h->ws;
    auto& rp = h->rp;
    const int rows = n / nranks;
    cudaError_t e;
    // (1) the full X on every rank (one all-gather of the input rows)
    const float* Xf = X;
    if (comm) {
        e = cudaMemcpyAsync(rp.xg + static_cast<int64_t>(rank) * rows * n, X, static_cast<size_t>(rows) * n * 4,
                            cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "row copy");
        int r = nccl().all_gather(rp.xg + static_cast<int64_t>(rank) * rows * n, rp.xg,
                                  static_cast<size_t>(rows) * n * 4, kNcclInt8, comm, st);
        if (r != 0) return nccl_fail(r, "ncclAllGather(X)");
        Xf = rp.xg;
    }
    // (2) bound (identical on every rank) and (3) scale + convert into the full X_0
    const int nblk = bound_blocks_per_matrix(n, 1);
    e = launch_frobenius_partials(Xf, n, 1, ws.partial, nblk, st);
    if (e == cudaSuccess) e = launch_finalize_bound(ws.partial, nblk, 1, ws.lambda, nullptr, ws.status, st);
    if (e == cudaSuccess)
        e = launch_scale_convert(ws.op, Xf, n, npad, 1, ws.lambda, 1.0, ws.op_buf[B_X0], nullptr, 1.0, nullptr, 0.0, st);
    if (e != cudaSuccess) return cuda_fail(e, "bound / scale");
    h->kernel_launches += 3;
    double sign_only = 0.0;
    std::vector<Step> steps = build_plan(h, want_sign, &sign_only);
    if (steps.empty()) return fail(PSD_EUNSUPPORTED, "row panels: filter without products");
    const int C = rp.chunks, ct = rp.ct;
    if (steps.size() * nranks * C > static_cast<size_t>(kMaxSteps)) return fail(PSD_EUNSUPPORTED, "too many products");
    e = cudaMemsetAsync(ws.counters, 0, steps.size() * nranks * C * sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "counter reset");
    const int ob = op_bytes(ws.op);
    const size_t tile_elems = 65536;
    std::vector<cudaEvent_t> used;
    // (4) the products: each rank its upper tiles, packed, chunk by chunk; chunk c's all-gather runs
    // on the communication stream while the compute stream does chunk c+1; unpack on every rank
    for (size_t si = 0; si < steps.size(); ++si) {
        const Step& s = steps[si];
        EpiParams ep{};
        ep.alpha = static_cast<float>(s.alpha);
        ep.alpha_dev = s.alpha_lambda ? ws.lambda : nullptr;
        ep.beta = static_cast<float>(s.beta);
        ep.out_scale = 1.0f;
        if (s.D >= 0) {
            ep.Dop = ws.op_buf[s.D];
        } else if (s.D == D_XIN) {
            ep.Df = Xf;
            ep.ldDf = n;
            ep.strideDf = static_cast<int64_t>(n) * n;
            ep.nDf = n;
        }
        ep.packed_f32 = s.outF ? 1 : 0;
        OperandMaps m;
        m.a = ws.tmap[s.A];
        m.b = ws.tmap[s.B];
        m.a_lo = m.a;
        m.b_lo = m.b;
        m.a_t = m.a_lo_t = ws.tmap64[s.A];
        m.b_t = m.b_lo_t = ws.tmap64[s.B];
        // upper-only operand storage (16-bit): the unpack writes each gathered tile without its
        // mirror and the loader reads the left part of a panel transposed
        const bool upper_only = ws.op != OpType::TF32 && debug_env("PSD_NO_UPPER_ONLY") == nullptr;
        const int r0 = comm ? rank : 0, r1 = comm ? rank + 1 : nranks;
        const size_t tbytes = tile_elems * (s.outF ? 4 : ob);             // one packed tile
        uint8_t* gathered = s.outF ? reinterpret_cast<uint8_t*>(rp.packed_f32) : static_cast<uint8_t*>(rp.packed_op);
        for (int c = 0; c < C; ++c) {
            for (int vr = r0; vr < r1; ++vr) {
                const int cnt = std::min(ct, rp.counts[vr] - c * ct);
                if (cnt <= 0) continue;
                ep.packed = gathered + (static_cast<size_t>(c) * nranks + vr) * ct * tbytes;
                GemmShape shape{npad, 1, rp.codes + static_cast<size_t>(vr) * rp.per + c * ct, cnt,
                                ws.counters + (si * C + c) * nranks + vr};
                shape.upper_only = upper_only ? 1 : 0;
                e = launch_sym_gemm_2cta(ws.op, false, m, shape, ep, st);
                if (e != cudaSuccess) return cuda_fail(e, "sym_gemm_2cta (row panel)");
                h->kernel_launches += 1;
            }
            if (comm) {
                cudaEvent_t ready = take_event(h);
                used.push_back(ready);
                cudaEventRecord(ready, st);
                cudaStreamWaitEvent(rp.cs, ready, 0);
                uint8_t* slab = gathered + static_cast<size_t>(c) * nranks * ct * tbytes;
                int r = nccl().all_gather(slab + static_cast<size_t>(rank) * ct * tbytes, slab, ct * tbytes, kNcclInt8,
                                          comm, rp.cs);
                if (r != 0) return nccl_fail(r, "ncclAllGather(tiles)");
            }
        }
        if (comm) {
            cudaEvent_t gathered_ev = take_event(h);
            used.push_back(gathered_ev);
            cudaEventRecord(gathered_ev, rp.cs);
            cudaStreamWaitEvent(st, gathered_ev, 0);
        }
        e = launch_unpack_tiles(s.outF ? 4 : ob, gathered, rp.codes_g, C * nranks * ct,
                                s.outF ? static_cast<void*>(rp.pfull) : ws.op_buf[s.out_op], npad, st,
                                s.outF || !upper_only);
        if (e != cudaSuccess) return cuda_fail(e, "unpack");
        h->kernel_launches += 1;
    }
    // cudaStreamWaitEvent binds to the record made before it, so the events can be re-recorded
    for (auto x : used) h->ev_pool.push_back(x);
    // (5) this rank's rows (all rows for the virtual ranks) of the result
    const int row0 = comm ? rank * rows : 0;
    const int nrows = comm ? rows : n;
    e = cudaMemcpy2DAsync(out, static_cast<size_t>(n) * 4, rp.pfull + static_cast<size_t>(row0) * npad,
                          static_cast<size_t>(npad) * 4, static_cast<size_t>(n) * 4, nrows, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "result copy");
    return PSD_OK;
}

// ------------------------------------------------------------------ peer-memory row panels
void free_peerpath(psd_filter_s* h) {
    auto& pp = h->pp;
    if (pp.base.empty() && !pp.codes && !pp.flags_dev) return;
    cudaDeviceSynchronize();
    for (size_t q = 0; q < pp.base.size(); ++q) {
        if (!pp.base[q]) continue;
        if (pp.ipc_opened[q]) cudaIpcCloseMemHandle(pp.base[q]);
        else cudaFree(pp.base[q]);
    }
    if (pp.flags_dev) cudaFree(pp.flags_dev);
    if (pp.codes) cudaFree(pp.codes);
    pp = psd_filter_s::PeerPath();
}

// Region layout: [B_COUNT operand buffers npad^2][pfull npad^2 fp32][X n^2 fp32][flags 64 x u64]
psd_status_t peer_layout(psd_filter_s* h, int n, int nranks, int rank, bool is_virtual) {
    auto& pp = h->pp;
    if (n < 256 || n > 65536 || nranks < 1 || nranks > kMaxPeers || n % nranks || rank < 0 || rank >= nranks)
        return fail(PSD_EINVAL, "peer row panels: 256 <= n, 1 <= nranks <= 8, n % nranks == 0");
    if ((n / nranks) % 32) return fail(PSD_EINVAL, "peer row panels: rows per rank must be a multiple of 32");
    if (split_of(h->prec)) return fail(PSD_EUNSUPPORTED, "row panels: FP16, BF16, TF32 only");
    if (h->bound != PSD_BOUND_FROBENIUS) return fail(PSD_EUNSUPPORTED, "row panels: Frobenius bound only");
    free_peerpath(h);
    pp.n = n;
    pp.npad = (n + 255) / 256 * 256;
    pp.nranks = nranks;
    pp.rank = rank;
    pp.is_virtual = is_virtual;
    pp.op = op_of(h->prec);
    auto up = [](size_t x) { return (x + 4095) / 4096 * 4096; };
    pp.op_bytes_buf = up(static_cast<size_t>(pp.npad) * pp.npad * op_bytes(pp.op));
    pp.pfull_off = B_COUNT * pp.op_bytes_buf;
    pp.xg_off = pp.pfull_off + up(static_cast<size_t>(pp.npad) * pp.npad * 4);
    pp.flags_off = pp.xg_off + up(static_cast<size_t>(n) * n * 4);
    pp.region_bytes = pp.flags_off + 4096;
    pp.base.assign(nranks, nullptr);
    pp.ipc_opened.assign(nranks, 0);
    return PSD_OK;
}

psd_status_t peer_alloc_local(psd_filter_s* h, int q) {
    auto& pp = h->pp;
    void* p = nullptr;
    if (cudaMalloc(&p, pp.region_bytes) != cudaSuccess) return fail(PSD_ENOMEM, "cudaMalloc peer region failed");
    cudaMemset(p, 0, pp.region_bytes);        // zero padding of every operand; zero flags
    pp.base[q] = static_cast<uint8_t*>(p);
    std::vector<CUtensorMap> maps(2 * B_COUNT);     // 128-row boxes, then 64 x 64 (transposed loads)
    for (int i = 0; i < B_COUNT; ++i)
        if (!make_operand_tmap(&maps[i], pp.base[q] + i * pp.op_bytes_buf, pp.op, pp.npad, 1) ||
            !make_operand_tmap(&maps[B_COUNT + i], pp.base[q] + i * pp.op_bytes_buf, pp.op, pp.npad, 1, 64))
            return fail(PSD_ECUDA, "cuTensorMapEncodeTiled failed");
    if (pp.tmaps.size() < static_cast<size_t>(pp.nranks)) pp.tmaps.resize(pp.nranks);
    pp.tmaps[q] = maps;
    return PSD_OK;
}

// tile codes + the device table of flag arrays, once every base is known
psd_status_t peer_finish(psd_filter_s* h) {
    auto& pp = h->pp;
    const int nt = pp.npad / 256;
    pp.per = rowpanel_tiles(nt, pp.nranks, 0, nullptr, 0);
    std::vector<uint32_t> codes(static_cast<size_t>(pp.nranks) * std::max(pp.per, 1));
    pp.counts.assign(pp.nranks, 0);
    for (int r = 0; r < pp.nranks; ++r) pp.counts[r] = rowpanel_tiles(nt, pp.nranks, r, codes.data() + r * pp.per, pp.per);
    std::vector<unsigned long long*> fl(pp.nranks);
    for (int q = 0; q < pp.nranks; ++q) fl[q] = reinterpret_cast<unsigned long long*>(pp.base[q] + pp.flags_off);
    if (cudaMalloc(&pp.codes, codes.size() * 4) != cudaSuccess ||
        cudaMalloc(&pp.flags_dev, fl.size() * sizeof(void*)) != cudaSuccess)
        return fail(PSD_ENOMEM, "cudaMalloc peer tables failed");
    cudaMemcpy(pp.codes, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(pp.flags_dev, fl.data(), fl.size() * sizeof(void*), cudaMemcpyHostToDevice);
    pp.attached = true;
    return PSD_OK;
}

// Algorithm 2 over row panels with the product-and-gather fused into the product kernels:
// X rows -> every rank's X copy (peer copies), barrier, bound + scale on every rank, then per
// product: this rank's upper tiles, the epilogue storing each tile (and its mirror) into every
// rank's operand buffer, barrier; the final product stores each fp32 block to the rank owning
// its rows.  Virtual mode: all `nranks` regions are local and every rank's kernels run here.
psd_status_t run_rowpanel_p2p(psd_filter_s* h, const float* X, float* out, bool want_sign, cudaStream_t st) {
    auto& pp = h->pp;
    if (!pp.attached) return fail(PSD_EINVAL, "peer row panels: region not set up / attached");
    const int n = pp.n, npad = pp.npad, P = pp.nranks, rows = n / P;
    psd_status_t rc = ensure_ws(h, npad, 1);
    if (rc != PSD_OK) return rc;
    Workspace& ws = h->ws;
    cudaError_t e;
    const int r_lo = pp.is_virtual ? 0 : pp.rank, r_hi = pp.is_virtual ? P : pp.rank + 1;
    auto region = [&](int q, size_t off) { return static_cast<void*>(pp.base[q] + off); };
    auto xg = [&](int q) { return reinterpret_cast<float*>(pp.base[q] + pp.xg_off); };
    auto barrier = [&]() -> psd_status_t {
        ++pp.epoch;
        for (int r = r_lo; r < r_hi; ++r) {
            if ((e = launch_peer_signal(pp.flags_dev, P, r, pp.epoch, st)) != cudaSuccess) return cuda_fail(e, "peer signal");
        }
        for (int r = r_lo; r < r_hi; ++r) {
            const auto* fl = reinterpret_cast<const unsigned long long*>(pp.base[r] + pp.flags_off);
            if ((e = launch_peer_wait(fl, P, pp.epoch, h->peer_timeout_ns, ws.status, st)) != cudaSuccess)
                return cuda_fail(e, "peer wait");
        }
        h->kernel_launches += 2 * (r_hi - r_lo);
        return PSD_OK;
    };
    // (1) X rows into every rank's X copy
    for (int r = r_lo; r < r_hi; ++r)
        for (int q = 0; q < P; ++q) {
            const float* src = pp.is_virtual ? X + static_cast<int64_t>(r) * rows * n : X;
            e = cudaMemcpyAsync(xg(q) + static_cast<int64_t>(r) * rows * n, src, static_cast<size_t>(rows) * n * 4,
                                cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "X rows to peers");
        }
    if ((rc = barrier()) != PSD_OK) return rc;
    // (2) bound (identical on every rank) and (3) X_0 into every local region
    const int nblk = bound_blocks_per_matrix(n, 1);
    e = launch_frobenius_partials(xg(r_lo), n, 1, ws.partial, nblk, st);
    if (e == cudaSuccess) e = launch_finalize_bound(ws.partial, nblk, 1, ws.lambda, nullptr, ws.status, st);
    for (int r = r_lo; r < r_hi && e == cudaSuccess; ++r)
        e = launch_scale_convert(pp.op, xg(r), n, npad, 1, ws.lambda, 1.0, region(r, B_X0 * pp.op_bytes_buf), nullptr,
                                 1.0, nullptr, 0.0, st);
    if (e != cudaSuccess) return cuda_fail(e, "bound / scale");
    h->kernel_launches += 2 + (r_hi - r_lo);
    double sign_only = 0.0;
    std::vector<Step> steps = build_plan(h, want_sign, &sign_only);
    if (steps.empty()) return fail(PSD_EUNSUPPORTED, "row panels: filter without products");
    if (steps.size() * P > static_cast<size_t>(kMaxSteps)) return fail(PSD_EUNSUPPORTED, "too many products");
    e = cudaMemsetAsync(ws.counters, 0, steps.size() * P * sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "counter reset");
    // (4) the products, each fused with its all-gather
    for (size_t si = 0; si < steps.size(); ++si) {
        const Step& s = steps[si];
        for (int r = r_lo; r < r_hi; ++r) {
            if (pp.counts[r] == 0) continue;
            EpiParams ep{};
            ep.alpha = static_cast<float>(s.alpha);
            ep.alpha_dev = s.alpha_lambda ? ws.lambda : nullptr;
            ep.beta = static_cast<float>(s.beta);
            ep.out_scale = 1.0f;
            if (s.D >= 0) {
                ep.Dop = region(r, s.D * pp.op_bytes_buf);
            } else if (s.D == D_XIN) {
                ep.Df = xg(r);
                ep.ldDf = n;
                ep.strideDf = static_cast<int64_t>(n) * n;
                ep.nDf = n;
            }
            if (s.out_op >= 0) {
                ep.npeers = P;
                for (int q = 0; q < P; ++q) ep.out_peers[q] = region(q, s.out_op * pp.op_bytes_buf);
                ep.out_op = ep.out_peers[r];
            }
            if (s.outF) {
                ep.peer_rows = rows;
                for (int q = 0; q < P; ++q) ep.outF_peers[q] = reinterpret_cast<float*>(region(q, pp.pfull_off));
                ep.outF = ep.outF_peers[r];
                ep.ldF = npad;
                ep.strideF = 0;
                ep.nF = n;
            }
            OperandMaps m;
            m.a = pp.tmaps[r][s.A];
            m.b = pp.tmaps[r][s.B];
            m.a_lo = m.a;
            m.b_lo = m.b;
            m.a_t = m.a_lo_t = pp.tmaps[r][B_COUNT + s.A];
            m.b_t = m.b_lo_t = pp.tmaps[r][B_COUNT + s.B];
            GemmShape shape{npad, 1, pp.codes + static_cast<size_t>(r) * pp.per, pp.counts[r],
                            ws.counters + si * P + r};
            // upper-only operand storage: each tile goes to the peers without its mirror (half the
            // NVLink bytes); the loader reads the left part of a panel transposed
            shape.upper_only = (pp.op != OpType::TF32) ? 1 : 0;
            ep.upper_only = shape.upper_only;
            e = launch_sym_gemm_2cta(pp.op, false, m, shape, ep, st);
            if (e != cudaSuccess) return cuda_fail(e, "sym_gemm_2cta (peer row panel)");
            h->kernel_launches += 1;
        }
        if ((rc = barrier()) != PSD_OK) return rc;
    }
    // (5) this rank's rows of the result (every rank's rows in virtual mode)
    for (int r = r_lo; r < r_hi; ++r) {
        float* dst = pp.is_virtual ? out + static_cast<int64_t>(r) * rows * n : out;
        const float* src = reinterpret_cast<const float*>(region(r, pp.pfull_off)) + static_cast<size_t>(r) * rows * npad;
        e = cudaMemcpy2DAsync(dst, static_cast<size_t>(n) * 4, src, static_cast<size_t>(npad) * 4,
                              static_cast<size_t>(n) * 4, rows, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "result rows");
    }
    return PSD_OK;
}

}  // namespace

namespace {

void free_polar(psd_filter_s* h) {
    auto& p = h->pol;
    if (p.H || p.S || p.lam || p.part) cudaDeviceSynchronize();
    if (p.H) cudaFree(p.H);
    if (p.S) cudaFree(p.S);
    if (p.lam) cudaFree(p.lam);
    if (p.part) cudaFree(p.part);
    if (p.tiles) cudaFree(p.tiles);
    p = psd_filter_s::Polar{};
}

}  // namespace

extern "C" {

const char* psd_version(void) { return "psdfilter 0.1 sm_100a"; }

const char* psd_last_error(void) { return g_last_error.c_str(); }

psd_status_t psd_filter_create(int T, const int* degrees, const double* coeffs, double eps, psd_filter_t* out) {
    if (!out) return fail(PSD_EINVAL, "null out");
    *out = nullptr;
    if (T < 1 || T > 64) return fail(PSD_EINVAL, "T must be in [1, 64]");
    if (!degrees || !coeffs) return fail(PSD_EINVAL, "null degrees or coeffs");
    if (!(eps > 0.0 && eps < 1.0)) return fail(PSD_EINVAL, "eps must be in (0, 1)");
    auto* h = new psd_filter_s();
    h->eps = eps;
    const double* c = coeffs;
    for (int t = 0; t < T; ++t) {
        const int d = degrees[t];
        if (d < 1 || d > 15 || (d % 2) == 0) {
            delete h;
            return fail(PSD_EINVAL, "stage " + std::to_string(t) + ": degree must be odd in [1, 15]");
        }
        std::vector<double> cc(c, c + (d + 1) / 2);
        for (double v : cc) {
            if (!std::isfinite(v)) {
                delete h;
                return fail(PSD_EINVAL, "stage " + std::to_string(t) + ": non-finite coefficient");
            }
        }
        c += (d + 1) / 2;
        h->degrees.push_back(d);
        h->coeffs.push_back(cc);
    }
    compute_scales(h);
    *out = h;
    g_last_error.clear();
    return PSD_OK;
}

void psd_filter_destroy(psd_filter_t h) {
    if (!h) return;
    free_polar(h);
    free_peerpath(h);
    free_rowpanel(h);
    free_hostpipe(h);
    free_graphs(h);
    if (h->capture_stream) cudaStreamDestroy(h->capture_stream);
    for (auto& p : h->ev_pairs) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto& e : h->ev_pool) cudaEventDestroy(e);
    if (h->ws.status) {
        cudaDeviceSynchronize();
        free_ws(h->ws);
    }
    delete h;
}

psd_status_t psd_filter_set_precision(psd_filter_t h, psd_precision_t prec) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (prec < PSD_PREC_FP16 || prec > PSD_PREC_BF16X3) return fail(PSD_EINVAL, "unknown precision");
    h->prec = prec;
    return PSD_OK;
}

psd_status_t psd_filter_set_bound(psd_filter_t h, psd_bound_t bound) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (bound != PSD_BOUND_FROBENIUS && bound != PSD_BOUND_USER && bound != PSD_BOUND_LANCZOS)
        return fail(PSD_EINVAL, "unknown bound");
    h->bound = bound;
    return PSD_OK;
}

psd_status_t psd_filter_set_lanczos(psd_filter_t h, int steps, double safety) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (steps < 1 || steps > 64) return fail(PSD_EINVAL, "Lanczos steps must be in [1, 64]");
    if (!(safety >= 1.0) || !(safety <= 2.0)) return fail(PSD_EINVAL, "safety factor must be in [1, 2]");
    h->lz_steps = steps;
    h->lz_safety = safety;
    free_graphs(h);
    return PSD_OK;
}

psd_status_t psd_filter_set_accum_chunk(psd_filter_t h, int64_t kchunk) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (kchunk < 0 || kchunk % 64 || kchunk > (1 << 20)) return fail(PSD_EINVAL, "kchunk must be 0 or a positive multiple of 64");
    if (h->kchunk != static_cast<int>(kchunk)) free_graphs(h);   // captured launches carry the old value
    h->kchunk = static_cast<int>(kchunk);
    return PSD_OK;
}

int psd_filter_gemm_count(psd_filter_t h, int for_project) {
    if (!h) return -1;
    int g = 0;
    for (int d : h->degrees) g += d > 1 ? (d + 1) / 2 : 0;
    return g + (for_project ? 1 : 0);
}

int64_t psd_workspace_bytes(psd_filter_t h, int64_t n, int64_t batch) {
    if (!h || n < 1 || batch < 1) return -1;
    return ws_bytes(op_of(h->prec), split_of(h->prec), padded_n(n, batch), batch);
}

psd_status_t psd_project(psd_filter_t h, const float* X, int64_t n, int64_t batch, float* out, void* stream) {
    if (h && h->bound == PSD_BOUND_USER) return fail(PSD_EINVAL, "PSD_BOUND_USER: use psd_project_ex");
    return run(h, X, n, batch, out, nullptr, nullptr, false, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_sign(psd_filter_t h, const float* X, int64_t n, int64_t batch, float* out, void* stream) {
    if (h && h->bound == PSD_BOUND_USER) return fail(PSD_EINVAL, "PSD_BOUND_USER: use psd_project_ex");
    return run(h, X, n, batch, out, nullptr, nullptr, true, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_project_ex(psd_filter_t h, const float* X, int64_t n, int64_t batch, float* out,
                            const double* lambda_in, double* lambda_out, int want_sign, void* stream) {
    return run(h, X, n, batch, out, lambda_in, lambda_out, want_sign != 0, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_admm_update(psd_filter_t h, const float* C, const float* Xk, const float* y, double sigma, int64_t n,
                             int64_t batch, float* S_out, float* X_out, void* stream) {
    if (!Xk || !X_out) return fail(PSD_EINVAL, "null Xk or X_out");
    if ((reinterpret_cast<uintptr_t>(Xk) & 15) || (reinterpret_cast<uintptr_t>(X_out) & 15))
        return fail(PSD_EINVAL, "Xk and X_out must be 16-byte aligned");
    if (!(sigma > 0.0) || !std::isfinite(sigma)) return fail(PSD_EINVAL, "sigma must be finite and > 0");
    if (S_out == X_out) return fail(PSD_EINVAL, "S_out and X_out must be distinct");
    if (h && h->bound == PSD_BOUND_USER) return fail(PSD_EUNSUPPORTED, "psd_admm_update needs a device bound");
    AdmmArgs a;
    a.form.Xk = Xk;
    a.form.y = y;
    a.form.inv_sigma = static_cast<float>(1.0 / sigma);
    a.sigma = static_cast<float>(sigma);
    a.x_out = X_out;
    // no graph cache: sigma and the extra pointers are kernel arguments of every launch
    return run_body(h, C, n, batch, S_out, nullptr, nullptr, false, static_cast<cudaStream_t>(stream), &a);
}

psd_status_t psd_polar(psd_filter_t h, const float* A, int64_t n, int64_t batch, float* out,
                       const double* lambda_in, double* lambda_out, void* stream) {
    return psd_polar_rect(h, A, n, n, batch, out, lambda_in, lambda_out, stream);
}

psd_status_t psd_polar_rect(psd_filter_t h, const float* A, int64_t rows, int64_t cols, int64_t batch, float* out,
                            const double* lambda_in, double* lambda_out, void* stream) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (!A || !out) return fail(PSD_EINVAL, "null A or out");
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
        return fail(PSD_EINVAL, "A and out must be 16-byte aligned");
    if (rows < 1 || cols < 1 || batch < 1) return fail(PSD_EINVAL, "rows, cols and batch must be >= 1");
    const int64_t n = rows > cols ? rows : cols;
    if (2 * n > (1 << 20) || batch > (1 << 24) || 4 * n * n * batch > (int64_t(1) << 40))
        return fail(PSD_EINVAL, "polar problem too large");
    if (h->bound == PSD_BOUND_USER && !lambda_in) return fail(PSD_EINVAL, "PSD_BOUND_USER needs lambda_in");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto& p = h->pol;
    // block edge m: a tile boundary of the kernel that will run H's products (256 for the CTA-pair
    // kernel, whose tile lists are built below; 128 for the 1-CTA kernel)
    const int64_t m256 = (n + 255) / 256 * 256;
    const bool pair = use_pair_kernel(2 * m256, batch);
    const int64_t m = pair ? m256 : (n + kTile - 1) / kTile * kTile;
    const int64_t N = 2 * m;
    const int nblk = polar_blocks_per_matrix(static_cast<int>(m), static_cast<int>(batch));
    if (p.n != m || p.batch < batch || (p.tiles != nullptr) != pair) {
        // stable buffers per (block edge, batch) -- the sign run on H is graph-cached on these pointers
        free_graphs(h);
        free_polar(h);
        const size_t hb = static_cast<size_t>(batch) * N * N * sizeof(float);
        if (cudaMalloc(&p.H, hb) != cudaSuccess || cudaMalloc(&p.S, hb) != cudaSuccess ||
            cudaMalloc(&p.lam, batch * sizeof(double)) != cudaSuccess ||
            cudaMalloc(&p.part, static_cast<size_t>(batch) * 512 * sizeof(double)) != cudaSuccess) {
            free_polar(h);
            return fail(PSD_ENOMEM, "cudaMalloc polar workspace failed");
        }
        if (pair) {
            const int mt = static_cast<int>(m / 256);
            std::vector<uint32_t> sym(static_cast<size_t>(mt) * (mt + 1) / 2), all;
            make_tile_order(mt, mt > 16 ? "grouped8" : "row", sym.data());
            p.nsym = static_cast<int>(sym.size());
            all = sym;                                                    // top-left block
            for (uint32_t c : sym) all.push_back(c + ((static_cast<uint32_t>(mt) << 16) | static_cast<uint32_t>(mt)));  // bottom-right
            for (int I = 0; I < mt; ++I)                                  // top-right block, row-major
                for (int J = mt; J < 2 * mt; ++J) all.push_back((static_cast<uint32_t>(I) << 16) | static_cast<uint32_t>(J));
            p.ntr = mt * mt;
            if (cudaMalloc(&p.tiles, all.size() * sizeof(uint32_t)) != cudaSuccess ||
                cudaMemcpy(p.tiles, all.data(), all.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
                free_polar(h);
                return fail(PSD_ENOMEM, "polar tile lists");
            }
        }
        p.n = m;
        p.batch = batch;
    }
    if (p.wide != (rows < cols)) {
        free_graphs(h);            // the cached sign runs on H carry the other Gram side's plan
        p.wide = rows < cols;
    }
    // the product workspace of n' = 2m (its status word receives the non-finite flag of the norm)
    psd_status_t rc = ensure_ws(h, static_cast<int>(padded_n(N, batch)), static_cast<int>(batch));
    if (rc != PSD_OK) return rc;
    cudaError_t e = launch_polar_embed(A, static_cast<int>(rows), static_cast<int>(cols), static_cast<int>(m),
                                       static_cast<int>(batch), p.H, p.part, nblk, st);
    if (e != cudaSuccess) return cuda_fail(e, "polar_embed");
    h->kernel_launches += 1;
    const psd_bound_t bound = h->bound;
    h->polar_m = static_cast<int>(m);
    h->polar_wide = rows < cols;
    if (bound == PSD_BOUND_FROBENIUS) {
        // lambda~ = ||A||_F (the Frobenius bound of A; ||H||_F would be sqrt(2) looser)
        e = launch_finalize_bound(p.part, nblk, static_cast<int>(batch), p.lam, nullptr, h->ws.status, st);
        if (e != cudaSuccess) {
            h->polar_m = 0;
            h->polar_wide = false;
            return cuda_fail(e, "polar norm");
        }
        h->kernel_launches += 1;
        h->bound = PSD_BOUND_USER;
        rc = run(h, p.H, N, batch, p.S, p.lam, lambda_out, true, st);
        h->bound = bound;
    } else {
        // USER: the caller's bound; LANCZOS: the Theorem-2 bound of H (||H||_2 = ||A||_2)
        rc = run(h, p.H, N, batch, p.S, bound == PSD_BOUND_USER ? lambda_in : nullptr, lambda_out, true, st);
    }
    h->polar_m = 0;
    h->polar_wide = false;
    if (rc != PSD_OK) return rc;
    e = launch_polar_extract(p.S, static_cast<int>(rows), static_cast<int>(cols), static_cast<int>(m),
                             static_cast<int>(batch), out, st);
    if (e != cudaSuccess) return cuda_fail(e, "polar_extract");
    h->kernel_launches += 1;
    return PSD_OK;
}

psd_status_t psd_filter_certificate(psd_filter_t h, double* sign_err, double* relu_err, double* sign_argmax,
                                    double* relu_argmax) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    cudaError_t e = certify_chain(h->coeffs, h->eps, relu_err, relu_argmax, sign_err, sign_argmax);
    if (e != cudaSuccess) return cuda_fail(e, "certificate");
    return PSD_OK;
}

psd_status_t psd_status(psd_filter_t h, void* stream) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (!h->ws.status) return PSD_OK;
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    unsigned v = 0;
    e = cudaMemcpy(&v, h->ws.status, sizeof(unsigned), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "status readback");
    cudaMemset(h->ws.status, 0, sizeof(unsigned));
    if (v & 2u) return fail(PSD_ETIMEOUT, "peer row panels: a peer did not reach the barrier in time");
    return v ? PSD_ENONFINITE : PSD_OK;
}

psd_status_t psd_profile(psd_filter_t h, int enable) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    h->profiling = enable != 0;
    return PSD_OK;
}

psd_status_t psd_profile_read(psd_filter_t h, double* product_ms, int64_t* product_launches,
                              int64_t* kernel_launches) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    double total = 0.0;
    for (auto& p : h->ev_pairs) {
        cudaError_t e = cudaEventSynchronize(p.second);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, p.first, p.second);
        total += ms;
        h->ev_pool.push_back(p.first);
        h->ev_pool.push_back(p.second);
    }
    h->ev_pairs.clear();
    if (product_ms) *product_ms = total;
    if (product_launches) *product_launches = h->product_launches_profiled;
    if (kernel_launches) *kernel_launches = h->kernel_launches;
    h->product_launches_profiled = 0;
    h->kernel_launches = 0;
    return PSD_OK;
}

psd_status_t psd_project_host(psd_filter_t h, const float* X_host, int64_t n, int64_t batch, float* out_host,
                              int chunks, void* stream) {
    psd_status_t rc = check_args(h, X_host, n, batch, out_host);
    if (rc != PSD_OK) return rc;
    if (chunks < 1) chunks = 1;
    if (chunks > batch) chunks = static_cast<int>(batch);
    const int64_t per = (batch + chunks - 1) / chunks;
    auto& hp = h->hp;
    const size_t mat = static_cast<size_t>(n) * n * sizeof(float);
    cudaError_t e;
    // chunk buffers: enough that the host-to-device copies never wait for a device-to-host copy to
    // free a slot (both copy directions are the bound at c4, profiles/r1s3_e2e_bound.md)
    int slots = std::min<int>(6, chunks + 1);
    if (const char* v = debug_env("PSD_HOST_SLOTS")) slots = std::atoi(v);   // A/B only
    slots = std::max(1, std::min(slots, psd_filter_s::HostPipe::kMaxSlots));
    if (hp.chunk_bytes < per * mat || hp.nslots != slots) {
        free_hostpipe(h);
        for (int i = 0; i < 3; ++i)
            if ((e = cudaStreamCreateWithFlags(&hp.s[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_fail(e, "cudaStreamCreate");
        hp.nslots = slots;
        for (int i = 0; i < slots; ++i) {
            if (cudaMalloc(&hp.dx[i], per * mat) != cudaSuccess || cudaMalloc(&hp.dout[i], per * mat) != cudaSuccess) {
                free_hostpipe(h);
                return fail(PSD_ENOMEM, "cudaMalloc host-pipeline buffers failed");
            }
        }
        hp.chunk_bytes = per * mat;
    }
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    auto ev = [&]() { return take_event(h); };
    auto give = [&](cudaEvent_t x) { h->ev_pool.push_back(x); };
    cudaEvent_t start = ev();
    cudaEventRecord(start, user);
    for (auto q : hp.s) cudaStreamWaitEvent(q, start, 0);
    cudaEvent_t freed[psd_filter_s::HostPipe::kMaxSlots] = {};
    std::vector<cudaEvent_t> used = {start};
    // chunk boundaries: the first and the last chunk are half-size (the pipeline's fill -- the first
    // host-to-device copy -- and its drain -- the last device-to-host copy -- are not overlapped)
    std::vector<std::pair<int64_t, int64_t>> parts;
    {
        int64_t b0 = 0;
        const int64_t edge = (chunks >= 4 && per >= 2) ? per / 2 : per;
        while (b0 < batch) {
            const int64_t rem = batch - b0;
            int64_t nb = parts.empty() ? edge : per;
            // leave a half-size tail; never more than `per` matrices (the slot buffers' size)
            if (rem - nb > 0 && rem - nb < per) nb = std::max<int64_t>(1, std::min(per, rem - edge));
            nb = std::min(nb, rem);
            parts.emplace_back(b0, nb);
            b0 += nb;
        }
    }
    for (size_t c = 0; c < parts.size(); ++c) {
        const int slot = static_cast<int>(c % hp.nslots);
        const int64_t b0 = parts[c].first;
        const int64_t nb = parts[c].second;
        if (freed[slot]) cudaStreamWaitEvent(hp.s[0], freed[slot], 0);
        e = cudaMemcpyAsync(hp.dx[slot], X_host + b0 * n * n, nb * mat, cudaMemcpyHostToDevice, hp.s[0]);
        if (e != cudaSuccess) return cuda_fail(e, "H2D");
        cudaEvent_t in = ev();
        used.push_back(in);
        cudaEventRecord(in, hp.s[0]);
        cudaStreamWaitEvent(hp.s[1], in, 0);
        rc = run(h, hp.dx[slot], n, nb, hp.dout[slot], nullptr, nullptr, false, hp.s[1]);
        if (rc != PSD_OK) return rc;
        cudaEvent_t comp = ev();
        used.push_back(comp);
        cudaEventRecord(comp, hp.s[1]);
        cudaStreamWaitEvent(hp.s[2], comp, 0);
        e = cudaMemcpyAsync(out_host + b0 * n * n, hp.dout[slot], nb * mat, cudaMemcpyDeviceToHost, hp.s[2]);
        if (e != cudaSuccess) return cuda_fail(e, "D2H");
        cudaEvent_t outd = ev();
        used.push_back(outd);
        cudaEventRecord(outd, hp.s[2]);
        freed[slot] = outd;      // chunk c+nslots may reuse this slot's X and out buffers after the D2H
    }
    cudaEvent_t done = ev();
    used.push_back(done);
    cudaEventRecord(done, hp.s[2]);
    cudaStreamWaitEvent(user, done, 0);
    // cudaStreamWaitEvent binds to the record made before it, so the events can be re-recorded
    for (auto x : used) give(x);
    return PSD_OK;
}

psd_status_t psd_nccl_unique_id(char id[128]) {
    if (!id) return fail(PSD_EINVAL, "null id");
    if (!nccl().ok) return fail(PSD_ENCCL, "libnccl.so.2 not available");
    int r = nccl().get_unique_id(id);
    return r ? nccl_fail(r, "ncclGetUniqueId") : PSD_OK;
}

psd_status_t psd_nccl_comm_create(const char id[128], int nranks, int rank, void** comm) {
    if (!id || !comm) return fail(PSD_EINVAL, "null id or comm");
    if (!nccl().ok) return fail(PSD_ENCCL, "libnccl.so.2 not available");
    NcclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    int r = nccl().comm_init_rank(comm, nranks, uid, rank);
    return r ? nccl_fail(r, "ncclCommInitRank") : PSD_OK;
}

psd_status_t psd_nccl_comm_destroy(void* comm) {
    if (!comm) return PSD_OK;
    if (!nccl().ok) return fail(PSD_ENCCL, "libnccl.so.2 not available");
    int r = nccl().comm_destroy(comm);
    return r ? nccl_fail(r, "ncclCommDestroy") : PSD_OK;
}

psd_status_t psd_project_rowpanel(psd_filter_t h, const float* X_rows, int64_t n, int rank, int nranks,
                                  float* out_rows, int want_sign, void* comm, void* stream) {
    if (!comm) return fail(PSD_EINVAL, "null communicator");
    return run_rowpanel(h, X_rows, n, rank, nranks, out_rows, want_sign != 0, comm, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_project_rowpanel_virtual(psd_filter_t h, const float* X, int64_t n, int nranks, float* out,
                                          int want_sign, void* stream) {
    return run_rowpanel(h, X, n, 0, nranks, out, want_sign != 0, nullptr, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_rowpanel_p2p_region(psd_filter_t h, int64_t n, int nranks, int rank, char handle[64]) {
    if (!h || !handle) return fail(PSD_EINVAL, "null handle / IPC handle buffer");
    psd_status_t rc = peer_layout(h, static_cast<int>(n), nranks, rank, false);
    if (rc != PSD_OK) return rc;
    if ((rc = peer_alloc_local(h, rank)) != PSD_OK) return rc;
    cudaIpcMemHandle_t ih;
    cudaError_t e = cudaIpcGetMemHandle(&ih, h->pp.base[rank]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    std::memcpy(handle, &ih, 64);
    return PSD_OK;
}

psd_status_t psd_rowpanel_p2p_attach(psd_filter_t h, const char* handles) {
    if (!h || !handles) return fail(PSD_EINVAL, "null handle / handles");
    auto& pp = h->pp;
    if (pp.base.empty() || pp.is_virtual || !pp.base[pp.rank]) return fail(PSD_EINVAL, "psd_rowpanel_p2p_region first");
    if (pp.attached) return PSD_OK;
    for (int q = 0; q < pp.nranks; ++q) {
        if (q == pp.rank) continue;
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, handles + 64 * q, 64);
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
        pp.base[q] = static_cast<uint8_t*>(p);
        pp.ipc_opened[q] = 1;
    }
    return peer_finish(h);
}

psd_status_t psd_project_rowpanel_p2p(psd_filter_t h, const float* X_rows, int64_t n, int rank, int nranks,
                                      float* out_rows, int want_sign, void* stream) {
    if (!h || !X_rows || !out_rows) return fail(PSD_EINVAL, "null handle / X / out");
    if (h->pp.is_virtual || h->pp.n != n || h->pp.nranks != nranks || h->pp.rank != rank)
        return fail(PSD_EINVAL, "peer row panels: (n, nranks, rank) differ from psd_rowpanel_p2p_region");
    return run_rowpanel_p2p(h, X_rows, out_rows, want_sign != 0, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_project_rowpanel_p2p_virtual(psd_filter_t h, const float* X, int64_t n, int nranks, float* out,
                                              int want_sign, void* stream) {
    if (!h || !X || !out) return fail(PSD_EINVAL, "null handle / X / out");
    auto& pp = h->pp;
    if (!(pp.is_virtual && pp.attached && pp.n == n && pp.nranks == nranks && pp.op == op_of(h->prec))) {
        psd_status_t rc = peer_layout(h, static_cast<int>(n), nranks, 0, true);
        if (rc != PSD_OK) return rc;
        for (int q = 0; q < nranks; ++q)
            if ((rc = peer_alloc_local(h, q)) != PSD_OK) return rc;
        if ((rc = peer_finish(h)) != PSD_OK) return rc;
    }
    return run_rowpanel_p2p(h, X, out, want_sign != 0, static_cast<cudaStream_t>(stream));
}

psd_status_t psd_rowpanel_p2p_timeout(psd_filter_t h, double seconds) {
    if (!h) return fail(PSD_EINVAL, "null handle");
    if (!(seconds > 0.0) || !(seconds <= 3600.0)) return fail(PSD_EINVAL, "timeout must be in (0, 3600] s");
    const unsigned long long ns = static_cast<unsigned long long>(seconds * 1e9);
    h->peer_timeout_ns = ns;
    return PSD_OK;
}

void psd_rowpanel_p2p_release(psd_filter_t h) {
    if (h) free_peerpath(h);
}

int psd_rowpanel_tiles(int64_t n, int nranks, int rank, uint32_t* codes, int cap) {
    if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks) return -1;
    const int nt = static_cast<int>((n + 255) / 256);
    return rowpanel_tiles(nt, nranks, rank, codes, cap);
}

psd_status_t psd_sym_product(psd_filter_t h, const float* A, const float* B, const float* D, double alpha,
                             double beta, int64_t n64, int64_t batch64, float* C, void* stream) {
    psd_status_t rc = check_args(h, A, n64, batch64, C);
    if (rc != PSD_OK) return rc;
    if (!B) return fail(PSD_EINVAL, "null B");
    const int n = static_cast<int>(n64), batch = static_cast<int>(batch64);
    const int npad = static_cast<int>(padded_n(n, batch));
    rc = ensure_ws(h, npad, batch);
    if (rc != PSD_OK) return rc;
    Workspace& ws = h->ws;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool split = ws.split;
    cudaError_t e = launch_scale_convert(ws.op, A, n, npad, batch, nullptr, 1.0, ws.op_buf[B_XA],
                                         split ? ws.op_buf[B_XA + B_COUNT] : nullptr, 1.0, nullptr, 0.0, st);
    if (e == cudaSuccess)
        e = launch_scale_convert(ws.op, B, n, npad, batch, nullptr, 1.0, ws.op_buf[B_XB],
                                 split ? ws.op_buf[B_XB + B_COUNT] : nullptr, 1.0, nullptr, 0.0, st);
    if (e != cudaSuccess) return cuda_fail(e, "scale_convert");
    EpiParams ep{};
    ep.alpha = static_cast<float>(alpha);
    ep.beta = static_cast<float>(beta);
    ep.out_scale = 1.0f;
    if (D) {
        ep.Df = D;
        ep.ldDf = n;
        ep.strideDf = static_cast<int64_t>(n) * n;
        ep.nDf = n;
    }
    ep.outF = C;
    ep.ldF = n;
    ep.strideF = static_cast<int64_t>(n) * n;
    ep.nF = n;
    if (debug_env("PSD_DEBUG_STAMPS")) ep.dbg = reinterpret_cast<unsigned long long*>(ws.partial);  // debug only
    e = cudaMemsetAsync(ws.counters, 0, sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "counter reset");
    GemmShape shape{npad, batch, ws.tiles, ws.tiles_per_matrix, ws.counters};
    shape.kchunk = product_kchunk(h, split, n, npad, batch);
    const bool bn64 = !(npad % 256 == 0 && use_pair_kernel(n, batch)) && sym_gemm_bn(npad, batch) == 64;
    const CUtensorMap* bmaps = bn64 ? ws.tmap64 : ws.tmap;
    OperandMaps m;
    m.a = ws.tmap[B_XA];
    m.b = bmaps[B_XB];
    m.a_lo = ws.tmap[split ? B_XA + B_COUNT : B_XA];
    m.b_lo = bmaps[split ? B_XB + B_COUNT : B_XB];
    const bool pair = npad % 256 == 0 && use_pair_kernel(n, batch);
    if (ep.dbg && pair) cudaMemsetAsync(ep.dbg, 0, 64, st);
    e = pair ? launch_sym_gemm_2cta(ws.op, split, m, shape, ep, st) : launch_sym_gemm(ws.op, split, m, shape, ep, st);
    if (e != cudaSuccess) return cuda_fail(e, "sym_gemm");
    h->kernel_launches += 3;
    if (ep.dbg && pair) {    // debug: summed over the leader MMA threads / epilogue warp 4 of every CTA
        unsigned long long t[7] = {};
        cudaStreamSynchronize(st);
        cudaMemcpy(t, ep.dbg, sizeof(t), cudaMemcpyDeviceToHost);
        const double tiles = t[4] ? double(t[4]) : 1.0;
        std::fprintf(stderr, "psd pair stamps n=%d (cycles per tile, %llu tiles): mma-loop %.0f = tile-id wait %.0f + "
                     "accumulator wait %.0f + operand wait %.0f + issue; epilogue: acc wait %.0f, work %.0f\n",
                     n, t[4], t[3] / tiles, t[0] / tiles, t[1] / tiles, t[2] / tiles, t[5] / (2 * tiles), t[6] / (2 * tiles));
    } else if (ep.dbg) {            // debug: print the kernel phase stamps (ns since the first)
        unsigned long long t[6] = {};
        cudaStreamSynchronize(st);
        cudaMemcpy(t, ep.dbg, sizeof(t), cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "psd stamps n=%d: prologue %.2f us, dep-wait %.2f us, mainloop %.2f us, epilogue %.2f us, teardown %.2f us\n",
                     n, (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
                     (t[5] - t[4]) * 1e-3);
    }
    return PSD_OK;
}

}  // extern "C"
