// Host side of libtnrd.so: the C ABI declared in include/tnrd.h.
//
// Owns the per-stage parameter store, scratch buffers, the stage loop
// (P Eq.13 iterated T times from u_0 = f), the
// row-slab path with its per-stage halo exchange (NCCL P2P or a single-device
// loopback), and per-launch CUDA-event instrumentation.  Every step of the
// computation runs in the sm_100a kernels of tnrd_kernels.cu.
#include "tnrd.h"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nccl.h"
#include "tnrd_internal.h"

using tnrd::StageArgs;

namespace {

thread_local std::string g_last_error;

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool loaded = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    const char *env = getenv("TNRD_NCCL_LIB");
    void *lib = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
        api.why = std::string("cannot dlopen NCCL: ") + dlerror();
        return api;
    }
#define TNRD_SYM(field, name)                                                   \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(lib, name));        \
    if (!api.field) { api.why = std::string("missing NCCL symbol ") + name; return api; }
    TNRD_SYM(GetUniqueId, "ncclGetUniqueId");
    TNRD_SYM(CommInitRank, "ncclCommInitRank");
    TNRD_SYM(CommDestroy, "ncclCommDestroy");
    TNRD_SYM(Send, "ncclSend");
    TNRD_SYM(Recv, "ncclRecv");
    TNRD_SYM(GroupStart, "ncclGroupStart");
    TNRD_SYM(GroupEnd, "ncclGroupEnd");
    TNRD_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    TNRD_SYM(CommAbort, "ncclCommAbort");
    TNRD_SYM(GetErrorString, "ncclGetErrorString");
#undef TNRD_SYM
    api.loaded = true;
    return api;
}

}  // namespace

struct tnrd_handle {
    tnrd_desc d{};
    int num_sms = 148;
    size_t total_mem = 0;          // device memory (bytes), queried once at create
    bool allow_large_tile = true;  // the 2x64x64 tile pair fits in shared memory
    int pstride_max = 0;
    std::vector<int> pstride;     // per stage
    std::vector<int> mode;        // per stage
    std::vector<float> lambda;    // per stage
    std::vector<char> is_set;     // per stage
    float *d_params = nullptr;    // [T][Nk][pstride_max]
    float4 *d_table = nullptr;    // MODE_TABLE: [T][Nk][table_stride] cubic intervals
    int table_stride = 0;
    // tensor-core engine (tnrd_tc.cu): per stage operand block [T][tc_stride]
    float *d_tc = nullptr;
    int tc_stride = 0;
    std::vector<char> tc_ok;      // per stage: block packed (Horner phi)
    int engine = TNRD_ENGINE_AUTO;
    int grad_max_f = 0;           // tnrd_set_grad_chunk: cap on filters per backward chunk (0 = auto)
    // raw stage parameters (training gradient, tnrd_loss_grad)
    std::vector<float> raw_mu0, raw_step, raw_gamma;   // host [T][Nk]
    float *d_raw = nullptr;       // device: k [T][Nk][m*m], kbar [T][Nk][m*m], w [T][Nk][M]
    float *g_buf = nullptr;       // tape + work images
    size_t g_buf_bytes = 0;
    float *g_partial = nullptr;   // per-block partial sums
    size_t g_partial_bytes = 0;
    double *g_red = nullptr;      // reduced sums
    size_t g_red_bytes = 0;
    float *scratch = nullptr;
    size_t scratch_bytes = 0;
    float *e2e_f = nullptr, *e2e_u = nullptr;
    size_t e2e_f_bytes = 0, e2e_u_bytes = 0;   // one capacity per buffer (grow() may free one)
    float *slab_buf[2] = {nullptr, nullptr};
    size_t slab_bytes[2] = {0, 0};
    std::vector<float *> lb_bufs;  // loopback slab buffers
    size_t lb_bytes = 0;
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    unsigned long long launches = 0;
    bool profile = false;
    std::vector<cudaEvent_t> ev;   // pairs (start, stop) per profiled launch
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;   // tnrd_denoise_host copy streams
    std::vector<cudaEvent_t> chunk_ev;               // 2 per pipelined chunk
    int ev_used = 0;
    // CUDA graphs of the T-stage loop (tnrd_denoise), keyed by every launch argument;
    // captured on a private stream, replayed on the caller's
    struct Graph {
        const float *f, *u, *scratch;
        int B, H, W, tc_oh, tile, profile;
        long long ld;
        cudaGraph_t graph = nullptr;             // kept: its nodes address the exec's event records
        cudaGraphExec_t exec = nullptr;
        std::vector<cudaGraphNode_t> ev_nodes;   // profiling: event-record nodes in launch order
        unsigned long long used = 0;
    };
    std::vector<Graph> graphs;
    unsigned long long graph_clock = 0;
    cudaStream_t s_cap = nullptr;
    int use_graphs = -1;          // -1: from TNRD_GRAPH (default on)
    std::string err;
};

namespace {

void drop_graphs(tnrd_handle *h);

tnrd_status fail(tnrd_handle *h, tnrd_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) h->err = buf;
    g_last_error = buf;
    return s;
}

tnrd_status cuda_fail(tnrd_handle *h, cudaError_t e, const char *what) {
    return fail(h, TNRD_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define TNRD_CUDA(h, call)                                          \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail((h), e_, #call);   \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

tnrd_status grow(tnrd_handle *h, float **p, size_t *have, size_t need, const char *what) {
    if (*have >= need) return TNRD_OK;
    if (*p) {
        cudaDeviceSynchronize();
        cudaFree(*p);
        *p = nullptr;
        *have = 0;
    }
    cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();   // a failed cudaMalloc is not sticky; do not leave it for later checks
        return fail(h, TNRD_ENOMEM, "cudaMalloc(%zu) for %s: %s", need, what, cudaGetErrorString(e));
    }
    *have = need;
    return TNRD_OK;
}

tnrd_status check_ready(tnrd_handle *h) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    for (int t = 0; t < h->d.T; ++t)
        if (!h->is_set[t]) return fail(h, TNRD_ESTATE, "stage %d parameters are not set", t);
    return TNRD_OK;
}

// Launch plan: engine and tile configuration.
struct Plan {
    int tile = 1;    // FP32 engine: 0 = "L" (tile pairs of 64x64), 1 = "S"
    int tc_oh = 0;   // > 0: tensor-core engine with tiles of tc_oh output rows
};

// The tensor-core engine can run every stage of this handle: a built (ksize, N_k)
// instantiation and Horner-unit or tabulated phi in every stage (R1 or R2).
bool tc_ready(const tnrd_handle *h) {
    if (!h->d_tc) return false;
    for (int t = 0; t < h->d.T; ++t)
        if (!h->tc_ok[t]) return false;
    return true;
}

// Engine: tnrd_set_engine (TNRD_ENGINE=fp32|tc in the environment overrides it
// for tests; TNRD_TC_ROWS=n forces the tensor engine's tile height); AUTO takes
// the tensor-core engine when it can run.  FP32 tile: "L"
// when there are enough tiles to fill the GPU, else "S"; TNRD_FORCE_TILE=L|S
// overrides (tests run every code path on small, fully oracle-checkable images).
// Results do not depend on the tile choice (per-pixel arithmetic is tiling-free).
Plan plan_for(const tnrd_handle *h, int B, int H, int W, bool allow_tc) {
    Plan p;
    static const char *env_engine = getenv("TNRD_ENGINE");
    int engine = h->engine;
    if (env_engine && env_engine[0] == 'f') engine = TNRD_ENGINE_FP32;
    if (env_engine && env_engine[0] == 't') engine = TNRD_ENGINE_TENSOR;
    if (allow_tc && engine != TNRD_ENGINE_FP32 && tc_ready(h)) {
        p.tc_oh = tnrd::tc_choose_rows(h->d.ksize, B, H, W, h->num_sms);
        static const char *rows = getenv("TNRD_TC_ROWS");  // tests: force the tile height
        if (rows && atoi(rows) >= 2 && atoi(rows) % 2 == 0) p.tc_oh = atoi(rows);
        return p;
    }
    static const char *force = getenv("TNRD_FORCE_TILE");
    if (force && (force[0] == 'L' || force[0] == 'l') && h->allow_large_tile) { p.tile = 0; return p; }
    if (force && (force[0] == 'S' || force[0] == 's')) { p.tile = 1; return p; }
    p.tile = h->allow_large_tile ? tnrd::choose_tile(h->d.ksize, B, H, W, h->num_sms) : 1;
    return p;
}

tnrd_status launch_one(tnrd_handle *h, int t, const Plan &plan, StageArgs &a, int B, cudaStream_t s) {
    a.params = h->d_params + (size_t)t * h->d.n_filters * h->pstride_max;
    a.Nk = h->d.n_filters;
    a.pstride = h->pstride[t];
    a.mode = h->mode[t];
    if (plan.tc_oh > 0) {
        a.params = h->d_tc + (size_t)t * h->tc_stride;
        a.pstride = tnrd::tc_pair_stride(h->d.n_rbf);
        a.tc_par_floats = h->tc_stride;
        a.tc_oh = plan.tc_oh;
    }
    a.table = h->d_table ? h->d_table + (size_t)t * h->d.n_filters * h->table_stride : nullptr;
    a.table_stride = h->table_stride;
    a.boundary = h->d.boundary;
    a.reaction = h->d.reaction;
    a.lambda = h->lambda[t];
    unsigned ev_flags = cudaEventRecordDefault;
    if (h->profile) {
        if ((size_t)h->ev_used + 2 > h->ev.size()) {
            for (int k = 0; k < 64; ++k) {
                cudaEvent_t e;
                TNRD_CUDA(h, cudaEventCreate(&e));
                h->ev.push_back(e);
            }
        }
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        TNRD_CUDA(h, cudaStreamIsCapturing(s, &cs));
        // captured: event-record nodes (run_graph swaps their events per replay)
        ev_flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
        TNRD_CUDA(h, cudaEventRecordWithFlags(h->ev[h->ev_used], s, ev_flags));
    }
    cudaError_t e = plan.tc_oh > 0 ? tnrd::launch_stage_tc(h->d.ksize, a, B, s)
                                   : tnrd::launch_stage(h->d.ksize, plan.tile, a, B, s);
    if (e != cudaSuccess) return cuda_fail(h, e, "stage kernel launch");
    if (h->profile) {
        TNRD_CUDA(h, cudaEventRecordWithFlags(h->ev[h->ev_used + 1], s, ev_flags));
        h->ev_used += 2;
    }
    h->launches++;
    return TNRD_OK;
}

// ---------------------------------------------------------------- slab machinery
// A slab buffer holds rows [row0 - halo, row0 + rows + halo) of u (dense, ld = W).
struct SlabExchange {
    virtual ~SlabExchange() = default;
    // Fill the top/bottom halo rows of slab `k`'s buffer `buf` for the coming stage.
    virtual tnrd_status exchange(int k, float *buf) = 0;
};

tnrd_status run_slab(tnrd_handle *h, const float *f_slab, long long f_ld, float *u_slab, long long u_ld,
                     int H, int W, int row0, int rows, float *buf0, float *buf1, SlabExchange &ex,
                     int k, int stage, cudaStream_t s) {
    // executes stage `stage` for slab k (stage 0 seeds the buffer with f first)
    const int halo = h->d.ksize - 1;
    float *in = (stage % 2 == 0) ? buf0 : buf1;
    float *out_buf = (stage % 2 == 0) ? buf1 : buf0;
    (void)in;
    StageArgs a{};
    a.u_in = {in, W, 0, row0 - halo};
    a.f = {f_slab, f_ld, 0, row0};
    const bool last = stage == h->d.T - 1;
    if (last) {
        a.u_out = u_slab; a.out_ld = u_ld; a.out_img_stride = 0; a.out_row_base = row0;
    } else {
        a.u_out = out_buf; a.out_ld = W; a.out_img_stride = 0; a.out_row_base = row0 - halo;
    }
    a.H = H; a.W = W;
    a.y_begin = row0; a.y_end = row0 + rows;
    a.avail_lo = row0 - halo < 0 ? 0 : row0 - halo;
    a.avail_hi = row0 + rows + halo > H ? H : row0 + rows + halo;
    const Plan plan = plan_for(h, 1, rows, W, true);
    (void)ex; (void)k;
    return launch_one(h, stage, plan, a, 1, s);
}

// Non-blocking poll of the communicator's asynchronous error (a failed or vanished
// peer, a NCCL-internal error): on error the communicator is aborted, so enqueued
// NCCL kernels return instead of waiting forever, and the handle reports ENCCL.
tnrd_status comm_async_check(tnrd_handle *h) {
    if (!h->comm) return TNRD_OK;
    NcclApi &api = nccl();
    ncclResult_t ae = ncclSuccess;
    const ncclResult_t r = api.CommGetAsyncError(h->comm, &ae);
    if (r == ncclSuccess && (ae == ncclSuccess || ae == ncclInProgress)) return TNRD_OK;
    const ncclResult_t bad = r != ncclSuccess ? r : ae;
    api.CommAbort(h->comm);
    h->comm = nullptr;
    return fail(h, TNRD_ENCCL, "NCCL asynchronous error (communicator aborted): %s", api.GetErrorString(bad));
}

struct NcclExchange : SlabExchange {
    tnrd_handle *h; int rows, W; cudaStream_t s;
    NcclExchange(tnrd_handle *h_, int rows_, int W_, cudaStream_t s_) : h(h_), rows(rows_), W(W_), s(s_) {}
    tnrd_status exchange(int, float *buf) override {
        NcclApi &api = nccl();
        const int halo = h->d.ksize - 1;
        const size_t n = (size_t)halo * W;
        ncclResult_t r = api.GroupStart();
        if (r == ncclSuccess && h->rank > 0) {
            r = api.Send(buf + (size_t)halo * W, n, ncclFloat32, h->rank - 1, h->comm, s);
            if (r == ncclSuccess) r = api.Recv(buf, n, ncclFloat32, h->rank - 1, h->comm, s);
        }
        if (r == ncclSuccess && h->rank < h->nranks - 1) {
            r = api.Send(buf + (size_t)rows * W, n, ncclFloat32, h->rank + 1, h->comm, s);
            if (r == ncclSuccess) r = api.Recv(buf + (size_t)(halo + rows) * W, n, ncclFloat32, h->rank + 1,
                                               h->comm, s);
        }
        ncclResult_t r2 = api.GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(h, TNRD_ENCCL, "halo exchange: %s", api.GetErrorString(r != ncclSuccess ? r : r2));
        return comm_async_check(h);   // a peer's failure surfaces here (non-blocking poll)
    }
};

// MODE_TABLE geometry and construction (tnrd_internal.h).
int table_intervals(int M) { return (M - 1 + 2 * tnrd::kTabPad) * tnrd::kTabPerCentre; }

// Cubic Hermite intervals of phi(x) = sum_j w_j exp(-rho^2 (x - j)^2 / 2) in centre
// units (the same function as P l.145 / S l.107 with x = (z - mu0)/step), from the
// exact values and slopes at the nodes, in double; out[n_int] = 0 (out of range).
void build_table(const float *w, int M, double rho, float4 *out) {
    const int S = tnrd::kTabPerCentre, n = table_intervals(M);
    const double h = 1.0 / S, x_lo = -tnrd::kTabPad;
    std::vector<double> f(n + 1), df(n + 1);
    for (int k = 0; k <= n; ++k) {
        const double x = x_lo + k * h;
        double s0 = 0.0, s1 = 0.0;
        for (int j = 0; j < M; ++j) {
            const double d = x - j, g = std::exp(-rho * rho * d * d / 2.0);
            s0 += w[j] * g;
            s1 += -w[j] * rho * rho * d * g;
        }
        f[k] = s0;
        df[k] = s1 * h;  // slope per interval length
    }
    for (int k = 0; k < n; ++k) {
        const double p0 = f[k], p1 = f[k + 1], m0 = df[k], m1 = df[k + 1];
        out[k] = make_float4((float)p0, (float)m0, (float)(3.0 * (p1 - p0) - 2.0 * m0 - m1),
                             (float)(2.0 * (p0 - p1) + m0 + m1));
    }
    out[n] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Horner units: R's exponent bound yrmax with sum|c| * 2^(7 yrmax) <= 2^126, so
// that R^7 (times the largest coefficient sum) stays finite (tnrd_internal.h).
double horner_yrmax(double sum_abs_c) {
    const double l2 = std::log2(std::max(sum_abs_c, 1e-30));
    return std::min(120.0, (126.0 - std::max(l2, -30.0)) / 7.0);
}
// ... and the Horner form is used only where the clamp t <= yrmax / (2 sg) binds
// exclusively on terms below 2^-20 of their weight: t_clamp >= 7 sg + 4.5.
bool horner_ok(double sg, double yrmax) { return yrmax / (2.0 * sg) >= 7.0 * sg + 4.5; }

// Host-side evaluation constants of one stage (layout in tnrd_internal.h),
// computed in double and rounded once to fp32.
void pack_stage(const tnrd_desc &d, const float *filters, const float *w, const float *mu0,
                const float *step, const float *gamma, int mode, int pstride, float *out) {
    const int K = d.ksize, M = d.n_rbf, K8 = tnrd::tap_pitch(K);
    const double sg_per_rho = std::sqrt(1.0 / (2.0 * std::log(2.0)));  // sqrt(log2(e)/2)
    for (int i = 0; i < d.n_filters; ++i) {
        float *p = out + (size_t)i * pstride;
        std::memset(p, 0, sizeof(float) * pstride);
        for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) p[a * K8 + b] = filters[(size_t)i * K * K + a * K + b];
        const double st = step[i], ga = gamma[i], m0 = mu0[i];
        const double rho = st / ga, sg = rho * sg_per_rho;
        const double a_s = sg / st, x_off = -m0 / st;
        float *fc = p + tnrd::tap_floats(K);
        float *units = fc + tnrd::kFc;
        const float *wi = w + (size_t)i * M;
        if (mode == tnrd::MODE_HORNER) {
            const int NB = (M + 7) / 8;
            double smax = 0.0;
            for (int b = 0; b < NB; ++b) {
                float *u = units + b * tnrd::kHornerUnit;
                u[0] = (float)(sg * (x_off - 8.0 * b));   // t of the block's first centre
                double s = 0.0;
                for (int e = 0; e < 8; ++e) {
                    const int j = 8 * b + e;
                    const double coef = j < M ? wi[j] * std::exp(-rho * rho * e * e / 2.0) : 0.0;
                    u[1 + e] = (float)coef;   // u[1..8] = c_0 .. c_7
                    s += std::fabs(coef);
                }
                smax = std::max(smax, s);
            }
            fc[0] = (float)a_s; fc[1] = (float)(2.0 * sg); fc[2] = (float)(1.0 / (8.0 * sg)); fc[3] = (float)NB;
            fc[4] = (float)horner_yrmax(smax);
            fc[5] = horner_ok(sg, horner_yrmax(smax)) ? 1.f : 0.f;   // host-side check only
        } else if (mode == tnrd::MODE_TABLE) {
            const double S = tnrd::kTabPerCentre, x_lo = -tnrd::kTabPad;
            const double b = -(m0 / st + x_lo) * S;
            fc[0] = (float)(S / st);
            fc[1] = (float)b;                       // hi word of the offset
            fc[2] = (float)table_intervals(M);
            fc[3] = (float)(b - (double)fc[1]);     // lo word: the rounding of fc[1]
        } else {
            fc[0] = (float)a_s; fc[1] = (float)(2.0 * sg); fc[2] = (float)(1.0 / sg); fc[3] = (float)M;
            for (int j = 0; j < M; ++j) {
                units[j * tnrd::kDirectUnit] = (float)(sg * (x_off - j));
                units[j * tnrd::kDirectUnit + 1] = wi[j];
            }
        }
    }
}

int pstride_for(const tnrd_desc &d, int mode) {
    const int M = d.n_rbf;
    const int units = mode == tnrd::MODE_HORNER ? ((M + 7) / 8) * tnrd::kHornerUnit
                      : mode == tnrd::MODE_TABLE ? 0 : M * tnrd::kDirectUnit;
    return (tnrd::tap_floats(d.ksize) + tnrd::kFc + units + 3) / 4 * 4;
}

// Tensor-core operand block of one stage (tnrd_internal.h): taps split as
// hi = tf32(x), lo = tf32(x - hi) (round to nearest) in the UMMA K-major layout,
// for the forward bank [Nk x KTP] and transposed for the adjoint bank [NZ x Nk],
// then the Horner phi constants of `phi_host` (pack_stage layout, stride ps) with a
// zero unit appended per filter.
float tf32_rn_host(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b = (b + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &b, 4);
    return r;
}

void pack_tc_stage(const tnrd_desc &d, const float *filters, const float *phi_host, int ps, int mode, float *out) {
    const int K = d.ksize, Nk = d.n_filters, M = d.n_rbf, KT = K * K;
    const int KTP = tnrd::tc_ktp(K), NZ = tnrd::tc_nz(K), PPS = tnrd::tc_pair_stride(M), NB = (M + 7) / 8;
    std::memset(out, 0, sizeof(float) * tnrd::tc_par_floats(K, Nk, M));
    float *bf_hi = out, *bf_lo = out + (size_t)Nk * KTP;
    float *ba_hi = out + 2 * (size_t)Nk * KTP, *ba_lo = ba_hi + (size_t)NZ * Nk;
    float *phi = ba_lo + (size_t)NZ * Nk;
    for (int n = 0; n < Nk; ++n)
        for (int t = 0; t < KT; ++t) {
            const float x = filters[(size_t)n * KT + t];
            const float hi = tf32_rn_host(x), lo = tf32_rn_host(x - hi);
            bf_hi[tnrd::tc_b_index(n, t, KTP)] = hi;   // forward-GEMM column t (taps row-major)
            bf_lo[tnrd::tc_b_index(n, t, KTP)] = lo;
            ba_hi[tnrd::tc_b_index(t, n, Nk)] = hi;
            ba_lo[tnrd::tc_b_index(t, n, Nk)] = lo;
        }
    if (mode == tnrd::MODE_TABLE) {  // tabulated phi: {a_t, b_t, n_int, b_lo} per filter
        for (int n = 0; n < Nk; ++n)
            std::memcpy(phi + 4 * (size_t)n, phi_host + (size_t)n * ps + tnrd::tap_floats(K), sizeof(float) * 4);
        return;
    }
    // phi of filter pairs, interleaved (tnrd_internal.h); units NB..2NB-1 stay 0.
    // Warp unit range (FP32 engine, phi_x2): u0 = ceil((a_s vmin + ct0 - kWindow) / (8 sg)),
    // u1 = floor((a_s vmax + ct0 + kCutT + 0.01) / (8 sg)), folded into one fma each;
    // the fp32 rounding of the folded constants (~1e-6 units) is far inside the
    // margins of kWindow (0.025 in t) and of the cut (0.0099 in t).
    for (int p = 0; p < Nk / 2; ++p) {
        float *q = phi + (size_t)p * PPS;
        for (int h = 0; h < 2; ++h) {
            const float *fc = phi_host + (size_t)(2 * p + h) * ps + tnrd::tap_floats(K);
            const float *units = fc + tnrd::kFc;
            const double inv = fc[2], a_s = fc[0], ct0 = units[0];
            q[0 + h] = fc[0];                                   // a_s
            q[2 + h] = fc[1];                                   // two_sg
            q[4 + h] = (float)(a_s * inv);                      // A
            q[6 + h] = (float)((ct0 - (double)tnrd::kWindow) * inv);       // B0
            q[8 + h] = (float)((ct0 + (double)tnrd::kCutT + 0.01) * inv);  // B1
            q[10 + h] = fc[4];                                  // yrmax
            int nbi = NB;                                       // NB as int bits
            std::memcpy(&q[12], &nbi, 4);
            for (int b = 0; b < NB; ++b)
                for (int e = 0; e < 9; ++e)  // ct, c0..c7
                    q[tnrd::kTcPairHdr + b * tnrd::kTcPairUnit + 2 * e + h] = units[b * tnrd::kHornerUnit + e];
        }
    }
}

}  // namespace

namespace {
// The T stage launches of one tnrd_denoise call as a CUDA graph: captured once per
// argument set on the handle's private stream (relaxed mode: the launchers query
// attributes), replayed on the caller's stream.  Stage parameters, engine and
// buffers are part of the key or invalidate the cache (tnrd_set_stage_params,
// tnrd_set_engine).  With profiling on, the per-launch events are event-record nodes
// whose events are swapped for fresh ones before every replay.
template <class F>
tnrd_status run_graph(tnrd_handle *h, const float *f, const float *u, int B, int H, int W, long long ld,
                      const Plan &plan, cudaStream_t s, const F &stages) {
    using G = tnrd_handle::Graph;
    const int prof = h->profile ? 1 : 0;
    G *g = nullptr;
    for (G &c : h->graphs)
        if (c.f == f && c.u == u && c.scratch == h->scratch && c.B == B && c.H == H && c.W == W && c.ld == ld &&
            c.tc_oh == plan.tc_oh && c.tile == plan.tile && c.profile == prof) { g = &c; break; }
    const int T = h->d.T;
    if (!g) {
        if (!h->s_cap) TNRD_CUDA(h, cudaStreamCreateWithFlags(&h->s_cap, cudaStreamNonBlocking));
        const int ev0 = h->ev_used;
        const unsigned long long l0 = h->launches;
        TNRD_CUDA(h, cudaStreamBeginCapture(h->s_cap, cudaStreamCaptureModeRelaxed));
        tnrd_status st = stages(h->s_cap);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(h->s_cap, &graph);
        h->launches = l0;
        if (st != TNRD_OK) { if (graph) cudaGraphDestroy(graph); return st; }
        if (ce != cudaSuccess) return cuda_fail(h, ce, "graph capture");
        G ng;
        ng.f = f; ng.u = u; ng.scratch = h->scratch; ng.B = B; ng.H = H; ng.W = W; ng.ld = ld;
        ng.tc_oh = plan.tc_oh; ng.tile = plan.tile; ng.profile = prof;
        if (prof) {   // event-record nodes in the order of the events they record
            size_t n = 0;
            cudaGraphGetNodes(graph, nullptr, &n);
            std::vector<cudaGraphNode_t> nodes(n);
            cudaGraphGetNodes(graph, nodes.data(), &n);
            ng.ev_nodes.assign(2 * (size_t)T, nullptr);
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType ty;
                cudaGraphNodeGetType(nd, &ty);
                if (ty != cudaGraphNodeTypeEventRecord) continue;
                cudaEvent_t e;
                cudaGraphEventRecordNodeGetEvent(nd, &e);
                for (int j = 0; j < 2 * T; ++j)
                    if (h->ev[ev0 + j] == e) ng.ev_nodes[j] = nd;
            }
            h->ev_used = ev0;
        }
        const cudaError_t ie = cudaGraphInstantiate(&ng.exec, graph, 0);
        if (ie != cudaSuccess) { cudaGraphDestroy(graph); return cuda_fail(h, ie, "graph instantiate"); }
        ng.graph = graph;
        if (h->graphs.size() >= 16) {   // evict the least recently used
            size_t lru = 0;
            for (size_t k = 1; k < h->graphs.size(); ++k)
                if (h->graphs[k].used < h->graphs[lru].used) lru = k;
            cudaGraphExecDestroy(h->graphs[lru].exec);
            cudaGraphDestroy(h->graphs[lru].graph);
            h->graphs.erase(h->graphs.begin() + (long)lru);
        }
        h->graphs.push_back(std::move(ng));
        g = &h->graphs.back();
    }
    g->used = ++h->graph_clock;
    if (prof) {
        while ((size_t)h->ev_used + 2 * T > h->ev.size()) {
            cudaEvent_t e;
            TNRD_CUDA(h, cudaEventCreate(&e));
            h->ev.push_back(e);
        }
        for (int j = 0; j < 2 * T; ++j)
            if (g->ev_nodes[j]) TNRD_CUDA(h, cudaGraphExecEventRecordNodeSetEvent(g->exec, g->ev_nodes[j], h->ev[h->ev_used + j]));
        h->ev_used += 2 * T;
    }
    TNRD_CUDA(h, cudaGraphLaunch(g->exec, s));
    h->launches += T;
    return TNRD_OK;
}

void drop_graphs(tnrd_handle *h) {
    for (auto &c : h->graphs) {
        cudaGraphExecDestroy(c.exec);
        cudaGraphDestroy(c.graph);
    }
    h->graphs.clear();
}
}  // namespace

extern "C" {

int tnrd_abi_version(void) { return TNRD_ABI_VERSION; }

const char *tnrd_status_string(tnrd_status s) {
    switch (s) {
        case TNRD_OK: return "TNRD_OK";
        case TNRD_EINVAL: return "TNRD_EINVAL";
        case TNRD_ESTATE: return "TNRD_ESTATE";
        case TNRD_ENOMEM: return "TNRD_ENOMEM";
        case TNRD_ECUDA: return "TNRD_ECUDA";
        case TNRD_ENCCL: return "TNRD_ENCCL";
        case TNRD_EUNSUPPORTED: return "TNRD_EUNSUPPORTED";
    }
    return "TNRD_UNKNOWN";
}

tnrd_status tnrd_create(const tnrd_desc *d, tnrd_handle **out) {
    if (!d || !out) return fail(nullptr, TNRD_EINVAL, "null argument");
    *out = nullptr;
    if (d->T < 1 || d->n_filters < 1 || d->n_rbf < 1 || d->n_rbf > 256)
        return fail(nullptr, TNRD_EINVAL, "need T >= 1, n_filters >= 1, 1 <= n_rbf <= 256");
    if (d->ksize < 3 || d->ksize % 2 == 0)
        return fail(nullptr, TNRD_EINVAL, "ksize must be odd and >= 3 (got %d)", d->ksize);
    if (d->ksize > 11) return fail(nullptr, TNRD_EUNSUPPORTED, "ksize %d not built (3, 5, 7, 9, 11)", d->ksize);
    if (d->boundary != 0 && d->boundary != 1) return fail(nullptr, TNRD_EINVAL, "bad boundary %d", d->boundary);
    if (d->phi_mode != TNRD_PHI_EXACT && d->phi_mode != TNRD_PHI_TABLE)
        return fail(nullptr, TNRD_EINVAL, "bad phi_mode %d", d->phi_mode);
    if (d->reaction < TNRD_REACTION_POISSON_PROX || d->reaction > TNRD_REACTION_POISSON_GRADIENT)
        return fail(nullptr, TNRD_EINVAL, "bad reaction %d", d->reaction);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    if (d->device < 0 || d->device >= ndev) return fail(nullptr, TNRD_EINVAL, "device %d of %d", d->device, ndev);
    DeviceGuard g(d->device);
    tnrd_handle *h = new tnrd_handle();
    h->d = *d;
    // on a failed allocation: free what exists (cudaFree(nullptr) is a no-op)
    const auto release = [](tnrd_handle *hh) {
        cudaFree(hh->d_params);
        cudaFree(hh->d_raw);
        cudaFree(hh->d_tc);
        cudaFree(hh->d_table);
        delete hh;
    };
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, d->device);
    {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) h->total_mem = total_b;
    }
    h->pstride_max = std::max(pstride_for(*d, tnrd::MODE_HORNER), pstride_for(*d, tnrd::MODE_DIRECT));
    h->pstride.assign(d->T, 0);
    h->mode.assign(d->T, 0);
    h->lambda.assign(d->T, 0.f);
    h->is_set.assign(d->T, 0);
    // shared-memory budget of the largest-stride stage on the small tile
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d->device);
    const size_t need_s = tnrd::stage_smem_bytes(d->ksize, 1, d->n_filters, h->pstride_max);
    if ((long long)need_s > smem_optin) {
        release(h);
        return fail(nullptr, TNRD_EUNSUPPORTED, "model needs %zu B shared memory (> %d)", need_s, smem_optin);
    }
    h->allow_large_tile = (long long)tnrd::stage_smem_bytes(d->ksize, 0, d->n_filters, h->pstride_max) <= smem_optin;
    const size_t bytes = sizeof(float) * (size_t)d->T * d->n_filters * h->pstride_max;
    e = cudaMalloc(&h->d_params, bytes);
    if (e != cudaSuccess) {
        release(h);
        return fail(nullptr, TNRD_ENOMEM, "cudaMalloc params: %s", cudaGetErrorString(e));
    }
    {
        const size_t mm = (size_t)d->ksize * d->ksize;
        e = cudaMalloc(&h->d_raw, sizeof(float) * (size_t)d->T * d->n_filters * (2 * mm + d->n_rbf + 3));
        if (e != cudaSuccess) {
            release(h);
            return fail(nullptr, TNRD_ENOMEM, "cudaMalloc raw params: %s", cudaGetErrorString(e));
        }
        h->raw_mu0.assign((size_t)d->T * d->n_filters, 0.f);
        h->raw_step = h->raw_mu0;
        h->raw_gamma = h->raw_mu0;
    }
    h->tc_ok.assign(d->T, 0);
    // tensor engine: a built (ksize, N_k) whose operands fit in shared memory with the
    // smallest tile (large M raises the phi constants: FP32 engine then)
    if (tnrd::tc_supported(d->ksize, d->n_filters) &&
        (long long)tnrd::tc_min_smem_bytes(d->ksize, d->n_filters,
                                           tnrd::tc_par_floats(d->ksize, d->n_filters, d->n_rbf)) <= smem_optin) {
        h->tc_stride = tnrd::tc_par_floats(d->ksize, d->n_filters, d->n_rbf);
        e = cudaMalloc(&h->d_tc, sizeof(float) * (size_t)d->T * h->tc_stride);
        if (e != cudaSuccess) {
            release(h);
            return fail(nullptr, TNRD_ENOMEM, "cudaMalloc tensor-core operands: %s", cudaGetErrorString(e));
        }
    }
    if (d->phi_mode == TNRD_PHI_TABLE) {
        h->table_stride = table_intervals(d->n_rbf) + 1;
        e = cudaMalloc(&h->d_table, sizeof(float4) * (size_t)d->T * d->n_filters * h->table_stride);
        if (e != cudaSuccess) {
            release(h);
            return fail(nullptr, TNRD_ENOMEM, "cudaMalloc phi tables: %s", cudaGetErrorString(e));
        }
    }
    *out = h;
    return TNRD_OK;
}

tnrd_status tnrd_set_stage_params(tnrd_handle *h, int t, const float *filters, const float *rbf_w,
                                  const float *rbf_mu0, const float *rbf_step, const float *rbf_gamma,
                                  float lambda) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    if (t < 0 || t >= h->d.T) return fail(h, TNRD_EINVAL, "stage %d out of [0, %d)", t, h->d.T);
    if (!filters || !rbf_w || !rbf_mu0 || !rbf_step || !rbf_gamma) return fail(h, TNRD_EINVAL, "null array");
    if (!std::isfinite(lambda) || lambda <= 0.f) return fail(h, TNRD_EINVAL, "lambda must be finite and > 0");
    const int Nk = h->d.n_filters, K = h->d.ksize, M = h->d.n_rbf;
    double rho_max = 0.0;
    for (int i = 0; i < Nk; ++i) {
        if (!std::isfinite(rbf_mu0[i]) || !std::isfinite(rbf_step[i]) || !std::isfinite(rbf_gamma[i]))
            return fail(h, TNRD_EINVAL, "non-finite RBF grid (filter %d)", i);
        if (rbf_step[i] <= 0.f || rbf_gamma[i] <= 0.f)
            return fail(h, TNRD_EINVAL, "RBF step and gamma must be > 0 (filter %d)", i);
        rho_max = std::max(rho_max, (double)rbf_step[i] / rbf_gamma[i]);
        for (int j = 0; j < K * K; ++j)
            if (!std::isfinite(filters[(size_t)i * K * K + j])) return fail(h, TNRD_EINVAL, "non-finite filter tap");
        for (int j = 0; j < M; ++j)
            if (!std::isfinite(rbf_w[(size_t)i * M + j])) return fail(h, TNRD_EINVAL, "non-finite RBF weight");
    }
    // Horner units when the clamp of R only touches negligible terms for every
    // filter; otherwise one unit per centre.  TNRD_PHI_TABLE:
    // cubic tables built here in double.
    (void)rho_max;
    int mode = h->d.phi_mode == TNRD_PHI_TABLE ? tnrd::MODE_TABLE : tnrd::MODE_HORNER;
    std::vector<float> host;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const int ps = pstride_for(h->d, mode);
        host.assign((size_t)Nk * ps, 0.f);
        pack_stage(h->d, filters, rbf_w, rbf_mu0, rbf_step, rbf_gamma, mode, ps, host.data());
        if (mode != tnrd::MODE_HORNER) break;
        bool ok = true;
        for (int i = 0; i < Nk; ++i) ok = ok && host[(size_t)i * ps + tnrd::tap_floats(K) + 5] != 0.f;
        if (ok) break;
        mode = tnrd::MODE_DIRECT;
    }
    {   // raw parameters for the training gradient: k, kbar = rot180(k), w; grid scalars on the host
        const size_t mm = (size_t)K * K, TN = (size_t)h->d.T * Nk;
        std::vector<float> kbar(mm * Nk);
        for (int i = 0; i < Nk; ++i)
            for (int a = 0; a < K; ++a)
                for (int b = 0; b < K; ++b)
                    kbar[i * mm + a * K + b] = filters[i * mm + (K - 1 - a) * K + (K - 1 - b)];
        DeviceGuard g(h->d.device);
        TNRD_CUDA(h, cudaMemcpy(h->d_raw + (size_t)t * Nk * mm, filters, sizeof(float) * mm * Nk,
                                cudaMemcpyHostToDevice));
        TNRD_CUDA(h, cudaMemcpy(h->d_raw + TN * mm + (size_t)t * Nk * mm, kbar.data(), sizeof(float) * mm * Nk,
                                cudaMemcpyHostToDevice));
        TNRD_CUDA(h, cudaMemcpy(h->d_raw + 2 * TN * mm + (size_t)t * Nk * M, rbf_w, sizeof(float) * (size_t)Nk * M,
                                cudaMemcpyHostToDevice));
        std::vector<float> g3((size_t)Nk * 3);
        for (int i = 0; i < Nk; ++i) {
            h->raw_mu0[(size_t)t * Nk + i] = rbf_mu0[i];
            h->raw_step[(size_t)t * Nk + i] = rbf_step[i];
            h->raw_gamma[(size_t)t * Nk + i] = rbf_gamma[i];
            g3[3 * i] = rbf_mu0[i]; g3[3 * i + 1] = rbf_step[i]; g3[3 * i + 2] = rbf_gamma[i];
        }
        TNRD_CUDA(h, cudaMemcpy(h->d_raw + 2 * TN * mm + TN * M + (size_t)t * Nk * 3, g3.data(),
                                sizeof(float) * 3 * Nk, cudaMemcpyHostToDevice));
    }
    if (mode == tnrd::MODE_TABLE) {
        std::vector<float4> tab((size_t)Nk * h->table_stride);
        for (int i = 0; i < Nk; ++i)
            build_table(rbf_w + (size_t)i * M, M, (double)rbf_step[i] / rbf_gamma[i], tab.data() + (size_t)i * h->table_stride);
        DeviceGuard g(h->d.device);
        TNRD_CUDA(h, cudaMemcpy(h->d_table + (size_t)t * Nk * h->table_stride, tab.data(),
                                sizeof(float4) * tab.size(), cudaMemcpyHostToDevice));
    }
    const int ps = pstride_for(h->d, mode);
    DeviceGuard g(h->d.device);
    TNRD_CUDA(h, cudaMemcpy(h->d_params + (size_t)t * Nk * h->pstride_max, host.data(),
                            sizeof(float) * host.size(), cudaMemcpyHostToDevice));
    h->tc_ok[t] = 0;
    if (h->d_tc && (mode == tnrd::MODE_HORNER || mode == tnrd::MODE_TABLE)) {
        std::vector<float> tc((size_t)h->tc_stride);
        pack_tc_stage(h->d, filters, host.data(), ps, mode, tc.data());
        TNRD_CUDA(h, cudaMemcpy(h->d_tc + (size_t)t * h->tc_stride, tc.data(), sizeof(float) * tc.size(),
                                cudaMemcpyHostToDevice));
        h->tc_ok[t] = 1;
    }
    h->pstride[t] = ps;
    h->mode[t] = mode;
    h->lambda[t] = lambda;
    h->is_set[t] = 1;
    drop_graphs(h);   // launch arguments (lambda, phi mode, engine eligibility) may have changed
    return TNRD_OK;
}

tnrd_status tnrd_set_grad_chunk(tnrd_handle *h, int max_filters) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    if (max_filters < 0) return fail(h, TNRD_EINVAL, "max_filters must be >= 0");
    h->grad_max_f = max_filters;
    return TNRD_OK;
}

tnrd_status tnrd_set_engine(tnrd_handle *h, int engine) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    if (engine < TNRD_ENGINE_AUTO || engine > TNRD_ENGINE_TENSOR) return fail(h, TNRD_EINVAL, "bad engine %d", engine);
    h->engine = engine;
    drop_graphs(h);
    return TNRD_OK;
}

int tnrd_engine_for(tnrd_handle *h, int B, int H, int W) {
    if (!h || check_ready(h) != TNRD_OK) return -1;
    return plan_for(h, B, H, W, true).tc_oh > 0 ? TNRD_ENGINE_TENSOR : TNRD_ENGINE_FP32;
}

tnrd_status tnrd_denoise(tnrd_handle *h, const float *f, float *u, int B, int H, int W, long long ld,
                         const float *peak, void *stream) {
    tnrd_status st = check_ready(h);
    if (st != TNRD_OK) return st;
    if (!f || !u) return fail(h, TNRD_EINVAL, "null image pointer");
    if (B < 1 || B > 65535) return fail(h, TNRD_EINVAL, "B must be in [1, 65535]");
    if (H < h->d.ksize || W < h->d.ksize) return fail(h, TNRD_EINVAL, "H, W must be >= ksize");
    if (ld < W) return fail(h, TNRD_EINVAL, "ld < W");
    const long long span = (long long)B * H * ld;
    if ((f < u && f + span > u) || (u < f && u + span > f) || f == u)
        return fail(h, TNRD_EINVAL, "u must not alias f (the prox reads f every stage)");
    if (peak)
        for (int b = 0; b < B; ++b)
            if (!std::isfinite(peak[b]) || peak[b] <= 0.f) return fail(h, TNRD_EINVAL, "peak[%d] must be > 0", b);
    DeviceGuard g(h->d.device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int T = h->d.T;
    if (T > 1) {
        st = grow(h, &h->scratch, &h->scratch_bytes, sizeof(float) * (size_t)B * H * W, "scratch");
        if (st != TNRD_OK) return st;
    }
    const Plan plan = plan_for(h, B, H, W, true);
    const tnrd::Image in_f{f, ld, (long long)H * ld, 0};
    const tnrd::Image in_s{h->scratch, W, (long long)H * W, 0};
    const tnrd::Image in_u{u, ld, (long long)H * ld, 0};
    const auto stages = [&](cudaStream_t cs) -> tnrd_status {
        for (int t = 0; t < T; ++t) {
            // ping-pong so that the last stage writes u: stage t writes u iff (T-1-t) is even
            const bool to_u = ((T - 1 - t) % 2) == 0;
            StageArgs a{};
            a.u_in = t == 0 ? in_f : (to_u ? in_s : in_u);
            a.f = in_f;
            if (to_u) { a.u_out = u; a.out_ld = ld; a.out_img_stride = (long long)H * ld; }
            else { a.u_out = h->scratch; a.out_ld = W; a.out_img_stride = (long long)H * W; }
            a.out_row_base = 0;
            a.H = H; a.W = W; a.y_begin = 0; a.y_end = H; a.avail_lo = 0; a.avail_hi = H;
            tnrd_status r = launch_one(h, t, plan, a, B, cs);
            if (r != TNRD_OK) return r;
        }
        return TNRD_OK;
    };
    if (h->use_graphs < 0) {
        const char *env = getenv("TNRD_GRAPH");
        h->use_graphs = !(env && env[0] == '0');
    }
    if (!h->use_graphs) return stages(s);
    return run_graph(h, f, u, B, H, W, ld, plan, s, stages);
}

tnrd_status tnrd_denoise_host(tnrd_handle *h, const float *f_host, float *u_host, int B, int H, int W,
                              const float *peak, void *stream) {
    tnrd_status st = check_ready(h);
    if (st != TNRD_OK) return st;
    if (!f_host || !u_host) return fail(h, TNRD_EINVAL, "null host pointer");
    if (B < 1 || H < 1 || W < 1) return fail(h, TNRD_EINVAL, "bad size");
    DeviceGuard g(h->d.device);
    const size_t bytes = sizeof(float) * (size_t)B * H * W;
    st = grow(h, &h->e2e_f, &h->e2e_f_bytes, bytes, "e2e f");
    if (st != TNRD_OK) return st;
    st = grow(h, &h->e2e_u, &h->e2e_u_bytes, bytes, "e2e u");
    if (st != TNRD_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // Pipeline over batch chunks: H2D of chunk c+1 and D2H of chunk c-1 (own
    // streams) overlap the stages of chunk c (caller's stream).  Chunks keep at
    // least ~4 tile pairs per SM so each stays on the large-tile kernel; the
    // per-pixel arithmetic does not depend on the chunking.
    const long long tiles_img = (long long)((H + 63) / 64) * ((W + 63) / 64);
    const int min_imgs = (int)std::max<long long>(1, (8LL * h->num_sms + tiles_img - 1) / tiles_img);
    const int nchunk = std::max(1, std::min(8, B / min_imgs));
    if (!h->s_h2d) {
        TNRD_CUDA(h, cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
        TNRD_CUDA(h, cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    }
    while ((int)h->chunk_ev.size() < 2 * nchunk + 1) {
        cudaEvent_t e;
        TNRD_CUDA(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->chunk_ev.push_back(e);
    }
    const size_t img = (size_t)H * W;
    for (int c = 0; c < nchunk; ++c) {
        const int b0 = (int)((long long)B * c / nchunk), b1 = (int)((long long)B * (c + 1) / nchunk);
        const size_t off = (size_t)b0 * img, cb = sizeof(float) * (size_t)(b1 - b0) * img;
        cudaEvent_t in = h->chunk_ev[2 * c], out = h->chunk_ev[2 * c + 1];
        if (c == 0) {  // the copy streams start after the caller's earlier work
            TNRD_CUDA(h, cudaEventRecord(h->chunk_ev[2 * nchunk], s));
            TNRD_CUDA(h, cudaStreamWaitEvent(h->s_h2d, h->chunk_ev[2 * nchunk], 0));
        }
        TNRD_CUDA(h, cudaMemcpyAsync(h->e2e_f + off, f_host + off, cb, cudaMemcpyHostToDevice, h->s_h2d));
        TNRD_CUDA(h, cudaEventRecord(in, h->s_h2d));
        TNRD_CUDA(h, cudaStreamWaitEvent(s, in, 0));
        st = tnrd_denoise(h, h->e2e_f + off, h->e2e_u + off, b1 - b0, H, W, W, peak ? peak + b0 : nullptr, stream);
        if (st != TNRD_OK) return st;
        TNRD_CUDA(h, cudaEventRecord(out, s));
        TNRD_CUDA(h, cudaStreamWaitEvent(h->s_d2h, out, 0));
        TNRD_CUDA(h, cudaMemcpyAsync(u_host + off, h->e2e_u + off, cb, cudaMemcpyDeviceToHost, h->s_d2h));
    }
    TNRD_CUDA(h, cudaEventRecord(h->chunk_ev[2 * nchunk], h->s_d2h));
    TNRD_CUDA(h, cudaStreamWaitEvent(s, h->chunk_ev[2 * nchunk], 0));  // caller's stream ordered after the copies
    TNRD_CUDA(h, cudaStreamSynchronize(s));
    return TNRD_OK;
}

tnrd_status tnrd_destroy(tnrd_handle *h) {
    if (!h) return TNRD_OK;
    {
        DeviceGuard g(h->d.device);
        cudaDeviceSynchronize();
        drop_graphs(h);
        if (h->s_cap) cudaStreamDestroy(h->s_cap);
        cudaFree(h->d_params);
        cudaFree(h->d_tc);
        cudaFree(h->d_table);
        cudaFree(h->d_raw);
        cudaFree(h->g_buf);
        cudaFree(h->g_partial);
        cudaFree(h->g_red);
        cudaFree(h->scratch);
        cudaFree(h->e2e_f);
        cudaFree(h->e2e_u);
        cudaFree(h->slab_buf[0]);
        cudaFree(h->slab_buf[1]);
        for (float *p : h->lb_bufs) cudaFree(p);
        for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
        for (cudaEvent_t e : h->chunk_ev) cudaEventDestroy(e);
        if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
        if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
        if (h->comm && nccl().loaded) nccl().CommDestroy(h->comm);
    }
    delete h;
    return TNRD_OK;
}

const char *tnrd_last_error(const tnrd_handle *h) {
    return h ? h->err.c_str() : g_last_error.c_str();
}

unsigned long long tnrd_launch_count(const tnrd_handle *h) { return h ? h->launches : 0ULL; }

tnrd_status tnrd_set_profiling(tnrd_handle *h, int enable) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    h->profile = enable != 0;
    h->ev_used = 0;
    return TNRD_OK;
}

tnrd_status tnrd_get_launch_times(tnrd_handle *h, float *ms_out, int n, int *n_out) {
    if (!h || !n_out) return fail(h, TNRD_EINVAL, "null argument");
    const int have = h->ev_used / 2;
    int k = 0;
    for (; k < have && k < n; ++k) {
        TNRD_CUDA(h, cudaEventSynchronize(h->ev[2 * k + 1]));
        TNRD_CUDA(h, cudaEventElapsedTime(&ms_out[k], h->ev[2 * k], h->ev[2 * k + 1]));
    }
    *n_out = have;
    return TNRD_OK;
}

tnrd_status tnrd_debug_phi(tnrd_handle *h, int t, int i, const float *v, float *out, long long n, void *stream) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    if (t < 0 || t >= h->d.T || !h->is_set[t]) return fail(h, TNRD_ESTATE, "stage %d not set", t);
    if (i < 0 || i >= h->d.n_filters) return fail(h, TNRD_EINVAL, "filter index");
    DeviceGuard g(h->d.device);
    const float4 *tab = h->d_table ? h->d_table + ((size_t)t * h->d.n_filters + i) * h->table_stride : nullptr;
    cudaError_t e = tnrd::launch_debug_phi(h->d_params + (size_t)t * h->d.n_filters * h->pstride_max,
                                           h->pstride[t], h->mode[t], tab, h->d.ksize, i, v, out, n,
                                           reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(h, e, "debug phi");
    h->launches++;
    return TNRD_OK;
}

tnrd_status tnrd_debug_prox(const float *ut, const float *f, float lambda, float *out, long long n, void *stream) {
    if (!(lambda > 0.f)) return fail(nullptr, TNRD_EINVAL, "lambda must be > 0");
    cudaError_t e = tnrd::launch_debug_prox(ut, f, lambda, out, n, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(nullptr, TNRD_ECUDA, "debug prox: %s", cudaGetErrorString(e));
    return TNRD_OK;
}

// ------------------------------------------------------------------ training gradient
tnrd_status tnrd_loss_grad(tnrd_handle *h, const float *f, const float *u_gt, int B, int H, int W, long long ld,
                           float *grad_filters, float *grad_rbf_w, float *grad_lambda, double *loss, void *stream) {
    tnrd_status st = check_ready(h);
    if (st != TNRD_OK) return st;
    if (!f || !u_gt || !grad_filters || !grad_rbf_w || !grad_lambda || !loss)
        return fail(h, TNRD_EINVAL, "null pointer");
    if (h->d.reaction != TNRD_REACTION_POISSON_PROX || h->d.phi_mode != TNRD_PHI_EXACT)
        return fail(h, TNRD_EUNSUPPORTED, "the training gradient is built for reaction 0 and exact phi");
    if (B < 1 || H < h->d.ksize || W < h->d.ksize || ld < W) return fail(h, TNRD_EINVAL, "bad image size");
    DeviceGuard g(h->d.device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int T = h->d.T, Nk = h->d.n_filters, K = h->d.ksize, M = h->d.n_rbf;
    const size_t mm = (size_t)K * K, n = (size_t)B * H * W, TN = (size_t)T * Nk;
    if (M > 64) return fail(h, TNRD_EUNSUPPORTED, "training gradient built for n_rbf <= 64");
    // filters per backward chunk: 5 per-filter images (x, a, b, w, t) within half the
    // device memory (at least 1 GB; from the total, not the free memory, so that the
    // chunking — and with it the summation order — is the same on every call with the
    // same batch); all N_k in one chunk enables the tensor banks (C4's 256 x 512^2
    // batch: 64 GB).  tnrd_set_grad_chunk caps F explicitly.  A failed allocation is
    // TNRD_ENOMEM: the chunk is never shrunk to what happens to be free.
    const size_t budget = std::max<size_t>((size_t)1 << 30, h->total_mem / 2);
    int F = (int)std::max<size_t>(1, std::min<size_t>((size_t)Nk, budget / (5 * n * sizeof(float))));
    if (h->grad_max_f > 0) F = std::min(F, h->grad_max_f);
    // tape u_0..u_T and ut_0..ut_{T-1} (2T+1 images) + g, gn, e + the chunk images
    st = grow(h, &h->g_buf, &h->g_buf_bytes, sizeof(float) * n * (2 * (size_t)T + 1 + 3 + 5 * (size_t)F),
              "gradient tape");
    if (st != TNRD_OK) return st;
    const int grid = tnrd::grad_grid((long long)n, h->num_sms);
    const int gx = tnrd::grad_chunk_grid((long long)n, F, h->num_sms);
    const int kg_nblk = tnrd::tc_kgrad_blocks(B, H, W, h->num_sms);
    const size_t part_floats = std::max((size_t)grid, (size_t)F * std::max(gx, kg_nblk) * std::max<size_t>(64, 2 * mm));
    st = grow(h, &h->g_partial, &h->g_partial_bytes, sizeof(float) * part_floats, "partials");
    if (st != TNRD_OK) return st;
    const size_t per_f = 2 * mm + M, nred = TN * per_f + T + 1;
    st = grow(h, reinterpret_cast<float **>(&h->g_red), &h->g_red_bytes, sizeof(double) * nred, "reductions");
    if (st != TNRD_OK) return st;
    float *tape_u = h->g_buf;                       // [T+1][n]
    float *tape_ut = tape_u + (size_t)(T + 1) * n;  // [T][n]
    float *wk = tape_ut + (size_t)T * n;
    float *gb = wk, *gn = wk + n, *e = wk + 2 * n;
    float *cx = wk + 3 * n, *ca = cx + (size_t)F * n, *cb = ca + (size_t)F * n, *cw = cb + (size_t)F * n,
          *ct = cw + (size_t)F * n;
    double *red_f = h->g_red, *red_lam = h->g_red + TN * per_f, *red_loss = red_lam + T;
    float *part = h->g_partial;
#define TNRD_K(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); } while (0)
    // ---- forward with tape (the fused stage kernel also writes ut)
    TNRD_K(cudaMemcpy2DAsync(tape_u, sizeof(float) * W, f, sizeof(float) * ld, sizeof(float) * W, (size_t)B * H,
                             cudaMemcpyDeviceToDevice, s));
    // the tape and the backward banks on the tensor cores unless the engine is FP32; the
    // tape's tensor stage kernel splits its operands with round-to-nearest (unbiased
    // errors); env TNRD_GRAD_TAPE=fp32 tapes on the FP32 engine
    const Plan bank_plan = plan_for(h, B, H, W, true);
    static const char *tape_env = getenv("TNRD_GRAD_TAPE");
    const Plan plan = (tape_env && tape_env[0] == 'f') ? plan_for(h, B, H, W, false) : bank_plan;
    for (int t = 0; t < T; ++t) {
        StageArgs a{};
        a.u_in = {tape_u + (size_t)t * n, W, (long long)H * W, 0};
        a.f = {f, ld, (long long)H * ld, 0};
        a.u_out = tape_u + (size_t)(t + 1) * n; a.out_ld = W; a.out_img_stride = (long long)H * W; a.out_row_base = 0;
        a.ut_out = tape_ut + (size_t)t * n;
        a.tc_rn = 1;
        a.H = H; a.W = W; a.y_begin = 0; a.y_end = H; a.avail_lo = 0; a.avail_hi = H;
        st = launch_one(h, t, plan, a, B, s);
        if (st != TNRD_OK) return st;
    }
    TNRD_K(tnrd::grad_loss(tape_u + (size_t)T * n, u_gt, ld, B, H, W, gb, part, grid, s));
    TNRD_K(tnrd::grad_reduce(part, grid, 1, 1, red_loss, s));
    // ---- backward, P Eq.14-20: per stage the prox backward, then chunks of F filters
    const float *raw_k = h->d_raw, *raw_kbar = h->d_raw + TN * mm, *raw_w = h->d_raw + 2 * TN * mm;
    const float *raw_g3 = raw_w + TN * M;
    for (int t = T - 1; t >= 0; --t) {
        TNRD_K(tnrd::grad_bw_prox(tape_ut + (size_t)t * n, f, ld, B, H, W, h->lambda[t], gb, e, gn, part, grid, s));
        TNRD_K(tnrd::grad_reduce(part, grid, 1, 1, red_lam + t, s));
        for (int i0 = 0; i0 < Nk; i0 += F) {
            tnrd::GradChunk c{};
            c.k = raw_k; c.kbar = raw_kbar; c.rw = raw_w; c.grid3 = raw_g3;
            c.fi0 = t * Nk + i0; c.F = std::min(F, Nk - i0);
            c.m = K; c.M = M; c.B = B; c.H = H; c.W = W; c.boundary = h->d.boundary; c.gx = gx; c.num_sms = h->num_sms;
            c.u = tape_u + (size_t)t * n; c.e = e;
            c.gn = gn; c.x = cx; c.a = ca; c.b = cb; c.w = cw; c.t = ct; c.partial = part;
            c.red = red_f + (size_t)(t * Nk + i0) * per_f; c.red_stride = (int)per_f;
            static const char *adj_env = getenv("TNRD_GRAD_ADJ");  // tests: "fp32" keeps the CUDA-core adjoint
            if (bank_plan.tc_oh > 0 && F == Nk && !(adj_env && adj_env[0] == 'f')) {
                c.tc_ba = h->d_tc + (size_t)t * h->tc_stride + 2 * (size_t)Nk * tnrd::tc_ktp(K);
                c.tc_bf = h->d_tc + (size_t)t * h->tc_stride;
                c.tc_oh = bank_plan.tc_oh;
                static const char *kg_env = getenv("TNRD_GRAD_KG");  // tests: "fp32" keeps the CUDA-core k-gradient
                if (!(kg_env && kg_env[0] == 'f')) c.tc_kg_nblk = kg_nblk;
            }
            TNRD_K(tnrd::grad_chunk(c, s));
        }
        std::swap(gb, gn);
    }
#undef TNRD_K
    std::vector<double> red(nred);
    TNRD_CUDA(h, cudaMemcpyAsync(red.data(), h->g_red, sizeof(double) * nred, cudaMemcpyDeviceToHost, s));
    TNRD_CUDA(h, cudaStreamSynchronize(s));
    for (size_t fi = 0; fi < TN; ++fi) {
        const double *rf = red.data() + fi * per_f;
        float *gk = grad_filters + fi * mm;
        for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) {
                // d l / d k = -(inner) - (outer): R1's outer kernel is kbar, so its taps map back by rot180
                const double outer = h->d.boundary == 1 ? rf[mm + a * K + b] : rf[mm + (K - 1 - a) * K + (K - 1 - b)];
                gk[a * K + b] = (float)(-(rf[a * K + b] + outer));
            }
        for (int j = 0; j < M; ++j) grad_rbf_w[fi * M + j] = (float)rf[2 * mm + j];
    }
    for (int t = 0; t < T; ++t) grad_lambda[t] = (float)red[TN * per_f + t];
    *loss = red[TN * per_f + T];
    return TNRD_OK;
}

// ------------------------------------------------------------------ data generation / evaluation
tnrd_status tnrd_sample_poisson(const float *u, float *f, int B, int H, int W, long long ld, unsigned long long seed,
                                void *stream) {
    if (!u || !f) return fail(nullptr, TNRD_EINVAL, "null pointer");
    if (B < 1 || H < 1 || W < 1 || ld < W) return fail(nullptr, TNRD_EINVAL, "bad size");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int *bad = nullptr;
    cudaError_t e = cudaMallocAsync(&bad, sizeof(int), s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ENOMEM, "cudaMallocAsync: %s", cudaGetErrorString(e));
    int hbad = 0;
    e = cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (e == cudaSuccess) e = tnrd::data_sample_poisson(u, f, B, H, W, ld, seed, bad, sms, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(bad, s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ECUDA, "sample_poisson: %s", cudaGetErrorString(e));
    if (hbad) return fail(nullptr, TNRD_EINVAL, "negative or NaN Poisson mean");
    return TNRD_OK;
}

tnrd_status tnrd_psnr(const float *u, const float *c, int B, int H, int W, long long ld, const float *peak,
                      double *out, void *stream) {
    if (!u || !c || !peak || !out) return fail(nullptr, TNRD_EINVAL, "null pointer");
    if (B < 1 || H < 1 || W < 1 || ld < W) return fail(nullptr, TNRD_EINVAL, "bad size");
    if (B > 65535) return fail(nullptr, TNRD_EINVAL, "B must be <= 65535 (grid.y)");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int nb = tnrd::data_sq_err_blocks((long long)H * W, sms);
    double *part = nullptr;
    cudaError_t e = cudaMallocAsync(&part, sizeof(double) * (size_t)B * nb, s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ENOMEM, "cudaMallocAsync: %s", cudaGetErrorString(e));
    std::vector<double> hp((size_t)B * nb);
    e = tnrd::data_sq_err(u, c, B, H, W, ld, part, nb, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), part, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(part, s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ECUDA, "psnr: %s", cudaGetErrorString(e));
    for (int b = 0; b < B; ++b) {
        double sse = 0.0;
        for (int j = 0; j < nb; ++j) sse += hp[(size_t)b * nb + j];
        const double mse = sse / ((double)H * W);
        out[b] = mse > 0.0 ? 10.0 * std::log10((double)peak[b] * peak[b] / mse) : INFINITY;
    }
    return TNRD_OK;
}

tnrd_status tnrd_scale_to_peak(const float *x, float *out, int B, int H, int W, long long ld, const float *peak,
                               void *stream) {
    if (!x || !out || !peak) return fail(nullptr, TNRD_EINVAL, "null pointer");
    if (B < 1 || H < 1 || W < 1 || ld < W) return fail(nullptr, TNRD_EINVAL, "bad size");
    if (B > 65535) return fail(nullptr, TNRD_EINVAL, "B must be <= 65535 (grid.y)");
    for (int b = 0; b < B; ++b)
        if (!std::isfinite(peak[b]) || peak[b] <= 0.f) return fail(nullptr, TNRD_EINVAL, "peak[%d] must be > 0", b);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // scratch: mx [B] (unsigned), bad (int), peak [B] (float)
    char *scr = nullptr;
    const size_t n_mx = sizeof(unsigned) * (size_t)B, n_bad = 16, n_pk = sizeof(float) * (size_t)B;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&scr), n_mx + n_bad + n_pk, s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ENOMEM, "cudaMallocAsync: %s", cudaGetErrorString(e));
    unsigned *mx = reinterpret_cast<unsigned *>(scr);
    int *bad = reinterpret_cast<int *>(scr + n_mx);
    float *pk = reinterpret_cast<float *>(scr + n_mx + n_bad);
    std::vector<unsigned> hm((size_t)B);
    int hbad = 0;
    e = cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pk, peak, n_pk, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = tnrd::data_scale_to_peak(x, out, B, H, W, ld, pk, mx, bad, sms, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hm.data(), mx, n_mx, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(scr, s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ECUDA, "scale_to_peak: %s", cudaGetErrorString(e));
    if (hbad) return fail(nullptr, TNRD_EINVAL, "scale_to_peak: negative or NaN input (out is undefined)");
    for (int b = 0; b < B; ++b)
        if (hm[b] == 0) return fail(nullptr, TNRD_EINVAL, "scale_to_peak: image %d is all zero (out is undefined)", b);
    return TNRD_OK;
}

tnrd_status tnrd_ssim(const float *u, const float *c, int B, int H, int W, long long ld, const float *peak,
                      double *out, void *stream) {
    if (!u || !c || !peak || !out) return fail(nullptr, TNRD_EINVAL, "null pointer");
    if (B < 1 || H < 11 || W < 11 || ld < W) return fail(nullptr, TNRD_EINVAL, "bad size (H, W >= 11)");
    if (B > 65535) return fail(nullptr, TNRD_EINVAL, "B must be <= 65535 (grid.y)");
    for (int b = 0; b < B; ++b)
        if (!std::isfinite(peak[b]) || peak[b] <= 0.f) return fail(nullptr, TNRD_EINVAL, "peak[%d] must be > 0", b);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const long long windows = (long long)(H - 10) * (W - 10);
    const int nb = tnrd::data_ssim_blocks(windows, sms);
    std::vector<double> hs((size_t)B);
    for (int b = 0; b < B; ++b) hs[b] = 255.0 / (double)peak[b];
    double *buf = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&buf), sizeof(double) * (size_t)B * (nb + 1), s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ENOMEM, "cudaMallocAsync: %s", cudaGetErrorString(e));
    double *scale = buf, *part = buf + B;
    std::vector<double> hp((size_t)B * nb);
    e = cudaMemcpyAsync(scale, hs.data(), sizeof(double) * (size_t)B, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = tnrd::data_ssim(u, c, B, H, W, ld, scale, part, nb, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), part, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(buf, s);
    if (e != cudaSuccess) return fail(nullptr, TNRD_ECUDA, "ssim: %s", cudaGetErrorString(e));
    for (int b = 0; b < B; ++b) {
        double sum = 0.0;
        for (int j = 0; j < nb; ++j) sum += hp[(size_t)b * nb + j];
        out[b] = sum / (double)windows;
    }
    return TNRD_OK;
}

// ------------------------------------------------------------------ slabs
tnrd_status tnrd_nccl_unique_id(void *id128) {
    if (!id128) return fail(nullptr, TNRD_EINVAL, "null id");
    NcclApi &api = nccl();
    if (!api.loaded) return fail(nullptr, TNRD_ENCCL, "%s", api.why.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, TNRD_ENCCL, "ncclGetUniqueId: %s", api.GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, 128);
    return TNRD_OK;
}

tnrd_status tnrd_comm_init(tnrd_handle *h, const void *id128, int rank, int nranks) {
    if (!h || !id128) return fail(h, TNRD_EINVAL, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(h, TNRD_EINVAL, "rank %d of %d", rank, nranks);
    NcclApi &api = nccl();
    if (!api.loaded) return fail(h, TNRD_ENCCL, "%s", api.why.c_str());
    DeviceGuard g(h->d.device);
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    if (h->comm) { api.CommDestroy(h->comm); h->comm = nullptr; }
    ncclResult_t r = api.CommInitRank(&h->comm, nranks, id, rank);
    if (r != ncclSuccess) return fail(h, TNRD_ENCCL, "ncclCommInitRank: %s", api.GetErrorString(r));
    h->rank = rank;
    h->nranks = nranks;
    return TNRD_OK;
}

namespace {
tnrd_status slab_args_ok(tnrd_handle *h, int H, int W, int row0, int rows, long long ld) {
    const int halo = h->d.ksize - 1;
    if (W < h->d.ksize || H < h->d.ksize) return fail(h, TNRD_EINVAL, "H, W must be >= ksize");
    if (rows < halo || rows < 1) return fail(h, TNRD_EINVAL, "slab rows (%d) must be >= ksize-1", rows);
    if (row0 < 0 || row0 + rows > H) return fail(h, TNRD_EINVAL, "slab [%d, %d) outside [0, %d)", row0, row0 + rows, H);
    if (ld < W) return fail(h, TNRD_EINVAL, "ld < W");
    return TNRD_OK;
}

// Run all T stages of one slab set.  `slabs` lists (row0, rows, buf0, buf1) per slab k;
// `ex` fills halos.  Stage order: for t: for k (exchange, then compute) -- the
// exchange of stage t only reads rows written by stage t-1.
struct SlabDesc { int row0, rows; float *buf[2]; const float *f; long long f_ld; float *u; long long u_ld; };

tnrd_status run_slabs(tnrd_handle *h, std::vector<SlabDesc> &sl, int H, int W, SlabExchange &ex, cudaStream_t s) {
    const int halo = h->d.ksize - 1;
    for (size_t k = 0; k < sl.size(); ++k) {  // seed buffer 0 with f (u_0 = f)
        cudaError_t e = tnrd::launch_copy_rows(sl[k].f, sl[k].f_ld, sl[k].buf[0] + (size_t)halo * W, W,
                                               sl[k].rows, W, s);
        if (e != cudaSuccess) return cuda_fail(h, e, "seed slab");
    }
    for (int t = 0; t < h->d.T; ++t) {
        for (size_t k = 0; k < sl.size(); ++k) {
            tnrd_status st = ex.exchange((int)k, sl[k].buf[t % 2]);
            if (st != TNRD_OK) return st;
        }
        for (size_t k = 0; k < sl.size(); ++k) {
            tnrd_status st = run_slab(h, sl[k].f, sl[k].f_ld, sl[k].u, sl[k].u_ld, H, W, sl[k].row0, sl[k].rows,
                                      sl[k].buf[0], sl[k].buf[1], ex, (int)k, t, s);
            if (st != TNRD_OK) return st;
        }
    }
    return TNRD_OK;
}

struct LoopbackExchange : SlabExchange {
    tnrd_handle *h; std::vector<SlabDesc> *sl; int W; cudaStream_t s; int t = 0;
    LoopbackExchange(tnrd_handle *h_, std::vector<SlabDesc> *sl_, int W_, cudaStream_t s_) : h(h_), sl(sl_), W(W_), s(s_) {}
    tnrd_status exchange(int k, float *buf) override {
        // halos of slab k come from the same-parity buffers of slabs k-1 and k+1
        const int halo = h->d.ksize - 1;
        std::vector<SlabDesc> &v = *sl;
        const int par = (buf == v[k].buf[0]) ? 0 : 1;
        const size_t n = sizeof(float) * (size_t)halo * W;
        if (k > 0) {
            const SlabDesc &up = v[k - 1];
            cudaError_t e = cudaMemcpyAsync(buf, up.buf[par] + (size_t)up.rows * W, n, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return cuda_fail(h, e, "loopback halo up");
        }
        if (k + 1 < (int)v.size()) {
            const SlabDesc &dn = v[k + 1];
            cudaError_t e = cudaMemcpyAsync(buf + (size_t)(halo + v[k].rows) * W, dn.buf[par] + (size_t)halo * W, n,
                                            cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return cuda_fail(h, e, "loopback halo down");
        }
        return TNRD_OK;
    }
};
// The slab halos of an nslabs partition moved by NCCL point-to-point on a 1-rank
// communicator (every send and receive has the caller's own rank as peer): one
// grouped exchange per stage, posted when the last slab's exchange is requested
// (the earlier slabs' buffers are complete by then).  NCCL matches sends and
// receives of one peer in posting order, so the sends list every slab's bottom
// owned rows then every slab's top owned rows, and the receives the matching halo
// rows of the neighbours in the same order.  Tests the NCCL transfer of the real
// slab buffers and sizes on one GPU (tnrd_denoise_slabs_nccl_self).
struct NcclSelfExchange : SlabExchange {
    tnrd_handle *h; std::vector<SlabDesc> *sl; int W; cudaStream_t s;
    NcclSelfExchange(tnrd_handle *h_, std::vector<SlabDesc> *sl_, int W_, cudaStream_t s_) : h(h_), sl(sl_), W(W_), s(s_) {}
    tnrd_status exchange(int k, float *buf) override {
        std::vector<SlabDesc> &v = *sl;
        if (k + 1 < (int)v.size()) return TNRD_OK;
        NcclApi &api = nccl();
        const int halo = h->d.ksize - 1, n = (int)v.size();
        const int par = (buf == v[k].buf[0]) ? 0 : 1;
        const size_t cnt = (size_t)halo * W;
        ncclResult_t r = api.GroupStart();
        for (int j = 0; j + 1 < n && r == ncclSuccess; ++j)   // bottom owned rows of j -> halo of j + 1
            r = api.Send(v[j].buf[par] + (size_t)v[j].rows * W, cnt, ncclFloat32, h->rank, h->comm, s);
        for (int j = 1; j < n && r == ncclSuccess; ++j)       // top owned rows of j -> halo of j - 1
            r = api.Send(v[j].buf[par] + (size_t)halo * W, cnt, ncclFloat32, h->rank, h->comm, s);
        for (int j = 1; j < n && r == ncclSuccess; ++j)
            r = api.Recv(v[j].buf[par], cnt, ncclFloat32, h->rank, h->comm, s);
        for (int j = 0; j + 1 < n && r == ncclSuccess; ++j)
            r = api.Recv(v[j].buf[par] + (size_t)(halo + v[j].rows) * W, cnt, ncclFloat32, h->rank, h->comm, s);
        ncclResult_t r2 = api.GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(h, TNRD_ENCCL, "self halo exchange: %s", api.GetErrorString(r != ncclSuccess ? r : r2));
        return TNRD_OK;
    }
};

// Slab descriptors of an nslabs partition of one image, with handle-owned buffers.
tnrd_status setup_loopback(tnrd_handle *h, const float *f, float *u, int H, int W, long long ld, int nslabs,
                           std::vector<SlabDesc> &sl) {
    const int halo = h->d.ksize - 1;
    sl.assign(nslabs, SlabDesc{});
    int maxrows = 0;
    for (int k = 0; k < nslabs; ++k) {
        const int r0 = (int)((long long)H * k / nslabs), r1 = (int)((long long)H * (k + 1) / nslabs);
        tnrd_status st = slab_args_ok(h, H, W, r0, r1 - r0, ld);
        if (st != TNRD_OK) return st;
        sl[k].row0 = r0; sl[k].rows = r1 - r0;
        maxrows = std::max(maxrows, r1 - r0);
    }
    const size_t bytes = sizeof(float) * (size_t)(maxrows + 2 * halo) * W;
    if ((int)h->lb_bufs.size() < 2 * nslabs || h->lb_bytes < bytes) {
        cudaDeviceSynchronize();
        for (float *p : h->lb_bufs) cudaFree(p);
        h->lb_bufs.clear();
        h->lb_bytes = 0;
        std::vector<float *> bufs(2 * nslabs, nullptr);
        for (auto &p : bufs) {
            cudaError_t e = cudaMalloc(&p, bytes);
            if (e != cudaSuccess) {   // release the partial set: the handle keeps none
                for (float *q : bufs) cudaFree(q);
                cudaGetLastError();
                return fail(h, TNRD_ENOMEM, "loopback buffers: %s", cudaGetErrorString(e));
            }
        }
        h->lb_bufs = bufs;
        h->lb_bytes = bytes;
    }
    for (int k = 0; k < nslabs; ++k) {
        sl[k].buf[0] = h->lb_bufs[2 * k];
        sl[k].buf[1] = h->lb_bufs[2 * k + 1];
        sl[k].f = f + (size_t)sl[k].row0 * ld; sl[k].f_ld = ld;
        sl[k].u = u + (size_t)sl[k].row0 * ld; sl[k].u_ld = ld;
    }
    return TNRD_OK;
}
}  // namespace

tnrd_status tnrd_denoise_slab(tnrd_handle *h, const float *f_slab, float *u_slab, int H, int W, int row0, int rows,
                              long long ld, float peak, void *stream) {
    tnrd_status st = check_ready(h);
    if (st != TNRD_OK) return st;
    if (!h->comm && h->nranks > 1) return fail(h, TNRD_ESTATE, "communicator not initialised");
    if (!f_slab || !u_slab || f_slab == u_slab) return fail(h, TNRD_EINVAL, "bad slab pointers");
    if (!std::isfinite(peak) || peak <= 0.f) return fail(h, TNRD_EINVAL, "peak must be > 0");
    st = slab_args_ok(h, H, W, row0, rows, ld);
    if (st != TNRD_OK) return st;
    DeviceGuard g(h->d.device);
    const int halo = h->d.ksize - 1;
    const size_t bytes = sizeof(float) * (size_t)(rows + 2 * halo) * W;
    for (int k = 0; k < 2; ++k) {
        st = grow(h, &h->slab_buf[k], &h->slab_bytes[k], bytes, "slab buffer");
        if (st != TNRD_OK) return st;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    std::vector<SlabDesc> sl{{row0, rows, {h->slab_buf[0], h->slab_buf[1]}, f_slab, ld, u_slab, ld}};
    NcclExchange ex(h, rows, W, s);
    if (h->nranks == 1) {
        struct NoExchange : SlabExchange { tnrd_status exchange(int, float *) override { return TNRD_OK; } } none;
        return run_slabs(h, sl, H, W, none, s);
    }
    return run_slabs(h, sl, H, W, ex, s);
}

tnrd_status tnrd_comm_wait(tnrd_handle *h, void *stream, int timeout_ms) {
    if (!h) return fail(nullptr, TNRD_EINVAL, "null handle");
    DeviceGuard g(h->d.device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return comm_async_check(h);
        if (q != cudaErrorNotReady) return cuda_fail(h, q, "stream");
        tnrd_status st = comm_async_check(h);
        if (st != TNRD_OK) return st;
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
        if (timeout_ms >= 0 && ms.count() > timeout_ms) {
            if (h->comm) {
                nccl().CommAbort(h->comm);
                h->comm = nullptr;
                return fail(h, TNRD_ENCCL, "timed out after %d ms waiting for the halo exchanges (communicator aborted)",
                            timeout_ms);
            }
            return fail(h, TNRD_ECUDA, "timed out after %d ms", timeout_ms);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

tnrd_status tnrd_denoise_slabs_loopback(tnrd_handle *h, const float *f, float *u, int H, int W, long long ld,
                                        int nslabs, void *stream) {
    tnrd_status st = check_ready(h);
    if (st != TNRD_OK) return st;
    if (!f || !u || f == u) return fail(h, TNRD_EINVAL, "bad pointers");
    if (nslabs < 1 || nslabs > H) return fail(h, TNRD_EINVAL, "nslabs");
    DeviceGuard g(h->d.device);
    std::vector<SlabDesc> sl;
    st = setup_loopback(h, f, u, H, W, ld, nslabs, sl);
    if (st != TNRD_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    LoopbackExchange ex(h, &sl, W, s);
    return run_slabs(h, sl, H, W, ex, s);
}

tnrd_status tnrd_denoise_slabs_nccl_self(tnrd_handle *h, const float *f, float *u, int H, int W, long long ld,
                                         int nslabs, void *stream) {
    tnrd_status st = check_ready(h);
    if (st != TNRD_OK) return st;
    if (!h->comm || h->nranks != 1) return fail(h, TNRD_ESTATE, "needs a 1-rank communicator (tnrd_comm_init)");
    if (!f || !u || f == u) return fail(h, TNRD_EINVAL, "bad pointers");
    if (nslabs < 1 || nslabs > H) return fail(h, TNRD_EINVAL, "nslabs");
    DeviceGuard g(h->d.device);
    std::vector<SlabDesc> sl;
    st = setup_loopback(h, f, u, H, W, ld, nslabs, sl);
    if (st != TNRD_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    NcclSelfExchange ex(h, &sl, W, s);
    return run_slabs(h, sl, H, W, ex, s);
}

}  // extern "C"
