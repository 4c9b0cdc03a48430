// lemix_api.cpp -- host side of the liblemix C ABI (include/lemix.h).
//
// Owns device memory, validates what can be validated on the host (profile,
// parameters, CSR metadata), launches the persistent event-loop kernel and the
// cell reduction on the context stream, and resolves NCCL at run time for the
// one cross-GPU summary all-reduce.  No scheduling arithmetic happens here.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lemix.h"
#include "lemix_internal.h"

namespace {

thread_local std::string g_create_error;

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    bool owned = true;
    ~DevBuf() { release(); }
    void release()
    {
        if (p && owned) cudaFree(p);
        p = nullptr;
        bytes = 0;
        owned = true;
    }
    cudaError_t ensure(size_t b)
    {
        if (owned && p && bytes >= b) return cudaSuccess;
        release();
        if (b == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        else p = nullptr;
        return e;
    }
    void borrow(const void *q)
    {
        release();
        p = const_cast<void *>(q);
        owned = false;
    }
};

bool is_pinned(const void *h)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

const char *field_name(int code)
{
    switch (code) {
    case lmx::kErrLen: return "len_batch_kind.length (must be 1..2048)";
    case lmx::kErrBatch: return "len_batch_kind.batch (must be 1..255)";
    case lmx::kErrKind: return "len_batch_kind.kind (must match the inference-first layout)";
    case lmx::kErrBits: return "len_batch_kind (bits 21-31 must be zero)";
    case lmx::kErrArrival: return "arrival (must be finite and >= 0)";
    case lmx::kErrOrder: return "arrival (inference tasks must be non-decreasing)";
    case lmx::kErrFixed: return "fixed_node (must be in [0, n_nodes))";
    case lmx::kErrSeparateN1: return "policy Separate needs n_nodes >= 2 when both kinds are present";
    case lmx::kErrOutLen: return "out_len (must be 0..2048)";
    case lmx::kErrResponse: return "profile/arrival: a candidate's response time R <= 0 (Eq. 3 undefined; eta too small for the arrival time)";
    default: return "unknown";
    }
}

// ---- NCCL, resolved at run time (the process may already have torch's copy) ----
typedef int (*nccl_get_unique_id_t)(void *);
typedef int (*nccl_comm_init_rank_t)(void **, int, /*ncclUniqueId by value*/ struct NcclId128, int);
struct NcclId128 { char internal[128]; };
typedef int (*nccl_comm_init_rank2_t)(void **, int, NcclId128, int);
typedef int (*nccl_all_reduce_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_group_t)();
typedef int (*nccl_comm_destroy_t)(void *);

struct Nccl {
    void *h = nullptr;
    nccl_get_unique_id_t get_unique_id = nullptr;
    nccl_comm_init_rank2_t comm_init_rank = nullptr;
    nccl_all_reduce_t all_reduce = nullptr;
    nccl_group_t group_start = nullptr, group_end = nullptr;
    nccl_comm_destroy_t comm_destroy = nullptr;
    bool load()
    {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        get_unique_id = (nccl_get_unique_id_t)dlsym(h, "ncclGetUniqueId");
        comm_init_rank = (nccl_comm_init_rank2_t)dlsym(h, "ncclCommInitRank");
        all_reduce = (nccl_all_reduce_t)dlsym(h, "ncclAllReduce");
        group_start = (nccl_group_t)dlsym(h, "ncclGroupStart");
        group_end = (nccl_group_t)dlsym(h, "ncclGroupEnd");
        comm_destroy = (nccl_comm_destroy_t)dlsym(h, "ncclCommDestroy");
        return get_unique_id && comm_init_rank && all_reduce && group_start && group_end && comm_destroy;
    }
};
Nccl g_nccl;
// ncclDataType_t / ncclRedOp_t values (stable NCCL ABI)
constexpr int kNcclInt64 = 4, kNcclFloat64 = 8, kNcclSum = 0;

}  // namespace

struct lmx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;

    // profile
    bool have_profile = false;
    int N = 0, S = 0;
    DevBuf eta;

    // traces
    bool have_traces = false;
    int64_t n_traces = 0, n_tasks = 0;
    // host task arrays borrowed until the next lmx_sync; lmx_run streams them
    // into HBM on copy_stream while the kernel runs (chunked, see wait_inputs)
    const double *h_arrival = nullptr;
    const uint32_t *h_lbk = nullptr;
    bool host_pending = false;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_armed = nullptr, ev_copied = nullptr;
    DevBuf ready;
    unsigned *h_seq = nullptr;      // pinned 1..n: the values written to *ready
    int64_t h_seq_len = 0;
    std::vector<int64_t> h_offsets;
    std::vector<int32_t> h_n_inf;
    bool has_fixed = false, has_out_len = false;
    DevBuf offsets, n_inf, arrival, lbk, fixed, out_len;

    // params
    bool have_params = false;
    lmx_params par{};

    // cells
    int32_t n_cells = 1;
    DevBuf cell_of, cell_i, cell_f;
    DevBuf cell_start, cell_order;   // CSR of the traces of each cell (lmx_set_cells)
    bool cells_set = false;

    // outputs / state
    int per_task = 1;
    DevBuf node_defer, decision_idx, completion, start_f1;
    DevBuf cand;           // debug_level 1: (II, R, f) per decision and node
    bool cand_valid = false;
    DevBuf ck;             // Separate's checkpoint lists (sync model)
    DevBuf cell_par;       // per-cell (lambda1, lambda2, tau)
    int32_t n_cell_par = 0;
    DevBuf summaries, trace_err, work, first_bad, ring_be;
    bool ran = false, synced = false;

    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    int32_t launches = 0, grid = 0, block = 0, lanes = 0, smem = 0;

    lmx_status fail(lmx_status s, const std::string &m)
    {
        err = m;
        return s;
    }
    lmx_status cuda(cudaError_t e, const char *what)
    {
        if (e == cudaSuccess) return LMX_OK;
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return LMX_ECUDA;
    }
};

extern "C" {

void lmx_params_default(lmx_params *p)
{
    if (!p) return;
    p->policy = LMX_LEMIX;
    p->deprioritize = 1;
    p->slo_mode = 0;
    p->qcap = 512;
    p->lambda1 = 1.0;
    p->lambda2 = 1.0;
    p->tau = 0.0;
    p->slo_mult = 5.0;
    p->slo_const = 0.0;
    p->sigma_floor = 1.0;
    p->lc0 = 0.0;
    p->alpha = 0.5;
    p->mem_enable = 0;     // unlimited memory: the executed path is the plan
    p->mem_pad = 0;
    p->mem_cap = 0;
    p->mem_dt = 0.0;
    p->mem_tmax = 0.0;
    p->mem_pen = 0.0;
    p->sync_interval = 0;  // co-located version proxy for every policy
    p->sync_pad = 0;
    p->sync_latency = 0.0;
    p->sep_dynamic = 0;    // static alpha partition
    p->sep_pad = 0;
    p->dyn_rate = 50.0;
    p->dyn_window = 10.0;
    p->debug_level = 0;
    p->debug_pad = 0;
    p->cb_cmax = 0;        // every request placed on its own
    p->eq4_mode = 0;       // R-14
    p->cb_tw = 0.0;
    p->luf_delay = 0.0;
}

lmx_status lmx_create(lmx_ctx **out, int device, void *cuda_stream)
{
    if (!out) {
        g_create_error = "lmx_create: out is NULL";
        return LMX_EINVAL;
    }
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || device < 0 || device >= n) {
        g_create_error = std::string("lmx_create: no CUDA device ") + std::to_string(device) +
                         (e != cudaSuccess ? std::string(" (") + cudaGetErrorString(e) + ")" : "");
        cudaGetLastError();
        return LMX_ECUDA;
    }
    if ((e = cudaSetDevice(device)) != cudaSuccess) {
        g_create_error = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
        return LMX_ECUDA;
    }
    lmx_ctx *c = new lmx_ctx();
    c->device = device;
    if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else {
        if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
            g_create_error = std::string("cudaStreamCreate: ") + cudaGetErrorString(e);
            delete c;
            return LMX_ECUDA;
        }
        c->own_stream = true;
    }
    cudaEventCreate(&c->ev0);
    cudaEventCreate(&c->ev1);
    cudaEventCreate(&c->ev2);
    cudaEventCreateWithFlags(&c->ev_armed, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_copied, cudaEventDisableTiming);
    // non-blocking: must never be serialised behind the kernel it feeds
    cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    lmx_params_default(&c->par);
    if (c->work.ensure(8) != cudaSuccess || c->first_bad.ensure(8) != cudaSuccess) {
        g_create_error = "lmx_create: device allocation failed";
        delete c;
        return LMX_ENOMEM;
    }
    *out = c;
    return LMX_OK;
}

void lmx_destroy(lmx_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->ev_armed) cudaEventDestroy(c->ev_armed);
    if (c->ev_copied) cudaEventDestroy(c->ev_copied);
    if (c->h_seq) cudaFreeHost(c->h_seq);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->ev2) cudaEventDestroy(c->ev2);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char *lmx_last_error(const lmx_ctx *c) { return c ? c->err.c_str() : g_create_error.c_str(); }

lmx_status lmx_load_profile(lmx_ctx *c, const lmx_profile *pr)
{
    if (!c) return LMX_EINVAL;
    if (!pr || !pr->eta_f || !pr->eta_b) return c->fail(LMX_EINVAL, "lmx_load_profile: NULL profile or table");
    if (pr->n_nodes < 1 || pr->n_nodes > 128)
        return c->fail(LMX_EINVAL, "profile.n_nodes must be in [1, 128], got " + std::to_string(pr->n_nodes));
    if (pr->n_stages < 1 || pr->n_stages > 16)
        return c->fail(LMX_EINVAL, "profile.n_stages must be in [1, 16], got " + std::to_string(pr->n_stages));
    const int NS = pr->n_nodes * pr->n_stages;
    // eta_f | eta_b | eta_d (+ one pad double: the kernel stages a multiple of 16 bytes)
    std::vector<double> h(3 * (size_t)NS + 1, 0.0);
    for (int k = 0; k < NS; ++k) {
        const double f = pr->eta_f[k], b = pr->eta_b[k];
        if (!(f > 0.0 && std::isfinite(f)))
            return c->fail(LMX_EINVAL, "profile.eta_f[" + std::to_string(k) + "] must be finite and > 0");
        if (!(b > 0.0 && std::isfinite(b)))
            return c->fail(LMX_EINVAL, "profile.eta_b[" + std::to_string(k) + "] must be finite and > 0");
        h[k] = f;
        h[NS + k] = b;
        if (pr->eta_d) {
            const double d = pr->eta_d[k];
            if (!(d >= 0.0 && std::isfinite(d)))
                return c->fail(LMX_EINVAL, "profile.eta_d[" + std::to_string(k) + "] must be finite and >= 0");
            h[2 * NS + k] = d;
        }
    }
    cudaSetDevice(c->device);
    if (c->eta.ensure(h.size() * sizeof(double)) != cudaSuccess) return c->fail(LMX_ENOMEM, "profile allocation");
    lmx_status s = c->cuda(cudaMemcpyAsync(c->eta.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice,
                                           c->stream),
                           "profile copy");
    if (s != LMX_OK) return s;
    s = c->cuda(cudaStreamSynchronize(c->stream), "profile copy");
    if (s != LMX_OK) return s;
    c->N = pr->n_nodes;
    c->S = pr->n_stages;
    c->have_profile = true;
    c->ran = false;
    return LMX_OK;
}

lmx_status lmx_load_traces(lmx_ctx *c, const lmx_traces *tr, lmx_mem mem)
{
    if (!c) return LMX_EINVAL;
    if (!c->have_profile) return c->fail(LMX_ESTATE, "lmx_load_traces: load the profile first");
    if (!tr || !tr->offsets || !tr->n_inf) return c->fail(LMX_EINVAL, "lmx_load_traces: NULL traces/offsets/n_inf");
    if (tr->n_traces < 0) return c->fail(LMX_EINVAL, "traces.n_traces must be >= 0");
    if (mem != LMX_HOST && mem != LMX_DEVICE) return c->fail(LMX_EINVAL, "lmx_load_traces: bad lmx_mem");
    const int64_t T = tr->n_traces;
    if (tr->offsets[0] != 0) return c->fail(LMX_EINVAL, "traces.offsets[0] must be 0");
    for (int64_t t = 0; t < T; ++t) {
        const int64_t len = tr->offsets[t + 1] - tr->offsets[t];
        if (len < 0) return c->fail(LMX_EINVAL, "traces.offsets must be non-decreasing (trace " + std::to_string(t) + ")");
        if (len > (int64_t(1) << 19))
            return c->fail(LMX_EINVAL, "trace " + std::to_string(t) + " has more than 2^19 tasks");
        if (tr->n_inf[t] < 0 || tr->n_inf[t] > len)
            return c->fail(LMX_EINVAL, "traces.n_inf[" + std::to_string(t) + "] must be in [0, trace length]");
    }
    const int64_t M = tr->offsets[T];
    if (M > 0 && (!tr->arrival || !tr->len_batch_kind))
        return c->fail(LMX_EINVAL, "traces.arrival / len_batch_kind are NULL");
    cudaSetDevice(c->device);
    c->h_offsets.assign(tr->offsets, tr->offsets + T + 1);
    c->h_n_inf.assign(tr->n_inf, tr->n_inf + T);
    if (c->offsets.ensure((T + 1) * 8) != cudaSuccess || c->n_inf.ensure(std::max<int64_t>(T, 1) * 4) != cudaSuccess)
        return c->fail(LMX_ENOMEM, "trace metadata allocation");
    lmx_status s = c->cuda(cudaMemcpyAsync(c->offsets.p, c->h_offsets.data(), (T + 1) * 8, cudaMemcpyHostToDevice,
                                           c->stream), "offsets copy");
    if (s == LMX_OK && T > 0)
        s = c->cuda(cudaMemcpyAsync(c->n_inf.p, c->h_n_inf.data(), T * 4, cudaMemcpyHostToDevice, c->stream),
                    "n_inf copy");
    if (s != LMX_OK) return s;
    c->has_fixed = tr->fixed_node != nullptr;
    c->has_out_len = tr->out_len != nullptr;
    if (mem == LMX_DEVICE) {
        c->arrival.borrow(tr->arrival);
        c->lbk.borrow(tr->len_batch_kind);
        if (c->has_fixed) c->fixed.borrow(tr->fixed_node);
        if (c->has_out_len) c->out_len.borrow(tr->out_len);
    } else {
        if (c->has_out_len) {   // decode lengths (continuous batching): copied here, not streamed
            if (c->out_len.ensure(std::max<int64_t>(M, 1) * 4) != cudaSuccess)
                return c->fail(LMX_ENOMEM, "out_len allocation");
            if (M > 0) {
                s = c->cuda(cudaMemcpyAsync(c->out_len.p, tr->out_len, M * 4, cudaMemcpyHostToDevice, c->stream),
                            "out_len copy");
                if (s == LMX_OK) s = c->cuda(cudaStreamSynchronize(c->stream), "out_len copy");
                if (s != LMX_OK) return s;
            }
        }
        if (c->arrival.ensure(std::max<int64_t>(M, 1) * 8) != cudaSuccess ||
            c->lbk.ensure(std::max<int64_t>(M, 1) * 4) != cudaSuccess ||
            (c->has_fixed && c->fixed.ensure(std::max<int64_t>(M, 1) * 4) != cudaSuccess))
            return c->fail(LMX_ENOMEM, "trace buffers allocation (" + std::to_string(M) + " tasks)");
        if (M > 0 && c->has_fixed) {
            s = c->cuda(cudaMemcpyAsync(c->fixed.p, tr->fixed_node, M * 4, cudaMemcpyHostToDevice, c->stream),
                        "fixed_node copy");
            if (s != LMX_OK) return s;
        }
        // arrival / len_batch_kind are streamed by lmx_run, overlapped with the kernel
        c->h_arrival = tr->arrival;
        c->h_lbk = tr->len_batch_kind;
        c->host_pending = M > 0;
        (void)is_pinned;
    }
    if (mem == LMX_DEVICE) c->host_pending = false;
    c->n_traces = T;
    c->n_tasks = M;
    c->have_traces = true;
    c->ran = false;
    if (!c->cells_set) c->n_cells = 1;
    return LMX_OK;
}

lmx_status lmx_set_params(lmx_ctx *c, const lmx_params *p)
{
    if (!c) return LMX_EINVAL;
    if (!p) return c->fail(LMX_EINVAL, "lmx_set_params: NULL params");
    if (p->policy < LMX_LEMIX || p->policy > LMX_MIXLUF) return c->fail(LMX_EINVAL, "params.policy out of range");
    if (p->cb_cmax < 0 || p->cb_cmax > 4096) return c->fail(LMX_EINVAL, "params.cb_cmax must be in [0, 4096]");
    if (p->cb_cmax > 0 && !(p->cb_tw >= 0.0 && std::isfinite(p->cb_tw)))
        return c->fail(LMX_EINVAL, "params.cb_tw must be finite and >= 0");
    if (p->cb_cmax > 0 && p->mem_enable)
        return c->fail(LMX_EINVAL, "params.cb_cmax: continuous batching is not combined with mem_enable");
    if (p->eq4_mode != 0 && p->eq4_mode != 1) return c->fail(LMX_EINVAL, "params.eq4_mode must be 0 or 1");
    if (!(p->luf_delay >= 0.0 && std::isfinite(p->luf_delay)))
        return c->fail(LMX_EINVAL, "params.luf_delay must be finite and >= 0");
    if (p->deprioritize != 0 && p->deprioritize != 1) return c->fail(LMX_EINVAL, "params.deprioritize must be 0 or 1");
    if (p->slo_mode != 0 && p->slo_mode != 1) return c->fail(LMX_EINVAL, "params.slo_mode must be 0 or 1");
    if (p->qcap < 1 || p->qcap > 65536) return c->fail(LMX_EINVAL, "params.qcap must be in [1, 65536]");
    if (!(p->lambda1 > 0.0 && std::isfinite(p->lambda1))) return c->fail(LMX_EINVAL, "params.lambda1 must be finite and > 0");
    if (!(p->lambda2 >= 0.0 && std::isfinite(p->lambda2))) return c->fail(LMX_EINVAL, "params.lambda2 must be finite and >= 0");
    if (!std::isfinite(p->tau)) return c->fail(LMX_EINVAL, "params.tau must be finite");
    if (!(p->slo_mult >= 0.0 && std::isfinite(p->slo_mult))) return c->fail(LMX_EINVAL, "params.slo_mult must be finite and >= 0");
    if (!std::isfinite(p->slo_const)) return c->fail(LMX_EINVAL, "params.slo_const must be finite");
    if (!(p->sigma_floor > 0.0 && std::isfinite(p->sigma_floor))) return c->fail(LMX_EINVAL, "params.sigma_floor must be finite and > 0");
    if (!std::isfinite(p->lc0)) return c->fail(LMX_EINVAL, "params.lc0 must be finite");
    if (!(p->alpha >= 0.0 && p->alpha <= 1.0)) return c->fail(LMX_EINVAL, "params.alpha must be in [0, 1]");
    if (p->mem_enable != 0 && p->mem_enable != 1) return c->fail(LMX_EINVAL, "params.mem_enable must be 0 or 1");
    if (p->sync_interval < 0) return c->fail(LMX_EINVAL, "params.sync_interval must be >= 0");
    if (!(p->sync_latency >= 0.0 && std::isfinite(p->sync_latency)))
        return c->fail(LMX_EINVAL, "params.sync_latency must be finite and >= 0");
    if (p->sep_dynamic != 0 && p->sep_dynamic != 1) return c->fail(LMX_EINVAL, "params.sep_dynamic must be 0 or 1");
    if (p->sep_dynamic && !(p->dyn_rate >= 0.0 && std::isfinite(p->dyn_rate)))
        return c->fail(LMX_EINVAL, "params.dyn_rate must be finite and >= 0");
    if (p->sep_dynamic && !(p->dyn_window > 0.0 && std::isfinite(p->dyn_window)))
        return c->fail(LMX_EINVAL, "params.dyn_window must be finite and > 0");
    if (p->debug_level != 0 && p->debug_level != 1) return c->fail(LMX_EINVAL, "params.debug_level must be 0 or 1");
    if (p->mem_enable) {   // Algorithm 2: Delta_t > 0 and a finite T_max bound the wait loop
        if (p->mem_cap < 0) return c->fail(LMX_EINVAL, "params.mem_cap must be >= 0");
        if (!(p->mem_dt > 0.0 && std::isfinite(p->mem_dt))) return c->fail(LMX_EINVAL, "params.mem_dt must be finite and > 0");
        if (!(p->mem_tmax > 0.0 && std::isfinite(p->mem_tmax))) return c->fail(LMX_EINVAL, "params.mem_tmax must be finite and > 0");
        if (!(p->mem_pen >= 0.0 && std::isfinite(p->mem_pen))) return c->fail(LMX_EINVAL, "params.mem_pen must be finite and >= 0");
        if (p->mem_tmax / p->mem_dt > 1048576.0) return c->fail(LMX_EINVAL, "params.mem_tmax / mem_dt must be <= 2^20");
    }
    c->par = *p;
    c->have_params = true;
    c->ran = false;
    return LMX_OK;
}

lmx_status lmx_set_cells(lmx_ctx *c, const int32_t *cell_of, int32_t n_cells)
{
    if (!c) return LMX_EINVAL;
    if (!c->have_traces) return c->fail(LMX_ESTATE, "lmx_set_cells: load traces first");
    if (!cell_of || n_cells <= 1) {
        c->n_cells = 1;
        c->cells_set = false;
        c->cell_of.release();
        return LMX_OK;
    }
    if (n_cells > 65536) return c->fail(LMX_EINVAL, "n_cells must be <= 65536");
    for (int64_t t = 0; t < c->n_traces; ++t)
        if (cell_of[t] < 0 || cell_of[t] >= n_cells)
            return c->fail(LMX_EINVAL, "cell_of_trace[" + std::to_string(t) + "] out of range");
    // per-cell CSR: a counting sort of the traces by cell (stable), so the
    // reduction visits each cell's traces only, in trace order
    std::vector<int64_t> start((size_t)n_cells + 1, 0), order((size_t)std::max<int64_t>(c->n_traces, 1));
    for (int64_t t = 0; t < c->n_traces; ++t) start[(size_t)cell_of[t] + 1]++;
    for (int32_t q = 0; q < n_cells; ++q) start[(size_t)q + 1] += start[q];
    {
        std::vector<int64_t> fill(start.begin(), start.end() - 1);
        for (int64_t t = 0; t < c->n_traces; ++t) order[(size_t)fill[(size_t)cell_of[t]]++] = t;
    }
    cudaSetDevice(c->device);
    if (c->cell_of.ensure(std::max<int64_t>(c->n_traces, 1) * 4) != cudaSuccess ||
        c->cell_start.ensure(start.size() * 8) != cudaSuccess || c->cell_order.ensure(order.size() * 8) != cudaSuccess)
        return c->fail(LMX_ENOMEM, "cells");
    lmx_status s = c->cuda(cudaMemcpyAsync(c->cell_of.p, cell_of, c->n_traces * 4, cudaMemcpyHostToDevice, c->stream),
                           "cells copy");
    if (s == LMX_OK)
        s = c->cuda(cudaMemcpyAsync(c->cell_start.p, start.data(), start.size() * 8, cudaMemcpyHostToDevice, c->stream),
                    "cells copy");
    if (s == LMX_OK)
        s = c->cuda(cudaMemcpyAsync(c->cell_order.p, order.data(), order.size() * 8, cudaMemcpyHostToDevice, c->stream),
                    "cells copy");
    if (s != LMX_OK) return s;
    s = c->cuda(cudaStreamSynchronize(c->stream), "cells copy");
    if (s != LMX_OK) return s;
    c->n_cells = n_cells;
    c->cells_set = true;
    return LMX_OK;
}

lmx_status lmx_set_cell_params(lmx_ctx *c, int32_t n_cells, const double *l1, const double *l2, const double *tau)
{
    if (!c) return LMX_EINVAL;
    if (n_cells == 0) {
        c->n_cell_par = 0;
        c->cell_par.release();
        return LMX_OK;
    }
    if (!c->have_params) return c->fail(LMX_ESTATE, "lmx_set_cell_params: set params first");
    if (!c->cells_set || c->n_cells != n_cells)
        return c->fail(LMX_ESTATE, "lmx_set_cell_params: lmx_set_cells with the same n_cells first");
    std::vector<double> h((size_t)n_cells * 3);
    for (int32_t k = 0; k < n_cells; ++k) {
        const double a = l1 ? l1[k] : c->par.lambda1, b = l2 ? l2[k] : c->par.lambda2, t = tau ? tau[k] : c->par.tau;
        if (!(a > 0.0 && std::isfinite(a)) || !(b >= 0.0 && std::isfinite(b)) || !std::isfinite(t))
            return c->fail(LMX_EINVAL, "cell params[" + std::to_string(k) + "]: lambda1 > 0, lambda2 >= 0, tau finite");
        h[3 * k] = a;
        h[3 * k + 1] = b;
        h[3 * k + 2] = t;
    }
    cudaSetDevice(c->device);
    if (c->cell_par.ensure(h.size() * sizeof(double)) != cudaSuccess) return c->fail(LMX_ENOMEM, "cell params");
    lmx_status s = c->cuda(cudaMemcpyAsync(c->cell_par.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice,
                                           c->stream), "cell params copy");
    if (s == LMX_OK) s = c->cuda(cudaStreamSynchronize(c->stream), "cell params copy");
    if (s != LMX_OK) return s;
    c->n_cell_par = n_cells;
    return LMX_OK;
}

lmx_status lmx_set_outputs(lmx_ctx *c, int per_task)
{
    if (!c) return LMX_EINVAL;
    c->per_task = per_task ? 1 : 0;
    return LMX_OK;
}

lmx_status lmx_run(lmx_ctx *c)
{
    if (!c) return LMX_EINVAL;
    if (!c->have_profile || !c->have_traces || !c->have_params)
        return c->fail(LMX_ESTATE, "lmx_run: load profile, traces and params first");
    const lmx_params &P = c->par;
    if (P.policy == LMX_FIXED && !c->has_fixed)
        return c->fail(LMX_EINVAL, "policy LMX_FIXED needs traces.fixed_node");
    if (P.cb_cmax > 0 && !c->has_out_len)
        return c->fail(LMX_EINVAL, "continuous batching (params.cb_cmax > 0) needs traces.out_len");
    cudaSetDevice(c->device);
    const int64_t T = c->n_traces, M = c->n_tasks;

    lmx::KParams k{};
    k.N = c->N;
    k.S = c->S;
    int Tl = 1;
    while (Tl < c->N && Tl < 32) Tl <<= 1;
    if (const char *tl_env = getenv("LMX_TILE_LANES")) {   // developer override: lanes per trace
        const int want = atoi(tl_env);
        if (want >= 1 && want <= 32 && (want & (want - 1)) == 0 && (c->N + want - 1) / want <= 4) Tl = want;
    }
    k.T = Tl;
    k.log2T = 0;
    while ((1 << k.log2T) < Tl) k.log2T++;
    k.npl = (c->N + Tl - 1) / Tl;
    k.npad = lmx::npl_bucket(k.npl) * Tl;
    k.policy = P.policy;
    k.deprioritize = P.deprioritize;
    k.slo_mode = P.slo_mode;
    k.qcap = P.qcap;
    int K = 1;
    while (K < P.qcap) K <<= 1;
    k.kmask = K - 1;
    {
        // Separate's training partition, PAPER.md:795 (host fp64, no contraction)
        const double raw = std::floor((double)c->N * P.alpha + 0.5);
        int ntr = (int)raw;
        if (ntr < 1) ntr = 1;
        if (ntr > c->N - 1) ntr = c->N - 1;
        k.n_tr_sep = ntr < 1 ? 1 : ntr;
    }
    k.s_pow2 = (c->S & (c->S - 1)) == 0;
    k.inv_S = 1.0 / (double)c->S;
    k.lambda1 = P.lambda1;
    k.lambda2 = P.lambda2;
    k.tau = P.tau;
    k.slo_mult = P.slo_mult;
    k.slo_const = P.slo_const;
    k.sigma_floor = P.sigma_floor;
    k.lc0 = P.lc0;
    k.mem_enable = P.mem_enable;
    k.mem_cap = P.mem_cap;
    k.mem_dt = P.mem_dt;
    k.mem_tmax = P.mem_tmax;
    k.mem_pen = P.mem_pen;
    k.sync_sep = (P.policy == LMX_SEPARATE && P.sync_interval > 0) ? 1 : 0;
    k.sync_interval = P.sync_interval > 0 ? P.sync_interval : 1;
    k.sync_latency = P.sync_latency;
    k.sep_dynamic = (P.policy == LMX_SEPARATE && P.sep_dynamic) ? 1 : 0;
    k.dyn_rate = P.dyn_rate;
    k.dyn_window = P.dyn_window;
    k.cb_cmax = P.cb_cmax;
    k.cb_tw = P.cb_tw;
    k.eq4_mode = P.eq4_mode;
    k.luf_delay = P.luf_delay;
    k.out_len = c->has_out_len ? (const uint32_t *)c->out_len.p : nullptr;
    if (c->n_cell_par > 0) {
        if (!c->cells_set || c->n_cells != c->n_cell_par)
            return c->fail(LMX_ESTATE, "lmx_run: cell params need lmx_set_cells with the same n_cells");
        k.cell_par = (const double *)c->cell_par.p;
        k.cell_of = (const int32_t *)c->cell_of.p;
    }
    k.n_traces = T;
    k.offsets = (const int64_t *)c->offsets.p;
    k.n_inf = (const int32_t *)c->n_inf.p;
    k.arrival = (const double *)c->arrival.p;
    k.lbk = (const uint32_t *)c->lbk.p;
    k.fixed = c->has_fixed ? (const int32_t *)c->fixed.p : nullptr;
    k.eta = (const double *)c->eta.p;

    k.want_outputs = c->per_task;
    k.want_cand = P.debug_level == 1;
    // geometry: persistent grid = resident CTAs, capped by the number of traces
    int occ_err = 0;
    const int per_sm = lmx::event_loop_occupancy(k, &occ_err);
    if (occ_err != 0 || per_sm < 1)
        return c->fail(LMX_ECUDA, std::string("event loop occupancy query failed: ") +
                                      cudaGetErrorString((cudaError_t)occ_err));
    int n_sm = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, c->device);
    const int block = lmx::event_loop_block_threads(k);
    const int tiles_per_block = lmx::event_loop_traces_per_block(k);
    int64_t grid = (int64_t)n_sm * per_sm;
    const int64_t need = (T + tiles_per_block - 1) / tiles_per_block;
    grid = std::max<int64_t>(1, std::min(grid, need));
    const int64_t tiles = grid * tiles_per_block;

    // device buffers
    const size_t ring_entries = (size_t)tiles * k.npad * K;
    if (c->ring_be.ensure(ring_entries * lmx::ring_words(c->S, P.mem_enable != 0) * sizeof(double2)) != cudaSuccess)
        return c->fail(LMX_ENOMEM, "queue ring allocation (" + std::to_string(ring_entries) + " entries; lower qcap)");
    if (k.sync_sep) {   // checkpoint list per tile slot: at most max_train / interval entries
        int64_t max_train = 0;
        for (int64_t t = 0; t < T; ++t)
            max_train = std::max<int64_t>(max_train, c->h_offsets[t + 1] - c->h_offsets[t] - c->h_n_inf[t]);
        const int64_t cap = max_train / k.sync_interval + 1;
        if (cap > INT32_MAX || c->ck.ensure((size_t)tiles * cap * sizeof(double)) != cudaSuccess)
            return c->fail(LMX_ENOMEM, "checkpoint list allocation");
        k.ck = (double *)c->ck.p;
        k.ck_cap = (int32_t)cap;
    }
    if (c->summaries.ensure(std::max<int64_t>(T, 1) * sizeof(lmx_summary)) != cudaSuccess ||
        c->trace_err.ensure(std::max<int64_t>(T, 1) * 8) != cudaSuccess ||
        c->cell_i.ensure((size_t)c->n_cells * LMX_CELL_NI * 8) != cudaSuccess ||
        c->cell_f.ensure((size_t)c->n_cells * LMX_CELL_NF * 8) != cudaSuccess)
        return c->fail(LMX_ENOMEM, "summary allocation");
    if (c->per_task) {
        if (c->node_defer.ensure(std::max<int64_t>(M, 1) * 4) != cudaSuccess ||
            c->decision_idx.ensure(std::max<int64_t>(M, 1) * 4) != cudaSuccess ||
            c->completion.ensure(std::max<int64_t>(M, 1) * 8) != cudaSuccess ||
            c->start_f1.ensure(std::max<int64_t>(M, 1) * 8) != cudaSuccess)
            return c->fail(LMX_ENOMEM, "per-task output allocation");
        k.node_defer = (uint32_t *)c->node_defer.p;
        k.decision_idx = (int32_t *)c->decision_idx.p;
        k.completion = (double *)c->completion.p;
        k.start_f1 = (double *)c->start_f1.p;
        // tasks a failed trace never decides keep defined sentinels (node/defer
        // all ones, decision -1, NaN times) instead of stale memory
        if (M > 0) {
            lmx_status s0 = c->cuda(cudaMemsetAsync(c->node_defer.p, 0xFF, M * 4, c->stream), "output init");
            if (s0 == LMX_OK) s0 = c->cuda(cudaMemsetAsync(c->decision_idx.p, 0xFF, M * 4, c->stream), "output init");
            if (s0 == LMX_OK) s0 = c->cuda(cudaMemsetAsync(c->completion.p, 0xFF, M * 8, c->stream), "output init");
            if (s0 == LMX_OK) s0 = c->cuda(cudaMemsetAsync(c->start_f1.p, 0xFF, M * 8, c->stream), "output init");
            if (s0 != LMX_OK) return s0;
        }
    }
    c->cand_valid = false;
    if (P.debug_level == 1) {
        const size_t nc = (size_t)std::max<int64_t>(M, 1) * c->N * 3;
        if (c->cand.ensure(nc * 8) != cudaSuccess) return c->fail(LMX_ENOMEM, "debug candidate output allocation");
        lmx_status s0 = c->cuda(cudaMemsetAsync(c->cand.p, 0xFF, nc * 8, c->stream), "debug output init");
        if (s0 != LMX_OK) return s0;
        k.cand = (double *)c->cand.p;
        c->cand_valid = true;
    }
    k.summaries = (lmx_summary *)c->summaries.p;
    k.trace_err = (int64_t *)c->trace_err.p;
    k.work = (unsigned long long *)c->work.p;
    k.first_bad = (unsigned long long *)c->first_bad.p;
    k.ring_be = (double2 *)c->ring_be.p;

    lmx_status s = c->cuda(cudaMemsetAsync(c->work.p, 0, 8, c->stream), "reset");
    if (s == LMX_OK) s = c->cuda(cudaMemsetAsync(c->first_bad.p, 0xFF, 8, c->stream), "reset");
    if (s != LMX_OK) return s;

    // streamed inputs: 2^22-task chunks (a multiple of 32 tasks, so chunk
    // boundaries are 128-byte aligned in both arrays and no cache line mixes
    // landed and in-flight data)
    const bool stream_in = c->host_pending;
    const int64_t chunk = int64_t(1) << 22;
    const int64_t n_chunks = stream_in ? (M + chunk - 1) / chunk : 0;
    if (stream_in) {
        if (c->ready.ensure(4) != cudaSuccess) return c->fail(LMX_ENOMEM, "ready flag");
        if (c->h_seq_len < n_chunks) {
            if (c->h_seq) cudaFreeHost(c->h_seq);
            c->h_seq = nullptr;
            c->h_seq_len = 0;
            if (cudaMallocHost(&c->h_seq, n_chunks * sizeof(unsigned)) != cudaSuccess)
                return c->fail(LMX_ENOMEM, "pinned chunk sequence");
            for (int64_t q = 0; q < n_chunks; ++q) c->h_seq[q] = (unsigned)(q + 1);
            c->h_seq_len = n_chunks;
        }
        s = c->cuda(cudaMemsetAsync(c->ready.p, 0, 4, c->stream), "ready reset");
        if (s != LMX_OK) return s;
        cudaEventRecord(c->ev_armed, c->stream);
        k.ready = (const unsigned *)c->ready.p;
        k.chunk_tasks = chunk;
        // Every copy is enqueued BEFORE the kernel that waits on them: the
        // copies run on a non-blocking stream while the kernel consumes the
        // chunks that have landed, and an execution that serialises the two
        // streams (ncu kernel replay, CUDA_DEVICE_MAX_CONNECTIONS=1) runs the
        // copies first instead of spinning forever.  A failed enqueue returns
        // here, before anything waits on the flag.
        cudaStreamWaitEvent(c->copy_stream, c->ev_armed, 0);
        for (int64_t q = 0; q < n_chunks && s == LMX_OK; ++q) {
            const int64_t b = q * chunk, e = std::min(M, b + chunk);
            s = c->cuda(cudaMemcpyAsync((double *)c->arrival.p + b, c->h_arrival + b, (e - b) * 8,
                                        cudaMemcpyHostToDevice, c->copy_stream), "arrival copy");
            if (s == LMX_OK)
                s = c->cuda(cudaMemcpyAsync((uint32_t *)c->lbk.p + b, c->h_lbk + b, (e - b) * 4,
                                            cudaMemcpyHostToDevice, c->copy_stream), "len_batch_kind copy");
            if (s == LMX_OK)
                s = c->cuda(cudaMemcpyAsync(c->ready.p, c->h_seq + q, 4, cudaMemcpyHostToDevice, c->copy_stream),
                            "ready flag");
        }
        if (s != LMX_OK) {
            cudaStreamSynchronize(c->copy_stream);
            return s;
        }
        cudaEventRecord(c->ev_copied, c->copy_stream);
    }
    c->launches = 0;
    cudaEventRecord(c->ev0, c->stream);
    if (T > 0) {
        int e = lmx::launch_event_loop(k, (int)grid, c->stream);
        if (e != 0) {
            if (stream_in) cudaStreamSynchronize(c->copy_stream);
            return c->cuda((cudaError_t)e, "event loop launch");
        }
        c->launches++;
    }
    cudaEventRecord(c->ev1, c->stream);
    if (stream_in) {
        // the context stream (cell reduction, later runs) waits for the copies
        cudaStreamWaitEvent(c->stream, c->ev_copied, 0);
        c->host_pending = false;   // the data now lives in the context's buffers
    }

    lmx::CellParams cp{};
    cp.n_traces = T;
    cp.n_cells = c->n_cells;
    cp.cell_start = c->cells_set ? (const int64_t *)c->cell_start.p : nullptr;
    cp.order = c->cells_set ? (const int64_t *)c->cell_order.p : nullptr;
    cp.summaries = (const lmx_summary *)c->summaries.p;
    cp.cell_i = (int64_t *)c->cell_i.p;
    cp.cell_f = (double *)c->cell_f.p;
    int e = lmx::launch_cells(cp, c->stream);
    if (e != 0) return c->cuda((cudaError_t)e, "cell reduction launch");
    c->launches++;
    cudaEventRecord(c->ev2, c->stream);

    c->grid = (int32_t)grid;
    c->block = block;
    c->lanes = k.T;
    c->smem = lmx::event_loop_smem_bytes(k);
    c->ran = true;
    c->synced = false;
    return LMX_OK;
}

lmx_status lmx_sync(lmx_ctx *c)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran) return c->fail(LMX_ESTATE, "lmx_sync: nothing was run");
    cudaSetDevice(c->device);
    lmx_status s = c->cuda(cudaStreamSynchronize(c->stream), "lmx_run");
    if (s != LMX_OK) return s;
    c->synced = true;
    unsigned long long bad = ~0ull;
    s = c->cuda(cudaMemcpy(&bad, c->first_bad.p, 8, cudaMemcpyDeviceToHost), "status read");
    if (s != LMX_OK) return s;
    if (bad == ~0ull) return LMX_OK;
    lmx_summary sm;
    int64_t info = 0;
    cudaMemcpy(&sm, (lmx_summary *)c->summaries.p + bad, sizeof sm, cudaMemcpyDeviceToHost);
    cudaMemcpy(&info, (int64_t *)c->trace_err.p + bad, 8, cudaMemcpyDeviceToHost);
    const int64_t task = info >> 8;
    const int code = (int)(info & 0xFF);
    char buf[512];
    if (sm.status == LMX_EINVAL)
        snprintf(buf, sizeof buf, "trace %llu, task %lld: invalid %s", (unsigned long long)bad, (long long)task,
                 field_name(code));
    else if (sm.status == LMX_EQCAP)
        snprintf(buf, sizeof buf, "trace %llu: a node's training queue exceeded params.qcap = %d", (unsigned long long)bad,
                 c->par.qcap);
    else
        snprintf(buf, sizeof buf, "trace %llu: decision budget exhausted", (unsigned long long)bad);
    c->err = buf;
    return (lmx_status)sm.status;
}

static lmx_status copy_out(lmx_ctx *c, void *dst, const DevBuf &src, size_t bytes, lmx_mem mem, const char *what)
{
    if (!dst || bytes == 0) return LMX_OK;
    return c->cuda(cudaMemcpy(dst, src.p, bytes, mem == LMX_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost),
                   what);
}

lmx_status lmx_get_assignments(lmx_ctx *c, uint32_t *node_defer, int32_t *decision_idx, lmx_mem mem)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran || !c->synced) return c->fail(LMX_ESTATE, "lmx_get_assignments: run and sync first");
    if (!c->per_task) return c->fail(LMX_ESTATE, "per-task outputs are off (lmx_set_outputs)");
    cudaSetDevice(c->device);
    lmx_status s = copy_out(c, node_defer, c->node_defer, c->n_tasks * 4, mem, "node_defer copy");
    if (s == LMX_OK) s = copy_out(c, decision_idx, c->decision_idx, c->n_tasks * 4, mem, "decision_idx copy");
    return s;
}

lmx_status lmx_get_times(lmx_ctx *c, double *completion, double *start_f1, lmx_mem mem)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran || !c->synced) return c->fail(LMX_ESTATE, "lmx_get_times: run and sync first");
    if (!c->per_task) return c->fail(LMX_ESTATE, "per-task outputs are off (lmx_set_outputs)");
    cudaSetDevice(c->device);
    lmx_status s = copy_out(c, completion, c->completion, c->n_tasks * 8, mem, "completion copy");
    if (s == LMX_OK) s = copy_out(c, start_f1, c->start_f1, c->n_tasks * 8, mem, "start_f1 copy");
    return s;
}

lmx_status lmx_get_candidates(lmx_ctx *c, double *cand, lmx_mem mem)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran || !c->synced) return c->fail(LMX_ESTATE, "lmx_get_candidates: run and sync first");
    if (!c->cand_valid) return c->fail(LMX_ESTATE, "lmx_get_candidates: the last run had debug_level 0");
    cudaSetDevice(c->device);
    return copy_out(c, cand, c->cand, (size_t)c->n_tasks * c->N * 3 * 8, mem, "candidate copy");
}

lmx_status lmx_get_summaries(lmx_ctx *c, lmx_summary *per_trace)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran || !c->synced) return c->fail(LMX_ESTATE, "lmx_get_summaries: run and sync first");
    cudaSetDevice(c->device);
    return copy_out(c, per_trace, c->summaries, c->n_traces * sizeof(lmx_summary), LMX_HOST, "summary copy");
}

lmx_status lmx_get_cells(lmx_ctx *c, lmx_cell_summary *cells)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran) return c->fail(LMX_ESTATE, "lmx_get_cells: run first");
    if (!cells) return c->fail(LMX_EINVAL, "lmx_get_cells: NULL output");
    cudaSetDevice(c->device);
    std::vector<int64_t> hi((size_t)c->n_cells * LMX_CELL_NI);
    std::vector<double> hf((size_t)c->n_cells * LMX_CELL_NF);
    lmx_status s = c->cuda(cudaMemcpyAsync(hi.data(), c->cell_i.p, hi.size() * 8, cudaMemcpyDeviceToHost, c->stream),
                           "cell copy");
    if (s == LMX_OK)
        s = c->cuda(cudaMemcpyAsync(hf.data(), c->cell_f.p, hf.size() * 8, cudaMemcpyDeviceToHost, c->stream),
                    "cell copy");
    if (s == LMX_OK) s = c->cuda(cudaStreamSynchronize(c->stream), "cell copy");
    if (s != LMX_OK) return s;
    for (int32_t q = 0; q < c->n_cells; ++q) {
        int64_t *I = &hi[(size_t)q * LMX_CELL_NI];
        double *F = &hf[(size_t)q * LMX_CELL_NF];
        lmx_cell_summary &o = cells[q];
        o.n_traces = I[0]; o.n_failed = I[1]; o.n_tasks = I[2]; o.n_inf = I[3]; o.n_train = I[4];
        o.n_slo_met = I[5]; o.n_deferrals = I[6]; o.sum_active_nodes = I[7]; o.sum_version = I[8];
        o.sum_makespan = F[0]; o.sum_throughput = F[1]; o.sum_ttft = F[2]; o.sum_mean_ttft = F[3];
        o.sum_slo_attainment = F[4]; o.sum_mean_util = F[5]; o.sum_mean_len_std = F[6];
    }
    return LMX_OK;
}

lmx_status lmx_allreduce_cells(lmx_ctx *c, void *comm)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran) return c->fail(LMX_ESTATE, "lmx_allreduce_cells: run first");
    if (!comm) return c->fail(LMX_EINVAL, "lmx_allreduce_cells: NULL communicator");
    if (!g_nccl.load()) return c->fail(LMX_ENCCL, "libnccl.so.2 not found");
    cudaSetDevice(c->device);
    int r = g_nccl.group_start();
    if (r == 0) r = g_nccl.all_reduce(c->cell_i.p, c->cell_i.p, (size_t)c->n_cells * LMX_CELL_NI, kNcclInt64, kNcclSum,
                                      comm, c->stream);
    if (r == 0) r = g_nccl.all_reduce(c->cell_f.p, c->cell_f.p, (size_t)c->n_cells * LMX_CELL_NF, kNcclFloat64,
                                      kNcclSum, comm, c->stream);
    int r2 = g_nccl.group_end();
    if (r != 0 || r2 != 0) return c->fail(LMX_ENCCL, "ncclAllReduce failed (" + std::to_string(r ? r : r2) + ")");
    return LMX_OK;
}

lmx_status lmx_nccl_unique_id(void *id128)
{
    if (!id128) return LMX_EINVAL;
    if (!g_nccl.load()) return LMX_ENCCL;
    return g_nccl.get_unique_id(id128) == 0 ? LMX_OK : LMX_ENCCL;
}

lmx_status lmx_nccl_comm_init(void **comm, int nranks, const void *id128, int rank, int device)
{
    if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return LMX_EINVAL;
    if (!g_nccl.load()) return LMX_ENCCL;
    if (cudaSetDevice(device) != cudaSuccess) return LMX_ECUDA;
    NcclId128 id;
    std::memcpy(id.internal, id128, 128);
    return g_nccl.comm_init_rank(comm, nranks, id, rank) == 0 ? LMX_OK : LMX_ENCCL;
}

lmx_status lmx_nccl_comm_destroy(void *comm)
{
    if (!comm) return LMX_OK;
    if (!g_nccl.load()) return LMX_ENCCL;
    return g_nccl.comm_destroy(comm) == 0 ? LMX_OK : LMX_ENCCL;
}

lmx_status lmx_get_timing(lmx_ctx *c, float *kernel_ms, float *run_ms, int32_t *launches)
{
    if (!c) return LMX_EINVAL;
    if (!c->ran || !c->synced) return c->fail(LMX_ESTATE, "lmx_get_timing: run and sync first");
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, c->ev0, c->ev1);
    cudaEventElapsedTime(&b, c->ev0, c->ev2);
    if (kernel_ms) *kernel_ms = a;
    if (run_ms) *run_ms = b;
    if (launches) *launches = c->launches;
    return LMX_OK;
}

lmx_status lmx_get_geometry(lmx_ctx *c, int32_t *grid, int32_t *block, int32_t *lanes, int32_t *smem)
{
    if (!c) return LMX_EINVAL;
    if (grid) *grid = c->grid;
    if (block) *block = c->block;
    if (lanes) *lanes = c->lanes;
    if (smem) *smem = c->smem;
    return LMX_OK;
}

}  // extern "C"
