/*
 * lemix.h -- C ABI of the B200-native LeMix placement-step library (liblemix.so).
 *
 * What it computes (arXiv 2507.21276, /root/reference/PAPER.md):
 *   For every decision of a discrete-event loop over independent synthetic
 *   traces, the pending task (an inference request or a training micro-batch)
 *   is planned on every node with Algorithm 1 ComputeIdleness (PAPER.md:432-476,
 *   §4.2) giving the idleness increase II and response time R, scored with
 *   Eq. 1 (idleness profit), Eq. 2 (length consistency,
 *   PAPER.md:555) and Eq. 3 (node priority f), and committed to
 *   the node with the highest f; training tasks are first
 *   checked against Eq. 4 queue-level deprioritisation.  The
 *   Separate / NaiveMix (round-robin) baselines and a fixed
 *   assignment run the same planner on their chosen node.  The exact
 *   semantics, the readings of garbled passages and the canonical fp64
 *   expression forms are in DESIGN.md; results are bit-identical to the CPU
 *   oracle in oracle/.
 *
 * Conventions
 *   - Ownership: the caller owns every buffer it passes.  lmx_load_* copy what
 *     they need unless stated otherwise; outputs are copied into
 *     caller-allocated arrays.
 *   - Sequencing: create -> load_profile -> load_traces -> set_params -> run
 *     -> sync -> get_*.  Profile/traces/params may be re-loaded between runs.
 *     A call out of order returns LMX_ESTATE.
 *   - Errors: every call returns an lmx_status; lmx_last_error() gives a
 *     message naming the offending field, trace and task index.
 *   - Asynchrony: lmx_run enqueues on the context's CUDA stream and returns;
 *     lmx_sync waits and returns the first per-trace error (LMX_OK if none).
 *   - Determinism: per-trace outputs, per-trace summaries and the per-cell
 *     aggregates of one rank are a pure function of (profile, traces, params)
 *     and the cell map; they do not depend on the launch geometry or the
 *     order in which traces are scheduled on the device (each cell is folded
 *     over its own traces in trace order).  After lmx_allreduce_cells the
 *     integer cell fields are exact, but the fp64 cell sums depend on how the
 *     traces are split across ranks and on NCCL's reduction order (they agree
 *     within 1e-12 relative, not bit for bit).
 *   - Not thread-safe: one context per thread / GPU.
 */
#ifndef LEMIX_H
#define LEMIX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lmx_ctx lmx_ctx;   /* opaque; owns device buffers on one GPU */

typedef enum {
    LMX_OK = 0,
    LMX_EINVAL = 1,   /* invalid argument or input data (field/trace/task in lmx_last_error) */
    LMX_ESTATE = 2,   /* call out of sequence */
    LMX_ENOMEM = 3,   /* device or pinned allocation failed */
    LMX_ECUDA = 4,    /* CUDA runtime error */
    LMX_ENCCL = 5,    /* NCCL unavailable or failed */
    LMX_EQCAP = 6,    /* per trace: a node's training queue Q_train^n exceeded params.qcap */
    LMX_EBUDGET = 7,  /* per trace: decision budget exhausted (cannot happen for valid input) */
    LMX_ETIMEOUT = 8  /* per trace: streamed host inputs did not land within 60 s (a copy never completed) */
} lmx_status;

/* LMX_MIXLUF: the Mix-LUF comparison system (DESIGN.md
 * R-luf): the node with the least busy time committed so far (lowest
 * average utilisation; ties -> lowest index), each decision dispatched after
 * a serialised utilisation query of params.luf_delay seconds. */
typedef enum { LMX_LEMIX = 0, LMX_RR = 1, LMX_SEPARATE = 2, LMX_FIXED = 3, LMX_MIXLUF = 4 } lmx_policy;
typedef enum { LMX_HOST = 0, LMX_DEVICE = 1 } lmx_mem;

/* Profile table (offline profiling, §4.1): stage latencies
 * Δ_F = eta_f·C·ℓ², Δ_B = eta_b·C·ℓ².  Host memory, node-major
 * [n_nodes * n_stages], every value finite and > 0.  1 <= n_nodes <= 128,
 * 1 <= n_stages <= 16.  eta_d (may be NULL = 0): seconds per context token
 * per item of one decode step on that GPU (continuous batching
 * only), finite and >= 0.  Copied. */
typedef struct {
    int32_t n_nodes;
    int32_t n_stages;
    const double *eta_f;
    const double *eta_b;
    const double *eta_d;
} lmx_profile;

/* Task packing of len_batch_kind: query length ℓ in bits 0-11 (1..2048),
 * batch size C in bits 12-19 (1..255), kind in bit 20 (0 inference,
 * 1 training), bits 21-31 zero. */
#define LMX_PACK(l, C, kind) ((uint32_t)(l) | ((uint32_t)(C) << 12) | ((uint32_t)(kind) << 20))

/* A CSR batch of independent traces.
 *   offsets[n_traces+1] (HOST memory): trace t owns tasks [offsets[t], offsets[t+1]),
 *     offsets[0] == 0, non-decreasing, at most 2^19 tasks per trace.
 *   n_inf[n_traces] (HOST memory): the first n_inf[t] tasks of trace t are
 *     inference tasks in non-decreasing arrival order, the rest are training
 *     tasks in release order.
 *   arrival[n_tasks]: inference arrival time, or a training task's earliest
 *     release a_min (seconds, finite, >= 0).
 *   len_batch_kind[n_tasks]: LMX_PACK; the kind bit must match the position.
 *   fixed_node[n_tasks]: node per task for LMX_FIXED, else may be NULL.
 * The task arrays live in the memory named by the lmx_mem argument of
 * lmx_load_traces.  Per-task field errors are detected on the device during
 * lmx_run and reported per trace (status LMX_EINVAL). */
typedef struct {
    int64_t n_traces;
    const int64_t *offsets;
    const int32_t *n_inf;
    const double *arrival;
    const uint32_t *len_batch_kind;
    const int32_t *fixed_node;
    /* out_len[n_tasks]: decode steps of an inference request (tokens after
     * the prefill's first, 0..2048).  Read only with continuous
     * batching (params.cb_cmax > 0), else may be NULL.  Same memory kind as
     * arrival. */
    const uint32_t *out_len;
} lmx_traces;

/* Scheduler parameters.  lmx_params_default() fills the DESIGN.md defaults:
 * LeMix, λ1 = λ2 = 1, τ = 0, slo_mult = 5, σ_floor = 1,
 * lc0 = 0, α = 0.5, deprioritise on, per-task τ_R, qcap = 512. */
typedef struct {
    int32_t policy;        /* lmx_policy */
    int32_t deprioritize;  /* 1: Eq. 4 on (LeMix only); 0: the "w/o prioritize" ablation */
    int32_t slo_mode;      /* 0: τ_R = slo_mult · Σ_s η_F^{0,s}·C·ℓ²; 1: τ_R = slo_const */
    int32_t qcap;          /* capacity of each Q_train^n (1..65536); overflow -> LMX_EQCAP */
    double lambda1;        /* Eq. 3, > 0 */
    double lambda2;        /* Eq. 3, >= 0 */
    double tau;            /* Eq. 1 threshold */
    double slo_mult;       /* >= 0 */
    double slo_const;      /* seconds, slo_mode 1 */
    double sigma_floor;    /* Eq. 2 σ floor, > 0 */
    double lc0;            /* Eq. 2 value for nodes with < 2 tasks of history */
    double alpha;          /* Separate: N_train = clamp(floor(N·α + 0.5), 1, N-1), α in [0, 1] */
    /* Algorithm 2 ExecuteTaskMemoryAware (DESIGN.md R-mem;
     * SURVEY.md §8f NEXT-1).  0 (default): unlimited memory -- the executed
     * path is Algorithm 1's plan.  1: before each stage forward the committed
     * task waits in mem_dt steps until the activation tokens (C·ℓ) held on
     * that GPU by queued training tasks plus its own fit in mem_cap; once the
     * wait reaches mem_tmax its activations are offloaded (forward longer by
     * mem_pen s per token) and it runs; the executed path replaces the plan
     * (calibration).  Invalid values (mem_cap < 0, mem_dt <= 0, mem_tmax not
     * finite and > 0, mem_tmax / mem_dt > 2^20, mem_pen < 0) -> LMX_EINVAL. */
    int32_t mem_enable;
    int32_t mem_pad;       /* zero */
    int64_t mem_cap;       /* M_threshold per stage GPU, in activation tokens (C·ℓ units) */
    double mem_dt;         /* check interval Δ_t, seconds */
    double mem_tmax;       /* maximum wait T_max, seconds */
    double mem_pen;        /* offload penalty, seconds per offloaded token */
    /* Separate's model synchronisation (DESIGN.md R-sync;
     * SURVEY.md §8f NEXT-3): with policy LMX_SEPARATE and sync_interval > 0,
     * a checkpoint is taken when every sync_interval-th training task (release
     * order) ends its backward and is loaded on the inference nodes
     * sync_latency seconds later; an inference task's version (summary
     * sum_version) is the training count of the newest checkpoint loaded by
     * its forward start.  0 (default): the co-located proxy (node's finished
     * training tasks) for every policy.  sync_interval < 0 or sync_latency not
     * finite and >= 0 -> LMX_EINVAL. */
    int32_t sync_interval;
    int32_t sync_pad;      /* zero */
    double sync_latency;   /* seconds */
    /* SeparateDynamic (DESIGN.md R-sepdyn; NEXT-3): with policy
     * LMX_SEPARATE and sep_dynamic = 1 the partition follows the inference
     * request rate over (now - dyn_window, now]: below dyn_rate requests/s
     * max(1, N/4) inference nodes ("1-3" at N = 4), otherwise the alpha
     * partition ("2-2").  dyn_rate not finite and >= 0 or dyn_window not
     * finite and > 0 (when enabled) -> LMX_EINVAL. */
    int32_t sep_dynamic;
    int32_t sep_pad;       /* zero */
    double dyn_rate;       /* requests/s (50 in the paper) */
    double dyn_window;     /* seconds */
    /* Stepwise debug output: 0 none (default); 1 keep, for
     * every decision and every node, Algorithm 1's II and R (PAPER.md:474,
     * line 20) and Eq. 3's f -- see lmx_get_candidates.
     * Costs 24·N bytes per task of device memory and the writes.  Any other
     * value -> LMX_EINVAL. */
    int32_t debug_level;
    int32_t debug_pad;     /* zero */
    /* Algorithm 3 ContinuousBatching with hybrid prefill/decode (PAPER.md:
     * 689-727; DESIGN.md R-cb).  cb_cmax = 0 (default):
     * every request is placed on its own.  cb_cmax = C >= 1: inference
     * requests are grouped FCFS into batches of up to C (a batch waits at
     * most cb_tw seconds after its first request and stops at a released
     * training task); a batch is placed as one task (C = its members' total,
     * l = the longest, padded) whose decode steps then run on the same node
     * (eta_d); per request TTFT and TBT are reported.  Not
     * combined with mem_enable (-> LMX_EINVAL). */
    int32_t cb_cmax;
    /* Eq. 4 reading: 0 = R-14 (the node's latest forward end), 1 = R-14b
     * (also counting the training task's own forward).  DESIGN.md. */
    int32_t eq4_mode;
    double cb_tw;          /* T_w seconds, finite and >= 0 */
    double luf_delay;      /* LMX_MIXLUF: scheduler latency per decision, seconds (>= 0) */
} lmx_params;

/* Per-trace summary (metrics of PAPER.md:786-790).  For a trace whose status
 * is not LMX_OK only n_tasks, n_inf, n_train and status are set. */
typedef struct {
    int64_t n_tasks, n_inf, n_train;
    int64_t n_slo_met;      /* inference tasks with TTFT <= τ_R */
    int64_t n_deferrals;    /* Eq. 4 deferrals */
    int64_t active_nodes;   /* nodes that ran >= 1 task (consolidation) */
    int64_t sum_version;    /* Σ over inference tasks of the node's completed-training count */
    int64_t status;         /* lmx_status of this trace */
    int64_t n_mem_wait;     /* Algorithm 2: stage forwards that waited for memory */
    int64_t n_offload;      /* Algorithm 2: stage forwards whose activations were offloaded */
    int64_t n_batches;      /* Algorithm 3: inference batches placed (cb_cmax > 0), else 0 */
    int64_t n_tbt;          /* Algorithm 3: requests with >= 1 decode step (TBT defined) */
    double makespan;        /* last completion - first arrival */
    double throughput;      /* tasks / makespan */
    double sum_ttft, mean_ttft;
    double slo_attainment;  /* n_slo_met / n_inf (1.0 when n_inf == 0) */
    double mean_util;       /* Σ busy / (N·S·makespan) */
    double mean_len_std;    /* mean over active nodes of the population σ of lengths */
    double sum_tbt, mean_tbt;   /* time-between-tokens: per request, the mean gap
                                   between its tokens; summed / averaged over requests */
} lmx_summary;

/* Aggregate of the per-trace summaries of one cell (e.g. one (rate, policy)
 * point of a sweep); the "sum_*" fields add the per-trace value over the
 * cell's LMX_OK traces.  Reduced across ranks by lmx_allreduce_cells. */
typedef struct {
    int64_t n_traces, n_failed, n_tasks, n_inf, n_train, n_slo_met, n_deferrals,
            sum_active_nodes, sum_version;
    double sum_makespan, sum_throughput, sum_ttft, sum_mean_ttft, sum_slo_attainment,
           sum_mean_util, sum_mean_len_std;
} lmx_cell_summary;

#define LMX_CELL_NI 9
#define LMX_CELL_NF 7

void lmx_params_default(lmx_params *p);

/* Create a context on CUDA device `device`; work is enqueued on `cuda_stream`
 * (a cudaStream_t, NULL = a stream owned by the context). */
lmx_status lmx_create(lmx_ctx **out, int device, void *cuda_stream);
void lmx_destroy(lmx_ctx *ctx);
const char *lmx_last_error(const lmx_ctx *ctx);

lmx_status lmx_load_profile(lmx_ctx *ctx, const lmx_profile *profile);

/* HOST: the task arrays are host memory (pinned for full overlap) borrowed
 * until the next lmx_sync; lmx_run streams them into device buffers owned by
 * the context on a second stream, in 2^22-task chunks, while the kernel
 * already consumes the chunks that have landed (later runs reuse the copy).
 * DEVICE: the task arrays are borrowed device pointers and must stay valid
 * until the next lmx_sync.  offsets and n_inf are always host memory and are
 * copied. */
lmx_status lmx_load_traces(lmx_ctx *ctx, const lmx_traces *traces, lmx_mem mem);

lmx_status lmx_set_params(lmx_ctx *ctx, const lmx_params *params);

/* Optional: group traces into cells for lmx_get_cells (host memory,
 * cell_of_trace[n_traces] in [0, n_cells)).  NULL / 1 = one cell. */
lmx_status lmx_set_cells(lmx_ctx *ctx, const int32_t *cell_of_trace, int32_t n_cells);

/* Optional (after lmx_set_cells with the same n_cells): per-cell values of
 * Eq. 3's λ1, λ2 and Eq. 1's τ (host arrays [n_cells]; a NULL array keeps the
 * lmx_params value), so one run sweeps the parameter study of PAPER.md
 * Fig. 15.  n_cells = 0 clears them.  Values are
 * validated like lmx_set_params (λ1 > 0, λ2 >= 0, finite) -> LMX_EINVAL;
 * without matching cells -> LMX_ESTATE.  LeMix on the tile kernel only. */
lmx_status lmx_set_cell_params(lmx_ctx *ctx, int32_t n_cells, const double *lambda1, const double *lambda2,
                               const double *tau);

/* Optional: keep per-task outputs (default on).  Off = summary-only runs. */
lmx_status lmx_set_outputs(lmx_ctx *ctx, int per_task);

/* Run every trace and reduce the per-cell summaries; asynchronous on the
 * context stream (LMX_ESTATE before profile, traces and params are loaded).
 * One persistent kernel runs the discrete-event loop of each trace: at every
 * decision point the next task (inference by arrival; training released at
 * the previous training task's S1 forward end) is deprioritised
 * by Eq. 4 or placed -- LeMix: Algorithm 1 ComputeIdleness
 * on every node, Eq. 1-3, the highest
 * f, lowest node on ties; RR / Separate / Fixed / Mix-LUF: PAPER.md:795-797
 * -- and committed (backward planning).  Algorithm 2
 * with params.mem_enable, Algorithm 3
 * with params.cb_cmax.  Returns LMX_OK when enqueued; per-trace failures
 * (LMX_EINVAL on bad task data, LMX_EQCAP, LMX_EBUDGET, LMX_ETIMEOUT) are
 * reported by lmx_sync and the summaries' status.  Outputs are a pure
 * function of (profile, traces, params): no launch-geometry or GPU-count
 * dependence (the cross-rank fp64 cell sums aside, see lmx_allreduce_cells). */
lmx_status lmx_run(lmx_ctx *ctx);
/* Wait for the last lmx_run; returns its first non-OK per-trace status (the
 * lowest failing trace, named with its task and field by lmx_last_error) --
 * the other traces' results stay valid -- or LMX_ECUDA on a device error.
 * Releases the borrow of HOST / DEVICE task arrays. */
lmx_status lmx_sync(lmx_ctx *ctx);

/* Per-task outputs (the assignment and completion times of SPEC.md:23's task
 * records; TTFT = completion - arrival for inference), indexed
 * like the task arrays, valid after lmx_sync (LMX_ESTATE before, or when the
 * run was summary-only).  node_defer = node index
 * (bits 0-15) | Eq. 4 deferral count saturated at 0xFFFF (bits 16-31);
 * decision_idx = the decision (0-based, per trace) that placed the task;
 * completion = inference end_f^S, training end_b^1; start_f1 = start_f^1.
 * Tasks a failed trace never decided read node_defer 0xFFFFFFFF,
 * decision_idx -1 and NaN times (the trace's status says why).
 * Any pointer may be NULL.  `mem` says where the destination lives. */
lmx_status lmx_get_assignments(lmx_ctx *ctx, uint32_t *node_defer, int32_t *decision_idx, lmx_mem mem);
lmx_status lmx_get_times(lmx_ctx *ctx, double *completion, double *start_f1, lmx_mem mem);

/* debug_level 1 only: per decision and node, (II, R, f) as three doubles,
 * [n_tasks][n_nodes][3], row offsets[t] + k = decision k of trace t
 * (decision k of a trace is its k-th placement; traces have one decision per
 * task).  LeMix: every node is planned and scored.  RR / Separate / Fixed:
 * only the chosen node is planned; its f and every other node's row are NaN.
 * Decisions a failed trace never reached are NaN.  `mem` says where the
 * destination lives.  LMX_ESTATE unless the last run had debug_level 1. */
lmx_status lmx_get_candidates(lmx_ctx *ctx, double *cand, lmx_mem mem);

/* Per-trace summaries [n_traces] (host memory; the metrics of PAPER.md:786-790:
 * throughput, SLO attainment with TTFT <= tau_R, mean TTFT, utilisation,
 * active nodes PAPER.md:569-573, the loss proxies of SPEC.md:439), valid after
 * lmx_sync.  SURVEY.md 8(b)'s `total` argument is lmx_get_cells (one cell =
 * all traces unless lmx_set_cells grouped them). */
lmx_status lmx_get_summaries(lmx_ctx *ctx, lmx_summary *per_trace);
/* Per-cell aggregates [n_cells] (host memory), valid after lmx_sync: integer
 * sums exact, fp64 sums over the cell's traces in trace order. */
lmx_status lmx_get_cells(lmx_ctx *ctx, lmx_cell_summary *cells);

/* Multi-GPU (8(b) calls it lmx_allreduce_summaries): one
 * grouped ncclAllReduce(sum) of the cell aggregates over `nccl_comm` (an
 * ncclComm_t) on the context stream, after lmx_sync.  Integer fields are exact
 * for any rank count; the fp64 sums depend on the NCCL reduction order (within
 * 1e-12 relative of a single-GPU run).  NCCL is resolved at run time (dlopen
 * "libnccl.so.2"); LMX_ENCCL if unavailable. */
lmx_status lmx_allreduce_cells(lmx_ctx *ctx, void *nccl_comm);
/* Helpers to build a communicator without a framework: rank 0 calls
 * lmx_nccl_unique_id, ships the 128 bytes to every rank, each calls
 * lmx_nccl_comm_init on its own device. */
lmx_status lmx_nccl_unique_id(void *id128);
lmx_status lmx_nccl_comm_init(void **comm, int nranks, const void *id128, int rank, int device);
lmx_status lmx_nccl_comm_destroy(void *comm);

/* Device time of the last run's event-loop kernel (CUDA events on the context
 * stream; valid after lmx_sync) and the number of kernels the library
 * launched in that run. */
lmx_status lmx_get_timing(lmx_ctx *ctx, float *kernel_ms, float *run_ms, int32_t *launches);

/* Launch geometry chosen for the last run (for reports). */
lmx_status lmx_get_geometry(lmx_ctx *ctx, int32_t *grid, int32_t *block, int32_t *lanes_per_trace,
                            int32_t *smem_bytes);

#ifdef __cplusplus
}
#endif
#endif /* LEMIX_H */
