/*
 * lemix_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, single-threaded CPU oracle of LeMix's placement step
 * (arXiv 2507.21276, §4.2 Algorithm 1, §4.3 Eq. 1-4, §6.1 baselines).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, constant or helper with the
 * CUDA product path (paper_2507_21276_b200/csrc, include/lemix.h).
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without an independent
 * pin say so in lemix_oracle.c ("parity unpinned").
 */
#ifndef LEMIX_ORACLE_H
#define LEMIX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_LEMIX = 0, ORC_RR = 1, ORC_SEPARATE = 2, ORC_FIXED = 3, ORC_MIXLUF = 4 };
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EQCAP = 6, ORC_EBUDGET = 7 };

typedef struct {
    int32_t n_nodes;       /* N */
    int32_t n_stages;      /* S (GPUs per node) */
    const double *eta_f;   /* [N*S] node-major: eta_F^n for stage s */
    const double *eta_b;   /* [N*S] node-major: eta_B^n for stage s */
    const double *eta_d;   /* [N*S] node-major: decode step cost eta_D^n per context token,
                              or NULL (no decode; only read with continuous batching) */
} orc_profile;

typedef struct {
    int32_t policy;        /* ORC_LEMIX / ORC_RR / ORC_SEPARATE / ORC_FIXED */
    int32_t deprioritize;  /* Eq. 4 on/off (ablation "w/o prioritize") */
    int32_t slo_mode;      /* 0: tau_R = slo_mult * forward latency on node 0; 1: slo_const */
    int32_t qcap;          /* capacity of Q_train^n; exceeding it stops the trace with ORC_EQCAP */
    double lambda1, lambda2, tau;   /* Eq. 1, Eq. 3 */
    double slo_mult, slo_const;     /* tau_R */
    double sigma_floor, lc0;        /* Eq. 2 singular cases */
    double alpha;                   /* Separate's training fraction */
    /* Algorithm 2 ExecuteTaskMemoryAware (
     * DESIGN.md reading R-mem).  mem_enable = 0: unlimited memory, the
     * executed path is the planned one. */
    int32_t mem_enable;
    int32_t mem_pad;
    int64_t mem_cap;                /* activation memory per stage GPU, in tokens (C*l units) */
    double mem_dt;                  /* check interval Delta_t */
    double mem_tmax;                /* maximum wait T_max */
    double mem_pen;                 /* offload penalty, seconds per offloaded token */
    /* Separate's model synchronisation (
     * DESIGN.md reading R-sync).  sync_interval = 0: every policy uses the
     * co-located version proxy (R-ver). */
    int32_t sync_interval;          /* checkpoint every this many training tasks (e.g. 100) */
    int32_t sync_pad;
    double sync_latency;            /* seconds from checkpoint to loaded on the inference nodes */
    /* SeparateDynamic (reading R-sepdyn): the
     * partition follows the request rate over (now - dyn_window, now]:
     * below dyn_rate one inference node ("1-3" at N = 4, max(1, N/4) in
     * general), otherwise the alpha partition ("2-2"). */
    int32_t sep_dynamic;
    int32_t sep_pad;
    double dyn_rate;                /* requests/s threshold (50 in the paper) */
    double dyn_window;              /* seconds */
    /* Algorithm 3 ContinuousBatching + hybrid prefill/decode (
     * SURVEY.md §8f NEXT-2; reading R-cb).  cb_cmax = 0: every
     * request is its own task (the hot-path model). */
    int32_t cb_cmax;                /* maximum batch size C (requests) */
    int32_t eq4_mode;               /* Eq. 4 reading: 0 = R-14 (default), 1 = R-14b */
    double cb_tw;                   /* maximum waiting time T_w, seconds */
    /* Mix-LUF (reading R-luf): per-decision
     * scheduler latency (utilisation query), seconds, serialised */
    double luf_delay;
} orc_params;

/* Per-trace summary.  Integer block then fp64 block. */
typedef struct {
    int64_t n_tasks, n_inf, n_train, n_slo_met, n_deferrals, active_nodes, sum_version, status;
    int64_t n_mem_wait, n_offload;  /* stage forwards that waited for memory / were offloaded (Alg. 2) */
    int64_t n_batches, n_tbt;       /* Alg. 3: inference batches; requests with >= 1 decode step (TBT defined) */
    double makespan, throughput, sum_ttft, mean_ttft, slo_attainment, mean_util, mean_len_std;
    double sum_tbt, mean_tbt;       /* Alg. 3: time-between-tokens */
} orc_summary;

/* Event counters used to derive algorithmic fp64 op counts. */
typedef struct {
    int64_t decisions, alg1_calls, stage_iters, scan_consumed, scan_break,
            offset_adds, lc_exp, lc_cold, commits_train, eq4_checks, deferrals,
            version_scan, max_qlen;
} orc_counters;

/*
 * Run one trace.  Tasks are [0, n_tasks): the first n_inf are inference tasks
 * (non-decreasing arrival), the rest training tasks in release order
 * (arrival = earliest release a_min).  lbk packs l (bits 0-11), C (bits 12-19),
 * kind (bit 20, 1 = training).  out_len[n_tasks] = decode steps (tokens after
 * the prefill's first) of an inference request (0..2048; read only with
 * continuous batching; may be NULL otherwise).  With continuous batching an inference task's completion is the
 * time of its last token.
 *
 * Outputs (any may be NULL): node_defer[n_tasks] = node | deferrals<<16;
 * decision_idx[n_tasks]; completion[n_tasks] (inference end_f^S, training
 * end_b^1); start_f1[n_tasks]; paths[n_tasks*S*4] = per stage
 * (start_f, end_f, start_b, end_b) (backward = 0 for inference);
 * cand[n_tasks*N*3] = per decision, per node (II, R, f) (NaN where Alg. 1 did
 * not run on that node).  Returns the trace status.
 */
int orc_run_trace(const orc_profile *prof, const orc_params *par,
                  int64_t n_tasks, int64_t n_inf,
                  const double *arrival, const uint32_t *lbk, const uint32_t *out_len, const int32_t *fixed_node,
                  uint32_t *node_defer, int32_t *decision_idx, double *completion,
                  double *start_f1, double *paths, double *cand,
                  orc_summary *summary, orc_counters *counters);

/* Loop of orc_run_trace over a CSR batch of traces (offsets[n_traces+1], n_inf[n_traces]). */
int orc_run_batch(const orc_profile *prof, const orc_params *par,
                  int64_t n_traces, const int64_t *offsets, const int32_t *n_inf,
                  const double *arrival, const uint32_t *lbk, const uint32_t *out_len, const int32_t *fixed_node,
                  uint32_t *node_defer, int32_t *decision_idx, double *completion,
                  double *start_f1, orc_summary *summaries, orc_counters *counters);

/* Exposed for pinning: the fully specified exp(-t) routine (reading R-exp). */
double orc_exp_neg(double t);

#ifdef __cplusplus
}
#endif
#endif
