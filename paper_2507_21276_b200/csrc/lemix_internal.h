// lemix_internal.h -- host<->device contract between lemix_api.cpp and
// lemix_kernels.cu (not part of the public ABI; see include/lemix.h).
#pragma once
#include <cstdint>

#include "lemix.h"

namespace lmx {

// double2 words of one Q_train entry: (start_b, end_b) per stage, then the
// backward durations in pairs (see dev::RingT)
// (+ one word (C*l tokens, offload mask) with the memory model of Algorithm 2)
__host__ __device__ constexpr inline int ring_words(int S, bool mem = false) { return S + (S + 1) / 2 + (mem ? 1 : 0); }

// Everything the persistent event-loop kernel needs, passed by value.
struct KParams {
    // geometry of the candidate sweep: a "tile" of T lanes owns one trace,
    // lane l handles nodes l, l+T, l+2T, ... (npl slots)
    int32_t N, S, T, log2T, npl;
    int32_t policy, deprioritize, slo_mode;
    int32_t qcap;        // logical capacity of Q_train^n
    int32_t kmask;       // ring allocation K - 1 (K = next power of two >= qcap)
    int32_t n_tr_sep;    // Separate: N_train when both kinds are present (host-computed)
    int32_t s_pow2;      // S is a power of two -> II/S == II * (1/S) exactly
    double inv_S;
    double lambda1, lambda2, tau, slo_mult, slo_const, sigma_floor, lc0;
    // Algorithm 2 (lmx_params.mem_*): the MEM kernel instantiations read these
    int32_t mem_enable;
    long long mem_cap;
    double mem_dt, mem_tmax, mem_pen;
    // Separate's checkpoint synchronisation (lmx_params.sync_*): sync_sep = 1
    // when it applies; ck = per tile slot ck_cap doubles (availability times,
    // kept as their suffix minima, non-decreasing)
    int32_t sync_sep, sync_interval;
    double sync_latency;
    // SeparateDynamic (lmx_params.sep_dynamic): rate threshold and window
    int32_t sep_dynamic;
    double dyn_rate, dyn_window;
    double *ck;
    int32_t ck_cap;
    // Algorithm 3 continuous batching (lmx_params.cb_*; MODE 2 instantiations),
    // Eq. 4 reading, Mix-LUF scheduler latency
    int32_t cb_cmax, eq4_mode;
    double cb_tw, luf_delay;
    const uint32_t *out_len;   // device [n_tasks] decode steps, or nullptr
    // per-cell (lambda1, lambda2, tau) of lmx_set_cell_params, or nullptr
    const double *cell_par;
    const int32_t *cell_of;

    int64_t n_traces;
    const int64_t *offsets;    // device [n_traces+1]
    const int32_t *n_inf;      // device [n_traces]
    const double *arrival;     // device [n_tasks]
    const uint32_t *lbk;       // device [n_tasks]
    const int32_t *fixed;      // device [n_tasks] or nullptr
    const double *eta;         // device [3*N*S + 1]: eta_f, eta_b, eta_d node-major (+ pad)
    // streamed inputs (lmx_run with host traces): chunks of chunk_tasks tasks
    // land in order; *ready = number of chunks copied (nullptr: all resident)
    const unsigned *ready;
    long long chunk_tasks;

    uint32_t *node_defer;      // outputs, nullptr = summary-only
    int32_t *decision_idx;
    double *completion;
    double *start_f1;
    double *cand;              // debug_level 1: [n_tasks * N][3] (II, R, f) per decision and node, or nullptr

    lmx_summary *summaries;    // device [n_traces]
    int64_t *trace_err;        // device [n_traces]: (task << 8) | field code, -1 none
    unsigned long long *work;  // device [1]: next trace to claim
    unsigned long long *first_bad;  // device [1]: min failing trace index

    double2 *ring_be;          // [tile_slots][Npad][K][ring_words(S)]: (start_b, end_b) per stage, dB pairs
    int32_t npad;              // npl * T
    // the run writes per-task outputs / debug candidates (set before the
    // kernel is picked, so geometry queries and the launch pick the same one)
    int32_t want_outputs, want_cand;
};

// field codes for trace_err (reported by lmx_last_error)
enum : int32_t {
    kErrNone = 0, kErrLen = 1, kErrBatch = 2, kErrKind = 3, kErrBits = 4, kErrArrival = 5,
    kErrOrder = 6, kErrFixed = 7, kErrSeparateN1 = 8, kErrResponse = 9, kErrOutLen = 10
};

struct CellParams {
    int64_t n_traces;
    int32_t n_cells;
    const int64_t *cell_start; // device [n_cells+1] CSR over `order`, or nullptr (one cell: all traces)
    const int64_t *order;      // device [n_traces]: trace indices sorted (stably) by cell
    const lmx_summary *summaries;
    int64_t *cell_i;           // [n_cells][LMX_CELL_NI]
    double *cell_f;            // [n_cells][LMX_CELL_NF]
};

// launchers (lemix_kernels.cu)
int max_stages_bucket(int S);                         // template bucket for S
int npl_bucket(int npl);                              // template bucket for nodes/lane
int event_loop_smem_bytes(const KParams &p);
int event_loop_block_threads(const KParams &p);
int event_loop_traces_per_block(const KParams &p);   // traces in flight per CTA
// blocks per SM the event loop can keep resident with this geometry
int event_loop_occupancy(const KParams &p, int *err);
int launch_event_loop(const KParams &p, int grid, void *stream);
int launch_cells(const CellParams &c, void *stream);

}  // namespace lmx
