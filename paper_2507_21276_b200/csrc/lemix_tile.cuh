// lemix_tile.cuh -- the tile-of-lanes persistent event-loop kernel template
// (included by lemix_tile_{lemix,base}{,_mem}.cu, one translation unit per
// policy class and memory model so the instantiations compile in parallel).
//
// K1 profile staging : the fp64 SoA profile table (eta_f, eta_b) is copied
//                      into shared memory once per CTA with a TMA bulk copy
//                      (cp.async.bulk + mbarrier).
// K2-K4 event loop   : one persistent kernel.  A "tile" of T lanes of a warp
//                      owns one trace at a time; lane l plans nodes l, l+T, ...
//                      (Algorithm 1) and scores them (Eq. 1-3,
//                      PAPER.md:546-565); a tile shuffle takes the arg-best with
//                      the lowest-index tie-break; the owning
//                      lane commits.  Eq. 4 is a tile min.
//                      Tiles claim traces from a global counter until none are
//                      left, so long and short traces balance across SMs.
//
// Layout of one lane's state: per-node hot values in registers; commit-only
// values, rarely used per-trace words and the newest W Q_train entries in
// shared memory (one conflict-free column per thread); older queue entries in
// a global ring (spilled on eviction only).  The decision body is executed by
// every lane of the warp (tiles without a trace ride along with live = false),
// so its shuffles are full-warp segment shuffles; work that only some tiles
// or lanes need is predicated on place / lane == owner.
//
// Compiled with --fmad=false: see lemix_device.cuh for the fp64 discipline.
#pragma once
#include <cuda_runtime.h>

#include <climits>
#include <cmath>

#include "lemix_device.cuh"
#include "lemix_internal.h"

#ifndef LMX_TILE_PF
#define LMX_TILE_PF false                   // up-front ring loads in Alg. 1 (see dev::plan)
#endif
#ifndef LMX_TILE_WIN
#define LMX_TILE_WIN 4                      // ring tail-window entries in shared memory (S <= 2)
#endif
#ifndef LMX_TILE_L1PF
#define LMX_TILE_L1PF 0                     // L1 prefetch of the next inputs at decision start (measured slower)
#endif
#ifndef LMX_TILE_MINB
#define LMX_TILE_MINB 4                     // resident CTAs/SM the register budget targets
                                            // (2 for deep pipelines / several nodes per lane:
                                            // their per-lane state would spill at 128 registers)
#endif

namespace lmx {
namespace tile {

constexpr int kBlock = 128;                 // 4 warps per CTA
constexpr int kTraceWords = 7;              // rarely used per-trace shared-memory words (c_tw; 4 without cell params)
using dev::kInf;
using dev::task_batch;
using dev::task_len;
using dev::task_w;

inline int stages_bucket(int S) { return S <= 1 ? 1 : S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : 16; }
inline int npl_bucket(int npl) { return npl <= 1 ? 1 : npl <= 2 ? 2 : 4; }
inline int window_entries(int S) { return stages_bucket(S) <= 2 ? LMX_TILE_WIN : 0; }
// bytes of the TMA-staged profile: eta_f | eta_b, plus eta_d with continuous
// batching, rounded up to the bulk copy's 16-byte granule
__host__ __device__ inline uint32_t profile_bytes(int NS, bool cb) { return cb ? (24u * NS + 15u) & ~15u : 16u * NS; }
// 8-byte shared-memory words of commit-only state per node slot and thread
// (+ 4 words of scoring state when a lane owns several nodes, see SCOLD)
__host__ __device__ inline int cold_words(int S, bool scold) { return 2 * S + 4 + (scold ? 4 : 0); }

// MODE of an instantiation: 0 the hot-path model; 1 Algorithm 2 memory-aware
// execution (NEXT-1); 2 Algorithm 3 continuous batching + decode (NEXT-2)
enum : int { kPlain = 0, kMem = 1, kCb = 2 };

template <int SMAX, bool EXACT, int NPL, bool LEMIX, int TT, int MODE>
__global__ void __launch_bounds__(kBlock, (SMAX >= 4 || NPL > 1) ? 2 : LMX_TILE_MINB) event_loop_kernel(const KParams p)
{
    // LEMIX: the policy is LeMix (all candidates planned and scored); else one
    // of the baselines (RR / Separate / Fixed / Mix-LUF) picks the node first.
    // MEM: the committed task is executed under Algorithm 2's memory model
    // (dev::execute_mem) and the executed path replaces the plan.
    // CB: inference requests are batched (Algorithm 3, DESIGN.md R-cb) and
    // each batch's decode steps occupy its node after the prefill.
    constexpr bool MEM = MODE == kMem, CB = MODE == kCb;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t s_bar;

    // S is a compile-time constant when it equals the template bucket (EXACT)
    const int N = p.N, S = EXACT ? SMAX : p.S, NS = p.N * S;
    double *s_eta = reinterpret_cast<double *>(smem_raw);
    // per-cell parameters (lmx_set_cell_params) are read by the generic-width
    // LeMix instantiations; the host picks one of those when they are set
    constexpr bool CPAR = LEMIX && TT == 0;

    // ---- K1: stage eta_f | eta_b (| eta_d) into shared memory via TMA ----
    const uint32_t pbytes = profile_bytes(NS, CB);
    if (threadIdx.x == 0) {
        dev::mbar_init(&s_bar, 1);
        dev::mbar_arrive_expect_tx(&s_bar, pbytes);
        dev::bulk_copy_g2s(s_eta, p.eta, pbytes, &s_bar);
    }
    __syncthreads();
    dev::mbar_wait(&s_bar, 0);
    uint32_t s_eta_u = dev::smem_u32(s_eta);
    dev::opaque(s_eta_u);
    const dev::SmemProfile prof{s_eta_u, NS, S};
    double ef0[SMAX];   // eta_F of node 0, for tau_R (R-16)
#pragma unroll
    for (int s = 0; s < SMAX; ++s) ef0[s] = (s < S) ? prof.f(0, s) : 0.0;

    // ---- tile geometry ----
    const int lane = threadIdx.x & 31;
    // TT > 0: the tile width is a compile-time constant (shuffle loops unroll)
    const int T = TT > 0 ? TT : p.T, log2T = TT > 0 ? __builtin_ctz(TT > 0 ? TT : 1) : p.log2T;
    const int tl = lane & (T - 1);
    const int tbase = lane & ~(T - 1);
    const unsigned tmask = (T == 32) ? 0xffffffffu : (((1u << T) - 1u) << tbase);
    const long long gtile = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> log2T;
    const long long K = (long long)p.kmask + 1;

    // the Q_train ring of each node this lane owns: a shared-memory tail
    // window, [slot jj][W][S+1][thread] (see dev::RingT), over a global ring
    constexpr int W = (SMAX <= 2) ? LMX_TILE_WIN : 0;   // see window_entries()
    constexpr uint32_t wstride = 16u * kBlock;            // (blockDim.x == kBlock)
    uint32_t ws[NPL];
    double2 *rbe[NPL];
#pragma unroll
    for (int jj = 0; jj < NPL; ++jj) {
        ws[jj] = dev::smem_u32(smem_raw + pbytes) + (uint32_t)(jj * (W > 0 ? W : 1) * ring_words(S, MEM)) * wstride +
                 16u * threadIdx.x;
        dev::opaque(ws[jj]);   // keep in a register: no per-iteration rematerialisation
        const long long rbase = (gtile * p.npad + (tl + jj * T)) * K;
        rbe[jj] = p.ring_be + rbase * ring_words(S, MEM);
        dev::opaque_ptr(rbe[jj]);
    }
    // commit-only per-node state in shared memory ("cold" words, 8 bytes each,
    // [word][thread] so each thread owns a conflict-free column): per slot jj
    // LB[s] (last planned backward end), busy[s], sum l, sum l^2, and
    // (training count, version pointer) -- see cold_words()
    constexpr uint32_t cstride = 8u * kBlock;   // (blockDim.x == kBlock): immediate offsets
    constexpr bool SCOLD = NPL > 1;
    const int CW = cold_words(S, SCOLD);   // words per node slot
    uint32_t cbase = dev::smem_u32(smem_raw + pbytes) +
                     (uint32_t)(W > 0 ? NPL * W * ring_words(S, MEM) : 0) * wstride + 8u * threadIdx.x;
    dev::opaque(cbase);
    auto c_lb = [&](int jj, int s) { return cbase + (uint32_t)(jj * CW + s) * cstride; };
    auto c_busy = [&](int jj, int s) { return cbase + (uint32_t)(jj * CW + S + s) * cstride; };
    auto c_sl = [&](int jj) { return cbase + (uint32_t)(jj * CW + 2 * S) * cstride; };
    auto c_sl2 = [&](int jj) { return cbase + (uint32_t)(jj * CW + 2 * S + 1) * cstride; };
    auto c_ntr = [&](int jj) { return cbase + (uint32_t)(jj * CW + 2 * S + 2) * cstride; };
    // the node's task count, stored only when its trace ends (for the summary)
    auto c_cnt = [&](int jj) { return cbase + (uint32_t)(jj * CW + 2 * S + 3) * cstride; };
    // rarely used per-trace words (same column layout, after the node slots):
    // 0 trace index, 1 first task offset, 2 t_first, 3 error (task << 8 | field),
    // 4-6 the trace's cell (lambda1, lambda2, tau) with lmx_set_cell_params
    auto c_tw = [&](int k) { return cbase + (uint32_t)(NPL * CW + k) * cstride; };
    // SCOLD (several nodes per lane): a_[-1], mu, 1/(2 sigma^2), 1/(sigma sqrt(2 pi))
    // of each node also live in shared memory (read once per decision)
    auto c_sc = [&](int jj, int f) { return cbase + (uint32_t)(jj * CW + 2 * S + 4 + f) * cstride; };

    // ---- per-trace (tile-replicated) state ----
    bool active = false, finished = false;
    long long t = 0;                      // (claim only; kept in c_tw(0) across the trace)
    const double *tarr = p.arrival;      // this trace's task arrays (32-bit indexing)
    const uint32_t *tlbk = p.lbk;
    int nI = 0, nT = 0, i = 0, j = 0, step = 0, iters = 0, rr = 0, sep_i = 0, sep_t = 0;
    int rate_lo = 0, rate_hi = 0;         // SeparateDynamic: inference arrivals in (now - W, now]
    int cur_defer = 0, status = LMX_OK;
    double r = kInf, t_last = -kInf, a_last_inf = -kInf, sum_ttft = 0.0;
    long long sum_ver = 0;
    int n_slo = 0, n_def = 0;             // (<= 2^19 tasks, <= 2^20 decisions per trace)
    int n_mwait = 0, n_moff = 0;          // Algorithm 2 counters (MEM)
    int n_ck = 0;                         // Separate's checkpoints so far (sync model)
    int n_batches = 0, n_tbt = 0;         // Algorithm 3 (CB): batches placed, requests with decode steps
    double sum_tbt = 0.0;
    double sched_free = -kInf;            // Mix-LUF: when the scheduler's previous query ends (R-luf)
    double *ckt = (!LEMIX && p.sync_sep) ? p.ck + gtile * p.ck_cap : nullptr;
    double a_inf = 0.0, a_inf2 = 0.0, a_tr = 0.0, a_tr2 = 0.0;   // 2-deep input prefetch
    uint32_t v_inf = 0, v_inf2 = 0, v_tr = 0, v_tr2 = 0;

    // ---- per-node state of this lane's slots (registers) ----
    double P[NPL][SMAX];
    double aprev[NPL], mu[NPL], kk[NPL], cc[NPL];
    int hasp[NPL], qh[NPL], qn[NPL], cnt[NPL];
    int sk[NPL][SMAX];   // stale-prefix pointers (see dev::plan)
    double skeb[NPL][SMAX];   // end_b^s of the last stale entry (see dev::plan)

    // Control flow inside the loop is structured (no continue/break out of a
    // branch) so tiles that took different branches reconverge right after it.
    while (!__all_sync(0xffffffffu, finished)) {
        if (!finished && !active) {
            // ---- claim the next trace ----
            unsigned long long tt = 0;
            if (tl == 0) tt = atomicAdd(p.work, 1ull);
            tt = __shfl_sync(tmask, tt, tbase);
            if (tt >= (unsigned long long)p.n_traces) {
                finished = true;
            } else {
                t = (long long)tt;
                const long long o = p.offsets[t];
                const int len = (int)(p.offsets[t + 1] - o);
                const bool landed = dev::wait_inputs(p.ready, p.chunk_tasks, o, o + len);
                nI = p.n_inf[t];
                nT = len - nI;
                tarr = p.arrival + o;
                tlbk = p.lbk + o;
                i = j = step = iters = rr = sep_i = sep_t = cur_defer = 0;
                rate_lo = rate_hi = 0;
                status = landed ? LMX_OK : LMX_ETIMEOUT;
                dev::sts_l(c_tw(0), t);
                dev::sts_l(c_tw(1), o);
                dev::sts_l(c_tw(3), kErrNone);
                n_slo = sum_ver = n_def = 0;
                n_mwait = n_moff = 0;
                n_ck = 0;
                n_batches = n_tbt = 0;
                sum_tbt = 0.0;
                sched_free = -kInf;
                sum_ttft = 0.0;
                t_last = -kInf;
                a_last_inf = -kInf;
                if (landed) {
                    if (nI > 0) { a_inf = __ldg(tarr); v_inf = __ldg(tlbk); }
                    if (nI > 1) { a_inf2 = __ldg(tarr + 1); v_inf2 = __ldg(tlbk + 1); }
                    if (nT > 0) { a_tr = __ldg(tarr + nI); v_tr = __ldg(tlbk + nI); }
                    if (nT > 1) { a_tr2 = __ldg(tarr + nI + 1); v_tr2 = __ldg(tlbk + nI + 1); }
                }
                r = (nT > 0) ? a_tr : kInf;
                double t_first = kInf;
                if (nI > 0) t_first = dev::dmin(t_first, a_inf);
                if (nT > 0) t_first = dev::dmin(t_first, a_tr);
                dev::sts_d(c_tw(2), t_first);
                if (CPAR && p.cell_par) {    // the trace's cell parameters (NEXT-4 sweeps)
                    const double *cp = p.cell_par + 3 * p.cell_of[t];
                    dev::sts_d(c_tw(4), cp[0]);
                    dev::sts_d(c_tw(5), cp[1]);
                    dev::sts_d(c_tw(6), cp[2]);
                }
#pragma unroll
                for (int jj = 0; jj < NPL; ++jj) {
                    hasp[jj] = qh[jj] = qn[jj] = cnt[jj] = 0;
                    aprev[jj] = mu[jj] = kk[jj] = cc[jj] = 0.0;
                    if (SCOLD)
#pragma unroll
                        for (int f = 0; f < 4; ++f) dev::sts_d(c_sc(jj, f), 0.0);
                    dev::sts_l(c_sl(jj), 0);
                    dev::sts_l(c_sl2(jj), 0);
                    dev::sts_l(c_ntr(jj), 0);      // training count | version pointer << 32
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) {
                        P[jj][s] = 0.0;
                        sk[jj][s] = 0;
                        skeb[jj][s] = 0.0;
                        if (s < S) {
                            dev::sts_d(c_lb(jj, s), -kInf);
                            dev::sts_d(c_busy(jj, s), 0.0);
                        }
                    }
                }
                if (!LEMIX && p.policy == LMX_SEPARATE && N == 1 && nI > 0 && nT > 0) {
                    status = LMX_EINVAL;
                    dev::sts_l(c_tw(3), kErrSeparateN1);
                }
                active = true;
            }
        }
        // Tiles without a trace (finished) stay in the loop as passengers
        // (live = false): every lane of the warp then reaches the full-warp
        // shuffles of the decision below together, so they need no
        // divergence-tolerant mask handling.
        const bool more = active & ((i < nI) | (j < nT));
        iters += more;
        if (more & (iters > 2 * (nI + nT) + 2)) status = LMX_EBUDGET;
        const bool done_trace = active & ((status != LMX_OK) | !more);
        const bool live = active & !done_trace;

        if (done_trace) {
            // ---- per-trace metrics, node folds in node order ----
            lmx_summary sm;
            sm.n_tasks = nI + nT;
            sm.n_inf = nI;
            sm.n_train = nT;
            sm.status = status;
            sm.n_slo_met = sm.n_deferrals = sm.active_nodes = sm.sum_version = 0;
            sm.n_mem_wait = sm.n_offload = sm.n_batches = sm.n_tbt = 0;
            sm.makespan = sm.throughput = sm.sum_ttft = sm.mean_ttft = sm.slo_attainment = 0.0;
            sm.mean_util = sm.mean_len_std = sm.sum_tbt = sm.mean_tbt = 0.0;
            if (status == LMX_OK) {
                const int ntask = nI + nT;
                sm.n_slo_met = n_slo;
                sm.n_deferrals = n_def;
                sm.sum_version = sum_ver;
                sm.n_mem_wait = n_mwait;
                sm.n_offload = n_moff;
                sm.n_batches = n_batches;
                sm.n_tbt = n_tbt;
                sm.sum_tbt = sum_tbt;
                sm.mean_tbt = (n_tbt > 0) ? sum_tbt / (double)n_tbt : 0.0;
                sm.sum_ttft = sum_ttft;
                sm.makespan = (ntask > 0) ? t_last - dev::lds_d(c_tw(2)) : 0.0;
                sm.throughput = (sm.makespan > 0.0) ? (double)ntask / sm.makespan : 0.0;
                sm.mean_ttft = (nI > 0) ? sum_ttft / (double)nI : 0.0;
                sm.slo_attainment = (nI > 0) ? (double)n_slo / (double)nI : 1.0;
                // node folds in node order by the tile's first lane, reading
                // every lane's shared-memory column (no shuffles in this
                // tile-divergent branch)
#pragma unroll
                for (int jj = 0; jj < NPL; ++jj) dev::sts_l(c_cnt(jj), cnt[jj]);
                __syncwarp(tmask);
                double U = 0.0, stds = 0.0;
                long long act = 0;
                if (tl == 0) {
                    for (int n = 0; n < N; ++n) {
                        // lane tbase + (n mod T), slot n / T: its column is (n mod T) columns right
                        const uint32_t col = 8u * (uint32_t)(n & (T - 1));
                        const int jn = n >> log2T;
                        const long long c = dev::lds_l(c_cnt(0) + (uint32_t)(jn * CW) * cstride + col);
                        const long long a1 = dev::lds_l(c_sl(0) + (uint32_t)(jn * CW) * cstride + col);
                        const long long a2 = dev::lds_l(c_sl2(0) + (uint32_t)(jn * CW) * cstride + col);
                        for (int s = 0; s < S; ++s) U = U + dev::lds_d(c_busy(0, s) + (uint32_t)(jn * CW) * cstride + col);
                        if (c > 0) {
                            act++;
                            stds = stds + sqrt((double)(c * a2 - a1 * a1)) / (double)c;
                        }
                    }
                }
                sm.active_nodes = act;
                sm.mean_util = (sm.makespan > 0.0) ? U / ((double)(N * S) * sm.makespan) : 0.0;
                sm.mean_len_std = (act > 0) ? stds / (double)act : 0.0;
            }
            if (tl == 0) {
                const long long tt = dev::lds_l(c_tw(0));
                p.summaries[tt] = sm;
                if (status != LMX_OK) {
                    p.trace_err[tt] = dev::lds_l(c_tw(3));
                    atomicMin(p.first_bad, (unsigned long long)tt);
                }
            }
            active = false;
        }
        {
            // ---- a1: event selection (ties -> inference) ----
#if LMX_TILE_L1PF
            // Pull the inputs the end-of-decision loads will read (two ahead in
            // each stream) into L1 now, without occupying registers, so those
            // loads -- which the next iteration's control flow waits on -- hit L1.
            dev::prefetch_l1(tarr + min(i + 2, nI - 1));
            dev::prefetch_l1(tlbk + min(i + 2, nI - 1));
            dev::prefetch_l1(tarr + nI + min(j + 2, nT - 1));
            dev::prefetch_l1(tlbk + nI + min(j + 2, nT - 1));
#endif
            const double t_inf = (i < nI) ? a_inf : kInf;
            const bool is_train = !(t_inf <= r);
            double now = is_train ? r : t_inf;
            const uint32_t v = is_train ? v_tr : v_inf;
            // CB: the unit placed is the batch request i opens (Algorithm 3,
            // PAPER.md:693-716; DESIGN.md R-cb): members i .. i + mb - 1, C_b
            // items padded to length lpad, decode work wd (exact token units)
            int mb = 1, lpad = task_len(v), cb_err = 0;
            long long cbt = task_batch(v), wd = 0, sum_l = task_len(v), sum_l2 = (long long)task_len(v) * task_len(v);
            if (CB && live && !is_train) {
                // lines 7-12: join while not full, not behind a released training
                // task (ties -> inference) and before the timer T_start + T_w
                while (i + mb < nI && mb < p.cb_cmax) {
                    const double ar = __ldg(tarr + i + mb);
                    if ((j < nT && r < ar) || !(t_inf + p.cb_tw > ar)) break;
                    const uint32_t vm = __ldg(tlbk + i + mb);
                    const unsigned lm = (unsigned)task_len(vm);
                    if (!(((vm >> 21) == 0u) & (lm - 1u < 2048u) & (task_batch(vm) >= 1) & (((vm >> 20) & 1u) == 0u) &
                          (ar < kInf) & (ar >= __ldg(tarr + i + mb - 1))))
                        cb_err = 1;   // (reported as the member's own field error below)
                    lpad = max(lpad, (int)lm);
                    cbt += task_batch(vm);
                    sum_l += lm;
                    sum_l2 += (long long)lm * lm;
                    mb++;
                }
                // line 15: full -> at the C-th arrival, else the timer or the training release
                now = (mb == p.cb_cmax) ? __ldg(tarr + i + mb - 1) : dev::dmin(t_inf + p.cb_tw, (j < nT) ? r : kInf);
                // decode steps 1 .. out_j of every member over the padded context
                // (SPEC.md:410): sum_j g(out_j), g(o) = o (lpad - 1) + o (o + 1) / 2
                const long long o0 = dev::lds_l(c_tw(1)) + i;
                for (int k = 0; k < mb; ++k) {
                    const long long ok = __ldg(p.out_len + o0 + k);
                    if (ok > 2048) cb_err = 2;
                    wd += ok * (lpad - 1) + ok * (ok + 1) / 2;
                }
            }
            // Inputs two ahead in the stream this decision consumes, loaded
            // now so they land while the decision runs (loaded at its end, the
            // loop-carried register copies at the top of the next iteration
            // would wait for them).  Discarded when the task is deferred.
            const bool pf_ok = live && (is_train ? nT > 0 : nI > 0);
            const int pf_idx = is_train ? nI + min(j + 2, nT - 1) : min(i + 2, nI - 1);
            const double pf_a = pf_ok ? __ldg(tarr + pf_idx) : 0.0;
            const uint32_t pf_v = pf_ok ? __ldg(tlbk + pf_idx) : 0u;
            bool deferred = false;
            if (LEMIX) {
                // ---- a2: Eq. 4 queue-level deprioritisation against the next
                // enqueued inference task (R-14/R-15);
                // the tile min is formed by every lane, used where it applies ----
                const bool eq4 = live && is_train && p.deprioritize && i < nI;
                const double wn = task_w(v_inf);
                double m = kInf;
#pragma unroll
                for (int jj = 0; jj < NPL; ++jj) {
                    const int n = tl + jj * T;
                    if (n < N) {
                        double latest = hasp[jj] ? dev::last_of(P[jj], S) : -kInf;
                        if (p.eq4_mode == 1) {
                            // R-14b: the training task's own forward, chained stage by
                            // stage after the node's last forward, comes first
                            const double wt = task_w(v);
                            double vv = now;
#pragma unroll
                            for (int s = 0; s < SMAX; ++s)
                                if (s < S) vv = dev::dmax(vv, hasp[jj] ? P[jj][s] : -kInf) + prof.f(n, s) * wt;
                            latest = vv;
                        }
                        m = dev::dmin(m, latest + prof.f(n, S - 1) * wn);
                    }
                }
                #pragma unroll
                for (int off = T >> 1; off > 0; off >>= 1) m = dev::dmin(m, dev::shfl_xor_w(m, off, T));
                if (eq4) {
                double tauR;
                if (p.slo_mode == 1) {
                    tauR = p.slo_const;
                } else {
                    double acc = 0.0;
#pragma unroll
                    for (int s = 0; s < SMAX; ++s)
                        if (s < S) acc = acc + ef0[s] * wn;
                    tauR = p.slo_mult * acc;
                }
                deferred = (m - t_inf) > tauR;
                if (deferred) {
                    r = t_inf;          // move behind the next inference task
                    cur_defer++;
                    n_def++;
                }
                }
            }
            const int task = is_train ? nI + j : i;
            if (live && !deferred) {
                // ---- input validation of the task being placed (one predicate;
                // the error code is worked out only on the rare failure path) ----
                const double arr = is_train ? a_tr : a_inf;
                const unsigned lv = (unsigned)task_len(v);
                bool ok = ((v >> 21) == 0u) & (lv - 1u < 2048u) & (task_batch(v) >= 1) &
                          ((int)((v >> 20) & 1u) == (int)is_train) & (arr >= 0.0) & (arr < kInf) &
                          (is_train | (arr >= a_last_inf));
                int fx = 0;
                if (!LEMIX && p.policy == LMX_FIXED) {
                    fx = __ldg(p.fixed + dev::lds_l(c_tw(1)) + task);
                    ok = ok & (fx >= 0) & (fx < N);
                }
                if (CB && cb_err) {
                    status = LMX_EINVAL;
                    dev::sts_l(c_tw(3), ((long long)task << 8) | (cb_err == 2 ? kErrOutLen : kErrBits));
                }
                if (!ok) {
                    int code = kErrFixed;
                    if (v >> 21) code = kErrBits;
                    else if (task_len(v) < 1 || task_len(v) > 2048) code = kErrLen;
                    else if (task_batch(v) < 1) code = kErrBatch;
                    else if ((int)((v >> 20) & 1u) != (int)is_train) code = kErrKind;
                    else if (!(arr >= 0.0 && arr < kInf)) code = kErrArrival;
                    else if (!is_train && arr < a_last_inf) code = kErrOrder;
                    status = LMX_EINVAL;
                    dev::sts_l(c_tw(3), ((long long)task << 8) | code);
                }
            }
            const bool place = live && !deferred && status == LMX_OK;   // this tile places a task
            {
                double a = now;                          // dispatch time (R-2)
                // the unit's C*l^2 (a batch: its items, padded, R-cb) and the
                // length Eq. 2 scores
                const double w = CB ? (double)(cbt * lpad * lpad) : task_w(v);
                const int l = CB ? lpad : task_len(v);

                // ---- a9: baseline selectors ----
                int chosen = -1;
                if (LEMIX || !place) {
                } else if (p.policy == LMX_RR) {
                    chosen = rr % N;
                    rr++;
                } else if (p.policy == LMX_SEPARATE) {
                    if (!(nI > 0 && nT > 0)) {
                        chosen = is_train ? (sep_t++ % N) : (sep_i++ % N);
                    } else {
                        int ninf = N - p.n_tr_sep;
                        if (p.sep_dynamic) {
                            // SeparateDynamic (R-sepdyn): request rate over
                            // the last dyn_window seconds -> "1-3" or the alpha partition
                            while (rate_hi < nI && __ldg(tarr + rate_hi) <= now) rate_hi++;
                            const double w_lo = now - p.dyn_window;
                            while (rate_lo < nI && __ldg(tarr + rate_lo) <= w_lo) rate_lo++;
                            const double rate = (double)(rate_hi - rate_lo) / p.dyn_window;
                            ninf = (rate < p.dyn_rate) ? (N / 4 > 1 ? N / 4 : 1) : ninf;
                        }
                        chosen = is_train ? ninf + (sep_t++ % (N - ninf)) : (sep_i++ % ninf);
                    }
                } else if (p.policy == LMX_MIXLUF) {
                    // Mix-LUF (R-luf): the node with the least busy
                    // time committed so far (busy columns of the tile's lanes,
                    // summed stage by stage), lowest index on ties; the decision
                    // waits for the serialised utilisation query
                    __syncwarp(tmask);
                    double ub = kInf;
                    chosen = 0;
                    for (int n = 0; n < N; ++n) {
                        const uint32_t col = 8u * (uint32_t)((n & (T - 1)) - tl);
                        const int jn = n >> log2T;
                        double u = 0.0;
                        for (int s = 0; s < S; ++s) u = u + dev::lds_d(c_busy(0, s) + (uint32_t)(jn * CW) * cstride + col);
                        if (u < ub) { ub = u; chosen = n; }
                    }
                    sched_free = dev::dmax(now, sched_free) + p.luf_delay;
                    a = sched_free;
                } else {
                    chosen = __ldg(p.fixed + dev::lds_l(c_tw(1)) + task);
                }

                // ---- a3-a7: Algorithm 1 + Eq. 1-3 for every candidate this lane owns ----
                double en_s[NPL][SMAX];
                double oc_s[NPL][SMAX];   // CB: occupancy ends (forward + the batch's decode steps)
                double st0_s[NPL];
                double f_best = 0.0;
                int n_best = INT_MAX;
                bool r_bad = false;   // a candidate with R <= 0 (Eq. 3 undefined)
                // Eq. 2 statistics of each owned node if this task is committed
                // there (DESIGN.md R-stat), computed here by every lane -- where
                // the work overlaps the other candidates' latency -- instead of
                // serially by the winning lane in the commit
                double mu_n[NPL], kk_n[NPL], cc_n[NPL];
                long long sl_n[NPL], sl2_n[NPL];
                bool ok_st = true;   // LMX_FASTDIV: every division / sqrt took its fast path
                auto spec_stats = [&](long long c, long long a1, long long a2, int jj) {
                    sl_n[jj] = a1;
                    sl2_n[jj] = a2;
                    const long long var = c * a2 - a1 * a1;
                    if (LMX_FASTDIV) {
                        bool ok1, ok2, ok3;
                        const double inv_c = dev::rcp_fastpath((double)c, ok1);
                        mu_n[jj] = (double)a1 * inv_c;
                        // (sqrt(+0) = +0: the argument is made nonzero, the fast path would not take 0)
                        double sq = dev::sqrt_fastpath((double)(var == 0 ? 1 : var), ok2);
                        sq = (var == 0) ? 0.0 : sq;
                        const double sigma = dev::dmax(sq * inv_c, p.sigma_floor);
                        const double inv_s = dev::rcp_fastpath(sigma, ok3);
                        kk_n[jj] = (0.5 * inv_s) * inv_s;
                        cc_n[jj] = inv_s * dev::kInvSqrt2Pi;
                        ok_st = ok1 && ok2 && ok3;
                    } else {
                        const double inv_c = 1.0 / (double)c;
                        mu_n[jj] = (double)a1 * inv_c;
                        const double sigma = dev::dmax(sqrt((double)var) * inv_c, p.sigma_floor);
                        const double inv_s = 1.0 / sigma;
                        kk_n[jj] = (0.5 * inv_s) * inv_s;
                        cc_n[jj] = inv_s * dev::kInvSqrt2Pi;
                    }
                };
                auto spec_stats_ieee = [&](long long c, long long a1, long long a2, int jj) {
                    const long long var = c * a2 - a1 * a1;
                    const double inv_c = 1.0 / (double)c;
                    mu_n[jj] = (double)a1 * inv_c;
                    const double sigma = dev::dmax(sqrt((double)var) * inv_c, p.sigma_floor);
                    const double inv_s = 1.0 / sigma;
                    kk_n[jj] = (0.5 * inv_s) * inv_s;
                    cc_n[jj] = inv_s * dev::kInvSqrt2Pi;
                };
#pragma unroll
                for (int jj = 0; jj < NPL; ++jj) {
                    const int n = tl + jj * T;
                    st0_s[jj] = 0.0;
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) en_s[jj][s] = 0.0;
                    mu_n[jj] = kk_n[jj] = cc_n[jj] = 0.0;
                    sl_n[jj] = sl2_n[jj] = 0;
                    if (place && n < N && (LEMIX || n == chosen)) {
                        // Eq. 2 of this candidate, ahead of (and
                        // independent of) Algorithm 1; exp_neg is evaluated for cold
                        // nodes too and discarded (its value is finite for t >= 0)
                        double LC = p.lc0;
                        if (LEMIX) {
                            const double mu_j = SCOLD ? dev::lds_d(c_sc(jj, 1)) : mu[jj];
                            const double kk_j = SCOLD ? dev::lds_d(c_sc(jj, 2)) : kk[jj];
                            const double cc_j = SCOLD ? dev::lds_d(c_sc(jj, 3)) : cc[jj];
                            const double d = (double)l - mu_j;
                            const double lw = cc_j * dev::exp_neg((d * d) * kk_j);
                            LC = (cnt[jj] < 2) ? p.lc0 : lw;
                        }
                        double II;
                        int gc;
                        const int qhead = qh[jj], qlen = qn[jj];
                        const dev::RingT<W, wstride, MEM> q{rbe[jj], p.kmask, S, ws[jj], wstride, qhead + qlen};
                        double efn[SMAX], ebn[SMAX];
                        prof.node<SMAX>(n, efn, ebn);
                        if (CB) {
                            // the batch's decode steps follow its prefill on each GPU
                            double tl_n[SMAX];
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) tl_n[s] = (s < S) ? prof.d(n, s) * (double)wd : 0.0;
                            dev::plan<SMAX, LMX_TILE_PF, dev::RingT<W, wstride, MEM>, true>(
                                P[jj], hasp[jj] != 0, S, efn, ebn, q, qhead, qlen, sk[jj], skeb[jj], w, a, now, en_s[jj],
                                st0_s[jj], II, gc, &tl_n, &oc_s[jj]);
                        } else {
                            dev::plan<SMAX, LMX_TILE_PF>(P[jj], hasp[jj] != 0, S, efn, ebn, q, qhead, qlen, sk[jj], skeb[jj],
                                                         w, a, now, en_s[jj], st0_s[jj], II, gc);
                        }
                        // lines 17-18: executed entries leave Q_train^n (a head advance:
                        // end_b^1 is non-decreasing along the queue)
                        qh[jj] = qhead + gc;
                        qn[jj] = qlen - gc;
                        if (LEMIX) {
                            const double R = dev::last_of(en_s[jj], S) - a;               // line 20
                            const double ap_j = SCOLD ? dev::lds_d(c_sc(jj, 0)) : aprev[jj];
                            const double a_last = hasp[jj] ? ap_j : a;                   // R-9
                            const double IIS = p.s_pow2 ? II * p.inv_S : II / (double)S;  // exact either way
                            const bool cpar = CPAR && p.cell_par != nullptr;              // (uniform)
                            const double lam1 = cpar ? dev::lds_d(c_tw(4)) : p.lambda1;
                            const double lam2 = cpar ? dev::lds_d(c_tw(5)) : p.lambda2;
                            const double tau = cpar ? dev::lds_d(c_tw(6)) : p.tau;
                            const double IP = -dev::dmax(IIS - (a - a_last), tau);        // Eq. 1
                            const double num = IP + lam2 * LC, den = lam1 * R;
                            double f;                                                     // Eq. 3
                            bool ok_f = true;
                            if (LMX_FASTDIV) {
                                // (see lemix_device.cuh; a zero numerator has the signed-zero
                                // quotient for a finite nonzero denominator)
                                const bool z = num == 0.0;
                                f = dev::div_fastpath(z ? 1.0 : num, den, ok_f);
                                f = z ? __longlong_as_double((__double_as_longlong(num) ^ __double_as_longlong(den)) &
                                                             (long long)0x8000000000000000ull)
                                      : f;
                            } else {
                                f = num / den;
                            }
                            // speculative statistics: count + members, sums + their l, l^2
                            const long long c = cnt[jj] + (CB ? mb : 1);
                            const long long a1 = dev::lds_l(c_sl(jj)) + (CB ? sum_l : l);
                            const long long a2 = dev::lds_l(c_sl2(jj)) + (CB ? sum_l2 : (long long)l * l);
                            spec_stats(c, a1, a2, jj);
                            if (LMX_FASTDIV && !(ok_f && ok_st)) {
                                f = num / den;
                                spec_stats_ieee(c, a1, a2, jj);
                            }
                            r_bad |= !(R > 0.0);
                            if (n_best == INT_MAX || f > f_best) { f_best = f; n_best = n; }
                            if (p.cand)   // debug_level 1: this candidate's (II, R, f) (uniform branch)
                                dev::put_cand(p.cand, (dev::lds_l(c_tw(1)) + step) * N + n, II, R, f);
                        } else {
                            if (p.cand)
                                dev::put_cand(p.cand, (dev::lds_l(c_tw(1)) + step) * N + n, II,
                                              dev::last_of(en_s[jj], S) - a, __longlong_as_double(-1ll));
                            // speculative statistics: count + members, sums + their l, l^2
                            const long long c = cnt[jj] + (CB ? mb : 1);
                            const long long a1 = dev::lds_l(c_sl(jj)) + (CB ? sum_l : l);
                            const long long a2 = dev::lds_l(c_sl2(jj)) + (CB ? sum_l2 : (long long)l * l);
                            spec_stats(c, a1, a2, jj);
                            if (LMX_FASTDIV && !ok_st) spec_stats_ieee(c, a1, a2, jj);
                        }
                    }
                }

                // R <= 0 (a forward too short to advance the clock): the trace
                // stops with LMX_EINVAL before anything is committed, as in the oracle
                bool place_c = place;
                if (LEMIX) {
                    const unsigned rb = __ballot_sync(0xffffffffu, r_bad);
                    if ((rb >> tbase) & (T == 32 ? 0xffffffffu : ((1u << T) - 1u))) {
                        if (place) {
                            status = LMX_EINVAL;
                            if (tl == 0) dev::sts_l(c_tw(3), ((long long)task << 8) | kErrResponse);
                        }
                        place_c = false;
                    }
                }

                // ---- a8: arg-best over the tile: highest f, then lowest node index ----
                int best;
                if (LEMIX && NPL == 1) {
                    // one node per lane (node = tile lane): the tile max of f by a
                    // butterfly, then the lowest lane holding it (a ballot) -- the
                    // same total order (f desc, node asc; +0 == -0, no NaN: R > 0)
                    const bool valid = n_best != INT_MAX;
                    double fm = valid ? f_best : -kInf;
#pragma unroll
                    for (int off = T >> 1; off > 0; off >>= 1) fm = dev::dmax(fm, dev::shfl_xor_w(fm, off, T));
                    const unsigned hit = __ballot_sync(0xffffffffu, valid && f_best == fm);
                    const unsigned seg = (hit >> tbase) & (T == 32 ? 0xffffffffu : ((1u << T) - 1u));
                    best = seg ? __ffs(seg) - 1 : 0;   // (empty only off the live path)
                } else if (LEMIX) {
#pragma unroll
                    for (int off = T >> 1; off > 0; off >>= 1) {
                        const double f2 = dev::shfl_xor_w(f_best, off, T);
                        const int n2 = __shfl_xor_sync(0xffffffffu, n_best, off, T);
                        if (n2 != INT_MAX &&
                            (n_best == INT_MAX || f2 > f_best || (f2 == f_best && n2 < n_best))) {
                            f_best = f2;
                            n_best = n2;
                        }
                    }
                    best = n_best;
                } else {
                    best = chosen;
                }

                // ---- a10: commit on the owning lane ----
                const int owner = tbase + (best & (T - 1));
                const int osrc = best & (T - 1);        // owner within the tile
                const int jb = best >> log2T;
                double c_done = 0.0, c_en0 = 0.0, c_st0 = 0.0;
                int c_ver = 0, c_status = LMX_OK, c_mem = 0;
                if (place_c && lane == owner) {
#pragma unroll
                    for (int jj = 0; jj < NPL; ++jj) {
                        if (NPL == 1 || jj == jb) {   // (one slot: the owner lane's node)
                            double ef[SMAX], eb[SMAX];
                            prof.node<SMAX>(best, ef, eb);
                            const dev::RingT<W, wstride, MEM> q{rbe[jj], p.kmask, S, ws[jj], wstride, qh[jj] + qn[jj]};
                            const long long tok = (long long)task_batch(v) * l;   // activation tokens C*l
                            int offm = 0;
                            if (MEM) {
                                // Algorithm 2: the executed path replaces the plan (calibration)
                                double ex_st[SMAX];
                                int nw = 0;
                                dev::execute_mem<SMAX>(P[jj], hasp[jj] != 0, S, ef, q, qh[jj], qn[jj], w, tok, a,
                                                       p.mem_cap, p.mem_dt, p.mem_tmax, p.mem_pen, ex_st, en_s[jj],
                                                       offm, nw);
                                st0_s[jj] = ex_st[0];
                                c_mem = nw | (__popc(offm) << 8);
                            }
                            double bz[SMAX];   // busy[s] (PAPER.md:787 utilisation), forward first
#pragma unroll
                            for (int s = 0; s < SMAX; ++s)
                                if (s < S) {
                                    P[jj][s] = CB ? oc_s[jj][s] : en_s[jj][s];   // (CB: busy through the decode steps)
                                    const double dFs = ef[s] * w;
                                    const double dur = (MEM && ((offm >> s) & 1)) ? dFs + p.mem_pen * (double)tok : dFs;
                                    bz[s] = dev::lds_d(c_busy(jj, s)) + dur;
                                    if (CB) bz[s] = bz[s] + prof.d(best, s) * (double)wd;   // the decode steps
                                }
                            const long long trv = dev::lds_l(c_ntr(jj));
                            int ntr = (int)(trv & 0xffffffffll), vp = (int)(trv >> 32);
                            hasp[jj] = 1;
                            if (SCOLD) dev::sts_d(c_sc(jj, 0), a); else aprev[jj] = a;
                            c_en0 = en_s[jj][0];
                            c_st0 = st0_s[jj];
                            c_done = dev::last_of(en_s[jj], S);
                            if (is_train && qn[jj] >= p.qcap) {
                                c_status = LMX_EQCAP;
                                c_ver = INT_MIN;   // (a version count is never negative)
                            } else if (is_train) {
                                // backward planning, stages S..1
                                double2 bw[SMAX];
                                double db[SMAX];
                                double x = c_done;
#pragma unroll
                                for (int s = SMAX - 1; s >= 0; --s) {
                                    bw[s] = make_double2(0.0, 0.0);
                                    db[s] = 0.0;
                                    if (s < S) {
                                        const double sb = dev::dmax(x, dev::lds_d(c_lb(jj, s)));
                                        db[s] = eb[s] * w;                 // dB_s (also line 16's offset)
                                        const double ebv = sb + db[s];
                                        dev::sts_d(c_lb(jj, s), ebv);
                                        bw[s] = make_double2(sb, ebv);
                                        x = ebv;
                                    }
                                }
                                q.push<SMAX>(qh[jj], bw, db, make_double2((double)tok, (double)offm));
                                qn[jj]++;
#pragma unroll
                                for (int s = 0; s < SMAX; ++s)
                                    if (s < S) bz[s] = bz[s] + eb[s] * w;
                                ntr++;
                                c_done = x;
                            } else {
                                // version-at-inference: completed backwards form a prefix of
                                // Q_train; start_f^1 of successive commits on a node is
                                // non-decreasing, so the boundary pointer only moves forward.
                                int k = vp > qh[jj] ? vp : qh[jj];
                                const int tail = qh[jj] + qn[jj];
                                while (k < tail && q.at(k, 0).y <= c_st0) k++;
                                vp = k;
                                c_ver = ntr - (tail - k);
                                if (!LEMIX && p.sync_sep) {
                                    // Separate: training count of the newest checkpoint loaded
                                    // by this forward start (DESIGN.md R-sync): the list holds
                                    // suffix minima of the load times, non-decreasing, so the
                                    // count of entries <= start_f^1 is that checkpoint's index
                                    int lo_k = 0, hi_k = n_ck;
                                    while (lo_k < hi_k) {
                                        const int mid = (lo_k + hi_k) >> 1;
                                        if (ckt[mid] <= c_st0) lo_k = mid + 1; else hi_k = mid;
                                    }
                                    c_ver = lo_k * p.sync_interval;
                                }
                            }
#pragma unroll
                            for (int s = 0; s < SMAX; ++s)
                                if (s < S) dev::sts_d(c_busy(jj, s), bz[s]);
                            dev::sts_l(c_ntr(jj), (long long)(unsigned)ntr | ((long long)vp << 32));
                            {
                                // cached Eq. 2 statistics (DESIGN.md R-stat), computed
                                // speculatively above; unused while cnt < 2.  (Also on a
                                // queue overflow: that trace stops, its state is dead.)
                                cnt[jj] += CB ? mb : 1;
                                dev::sts_l(c_sl(jj), sl_n[jj]);
                                dev::sts_l(c_sl2(jj), sl2_n[jj]);
                                if (SCOLD) {
                                    dev::sts_d(c_sc(jj, 1), mu_n[jj]);
                                    dev::sts_d(c_sc(jj, 2), kk_n[jj]);
                                    dev::sts_d(c_sc(jj, 3), cc_n[jj]);
                                } else {
                                    mu[jj] = mu_n[jj];
                                    kk[jj] = kk_n[jj];
                                    cc[jj] = cc_n[jj];
                                }
                            }
                        }
                    }
                }
                c_done = dev::shfl_w(c_done, osrc, T);
                c_en0 = dev::shfl_w(c_en0, osrc, T);
                if (p.node_defer) c_st0 = dev::shfl_w(c_st0, osrc, T);
                c_ver = __shfl_sync(0xffffffffu, c_ver, osrc, T);
                if (MEM) {
                    c_mem = __shfl_sync(0xffffffffu, c_mem, osrc, T);
                    if (place_c && c_ver != INT_MIN) { n_mwait += c_mem & 0xff; n_moff += c_mem >> 8; }
                }
                if (!place_c) {
                } else if (c_ver == INT_MIN) {
                    status = LMX_EQCAP;
                } else if (CB && !is_train) {
                    // ---- a11 for a batch (R-cb): every member's first token at the
                    // prefill end, its last after its own decode steps; TTFT, SLO,
                    // TBT per member, in member order ----
                    const double edS = prof.d(best, S - 1);
                    const long long o0 = dev::lds_l(c_tw(1)) + i;
                    for (int k = 0; k < mb; ++k) {
                        const double ar = __ldg(tarr + i + k);
                        const uint32_t vk = __ldg(tlbk + i + k);
                        const long long ok = __ldg(p.out_len + o0 + k);
                        // decode work up to its last step: sum_j g(min(out_k, out_j))
                        long long wk = 0;
                        for (int jm = 0; jm < mb; ++jm) {
                            const long long oj = __ldg(p.out_len + o0 + jm);
                            const long long mn = oj < ok ? oj : ok;
                            wk += mn * (lpad - 1) + mn * (mn + 1) / 2;
                        }
                        const double dec = edS * (double)wk;
                        const double fin = c_done + dec;
                        const double ttft = c_done - ar;
                        double tauR;
                        if (p.slo_mode == 1) {
                            tauR = p.slo_const;
                        } else {
                            const double wk2 = task_w(vk);
                            double acc = 0.0;
#pragma unroll
                            for (int s = 0; s < SMAX; ++s)
                                if (s < S) acc = acc + ef0[s] * wk2;
                            tauR = p.slo_mult * acc;
                        }
                        sum_ttft = sum_ttft + ttft;
                        n_slo += (ttft <= tauR) ? 1 : 0;
                        sum_ver += c_ver;
                        if (ok >= 1) {
                            sum_tbt = sum_tbt + dec / (double)ok;
                            n_tbt++;
                        }
                        t_last = dev::dmax(t_last, fin);
                        if (tl == 0 && p.node_defer) {
                            p.node_defer[o0 + k] = (uint32_t)best;
                            p.decision_idx[o0 + k] = step;
                            p.completion[o0 + k] = fin;
                            p.start_f1[o0 + k] = c_st0;
                        }
                    }
                    n_batches++;
                    step++;
                    a_last_inf = __ldg(tarr + i + mb - 1);
                    i += mb;
                    a_inf = (i < nI) ? __ldg(tarr + i) : 0.0;
                    v_inf = (i < nI) ? __ldg(tlbk + i) : 0u;
                    a_inf2 = (i + 1 < nI) ? __ldg(tarr + i + 1) : 0.0;
                    v_inf2 = (i + 1 < nI) ? __ldg(tlbk + i + 1) : 0u;
                } else {
                    // ---- a11: outputs + per-trace folds ----
                    if (tl == 0 && p.node_defer) {
                        const long long o = dev::lds_l(c_tw(1));
                        const unsigned dsat = is_train ? (unsigned)min(cur_defer, 0xFFFF) : 0u;
                        p.node_defer[o + task] = (uint32_t)best | (dsat << 16);
                        p.decision_idx[o + task] = step;
                        p.completion[o + task] = c_done;
                        p.start_f1[o + task] = c_st0;
                    }
                    t_last = dev::dmax(t_last, c_done);
                    step++;
                    // both kinds' folds as selects (no divergence between tiles
                    // that placed a training and an inference task)
                    const bool inf = !is_train;
                    const double ttft = c_done - a_inf;        // R from arrival
                    double tauR;
                    if (p.slo_mode == 1) {
                        tauR = p.slo_const;
                    } else {
                        double acc = 0.0;
#pragma unroll
                        for (int s = 0; s < SMAX; ++s)
                            if (s < S) acc = acc + ef0[s] * w;
                        tauR = p.slo_mult * acc;
                    }
                    const double sum_ttft_n = sum_ttft + ttft;
                    sum_ttft = inf ? sum_ttft_n : sum_ttft;
                    n_slo += (inf && ttft <= tauR) ? 1 : 0;   // SLO: TTFT <= 5x forward latency
                    sum_ver += inf ? c_ver : 0;
                    a_last_inf = inf ? a_inf : a_last_inf;
                    i += inf ? 1 : 0;
                    j += inf ? 0 : 1;
                    cur_defer = inf ? cur_defer : 0;
                    // the consumed stream advances; its task two ahead was loaded above
                    a_inf = inf ? a_inf2 : a_inf;
                    v_inf = inf ? v_inf2 : v_inf;
                    a_inf2 = inf ? pf_a : a_inf2;
                    v_inf2 = inf ? pf_v : v_inf2;
                    a_tr = inf ? a_tr : a_tr2;
                    v_tr = inf ? v_tr : v_tr2;
                    a_tr2 = inf ? a_tr2 : pf_a;
                    v_tr2 = inf ? v_tr2 : pf_v;
                    if (!LEMIX && p.sync_sep && !inf && j % p.sync_interval == 0) {
                        // Separate: checkpoint after this training task's backward, loaded
                        // sync_latency later (R-sync); every lane of the tile
                        // writes the same values (each reads back only its own writes)
                        const double av = c_done + p.sync_latency;
                        ckt[n_ck] = av;
                        for (int k = n_ck - 1; k >= 0 && ckt[k] > av; --k) ckt[k] = av;   // suffix minima
                        n_ck++;
                    }
                    // next release: max(a_min, this task's S1 forward end)
                    const double r_n = (j < nT) ? dev::dmax(a_tr, c_en0) : kInf;
                    r = inf ? r : r_n;
                }
            }
        }
    }
}


typedef void (*kernel_fn)(const KParams);

template <int SMAX, bool EXACT, bool LEMIX, int MODE>
kernel_fn pick_npl(int npl)
{
    switch (npl) {
    case 1: return event_loop_kernel<SMAX, EXACT, 1, LEMIX, 0, MODE>;
    case 2: return event_loop_kernel<SMAX, EXACT, 2, LEMIX, 0, MODE>;
    default: return event_loop_kernel<SMAX, EXACT, 4, LEMIX, 0, MODE>;
    }
}

template <bool LEMIX, int MODE>
kernel_fn pick(const KParams &p)
{
    const int nb = npl_bucket(p.npl);
    switch (stages_bucket(p.S)) {
    case 1: return pick_npl<1, true, LEMIX, MODE>(nb);
    case 2:
        // the bench shape (4 nodes x 2 stages): tile width fixed at compile time
        if (p.S == 2 && nb == 1 && p.T == 4 && !p.cell_par) return event_loop_kernel<2, true, 1, LEMIX, 4, MODE>;
        return p.S == 2 ? pick_npl<2, true, LEMIX, MODE>(nb) : pick_npl<2, false, LEMIX, MODE>(nb);
    case 4: return p.S == 4 ? pick_npl<4, true, LEMIX, MODE>(nb) : pick_npl<4, false, LEMIX, MODE>(nb);
    case 8: return p.S == 8 ? pick_npl<8, true, LEMIX, MODE>(nb) : pick_npl<8, false, LEMIX, MODE>(nb);
    default: return p.S == 16 ? pick_npl<16, true, LEMIX, MODE>(nb) : pick_npl<16, false, LEMIX, MODE>(nb);
    }
}

}  // namespace tile
}  // namespace lmx
