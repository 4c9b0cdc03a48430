// lemix_lane.cuh -- lane-per-trace persistent event-loop kernel (small
// clusters: N <= NMAX nodes, S = SMAX stages), the default for the MC / sweep /
// tiny shapes (N = 4, S = 2).
//
// One thread owns one trace at a time and plans + scores all N candidate
// nodes itself (Algorithm 1; Eq. 1-3), the
// candidate loop fully unrolled: the N plans are N independent dependency
// chains the scheduler interleaves (instruction-level parallelism instead of
// lanes), the arg-best is an in-order scan (highest f, lowest
// index on ties), the commit and the Eq. 2 statistics are done once, by the
// trace's own thread, and nothing is replicated or masked: a warp advances 32
// traces per iteration with no shuffles.  (The tile kernel, lemix_tile.cuh,
// spreads one trace's candidates over T lanes; it serves the larger N.)
//
// State placement, per thread:
//   registers : per node the previous forward ends P[s], Q_train^n head and
//               length, stale-prefix pointers and their cached end_b, a_[-1],
//               the cached Eq. 2 statistics (mu, 1/(2 sigma^2), 1/(sigma
//               sqrt(2 pi))) and the task count; the per-trace folds;
//   shared    : the TMA-staged profile, per node the newest kW Q_train entries
//               (a tail window, one 16-byte column per thread) and the
//               commit-only words (last backward end per stage, busy time,
//               length sums, training count | version pointer), one 8-byte
//               column per thread (no bank conflicts);
//   global    : Q_train entries older than the window (spilled on eviction).
// The block is 128 threads and 2 blocks share an SM (8 warps), so the register
// budget is 255 per thread and the per-node state never spills.
//
// Arithmetic is identical, operation by operation, to the oracle and the tile
// kernel (--fmad=false).
#pragma once
#include <cuda_runtime.h>

#include <climits>
#include <cmath>

#include "lemix_device.cuh"
#include "lemix_internal.h"

#ifndef LMX_LANE_MINB
#define LMX_LANE_MINB 2
#endif
#ifndef LMX_LANE_W
#define LMX_LANE_W 2                        // tail-window entries per node in shared memory
#endif

namespace lmx {
namespace lane {

constexpr int kBlock = 128;
constexpr int kW = LMX_LANE_W;
constexpr int kTraceWords = 4;              // trace index, first task offset, t_first, error
using dev::dmax;
using dev::dmin;
using dev::kInf;
using dev::task_batch;
using dev::task_len;
using dev::task_w;

__host__ __device__ constexpr inline int cold_words(int S) { return 2 * S + 3; }

// dynamic shared memory of one block
__host__ inline int smem_bytes(int N, int S, int NMAX)
{
    return 16 * N * S + NMAX * kW * ring_words(S) * 16 * kBlock + (NMAX * cold_words(S) + kTraceWords) * 8 * kBlock;
}

template <int NMAX, int SMAX, bool LEMIX>
__global__ void __launch_bounds__(kBlock, LMX_LANE_MINB) lane_kernel(const KParams p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t s_bar;
    constexpr int S = SMAX;
    constexpr int RW = ring_words(SMAX);
    constexpr uint32_t wstride = 16u * kBlock;   // bytes between a thread's consecutive window words
    constexpr uint32_t cstride = 8u * kBlock;    // bytes between a thread's consecutive cold words
    constexpr int CW = cold_words(SMAX);
    const int N = p.N, NS = p.N * S;

    // ---- K1: stage eta_f | eta_b (16*N*S bytes) into shared memory via TMA ----
    double *s_eta = reinterpret_cast<double *>(smem_raw);
    if (threadIdx.x == 0) {
        dev::mbar_init(&s_bar, 1);
        dev::mbar_arrive_expect_tx(&s_bar, 16u * (uint32_t)NS);
        dev::bulk_copy_g2s(s_eta, p.eta, 16u * (uint32_t)NS, &s_bar);
    }
    __syncthreads();
    dev::mbar_wait(&s_bar, 0);
    uint32_t s_eta_u = dev::smem_u32(s_eta);
    dev::opaque(s_eta_u);
    const dev::SmemProfile prof{s_eta_u, NS, S};
    double ef0[SMAX];   // eta_F of node 0, for tau_R (R-16)
#pragma unroll
    for (int s = 0; s < SMAX; ++s) ef0[s] = prof.f(0, s);

    // ---- per-thread shared-memory columns ----
    const int tid = threadIdx.x;
    const long long gthread = (long long)blockIdx.x * kBlock + tid;
    const long long K = (long long)p.kmask + 1;
    uint32_t wbase0 = dev::smem_u32(smem_raw) + 16u * (uint32_t)NS + 16u * tid;   // window of node 0
    dev::opaque(wbase0);
    constexpr uint32_t wnode = (uint32_t)(kW * RW) * wstride;                    // node-to-node window offset
    uint32_t cbase = dev::smem_u32(smem_raw) + 16u * (uint32_t)NS + (uint32_t)NMAX * wnode + 8u * tid;
    dev::opaque(cbase);
    auto c_lb = [&](int n, int s) { return cbase + (uint32_t)(n * CW + s) * cstride; };
    auto c_busy = [&](int n, int s) { return cbase + (uint32_t)(n * CW + S + s) * cstride; };
    auto c_sl = [&](int n) { return cbase + (uint32_t)(n * CW + 2 * S) * cstride; };
    auto c_sl2 = [&](int n) { return cbase + (uint32_t)(n * CW + 2 * S + 1) * cstride; };
    auto c_ntr = [&](int n) { return cbase + (uint32_t)(n * CW + 2 * S + 2) * cstride; };   // training count | version ptr << 32
    auto c_tw = [&](int k) { return cbase + (uint32_t)(NMAX * CW + k) * cstride; };
    double2 *ring0 = p.ring_be + gthread * NMAX * K * RW;                        // global ring of node 0
    dev::opaque_ptr(ring0);
    // Q_train^n of node n (window over the global ring); tail = head + length
    auto queue = [&](int n, int tail) {
        return dev::RingT<kW, wstride, false>{ring0 + (long long)n * K * RW, p.kmask, S, wbase0 + (uint32_t)n * wnode,
                                              wstride, tail};
    };

    // ---- per-trace state ----
    bool active = false, finished = false;
    const double *tarr = p.arrival;
    const uint32_t *tlbk = p.lbk;
    int nI = 0, nT = 0, i = 0, j = 0, step = 0, iters = 0, rr = 0, sep_i = 0, sep_t = 0;
    int rate_lo = 0, rate_hi = 0, cur_defer = 0, status = LMX_OK, n_slo = 0, n_def = 0, n_ck = 0;
    double r = kInf, t_last = -kInf, a_last_inf = -kInf, sum_ttft = 0.0;
    long long sum_ver = 0;
    double *ckt = (!LEMIX && p.sync_sep) ? p.ck + gthread * p.ck_cap : nullptr;
    double a_inf = 0.0, a_inf2 = 0.0, a_tr = 0.0, a_tr2 = 0.0;   // 2-deep input prefetch
    uint32_t v_inf = 0, v_inf2 = 0, v_tr = 0, v_tr2 = 0;

    // ---- per-node state (registers) ----
    double P[NMAX][SMAX], skeb[NMAX][SMAX], aprev[NMAX], mu[NMAX], kk[NMAX], cc[NMAX];
    int qh[NMAX], qn[NMAX], cnt[NMAX], sk[NMAX][SMAX];
    unsigned hasp = 0;   // bit n: node n has run a task

    while (!__all_sync(0xffffffffu, finished)) {
        if (!finished && !active) {
            // ---- claim the next trace ----
            const unsigned long long tt = atomicAdd(p.work, 1ull);
            if (tt >= (unsigned long long)p.n_traces) {
                finished = true;
            } else {
                const long long t = (long long)tt;
                const long long o = p.offsets[t];
                const int len = (int)(p.offsets[t + 1] - o);
                dev::wait_inputs(p.ready, p.chunk_tasks, o, o + len);
                nI = p.n_inf[t];
                nT = len - nI;
                tarr = p.arrival + o;
                tlbk = p.lbk + o;
                i = j = step = iters = rr = sep_i = sep_t = cur_defer = rate_lo = rate_hi = 0;
                n_slo = n_def = n_ck = 0;
                status = LMX_OK;
                sum_ver = 0;
                sum_ttft = 0.0;
                t_last = -kInf;
                a_last_inf = -kInf;
                dev::sts_l(c_tw(0), t);
                dev::sts_l(c_tw(1), o);
                dev::sts_l(c_tw(3), kErrNone);
                if (nI > 0) { a_inf = __ldg(tarr); v_inf = __ldg(tlbk); }
                if (nI > 1) { a_inf2 = __ldg(tarr + 1); v_inf2 = __ldg(tlbk + 1); }
                if (nT > 0) { a_tr = __ldg(tarr + nI); v_tr = __ldg(tlbk + nI); }
                if (nT > 1) { a_tr2 = __ldg(tarr + nI + 1); v_tr2 = __ldg(tlbk + nI + 1); }
                r = (nT > 0) ? a_tr : kInf;
                double t_first = kInf;
                if (nI > 0) t_first = dmin(t_first, a_inf);
                if (nT > 0) t_first = dmin(t_first, a_tr);
                dev::sts_d(c_tw(2), t_first);
                hasp = 0;
#pragma unroll
                for (int n = 0; n < NMAX; ++n) {
                    qh[n] = qn[n] = cnt[n] = 0;
                    aprev[n] = mu[n] = kk[n] = cc[n] = 0.0;
                    dev::sts_l(c_sl(n), 0);
                    dev::sts_l(c_sl2(n), 0);
                    dev::sts_l(c_ntr(n), 0);
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) {
                        P[n][s] = 0.0;
                        sk[n][s] = 0;
                        skeb[n][s] = 0.0;
                        dev::sts_d(c_lb(n, s), -kInf);
                        dev::sts_d(c_busy(n, s), 0.0);
                    }
                }
                if (!LEMIX && p.policy == LMX_SEPARATE && N == 1 && nI > 0 && nT > 0) {
                    status = LMX_EINVAL;
                    dev::sts_l(c_tw(3), kErrSeparateN1);
                }
                active = true;
            }
        }
        const bool more = active & ((i < nI) | (j < nT));
        iters += more;
        if (more & (iters > 2 * (nI + nT) + 2)) status = LMX_EBUDGET;
        const bool done_trace = active & ((status != LMX_OK) | !more);

        if (done_trace) {
            // ---- per-trace metrics, node folds in node order ----
            lmx_summary sm;
            sm.n_tasks = nI + nT;
            sm.n_inf = nI;
            sm.n_train = nT;
            sm.status = status;
            sm.n_slo_met = sm.n_deferrals = sm.active_nodes = sm.sum_version = 0;
            sm.n_mem_wait = sm.n_offload = 0;
            sm.makespan = sm.throughput = sm.sum_ttft = sm.mean_ttft = sm.slo_attainment = 0.0;
            sm.mean_util = sm.mean_len_std = 0.0;
            if (status == LMX_OK) {
                const int ntask = nI + nT;
                sm.n_slo_met = n_slo;
                sm.n_deferrals = n_def;
                sm.sum_version = sum_ver;
                sm.sum_ttft = sum_ttft;
                sm.makespan = (ntask > 0) ? t_last - dev::lds_d(c_tw(2)) : 0.0;
                sm.throughput = (sm.makespan > 0.0) ? (double)ntask / sm.makespan : 0.0;
                sm.mean_ttft = (nI > 0) ? sum_ttft / (double)nI : 0.0;
                sm.slo_attainment = (nI > 0) ? (double)n_slo / (double)nI : 1.0;
                double U = 0.0, stds = 0.0;
                long long act = 0;
#pragma unroll
                for (int n = 0; n < NMAX; ++n) {
                    if (n < N) {
#pragma unroll
                        for (int s = 0; s < SMAX; ++s) U = U + dev::lds_d(c_busy(n, s));
                        const long long c = cnt[n], a1 = dev::lds_l(c_sl(n)), a2 = dev::lds_l(c_sl2(n));
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
            const long long tt = dev::lds_l(c_tw(0));
            p.summaries[tt] = sm;
            if (status != LMX_OK) {
                p.trace_err[tt] = dev::lds_l(c_tw(3));
                atomicMin(p.first_bad, (unsigned long long)tt);
            }
            active = false;
        }

        if (active) {
            // ---- a1: event selection (ties -> inference) ----
            const double t_inf = (i < nI) ? a_inf : kInf;
            const bool is_train = !(t_inf <= r);
            const double now = is_train ? r : t_inf;
            const uint32_t v = is_train ? v_tr : v_inf;
            // the input two ahead in the consumed stream, loaded now so it
            // lands while the decision runs (discarded when the task is deferred)
            const int pf_idx = is_train ? nI + min(j + 2, nT - 1) : min(i + 2, nI - 1);
            const double pf_a = __ldg(tarr + pf_idx);
            const uint32_t pf_v = __ldg(tlbk + pf_idx);
            bool deferred = false;
            if (LEMIX && is_train && p.deprioritize && i < nI) {
                // ---- a2: Eq. 4 against the next enqueued inference task
                // (R-14/R-15) ----
                const double wn = task_w(v_inf);
                double m = kInf;
#pragma unroll
                for (int n = 0; n < NMAX; ++n)
                    if (n < N) {
                        const double latest = ((hasp >> n) & 1u) ? P[n][S - 1] : -kInf;
                        m = dmin(m, latest + prof.f(n, S - 1) * wn);
                    }
                double tauR;
                if (p.slo_mode == 1) {
                    tauR = p.slo_const;
                } else {
                    double acc = 0.0;
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) acc = acc + ef0[s] * wn;
                    tauR = p.slo_mult * acc;
                }
                deferred = (m - t_inf) > tauR;
                if (deferred) {
                    r = t_inf;          // move behind the next inference task
                    cur_defer++;
                    n_def++;
                }
            }
            const int task = is_train ? nI + j : i;
            if (!deferred) {
                // ---- input validation of the task being placed ----
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
                if (ok) {
                    const double a = now;                    // dispatch time (R-2)
                    const double w = task_w(v);
                    const int l = task_len(v);
                    const long long cslot = p.cand ? (dev::lds_l(c_tw(1)) + step) * N : 0;
                    double en_b[SMAX], st0_b = 0.0;
                    int best = 0;
                    bool r_bad = false;
                    if (LEMIX) {
                        // ---- a3-a7: Algorithm 1 + Eq. 1-3 on every node (independent chains) ----
                        double f[NMAX], en[NMAX][SMAX], st0[NMAX];
#pragma unroll
                        for (int n = 0; n < NMAX; ++n) {
                            f[n] = -kInf;
                            st0[n] = 0.0;
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) en[n][s] = 0.0;
                            if (n < N) {
                                // Eq. 2: cold nodes take lc0; exp_neg is
                                // evaluated anyway (finite for t >= 0) and discarded
                                const double d = (double)l - mu[n];
                                const double lw = cc[n] * dev::exp_neg((d * d) * kk[n]);
                                const double LC = (cnt[n] < 2) ? p.lc0 : lw;
                                double efn[SMAX], ebn[SMAX], II;
                                int gc;
                                prof.node<SMAX>(n, efn, ebn);
                                const auto q = queue(n, qh[n] + qn[n]);
                                dev::plan<SMAX, false>(P[n], (hasp >> n) & 1u, S, efn, ebn, q, qh[n], qn[n], sk[n],
                                                       skeb[n], w, a, now, en[n], st0[n], II, gc);
                                qh[n] += gc;                     // lines 17-18: executed entries leave Q_train^n
                                qn[n] -= gc;
                                const double R = en[n][S - 1] - a;                                // line 20
                                const double a_last = ((hasp >> n) & 1u) ? aprev[n] : a;          // R-9
                                const double IIS = p.s_pow2 ? II * p.inv_S : II / (double)S;      // exact either way
                                const double IP = -dmax(IIS - (a - a_last), p.tau);              // Eq. 1
                                f[n] = (IP + p.lambda2 * LC) / (p.lambda1 * R);                  // Eq. 3
                                r_bad |= !(R > 0.0);
                                if (p.cand) dev::put_cand(p.cand, cslot + n, II, R, f[n]);
                            }
                        }
                        // ---- a8: highest f, ties -> lowest node index (strict >) ----
                        double fb = f[0];
#pragma unroll
                        for (int n = 1; n < NMAX; ++n)
                            if (n < N && f[n] > fb) { fb = f[n]; best = n; }
                        st0_b = st0[0];
#pragma unroll
                        for (int s = 0; s < SMAX; ++s) en_b[s] = en[0][s];
#pragma unroll
                        for (int n = 1; n < NMAX; ++n)
                            if (n == best) {
                                st0_b = st0[n];
#pragma unroll
                                for (int s = 0; s < SMAX; ++s) en_b[s] = en[n][s];
                            }
                    } else {
                        // ---- a9: baseline selectors, then Alg. 1 there ----
                        if (p.policy == LMX_RR) {
                            best = rr % N;
                            rr++;
                        } else if (p.policy == LMX_SEPARATE) {
                            if (!(nI > 0 && nT > 0)) {
                                best = is_train ? (sep_t++ % N) : (sep_i++ % N);
                            } else {
                                int ninf = N - p.n_tr_sep;
                                if (p.sep_dynamic) {
                                    // SeparateDynamic (R-sepdyn)
                                    while (rate_hi < nI && __ldg(tarr + rate_hi) <= now) rate_hi++;
                                    const double w_lo = now - p.dyn_window;
                                    while (rate_lo < nI && __ldg(tarr + rate_lo) <= w_lo) rate_lo++;
                                    const double rate = (double)(rate_hi - rate_lo) / p.dyn_window;
                                    ninf = (rate < p.dyn_rate) ? (N / 4 > 1 ? N / 4 : 1) : ninf;
                                }
                                best = is_train ? ninf + (sep_t++ % (N - ninf)) : (sep_i++ % ninf);
                            }
                        } else {
                            best = fx;
                        }
                        double Pc[SMAX], skebc[SMAX], efn[SMAX], ebn[SMAX], II;
                        int skc[SMAX], qhc = 0, qnc = 0, gc;
#pragma unroll
                        for (int s = 0; s < SMAX; ++s) { Pc[s] = 0.0; skebc[s] = 0.0; skc[s] = 0; }
#pragma unroll
                        for (int n = 0; n < NMAX; ++n)
                            if (n == best) {
                                qhc = qh[n];
                                qnc = qn[n];
#pragma unroll
                                for (int s = 0; s < SMAX; ++s) { Pc[s] = P[n][s]; skc[s] = sk[n][s]; skebc[s] = skeb[n][s]; }
                            }
                        prof.node<SMAX>(best, efn, ebn);
                        const auto q = queue(best, qhc + qnc);
                        dev::plan<SMAX, false>(Pc, (hasp >> best) & 1u, S, efn, ebn, q, qhc, qnc, skc, skebc, w, a,
                                               now, en_b, st0_b, II, gc);
#pragma unroll
                        for (int n = 0; n < NMAX; ++n)
                            if (n == best) {
                                qh[n] = qhc + gc;
                                qn[n] = qnc - gc;
#pragma unroll
                                for (int s = 0; s < SMAX; ++s) { sk[n][s] = skc[s]; skeb[n][s] = skebc[s]; }
                            }
                        if (p.cand)
                            dev::put_cand(p.cand, cslot + best, II, en_b[S - 1] - a, __longlong_as_double(-1ll));
                    }

                    if (r_bad) {
                        // R <= 0 (a forward too short to move the clock): Eq. 3 is
                        // undefined; the trace stops, as in the oracle
                        status = LMX_EINVAL;
                        dev::sts_l(c_tw(3), ((long long)task << 8) | kErrResponse);
                    } else {
                        // ---- a10: commit on node `best` ----
                        int qhb = 0, qnb = 0;
#pragma unroll
                        for (int n = 0; n < NMAX; ++n)
                            if (n == best) { qhb = qh[n]; qnb = qn[n]; }
                        const auto q = queue(best, qhb + qnb);
                        double efb[SMAX], ebb[SMAX];
                        prof.node<SMAX>(best, efb, ebb);
                        double bz[SMAX];   // busy[s] (PAPER.md:787 utilisation), forward first
#pragma unroll
                        for (int s = 0; s < SMAX; ++s) bz[s] = dev::lds_d(c_busy(best, s)) + efb[s] * w;
#pragma unroll
                        for (int n = 0; n < NMAX; ++n)
                            if (n == best) {
#pragma unroll
                                for (int s = 0; s < SMAX; ++s) P[n][s] = en_b[s];
                                aprev[n] = a;
                            }
                        hasp |= 1u << best;
                        const long long trv = dev::lds_l(c_ntr(best));
                        int ntr = (int)(trv & 0xffffffffll), vp = (int)(trv >> 32);
                        double c_done = en_b[S - 1];
                        int c_ver = 0;
                        if (is_train && qnb >= p.qcap) {
                            status = LMX_EQCAP;
                        } else if (is_train) {
                            // backward planning, stages S..1
                            double2 bw[SMAX];
                            double db[SMAX];
                            double x = c_done;
#pragma unroll
                            for (int s = SMAX - 1; s >= 0; --s) {
                                const double sb = dmax(x, dev::lds_d(c_lb(best, s)));
                                db[s] = ebb[s] * w;                 // dB_s (also line 16's offset)
                                const double ebv = sb + db[s];
                                dev::sts_d(c_lb(best, s), ebv);
                                bw[s] = make_double2(sb, ebv);
                                x = ebv;
                            }
                            q.push<SMAX>(qhb, bw, db);
#pragma unroll
                            for (int n = 0; n < NMAX; ++n)
                                if (n == best) qn[n] = qnb + 1;
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) bz[s] = bz[s] + ebb[s] * w;
                            ntr++;
                            c_done = x;
                        } else {
                            // version-at-inference: completed backwards form a prefix of
                            // Q_train; start_f^1 of successive commits on a node is
                            // non-decreasing, so the boundary pointer only moves forward
                            int k = vp > qhb ? vp : qhb;
                            const int tail = qhb + qnb;
                            while (k < tail && q.at(k, 0).y <= st0_b) k++;
                            vp = k;
                            c_ver = ntr - (tail - k);
                            if (!LEMIX && p.sync_sep) {
                                // Separate: training count of the newest checkpoint loaded by
                                // this forward start (DESIGN.md R-sync; suffix minima, sorted)
                                int lo_k = 0, hi_k = n_ck;
                                while (lo_k < hi_k) {
                                    const int mid = (lo_k + hi_k) >> 1;
                                    if (ckt[mid] <= st0_b) lo_k = mid + 1; else hi_k = mid;
                                }
                                c_ver = lo_k * p.sync_interval;
                            }
                        }
                        if (status == LMX_OK) {
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) dev::sts_d(c_busy(best, s), bz[s]);
                            dev::sts_l(c_ntr(best), (long long)(unsigned)ntr | ((long long)vp << 32));
                            // Eq. 2 history of the chosen node and its cached statistics
                            // (DESIGN.md R-stat; unused while the count is below 2)
                            const long long a1 = dev::lds_l(c_sl(best)) + l;
                            const long long a2 = dev::lds_l(c_sl2(best)) + (long long)l * l;
                            dev::sts_l(c_sl(best), a1);
                            dev::sts_l(c_sl2(best), a2);
                            int c = 0;
#pragma unroll
                            for (int n = 0; n < NMAX; ++n)
                                if (n == best) c = cnt[n] + 1;
                            const double inv_c = 1.0 / (double)c;
                            const double mu_n = (double)a1 * inv_c;
                            const long long var = (long long)c * a2 - a1 * a1;
                            const double sigma = dmax(sqrt((double)var) * inv_c, p.sigma_floor);
                            const double inv_s = 1.0 / sigma;
                            const double kk_n = (0.5 * inv_s) * inv_s;
                            const double cc_n = inv_s * dev::kInvSqrt2Pi;
#pragma unroll
                            for (int n = 0; n < NMAX; ++n)
                                if (n == best) { cnt[n] = c; mu[n] = mu_n; kk[n] = kk_n; cc[n] = cc_n; }

                            // ---- a11: outputs + per-trace folds ----
                            if (p.node_defer) {
                                const long long o = dev::lds_l(c_tw(1));
                                const unsigned dsat = is_train ? (unsigned)min(cur_defer, 0xFFFF) : 0u;
                                p.node_defer[o + task] = (uint32_t)best | (dsat << 16);
                                p.decision_idx[o + task] = step;
                                p.completion[o + task] = c_done;
                                p.start_f1[o + task] = st0_b;
                            }
                            t_last = dmax(t_last, c_done);
                            step++;
                            const bool inf = !is_train;
                            const double ttft = c_done - a;            // R from arrival
                            double tauR;
                            if (p.slo_mode == 1) {
                                tauR = p.slo_const;
                            } else {
                                double acc = 0.0;
#pragma unroll
                                for (int s = 0; s < SMAX; ++s) acc = acc + ef0[s] * w;
                                tauR = p.slo_mult * acc;
                            }
                            const double sum_ttft_n = sum_ttft + ttft;
                            sum_ttft = inf ? sum_ttft_n : sum_ttft;
                            n_slo += (inf && ttft <= tauR) ? 1 : 0;   // SLO: TTFT <= 5x forward latency
                            sum_ver += inf ? c_ver : 0;
                            a_last_inf = inf ? a : a_last_inf;
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
                                // Separate: checkpoint after this training task's backward,
                                // loaded sync_latency later (R-sync)
                                const double av = c_done + p.sync_latency;
                                ckt[n_ck] = av;
                                for (int k = n_ck - 1; k >= 0 && ckt[k] > av; --k) ckt[k] = av;   // suffix minima
                                n_ck++;
                            }
                            // next release: max(a_min, this task's S1 forward end)
                            const double r_n = (j < nT) ? dmax(a_tr, en_b[0]) : kInf;
                            r = inf ? r : r_n;
                        }
                    }
                }
            }
        }
    }
}

typedef void (*kernel_fn)(const KParams);

// the instantiations this translation unit carries (lemix_lane.cu)
template <bool LEMIX>
kernel_fn pick(const KParams &p)
{
    if (p.S == 2) return p.N <= 2 ? lane_kernel<2, 2, LEMIX> : lane_kernel<4, 2, LEMIX>;
    return p.N <= 2 ? lane_kernel<2, 1, LEMIX> : lane_kernel<4, 1, LEMIX>;
}

inline int nmax_bucket(int N) { return N <= 2 ? 2 : 4; }

}  // namespace lane
}  // namespace lmx
