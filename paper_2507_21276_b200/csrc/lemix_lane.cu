// lemix_lane.cu -- lane-per-trace variant of the persistent event loop
// (small clusters: N <= 8 nodes, S <= 4 stages).
//
// Each thread owns one trace at a time and sweeps all N candidate nodes itself
// with the candidate loop fully unrolled, so the N Algorithm-1 plans and Eq. 1-3
// scores are N independent dependency chains the scheduler can interleave
// (instruction-level parallelism instead of lanes), the arg-best is a plain
// in-order scan (lowest index wins ties) and the commit needs no
// shuffles.  A warp therefore advances 32 traces per step instead of 8, and
// no lane idles while one lane commits.
//
// State placement (per thread):
//   registers : per node the prev forward ends P[s] and the queue head/length;
//   shared    : profile table (TMA bulk copy), and per node a_[-1], the cached
//               Eq. 2 statistics, the stale-prefix / version pointers and the
//               commit-only state (last backward end per stage, busy time,
//               length sums), laid out [field][node][thread] (no bank
//               conflicts: each thread touches its own column);
//   global    : the Q_train^n rings (L1/L2 resident; only the head is hot).
//
// Arithmetic is identical, operation by operation, to lemix_kernels.cu and to
// the canonical expression sheet in DESIGN.md (--fmad=false).
#include <cuda_runtime.h>

#include <climits>
#include <cmath>

#include "lemix_device.cuh"
#include "lemix_internal.h"

namespace lmx {

namespace {

constexpr int kLaneBlock = 128;
#ifndef LMX_LANE_PF
#define LMX_LANE_PF true                    // up-front ring loads in Alg. 1 (see dev::plan)
#endif
#ifndef LMX_LANE_MINB
#define LMX_LANE_MINB 4   // resident CTAs/SM the register budget targets
#endif
using dev::dmax;
using dev::dmin;
using dev::kInf;
using dev::task_batch;
using dev::task_len;
using dev::task_w;

// shared-memory bytes per thread: doubles (LB, busy per stage; a_[-1], mu,
// 1/(2 sigma^2), 1/(sigma sqrt(2 pi))), 64-bit length sums, 32-bit ints
// (stale-prefix pointer per stage, version pointer, count, training count)
template <int NMAX, int SMAX>
struct LaneSmem {
    static constexpr int kDoubles = NMAX * (2 * SMAX + 4);
    static constexpr int kLongs = NMAX * 2;
    static constexpr int kInts = NMAX * (SMAX + 3);
    static constexpr int kBytesPerThread = 8 * (kDoubles + kLongs) + 4 * kInts;
};

template <int NMAX, int SMAX, bool EXACT>
__global__ void __launch_bounds__(kLaneBlock, LMX_LANE_MINB) lane_loop_kernel(const KParams p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t s_bar;

    // S is a compile-time constant when it equals the template bucket (EXACT)
    const int N = p.N, S = EXACT ? SMAX : p.S, NS = p.N * S;
    double *s_eta = reinterpret_cast<double *>(smem_raw);
    if (threadIdx.x == 0) {
        dev::mbar_init(&s_bar, 1);
        dev::mbar_arrive_expect_tx(&s_bar, 16u * (uint32_t)NS);
        dev::bulk_copy_g2s(s_eta, p.eta, 16u * (uint32_t)NS, &s_bar);
    }
    __syncthreads();
    dev::mbar_wait(&s_bar, 0);
    const double *s_ef = s_eta;
    const double *s_eb = s_eta + NS;
    double ef0[SMAX];   // eta_F of node 0, for tau_R (R-16)
#pragma unroll
    for (int s = 0; s < SMAX; ++s) ef0[s] = (s < S) ? s_ef[s] : 0.0;

    const int B = blockDim.x, tid = threadIdx.x;
    double *c_LB = s_eta + 2 * NS;                        // [SMAX][NMAX][B]
    double *c_busy = c_LB + SMAX * NMAX * B;              // [SMAX][NMAX][B]
    double *c_aprev = c_busy + SMAX * NMAX * B;           // [NMAX][B]
    double *c_mu = c_aprev + NMAX * B;
    double *c_kk = c_mu + NMAX * B;
    double *c_cc = c_kk + NMAX * B;
    long long *c_sl = reinterpret_cast<long long *>(c_cc + NMAX * B);
    long long *c_sl2 = c_sl + NMAX * B;
    int *c_sk = reinterpret_cast<int *>(c_sl2 + NMAX * B);   // [SMAX][NMAX][B]
    int *c_vp = c_sk + SMAX * NMAX * B;
    int *c_cnt = c_vp + NMAX * B;
    int *c_ntr = c_cnt + NMAX * B;
#define LB_(n, s) c_LB[((s) * NMAX + (n)) * B + tid]
#define BUSY_(n, s) c_busy[((s) * NMAX + (n)) * B + tid]
#define SK_(n, s) c_sk[((s) * NMAX + (n)) * B + tid]
#define APREV_(n) c_aprev[(n) * B + tid]
#define MU_(n) c_mu[(n) * B + tid]
#define KK_(n) c_kk[(n) * B + tid]
#define CC_(n) c_cc[(n) * B + tid]
#define SL_(n) c_sl[(n) * B + tid]
#define SL2_(n) c_sl2[(n) * B + tid]
#define VP_(n) c_vp[(n) * B + tid]
#define CNT_(n) c_cnt[(n) * B + tid]
#define NTR_(n) c_ntr[(n) * B + tid]

    const long long gthread = (long long)blockIdx.x * B + tid;
    const long long K = (long long)p.kmask + 1;
    const long long rb0 = gthread * NMAX * K;               // ring of node n: rb0 + n*K
    double2 *ring_be = p.ring_be;   // written in this kernel: coherent loads only

    // ---- hot per-node state (registers) ----
    double P[NMAX][SMAX];
    int qh[NMAX], qn[NMAX];
    unsigned hasp = 0, warm = 0;   // bit n: node n ran a task / has >= 2 tasks of history

    for (;;) {
        // ---- claim a trace ----
        const unsigned long long tt = atomicAdd(p.work, 1ull);
        if (tt >= (unsigned long long)p.n_traces) break;
        const long long t = (long long)tt;
        const long long o = p.offsets[t];
        const int nI = p.n_inf[t];
        const int nT = (int)(p.offsets[t + 1] - o) - nI;
        dev::wait_inputs(p.ready, p.chunk_tasks, o, o + nI + nT);

        int i = 0, j = 0, step = 0, iters = 0, rr = 0, sep_i = 0, sep_t = 0, cur_defer = 0;
        int n_ck = 0;   // Separate's checkpoints so far (sync model, DESIGN.md R-sync)
        int rate_lo = 0, rate_hi = 0;   // SeparateDynamic window pointers
        double *ckt = p.sync_sep ? p.ck + gthread * p.ck_cap : nullptr;
        int status = LMX_OK, err_task = 0, err_code = kErrNone;
        double t_last = -kInf, a_last_inf = -kInf, sum_ttft = 0.0;
        long long n_slo = 0, sum_ver = 0, n_def = 0;
        double a_inf = 0.0, a_inf2 = 0.0, a_tr = 0.0, a_tr2 = 0.0;
        uint32_t v_inf = 0, v_inf2 = 0, v_tr = 0, v_tr2 = 0;
        if (nI > 0) { a_inf = __ldg(p.arrival + o); v_inf = __ldg(p.lbk + o); }
        if (nI > 1) { a_inf2 = __ldg(p.arrival + o + 1); v_inf2 = __ldg(p.lbk + o + 1); }
        if (nT > 0) { a_tr = __ldg(p.arrival + o + nI); v_tr = __ldg(p.lbk + o + nI); }
        if (nT > 1) { a_tr2 = __ldg(p.arrival + o + nI + 1); v_tr2 = __ldg(p.lbk + o + nI + 1); }
        double r = (nT > 0) ? a_tr : kInf;
        double t_first = kInf;
        if (nI > 0) t_first = dmin(t_first, a_inf);
        if (nT > 0) t_first = dmin(t_first, a_tr);
        hasp = warm = 0;
#pragma unroll
        for (int n = 0; n < NMAX; ++n) {
            qh[n] = qn[n] = 0;
#pragma unroll
            for (int s = 0; s < SMAX; ++s) {
                P[n][s] = 0.0;
                LB_(n, s) = -kInf;
                BUSY_(n, s) = 0.0;
                SK_(n, s) = 0;
            }
            APREV_(n) = MU_(n) = KK_(n) = CC_(n) = 0.0;
            SL_(n) = 0;
            SL2_(n) = 0;
            VP_(n) = 0;
            CNT_(n) = 0;
            NTR_(n) = 0;
        }
        if (p.policy == LMX_SEPARATE && N == 1 && nI > 0 && nT > 0) {
            status = LMX_EINVAL;
            err_code = kErrSeparateN1;
        }

        // ---- the event loop of this trace ----
        // Control flow is kept structured (no continue/break out of the
        // decision) so divergent lanes reconverge right after each branch.
        while (status == LMX_OK && (i < nI || j < nT)) {
            if (++iters > 2 * (nI + nT) + 2) status = LMX_EBUDGET;
            // a1: event selection (ties -> inference)
            const double t_inf = (i < nI) ? a_inf : kInf;
            const bool is_train = !(t_inf <= r);
            const double now = is_train ? r : t_inf;
            const uint32_t v = is_train ? v_tr : v_inf;
            bool deferred = false;
            if (status == LMX_OK && is_train && p.policy == LMX_LEMIX && p.deprioritize && i < nI) {
                // a2: Eq. 4 against the next enqueued inference task
                const double wn = task_w(v_inf);
                double m = kInf;
#pragma unroll
                for (int n = 0; n < NMAX; ++n)
                    if (n < N) {
                        const double latest = ((hasp >> n) & 1u) ? dev::last_of(P[n], S) : -kInf;
                        m = dmin(m, latest + s_ef[n * S + S - 1] * wn);
                    }
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
                    r = t_inf;            // behind the next inference task
                    cur_defer++;
                    n_def++;
                }
            }
            const int task = is_train ? nI + j : i;
            if (status == LMX_OK && !deferred) {   // input validation of the task being placed
                const double arr = is_train ? a_tr : a_inf;
                int code = kErrNone;
                if (v >> 21) code = kErrBits;
                else if (task_len(v) < 1 || task_len(v) > 2048) code = kErrLen;
                else if (task_batch(v) < 1) code = kErrBatch;
                else if ((int)((v >> 20) & 1u) != (int)is_train) code = kErrKind;
                else if (!(arr >= 0.0 && arr < kInf)) code = kErrArrival;
                else if (!is_train && arr < a_last_inf) code = kErrOrder;
                if (p.policy == LMX_FIXED && code == kErrNone) {
                    const int fx = __ldg(p.fixed + o + task);
                    if (fx < 0 || fx >= N) code = kErrFixed;
                }
                if (code != kErrNone) {
                    status = LMX_EINVAL;
                    err_task = task;
                    err_code = code;
                }
            }
            if (status == LMX_OK && !deferred) {
                const double a = now;
                const double w = task_w(v);
                const int l = task_len(v);

                double en_b[SMAX];
                double st0_b = 0.0;
                int best = 0;
                if (p.policy == LMX_LEMIX) {
                    // a3-a7: plan and score every node (independent chains, unrolled)
                    double f[NMAX];
                    double en[NMAX][SMAX], st0[NMAX];
#pragma unroll
                    for (int n = 0; n < NMAX; ++n) {
                        if (n < N) {
                            int sk[SMAX];
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) sk[s] = SK_(n, s);
                            double II;
                            int gc;
                            const dev::Ring q{ring_be + (rb0 + n * K) * ring_words(S), p.kmask, S, 0u, 0u, qh[n] + qn[n]};
                            double efn[SMAX], ebn[SMAX];
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) { efn[s] = (s < S) ? s_ef[n * S + s] : 0.0; ebn[s] = (s < S) ? s_eb[n * S + s] : 0.0; }
                            double skeb[SMAX];   // (no cache here: read the last stale entry)
#pragma unroll
                            for (int s = 0; s < SMAX; ++s)
                                skeb[s] = (s < S && sk[s] > qh[n]) ? q.at(sk[s] - 1, s).y : 0.0;
                            dev::plan<SMAX, LMX_LANE_PF>(P[n], (hasp >> n) & 1u, S, efn, ebn, q, qh[n], qn[n],
                                            sk, skeb, w, a, now, en[n], st0[n], II, gc);
#pragma unroll
                            for (int s = 0; s < SMAX; ++s)
                                if (s < S) SK_(n, s) = sk[s];
                            qh[n] += gc;
                            qn[n] -= gc;
                            const double R = dev::last_of(en[n], S) - a;                         // line 20
                            const double a_last = ((hasp >> n) & 1u) ? APREV_(n) : a;            // R-9
                            const double IIS = p.s_pow2 ? II * p.inv_S : II / (double)S;
                            const double IP = -dmax(IIS - (a - a_last), p.tau);                 // Eq. 1
                            double LC;                                                           // Eq. 2
                            if (!((warm >> n) & 1u)) {
                                LC = p.lc0;
                            } else {
                                const double d = (double)l - MU_(n);
                                LC = CC_(n) * dev::exp_neg((d * d) * KK_(n));
                            }
                            f[n] = (IP + p.lambda2 * LC) / (p.lambda1 * R);                     // Eq. 3
                        }
                    }
                    // a8: highest f, ties -> lowest index
#pragma unroll
                    for (int n = 1; n < NMAX; ++n)
                        if (n < N && f[n] > f[best]) best = n;
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) {
                        en_b[s] = en[0][s];
#pragma unroll
                        for (int n = 1; n < NMAX; ++n)
                            if (n == best) en_b[s] = en[n][s];
                    }
                    st0_b = st0[0];
#pragma unroll
                    for (int n = 1; n < NMAX; ++n)
                        if (n == best) st0_b = st0[n];
                } else {
                    // a9: baseline selectors, then Alg. 1 on that node only
                    if (p.policy == LMX_RR) {
                        best = rr % N;
                        rr++;
                    } else if (p.policy == LMX_SEPARATE) {
                        if (!(nI > 0 && nT > 0)) best = is_train ? (sep_t++ % N) : (sep_i++ % N);
                        else {
                            int ninf = N - p.n_tr_sep;
                            if (p.sep_dynamic) {   // SeparateDynamic (R-sepdyn)
                                while (rate_hi < nI && __ldg(p.arrival + o + rate_hi) <= now) rate_hi++;
                                const double w_lo = now - p.dyn_window;
                                while (rate_lo < nI && __ldg(p.arrival + o + rate_lo) <= w_lo) rate_lo++;
                                const double rate = (double)(rate_hi - rate_lo) / p.dyn_window;
                                ninf = (rate < p.dyn_rate) ? (N / 4 > 1 ? N / 4 : 1) : ninf;
                            }
                            best = is_train ? ninf + (sep_t++ % (N - ninf)) : (sep_i++ % ninf);
                        }
                    } else {
                        best = __ldg(p.fixed + o + task);
                    }
                    double Pc[SMAX];
                    int qhc = qh[0], qnc = qn[0];
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) Pc[s] = P[0][s];
#pragma unroll
                    for (int n = 1; n < NMAX; ++n)
                        if (n == best) {
                            qhc = qh[n];
                            qnc = qn[n];
#pragma unroll
                            for (int s = 0; s < SMAX; ++s) Pc[s] = P[n][s];
                        }
                    int sk[SMAX];
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) sk[s] = SK_(best, s);
                    double II;
                    int gc;
                    const dev::Ring q{ring_be + (rb0 + best * K) * ring_words(S), p.kmask, S, 0u, 0u, qhc + qnc};
                    double efb[SMAX], ebb[SMAX];
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) { efb[s] = (s < S) ? s_ef[best * S + s] : 0.0; ebb[s] = (s < S) ? s_eb[best * S + s] : 0.0; }
                    double skeb[SMAX];
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) skeb[s] = (s < S && sk[s] > qhc) ? q.at(sk[s] - 1, s).y : 0.0;
                    dev::plan<SMAX, LMX_LANE_PF>(Pc, (hasp >> best) & 1u, S, efb, ebb, q, qhc, qnc, sk,
                                    skeb, w, a, now, en_b, st0_b, II, gc);
#pragma unroll
                    for (int s = 0; s < SMAX; ++s)
                        if (s < S) SK_(best, s) = sk[s];
#pragma unroll
                    for (int n = 0; n < NMAX; ++n)
                        if (n == best) { qh[n] += gc; qn[n] -= gc; }
                }

                // ---- a10: commit the task to node `best` ----
                const double *ef = s_ef + best * S;
                const double *eb = s_eb + best * S;
                int qhb = qh[0], qnb = qn[0];
#pragma unroll
                for (int n = 1; n < NMAX; ++n)
                    if (n == best) { qhb = qh[n]; qnb = qn[n]; }
                double2 *rbe = p.ring_be + (rb0 + best * K) * ring_words(S);
                const dev::Ring qb{rbe, p.kmask, S, 0u, 0u, qhb + qnb};
#pragma unroll
                for (int s = 0; s < SMAX; ++s)
                    if (s < S) BUSY_(best, s) = BUSY_(best, s) + ef[s] * w;
                double done = dev::last_of(en_b, S);
                int ver = 0;
                if (is_train && qnb >= p.qcap) {
                    status = LMX_EQCAP;
                } else if (is_train) {
                    // backward planning, stages S..1
                    double2 bw[SMAX];
                    double db[SMAX];
                    double x = done;
#pragma unroll
                    for (int s = SMAX - 1; s >= 0; --s) {
                        bw[s] = make_double2(0.0, 0.0);
                        db[s] = 0.0;
                        if (s < S) {
                            const double sb = dmax(x, LB_(best, s));
                            db[s] = eb[s] * w;                 // dB_s (also line 16's offset)
                            const double ebv = sb + db[s];
                            LB_(best, s) = ebv;
                            bw[s] = make_double2(sb, ebv);
                            x = ebv;
                        }
                    }
                    qb.push<SMAX>(qhb, bw, db);
                    qnb++;
#pragma unroll
                    for (int n = 0; n < NMAX; ++n)
                        if (n == best) qn[n] = qnb;
#pragma unroll
                    for (int s = 0; s < SMAX; ++s)
                        if (s < S) BUSY_(best, s) = BUSY_(best, s) + eb[s] * w;
                    NTR_(best) = NTR_(best) + 1;
                    done = x;
                } else {
                    // version-at-inference: backwards completed by start_f^1 form a
                    // prefix of Q_train (end_b^1 non-decreasing); start_f^1 of
                    // successive commits on a node is non-decreasing, so the
                    // boundary pointer only moves forward.
                    int k = VP_(best);
                    if (k < qhb) k = qhb;
                    while (k < qhb + qnb && qb.at(k, 0).y <= st0_b) k++;
                    VP_(best) = k;
                    ver = NTR_(best) - (qhb + qnb - k);
                    if (p.sync_sep) {   // Separate: newest checkpoint loaded by start_f^1
                        int lo_k = 0, hi_k = n_ck;
                        while (lo_k < hi_k) {
                            const int mid = (lo_k + hi_k) >> 1;
                            if (ckt[mid] <= st0_b) lo_k = mid + 1; else hi_k = mid;
                        }
                        ver = lo_k * p.sync_interval;
                    }
                }
                if (status == LMX_OK) {
                    {   // P, a_[-1], Eq. 2 history of the chosen node
                        const int c = CNT_(best) + 1;
                        const long long s1 = SL_(best) + l, s2 = SL2_(best) + (long long)l * l;
                        CNT_(best) = c;
                        SL_(best) = s1;
                        SL2_(best) = s2;
                        APREV_(best) = a;
                        if (c >= 2) {   // cached Eq. 2 statistics (DESIGN.md R-stat)
                            const double inv_c = 1.0 / (double)c;
                            MU_(best) = (double)s1 * inv_c;
                            const long long var = (long long)c * s2 - s1 * s1;
                            const double sigma = dmax(sqrt((double)var) * inv_c, p.sigma_floor);
                            const double inv_s = 1.0 / sigma;
                            KK_(best) = (0.5 * inv_s) * inv_s;
                            CC_(best) = inv_s * dev::kInvSqrt2Pi;
                            warm |= 1u << best;
                        }
#pragma unroll
                        for (int n = 0; n < NMAX; ++n)
                            if (n == best) {
#pragma unroll
                                for (int s = 0; s < SMAX; ++s) P[n][s] = en_b[s];
                            }
                        hasp |= 1u << best;
                    }

                    // ---- a11: outputs + per-trace folds ----
                    if (p.node_defer) {
                        const unsigned dsat = is_train ? (unsigned)min(cur_defer, 0xFFFF) : 0u;
                        p.node_defer[o + task] = (uint32_t)best | (dsat << 16);
                        p.decision_idx[o + task] = step;
                        p.completion[o + task] = done;
                        p.start_f1[o + task] = st0_b;
                    }
                    t_last = dmax(t_last, done);
                    step++;
                    if (is_train) {
                        j++;
                        cur_defer = 0;
                        a_tr = a_tr2;
                        v_tr = v_tr2;
                        if (j + 1 < nT) {
                            a_tr2 = __ldg(p.arrival + o + nI + j + 1);
                            v_tr2 = __ldg(p.lbk + o + nI + j + 1);
                        }
                        if (p.sync_sep && j % p.sync_interval == 0) {   // checkpoint (R-sync)
                            const double av = done + p.sync_latency;
                            ckt[n_ck] = av;
                            for (int k = n_ck - 1; k >= 0 && ckt[k] > av; --k) ckt[k] = av;
                            n_ck++;
                        }
                        r = (j < nT) ? dmax(a_tr, en_b[0]) : kInf;      // release
                    } else {
                        const double ttft = dev::last_of(en_b, S) - a;
                        sum_ttft = sum_ttft + ttft;
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
                        if (ttft <= tauR) n_slo++;
                        sum_ver += ver;
                        a_last_inf = a;
                        i++;
                        a_inf = a_inf2;
                        v_inf = v_inf2;
                        if (i + 1 < nI) {
                            a_inf2 = __ldg(p.arrival + o + i + 1);
                            v_inf2 = __ldg(p.lbk + o + i + 1);
                        }
                    }
                }
            }
        }

        // ---- per-trace metrics, node folds in node order ----
        lmx_summary sm;
        sm.n_tasks = nI + nT;
        sm.n_inf = nI;
        sm.n_train = nT;
        sm.status = status;
        sm.n_slo_met = sm.n_deferrals = sm.active_nodes = sm.sum_version = 0;
        sm.n_mem_wait = sm.n_offload = 0;   // (Algorithm 2 runs on the tile kernel only)
        sm.makespan = sm.throughput = sm.sum_ttft = sm.mean_ttft = sm.slo_attainment = 0.0;
        sm.mean_util = sm.mean_len_std = 0.0;
        if (status == LMX_OK) {
            const int ntask = nI + nT;
            sm.n_slo_met = n_slo;
            sm.n_deferrals = n_def;
            sm.sum_version = sum_ver;
            sm.sum_ttft = sum_ttft;
            sm.makespan = (ntask > 0) ? t_last - t_first : 0.0;
            sm.throughput = (sm.makespan > 0.0) ? (double)ntask / sm.makespan : 0.0;
            sm.mean_ttft = (nI > 0) ? sum_ttft / (double)nI : 0.0;
            sm.slo_attainment = (nI > 0) ? (double)n_slo / (double)nI : 1.0;
            double U = 0.0, stds = 0.0;
            long long act = 0;
            for (int n = 0; n < N; ++n) {
                for (int s = 0; s < S; ++s) U = U + BUSY_(n, s);
                const long long c = CNT_(n);
                if (c > 0) {
                    act++;
                    const long long v2 = c * SL2_(n) - SL_(n) * SL_(n);
                    stds = stds + sqrt((double)v2) / (double)c;
                }
            }
            sm.active_nodes = act;
            sm.mean_util = (sm.makespan > 0.0) ? U / ((double)(N * S) * sm.makespan) : 0.0;
            sm.mean_len_std = (act > 0) ? stds / (double)act : 0.0;
        }
        p.summaries[t] = sm;
        if (status != LMX_OK) {
            p.trace_err[t] = ((long long)err_task << 8) | err_code;
            atomicMin(p.first_bad, (unsigned long long)t);
        }
    }
#undef LB_
#undef BUSY_
#undef SK_
#undef APREV_
#undef MU_
#undef KK_
#undef CC_
#undef SL_
#undef SL2_
#undef VP_
#undef CNT_
#undef NTR_
}

typedef void (*kernel_fn)(const KParams);

int nodes_bucket(int N) { return N <= 2 ? 2 : N <= 4 ? 4 : 8; }
int stages_bucket(int S) { return S <= 1 ? 1 : S <= 2 ? 2 : 4; }

template <int NMAX, int SMAX>
kernel_fn pick_exact(int S)
{
    return S == SMAX ? lane_loop_kernel<NMAX, SMAX, true> : lane_loop_kernel<NMAX, SMAX, false>;
}

kernel_fn pick(int N, int S)
{
    if (N < 1 || N > 8 || S < 1 || S > 4) return nullptr;
    switch (nodes_bucket(N) * 10 + stages_bucket(S)) {
    case 21: return pick_exact<2, 1>(S);
    case 22: return pick_exact<2, 2>(S);
    case 24: return pick_exact<2, 4>(S);
    case 41: return pick_exact<4, 1>(S);
    case 42: return pick_exact<4, 2>(S);
    case 44: return pick_exact<4, 4>(S);
    case 81: return pick_exact<8, 1>(S);
    case 82: return pick_exact<8, 2>(S);
    default: return nullptr;
    }
}

int per_thread_bytes(int N, int S)
{
    switch (nodes_bucket(N) * 10 + stages_bucket(S)) {
    case 21: return LaneSmem<2, 1>::kBytesPerThread;
    case 22: return LaneSmem<2, 2>::kBytesPerThread;
    case 24: return LaneSmem<2, 4>::kBytesPerThread;
    case 41: return LaneSmem<4, 1>::kBytesPerThread;
    case 42: return LaneSmem<4, 2>::kBytesPerThread;
    case 44: return LaneSmem<4, 4>::kBytesPerThread;
    case 81: return LaneSmem<8, 1>::kBytesPerThread;
    default: return LaneSmem<8, 2>::kBytesPerThread;
    }
}

int smem_bytes(int N, int S) { return 16 * N * S + kLaneBlock * per_thread_bytes(N, S); }

}  // namespace

bool lane_supported(int N, int S) { return pick(N, S) != nullptr; }

int lane_smem_bytes(const KParams &p) { return smem_bytes(p.N, p.S); }

int lane_block_threads() { return kLaneBlock; }

int lane_nodes_bucket(int N) { return nodes_bucket(N); }

int lane_occupancy(const KParams &p, int *err)
{
    kernel_fn f = pick(p.N, p.S);
    const int smem = smem_bytes(p.N, p.S);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int blocks = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f, kLaneBlock, smem);
    *err = (int)e;
    return blocks;
}

int launch_lane_loop(const KParams &p, int grid, void *stream)
{
    kernel_fn f = pick(p.N, p.S);
    f<<<grid, kLaneBlock, smem_bytes(p.N, p.S), (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace lmx
