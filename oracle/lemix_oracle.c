/*
 * lemix_oracle.c -- TEST INFRASTRUCTURE ONLY (see lemix_oracle.h).
 *
 * A plain, slow, obviously-correct, single-threaded CPU implementation of the
 * LeMix placement step, written from the paper (arXiv 2507.21276, file
 * /root/reference/PAPER.md) in the paper's order and notation:
 *
 *   - latency model            Δ_F = η_F^n·C·ℓ², Δ_B = η_B^n·C·ℓ²     PAPER.md:383 (§4.1)
 *   - ComputeIdleness          Algorithm 1, lines 1-21                PAPER.md:432-476 (§4.2)
 *   - backward planning                                                PAPER.md:490-491 (§4.2)
 *   - idleness profit IP       Eq. 1 (eq:idle_profit)                 PAPER.md:544-549 (§4.3)
 *   - length consistency LC    Eq. 2 (eq:length_heterogeneity)        PAPER.md:552-557 (§4.3)
 *   - node priority f          Eq. 3 (eq:node_fitness), highest wins  PAPER.md:562-568 (§4.3)
 *   - queue-level deprioritise Eq. 4                                   PAPER.md:586-597 (§4.3)
 *   - global queue order       inference by arrival, training by the
 *                              previous training task's S1 forward end PAPER.md:224 (§3)
 *   - baselines Separate / NaiveMix(RR)                                PAPER.md:795-796 (§6.1)
 *   - metrics (throughput, SLO = TTFT <= 5x forward latency)          PAPER.md:786-790 (§6.1)
 *   - ExecuteTaskMemoryAware   Algorithm 2, lines 1-20 (optional)      PAPER.md:608-641 (§4.4)
 *   - ContinuousBatching       Algorithm 3, lines 1-17 (optional), with
 *                              hybrid prefill/decode and TBT           PAPER.md:689-727, 789 (§5.4, §6.1)
 *   - Mix-LUF baseline         lowest average utilisation first        PAPER.md:797, 1101 (§6.1, Table 2)
 *
 * Where the paper is silent or garbled the DESIGN.md reading is cited as
 * [R-n] (DESIGN.md §"Readings").  Floating point: IEEE binary64, built with
 * -O2 -ffp-contract=off (no FMA contraction, no reassociation).  The
 * expression forms follow DESIGN.md §"Canonical fp64 expression sheet".
 *
 * Data structures are deliberately literal: per-node trace queues hold task
 * indices (Q^n, Q_train^n), Q_temp is a fresh copy per call, removal is a
 * list deletion, every task keeps its full planned path.  Nothing here is
 * blocked, fused or reordered.
 */
#include "lemix_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXS 16

/* MAX/MIN as ternaries ([R-maxmin]: fmax/fmin leave the sign of zero unspecified). */
static double MAX(double x, double y) { return (y > x) ? y : x; }
static double MIN(double x, double y) { return (y < x) ? y : x; }

/* ---------------------------------------------------------------------------
 * exp(-t), t >= 0: the fully specified routine of DESIGN.md [R-exp] (the
 * paper only says "exp", Eq. 2; both sides must round identically):
 *   k = rint(-t * log2(e)); r = (-t - k*LN2_HI) - k*LN2_LO
 *   p = the degree-13 Taylor polynomial of e^r evaluated by Estrin's scheme
 *       (pairs c_2i + c_2i+1*r, then powers r^2, r^4, r^8), each a*b+c as a
 *       multiply then an add, no FMA
 *   result = p * 2^k (exact; normal for t <= 700), 0 beyond t = 700.
 * Pinned against libm in tests/test_oracle_units.py (<= 2 ulp), exact at 0.
 * ------------------------------------------------------------------------- */
double orc_exp_neg(double t)
{
    static const double C[14] = {
        0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
        0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
        0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
        0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};   /* 1/i! */
    if (t > 700.0) return 0.0;
#ifdef ORC_TEXTBOOK
    /* SURVEY.md 8c.4 text form (Horner, degree 13), kept only to test that
     * the Estrin form above [R-exp] changes no scheduling result */
    {
        double x = -t;
        double k = rint(x * 0x1.71547652b82fep0);
        double r = (x - k * 0x1.62e42fee00000p-1) - k * 0x1.a39ef35793c76p-33;
        double p = C[13];
        for (int i = 12; i >= 0; --i) p = p * r + C[i];
        return ldexp(p, (int)k);
    }
#endif
    double x = -t;
    double k = rint(x * 0x1.71547652b82fep0);       /* round half to even */
    double hi = x - k * 0x1.62e42fee00000p-1;      /* ln2 high part */
    double lo = k * 0x1.a39ef35793c76p-33;         /* ln2 low part */
    double r = hi - lo;
    double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    double q[7];
    for (int i = 0; i < 7; ++i) q[i] = C[2 * i] + C[2 * i + 1] * r;   /* c_2i + c_2i+1 r */
    double s0 = q[0] + q[1] * r2, s1 = q[2] + q[3] * r2, s2 = q[4] + q[5] * r2, s3 = q[6];
    double u0 = s0 + s1 * r4, u1 = s2 + s3 * r4;
    double p = u0 + u1 * r8;
    return ldexp(p, (int)k);
}

/* ---------------------------------------------------------------------------
 * Per-trace state
 * ------------------------------------------------------------------------- */
typedef struct {
    double sf[MAXS], ef[MAXS];   /* forward path  start_f^s, end_f^s */
    double oe[MAXS];             /* occupancy end of GPU (n, s): end_f^s + the decode steps that
                                    follow the prefill there ([R-cb]); = end_f^s without batching */
    double sb[MAXS], eb[MAXS];   /* backward path start_b^s, end_b^s (training only) */
    int off[MAXS];               /* Algorithm 2: activations offloaded from GPU s (line 10) */
} path_t;

typedef struct {
    int64_t last_task;      /* Q^n[-1], -1 if the node never ran a task */
    double a_last;          /* a_[-1]: dispatch time of that task (Eq. 1, [R-9]) */
    int has_efS;            /* Q^n non-empty */
    double max_efS;         /* max over task in Q^n of end_f^S (Eq. 4 inner max, [R-14]) */
    int64_t *q_train;       /* Q_train^n: task indices, enqueue order */
    int64_t q_len;
    int64_t hist_cnt, hist_sum, hist_sumsq;   /* lengths of tasks previously run here ([R-10]) */
    double busy[MAXS];
    int64_t n_train_on;     /* training tasks committed here (co-located model version) */
} node_t;

typedef struct {
    const orc_profile *prof;
    const orc_params *par;
    int N, S;
    const double *arrival;
    const uint32_t *lbk;
    const uint32_t *out_len;
    path_t *path;           /* per task */
    node_t *node;
    orc_counters *cnt;
} trace_t;

static int task_len(uint32_t v) { return (int)(v & 0xFFFu); }
static int task_batch(uint32_t v) { return (int)((v >> 12) & 0xFFu); }
static int task_kind(uint32_t v) { return (int)((v >> 20) & 1u); }

/* C·ℓ² as an exact double (< 2^53). */
static double task_w(uint32_t v)
{
    int64_t l = task_len(v), C = task_batch(v);
    return (double)(C * l * l);
}

static double eta_f(const trace_t *T, int n, int s) { return T->prof->eta_f[n * T->S + s]; }
static double eta_b(const trace_t *T, int n, int s) { return T->prof->eta_b[n * T->S + s]; }
static double eta_d(const trace_t *T, int n, int s) { return T->prof->eta_d ? T->prof->eta_d[n * T->S + s] : 0.0; }

/* ---------------------------------------------------------------------------
 * Algorithm 1  ComputeIdleness.  Line numbers below are
 * the algorithm's own.  Returns II and R; writes the planned forward path of
 * the new task into sf/ef (and its occupancy ends into oe).  Entries of
 * Q_train^n for which CheckExecuted holds (lines 17-18) are removed from the
 * node's queue on return.
 *
 * w = C*l^2 of the task.  tail[s] (NULL = none) is the decode work a
 * continuous batch runs on GPU s right after its prefill ([R-cb]): the GPU is
 * busy until end + tail[s], so that occupancy end is what must fit before a
 * pending backward (line 10) and what the next task on the node starts after
 * (line 3's task_prev); the next stage still starts at the prefill end (the
 * first token flows on).  With no tail every occ equals end bit for bit.
 * ------------------------------------------------------------------------- */
static void compute_idleness(trace_t *T, int n, double w, const double *tail, double a, double now,
                             double *II_out, double *R_out, double *sf, double *ef, double *oe)
{
    const int S = T->S;
    node_t *nd = &T->node[n];
    T->cnt->alg1_calls++;

    /* line 3: task_prev <- Q^n[-1].  A node that never ran a task has a
     * virtual predecessor that ends each stage exactly when the new task could
     * start it ([R-1]); its a_[-1] is a itself ([R-9]). */
    double prev_ef[MAXS];
    if (nd->last_task >= 0) {
        for (int s = 0; s < S; ++s) prev_ef[s] = T->path[nd->last_task].oe[s];
    } else {
        double v = a;
        for (int s = 0; s < S; ++s) { prev_ef[s] = v; v = v + eta_f(T, n, s) * w; }
    }

    /* line 3: Q_temp <- Q_train^n (a copy; dequeue = advance the front). */
    int64_t qlen = nd->q_len;
    int64_t *qtemp = (int64_t *)malloc((size_t)(qlen > 0 ? qlen : 1) * sizeof(int64_t));
    memcpy(qtemp, nd->q_train, (size_t)qlen * sizeof(int64_t));
    int64_t front = 0;
    int *remove = (int *)calloc((size_t)(qlen > 0 ? qlen : 1), sizeof(int));

    double II = 0.0;                                   /* line 3 */
    double end_prev_stage = a;                         /* end_f^0 := a ([R-2]) */
    for (int s = 0; s < S; ++s) {                      /* line 4 */
        T->cnt->stage_iters++;
        const double dF = eta_f(T, n, s) * w;
        const double dD = tail ? tail[s] : 0.0;
        double start = MAX(end_prev_stage, prev_ef[s]);  /* line 5 */
        double end = start + dF;                          /* line 6 */
        double occ = end + dD;
        double offset = 0.0;                              /* line 7 */
        while (front < qlen) {                            /* line 8 */
            int64_t k = front;
            int64_t tt = qtemp[front++];                  /* line 9: dequeue */
            const path_t *pt = &T->path[tt];
            if (occ <= pt->sb[s]) {                       /* line 10 */
                front--;                                  /* line 11: reinstated at the front ([R-3]) */
                T->cnt->scan_break++;
                break;                                    /* line 12 */
            }
            T->cnt->scan_consumed++;
            start = MAX(start, pt->eb[s]);                /* line 13 */
            end = start + dF;                             /* line 14 */
            occ = end + dD;
            if (prev_ef[s] <= pt->sb[s]) {                /* line 15 */
                offset = offset + eta_b(T, n, s) * task_w(T->lbk[tt]);   /* line 16 ([R-7]) */
                T->cnt->offset_adds++;
            }
            if (s == 0 && pt->eb[0] <= now) {             /* line 17: CheckExecuted ([R-5]) */
                /* line 18: remove from Q_train^n (index k of the original queue,
                 * which Q_temp copied in order). */
                remove[k] = 1;
            }
        }
        II = II + ((start - prev_ef[s]) - offset);        /* line 19 ([R-8], grouping [R-II]) */
        sf[s] = start;
        ef[s] = end;
        oe[s] = occ;
        end_prev_stage = end;
    }
    *II_out = II;
    *R_out = ef[S - 1] - a;                               /* line 20 */

    /* apply line-18 removals to Q_train^n */
    int64_t m = 0;
    for (int64_t k = 0; k < qlen; ++k)
        if (!remove[k]) nd->q_train[m++] = nd->q_train[k];
    nd->q_len = m;
    free(remove);
    free(qtemp);
}

/* Eq. 1: IP = -max{ II/S - (a - a_[-1]), tau }. */
static double idleness_profit(double II, int S, double a, double a_last, double tau)
{
    return -MAX(II / (double)S - (a - a_last), tau);
}

/* Eq. 2: LC = 1/(σ√(2π)) · exp{-(ℓ-μ)²/(2σ²)} with μ, σ the population mean
 * and standard deviation of lengths previously run on the node ([R-10]);
 * σ floored at sigma_floor, fewer than two samples -> lc0 ([R-11]).
 * Arithmetic per DESIGN.md [R-stat]: one reciprocal of the count and one of σ
 *   inv_c = 1/cnt; μ = Σℓ·inv_c; σ = max(√(cnt·Σℓ² − (Σℓ)²)·inv_c, floor);
 *   inv_σ = 1/σ; k = (0.5·inv_σ)·inv_σ = 1/(2σ²); c = inv_σ·(1/√(2π)).
 * parity unpinned for lc0 (a reading, not a formula). */
static double length_consistency(const trace_t *T, const node_t *nd, int l)
{
    const orc_params *P = T->par;
    if (nd->hist_cnt < 2) { T->cnt->lc_cold++; return P->lc0; }
    T->cnt->lc_exp++;
#ifdef ORC_TEXTBOOK
    /* SURVEY.md 8c.4 text form (true divisions), kept only to test that the
     * reciprocal form below [R-stat] changes no scheduling result */
    {
        double mu = (double)nd->hist_sum / (double)nd->hist_cnt;
        int64_t var = nd->hist_cnt * nd->hist_sumsq - nd->hist_sum * nd->hist_sum;
        double sigma = MAX(sqrt((double)var) / (double)nd->hist_cnt, P->sigma_floor);
        double k = 0.5 / (sigma * sigma);
        double c = 1.0 / (sigma * 0x1.40d931ff62705p+1);         /* sqrt(2 pi) */
        double d = (double)l - mu;
        return c * orc_exp_neg((d * d) * k);
    }
#endif
    double inv_c = 1.0 / (double)nd->hist_cnt;
    double mu = (double)nd->hist_sum * inv_c;
    int64_t var_num = nd->hist_cnt * nd->hist_sumsq - nd->hist_sum * nd->hist_sum; /* cnt²·Var, exact */
    double sigma = MAX(sqrt((double)var_num) * inv_c, P->sigma_floor);
    double inv_s = 1.0 / sigma;
    double k = (0.5 * inv_s) * inv_s;                       /* 1/(2σ²) */
    double c = inv_s * 0x1.9884533d43651p-2;                /* 1/(σ√(2π)) */
    double d = (double)l - mu;
    return c * orc_exp_neg((d * d) * k);
}

/* Eq. 3: f = (IP + λ2·LC) / (λ1·R). */
static double priority(const orc_params *P, double IP, double LC, double R)
{
    return (IP + P->lambda2 * LC) / (P->lambda1 * R);
}

/* tau_R for an inference task: slo_mult x its uncontended forward latency on
 * node 0 ([R-16]) or a constant. */
static double tau_R(const trace_t *T, uint32_t v)
{
    const orc_params *P = T->par;
    if (P->slo_mode == 1) return P->slo_const;
    double w = task_w(v);
    double acc = 0.0;
    for (int s = 0; s < T->S; ++s) acc = acc + eta_f(T, 0, s) * w;
    return P->slo_mult * acc;
}

/* Eq. 4: defer the training task iff
 *   min_n { max_{task in Q^n} end_f^S + η_F^n·C'ℓ'² } - a' > tau_R
 * for the next enqueued inference task (a', ℓ', C') ([R-14], [R-15]).
 * eq4_mode 1 ([R-14b]): the inner term also counts the training task's own
 * forward, as if it went to node n ahead of the inference task: its forward
 * chained stage by stage after the node's last forward ends (no backward
 * scan), x_n = that end + η_F^{n,S}·C'ℓ'². */
static int should_deprioritize(trace_t *T, uint32_t next_lbk, double a_next, double a_train, double w_train)
{
    const int N = T->N, S = T->S;
    T->cnt->eq4_checks++;
    double w = task_w(next_lbk);
    double m = INFINITY;
    for (int n = 0; n < N; ++n) {
        const node_t *nd = &T->node[n];
        double latest;
        if (T->par->eq4_mode == 1) {
            double v = a_train;
            for (int s = 0; s < S; ++s) {
                double pe = (nd->last_task >= 0) ? T->path[nd->last_task].oe[s] : -INFINITY;
                v = MAX(v, pe) + eta_f(T, n, s) * w_train;
            }
            latest = v;
        } else {
            latest = nd->has_efS ? nd->max_efS : -INFINITY;   /* max over empty Q^n */
        }
        double x = latest + eta_f(T, n, S - 1) * w;
        m = MIN(m, x);
    }
    return (m - a_next) > tau_R(T, next_lbk);
}

/* ---------------------------------------------------------------------------
 * Algorithm 3  ContinuousBatching, lines 2-15, on the
 * FCFS inference stream ([R-cb]).  The batch opens at the arrival of request
 * i (line 5: T_start).  The next request joins (line 10) while the batch has
 * fewer than C members (line 7), it is not preceded by a released training
 * task (line 9: a training task at the head of the queue -- released at
 * r_train before the request arrives; ties go to inference, [R-19]) and the
 * timer has not run out (line 9: T_start + T_w > the request's arrival).  The
 * batch executes (line 15) as soon as it is full -- at its C-th member's
 * arrival -- else when the timer expires or the training task is released,
 * whichever is first.  Returns the member count; *t_exec = that time.
 * ------------------------------------------------------------------------- */
static int64_t continuous_batch(const double *arrival, int64_t i, int64_t nI, int64_t C, double Tw,
                                int train_pending, double r_train, double *t_exec)
{
    const double T_start = arrival[i];                    /* line 5 */
    int64_t m = 1;                                        /* line 10: request i */
    while (i + m < nI && m < C) {                         /* line 7 */
        const double ar = arrival[i + m];                 /* line 8: get_next_request */
        if (train_pending && r_train < ar) break;         /* line 9: require_backward -> line 12 */
        if (!(T_start + Tw > ar)) break;                  /* line 9: timer -> line 12 */
        m++;                                              /* line 10 */
    }
    if (m == C) *t_exec = arrival[i + m - 1];             /* full */
    else *t_exec = MIN(T_start + Tw, train_pending ? r_train : INFINITY);
    return m;
}

/* Decode work ([R-cb]): after the prefill, the batch
 * decodes with hybrid iteration-level batching: step k = 1, 2,
 * ... advances every member that still needs a token (C_k = members with
 * out >= k; out = decode steps of a request, 0 = none) over a context padded
 * to the batch's prompt length, l_pad + k - 1 tokens, at
 * eta_D * C_k * (l_pad + k - 1) seconds on each GPU ("step latency = max over
 * members of eta_D * C_batch * l_ctx").  Returns the work of
 * steps 1 .. upto in exact integer token units, summed step by step; the
 * seconds are eta_D times it (one rounding, like Delta_F = eta_F * C l^2). */
static int64_t decode_work(const uint32_t *out, int64_t m, int64_t l_pad, int64_t upto)
{
    int64_t W = 0;
    for (int64_t k = 1; k <= upto; ++k) {
        int64_t Ck = 0;
        for (int64_t jj = 0; jj < m; ++jj)
            if ((int64_t)out[jj] >= k) Ck++;               /* members still decoding at step k */
        W += Ck * (l_pad + k - 1);
    }
    return W;
}

/* Backward planning: immediately after the forward path,
 * stages S..1 in reverse, each after the previous stage's backward and after
 * every backward already planned on that GPU. */
static void plan_backward(trace_t *T, int n, uint32_t v, path_t *p)
{
    const int S = T->S;
    node_t *nd = &T->node[n];
    double w = task_w(v);
    double x = p->ef[S - 1];
    for (int s = S - 1; s >= 0; --s) {
        /* latest planned backward end on GPU (n, s).  Entries already removed
         * from Q_train^n ended before `now`, which precedes x, so the queue
         * holds every backward that can matter. */
        double latest = -INFINITY;
        for (int64_t k = 0; k < nd->q_len; ++k) latest = MAX(latest, T->path[nd->q_train[k]].eb[s]);
        p->sb[s] = MAX(x, latest);
        p->eb[s] = p->sb[s] + eta_b(T, n, s) * w;
        x = p->eb[s];
    }
}

/* ---------------------------------------------------------------------------
 * Algorithm 2  ExecuteTaskMemoryAware, for the task just
 * placed on node n, under the memory model of DESIGN.md [R-mem]:
 *   - a forward of a task on stage s needs C*l tokens of activation memory
 *     on GPU (n, s); a training task holds them until its stage-s backward
 *     ends, an inference task releases them when its forward ends;
 *   - MemoryAvailable(n, s) at time t (line 7): the tokens held at t by the
 *     training tasks in Q_train^n (end_b^s > t, not offloaded from s) plus
 *     the task's own need fit in mem_cap (= M_threshold, in tokens);
 *   - lines 6-11: wait in steps of Delta_t; once the wait reaches T_max the
 *     task's activations on s are offloaded (it then needs 0 tokens there)
 *     and its forward on s takes mem_pen seconds per offloaded token longer;
 *   - lines 12-14: Forward at the planned start plus the wait; calibration:
 *     the executed interval replaces the planned one -- a forward that was
 *     planned into the gap before a pending backward and no longer fits is
 *     postponed past it exactly as Algorithm 1 lines 10-14 do;
 *   - lines 15-17: the backward is planned after the executed forward path
 *     (plan_backward), so the queues hold executed times.
 * Only forwards are gated (Algorithm 2 checks memory before Forward only).
 * With no waits the executed path equals Algorithm 1's plan.
 * Writes the executed forward path to sf/ef and the offload flags to off;
 * returns the number of stages that waited (the offloads are in off).
 * ------------------------------------------------------------------------- */
static int memory_available(const trace_t *T, int n, int s, double t, int64_t need)
{
    const node_t *nd = &T->node[n];
    int64_t held = 0;
    for (int64_t k = 0; k < nd->q_len; ++k) {
        const path_t *q = &T->path[nd->q_train[k]];
        if (q->eb[s] > t && !q->off[s]) {
            uint32_t v = T->lbk[nd->q_train[k]];
            held += (int64_t)task_batch(v) * task_len(v);
        }
    }
    return held + need <= T->par->mem_cap;
}

static int execute_memory_aware(trace_t *T, int n, uint32_t v, double a, double *sf, double *ef, int *off)
{
    const int S = T->S;
    const orc_params *P = T->par;
    node_t *nd = &T->node[n];
    const double w = task_w(v);
    const int64_t tok = (int64_t)task_batch(v) * task_len(v);
    double prev_ef[MAXS];
    if (nd->last_task >= 0) {
        for (int s = 0; s < S; ++s) prev_ef[s] = T->path[nd->last_task].oe[s];
    } else {
        double x = a;
        for (int s = 0; s < S; ++s) { prev_ef[s] = x; x = x + eta_f(T, n, s) * w; }
    }
    int64_t front = 0;                                   /* Q_temp cursor over Q_train^n */
    int waited = 0;
    double e = a;
    for (int s = 0; s < S; ++s) {
        const double dF = eta_f(T, n, s) * w;
        double start = MAX(e, prev_ef[s]);               /* Alg. 1 lines 5-6: planned start */
        double end = start + dF;
        while (front < nd->q_len) {                      /* Alg. 1 lines 8-14 */
            const path_t *q = &T->path[nd->q_train[front]];
            if (end <= q->sb[s]) break;
            start = MAX(start, q->eb[s]);
            end = start + dF;
            front++;
        }
        /* Alg. 2 lines 6-11: wait-or-drop before Forward(task, s) */
        double wait = 0.0;
        off[s] = 0;
        while (!memory_available(T, n, s, start + wait, tok)) {   /* line 7 */
            wait = wait + P->mem_dt;                               /* line 8 */
            if (wait >= P->mem_tmax) {                             /* line 9 */
                off[s] = 1;                                        /* line 10: offload */
                break;                                             /* line 11 */
            }
        }
        /* line 12: after an offload the task needs no memory on GPU s, and the
         * tokens held never exceed mem_cap (every admission was checked), so
         * the check holds and the forward runs (see DESIGN.md [R-mem]). */
        if (wait > 0.0) {
            waited++;
            const double dur = off[s] ? dF + P->mem_pen * (double)tok : dF;
            start = start + wait;                        /* lines 13-14: calibrate */
            end = start + dur;
            while (front < nd->q_len) {                  /* no overlap with pending backwards */
                const path_t *q = &T->path[nd->q_train[front]];
                if (end <= q->sb[s]) break;
                start = MAX(start, q->eb[s]);
                end = start + dur;
                front++;
            }
        }
        sf[s] = start;
        ef[s] = end;
        e = end;
    }
    return waited;
}

int orc_run_trace(const orc_profile *prof, const orc_params *par,
                  int64_t n_tasks, int64_t n_inf,
                  const double *arrival, const uint32_t *lbk, const uint32_t *out_len, const int32_t *fixed_node,
                  uint32_t *node_defer, int32_t *decision_idx, double *completion,
                  double *start_f1, double *paths, double *cand,
                  orc_summary *summary, orc_counters *counters)
{
    const int N = prof->n_nodes, S = prof->n_stages;
    orc_summary sm;
    memset(&sm, 0, sizeof sm);
    orc_counters dummy;
    memset(&dummy, 0, sizeof dummy);
    if (!counters) counters = &dummy;

    const int64_t nI = n_inf, nT = n_tasks - n_inf;
    sm.n_tasks = n_tasks; sm.n_inf = nI; sm.n_train = nT;
    const int cb = par->cb_cmax > 0;   /* continuous batching (Algorithm 3) */

    /* ---- input validation (inputs must be finite, ordered and in range) ---- */
    int bad = (N < 1 || S < 1 || S > MAXS || nI < 0 || nT < 0 || par->qcap < 1 || !(par->lambda1 > 0.0));
    bad = bad || par->policy < ORC_LEMIX || par->policy > ORC_MIXLUF;
    bad = bad || par->sync_interval < 0 || !(par->sync_latency >= 0.0 && par->sync_latency < INFINITY);
    bad = bad || par->cb_cmax < 0 || (par->eq4_mode != 0 && par->eq4_mode != 1);
    bad = bad || !(par->luf_delay >= 0.0 && par->luf_delay < INFINITY);
    if (cb)   /* T_w finite, decode costs and output lengths given; not combined with Algorithm 2 */
        bad = bad || !(par->cb_tw >= 0.0 && par->cb_tw < INFINITY) || par->mem_enable || (nI > 0 && !out_len);
    if (par->sep_dynamic)
        bad = bad || !(par->dyn_rate >= 0.0 && par->dyn_rate < INFINITY) ||
              !(par->dyn_window > 0.0 && par->dyn_window < INFINITY);
    if (par->mem_enable)   /* Delta_t > 0 and T_max finite bound the wait loop */
        bad = bad || par->mem_cap < 0 || !(par->mem_dt > 0.0) || !(par->mem_tmax > 0.0 && par->mem_tmax < INFINITY) ||
              !(par->mem_pen >= 0.0 && par->mem_pen < INFINITY) || par->mem_tmax / par->mem_dt > 1048576.0;
    for (int k = 0; k < N * S && !bad; ++k)
        bad = !(prof->eta_f[k] > 0.0 && prof->eta_f[k] < INFINITY && prof->eta_b[k] > 0.0 && prof->eta_b[k] < INFINITY) ||
              (cb && prof->eta_d && !(prof->eta_d[k] >= 0.0 && prof->eta_d[k] < INFINITY));
    for (int64_t t = 0; t < n_tasks && !bad; ++t) {
        uint32_t v = lbk[t];
        bad = (v >> 21) != 0 || task_len(v) < 1 || task_len(v) > 2048 || task_batch(v) < 1 ||
              task_kind(v) != (t >= nI) || !(arrival[t] >= 0.0 && arrival[t] < INFINITY) ||
              (t > 0 && t < nI && arrival[t] < arrival[t - 1]) ||
              (cb && t < nI && out_len[t] > 2048u) ||
              (par->policy == ORC_FIXED && (fixed_node[t] < 0 || fixed_node[t] >= N));
    }
    if (!bad && par->policy == ORC_SEPARATE && N == 1 && nI > 0 && nT > 0) bad = 1;
    if (bad) {
        sm.status = ORC_EINVAL;
        if (summary) *summary = sm;
        return ORC_EINVAL;
    }

    trace_t T;
    T.prof = prof; T.par = par; T.N = N; T.S = S;
    T.arrival = arrival; T.lbk = lbk; T.out_len = out_len; T.cnt = counters;
    T.path = (path_t *)calloc((size_t)(n_tasks > 0 ? n_tasks : 1), sizeof(path_t));
    T.node = (node_t *)calloc((size_t)N, sizeof(node_t));
    for (int n = 0; n < N; ++n) {
        T.node[n].last_task = -1;
        T.node[n].q_train = (int64_t *)malloc((size_t)par->qcap * sizeof(int64_t));
    }
    uint32_t *defer = (uint32_t *)calloc((size_t)(n_tasks > 0 ? n_tasks : 1), sizeof(uint32_t));
    /* Separate's checkpoints ([R-sync]): availability time on the inference
     * nodes of checkpoint k = 1, 2, ... (taken when the (k*interval)-th
     * training task in release order ends its backward) */
    const int sync_sep = (par->policy == ORC_SEPARATE && par->sync_interval > 0);
    double *ck_avail = (double *)malloc((size_t)(nT / (sync_sep ? par->sync_interval : 1) + 1) * sizeof(double));
    int64_t n_ck = 0;

    /* Separate's partition ([R-20]) */
    int n_tr_nodes = 0, n_inf_nodes = N;
    if (par->policy == ORC_SEPARATE && nI > 0 && nT > 0) {
        n_tr_nodes = (int)floor((double)N * par->alpha + 0.5);
        if (n_tr_nodes < 1) n_tr_nodes = 1;
        if (n_tr_nodes > N - 1) n_tr_nodes = N - 1;
        n_inf_nodes = N - n_tr_nodes;
    }

    /* ---- the global queue: inference by arrival, training released at the
     * previous training task's S1 forward end ([R-18]) ---- */
    int64_t i = 0, j = 0, step = 0, iters = 0, rr = 0, sep_i = 0, sep_t = 0;
    int64_t rate_lo = 0, rate_hi = 0;   /* SeparateDynamic: arrivals in (now - W, now] */
    double r = (nT > 0) ? arrival[nI] : INFINITY;
    double t_last = -INFINITY;
    double sched_free = -INFINITY;      /* Mix-LUF: when the scheduler finishes its previous query ([R-luf]) */
    int status = ORC_OK;
    double IIv[256], Rv[256], fv[256];
    double (*sfv)[MAXS] = (double (*)[MAXS])malloc((size_t)N * sizeof(double[MAXS]));
    double (*efv)[MAXS] = (double (*)[MAXS])malloc((size_t)N * sizeof(double[MAXS]));
    double (*oev)[MAXS] = (double (*)[MAXS])malloc((size_t)N * sizeof(double[MAXS]));
    double *IIa = N <= 256 ? IIv : (double *)malloc((size_t)N * sizeof(double));
    double *Ra = N <= 256 ? Rv : (double *)malloc((size_t)N * sizeof(double));
    double *fa = N <= 256 ? fv : (double *)malloc((size_t)N * sizeof(double));
    double (*tails)[MAXS] = (double (*)[MAXS])malloc((size_t)N * sizeof(double[MAXS]));

    while (i < nI || j < nT) {
        if (++iters > 2 * (nI + nT) + 2) { status = ORC_EBUDGET; break; }
        double t_inf = (i < nI) ? arrival[i] : INFINITY;
        int64_t task, m = 1;            /* the decision places tasks task .. task + m - 1 */
        double now;
        if (t_inf <= r) {               /* ties: inference first ([R-19]) */
            task = i; now = t_inf;
            if (cb)                     /* Algorithm 3: the batch this request opens */
                m = continuous_batch(arrival, i, nI, par->cb_cmax, par->cb_tw, j < nT, r, &now);
        } else {
            task = nI + j; now = r;
            /* queue-level deprioritisation (Eq. 4) against the next enqueued
             * inference task; the training task moves behind it ([R-15]). */
            if (par->policy == ORC_LEMIX && par->deprioritize && i < nI &&
                should_deprioritize(&T, lbk[i], arrival[i], now, task_w(lbk[task]))) {
                r = arrival[i];
                defer[task]++;
                counters->deferrals++;
                sm.n_deferrals++;
                continue;
            }
        }
        const uint32_t v = lbk[task];
        const int is_train = task_kind(v);
        double a = now;                 /* dispatch time ([R-2]) */
        if (par->policy == ORC_MIXLUF) {
            /* Mix-LUF's utilisation query takes luf_delay and the scheduler
             * serves one decision at a time ([R-luf]) */
            sched_free = MAX(now, sched_free) + par->luf_delay;
            a = sched_free;
        }

        /* ---- the unit being placed: one task, or a batch of m requests
         * ([R-cb]: C_b = sum of the members' C, padded to the longest) ---- */
        int64_t l_pad = task_len(v), C_b = task_batch(v), W_D = 0;
        for (int64_t k = 1; k < m; ++k) {
            if (task_len(lbk[task + k]) > l_pad) l_pad = task_len(lbk[task + k]);
            C_b += task_batch(lbk[task + k]);
        }
        const double w = (double)(C_b * l_pad * l_pad);
        if (cb && !is_train) {
            uint32_t mx = 0;
            for (int64_t k = 0; k < m; ++k) if (out_len[task + k] > mx) mx = out_len[task + k];
            W_D = decode_work(out_len + task, m, l_pad, (int64_t)mx);
        }
        for (int n = 0; n < N; ++n)
            for (int s = 0; s < S; ++s) tails[n][s] = eta_d(&T, n, s) * (double)W_D;
        path_t *p = &T.path[task];

        /* ---- task-level node allocation ---- */
        int best = 0;
        for (int n = 0; n < N && cand; ++n) {
            cand[(step * N + n) * 3 + 0] = NAN;
            cand[(step * N + n) * 3 + 1] = NAN;
            cand[(step * N + n) * 3 + 2] = NAN;
        }
        if (par->policy == ORC_LEMIX) {
            for (int n = 0; n < N; ++n) {
                compute_idleness(&T, n, w, W_D ? tails[n] : NULL, a, now, &IIa[n], &Ra[n], sfv[n], efv[n], oev[n]);
                const node_t *nd = &T.node[n];
                double a_last = (nd->last_task >= 0) ? nd->a_last : a;
                double IP = idleness_profit(IIa[n], S, a, a_last, par->tau);
                double LC = length_consistency(&T, nd, (int)l_pad);
                fa[n] = priority(par, IP, LC, Ra[n]);
                if (cand) {
                    cand[(step * N + n) * 3 + 0] = IIa[n];
                    cand[(step * N + n) * 3 + 1] = Ra[n];
                    cand[(step * N + n) * 3 + 2] = fa[n];
                }
            }
            /* Eq. 3 needs R > 0: a forward too short to move the
             * clock past a makes f undefined; the trace stops as invalid input */
            int r_bad = 0;
            for (int n = 0; n < N; ++n) r_bad |= !(Ra[n] > 0.0);
            if (r_bad) { status = ORC_EINVAL; break; }
            /* highest f wins; ties -> lowest node index ([R-13]) */
            best = 0;
            for (int n = 1; n < N; ++n)
                if (fa[n] > fa[best]) best = n;
        } else {
            if (par->policy == ORC_RR) {
                best = (int)(rr % N); rr++;
            } else if (par->policy == ORC_SEPARATE) {
                if (n_tr_nodes == 0) {                                    /* one kind only */
                    if (is_train) best = (int)(sep_t++ % N); else best = (int)(sep_i++ % N);
                } else {
                    int ninf = n_inf_nodes;
                    if (par->sep_dynamic) {
                        /* request rate over the last dyn_window seconds ([R-sepdyn]) */
                        while (rate_hi < nI && arrival[rate_hi] <= now) rate_hi++;
                        const double w_lo = now - par->dyn_window;
                        while (rate_lo < nI && arrival[rate_lo] <= w_lo) rate_lo++;
                        const double rate = (double)(rate_hi - rate_lo) / par->dyn_window;
                        ninf = (rate < par->dyn_rate) ? (N / 4 > 1 ? N / 4 : 1) : n_inf_nodes;  /* "1-3" : "2-2" */
                    }
                    if (is_train) best = ninf + (int)(sep_t++ % (N - ninf));
                    else best = (int)(sep_i++ % ninf);
                }
            } else if (par->policy == ORC_MIXLUF) {
                /* lowest average utilisation first ([R-luf]): the
                 * node whose GPUs have the least busy time committed so far
                 * (the common denominator S * elapsed time does not change the
                 * order); ties -> lowest index */
                best = 0;
                double ub = INFINITY;
                for (int n = 0; n < N; ++n) {
                    double u = 0.0;
                    for (int s = 0; s < S; ++s) u = u + T.node[n].busy[s];
                    if (u < ub) { ub = u; best = n; }
                }
            } else {
                best = fixed_node[task];
            }
            compute_idleness(&T, best, w, W_D ? tails[best] : NULL, a, now, &IIa[best], &Ra[best], sfv[best],
                             efv[best], oev[best]);
            if (cand) {
                cand[(step * N + best) * 3 + 0] = IIa[best];
                cand[(step * N + best) * 3 + 1] = Ra[best];
                cand[(step * N + best) * 3 + 2] = NAN;
            }
        }

        /* ---- commit: the task (or batch) joins Q^best ---- */
        node_t *nd = &T.node[best];
        if (par->mem_enable) {
            /* Algorithm 2: execute (wait-or-drop) and calibrate */
            sm.n_mem_wait += execute_memory_aware(&T, best, v, a, p->sf, p->ef, p->off);
            for (int s = 0; s < S; ++s) {
                p->oe[s] = p->ef[s];
                sm.n_offload += p->off[s];
                const double dF = eta_f(&T, best, s) * w;
                const double dur = p->off[s] ? dF + par->mem_pen * (double)((int64_t)task_batch(v) * task_len(v)) : dF;
                nd->busy[s] = nd->busy[s] + dur;
            }
        } else {
            for (int s = 0; s < S; ++s) {
                p->sf[s] = sfv[best][s]; p->ef[s] = efv[best][s]; p->oe[s] = oev[best][s]; p->off[s] = 0;
            }
            /* busy: the prefill (or forward), then the decode steps that follow it */
            for (int s = 0; s < S; ++s) nd->busy[s] = (nd->busy[s] + eta_f(&T, best, s) * w) + tails[best][s];
        }
        double done = 0.0;
        int64_t ver = 0;
        if (is_train) {
            if (nd->q_len >= par->qcap) { status = ORC_EQCAP; break; }
            plan_backward(&T, best, v, p);
            nd->q_train[nd->q_len++] = task;
            if (nd->q_len > counters->max_qlen) counters->max_qlen = nd->q_len;
            for (int s = 0; s < S; ++s) nd->busy[s] = nd->busy[s] + eta_b(&T, best, s) * w;
            nd->n_train_on++;
            counters->commits_train++;
            done = p->eb[0];
        } else {
            /* version-at-inference: training tasks on this node whose backward
             * (stage 1) ended by this task's forward start. */
            int64_t pending = 0;
            for (int64_t k = 0; k < nd->q_len; ++k) {
                counters->version_scan++;
                if (T.path[nd->q_train[k]].eb[0] > p->sf[0]) pending++;
            }
            if (sync_sep) {
                /* Separate: the newest checkpoint loaded on the inference node by
                 * this task's forward start ([R-sync]) */
                int64_t kmax = 0;
                for (int64_t k = 0; k < n_ck; ++k)
                    if (ck_avail[k] <= p->sf[0] && k + 1 > kmax) kmax = k + 1;
                ver = kmax * par->sync_interval;
            } else {
                ver = nd->n_train_on - pending;
            }
            if (cb) sm.n_batches++;
        }
        /* per member (one for a single task): completion, TTFT / SLO, TBT */
        for (int64_t k = 0; k < m; ++k) {
            const int64_t tk = task + k;
            if (k > 0) T.path[tk] = *p;                          /* the batch's path */
            double fin = done;
            if (!is_train) {
                fin = p->ef[S - 1];                              /* first token (prefill end) */
                double ttft = p->ef[S - 1] - arrival[tk];        /* TTFT = R from arrival */
                sm.sum_ttft = sm.sum_ttft + ttft;
                if (ttft <= tau_R(&T, lbk[tk])) sm.n_slo_met++;
                sm.sum_version += ver;
                if (cb) {
                    /* its last token: after decode steps 1 .. out on GPU (best, S) */
                    const int64_t o = (int64_t)out_len[tk];
                    const double dec = eta_d(&T, best, S - 1) * (double)decode_work(out_len + task, m, l_pad, o);
                    fin = p->ef[S - 1] + dec;
                    if (o >= 1) {                                /* TBT: mean gap between its tokens */
                        sm.sum_tbt = sm.sum_tbt + dec / (double)o;
                        sm.n_tbt++;
                    }
                }
            }
            t_last = MAX(t_last, fin);
            if (node_defer) node_defer[tk] = (uint32_t)best | ((defer[tk] > 0xFFFFu ? 0xFFFFu : defer[tk]) << 16);
            if (decision_idx) decision_idx[tk] = (int32_t)step;
            if (completion) completion[tk] = fin;
            if (start_f1) start_f1[tk] = p->sf[0];
            if (paths)
                for (int s = 0; s < S; ++s) {
                    paths[(tk * S + s) * 4 + 0] = p->sf[s];
                    paths[(tk * S + s) * 4 + 1] = p->ef[s];
                    paths[(tk * S + s) * 4 + 2] = is_train ? p->sb[s] : 0.0;
                    paths[(tk * S + s) * 4 + 3] = is_train ? p->eb[s] : 0.0;
                }
            /* Eq. 2 history: the lengths of every task run on the node ([R-10]) */
            nd->hist_cnt += 1;
            nd->hist_sum += task_len(lbk[tk]);
            nd->hist_sumsq += (int64_t)task_len(lbk[tk]) * task_len(lbk[tk]);
        }
        nd->last_task = task + m - 1;
        nd->a_last = a;
        if (!nd->has_efS || p->oe[S - 1] > nd->max_efS) nd->max_efS = p->oe[S - 1];
        nd->has_efS = 1;
        step++;
        counters->decisions++;
        if (is_train) {
            j++;
            if (sync_sep && j % par->sync_interval == 0)               /* checkpoint ([R-sync]) */
                ck_avail[n_ck++] = p->eb[0] + par->sync_latency;
            r = (j < nT) ? MAX(arrival[nI + j], p->ef[0]) : INFINITY;
        } else {
            i += m;
        }
    }

    if (status == ORC_OK) {
        /* ---- per-trace metrics ---- */
        double t_first = INFINITY;
        if (nI > 0) t_first = MIN(t_first, arrival[0]);
        if (nT > 0) t_first = MIN(t_first, arrival[nI]);
        sm.makespan = (n_tasks > 0) ? t_last - t_first : 0.0;
        sm.throughput = (sm.makespan > 0.0) ? (double)n_tasks / sm.makespan : 0.0;
        sm.mean_ttft = (nI > 0) ? sm.sum_ttft / (double)nI : 0.0;
        sm.slo_attainment = (nI > 0) ? (double)sm.n_slo_met / (double)nI : 1.0;
        sm.mean_tbt = (sm.n_tbt > 0) ? sm.sum_tbt / (double)sm.n_tbt : 0.0;
        double U = 0.0, stds = 0.0;
        for (int n = 0; n < N; ++n) {
            for (int s = 0; s < S; ++s) U = U + T.node[n].busy[s];
            if (T.node[n].hist_cnt > 0) {
                const node_t *q = &T.node[n];
                sm.active_nodes++;
                int64_t var_num = q->hist_cnt * q->hist_sumsq - q->hist_sum * q->hist_sum;
                stds = stds + sqrt((double)var_num) / (double)q->hist_cnt;
            }
        }
        sm.mean_util = (sm.makespan > 0.0) ? U / ((double)(N * S) * sm.makespan) : 0.0;
        sm.mean_len_std = (sm.active_nodes > 0) ? stds / (double)sm.active_nodes : 0.0;
    } else {
        orc_summary e;
        memset(&e, 0, sizeof e);
        e.n_tasks = n_tasks; e.n_inf = nI; e.n_train = nT;
        sm = e;
    }
    sm.status = status;
    if (summary) *summary = sm;

    if (IIa != IIv) { free(IIa); free(Ra); free(fa); }
    free(sfv); free(efv); free(oev); free(tails);
    for (int n = 0; n < N; ++n) free(T.node[n].q_train);
    free(T.node); free(T.path); free(defer); free(ck_avail);
    return status;
}

int orc_run_batch(const orc_profile *prof, const orc_params *par,
                  int64_t n_traces, const int64_t *offsets, const int32_t *n_inf,
                  const double *arrival, const uint32_t *lbk, const uint32_t *out_len, const int32_t *fixed_node,
                  uint32_t *node_defer, int32_t *decision_idx, double *completion,
                  double *start_f1, orc_summary *summaries, orc_counters *counters)
{
    int first_err = ORC_OK;
    for (int64_t t = 0; t < n_traces; ++t) {
        int64_t o = offsets[t], n = offsets[t + 1] - offsets[t];
        int st = orc_run_trace(prof, par, n, n_inf[t], arrival + o, lbk + o, out_len ? out_len + o : NULL,
                               fixed_node ? fixed_node + o : NULL,
                               node_defer ? node_defer + o : NULL,
                               decision_idx ? decision_idx + o : NULL,
                               completion ? completion + o : NULL,
                               start_f1 ? start_f1 + o : NULL, NULL, NULL,
                               summaries ? summaries + t : NULL, counters);
        if (st != ORC_OK && first_err == ORC_OK) first_err = st;
    }
    return first_err;
}
