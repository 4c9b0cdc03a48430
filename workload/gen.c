/*
 * gen.c -- seeded synthetic workload traces (DESIGN.md §"Input recipe").
 *
 * Shared input generator for BOTH the oracle and the CUDA path.  It contains
 * none of the scheduling method's arithmetic: it only draws arrival times and
 * lengths.  Each trace t draws from its own xoshiro256** stream seeded by
 * SplitMix64(seed_base + t), so the output is independent of the thread count.
 *
 * Shapes follow the paper's workloads:
 *   - Poisson arrivals, exponential inter-arrival gaps      PAPER.md:780 (§6.1)
 *   - bursty arrivals: Gamma renewal process, CV = 3         (LMSYS-shaped)
 *   - heavy-tailed LogNormal lengths clamped to [16, 2048]
 *   - continuous retraining: training a_min = 0
 * Task packing: l bits 0-11, C bits 12-19, kind bit 20 (1 = training).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n_inf, n_train;          /* tasks per trace */
    int32_t arrival_kind;            /* 0 Poisson, 1 Gamma renewal (bursty) */
    int32_t train_kind;              /* 0 Poisson a_min at rate_train, 1 continuous (a_min = 0) */
    double rate_inf;                 /* inference arrivals / s */
    double rate_train;               /* training arrivals / s (train_kind 0) */
    double cv;                       /* Gamma renewal coefficient of variation */
    double len_inf_median, len_inf_sigma;
    double len_train_median, len_train_sigma;
    int32_t len_min, len_max;
    int32_t batch_inf, batch_train;
    double out_median, out_sigma;
} wl_spec;

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t splitmix64(uint64_t *x)
{
    uint64_t z = (*x += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t next_u64(rng_t *r)
{
    uint64_t *s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}

static void rng_seed(rng_t *r, uint64_t seed)
{
    uint64_t x = seed;
    for (int k = 0; k < 4; ++k) r->s[k] = splitmix64(&x);
}

/* U in [0, 1) with 53 random bits */
static double uniform(rng_t *r) { return (double)(next_u64(r) >> 11) * 0x1p-53; }

static double exponential(rng_t *r, double rate) { return -log1p(-uniform(r)) / rate; }

static double normal(rng_t *r)
{
    double u1 = 1.0 - uniform(r);            /* (0, 1] */
    double u2 = uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* Gamma(shape k, scale 1): Marsaglia-Tsang; k < 1 via the U^(1/k) boost. */
static double gamma1(rng_t *r, double k)
{
    double boost = 1.0;
    if (k < 1.0) {
        boost = pow(1.0 - uniform(r), 1.0 / k);
        k += 1.0;
    }
    double d = k - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    for (;;) {
        double x, v;
        do { x = normal(r); v = 1.0 + c * x; } while (v <= 0.0);
        v = v * v * v;
        double u = uniform(r);
        if (u < 1.0 - 0.0331 * x * x * x * x) return boost * d * v;
        if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return boost * d * v;
    }
}

static int lognormal_len(rng_t *r, double median, double sigma, int lo, int hi)
{
    double x = median * exp(sigma * normal(r));
    double l = floor(x + 0.5);
    if (l < lo) l = lo;
    if (l > hi) l = hi;
    return (int)l;
}

static uint32_t pack(int l, int C, int kind)
{
    return (uint32_t)l | ((uint32_t)C << 12) | ((uint32_t)kind << 20);
}

static void gen_trace(const wl_spec *sp, uint64_t seed, double *arr, uint32_t *lbk, uint32_t *out_len)
{
    rng_t r;
    rng_seed(&r, seed);
    double t = 0.0;
    double shape = 1.0 / (sp->cv * sp->cv);
    for (int64_t k = 0; k < sp->n_inf; ++k) {
        double gap = (sp->arrival_kind == 1) ? gamma1(&r, shape) / (shape * sp->rate_inf)
                                             : exponential(&r, sp->rate_inf);
        t += gap;
        arr[k] = t;
        lbk[k] = pack(lognormal_len(&r, sp->len_inf_median, sp->len_inf_sigma, sp->len_min, sp->len_max),
                      sp->batch_inf, 0);
        /* always drawn, so the stream does not depend on whether it is kept */
        uint32_t ol = (uint32_t)lognormal_len(&r, sp->out_median, sp->out_sigma, 1, 2048);
        if (out_len) out_len[k] = ol;
    }
    t = 0.0;
    for (int64_t k = 0; k < sp->n_train; ++k) {
        int64_t o = sp->n_inf + k;
        if (sp->train_kind == 1) {
            arr[o] = 0.0;
        } else {
            t += exponential(&r, sp->rate_train);
            arr[o] = t;
        }
        lbk[o] = pack(lognormal_len(&r, sp->len_train_median, sp->len_train_sigma, sp->len_min, sp->len_max),
                      sp->batch_train, 1);
        if (out_len) out_len[o] = 0;
    }
}

typedef struct {
    const wl_spec *sp;
    uint64_t seed_base;
    const uint64_t *seeds;   /* non-NULL: trace t uses seeds[t] */
    int64_t t0, t1;
    double *arr;
    uint32_t *lbk, *out_len;
} job_t;

static void *worker(void *p)
{
    job_t *j = (job_t *)p;
    int64_t per = j->sp->n_inf + j->sp->n_train;
    for (int64_t t = j->t0; t < j->t1; ++t)
        gen_trace(j->sp, j->seeds ? j->seeds[t] : j->seed_base + (uint64_t)t, j->arr + t * per, j->lbk + t * per,
                  j->out_len ? j->out_len + t * per : NULL);
    return NULL;
}

static int generate(const wl_spec *sp, int64_t n_traces, uint64_t seed_base, const uint64_t *seeds,
                    double *arrival, uint32_t *lbk, uint32_t *out_len, int n_threads)
{
    if (!sp || n_traces < 0 || sp->n_inf < 0 || sp->n_train < 0) return 1;
    if (sp->n_inf > 0 && !(sp->rate_inf > 0.0)) return 1;
    if (sp->n_train > 0 && sp->train_kind == 0 && !(sp->rate_train > 0.0)) return 1;
    if (sp->arrival_kind == 1 && !(sp->cv > 0.0)) return 1;
    if (sp->len_min < 1 || sp->len_max > 2048 || sp->len_min > sp->len_max) return 1;
    if (sp->batch_inf < 1 || sp->batch_inf > 255 || sp->batch_train < 1 || sp->batch_train > 255) return 1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads > n_traces) n_threads = (int)(n_traces > 0 ? n_traces : 1);
    pthread_t th[256];
    job_t jobs[256];
    for (int k = 0; k < n_threads; ++k) {
        jobs[k].sp = sp; jobs[k].seed_base = seed_base; jobs[k].seeds = seeds;
        jobs[k].t0 = n_traces * k / n_threads; jobs[k].t1 = n_traces * (k + 1) / n_threads;
        jobs[k].arr = arrival; jobs[k].lbk = lbk; jobs[k].out_len = out_len;
    }
    if (n_threads == 1) { worker(&jobs[0]); return 0; }
    for (int k = 0; k < n_threads; ++k) pthread_create(&th[k], NULL, worker, &jobs[k]);
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
    return 0;
}

/* Fill n_traces fixed-size traces (n_inf + n_train tasks each, contiguous).
 * Trace t uses seed seed_base + t.  Returns 0 on success. */
int wl_generate(const wl_spec *sp, int64_t n_traces, uint64_t seed_base,
                double *arrival, uint32_t *lbk, uint32_t *out_len, int n_threads)
{
    return generate(sp, n_traces, seed_base, NULL, arrival, lbk, out_len, n_threads);
}

/* The same for an explicit seed list: trace t uses seeds[t] (a rank's shard
 * of a fixed seed set).  Returns 0 on success. */
int wl_generate_seeds(const wl_spec *sp, int64_t n_traces, const uint64_t *seeds,
                      double *arrival, uint32_t *lbk, uint32_t *out_len, int n_threads)
{
    if (!seeds && n_traces > 0) return 1;
    return generate(sp, n_traces, 0, seeds, arrival, lbk, out_len, n_threads);
}
