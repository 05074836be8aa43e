/*
 * hb_oracle.c -- CPU restatement of the HyperBall hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_1308_2144_b200) never links, loads or
 * calls it, and has no CPU fallback.
 *
 * Every function restates the reference's algorithm (Python + numba, read from
 * /root/reference/pkg/src/hyperball) in plain C, in the same evaluation order,
 * so that its outputs are bit-identical to the reference:
 *
 *   orc_mix64 / orc_hash           hll.py:70-88      (_mix64, hash_items)
 *   orc_register_value             hll.py:147-158    (register_values, rho_max 138-141)
 *   orc_alpha / orc_constants      hll.py:33,40-48; engine.py:149-151
 *   orc_estimate_row               _kernels.py:15-34 (ascending-j fp64 sum; libm log)
 *   orc_seed                       engine.py:100-119,153-162 -> _kernels.py:43-51,37-40
 *   orc_union_range                _kernels.py:67-114 (destination-level skip rule)
 *   orc_iterate_mt                 engine.py:351-399 (arc-balanced worker ranges)
 *   orc_accumulate                 centrality.py:132-150 (numpy elementwise, each op rounded)
 *   orc_finalize                   centrality.py:153-171
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against the
 * fixtures in tests/golden/, which tests/golden/make_golden.py produced by
 * running the reference package itself.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -ffast-math: the fp64
 * sums and the accumulate must keep IEEE evaluation order and rounding).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MIX_C1 0xBF58476D1CE4E5B9ULL
#define MIX_C2 0x94D049BB133111EBULL

/* hll.py:70-76 */
uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX_C1;
    z = (z ^ (z >> 27)) * MIX_C2;
    return z ^ (z >> 31);
}

/* hll.py:79-88: key = mix(replica + mix(seed)); h = mix(item + key) (wrapping u64) */
uint64_t orc_hash(uint64_t item, uint64_t replica, uint64_t seed) {
    uint64_t key = orc_mix64(replica + orc_mix64(seed));
    return orc_mix64(item + key);
}

void orc_hash_items(int64_t n, const uint64_t *items, const uint64_t *replicas,
                    uint64_t seed, uint64_t *out) {
    for (int64_t i = 0; i < n; i++) out[i] = orc_hash(items[i], replicas[i], seed);
}

static int bit_length_u64(uint64_t x) {
    int bl = 0;
    while (x) { bl++; x >>= 1; }
    return bl;
}

/* hll.py:147-158: idx = h & (p-1); rho = min((64-b+1) - bit_length(h >> b), 2^w - 1) */
void orc_register_value(uint64_t h, int b, int width, int64_t *idx, uint8_t *rho) {
    uint64_t p = 1ULL << b;
    *idx = (int64_t)(h & (p - 1));
    int r = (64 - b + 1) - bit_length_u64(h >> b);
    int sat = (1 << width) - 1;
    if (r > sat) r = sat;
    *rho = (uint8_t)r;
}

/* hll.py:40-48 */
double orc_alpha(int64_t p) {
    if (p == 16) return 0.673;
    if (p == 32) return 0.697;
    if (p == 64) return 0.709;
    return 0.7213 / (1.0 + 1.079 / (double)p);
}

/* engine.py:149-151: alpha_p2 = alpha(p) * p * p (left to right), lc_cut = 2.5 * p */
void orc_constants(int b, double *alpha_p2, double *lc_cut, double *p_float) {
    int64_t p = 1LL << b;
    *alpha_p2 = (orc_alpha(p) * (double)p) * (double)p;
    *lc_cut = 2.5 * (double)p;
    *p_float = (double)p;
}

/* hll.py:33: POW2NEG[r] = 2.0 ** -r (exact powers of two), tabulated once */
static double POW2NEG_TAB[256];
static pthread_once_t pow2neg_once = PTHREAD_ONCE_INIT;
static void pow2neg_init(void) {
    for (int r = 0; r < 256; r++) POW2NEG_TAB[r] = ldexp(1.0, -r);
}
static inline double pow2neg(int r) { return POW2NEG_TAB[r]; }

/* _kernels.py:15-34: ascending-index fp64 sum of 2^-M[j]; raw harmonic-mean estimate;
 * linear counting p*ln(p/V) when raw <= 2.5p and V > 0. */
double orc_estimate_row(const uint8_t *row, int64_t p, double alpha_p2, double lc_cut,
                        double p_float) {
    pthread_once(&pow2neg_once, pow2neg_init);
    double s = 0.0;
    int64_t zeros = 0;
    for (int64_t j = 0; j < p; j++) {
        uint8_t r = row[j];
        s += pow2neg(r);
        if (r == 0) zeros++;
    }
    double e = alpha_p2 / s;
    if (e <= lc_cut && zeros > 0) e = p_float * log(p_float / (double)zeros);
    return e;
}

void orc_estimate_rows(const uint8_t *regs, int64_t lo, int64_t hi, int b, double *out) {
    double a2, lc, pf;
    orc_constants(b, &a2, &lc, &pf);
    int64_t p = 1LL << b;
    for (int64_t v = lo; v < hi; v++) out[v] = orc_estimate_row(regs + v * p, p, a2, lc, pf);
}

/* engine.py:100-119 (_replica_items), 153-162 (seed) -> _kernels.py:43-51 scatter_max,
 * 37-40 estimate_register_rows.  weights may be NULL (one item (v, replica=1) per node);
 * otherwise node v contributes items (v, 1..weights[v]). regs must be zeroed [n, p]. */
void orc_seed(int64_t n, int b, int width, uint64_t seed, const int64_t *weights,
              uint8_t *regs, double *est) {
    int64_t p = 1LL << b;
    for (int64_t v = 0; v < n; v++) {
        int64_t w = weights ? weights[v] : 1;
        for (int64_t r = 1; r <= w; r++) {
            uint64_t h = orc_hash((uint64_t)v, (uint64_t)r, seed);
            int64_t idx;
            uint8_t rho;
            orc_register_value(h, b, width, &idx, &rho);
            if (rho > regs[v * p + idx]) regs[v * p + idx] = rho;
        }
    }
    if (n) orc_estimate_rows(regs, 0, n, b, est);
}

/* _kernels.py:67-114, line for line: a node is recomputed only if it or one of its
 * successors changed in the previous step (82-87); stable nodes copy their row and
 * reuse the cached estimate (88-93); otherwise byte-wise max over successor rows
 * (94-101), change test (102-106), estimate of changed rows (107-113). */
/* dst[j] = max(dst[j], src[j]); restrict-qualified so the loop vectorises */
static inline void max_into(uint8_t *restrict dst, const uint8_t *restrict src, int64_t p) {
    for (int64_t j = 0; j < p; j++) dst[j] = src[j] > dst[j] ? src[j] : dst[j];
}

/* target_clones: the reference's numba kernels are JIT-compiled for the host CPU, so the
 * port dispatches at load time to an AVX2 build where the CPU has it (same results: the
 * byte max is exact in any width). */
__attribute__((target_clones("avx2", "default")))
int64_t orc_union_range(int64_t lo, int64_t hi, const int64_t *offsets, const int64_t *succ,
                        const uint8_t *cur, uint8_t *nxt, const uint8_t *changed_prev,
                        uint8_t *changed_now, const double *est, double *new_est, int b,
                        int skip_stable) {
    double a2, lc, pf;
    orc_constants(b, &a2, &lc, &pf);
    int64_t p = 1LL << b;
    int64_t nch = 0;
    for (int64_t v = lo; v < hi; v++) {
        int active = changed_prev[v] != 0;
        if (!active) {
            for (int64_t k = offsets[v]; k < offsets[v + 1]; k++) {
                if (changed_prev[succ[k]]) { active = 1; break; }
            }
        }
        const uint8_t *cv = cur + v * p;
        uint8_t *nv = nxt + v * p;
        if (skip_stable && !active) {
            memcpy(nv, cv, (size_t)p);
            changed_now[v] = 0;
            new_est[v] = est[v];
            continue;
        }
        memcpy(nv, cv, (size_t)p);
        for (int64_t k = offsets[v]; k < offsets[v + 1]; k++) {
            max_into(nv, cur + succ[k] * p, p);
        }
        int changed = memcmp(nv, cv, (size_t)p) != 0;
        changed_now[v] = (uint8_t)changed;
        if (changed) {
            nch++;
            new_est[v] = orc_estimate_row(nv, p, a2, lc, pf);
        } else {
            new_est[v] = est[v];
        }
    }
    return nch;
}

/* engine.py:351-359: arc-balanced contiguous node ranges.  numpy.linspace(0, m, W+1)
 * then searchsorted(offsets, targets) (side='left'); the first bound is 0, the last n,
 * then a running max.  Any partition gives identical results (row-local writes), so
 * only the balance matters here. */
static void worker_bounds(const int64_t *offsets, int64_t n, int workers, int64_t *bounds) {
    int64_t m = offsets[n];
    for (int w = 0; w <= workers; w++) {
        double target = (double)m * (double)w / (double)workers;
        int64_t lo = 0, hi = n + 1;  /* first index with offsets[i] >= target */
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if ((double)offsets[mid] < target) lo = mid + 1; else hi = mid;
        }
        bounds[w] = lo;
    }
    bounds[0] = 0;
    bounds[workers] = n;
    for (int w = 1; w <= workers; w++)
        if (bounds[w] < bounds[w - 1]) bounds[w] = bounds[w - 1];
}

typedef struct {
    int64_t lo, hi;
    const int64_t *offsets, *succ;
    const uint8_t *cur;
    uint8_t *nxt;
    const uint8_t *chg_prev;
    uint8_t *chg_now;
    const double *est;
    double *new_est;
    int b, skip;
    int64_t nch;
} orc_job;

static void *orc_job_run(void *arg) {
    orc_job *j = (orc_job *)arg;
    j->nch = orc_union_range(j->lo, j->hi, j->offsets, j->succ, j->cur, j->nxt, j->chg_prev,
                             j->chg_now, j->est, j->new_est, j->b, j->skip);
    return NULL;
}

/* engine.py:362-390: one union pass over nodes [lo, hi) split into arc-balanced ranges
 * over `workers` threads; returns the total changed count (the `sum(f.result() ...)`
 * barrier).  All arrays are full-size (indexed by global node id). */
int64_t orc_iterate_range_mt(int64_t lo, int64_t hi, const int64_t *offsets,
                             const int64_t *succ, const uint8_t *cur, uint8_t *nxt,
                             const uint8_t *chg_prev, uint8_t *chg_now, const double *est,
                             double *new_est, int b, int skip, int workers) {
    int64_t n = hi - lo;
    if (n <= 0) return 0;
    if (workers < 1) workers = 1;
    if (workers > n) workers = (int)n;
    if (workers == 1)
        return orc_union_range(lo, hi, offsets, succ, cur, nxt, chg_prev, chg_now, est,
                               new_est, b, skip);
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(workers + 1));
    orc_job *jobs = (orc_job *)calloc((size_t)workers, sizeof(orc_job));
    pthread_t *th = (pthread_t *)calloc((size_t)workers, sizeof(pthread_t));
    /* bounds over the sub-range: shift offsets so the range starts at arc 0 */
    int64_t *sub = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i <= n; i++) sub[i] = offsets[lo + i] - offsets[lo];
    worker_bounds(sub, n, workers, bounds);
    free(sub);
    for (int w = 0; w < workers; w++) {
        orc_job *j = &jobs[w];
        j->lo = lo + bounds[w]; j->hi = lo + bounds[w + 1];
        j->offsets = offsets; j->succ = succ; j->cur = cur; j->nxt = nxt;
        j->chg_prev = chg_prev; j->chg_now = chg_now; j->est = est; j->new_est = new_est;
        j->b = b; j->skip = skip; j->nch = 0;
        if (j->hi > j->lo) pthread_create(&th[w], NULL, orc_job_run, j);
    }
    int64_t nch = 0;
    for (int w = 0; w < workers; w++) {
        if (jobs[w].hi > jobs[w].lo) { pthread_join(th[w], NULL); nch += jobs[w].nch; }
    }
    free(bounds); free(jobs); free(th);
    return nch;
}

int64_t orc_iterate_mt(int64_t n, const int64_t *offsets, const int64_t *succ,
                       const uint8_t *cur, uint8_t *nxt, const uint8_t *chg_prev,
                       uint8_t *chg_now, const double *est, double *new_est, int b, int skip,
                       int workers) {
    return orc_iterate_range_mt(0, n, offsets, succ, cur, nxt, chg_prev, chg_now, est, new_est,
                                b, skip, workers);
}

/* numpy.maximum(x, 0.0): returns x when x >= 0 or x is NaN, else 0.0 */
static inline double np_max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }

/* centrality.py:132-135,143-148: delta = maximum(new - old, 0); sum_dist += t * delta;
 * sum_recip += delta / t.  Each op is a separately rounded numpy fp64 op. */
void orc_accumulate(int64_t n, int64_t t, const double *old_est, const double *new_est,
                    double *sum_dist, double *sum_recip) {
    double tf = (double)t;
    for (int64_t v = 0; v < n; v++) {
        double d = np_max0(new_est[v] - old_est[v]);
        double td = tf * d;
        sum_dist[v] = sum_dist[v] + td;
        double dt = d / tf;
        sum_recip[v] = sum_recip[v] + dt;
    }
}

/* centrality.py:153-171 */
void orc_finalize(int64_t n, const double *sum_dist, const double *sum_recip,
                  const double *coreach, double *closeness, double *harmonic, double *lin) {
    for (int64_t v = 0; v < n; v++) {
        double s = sum_dist[v];
        closeness[v] = s > 0 ? 1.0 / s : 0.0;
        harmonic[v] = sum_recip[v];
        lin[v] = s > 0 ? (coreach[v] * coreach[v]) / s : 1.0;
    }
}
