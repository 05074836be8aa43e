/*
 * graphgen.c -- deterministic synthetic graph builders for the five BASELINE configs,
 * emitting the CSR of the TRANSPOSE graph (the engine runs on G^T: cli.py:213-216,
 * SURVEY.md Appendix B).  Host C, multithreaded with pthreads.
 *
 * The reference builds graphs with CsrGraph.from_edges (graph.py:52-80: lexsort,
 * dedup, CSR) and transpose (graph.py:145-155).  This file produces the same normalised
 * object -- successor lists sorted ascending, duplicate arcs removed -- for G^T directly,
 * and additionally drops self-loops as BASELINE.json's configs ask.
 *
 * Randomness is counter-based (splitmix64 finaliser chains keyed by (seed, stream,
 * index)), so every arc is a pure function of its index: the output is bit-identical
 * for any thread count and on any x86-64 host, which is what lets the GPU run, the CPU
 * oracle and the golden fixtures agree on "the same graph" without shipping it.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define C1 0xBF58476D1CE4E5B9ULL
#define C2 0x94D049BB133111EBULL

static inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * C1;
    z = (z ^ (z >> 27)) * C2;
    return z ^ (z >> 31);
}
static inline uint64_t rng3(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    return mix(mix(mix(seed * 0x9E3779B97F4A7C15ULL + stream) + a) + b);
}
static inline double u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
static inline uint64_t below(uint64_t x, uint64_t n) {
    return (uint64_t)(((__uint128_t)x * (__uint128_t)n) >> 64);
}

enum { GEN_ER = 1, GEN_RMAT = 2, GEN_DISC = 3, GEN_WEB = 4, GEN_EDGES = 5 };

typedef struct {
    int kind;
    int64_t n;
    int64_t m_target;  /* R-MAT: number of generated arcs */
    uint64_t seed;
    double mean;       /* Poisson mean (ER, disconnected) */
    double a, b, c;    /* R-MAT quadrant probabilities */
    int scale;
    int64_t giant;     /* disconnected: giant block size */
    double geo_p;      /* disconnected: Geometric(p) block sizes */
    double alpha;      /* web: Zipf exponent */
    int64_t kmin, kmax;/* web: Zipf support */
    double p_local;    /* web: probability of a local arc */
    int64_t window;    /* web: local arc offset range 1..window */
} gen_params;

typedef struct {
    int64_t n, m;
    int64_t *offsets;  /* [n+1] */
    int32_t *succ;     /* [m] */
} hbg_graph;

static int nthreads_default(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

/* ---------------------------------------------------------------- thread helper */
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi, int tid);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; int tid; } par_job;
static void *par_run(void *a) {
    par_job *j = (par_job *)a;
    j->fn(j->ctx, j->lo, j->hi, j->tid);
    return NULL;
}
static void parallel_for(int64_t n, int threads, range_fn fn, void *ctx) {
    if (threads < 1) threads = 1;
    if (n < 4096 || threads == 1) { fn(ctx, 0, n, 0); return; }
    pthread_t th[256];
    par_job jobs[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; t++) {
        jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].tid = t;
        jobs[t].lo = n * t / threads; jobs[t].hi = n * (t + 1) / threads;
        pthread_create(&th[t], NULL, par_run, &jobs[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- distributions */
typedef struct { double cdf[256]; int kmax; } poisson_tab;
static void poisson_init(poisson_tab *t, double lam) {
    double pk = exp(-lam), acc = 0.0;
    int k;
    for (k = 0; k < 255; k++) {
        acc += pk;
        t->cdf[k] = acc;
        pk = pk * lam / (double)(k + 1);
        if (acc >= 1.0 - 1e-17 && k > lam) break;
    }
    t->kmax = k;
    t->cdf[k] = 2.0;  /* sentinel: any u < 1 stops here */
}
static inline int poisson_draw(const poisson_tab *t, double u) {
    int k = 0;
    while (u >= t->cdf[k]) k++;
    return k;
}

typedef struct { double *cdf; int64_t kmin, kmax; } zipf_tab;
static void zipf_init(zipf_tab *z, double alpha, int64_t kmin, int64_t kmax) {
    int64_t len = kmax - kmin + 1;
    z->cdf = (double *)malloc(sizeof(double) * (size_t)len);
    z->kmin = kmin; z->kmax = kmax;
    double tot = 0.0;
    for (int64_t i = 0; i < len; i++) tot += pow((double)(kmin + i), -alpha);
    double acc = 0.0;
    for (int64_t i = 0; i < len; i++) {
        acc += pow((double)(kmin + i), -alpha) / tot;
        z->cdf[i] = acc;
    }
    z->cdf[len - 1] = 2.0;
}
static inline int64_t zipf_draw(const zipf_tab *z, double u) {
    int64_t lo = 0, hi = z->kmax - z->kmin;  /* first i with u < cdf[i] */
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (u < z->cdf[mid]) hi = mid; else lo = mid + 1;
    }
    return z->kmin + lo;
}

/* ---------------------------------------------------------------- arc generation */
typedef struct {
    const gen_params *P;
    poisson_tab pois;
    zipf_tab zipf;
    int64_t *block_lo;      /* disconnected: block start of node v */
    int64_t *block_hi;
    int64_t *deg;           /* per-source out-degree (pre-dedup), then offsets */
    uint32_t *src, *dst;
} arc_ctx;

static int64_t out_degree(arc_ctx *c, int64_t u) {
    const gen_params *P = c->P;
    switch (P->kind) {
    case GEN_ER:
    case GEN_DISC:
        return poisson_draw(&c->pois, u01(rng3(P->seed, 1, (uint64_t)u, 0)));
    case GEN_WEB:
        return zipf_draw(&c->zipf, u01(rng3(P->seed, 1, (uint64_t)u, 0)));
    }
    return 0;
}

static void deg_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    arc_ctx *c = (arc_ctx *)ctx;
    for (int64_t u = lo; u < hi; u++) c->deg[u] = out_degree(c, u);
}

static void fill_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    arc_ctx *c = (arc_ctx *)ctx;
    const gen_params *P = c->P;
    int64_t n = P->n;
    for (int64_t u = lo; u < hi; u++) {
        int64_t base = c->deg[u], k = c->deg[u + 1] - base;
        for (int64_t j = 0; j < k; j++) {
            uint64_t r = rng3(P->seed, 2, (uint64_t)u, (uint64_t)j);
            int64_t v;
            if (P->kind == GEN_ER) {
                /* uniform on V \ {u} */
                v = (int64_t)below(r, (uint64_t)(n - 1));
                if (v >= u) v++;
            } else if (P->kind == GEN_DISC) {
                int64_t blo = c->block_lo[u], bhi = c->block_hi[u];
                v = blo + (int64_t)below(r, (uint64_t)(bhi - blo));
            } else { /* GEN_WEB */
                uint64_t r2 = rng3(P->seed, 3, (uint64_t)u, (uint64_t)j);
                if (u01(r) < P->p_local) {
                    int64_t off = 1 + (int64_t)below(r2 >> 1, (uint64_t)P->window);
                    v = (r2 & 1) ? u + off : u - off;
                    v %= n;
                    if (v < 0) v += n;
                } else {
                    v = (int64_t)below(r2, (uint64_t)n);
                }
            }
            c->src[base + j] = (uint32_t)u;
            c->dst[base + j] = (uint32_t)v;
        }
    }
}

static void rmat_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    arc_ctx *c = (arc_ctx *)ctx;
    const gen_params *P = c->P;
    const uint64_t A = (uint64_t)(P->a * 4294967296.0);
    const uint64_t AB = (uint64_t)((P->a + P->b) * 4294967296.0);
    const uint64_t ABC = (uint64_t)((P->a + P->b + P->c) * 4294967296.0);
    for (int64_t k = lo; k < hi; k++) {
        uint64_t s = 0, d = 0, r = 0;
        for (int l = 0; l < P->scale; l++) {
            uint64_t x;
            if ((l & 1) == 0) { r = rng3(P->seed, 4, (uint64_t)k, (uint64_t)(l >> 1)); x = r & 0xffffffffULL; }
            else x = r >> 32;
            int q = x < A ? 0 : (x < AB ? 1 : (x < ABC ? 2 : 3));
            s = (s << 1) | (uint64_t)(q >> 1);
            d = (d << 1) | (uint64_t)(q & 1);
        }
        c->src[k] = (uint32_t)s;
        c->dst[k] = (uint32_t)d;
    }
}

/* ---------------------------------------------------------------- transpose build */
typedef struct {
    int64_t n, M;
    const uint32_t *src, *dst;
    int64_t *cnt;          /* in-degree counts -> offsets */
    int64_t *cursor;
    int32_t *tmp;          /* scattered G^T rows (pre-sort) */
    int64_t *newdeg;
    int64_t *out_off;
    int32_t *out;
} tr_ctx;

static void count_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    tr_ctx *c = (tr_ctx *)ctx;
    for (int64_t k = lo; k < hi; k++) {
        if (c->src[k] == c->dst[k]) continue;  /* self-loop dropped */
        __atomic_fetch_add(&c->cnt[c->dst[k]], 1, __ATOMIC_RELAXED);
    }
}
static void scatter_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    tr_ctx *c = (tr_ctx *)ctx;
    for (int64_t k = lo; k < hi; k++) {
        uint32_t u = c->src[k], v = c->dst[k];
        if (u == v) continue;
        int64_t pos = __atomic_fetch_add(&c->cursor[v], 1, __ATOMIC_RELAXED);
        c->tmp[pos] = (int32_t)u;
    }
}
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}
static void sortrow_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    tr_ctx *c = (tr_ctx *)ctx;
    for (int64_t v = lo; v < hi; v++) {
        int32_t *row = c->tmp + c->cnt[v];
        int64_t len = c->cnt[v + 1] - c->cnt[v];
        if (len > 32) qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
        else {
            for (int64_t i = 1; i < len; i++) {
                int32_t x = row[i];
                int64_t j = i - 1;
                while (j >= 0 && row[j] > x) { row[j + 1] = row[j]; j--; }
                row[j + 1] = x;
            }
        }
        int64_t w = 0;
        for (int64_t i = 0; i < len; i++)
            if (w == 0 || row[i] != row[w - 1]) row[w++] = row[i];
        c->newdeg[v] = w;
    }
}
static void compact_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    tr_ctx *c = (tr_ctx *)ctx;
    for (int64_t v = lo; v < hi; v++)
        memcpy(c->out + c->out_off[v], c->tmp + c->cnt[v], sizeof(int32_t) * (size_t)c->newdeg[v]);
}

static void exclusive_scan(int64_t *a, int64_t n) { /* a[0..n) -> offsets in a[0..n] */
    int64_t acc = 0;
    for (int64_t i = 0; i < n; i++) { int64_t x = a[i]; a[i] = acc; acc += x; }
    a[n] = acc;
}

static hbg_graph *transpose_build(int64_t n, int64_t M, const uint32_t *src,
                                  const uint32_t *dst, int threads) {
    tr_ctx c;
    memset(&c, 0, sizeof(c));
    c.n = n; c.M = M; c.src = src; c.dst = dst;
    c.cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    parallel_for(M, threads, count_fn, &c);
    exclusive_scan(c.cnt, n);
    c.cursor = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    memcpy(c.cursor, c.cnt, sizeof(int64_t) * ((size_t)n + 1));
    c.tmp = (int32_t *)malloc(sizeof(int32_t) * ((size_t)c.cnt[n] + 1));
    parallel_for(M, threads, scatter_fn, &c);
    free(c.cursor);
    c.newdeg = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    parallel_for(n, threads, sortrow_fn, &c);
    c.out_off = c.newdeg;  /* scan in place */
    exclusive_scan(c.out_off, n);
    /* newdeg is gone after the scan; compact needs lengths: recompute from out_off */
    hbg_graph *g = (hbg_graph *)calloc(1, sizeof(hbg_graph));
    g->n = n;
    g->m = c.out_off[n];
    g->offsets = c.out_off;
    g->succ = (int32_t *)malloc(sizeof(int32_t) * ((size_t)g->m + 1));
    c.out = g->succ;
    /* restore per-row lengths for compact_fn */
    int64_t *lens = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t v = 0; v < n; v++) lens[v] = c.out_off[v + 1] - c.out_off[v];
    c.newdeg = lens;
    parallel_for(n, threads, compact_fn, &c);
    free(lens);
    free(c.tmp);
    free(c.cnt);
    return g;
}

/* ---------------------------------------------------------------- public C-ABI */
static hbg_graph *generate(const gen_params *P, int threads) {
    if (threads <= 0) threads = nthreads_default();
    int64_t n = P->n;
    arc_ctx c;
    memset(&c, 0, sizeof(c));
    c.P = P;
    int64_t M;
    if (P->kind == GEN_RMAT) {
        M = P->m_target;
        c.src = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)M + 1));
        c.dst = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)M + 1));
        parallel_for(M, threads, rmat_fn, &c);
    } else {
        if (P->kind == GEN_ER || P->kind == GEN_DISC) poisson_init(&c.pois, P->mean);
        if (P->kind == GEN_WEB) zipf_init(&c.zipf, P->alpha, P->kmin, P->kmax);
        if (P->kind == GEN_DISC) {
            c.block_lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
            c.block_hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
            int64_t g = P->giant < n ? P->giant : n;
            for (int64_t v = 0; v < g; v++) { c.block_lo[v] = 0; c.block_hi[v] = g; }
            int64_t pos = g, blk = 0;
            while (pos < n) {
                int64_t size = 1;  /* Geometric(p) on {1, 2, ...}: trials to first success */
                while (u01(rng3(P->seed, 5, (uint64_t)blk, (uint64_t)size)) >= P->geo_p) size++;
                int64_t hi = pos + size < n ? pos + size : n;
                for (int64_t v = pos; v < hi; v++) { c.block_lo[v] = pos; c.block_hi[v] = hi; }
                pos = hi;
                blk++;
            }
        }
        c.deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
        parallel_for(n, threads, deg_fn, &c);
        exclusive_scan(c.deg, n);
        M = c.deg[n];
        c.src = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)M + 1));
        c.dst = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)M + 1));
        parallel_for(n, threads, fill_fn, &c);
        free(c.deg);
        free(c.block_lo);
        free(c.block_hi);
        free(c.zipf.cdf);
    }
    hbg_graph *g = transpose_build(n, M, c.src, c.dst, threads);
    free(c.src);
    free(c.dst);
    return g;
}

void *hbg_er(int64_t n, double mean, uint64_t seed, int threads) {
    gen_params P; memset(&P, 0, sizeof(P));
    P.kind = GEN_ER; P.n = n; P.mean = mean; P.seed = seed;
    return generate(&P, threads);
}

void *hbg_rmat(int scale, int64_t m, double a, double b, double c, uint64_t seed, int threads) {
    gen_params P; memset(&P, 0, sizeof(P));
    P.kind = GEN_RMAT; P.scale = scale; P.n = 1LL << scale; P.m_target = m;
    P.a = a; P.b = b; P.c = c; P.seed = seed;
    return generate(&P, threads);
}

void *hbg_disconnected(int64_t n, int64_t giant, double geo_p, double mean, uint64_t seed,
                       int threads) {
    gen_params P; memset(&P, 0, sizeof(P));
    P.kind = GEN_DISC; P.n = n; P.giant = giant; P.geo_p = geo_p; P.mean = mean; P.seed = seed;
    return generate(&P, threads);
}

void *hbg_weblike(int64_t n, double alpha, int64_t kmin, int64_t kmax, double p_local,
                  int64_t window, uint64_t seed, int threads) {
    gen_params P; memset(&P, 0, sizeof(P));
    P.kind = GEN_WEB; P.n = n; P.alpha = alpha; P.kmin = kmin; P.kmax = kmax;
    P.p_local = p_local; P.window = window; P.seed = seed;
    return generate(&P, threads);
}

/* Transpose + normalise an explicit arc list (graph.py:52-80 + 145-155, self-loops
 * dropped). */
void *hbg_from_arcs(int64_t n, int64_t M, const uint32_t *src, const uint32_t *dst,
                    int threads) {
    if (threads <= 0) threads = nthreads_default();
    return transpose_build(n, M, src, dst, threads);
}

/* The CDF tables the degree draws use (for the device builders, which must draw
 * bit-identical degrees: hb_gen_degrees).  hbg_poisson_cdf writes up to 256 entries and
 * returns the count (the last one is the 2.0 sentinel); hbg_zipf_cdf writes kmax-kmin+1. */
int hbg_poisson_cdf(double lam, double *out) {
    poisson_tab t;
    poisson_init(&t, lam);
    memcpy(out, t.cdf, sizeof(double) * (size_t)(t.kmax + 1));
    return t.kmax + 1;
}
void hbg_zipf_cdf(double alpha, int64_t kmin, int64_t kmax, double *out) {
    zipf_tab z;
    zipf_init(&z, alpha, kmin, kmax);
    memcpy(out, z.cdf, sizeof(double) * (size_t)(kmax - kmin + 1));
    free(z.cdf);
}

/* Rank-local CSR for multi-GPU runs: rows[i] (old row ids, int32
 * [nrows]) of a host CSR (offsets int64 [n+1], successors int32 or int64 by
 * succ_bytes = 4 / 8) packed into out_off (int64 [nrows+1], local positions) and out
 * (int32, narrowed ids), so each rank uploads only the ~m/W ids of the rows it owns. */
typedef struct {
    const int64_t *off;
    const void *succ;
    int succ_bytes;
    const int32_t *rows;
    const int64_t *out_off;
    int32_t *out;
} gather_ctx;

static void gather_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    gather_ctx *c = (gather_ctx *)ctx;
    for (int64_t i = lo; i < hi; i++) {
        const int64_t r = c->rows[i], b = c->off[r], len = c->off[r + 1] - b;
        int32_t *dst = c->out + c->out_off[i];
        if (c->succ_bytes == 4) {
            memcpy(dst, (const int32_t *)c->succ + b, sizeof(int32_t) * (size_t)len);
        } else {
            const int64_t *src = (const int64_t *)c->succ + b;
            for (int64_t k = 0; k < len; k++) dst[k] = (int32_t)src[k];
        }
    }
}

int64_t hbg_gather_rows(const int64_t *off, const void *succ, int succ_bytes,
                        const int32_t *rows, int64_t nrows, int64_t *out_off, int32_t *out,
                        int threads) {
    if (threads <= 0) threads = nthreads_default();
    int64_t acc = 0;
    for (int64_t i = 0; i < nrows; i++) {
        out_off[i] = acc;
        acc += off[rows[i] + 1] - off[rows[i]];
    }
    out_off[nrows] = acc;
    if (out == NULL) return acc;            /* size query */
    gather_ctx c = {off, succ, succ_bytes, rows, out_off, out};
    parallel_for(nrows, threads, gather_fn, &c);
    return acc;
}

/* Staging for uploads from pageable host memory (schedule.py _upload_slices): n elements
 * of src (src_bytes = 4: int32, copied; 8: the reference's int64 ids, narrowed to int32)
 * into dst (a pinned buffer the caller then copies to the device), over `threads`
 * pthreads -- the narrowing and the page walk run at host-memory speed on every core
 * while the previous slice crosses PCIe.  hbg_stage_bytes: the same as a plain copy. */
typedef struct {
    const void *src;
    int src_bytes;
    void *dst;
} stage_ctx;

static void stage_fn(void *ctx, int64_t lo, int64_t hi, int tid) {
    (void)tid;
    stage_ctx *c = (stage_ctx *)ctx;
    if (c->src_bytes == 8) {
        const int64_t *s = (const int64_t *)c->src;
        int32_t *d = (int32_t *)c->dst;
        for (int64_t i = lo; i < hi; i++) d[i] = (int32_t)s[i];
    } else {
        memcpy((char *)c->dst + (size_t)lo * (size_t)c->src_bytes,
               (const char *)c->src + (size_t)lo * (size_t)c->src_bytes,
               (size_t)(hi - lo) * (size_t)c->src_bytes);
    }
}

int hbg_stage_ids(const void *src, int src_bytes, int64_t n, int32_t *dst, int threads) {
    if (src_bytes != 4 && src_bytes != 8) return -1;
    if (threads <= 0) threads = nthreads_default();
    stage_ctx c = {src, src_bytes, dst};
    parallel_for(n, threads, stage_fn, &c);
    return 0;
}

void hbg_stage_bytes(const void *src, int64_t nbytes, void *dst, int threads) {
    if (threads <= 0) threads = nthreads_default();
    stage_ctx c = {src, 1, dst};
    parallel_for(nbytes, threads, stage_fn, &c);
}

int64_t hbg_n(void *h) { return ((hbg_graph *)h)->n; }
int64_t hbg_m(void *h) { return ((hbg_graph *)h)->m; }
void hbg_copy(void *h, int64_t *offsets, int32_t *succ) {
    hbg_graph *g = (hbg_graph *)h;
    memcpy(offsets, g->offsets, sizeof(int64_t) * ((size_t)g->n + 1));
    memcpy(succ, g->succ, sizeof(int32_t) * (size_t)g->m);
}
void hbg_free(void *h) {
    hbg_graph *g = (hbg_graph *)h;
    if (!g) return;
    free(g->offsets);
    free(g->succ);
    free(g);
}
