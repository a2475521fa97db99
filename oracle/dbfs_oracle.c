/*
 * dbfs_oracle.c -- CPU restatement of the reference delegate-BFS path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1803_03922_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product never links or calls it.
 *
 * It restates, function by function, the reference package
 * /root/reference/pkg/src/delegate_bfs (pure Python/numpy):
 *   - generation      rmat.py:107-122 (_mix64, _uniform_draws),
 *                     rmat.py:125-150 (generate_rmat),
 *                     rmat.py:153-182 (hash_randomize_vertices),
 *                     rmat.py:185-189 (symmetrize)
 *   - partition       partition.py:103-117 (degrees, classification),
 *                     partition.py:156-177 (distribute_edges, Alg. 1),
 *                     partition.py:132-137 + 295-340 (stable CSR build)
 *   - BFS engine      engine.py:98-330 (run_bfs) with traversal.py:58-163
 *                     (previsit, visit_forward, visit_backward,
 *                     estimate_backward_workload, decide_direction) and
 *                     comm.py:75-197 (mask reduction, normal exchange)
 *   - NEW (no reference): min-ID parents and the Graph500
 *     certificate.
 *
 * Pinned against the reference by tests/golden (fixtures produced by
 * tests/golden/make_golden.py from the reference itself) and, when
 * /root/reference is present, by live comparison in tests/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ERANGE 2
#define ORC_ECAPACITY 3
#define ORC_ENOMEM 4

enum { NN = 0, ND = 1, DN = 2, DD = 3 };
enum { FWD = 0, BWD = 1 };

/* ------------------------------------------------------------------ */
/* Generation: rmat.py:107-189                                         */
/* ------------------------------------------------------------------ */

static inline uint64_t mix64(uint64_t x) { /* rmat.py:107-115 */
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

/* r = (base >> 11) * 2^-53 is exactly k * 2^-53 with k an integer < 2^53,
 * so r >= t  <=>  k >= ceil(t * 2^53).  t * 2^53 is exact in binary64. */
static uint64_t threshold53(double t) {
    double x = t * 9007199254740992.0;
    if (x <= 0.0) return 0;
    if (x >= 9007199254740992.0) return 1ULL << 53;
    uint64_t k = (uint64_t)x;
    if ((double)k < x) k++;
    return k;
}

typedef struct {
    int scale;
    int64_t n, m0;
    uint64_t key;
    uint64_t ta, tab, tabc;
    int randomize;               /* bit 0: reference hash; bit 1: Feistel scramble (this build) */
    uint64_t mask, c1, m1, m2;
    int s1, s2;
    uint64_t skey;
} rmat_gen;

static void rmat_gen_init(rmat_gen *g, int scale, int64_t ef, double a, double b,
                          double c, uint64_t seed, int randomize) {
    g->scale = scale;
    g->n = (int64_t)1 << scale;
    g->m0 = g->n * ef;
    g->key = mix64(seed); /* rmat.py:120 */
    double ab = a + b, abc = ab + c; /* rmat.py:130-131 */
    g->ta = threshold53(a);
    g->tab = threshold53(ab);
    g->tabc = threshold53(abc);
    g->randomize = randomize;
    /* rmat.py:164-171 */
    g->mask = (uint64_t)g->n - 1;
    int k = scale;
    g->s1 = k / 3 > 1 ? k / 3 : 1;
    g->s2 = k / 2 > 1 ? k / 2 : 1;
    g->c1 = mix64(seed) & g->mask;
    g->m1 = (0x9E3779B97F4A7C15ULL & 0x7FFFFFFFFFFFFFFFULL) | 1ULL;
    g->m2 = (0xBF58476D1CE4E5B9ULL & 0x7FFFFFFFFFFFFFFFULL) | 1ULL;
    g->skey = mix64(seed ^ 0x5CA3B1E5D00DF00DULL);
}

static inline uint64_t hash_perm(const rmat_gen *g, uint64_t v) { /* rmat.py:173-180 */
    v = (v * g->m1) & g->mask;
    v ^= (v << g->s1) & g->mask;
    v = (v + g->c1) & g->mask;
    v = (v * g->m2) & g->mask;
    v ^= (v << g->s2) & g->mask;
    return v;
}

/* Optional relabeling of this build (not in the reference): a 3-round Feistel
 * bijection on the scale bits, applied after the reference hash.  The
 * reference hash keeps low id bits a function of low bits only, so owners
 * v mod p inherit RMAT's bit-pattern degree skew; the scramble makes every id
 * bit depend on all of them.  Same function as csrc/build.cu scramble(). */
static inline uint64_t scramble(const rmat_gen *g, uint64_t v) {
    int k = g->scale;
    if (k < 2) return v;
    int j = k / 2;
    uint64_t lm = (1ULL << j) - 1, hm = (1ULL << (k - j)) - 1;
    uint64_t lo = v & lm, hi = v >> j;
    lo ^= mix64(hi ^ g->skey) & lm;
    hi ^= mix64(lo ^ (g->skey + 1)) & hm;
    lo ^= mix64(hi ^ (g->skey + 2)) & lm;
    return (hi << j) | lo;
}

/* One original (undoubled) RMAT edge, rmat.py:139-148. */
static inline void rmat_edge(const rmat_gen *g, uint64_t e, uint64_t *u, uint64_t *v) {
    uint64_t su = 0, sv = 0;
    for (int l = 0; l < g->scale; l++) {
        uint64_t cnt = e * (uint64_t)g->scale + (uint64_t)l;
        uint64_t k = mix64(g->key ^ cnt) >> 11;
        uint64_t ub = k >= g->tab;
        uint64_t vb = (k >= g->ta && k < g->tab) || k >= g->tabc;
        su |= ub << (g->scale - 1 - l);
        sv |= vb << (g->scale - 1 - l);
    }
    if (g->randomize & 1) {
        su = hash_perm(g, su);
        sv = hash_perm(g, sv);
    }
    if (g->randomize & 2) {
        su = scramble(g, su);
        sv = scramble(g, sv);
    }
    *u = su;
    *v = sv;
}

/* Edges [begin, end) of the (optionally symmetrized) RMAT edge list built by
 * build_rmat_graph (rmat.py:200-208): index e < m0 is original edge e, index
 * e >= m0 is the reverse of original edge e - m0 (rmat.py:185-189). */
typedef struct {
    const rmat_gen *g;
    int64_t begin, lo, hi;
    int64_t *src, *dst;
} gen_job;

static void *gen_worker(void *arg) {
    gen_job *j = (gen_job *)arg;
    const rmat_gen *g = j->g;
    for (int64_t i = j->lo; i < j->hi; i++) {
        uint64_t u, v;
        int64_t e = i >= g->m0 ? i - g->m0 : i;
        rmat_edge(g, (uint64_t)e, &u, &v);
        if (i >= g->m0) { uint64_t t = u; u = v; v = t; }
        j->src[i - j->begin] = (int64_t)u;
        j->dst[i - j->begin] = (int64_t)v;
    }
    return NULL;
}

static int orc_threads(void) {
    const char *e = getenv("ORC_THREADS");
    long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 256) t = 256;
    return (int)t;
}

int orc_rmat_edges(int scale, int64_t edge_factor, double a, double b, double c,
                   uint64_t seed, int randomize, int symmetrize, int64_t begin,
                   int64_t end, int64_t *src, int64_t *dst) {
    if (scale < 0 || scale > 40 || edge_factor < 1) return ORC_EINVAL;
    rmat_gen g;
    rmat_gen_init(&g, scale, edge_factor, a, b, c, seed, randomize);
    int64_t m = symmetrize ? 2 * g.m0 : g.m0;
    if (begin < 0 || end > m || begin > end) return ORC_ERANGE;
    int T = orc_threads();
    if (end - begin < (1 << 16)) T = 1;
    pthread_t th[256];
    gen_job jobs[256];
    int64_t per = (end - begin + T - 1) / T;
    for (int t = 0; t < T; t++) {
        jobs[t].g = &g; jobs[t].begin = begin; jobs[t].src = src; jobs[t].dst = dst;
        jobs[t].lo = begin + per * t < end ? begin + per * t : end;
        jobs[t].hi = jobs[t].lo + per < end ? jobs[t].lo + per : end;
        if (T > 1) pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
        else gen_worker(&jobs[t]);
    }
    if (T > 1) for (int t = 0; t < T; t++) pthread_join(th[t], NULL);
    return ORC_OK;
}

/* Graph summary straight from the counter-based generator, without storing
 * the edge list: out-degrees (partition.py:103-104, bincount over the
 * symmetrized list, i.e. deg(u)++ and deg(v)++ per original edge), the
 * delegate count d = |{v : deg(v) > theta}| (partition.py:79-117) and the
 * kind totals (partition.py:312-318; the kind of an edge depends only on its
 * endpoints' classes).  Two multithreaded passes over the m0 original edges,
 * so graphs far larger than the host could partition (scale 26-30) can be
 * checked against the device build. */
typedef struct {
    const rmat_gen *g;
    int64_t lo, hi;
    uint32_t *deg;
    const uint32_t *deg_ro;
    int64_t theta;
    int64_t kinds[4];
} sum_job;

static void *sum_deg_worker(void *arg) {
    sum_job *j = (sum_job *)arg;
    for (int64_t e = j->lo; e < j->hi; e++) {
        uint64_t u, v;
        rmat_edge(j->g, (uint64_t)e, &u, &v);
        __atomic_fetch_add(&j->deg[u], 1u, __ATOMIC_RELAXED);
        __atomic_fetch_add(&j->deg[v], 1u, __ATOMIC_RELAXED);
    }
    return NULL;
}

static void *sum_kind_worker(void *arg) {
    sum_job *j = (sum_job *)arg;
    int64_t k[4] = {0, 0, 0, 0};
    for (int64_t e = j->lo; e < j->hi; e++) {
        uint64_t u, v;
        rmat_edge(j->g, (uint64_t)e, &u, &v);
        int du = (int64_t)j->deg_ro[u] > j->theta, dv = (int64_t)j->deg_ro[v] > j->theta;
        k[(du << 1) | dv]++;  /* original edge u->v */
        k[(dv << 1) | du]++;  /* its reverse (symmetrize) */
    }
    for (int i = 0; i < 4; i++) j->kinds[i] = k[i];
    return NULL;
}

int orc_rmat_summary(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                     int randomize, int64_t theta, uint32_t *deg_out, int64_t *d_out,
                     int64_t *kind_totals) {
    if (scale < 0 || scale > 40 || edge_factor < 1 || theta < 0) return ORC_EINVAL;
    rmat_gen g;
    rmat_gen_init(&g, scale, edge_factor, a, b, c, seed, randomize);
    memset(deg_out, 0, sizeof(uint32_t) * (size_t)g.n);
    int T = orc_threads();
    if (g.m0 < (1 << 16)) T = 1;
    pthread_t th[256];
    sum_job jobs[256];
    int64_t per = (g.m0 + T - 1) / T;
    for (int pass = 0; pass < 2; pass++) {
        for (int t = 0; t < T; t++) {
            memset(&jobs[t], 0, sizeof(sum_job));
            jobs[t].g = &g; jobs[t].deg = deg_out; jobs[t].deg_ro = deg_out; jobs[t].theta = theta;
            jobs[t].lo = per * t < g.m0 ? per * t : g.m0;
            jobs[t].hi = jobs[t].lo + per < g.m0 ? jobs[t].lo + per : g.m0;
            void *(*fn)(void *) = pass == 0 ? sum_deg_worker : sum_kind_worker;
            if (T > 1) pthread_create(&th[t], NULL, fn, &jobs[t]);
            else fn(&jobs[t]);
        }
        if (T > 1) for (int t = 0; t < T; t++) pthread_join(th[t], NULL);
    }
    int64_t d = 0;
    for (int64_t v = 0; v < g.n; v++) d += (int64_t)deg_out[v] > theta;
    *d_out = d;
    for (int i = 0; i < 4; i++) {
        kind_totals[i] = 0;
        for (int t = 0; t < T; t++) kind_totals[i] += jobs[t].kinds[i];
    }
    return ORC_OK;
}

/* hash_randomize_vertices on an arbitrary id array (rmat.py:153-182). */
int orc_hash_vertices(int64_t n, uint64_t seed, const int64_t *in, int64_t *out,
                      int64_t count) {
    if (n <= 0 || (n & (n - 1))) return ORC_EINVAL;
    int k = 0;
    while (((int64_t)1 << k) < n) k++;
    rmat_gen g;
    rmat_gen_init(&g, k, 1, 0.25, 0.25, 0.25, seed, 1);
    for (int64_t i = 0; i < count; i++) out[i] = (int64_t)hash_perm(&g, (uint64_t)in[i]);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Partition: partition.py:103-177, 295-340                           */
/* ------------------------------------------------------------------ */

typedef struct {
    int64_t rows, nnz;
    int64_t *off;  /* rows + 1, relative to cols */
    void *cols;    /* int64 for nn, uint32 otherwise (storage.py:19-31) */
} orc_csr;

typedef struct {
    int64_t n_local;
    orc_csr csr[4];
    int64_t n_nd_src;
    int64_t *nd_src;  /* partition.py:330 */
    uint8_t *dn_mask; /* partition.py:331 */
    uint8_t *dd_mask; /* partition.py:332 */
} orc_worker;

typedef struct orc_graph {
    int64_t n, m, theta, d;
    int p_rank, p_gpu, p;
    int64_t *degree;   /* partition.py:103-104 */
    int64_t *del_gid;  /* partition.py:111 */
    int64_t *del_id;   /* partition.py:96-100 (-1 for normals) */
    int64_t kind_total[4];
    orc_worker *w;
} orc_graph;

static int64_t n_local_of(int64_t n, int p, int w) { /* partition.py:314 */
    return w < n ? (n - w + p - 1) / p : 0;
}

void orc_graph_free(orc_graph *g) {
    if (!g) return;
    if (g->w) {
        for (int w = 0; w < g->p; w++) {
            for (int k = 0; k < 4; k++) {
                free(g->w[w].csr[k].off);
                free(g->w[w].csr[k].cols);
            }
            free(g->w[w].nd_src);
            free(g->w[w].dn_mask);
            free(g->w[w].dd_mask);
        }
        free(g->w);
    }
    free(g->degree);
    free(g->del_gid);
    free(g->del_id);
    free(g);
}

/* partition_graph(g, theta, ClusterShape(p_rank, p_gpu)) (partition.py:343-351). */
int orc_partition(const int64_t *src, const int64_t *dst, int64_t m, int64_t n,
                  int64_t theta, int p_rank, int p_gpu, orc_graph **out) {
    *out = NULL;
    if (theta < 0 || p_rank < 1 || p_gpu < 1 || n < 0 || m < 0) return ORC_EINVAL;
    for (int64_t i = 0; i < m; i++)
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return ORC_ERANGE;
    orc_graph *g = calloc(1, sizeof(orc_graph));
    if (!g) return ORC_ENOMEM;
    g->n = n; g->m = m; g->theta = theta;
    g->p_rank = p_rank; g->p_gpu = p_gpu; g->p = p_rank * p_gpu;
    int p = g->p;
    g->degree = calloc(n > 0 ? n : 1, sizeof(int64_t));
    g->del_id = malloc((n > 0 ? n : 1) * sizeof(int64_t));
    if (!g->degree || !g->del_id) { orc_graph_free(g); return ORC_ENOMEM; }
    for (int64_t i = 0; i < m; i++) g->degree[src[i]]++;
    int64_t d = 0;
    for (int64_t v = 0; v < n; v++) {
        if (g->degree[v] > theta) g->del_id[v] = d++;
        else g->del_id[v] = -1;
    }
    g->d = d;
    /* CapacityError, partition.py:308-309 */
    if ((n + p - 1) / p >= ((int64_t)1 << 32) || d >= ((int64_t)1 << 32)) {
        orc_graph_free(g);
        return ORC_ECAPACITY;
    }
    g->del_gid = malloc((d > 0 ? d : 1) * sizeof(int64_t));
    for (int64_t v = 0; v < n; v++)
        if (g->del_id[v] >= 0) g->del_gid[g->del_id[v]] = v;

    /* Composite key space: per worker nn rows | nd rows | dn rows | dd rows.
     * A stable counting sort over it in edge order reproduces both the
     * stable (worker, kind) grouping (partition.py:132-137) and the stable
     * per-CSR row sort (partition.py:295-301). */
    g->w = calloc(p, sizeof(orc_worker));
    int64_t *base = malloc((size_t)(4 * p + 1) * sizeof(int64_t));
    int64_t acc = 0;
    for (int w = 0; w < p; w++) {
        int64_t nl = n_local_of(n, p, w);
        g->w[w].n_local = nl;
        int64_t rows[4] = {nl, nl, d, d};
        for (int k = 0; k < 4; k++) { base[4 * w + k] = acc; acc += rows[k]; }
    }
    base[4 * p] = acc;
    int64_t nkeys = acc;
    int64_t *cnt = calloc(nkeys + 1, sizeof(int64_t));
    uint32_t *kind_of = malloc((m > 0 ? m : 1) * sizeof(uint32_t)); /* worker*4+kind */
    int64_t *key = malloc((m > 0 ? m : 1) * sizeof(int64_t));
    if (!cnt || !kind_of || !key) { free(cnt); free(kind_of); free(key); free(base); orc_graph_free(g); return ORC_ENOMEM; }
    for (int64_t i = 0; i < m; i++) {
        int64_t u = src[i], v = dst[i];
        int du = g->del_id[u] >= 0, dv = g->del_id[v] >= 0;
        int64_t home_u = u % p, home_v = v % p;
        int64_t worker;
        /* distribute_edges, partition.py:165-174 */
        if (!du) worker = home_u;
        else if (!dv) worker = home_v;
        else {
            int64_t gu = g->degree[u], gv = g->degree[v];
            int to_u = gu < gv || (gu == gv && u <= v);
            worker = to_u ? home_u : home_v;
        }
        int kind = (du << 1) | dv; /* partition.py:175 */
        int64_t row = (kind == NN || kind == ND) ? u / p : g->del_id[u]; /* partition.py:319 */
        kind_of[i] = (uint32_t)(worker * 4 + kind);
        key[i] = base[worker * 4 + kind] + row;
        cnt[key[i] + 1]++;
        g->kind_total[kind]++;
    }
    for (int64_t k = 0; k < nkeys; k++) cnt[k + 1] += cnt[k];
    /* per-(worker,kind) edge counts */
    int64_t *bucket_nnz = calloc(4 * p, sizeof(int64_t));
    for (int64_t i = 0; i < m; i++) bucket_nnz[kind_of[i]]++;
    for (int w = 0; w < p; w++) {
        for (int k = 0; k < 4; k++) {
            orc_csr *c = &g->w[w].csr[k];
            int64_t rows = (k == NN || k == ND) ? g->w[w].n_local : d;
            c->rows = rows;
            c->nnz = bucket_nnz[4 * w + k];
            c->off = malloc((rows + 1) * sizeof(int64_t));
            int64_t b = base[4 * w + k];
            int64_t first = cnt[b];
            for (int64_t r = 0; r <= rows; r++) c->off[r] = cnt[b + r] - first;
            c->cols = malloc((c->nnz > 0 ? c->nnz : 1) * (k == NN ? 8 : 4));
        }
    }
    /* stable scatter in edge order */
    int64_t *cursor = malloc((nkeys > 0 ? nkeys : 1) * sizeof(int64_t));
    memcpy(cursor, cnt, nkeys * sizeof(int64_t));
    for (int64_t i = 0; i < m; i++) {
        int wk = (int)kind_of[i];
        int w = wk >> 2, k = wk & 3;
        int64_t b = base[wk];
        int64_t pos = cursor[key[i]]++ - cnt[b];
        int64_t v = dst[i];
        orc_csr *c = &g->w[w].csr[k];
        if (k == NN) ((int64_t *)c->cols)[pos] = v;                          /* int64 global */
        else if (k == DN) ((uint32_t *)c->cols)[pos] = (uint32_t)(v / p);    /* local */
        else ((uint32_t *)c->cols)[pos] = (uint32_t)g->del_id[v];            /* delegate id */
    }
    free(cursor); free(cnt); free(kind_of); free(key); free(base); free(bucket_nnz);
    for (int w = 0; w < p; w++) {
        orc_worker *W = &g->w[w];
        orc_csr *nd = &W->csr[ND];
        int64_t cntnd = 0;
        for (int64_t r = 0; r < nd->rows; r++) cntnd += nd->off[r + 1] > nd->off[r];
        W->n_nd_src = cntnd;
        W->nd_src = malloc((cntnd > 0 ? cntnd : 1) * sizeof(int64_t));
        cntnd = 0;
        for (int64_t r = 0; r < nd->rows; r++)
            if (nd->off[r + 1] > nd->off[r]) W->nd_src[cntnd++] = r;
        W->dn_mask = malloc(d > 0 ? d : 1);
        W->dd_mask = malloc(d > 0 ? d : 1);
        for (int64_t r = 0; r < d; r++) {
            W->dn_mask[r] = W->csr[DN].off[r + 1] > W->csr[DN].off[r];
            W->dd_mask[r] = W->csr[DD].off[r + 1] > W->csr[DD].off[r];
        }
    }
    *out = g;
    return ORC_OK;
}

/* Build the partition straight from RMAT parameters (same result as
 * partition_graph(build_rmat_graph(params), ...)). */
int orc_partition_rmat_flags(int scale, int64_t edge_factor, double a, double b, double c,
                             uint64_t seed, int gen_flags, int64_t theta, int p_rank, int p_gpu,
                             orc_graph **out);

int orc_partition_rmat(int scale, int64_t edge_factor, double a, double b, double c,
                       uint64_t seed, int64_t theta, int p_rank, int p_gpu,
                       orc_graph **out) {
    return orc_partition_rmat_flags(scale, edge_factor, a, b, c, seed, 1, theta, p_rank, p_gpu, out);
}

/* gen_flags: the `randomize` bits of orc_rmat_edges (1 = reference hash, 3 = + scramble). */
int orc_partition_rmat_flags(int scale, int64_t edge_factor, double a, double b, double c,
                             uint64_t seed, int gen_flags, int64_t theta, int p_rank, int p_gpu,
                             orc_graph **out) {
    *out = NULL;
    if (scale < 0 || scale > 36 || edge_factor < 1) return ORC_EINVAL;
    int64_t n = (int64_t)1 << scale;
    int64_t m = 2 * n * edge_factor;
    int64_t *src = malloc(m * sizeof(int64_t));
    int64_t *dst = malloc(m * sizeof(int64_t));
    if (!src || !dst) { free(src); free(dst); return ORC_ENOMEM; }
    int rc = orc_rmat_edges(scale, edge_factor, a, b, c, seed, gen_flags, 1, 0, m, src, dst);
    if (rc == ORC_OK) rc = orc_partition(src, dst, m, n, theta, p_rank, p_gpu, out);
    free(src);
    free(dst);
    return rc;
}

/* Construct an oracle graph from an externally built partition (e.g. the CSR
 * exported from the device): used to time the CPU restatement on exactly the
 * graph the GPU traverses.  Arrays are copied.  cols are int64 for nn and
 * uint32 otherwise, as in the reference (storage.py:19-31). */
orc_graph *orc_graph_new(int64_t n, int64_t m, int64_t theta, int p_rank, int p_gpu, int64_t d,
                         const int64_t *del_gid) {
    orc_graph *g = calloc(1, sizeof(orc_graph));
    g->n = n; g->m = m; g->theta = theta; g->d = d;
    g->p_rank = p_rank; g->p_gpu = p_gpu; g->p = p_rank * p_gpu;
    g->degree = calloc(n > 0 ? n : 1, sizeof(int64_t));
    g->del_gid = malloc((d > 0 ? d : 1) * sizeof(int64_t));
    g->del_id = malloc((n > 0 ? n : 1) * sizeof(int64_t));
    memcpy(g->del_gid, del_gid, d * sizeof(int64_t));
    for (int64_t v = 0; v < n; v++) g->del_id[v] = -1;
    for (int64_t x = 0; x < d; x++) g->del_id[del_gid[x]] = x;
    g->w = calloc(g->p, sizeof(orc_worker));
    for (int w = 0; w < g->p; w++) g->w[w].n_local = n_local_of(n, g->p, w);
    return g;
}

int orc_graph_set_csr(orc_graph *g, int w, int k, int64_t rows, const int64_t *off, const void *cols) {
    if (w < 0 || w >= g->p || k < 0 || k > 3) return ORC_EINVAL;
    orc_csr *c = &g->w[w].csr[k];
    c->rows = rows;
    c->nnz = off[rows];
    c->off = malloc((rows + 1) * sizeof(int64_t));
    memcpy(c->off, off, (rows + 1) * sizeof(int64_t));
    size_t wdt = k == NN ? 8 : 4;
    c->cols = malloc((c->nnz > 0 ? c->nnz : 1) * wdt);
    memcpy(c->cols, cols, c->nnz * wdt);
    g->kind_total[k] += c->nnz;
    return ORC_OK;
}

int orc_graph_finalize(orc_graph *g) {
    for (int w = 0; w < g->p; w++) {
        orc_worker *W = &g->w[w];
        orc_csr *nd = &W->csr[ND];
        int64_t cnt = 0;
        for (int64_t r = 0; r < nd->rows; r++) cnt += nd->off[r + 1] > nd->off[r];
        W->n_nd_src = cnt;
        W->nd_src = malloc((cnt > 0 ? cnt : 1) * sizeof(int64_t));
        cnt = 0;
        for (int64_t r = 0; r < nd->rows; r++) if (nd->off[r + 1] > nd->off[r]) W->nd_src[cnt++] = r;
        W->dn_mask = malloc(g->d > 0 ? g->d : 1);
        W->dd_mask = malloc(g->d > 0 ? g->d : 1);
        for (int64_t r = 0; r < g->d; r++) {
            W->dn_mask[r] = W->csr[DN].off[r + 1] > W->csr[DN].off[r];
            W->dd_mask[r] = W->csr[DD].off[r + 1] > W->csr[DD].off[r];
        }
    }
    return ORC_OK;
}

int64_t orc_graph_n(const orc_graph *g) { return g->n; }
int64_t orc_graph_m(const orc_graph *g) { return g->m; }
int64_t orc_graph_d(const orc_graph *g) { return g->d; }
int orc_graph_p(const orc_graph *g) { return g->p; }
int64_t orc_graph_kind_total(const orc_graph *g, int k) { return g->kind_total[k]; }
const int64_t *orc_graph_degrees(const orc_graph *g) { return g->degree; }
const int64_t *orc_graph_delegates(const orc_graph *g) { return g->del_gid; }
int64_t orc_graph_n_local(const orc_graph *g, int w) { return g->w[w].n_local; }
int64_t orc_graph_csr_rows(const orc_graph *g, int w, int k) { return g->w[w].csr[k].rows; }
int64_t orc_graph_csr_nnz(const orc_graph *g, int w, int k) { return g->w[w].csr[k].nnz; }
const int64_t *orc_graph_csr_off(const orc_graph *g, int w, int k) { return g->w[w].csr[k].off; }
const void *orc_graph_csr_cols(const orc_graph *g, int w, int k) { return g->w[w].csr[k].cols; }
int64_t orc_graph_n_nd_src(const orc_graph *g, int w) { return g->w[w].n_nd_src; }
const int64_t *orc_graph_nd_src(const orc_graph *g, int w) { return g->w[w].nd_src; }
const uint8_t *orc_graph_dn_mask(const orc_graph *g, int w) { return g->w[w].dn_mask; }
const uint8_t *orc_graph_dd_mask(const orc_graph *g, int w) { return g->w[w].dd_mask; }

/* ------------------------------------------------------------------ */
/* Direction rule: traversal.py:142-163                                */
/* ------------------------------------------------------------------ */

static int bitlen128(unsigned __int128 x) {
    int b = 0;
    while (x) { b++; x >>= 1; }
    return b;
}

/* Correctly rounded N / D for non-negative integers, as Python's int / int. */
double orc_div_rn(unsigned __int128 N, uint64_t D) {
    if (N == 0) return 0.0;
    if (N < ((unsigned __int128)1 << 53) && D < (1ULL << 53)) return (double)(uint64_t)N / (double)D;
    int shift = 56 - bitlen128(N) + bitlen128(D);
    if (shift < 0) shift = 0;
    unsigned __int128 num = N << shift;
    unsigned __int128 Q = num / D;
    int sticky = (num % D) != 0;
    int qb = bitlen128(Q);
    int drop = qb - 53;
    unsigned __int128 mant = Q >> drop;
    unsigned __int128 rem = Q & ((((unsigned __int128)1) << drop) - 1);
    unsigned __int128 half = ((unsigned __int128)1) << (drop - 1);
    if (rem > half || (rem == half && (sticky || (mant & 1)))) mant++;
    if (mant == ((unsigned __int128)1 << 53)) { mant >>= 1; drop++; }
    return ldexp((double)(uint64_t)mant, drop - shift);
}

/* estimate_backward_workload(u, q, s) with exact ints (traversal.py:142-148) */
double orc_bv(int64_t u, int64_t q, int64_t s) {
    if (q == 0) return INFINITY;
    return orc_div_rn((unsigned __int128)(uint64_t)u * (unsigned __int128)(uint64_t)(q + s), (uint64_t)q);
}

/* decide_direction (traversal.py:151-163): int fv compared exactly to a float */
int orc_decide(int dir, int64_t fv, double bv, double f0, double f1, int allow_back) {
    double fvd = (double)fv; /* fv <= m < 2^53: exact */
    if (dir == FWD) {
        if (isfinite(bv) && fvd > f0 * bv) return BWD;
        return FWD;
    }
    if (allow_back && fvd < f1 * bv) return FWD;
    return BWD;
}

/* ------------------------------------------------------------------ */
/* BFS engine: engine.py:98-330                                        */
/* ------------------------------------------------------------------ */

typedef struct { int64_t *a; int64_t n, cap; } vec64;
static void v_push(vec64 *v, int64_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 64;
        v->a = realloc(v->a, v->cap * sizeof(int64_t));
    }
    v->a[v->n++] = x;
}
static void v_clear(vec64 *v) { v->n = 0; }
static void v_free(vec64 *v) { free(v->a); v->a = NULL; v->n = v->cap = 0; }

typedef struct {
    int mode; /* 0 bfs, 1 dobfs */
    int64_t source;
    double f0[4], f1[4]; /* indexed by kind code; nn unused */
    int allow_switch_back, local_all2all, uniquify;
} orc_bfs_opts;

typedef struct orc_run {
    int64_t n;
    int p;
    int32_t *levels;
    int64_t iterations;
    int64_t insp[4][2];
    int64_t cap;
    /* per iteration */
    int8_t *dirs;      /* [it][p][4] */
    int64_t *it_insp;  /* [it][4] */
    int64_t *it_fv;    /* [it][4] */
    double *it_bv;     /* [it][p][4] (nn slot unused) */
    double *mask_bytes;
    int64_t *normal_bytes, *messages, *pairs;
    double b_measured;
} orc_run;

void orc_run_free(orc_run *r) {
    if (!r) return;
    free(r->levels); free(r->dirs); free(r->it_insp); free(r->it_fv); free(r->it_bv);
    free(r->mask_bytes); free(r->normal_bytes); free(r->messages); free(r->pairs);
    free(r);
}

static void run_grow(orc_run *r) {
    int64_t cap = r->cap ? 2 * r->cap : 16;
    int p = r->p;
    r->dirs = realloc(r->dirs, cap * p * 4);
    r->it_insp = realloc(r->it_insp, cap * 4 * sizeof(int64_t));
    r->it_fv = realloc(r->it_fv, cap * 4 * sizeof(int64_t));
    r->it_bv = realloc(r->it_bv, cap * p * 4 * sizeof(double));
    r->mask_bytes = realloc(r->mask_bytes, cap * sizeof(double));
    r->normal_bytes = realloc(r->normal_bytes, cap * sizeof(int64_t));
    r->messages = realloc(r->messages, cap * sizeof(int64_t));
    r->pairs = realloc(r->pairs, cap * sizeof(int64_t));
    r->cap = cap;
}

static inline int64_t csr_deg(const orc_csr *c, int64_t r) { return c->off[r + 1] - c->off[r]; }
static inline int64_t csr_col(const orc_csr *c, int k, int64_t i) {
    return k == NN ? ((const int64_t *)c->cols)[i] : (int64_t)((const uint32_t *)c->cols)[i];
}

/* visit_backward (traversal.py:111-139): returns inspections, appends found. */
static int64_t visit_backward(const orc_csr *rev, int kind, const int64_t *srcs, int64_t ns,
                              const int32_t *parent_levels, int32_t level, vec64 *found) {
    int64_t insp = 0;
    for (int64_t i = 0; i < ns; i++) {
        int64_t s = srcs[i];
        int64_t b = rev->off[s], e = rev->off[s + 1];
        if (e == b) continue;
        int64_t j;
        for (j = b; j < e; j++)
            if (parent_levels[csr_col(rev, kind, j)] == level) break;
        if (j < e) { insp += j - b + 1; v_push(found, s); }
        else insp += e - b;
    }
    return insp;
}

int orc_run_bfs(const orc_graph *g, const orc_bfs_opts *o, orc_run **out) {
    *out = NULL;
    const int p = g->p;
    const int64_t n = g->n, d = g->d;
    if (!(0 <= o->source && o->source < n)) return ORC_ERANGE; /* engine.py:105-106 */
    orc_run *R = calloc(1, sizeof(orc_run));
    R->n = n; R->p = p;

    int32_t **nlev = malloc(p * sizeof(int32_t *));
    int32_t **nstamp = malloc(p * sizeof(int32_t *));
    for (int w = 0; w < p; w++) {
        int64_t nl = g->w[w].n_local;
        nlev[w] = malloc((nl > 0 ? nl : 1) * sizeof(int32_t));
        nstamp[w] = calloc(nl > 0 ? nl : 1, sizeof(int32_t));
        for (int64_t i = 0; i < nl; i++) nlev[w][i] = -1;
    }
    int32_t *dlev = malloc((d > 0 ? d : 1) * sizeof(int32_t));
    int32_t *dstamp = calloc(d > 0 ? d : 1, sizeof(int32_t));
    for (int64_t i = 0; i < d; i++) dlev[i] = -1;
    int32_t stamp = 0;
    int *dirs = malloc(p * 4 * sizeof(int));
    for (int i = 0; i < p * 4; i++) dirs[i] = FWD;

    vec64 *new_normals = calloc(p, sizeof(vec64));
    vec64 new_delegates = {0};
    vec64 *inbox = calloc(p, sizeof(vec64)); /* gids; level = current level */
    vec64 *cand = calloc(p, sizeof(vec64));
    vec64 *qn_nn = calloc(p, sizeof(vec64)), *qn_nd = calloc(p, sizeof(vec64));
    vec64 *qd_dn = calloc(p, sizeof(vec64)), *qd_dd = calloc(p, sizeof(vec64));
    vec64 *local_new = calloc(p, sizeof(vec64));
    vec64 *outbox = calloc((size_t)p * p, sizeof(vec64)); /* [sender][dest] */
    vec64 found = {0}, srcs = {0};
    uint8_t **mask = malloc(p * sizeof(uint8_t *));
    int *dirty = calloc(p, sizeof(int));
    for (int w = 0; w < p; w++) mask[w] = calloc(d > 0 ? d : 1, 1);
    int64_t *fv = malloc(p * 4 * sizeof(int64_t));
    int64_t *U = malloc(p * 4 * sizeof(int64_t)), *Q = malloc(p * 4 * sizeof(int64_t)), *S = malloc(p * 4 * sizeof(int64_t));
    int32_t *seen_n = NULL; /* uniquify scratch over global ids */

    /* seeding, engine.py:131-139 */
    int64_t sd = g->del_id[o->source];
    if (sd >= 0) { dlev[sd] = 0; v_push(&new_delegates, sd); }
    else {
        int owner = (int)(o->source % p);
        int64_t local = o->source / p;
        nlev[owner][local] = 0;
        v_push(&new_normals[owner], local);
    }

    int32_t level = 0;
    for (;;) {
        /* -- ingest inboxes, engine.py:147-157 */
        for (int w = 0; w < p; w++) {
            v_clear(&cand[w]);
            for (int64_t i = 0; i < new_normals[w].n; i++) v_push(&cand[w], new_normals[w].a[i]);
            for (int64_t i = 0; i < inbox[w].n; i++) {
                int64_t loc = inbox[w].a[i] / p;
                v_push(&cand[w], loc);
                if (nlev[w][loc] < 0) nlev[w][loc] = level;
            }
        }
        /* -- previsit + estimates + directions, engine.py:161-197 */
        for (int w = 0; w < p; w++) {
            const orc_worker *W = &g->w[w];
            v_clear(&qn_nn[w]); v_clear(&qn_nd[w]); v_clear(&qd_dn[w]); v_clear(&qd_dd[w]);
            int64_t fnn = 0, fnd = 0, fdn = 0, fdd = 0;
            /* previsit (traversal.py:58-73): unique, keep lv<0 or lv==L */
            stamp++;
            for (int64_t i = 0; i < cand[w].n; i++) {
                int64_t v = cand[w].a[i];
                if (nstamp[w][v] == stamp) continue;
                nstamp[w][v] = stamp;
                if (!(nlev[w][v] < 0 || nlev[w][v] == level)) continue;
                nlev[w][v] = level;
                int64_t a = csr_deg(&W->csr[NN], v), b = csr_deg(&W->csr[ND], v);
                if (a > 0) { v_push(&qn_nn[w], v); fnn += a; }
                if (b > 0) { v_push(&qn_nd[w], v); fnd += b; }
            }
            stamp++;
            for (int64_t i = 0; i < new_delegates.n; i++) {
                int64_t x = new_delegates.a[i];
                if (dstamp[x] == stamp) continue;
                dstamp[x] = stamp;
                if (!(dlev[x] < 0 || dlev[x] == level)) continue;
                dlev[x] = level;
                int64_t a = csr_deg(&W->csr[DN], x), b = csr_deg(&W->csr[DD], x);
                if (a > 0) { v_push(&qd_dn[w], x); fdn += a; }
                if (b > 0) { v_push(&qd_dd[w], x); fdd += b; }
            }
            int64_t u_nd = 0, u_dn = 0, u_dd = 0;
            for (int64_t i = 0; i < W->n_nd_src; i++) u_nd += nlev[w][W->nd_src[i]] < 0;
            for (int64_t x = 0; x < d; x++) {
                if (dlev[x] < 0) { u_dn += W->dn_mask[x]; u_dd += W->dd_mask[x]; }
            }
            int64_t *F = fv + 4 * w;
            F[NN] = fnn; F[ND] = fnd; F[DN] = fdn; F[DD] = fdd;
            /* engine.py:181-189 */
            U[4 * w + ND] = u_dn; Q[4 * w + ND] = qn_nd[w].n; S[4 * w + ND] = u_nd;
            U[4 * w + DN] = u_nd; Q[4 * w + DN] = qd_dn[w].n; S[4 * w + DN] = u_dn;
            U[4 * w + DD] = u_dd; Q[4 * w + DD] = qd_dd[w].n; S[4 * w + DD] = u_dd;
            if (o->mode == 1) {
                for (int k = ND; k <= DD; k++) {
                    double bv = orc_bv(U[4 * w + k], Q[4 * w + k], S[4 * w + k]);
                    dirs[4 * w + k] = orc_decide(dirs[4 * w + k], F[k], bv, o->f0[k], o->f1[k],
                                                 o->allow_switch_back);
                }
            }
        }
        /* -- visits, engine.py:199-263 */
        int64_t it_insp[4] = {0, 0, 0, 0};
        for (int w = 0; w < p; w++) {
            memset(mask[w], 0, d > 0 ? d : 1);
            dirty[w] = 0;
            v_clear(&local_new[w]);
            for (int q = 0; q < p; q++) v_clear(&outbox[w * p + q]);
        }
        for (int w = 0; w < p; w++) {
            const orc_worker *W = &g->w[w];
            const int *D = dirs + 4 * w;
            /* nn: forward, dedupe=False (engine.py:207-222) */
            {
                const orc_csr *c = &W->csr[NN];
                int64_t insp = 0;
                for (int64_t i = 0; i < qn_nn[w].n; i++) {
                    int64_t u = qn_nn[w].a[i];
                    for (int64_t j = c->off[u]; j < c->off[u + 1]; j++) {
                        int64_t v = ((const int64_t *)c->cols)[j];
                        insp++;
                        int owner = (int)(v % p);
                        if (owner == w) v_push(&local_new[w], v / p);
                        else v_push(&outbox[w * p + owner], v);
                    }
                }
                it_insp[NN] += insp; R->insp[NN][FWD] += insp;
            }
            /* nd (engine.py:225-235) */
            if (D[ND] == FWD || o->mode == 0) {
                const orc_csr *c = &W->csr[ND];
                int64_t insp = 0;
                for (int64_t i = 0; i < qn_nd[w].n; i++) {
                    int64_t u = qn_nd[w].a[i];
                    for (int64_t j = c->off[u]; j < c->off[u + 1]; j++) {
                        uint32_t x = ((const uint32_t *)c->cols)[j];
                        insp++;
                        if (dlev[x] < 0) { mask[w][x] = 1; dirty[w] = 1; }
                    }
                }
                it_insp[ND] += insp; R->insp[ND][FWD] += insp;
            } else {
                v_clear(&srcs); v_clear(&found);
                for (int64_t x = 0; x < d; x++) if (W->dn_mask[x] && dlev[x] < 0) v_push(&srcs, x);
                int64_t insp = visit_backward(&W->csr[DN], DN, srcs.a, srcs.n, nlev[w], level, &found);
                for (int64_t i = 0; i < found.n; i++) { mask[w][found.a[i]] = 1; dirty[w] = 1; }
                it_insp[ND] += insp; R->insp[ND][BWD] += insp;
            }
            /* dn (engine.py:238-250) */
            if (D[DN] == FWD || o->mode == 0) {
                const orc_csr *c = &W->csr[DN];
                int64_t insp = 0;
                for (int64_t i = 0; i < qd_dn[w].n; i++) {
                    int64_t x = qd_dn[w].a[i];
                    for (int64_t j = c->off[x]; j < c->off[x + 1]; j++) {
                        uint32_t v = ((const uint32_t *)c->cols)[j];
                        insp++;
                        if (nlev[w][v] < 0) v_push(&local_new[w], v);
                    }
                }
                it_insp[DN] += insp; R->insp[DN][FWD] += insp;
            } else {
                v_clear(&srcs); v_clear(&found);
                for (int64_t i = 0; i < W->n_nd_src; i++)
                    if (nlev[w][W->nd_src[i]] < 0) v_push(&srcs, W->nd_src[i]);
                int64_t insp = visit_backward(&W->csr[ND], ND, srcs.a, srcs.n, dlev, level, &found);
                for (int64_t i = 0; i < found.n; i++) v_push(&local_new[w], found.a[i]);
                it_insp[DN] += insp; R->insp[DN][BWD] += insp;
            }
            /* dd (engine.py:253-263) */
            if (D[DD] == FWD || o->mode == 0) {
                const orc_csr *c = &W->csr[DD];
                int64_t insp = 0;
                for (int64_t i = 0; i < qd_dd[w].n; i++) {
                    int64_t x = qd_dd[w].a[i];
                    for (int64_t j = c->off[x]; j < c->off[x + 1]; j++) {
                        uint32_t y = ((const uint32_t *)c->cols)[j];
                        insp++;
                        if (dlev[y] < 0) { mask[w][y] = 1; dirty[w] = 1; }
                    }
                }
                it_insp[DD] += insp; R->insp[DD][FWD] += insp;
            } else {
                v_clear(&srcs); v_clear(&found);
                for (int64_t x = 0; x < d; x++) if (W->dd_mask[x] && dlev[x] < 0) v_push(&srcs, x);
                int64_t insp = visit_backward(&W->csr[DD], DD, srcs.a, srcs.n, dlev, level, &found);
                for (int64_t i = 0; i < found.n; i++) { mask[w][found.a[i]] = 1; dirty[w] = 1; }
                it_insp[DD] += insp; R->insp[DD][BWD] += insp;
            }
        }
        /* -- barrier: mask reduction (comm.py:75-98), engine.py:266-268 */
        int any_dirty = 0;
        for (int w = 0; w < p; w++) any_dirty |= dirty[w];
        double mask_bytes = any_dirty ? 2.0 * (double)d * (double)g->p_rank / 8.0 : 0.0;
        v_clear(&new_delegates);
        if (any_dirty) {
            for (int64_t x = 0; x < d; x++) {
                int r = 0;
                for (int w = 0; w < p; w++) r |= mask[w][x];
                if (r && dlev[x] < 0) { v_push(&new_delegates, x); }
            }
            for (int64_t i = 0; i < new_delegates.n; i++) dlev[new_delegates.a[i]] = level + 1;
        }
        /* -- exchange (comm.py:138-197), engine.py:270-277 */
        int64_t nbytes = 0, msgs = 0;
        for (int w = 0; w < p; w++) v_clear(&inbox[w]);
        if (o->uniquify && !seen_n) seen_n = calloc(n > 0 ? n : 1, sizeof(int32_t));
        /* staged groups: key (final_sender, dest) visited in sorted order */
        for (int fs = 0; fs < p; fs++) {
            for (int dest = 0; dest < p; dest++) {
                int64_t count = 0;
                int any = 0;
                if (o->uniquify) stamp++;
                for (int s = 0; s < p; s++) {
                    int final_sender = s;
                    if (o->local_all2all) {
                        int r = s % g->p_rank;
                        int g2 = dest / g->p_rank;
                        final_sender = r + g->p_rank * g2;
                    }
                    if (final_sender != fs) continue;
                    vec64 *ob = &outbox[s * p + dest];
                    if (ob->n == 0) continue;
                    any = 1;
                    for (int64_t i = 0; i < ob->n; i++) {
                        int64_t gid = ob->a[i];
                        if (o->uniquify) {
                            if (seen_n[gid] == stamp) continue;
                            seen_n[gid] = stamp;
                        }
                        v_push(&inbox[dest], gid);
                        count++;
                    }
                }
                if (any) { nbytes += 4 * count; msgs += 1; }
            }
        }
        int64_t pair_cap = o->local_all2all ? (int64_t)p * p / g->p_gpu : (int64_t)p * p;
        /* -- apply local updates, engine.py:280-289 */
        int any_local = 0;
        for (int w = 0; w < p; w++) {
            v_clear(&new_normals[w]);
            stamp++;
            for (int64_t i = 0; i < local_new[w].n; i++) {
                int64_t v = local_new[w].a[i];
                if (nstamp[w][v] == stamp) continue;
                nstamp[w][v] = stamp;
                if (nlev[w][v] < 0) { nlev[w][v] = level + 1; v_push(&new_normals[w], v); }
            }
            if (new_normals[w].n) any_local = 1;
        }
        /* -- per-iteration record, engine.py:291-302 */
        if (R->iterations == R->cap) run_grow(R);
        int64_t it = R->iterations;
        for (int w = 0; w < p; w++) {
            for (int k = 0; k < 4; k++) {
                int dk = (k == NN || o->mode == 0) ? FWD : dirs[4 * w + k];
                R->dirs[(it * p + w) * 4 + k] = (int8_t)dk;
                R->it_bv[(it * p + w) * 4 + k] =
                    k == NN ? INFINITY : orc_bv(U[4 * w + k], Q[4 * w + k], S[4 * w + k]);
            }
        }
        for (int k = 0; k < 4; k++) {
            R->it_insp[it * 4 + k] = it_insp[k];
            int64_t s = 0;
            for (int w = 0; w < p; w++) s += fv[4 * w + k];
            R->it_fv[it * 4 + k] = s;
        }
        R->mask_bytes[it] = mask_bytes;
        R->normal_bytes[it] = nbytes;
        R->messages[it] = msgs;
        R->pairs[it] = pair_cap;
        R->iterations++;
        level++;
        int inbox_pending = 0;
        for (int w = 0; w < p; w++) inbox_pending |= inbox[w].n > 0;
        if (!any_local && new_delegates.n == 0 && !inbox_pending) break;
    }
    /* -- assemble, engine.py:308-314 */
    R->levels = malloc((n > 0 ? n : 1) * sizeof(int32_t));
    for (int64_t v = 0; v < n; v++) R->levels[v] = -1;
    for (int w = 0; w < p; w++)
        for (int64_t i = 0; i < g->w[w].n_local; i++) R->levels[i * p + w] = nlev[w][i];
    for (int64_t x = 0; x < d; x++) R->levels[g->del_gid[x]] = dlev[x];
    int64_t bwd_del = R->insp[ND][BWD] + R->insp[DD][BWD];
    R->b_measured = d ? (double)bwd_del / (double)(d * p) : 0.0;

    for (int w = 0; w < p; w++) {
        free(nlev[w]); free(nstamp[w]); free(mask[w]);
        v_free(&new_normals[w]); v_free(&inbox[w]); v_free(&cand[w]);
        v_free(&qn_nn[w]); v_free(&qn_nd[w]); v_free(&qd_dn[w]); v_free(&qd_dd[w]);
        v_free(&local_new[w]);
        for (int q = 0; q < p; q++) v_free(&outbox[w * p + q]);
    }
    free(nlev); free(nstamp); free(mask); free(dirty); free(dlev); free(dstamp); free(dirs);
    free(new_normals); free(inbox); free(cand); free(qn_nn); free(qn_nd); free(qd_dn); free(qd_dd);
    free(local_new); free(outbox); free(fv); free(U); free(Q); free(S); free(seen_n);
    v_free(&new_delegates); v_free(&found); v_free(&srcs);
    *out = R;
    return ORC_OK;
}

const int32_t *orc_run_levels(const orc_run *r) { return r->levels; }
int64_t orc_run_iterations(const orc_run *r) { return r->iterations; }
int64_t orc_run_insp(const orc_run *r, int k, int dir) { return r->insp[k][dir]; }
double orc_run_b_measured(const orc_run *r) { return r->b_measured; }
const int8_t *orc_run_dirs(const orc_run *r) { return r->dirs; }
const int64_t *orc_run_it_insp(const orc_run *r) { return r->it_insp; }
const int64_t *orc_run_it_fv(const orc_run *r) { return r->it_fv; }
const double *orc_run_it_bv(const orc_run *r) { return r->it_bv; }
const double *orc_run_mask_bytes(const orc_run *r) { return r->mask_bytes; }
const int64_t *orc_run_normal_bytes(const orc_run *r) { return r->normal_bytes; }
const int64_t *orc_run_messages(const orc_run *r) { return r->messages; }
const int64_t *orc_run_pairs(const orc_run *r) { return r->pairs; }

/* ------------------------------------------------------------------ */
/* Plain BFS over an edge list: oracle.py:36-53 (any n)               */
/* ------------------------------------------------------------------ */

int orc_bfs_levels_edges(const int64_t *src, const int64_t *dst, int64_t m, int64_t n,
                         int64_t source, int32_t *levels) {
    if (!(0 <= source && source < n)) return ORC_ERANGE;
    int64_t *off = calloc(n + 1, sizeof(int64_t));
    int64_t *adj = malloc((m > 0 ? m : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < m; i++) off[src[i] + 1]++;
    for (int64_t v = 0; v < n; v++) off[v + 1] += off[v];
    int64_t *cur = malloc((n > 0 ? n : 1) * sizeof(int64_t));
    memcpy(cur, off, n * sizeof(int64_t));
    for (int64_t i = 0; i < m; i++) adj[cur[src[i]]++] = dst[i];
    for (int64_t v = 0; v < n; v++) levels[v] = -1;
    int64_t *q = malloc((n > 0 ? n : 1) * sizeof(int64_t));
    int64_t head = 0, tail = 0;
    levels[source] = 0;
    q[tail++] = source;
    while (head < tail) {
        int64_t u = q[head++];
        for (int64_t j = off[u]; j < off[u + 1]; j++) {
            int64_t v = adj[j];
            if (levels[v] < 0) { levels[v] = levels[u] + 1; q[tail++] = v; }
        }
    }
    free(off); free(adj); free(cur); free(q);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* NEW (no reference): min-ID parents             */
/*   parent[root] = root; parent[v] = min{u : (u->v) in E,             */
/*   level[u] = level[v]-1}; -1 if unreached.                          */
/* ------------------------------------------------------------------ */

int orc_min_parents(const int64_t *src, const int64_t *dst, int64_t m, int64_t n,
                    int64_t root, const int32_t *levels, int64_t *parents) {
    for (int64_t v = 0; v < n; v++) parents[v] = levels[v] >= 0 ? INT64_MAX : -1;
    for (int64_t i = 0; i < m; i++) {
        int64_t u = src[i], v = dst[i];
        if (levels[u] >= 0 && levels[v] == levels[u] + 1 && u < parents[v]) parents[v] = u;
    }
    parents[root] = root;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* NEW: Graph500-style certificate, SURVEY.md §8(a) A20.               */
/* Returns a bitmask of failed checks (0 = valid):                     */
/*  1 root level/parent, 2 edge spans > 1 level, 4 edge joins reached  */
/*  and unreached, 8 level[parent[v]] != level[v]-1, 16 tree edge not  */
/*  in E, 32 unreached vertex has a parent / reached one has none.     */
/* ------------------------------------------------------------------ */

int orc_validate(const int64_t *src, const int64_t *dst, int64_t m, int64_t n, int64_t root,
                 const int32_t *levels, const int64_t *parents) {
    int bad = 0;
    if (root < 0 || root >= n) return 1;
    if (levels[root] != 0 || parents[root] != root) bad |= 1;
    uint8_t *ok = calloc(n > 0 ? n : 1, 1);
    for (int64_t i = 0; i < m; i++) {
        int64_t u = src[i], v = dst[i];
        int32_t lu = levels[u], lv = levels[v];
        if ((lu >= 0) != (lv >= 0)) bad |= 4;
        else if (lu >= 0 && (lu - lv > 1 || lv - lu > 1)) bad |= 2;
        if (lv >= 0 && parents[v] == u) ok[v] = 1;
    }
    for (int64_t v = 0; v < n; v++) {
        if (levels[v] < 0) { if (parents[v] != -1) bad |= 32; continue; }
        if (v == root) continue;
        int64_t pv = parents[v];
        if (pv < 0 || pv >= n) { bad |= 32; continue; }
        if (levels[pv] != levels[v] - 1) bad |= 8;
        if (!ok[v]) bad |= 16;
    }
    free(ok);
    return bad;
}
