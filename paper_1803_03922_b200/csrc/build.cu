// build.cu -- device-side graph construction.
//
//   k_rmat_*      generate_rmat + hash_randomize_vertices + symmetrize
//                 (rmat.py:107-208), counter-based and regenerated per pass so
//                 the edge list is never materialised for RMAT inputs.
//   k_degree      compute_out_degrees (partition.py:103-104)
//   k_classify    classify_vertices / delegate_id_map (partition.py:96-117)
//   k_route       distribute_edges (Alg. 1, partition.py:156-177) and the CSR
//                 row/column renumbering of build_partitioned_graph
//                 (partition.py:304-340) into one composite key per edge
//   radix sort    stable by composite key == stable (worker,kind) grouping then
//                 stable row sort (partition.py:132-137, 295-301)
//   k_src_bits    nd_source_list / dn_source_mask / dd_source_mask
//                 (partition.py:330-332) as bitmaps
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace dbfs {

// ------------------------------------------------------------ RMAT generator

struct RmatGen {
    int scale;
    int randomize;
    int scramble;     // Feistel relabeling after the reference hash (this build's option)
    int64_t m0;       // undoubled edges
    uint64_t key, ta, tab, tabc, mask, c1, m1, m2, skey;
    int s1, s2;
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rmat.py:107-115
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

// r = (base>>11)*2^-53 is k*2^-53 exactly, so r >= t <=> k >= ceil(t*2^53).
static uint64_t threshold53(double t) {
    double x = t * 9007199254740992.0;
    if (x <= 0.0) return 0;
    if (x >= 9007199254740992.0) return 1ULL << 53;
    uint64_t k = (uint64_t)x;
    if ((double)k < x) k++;
    return k;
}

static RmatGen make_gen(const dbfs_rmat_params &p) {
    RmatGen g;
    g.scale = p.scale;
    g.randomize = p.randomize;
    int64_t n = (int64_t)1 << p.scale;
    g.m0 = n * p.edge_factor;
    g.key = mix64(p.seed);
    double ab = p.a + p.b, abc = ab + p.c;  // rmat.py:130-131
    g.ta = threshold53(p.a);
    g.tab = threshold53(ab);
    g.tabc = threshold53(abc);
    g.mask = (uint64_t)n - 1;  // rmat.py:164-171
    int k = p.scale;
    g.s1 = std::max(1, k / 3);
    g.s2 = std::max(1, k / 2);
    g.c1 = mix64(p.seed) & g.mask;
    g.m1 = (0x9E3779B97F4A7C15ULL & 0x7FFFFFFFFFFFFFFFULL) | 1ULL;
    g.m2 = (0xBF58476D1CE4E5B9ULL & 0x7FFFFFFFFFFFFFFFULL) | 1ULL;
    g.scramble = p.scramble;
    g.skey = mix64(p.seed ^ 0x5CA3B1E5D00DF00DULL);
    return g;
}

// 3-round Feistel bijection on the scale bits (oracle/dbfs_oracle.c scramble()):
// the reference hash keeps low id bits a function of low bits only, so owners
// v mod p inherit RMAT's bit-pattern degree skew; this mixes all bits.
__host__ __device__ __forceinline__ uint64_t scramble(const RmatGen &g, uint64_t v) {
    const int k = g.scale;
    if (k < 2) return v;
    const int j = k / 2;
    const uint64_t lm = (1ULL << j) - 1, hm = (1ULL << (k - j)) - 1;
    uint64_t lo = v & lm, hi = v >> j;
    lo ^= mix64(hi ^ g.skey) & lm;
    hi ^= mix64(lo ^ (g.skey + 1)) & hm;
    lo ^= mix64(hi ^ (g.skey + 2)) & lm;
    return (hi << j) | lo;
}

__device__ __forceinline__ uint64_t hash_perm(const RmatGen &g, uint64_t v) {  // rmat.py:173-180
    v = (v * g.m1) & g.mask;
    v ^= (v << g.s1) & g.mask;
    v = (v + g.c1) & g.mask;
    v = (v * g.m2) & g.mask;
    v ^= (v << g.s2) & g.mask;
    return v;
}

// Original edge e: quadrant bits MSB first (rmat.py:139-148), then the hash.
__device__ __forceinline__ void rmat_edge(const RmatGen &g, uint64_t e, uint32_t &u, uint32_t &v) {
    uint32_t su = 0, sv = 0;
    uint64_t cnt = e * (uint64_t)g.scale;
    for (int l = 0; l < g.scale; l++) {
        uint64_t k = mix64(g.key ^ (cnt + (uint64_t)l)) >> 11;
        uint32_t ub = k >= g.tab;
        uint32_t vb = (k >= g.ta && k < g.tab) || k >= g.tabc;
        su = (su << 1) | ub;
        sv = (sv << 1) | vb;
    }
    if (g.randomize) {
        su = (uint32_t)hash_perm(g, su);
        sv = (uint32_t)hash_perm(g, sv);
    }
    if (g.scramble) {
        su = (uint32_t)scramble(g, su);
        sv = (uint32_t)scramble(g, sv);
    }
    u = su;
    v = sv;
}

// Edge source: either the counter-based RMAT generator (doubled index space
// when symmetrize: e >= m0 is the reverse of e - m0, rmat.py:185-189) or an
// explicit device edge list.
struct EdgeSrc {
    RmatGen gen;
    int symmetrize;
    const int64_t *src, *dst;  // explicit mode when non-null
    __device__ __forceinline__ void get(int64_t e, uint32_t &u, uint32_t &v) const {
        if (src) {
            u = (uint32_t)src[e];
            v = (uint32_t)dst[e];
            return;
        }
        if (symmetrize && e >= gen.m0) {
            rmat_edge(gen, (uint64_t)(e - gen.m0), v, u);
        } else {
            rmat_edge(gen, (uint64_t)e, u, v);
        }
    }
};

__global__ void k_rmat_to_host_layout(EdgeSrc es, int64_t begin, int64_t count, int64_t *src, int64_t *dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t u, v;
        es.get(begin + i, u, v);
        src[i] = u;
        dst[i] = v;
    }
}

void rmat_generate_host(Ctx &ctx, const dbfs_rmat_params &prm, int64_t begin, int64_t end, int64_t *src,
                        int64_t *dst) {
    DBFS_CHECK(prm.scale >= 0 && prm.scale <= 32 && prm.edge_factor >= 1, DBFS_EINVAL, "bad RMAT params");
    EdgeSrc es{};
    es.gen = make_gen(prm);
    es.symmetrize = prm.symmetrize;
    int64_t m = es.gen.m0 * (prm.symmetrize ? 2 : 1);
    DBFS_CHECK(0 <= begin && begin <= end && end <= m, DBFS_ERANGE, "edge range out of bounds");
    const int64_t CH = 1 << 26;
    DArray<int64_t> ds, dd;
    ds.alloc(std::min<int64_t>(CH, std::max<int64_t>(end - begin, 1)));
    dd.alloc(std::min<int64_t>(CH, std::max<int64_t>(end - begin, 1)));
    for (int64_t b = begin; b < end; b += CH) {
        int64_t c = std::min(CH, end - b);
        k_rmat_to_host_layout<<<ctx.num_sms * 8, 256, 0, ctx.stream>>>(es, b, c, ds.p, dd.p);
        DBFS_LAUNCHED();
        DBFS_CUDA(cudaMemcpyAsync(src + (b - begin), ds.p, c * 8, cudaMemcpyDeviceToHost, ctx.stream));
        DBFS_CUDA(cudaMemcpyAsync(dst + (b - begin), dd.p, c * 8, cudaMemcpyDeviceToHost, ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
}

__global__ void k_hash_ids(RmatGen g, const int64_t *__restrict__ in, int64_t *__restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)hash_perm(g, (uint64_t)in[i]);
}

void hash_vertices_host(Ctx &ctx, int64_t n, uint64_t seed, const int64_t *in, int64_t *out, int64_t count) {
    DBFS_CHECK(n > 0 && (n & (n - 1)) == 0, DBFS_EINVAL, "n=" + std::to_string(n) + " is not a power of two; hashing undefined");
    dbfs_rmat_params prm{};
    int k = 0;
    while (((int64_t)1 << k) < n) k++;
    prm.scale = k;
    prm.edge_factor = 1;
    prm.seed = seed;
    RmatGen g = make_gen(prm);
    if (count == 0) return;
    DArray<int64_t> a, b;
    a.alloc(count);
    b.alloc(count);
    DBFS_CUDA(cudaMemcpyAsync(a.p, in, 8 * count, cudaMemcpyHostToDevice, ctx.stream));
    k_hash_ids<<<ctx.num_sms * 8, 256, 0, ctx.stream>>>(g, a.p, b.p, count);
    DBFS_LAUNCHED();
    DBFS_CUDA(cudaMemcpyAsync(out, b.p, 8 * count, cudaMemcpyDeviceToHost, ctx.stream));
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

// ------------------------------------------------------------------ degrees

// For symmetrized RMAT only the m0 originals are generated; each adds one
// out-edge to both endpoints (bincount over the doubled src == deg(u)+deg(v)).
__global__ void k_degree(EdgeSrc es, int64_t begin, int64_t end, int both, uint32_t *__restrict__ deg) {
    for (int64_t e = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < end;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t u, v;
        es.get(e, u, v);
        atomicAdd(&deg[u], 1u);
        if (both) atomicAdd(&deg[v], 1u);
    }
}

__global__ void k_flag_delegates(const uint32_t *__restrict__ deg, int64_t n, int64_t theta,
                                 uint32_t *__restrict__ flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        flag[v] = (int64_t)deg[v] > theta;  // partition.py:111
}

__global__ void k_classify(const uint32_t *__restrict__ flag, const int64_t *__restrict__ pos, int64_t n,
                           uint32_t *__restrict__ del_id, int64_t *__restrict__ del_gid) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (flag[v]) {
            int64_t id = pos[v];
            del_id[v] = (uint32_t)id;
            del_gid[id] = v;
        } else {
            del_id[v] = 0xffffffffu;
        }
    }
}

// ------------------------------------------------------------------- routing

struct RouteParams {
    int p;            // total workers
    int first, W;     // local workers [first, first+W)
    PDiv pd;
    int64_t base[MAXW][4];  // key base per local worker/kind (index by w - first)
};

// Alg. 1 (partition.py:165-175): the worker of edge (u,v) and its kind.
__device__ __forceinline__ void route_edge(uint32_t u, uint32_t v, const uint32_t *__restrict__ deg,
                                           const uint32_t *__restrict__ del_id, const PDiv &pd, int &worker,
                                           int &kind, uint32_t &du_id, uint32_t &dv_id) {
    du_id = del_id[u];
    dv_id = del_id[v];
    bool du = du_id != 0xffffffffu, dv = dv_id != 0xffffffffu;
    uint32_t home_u = pd.mod(u), home_v = pd.mod(v);
    if (!du) worker = home_u;
    else if (!dv) worker = home_v;
    else {
        uint32_t gu = deg[u], gv = deg[v];
        bool to_u = gu < gv || (gu == gv && u <= v);
        worker = to_u ? home_u : home_v;
    }
    kind = ((int)du << 1) | (int)dv;
}

// Pass 1 of the route: count rows (composite-key histogram), kind totals and
// per-(worker,dest) remote nn capacities.  Pass 2 writes keys/values.
template <bool WRITE>
__global__ void k_route(EdgeSrc es, int64_t begin, int64_t end, const uint32_t *__restrict__ deg,
                        const uint32_t *__restrict__ del_id, const RouteParams *__restrict__ rp,
                        uint32_t *__restrict__ key_cnt, unsigned long long *__restrict__ kind_tot,
                        unsigned long long *__restrict__ remote, uint32_t *__restrict__ keys,
                        uint32_t *__restrict__ vals) {
    __shared__ unsigned long long s_kind[4];
    if (threadIdx.x < 4) s_kind[threadIdx.x] = 0;
    __syncthreads();
    const int first = rp->first, W = rp->W;
    const PDiv pd = rp->pd;
    for (int64_t e = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < end;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t u, v, du, dv;
        int worker, kind;
        es.get(e, u, v);
        route_edge(u, v, deg, del_id, pd, worker, kind, du, dv);
        int lw = worker - first;
        if (lw < 0 || lw >= W) continue;  // dist: edge belongs to another rank (never for local build)
        uint32_t row = (kind == KIND_NN || kind == KIND_ND) ? pd.div(u) : du;  // partition.py:319
        uint32_t col = kind == KIND_NN ? v : (kind == KIND_DN ? pd.div(v) : dv);  // partition.py:320-325
        uint32_t key = (uint32_t)(rp->base[lw][kind] + row);
        if (!WRITE) {
            atomicAdd(&key_cnt[key], 1u);
            atomicAdd(&s_kind[kind], 1ull);
            if (kind == KIND_NN) {
                int o = pd.mod(v);
                if (o != worker) atomicAdd(&remote[lw * MAXW + o], 1ull);
            }
        } else {
            keys[e - begin] = key;
            vals[e - begin] = col;
        }
    }
    if (!WRITE) {
        __syncthreads();
        if (threadIdx.x < 4 && s_kind[threadIdx.x]) atomicAdd(&kind_tot[threadIdx.x], s_kind[threadIdx.x]);
    }
}

// Dist mode: route pass that emits (dest worker, key, col) for the all-to-all.
__global__ void k_route_dest(EdgeSrc es, int64_t begin, int64_t end, const uint32_t *__restrict__ deg,
                             const uint32_t *__restrict__ del_id, PDiv pd, const int64_t *__restrict__ wbase,
                             uint32_t *__restrict__ dest, uint32_t *__restrict__ keys,
                             uint32_t *__restrict__ vals, unsigned long long *__restrict__ kind_tot) {
    for (int64_t e = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < end;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t u, v, du, dv;
        int worker, kind;
        es.get(e, u, v);
        route_edge(u, v, deg, del_id, pd, worker, kind, du, dv);
        uint32_t row = (kind == KIND_NN || kind == KIND_ND) ? pd.div(u) : du;
        uint32_t col = kind == KIND_NN ? v : (kind == KIND_DN ? pd.div(v) : dv);
        dest[e - begin] = (uint32_t)worker;
        keys[e - begin] = (uint32_t)(wbase[worker * 4 + kind] + row);
        vals[e - begin] = col;
        atomicAdd(&kind_tot[kind], 1ull);
    }
}

__global__ void k_src_bits(const int64_t *__restrict__ off, int64_t rows, uint32_t *__restrict__ bits,
                           unsigned long long *__restrict__ count) {
    int64_t nw = nwords(rows);
    unsigned long long c = 0;
    for (int64_t wi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wi < nw; wi += (int64_t)gridDim.x * blockDim.x) {
        uint32_t word = 0;
        int64_t r0 = wi * 32;
        for (int b = 0; b < 32; b++) {
            int64_t r = r0 + b;
            if (r < rows && off[r + 1] > off[r]) word |= 1u << b;
        }
        bits[wi] = word;
        c += __popc(word);
    }
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(count, c);
}

__global__ void k_row_degrees(const int64_t *__restrict__ off, int64_t rows, uint32_t *__restrict__ deg) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        deg[r] = (uint32_t)(off[r + 1] - off[r]);
}

__global__ void k_remote_caps_keys(const uint32_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                                   int64_t m, int64_t nn_rows, PDiv pd, int w,
                                   unsigned long long *__restrict__ remote) {
    // dist mode: keys < nn_rows are nn edges of this worker (base 0)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        if ((int64_t)keys[e] < nn_rows) {
            int o = pd.mod(vals[e]);
            if (o != w) atomicAdd(&remote[o], 1ull);
        }
    }
}

// ------------------------------------------------------------------- driver

static int64_t n_local_of(int64_t n, int p, int w) { return w < n ? (n - w + p - 1) / p : 0; }  // partition.py:314

static int bits_for(int64_t x) {
    int b = 0;
    while (b < 63 && ((int64_t)1 << b) < x) b++;
    return b;
}

static void finish_workers(Graph &g, int64_t nkeys, const std::vector<int64_t> &wbase_all) {
    Ctx &ctx = *g.ctx;
    unsigned long long *dcount;
    DBFS_CUDA(cudaMalloc(&dcount, sizeof(unsigned long long) * 4));
    for (auto &W : g.workers) {
        int lw = W.w - g.first_worker;
        for (int k = 0; k < 4; k++) {
            W.base[k] = wbase_all[(size_t)lw * 4 + k];
            W.rows[k] = (k == KIND_NN || k == KIND_ND) ? W.n_local : g.d;
        }
        int64_t offs[5];
        for (int k = 0; k < 4; k++)
            DBFS_CUDA(cudaMemcpy(&offs[k], g.off_all.p + W.base[k], 8, cudaMemcpyDeviceToHost));
        DBFS_CUDA(cudaMemcpy(&offs[4], g.off_all.p + W.base[3] + W.rows[3], 8, cudaMemcpyDeviceToHost));
        for (int k = 0; k < 4; k++) W.nnz[k] = offs[k + 1] - offs[k];
        DBFS_CUDA(cudaMemset(dcount, 0, sizeof(unsigned long long) * 4));
        for (int k = 0; k < 4; k++) {
            W.src_bits[k].alloc(std::max<int64_t>(nwords(W.rows[k]), 1));
            DBFS_CUDA(cudaMemsetAsync(W.src_bits[k].p, 0, W.src_bits[k].bytes(), ctx.stream));
            if (W.rows[k] > 0) {
                int blocks = (int)std::min<int64_t>(ceil_div(nwords(W.rows[k]), 256), ctx.num_sms * 16);
                k_src_bits<<<blocks, 256, 0, ctx.stream>>>(g.off_all.p + W.base[k], W.rows[k], W.src_bits[k].p,
                                                           dcount + k);
                DBFS_LAUNCHED();
            }
        }
        unsigned long long hc[4];
        DBFS_CUDA(cudaMemcpyAsync(hc, dcount, sizeof(hc), cudaMemcpyDeviceToHost, ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
        for (int k = 0; k < 4; k++) W.n_src[k] = (int64_t)hc[k];
        // compact row lengths: nd per local normal, dn / dd per delegate
        W.deg[KIND_ND].alloc(std::max<int64_t>(W.rows[KIND_ND], 1));
        W.deg[KIND_DN].alloc(std::max<int64_t>(W.rows[KIND_DN], 1));
        W.deg[KIND_DD].alloc(std::max<int64_t>(W.rows[KIND_DD], 1));
        for (int k = 1; k < 4; k++)
            if (W.rows[k] > 0) {
                int blocks = (int)std::min<int64_t>(ceil_div(W.rows[k], 256), ctx.num_sms * 16);
                k_row_degrees<<<blocks, 256, 0, ctx.stream>>>(g.off_all.p + W.base[k], W.rows[k], W.deg[k].p);
                DBFS_LAUNCHED();
            }
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    cudaFree(dcount);
    (void)nkeys;
}

// Shared tail of the single-process build: route -> key histogram -> offsets ->
// stable radix sort of (key, col) -> CSR views and source bitmaps.
static void build_local(Graph &g, const EdgeSrc &es, int64_t m) {
    Ctx &ctx = *g.ctx;
    const int p = g.p;
    const int64_t n = g.n, d = g.d;
    // composite key layout: [w][nn rows | nd rows | dn rows | dd rows]
    RouteParams rp{};
    rp.p = p;
    rp.first = 0;
    rp.W = p;
    rp.pd.init((uint32_t)p);
    std::vector<int64_t> wbase((size_t)p * 4);
    int64_t acc = 0;
    g.workers.resize(p);
    for (int w = 0; w < p; w++) {
        g.workers[w].w = w;
        g.workers[w].n_local = n_local_of(n, p, w);
        int64_t rows[4] = {g.workers[w].n_local, g.workers[w].n_local, d, d};
        for (int k = 0; k < 4; k++) {
            rp.base[w][k] = acc;
            wbase[(size_t)w * 4 + k] = acc;
            acc += rows[k];
        }
    }
    const int64_t nkeys = acc;
    DBFS_CHECK(nkeys < ((int64_t)1 << 32), DBFS_ECAPACITY, "composite row space exceeds 32 bits");
    DArray<RouteParams> drp;
    drp.alloc(1);
    DBFS_CUDA(cudaMemcpy(drp.p, &rp, sizeof(rp), cudaMemcpyHostToDevice));
    DArray<uint32_t> key_cnt;
    key_cnt.alloc(std::max<int64_t>(nkeys, 1));
    DBFS_CUDA(cudaMemsetAsync(key_cnt.p, 0, key_cnt.bytes(), ctx.stream));
    DArray<unsigned long long> kt, remote;
    kt.alloc(4);
    remote.alloc((int64_t)MAXW * MAXW);
    DBFS_CUDA(cudaMemsetAsync(kt.p, 0, kt.bytes(), ctx.stream));
    DBFS_CUDA(cudaMemsetAsync(remote.p, 0, remote.bytes(), ctx.stream));
    const int gblocks = ctx.num_sms * 16;
    if (m > 0) {
        k_route<false><<<gblocks, 256, 0, ctx.stream>>>(es, 0, m, g.degree.p, g.del_id.p, drp.p, key_cnt.p, kt.p,
                                                        remote.p, nullptr, nullptr);
        DBFS_LAUNCHED();
    }
    g.off_all.alloc(nkeys + 1);
    exclusive_scan_u32_to_i64(ctx, key_cnt.p, g.off_all.p, nkeys);
    key_cnt.release();
    unsigned long long ktot[4];
    DBFS_CUDA(cudaMemcpy(ktot, kt.p, sizeof(ktot), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 4; k++) g.kind_totals[k] = (int64_t)ktot[k];
    std::vector<unsigned long long> rem((size_t)MAXW * MAXW);
    DBFS_CUDA(cudaMemcpy(rem.data(), remote.p, remote.bytes(), cudaMemcpyDeviceToHost));
    for (int w = 0; w < p; w++)
        for (int o = 0; o < MAXW; o++) g.workers[w].remote_cap[o] = (int64_t)rem[(size_t)w * MAXW + o];

    // keys/values, then the stable sort
    g.col_all.alloc(std::max<int64_t>(m, 1));
    if (m > 0) {
        DArray<uint32_t> keys, keys2, vals2;
        keys.alloc(m);
        keys2.alloc(m);
        vals2.alloc(m);
        k_route<true><<<gblocks, 256, 0, ctx.stream>>>(es, 0, m, g.degree.p, g.del_id.p, drp.p, nullptr, nullptr,
                                                       nullptr, keys.p, g.col_all.p);
        DBFS_LAUNCHED();
        bool alt = false;
        radix_sort_pairs(ctx, keys.p, g.col_all.p, keys2.p, vals2.p, m, bits_for(nkeys), &alt);
        if (alt)
            DBFS_CUDA(cudaMemcpyAsync(g.col_all.p, vals2.p, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice,
                                      ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    finish_workers(g, nkeys, wbase);
}

// degrees + classification; fills g.degree, g.del_id, g.del_gid, g.d
static void classify(Graph &g) {
    Ctx &ctx = *g.ctx;
    const int64_t n = g.n;
    DArray<uint32_t> flag;
    DArray<int64_t> pos;
    flag.alloc(std::max<int64_t>(n, 1));
    pos.alloc(n + 1);
    int blocks = (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), ctx.num_sms * 16);
    k_flag_delegates<<<blocks, 256, 0, ctx.stream>>>(g.degree.p, n, g.theta, flag.p);
    DBFS_LAUNCHED();
    exclusive_scan_u32_to_i64(ctx, flag.p, pos.p, n);
    DBFS_CUDA(cudaMemcpy(&g.d, pos.p + n, 8, cudaMemcpyDeviceToHost));
    // CapacityError (partition.py:308-309)
    DBFS_CHECK(ceil_div(n, g.p) < ((int64_t)1 << 32) && g.d < ((int64_t)1 << 32) - 1, DBFS_ECAPACITY,
               "local id space exceeds 32 bits");
    g.del_id.alloc(std::max<int64_t>(n, 1));
    g.del_gid.alloc(std::max<int64_t>(g.d, 1));
    k_classify<<<blocks, 256, 0, ctx.stream>>>(flag.p, pos.p, n, g.del_id.p, g.del_gid.p);
    DBFS_LAUNCHED();
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

// A partition built elsewhere (the reference's PartitionedGraph,
// partition.py:263-292, or a DPG1 file set) straight into the device layout:
// per worker the four CSRs (int64 offsets; int64 nn / uint32 other columns),
// concatenated in the composite row order [w][nn | nd | dn | dd] with absolute
// offsets, then the same per-worker aids (source bitmaps, row lengths) the
// device build derives.  No edge list, no re-sort: the rows keep the caller's
// neighbour order, which the BFS counters depend on.
void upload_partitioned(Graph &g, const int64_t *degree, const int64_t *dgid, const int64_t *const *off,
                        const void *const *cols) {
    Ctx &ctx = *g.ctx;
    const int p = g.p;
    const int64_t n = g.n, d = g.d;
    DBFS_CHECK(ctx.nranks == 1, DBFS_EINVAL, "upload builds a single-process partition");
    DBFS_CHECK(p >= 1 && p <= MAXW, DBFS_ECAPACITY, "at most 64 workers");
    DBFS_CHECK(ceil_div(n, p) < ((int64_t)1 << 32) && d < ((int64_t)1 << 32) - 1, DBFS_ECAPACITY,
               "local id space exceeds 32 bits");
    // classification: degrees, delegate ids (ascending global ids)
    {
        std::vector<uint32_t> h((size_t)std::max<int64_t>(n, 1), 0);
        for (int64_t v = 0; v < n; v++) {
            DBFS_CHECK(degree[v] >= 0 && degree[v] < ((int64_t)1 << 32), DBFS_ECAPACITY, "degree exceeds 32 bits");
            h[v] = (uint32_t)degree[v];
        }
        g.degree.alloc(std::max<int64_t>(n, 1));
        DBFS_CUDA(cudaMemcpy(g.degree.p, h.data(), 4 * (size_t)std::max<int64_t>(n, 1), cudaMemcpyHostToDevice));
        std::fill(h.begin(), h.end(), 0xffffffffu);
        for (int64_t x = 0; x < d; x++) {
            DBFS_CHECK(dgid[x] >= 0 && dgid[x] < n && (x == 0 || dgid[x] > dgid[x - 1]), DBFS_ESTRUCT,
                       "delegate ids must be ascending global ids");
            h[dgid[x]] = (uint32_t)x;
        }
        g.del_id.alloc(std::max<int64_t>(n, 1));
        DBFS_CUDA(cudaMemcpy(g.del_id.p, h.data(), 4 * (size_t)std::max<int64_t>(n, 1), cudaMemcpyHostToDevice));
        g.del_gid.alloc(std::max<int64_t>(d, 1));
        if (d) DBFS_CUDA(cudaMemcpy(g.del_gid.p, dgid, 8 * d, cudaMemcpyHostToDevice));
    }
    // composite layout and absolute offsets
    g.workers.resize(p);
    std::vector<int64_t> wbase((size_t)p * 4);
    int64_t nkeys = 0, m = 0;
    for (int w = 0; w < p; w++) {
        g.workers[w].w = w;
        g.workers[w].n_local = n_local_of(n, p, w);
        for (int k = 0; k < 4; k++) {
            const int64_t rows = k < 2 ? g.workers[w].n_local : d;
            const int64_t *o = off[(size_t)w * 4 + k];
            DBFS_CHECK(o[0] == 0, DBFS_ESTRUCT, "row offsets must start at 0");
            for (int64_t r = 0; r < rows; r++)
                DBFS_CHECK(o[r + 1] >= o[r], DBFS_ESTRUCT, "row offsets must be non-decreasing");
            wbase[(size_t)w * 4 + k] = nkeys;
            nkeys += rows;
            m += o[rows];
        }
    }
    DBFS_CHECK(m == g.m, DBFS_ESTRUCT, "the workers' CSRs must hold the graph's m edges");
    DBFS_CHECK(nkeys < ((int64_t)1 << 32), DBFS_ECAPACITY, "composite row space exceeds 32 bits");
    std::vector<int64_t> hoff((size_t)nkeys + 1);
    std::vector<uint32_t> hcol((size_t)std::max<int64_t>(m, 1));
    int64_t acc = 0;
    for (int k = 0; k < 4; k++) g.kind_totals[k] = 0;
    for (int w = 0; w < p; w++) {
        for (int o = 0; o < MAXW; o++) g.workers[w].remote_cap[o] = 0;
        for (int k = 0; k < 4; k++) {
            const int64_t rows = k < 2 ? g.workers[w].n_local : d;
            const int64_t *o = off[(size_t)w * 4 + k];
            const int64_t base = wbase[(size_t)w * 4 + k];
            for (int64_t r = 0; r < rows; r++) hoff[base + r] = acc + o[r];
            const int64_t nnz = o[rows];
            const int64_t lim = k == KIND_NN ? n : (k == KIND_DN ? g.workers[w].n_local : d);
            for (int64_t j = 0; j < nnz; j++) {
                const int64_t c = k == KIND_NN ? static_cast<const int64_t *>(cols[(size_t)w * 4 + k])[j]
                                               : (int64_t) static_cast<const uint32_t *>(cols[(size_t)w * 4 + k])[j];
                DBFS_CHECK(c >= 0 && c < lim, DBFS_ESTRUCT, "column out of range for its kind");
                hcol[acc + j] = (uint32_t)c;
                if (k == KIND_NN && (int)(c % p) != w) g.workers[w].remote_cap[c % p]++;
            }
            acc += nnz;
            g.kind_totals[k] += nnz;
        }
    }
    hoff[nkeys] = acc;
    g.off_all.alloc(nkeys + 1);
    DBFS_CUDA(cudaMemcpy(g.off_all.p, hoff.data(), 8 * hoff.size(), cudaMemcpyHostToDevice));
    g.col_all.alloc(std::max<int64_t>(m, 1));
    if (m) DBFS_CUDA(cudaMemcpy(g.col_all.p, hcol.data(), 4 * (size_t)m, cudaMemcpyHostToDevice));
    finish_workers(g, nkeys, wbase);
}

static void build_dist(Graph &g, const EdgeSrc &es, int64_t begin, int64_t end);

void mem_note(const Ctx &ctx, const char *what) {
    static const bool on = getenv("DBFS_VERBOSE") && getenv("DBFS_VERBOSE")[0] == '1';
    if (!on) return;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    fprintf(stderr, "[dbfs rank %d dev %d] %s: %zu MiB free of %zu\n", ctx.rank, ctx.device, what, fr >> 20, tot >> 20);
}

void build_graph_rmat(Graph &g, const dbfs_rmat_params &prm) {
    Ctx &ctx = *g.ctx;
    DBFS_CHECK(prm.scale >= 0 && prm.scale <= 32 && prm.edge_factor >= 1, DBFS_EINVAL, "bad RMAT params");
    DBFS_CHECK(g.p >= 1 && g.p <= MAXW, DBFS_EINVAL, "p must be in [1, 64]");
    EdgeSrc es{};
    es.gen = make_gen(prm);
    es.symmetrize = prm.symmetrize;
    es.src = es.dst = nullptr;
    g.n = (int64_t)1 << prm.scale;
    g.m = es.gen.m0 * (prm.symmetrize ? 2 : 1);
    g.degree.alloc(g.n);
    DBFS_CUDA(cudaMemsetAsync(g.degree.p, 0, g.degree.bytes(), ctx.stream));
    const int gblocks = ctx.num_sms * 16;
    int64_t rb = 0, re = prm.symmetrize ? es.gen.m0 : g.m;
    if (g.dist) {  // every rank generates a slice; degrees all-reduced
        int64_t per = ceil_div(re, ctx.nranks);
        rb = std::min(re, per * ctx.rank);
        re = std::min(re, rb + per);
    }
    if (re > rb) {
        k_degree<<<gblocks, 256, 0, ctx.stream>>>(es, rb, re, prm.symmetrize, g.degree.p);
        DBFS_LAUNCHED();
    }
    if (g.dist) nccl_allreduce_u32_sum(ctx, g.degree.p, g.n);
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    mem_note(ctx, "degrees");
    classify(g);
    mem_note(ctx, "classified");
    if (g.dist) {
        int64_t per = ceil_div(g.m, ctx.nranks);
        int64_t b = std::min(g.m, per * ctx.rank), e = std::min(g.m, b + per);
        build_dist(g, es, b, e);
    } else {
        build_local(g, es, g.m);
    }
}

__global__ void k_degree_explicit(const int64_t *__restrict__ src, int64_t m, uint32_t *__restrict__ deg) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&deg[src[e]], 1u);
}

void build_graph_edges(Graph &g, const int64_t *src, const int64_t *dst, int64_t m_local) {
    Ctx &ctx = *g.ctx;
    DBFS_CHECK(g.p >= 1 && g.p <= MAXW, DBFS_EINVAL, "p must be in [1, 64]");
    DBFS_CHECK(g.n >= 0 && g.n <= ((int64_t)1 << 32), DBFS_ECAPACITY, "n must fit 32-bit vertex ids");
    for (int64_t i = 0; i < m_local; i++)
        DBFS_CHECK(src[i] >= 0 && src[i] < g.n && dst[i] >= 0 && dst[i] < g.n, DBFS_ERANGE,
                   "edge endpoint out of range");
    DArray<int64_t> ds, dd;
    ds.alloc(std::max<int64_t>(m_local, 1));
    dd.alloc(std::max<int64_t>(m_local, 1));
    if (m_local) {
        DBFS_CUDA(cudaMemcpyAsync(ds.p, src, 8 * m_local, cudaMemcpyHostToDevice, ctx.stream));
        DBFS_CUDA(cudaMemcpyAsync(dd.p, dst, 8 * m_local, cudaMemcpyHostToDevice, ctx.stream));
    }
    g.degree.alloc(std::max<int64_t>(g.n, 1));
    DBFS_CUDA(cudaMemsetAsync(g.degree.p, 0, g.degree.bytes(), ctx.stream));
    if (m_local) {
        k_degree_explicit<<<ctx.num_sms * 16, 256, 0, ctx.stream>>>(ds.p, m_local, g.degree.p);
        DBFS_LAUNCHED();
    }
    if (g.dist) {
        nccl_allreduce_u32_sum(ctx, g.degree.p, g.n);
        int64_t mt = m_local;
        DArray<int64_t> t;
        t.alloc(1);
        DBFS_CUDA(cudaMemcpy(t.p, &mt, 8, cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx, t.p, 1, 0);
        DBFS_CUDA(cudaMemcpy(&g.m, t.p, 8, cudaMemcpyDeviceToHost));
    } else {
        g.m = m_local;
    }
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    classify(g);
    EdgeSrc es{};
    es.src = ds.p;
    es.dst = dd.p;
    if (g.dist) build_dist(g, es, 0, m_local);
    else build_local(g, es, m_local);
}

// Distributed build: this rank routes its slice [begin,end) of the global edge
// order, the (key, col) records travel to their owner rank (all-to-all, rank
// order preserved => global edge order preserved), then a local stable sort.
// Everything stays in device memory; only p-sized count vectors reach the host.
__global__ void k_iota(uint32_t *__restrict__ a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

__global__ void k_pack_records(const uint32_t *__restrict__ idx, const uint32_t *__restrict__ keys,
                               const uint32_t *__restrict__ vals, int64_t n, uint2 *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t j = idx[i];
        out[i] = make_uint2(keys[j], vals[j]);
    }
}

__global__ void k_count_dest(const uint32_t *__restrict__ dest, int64_t n, unsigned long long *__restrict__ cnt) {
    __shared__ unsigned long long s[MAXW];
    for (int i = threadIdx.x; i < MAXW; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&s[dest[i]], 1ull);
    __syncthreads();
    for (int i = threadIdx.x; i < MAXW; i += blockDim.x)
        if (s[i]) atomicAdd(&cnt[i], s[i]);
}

__global__ void k_unpack_records(const uint2 *__restrict__ rec, int64_t n, uint32_t *__restrict__ keys,
                                 uint32_t *__restrict__ vals, uint32_t *__restrict__ key_cnt, int64_t nn_rows,
                                 PDiv pd, int self, unsigned long long *__restrict__ remote) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint2 r = rec[i];
        keys[i] = r.x;
        vals[i] = r.y;
        atomicAdd(&key_cnt[r.x], 1u);
        if ((int64_t)r.x < nn_rows) {  // nn edge: capacity of remote records to the column's owner
            int o = pd.mod(r.y);
            if (o != self) atomicAdd(&remote[o], 1ull);
        }
    }
}

static void build_dist(Graph &g, const EdgeSrc &es, int64_t begin, int64_t end) {
    Ctx &ctx = *g.ctx;
    const int p = g.p, r = ctx.rank;
    DBFS_CHECK(p == ctx.nranks, DBFS_EINVAL, "distributed build needs p == number of ranks");
    PDiv pd;
    pd.init((uint32_t)p);
    const int64_t n = g.n, d = g.d;
    std::vector<int64_t> wbase((size_t)p * 4);
    for (int w = 0; w < p; w++) {  // key space is per destination worker
        int64_t nl = n_local_of(n, p, w);
        int64_t rows[4] = {nl, nl, d, d};
        int64_t acc = 0;
        for (int k = 0; k < 4; k++) {
            wbase[(size_t)w * 4 + k] = acc;
            acc += rows[k];
        }
    }
    DArray<int64_t> dwbase;
    dwbase.alloc((int64_t)p * 4);
    DBFS_CUDA(cudaMemcpy(dwbase.p, wbase.data(), 8 * p * 4, cudaMemcpyHostToDevice));
    const int64_t ml = end - begin;
    const int blocks = ctx.num_sms * 16;
    // The slice is routed in chunks of <= 2^29 edges (bounded temporaries,
    // 32-bit indices at any scale).  A counting pass sizes every (source rank,
    // chunk) segment first, so each chunk's all-to-all lands at its place in
    // global edge order on the receiver.
    const int64_t CH = (int64_t)1 << 29;
    int64_t nch = std::max<int64_t>(1, ceil_div(ml, CH));
    {
        DArray<int64_t> t;
        t.alloc(1);
        DBFS_CUDA(cudaMemcpy(t.p, &nch, 8, cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx, t.p, 1, 2);  // max over ranks: the chunk loop is collective
        DBFS_CUDA(cudaMemcpy(&nch, t.p, 8, cudaMemcpyDeviceToHost));
    }
    const int64_t cap = std::max<int64_t>(1, std::min(ml, CH));
    auto chunk = [&](int64_t c, int64_t &c0, int64_t &c1) {
        c0 = std::min(end, begin + c * CH);
        c1 = std::min(end, c0 + CH);
    };
    DArray<unsigned long long> kt, dcnt, kt_dummy;
    kt.alloc(4);
    kt_dummy.alloc(4);
    dcnt.alloc(MAXW);
    DBFS_CUDA(cudaMemsetAsync(kt.p, 0, kt.bytes(), ctx.stream));
    DArray<uint32_t> dest, keys, vals, idx, dest2, idx2;
    dest.alloc(cap);
    keys.alloc(cap);
    vals.alloc(cap);
    idx.alloc(cap);
    dest2.alloc(cap);
    idx2.alloc(cap);
    // pass 1: records per (chunk, destination)
    std::vector<int64_t> cnt_local((size_t)nch * p, 0);
    for (int64_t c = 0; c < nch; c++) {
        int64_t c0, c1;
        chunk(c, c0, c1);
        if (c1 <= c0) continue;
        DBFS_CUDA(cudaMemsetAsync(dcnt.p, 0, dcnt.bytes(), ctx.stream));
        k_route_dest<<<blocks, 256, 0, ctx.stream>>>(es, c0, c1, g.degree.p, g.del_id.p, pd, dwbase.p, dest.p, keys.p,
                                                     vals.p, kt.p);
        DBFS_LAUNCHED();
        k_count_dest<<<blocks, 256, 0, ctx.stream>>>(dest.p, c1 - c0, dcnt.p);
        DBFS_LAUNCHED();
        std::vector<unsigned long long> h(MAXW);
        DBFS_CUDA(cudaMemcpy(h.data(), dcnt.p, 8 * MAXW, cudaMemcpyDeviceToHost));
        for (int o = 0; o < p; o++) cnt_local[(size_t)c * p + o] = (int64_t)h[o];
    }
    // global kind totals
    {
        DArray<int64_t> t;
        t.alloc(4);
        unsigned long long h[4];
        DBFS_CUDA(cudaMemcpy(h, kt.p, sizeof(h), cudaMemcpyDeviceToHost));
        int64_t hv[4] = {(int64_t)h[0], (int64_t)h[1], (int64_t)h[2], (int64_t)h[3]};
        DBFS_CUDA(cudaMemcpy(t.p, hv, sizeof(hv), cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx, t.p, 4, 0);
        DBFS_CUDA(cudaMemcpy(hv, t.p, sizeof(hv), cudaMemcpyDeviceToHost));
        for (int k = 0; k < 4; k++) g.kind_totals[k] = hv[k];
    }
    // every rank's counts [source][chunk][dest]
    const int64_t CPS = nch * p;
    std::vector<int64_t> all((size_t)p * CPS);
    {
        DArray<int64_t> sc, rc;
        sc.alloc(CPS);
        rc.alloc((int64_t)p * CPS);
        DBFS_CUDA(cudaMemcpy(sc.p, cnt_local.data(), 8 * CPS, cudaMemcpyHostToDevice));
        nccl_allgather_bytes(ctx, sc.p, rc.p, 8 * CPS);
        DBFS_CUDA(cudaMemcpy(all.data(), rc.p, 8 * p * CPS, cudaMemcpyDeviceToHost));
    }
    auto count = [&](int s, int64_t c, int o) { return all[(size_t)s * CPS + (size_t)c * p + o]; };
    // receive layout: source-major, then chunk (== global edge order)
    std::vector<int64_t> rseg((size_t)p * nch);
    int64_t racc = 0;
    for (int s = 0; s < p; s++)
        for (int64_t c = 0; c < nch; c++) {
            rseg[(size_t)s * nch + c] = racc;
            racc += count(s, c, r);
        }
    DArray<uint2> rbuf, sbuf;
    mem_note(ctx, "counted");
    rbuf.alloc(std::max<int64_t>(racc, 1));
    sbuf.alloc(cap);
    mem_note(ctx, "exchange buffers");
    // pass 2: route, bucket by destination (stable), exchange
    for (int64_t c = 0; c < nch; c++) {
        int64_t c0, c1;
        chunk(c, c0, c1);
        const int64_t cm = std::max<int64_t>(c1 - c0, 0);
        if (cm > 0) {
            k_route_dest<<<blocks, 256, 0, ctx.stream>>>(es, c0, c1, g.degree.p, g.del_id.p, pd, dwbase.p, dest.p,
                                                         keys.p, vals.p, kt_dummy.p);
            DBFS_LAUNCHED();
            k_iota<<<blocks, 256, 0, ctx.stream>>>(idx.p, cm);
            DBFS_LAUNCHED();
            bool alt = false;  // stable bucket by destination (edge order kept inside a bucket)
            radix_sort_pairs(ctx, dest.p, idx.p, dest2.p, idx2.p, cm, std::max(1, bits_for(p)), &alt);
            k_pack_records<<<blocks, 256, 0, ctx.stream>>>(alt ? idx2.p : idx.p, keys.p, vals.p, cm, sbuf.p);
            DBFS_LAUNCHED();
        }
        std::vector<int64_t> soff(p), sbytes(p), roff(p), rbytes(p);
        int64_t acc = 0;
        for (int o = 0; o < p; o++) {
            soff[o] = acc * 8;
            sbytes[o] = count(r, c, o) * 8;
            acc += count(r, c, o);
            roff[o] = rseg[(size_t)o * nch + c] * 8;
            rbytes[o] = count(o, c, r) * 8;
        }
        nccl_alltoallv_bytes(ctx, sbuf.p, soff.data(), sbytes.data(), rbuf.p, roff.data(), rbytes.data());
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
        mem_note(ctx, "chunk exchanged");
    }
    sbuf.release();
    dest.release();
    keys.release();
    vals.release();
    idx.release();
    dest2.release();
    idx2.release();
    // local CSR from the received records (source-rank order == global edge order)
    g.workers.clear();
    g.workers.resize(1);
    WorkerHost &me = g.workers[0];
    me.w = r;
    me.n_local = n_local_of(n, p, r);
    const int64_t nkeys = 2 * me.n_local + 2 * d;
    DBFS_CHECK(nkeys < ((int64_t)1 << 32), DBFS_ECAPACITY, "local row space exceeds 32 bits");
    DArray<uint32_t> kk, kk2, vv2, cnt;
    DArray<unsigned long long> remote;
    kk.alloc(std::max<int64_t>(racc, 1));
    kk2.alloc(std::max<int64_t>(racc, 1));
    vv2.alloc(std::max<int64_t>(racc, 1));
    cnt.alloc(std::max<int64_t>(nkeys, 1));
    remote.alloc(MAXW);
    g.col_all.alloc(std::max<int64_t>(racc, 1));
    mem_note(ctx, "local sort buffers");
    DBFS_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), ctx.stream));
    DBFS_CUDA(cudaMemsetAsync(remote.p, 0, remote.bytes(), ctx.stream));
    if (racc) {
        k_unpack_records<<<blocks, 256, 0, ctx.stream>>>(rbuf.p, racc, kk.p, g.col_all.p, cnt.p, me.n_local, pd, r,
                                                         remote.p);
        DBFS_LAUNCHED();
    }
    rbuf.release();
    g.off_all.alloc(nkeys + 1);
    exclusive_scan_u32_to_i64(ctx, cnt.p, g.off_all.p, nkeys);
    {
        std::vector<unsigned long long> h(MAXW);
        DBFS_CUDA(cudaMemcpy(h.data(), remote.p, 8 * MAXW, cudaMemcpyDeviceToHost));
        for (int o = 0; o < MAXW; o++) me.remote_cap[o] = (int64_t)h[o];
    }
    bool alt3 = false;
    radix_sort_pairs(ctx, kk.p, g.col_all.p, kk2.p, vv2.p, racc, bits_for(nkeys), &alt3);
    if (alt3 && racc) DBFS_CUDA(cudaMemcpy(g.col_all.p, vv2.p, 4 * racc, cudaMemcpyDeviceToDevice));
    std::vector<int64_t> wb = {wbase[(size_t)r * 4 + 0], wbase[(size_t)r * 4 + 1], wbase[(size_t)r * 4 + 2],
                               wbase[(size_t)r * 4 + 3]};
    g.first_worker = r;
    g.W = 1;
    finish_workers(g, nkeys, wb);
}

// ------------------------------------------------- degree-ordered dd rows

__global__ void k_deg_keys(const uint32_t *__restrict__ col, const int64_t *__restrict__ off0, int64_t nnz,
                           const uint32_t *__restrict__ deg, const int64_t *__restrict__ del_gid,
                           uint32_t *__restrict__ key, uint32_t *__restrict__ idx) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t dg = deg[del_gid[col[off0[0] + j]]];
        key[j] = 0xffffffffu - dg;  // descending degree
        idx[j] = (uint32_t)j;
    }
}

__global__ void k_row_ids(const int64_t *__restrict__ off, int64_t rows, uint32_t *__restrict__ rowid) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, TW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t b0 = off[0];
    for (int64_t r = gw; r < rows; r += TW)
        for (int64_t j = off[r] - b0 + lane_id(); j < off[r + 1] - b0; j += 32) rowid[j] = (uint32_t)r;
}

__global__ void k_row_keys(const uint32_t *__restrict__ idx, const uint32_t *__restrict__ rowid, int64_t nnz,
                           uint32_t *__restrict__ key) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
        key[j] = rowid[idx[j]];
}

__global__ void k_gather_cols(const uint32_t *__restrict__ idx, const uint32_t *__restrict__ col, int64_t base,
                              int64_t nnz, uint32_t *__restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
        out[base + j] = col[base + idx[j]];
}

// For every local worker: a copy of the dd rows with neighbours ordered by
// descending degree (two stable radix passes: degree, then row).  Used only
// by executor pulls of FORWARD-reported dd levels, where scan order is free.
void build_sorted_dd(Graph &g) {
    Ctx &ctx = *g.ctx;
    for (auto &W : g.workers) {
        const int64_t nnz = W.nnz[KIND_DD], rows = W.rows[KIND_DD];
        if (nnz == 0 || W.col_sorted.n) continue;
        const int64_t *off = g.off_all.p + W.base[KIND_DD];
        std::vector<int64_t> h(rows + 1);
        DBFS_CUDA(cudaMemcpy(h.data(), off, 8 * (rows + 1), cudaMemcpyDeviceToHost));
        W.dd_base = h[0];
        W.col_sorted.alloc(nnz);
        // row batches of <= 2^29 entries (a longer row is a batch of its own):
        // 32-bit entry indices and bounded sort temporaries at any scale
        const int64_t B = (int64_t)1 << 29;
        int64_t cap = 0;
        for (int64_t r0 = 0, r1; r0 < rows; r0 = r1) {
            r1 = r0 + 1;
            while (r1 < rows && h[r1 + 1] - h[r0] <= B) r1++;
            cap = std::max(cap, h[r1] - h[r0]);
        }
        DBFS_CHECK(cap < ((int64_t)1 << 32), DBFS_ECAPACITY, "a dd row exceeds 2^32 edges");
        DArray<uint32_t> key, idx, key2, idx2, rowid;
        key.alloc(cap);
        idx.alloc(cap);
        key2.alloc(cap);
        idx2.alloc(cap);
        rowid.alloc(cap);
        const int blocks = ctx.num_sms * 16;
        for (int64_t r0 = 0, r1; r0 < rows; r0 = r1) {
            r1 = r0 + 1;
            while (r1 < rows && h[r1 + 1] - h[r0] <= B) r1++;
            const int64_t bn = h[r1] - h[r0], brows = r1 - r0;
            if (bn == 0) continue;
            k_deg_keys<<<blocks, 256, 0, ctx.stream>>>(g.col_all.p, off + r0, bn, g.degree.p, g.del_gid.p, key.p,
                                                       idx.p);
            DBFS_LAUNCHED();
            bool alt = false;
            radix_sort_pairs(ctx, key.p, idx.p, key2.p, idx2.p, bn, 32, &alt);
            uint32_t *sidx = alt ? idx2.p : idx.p;
            k_row_ids<<<blocks, 256, 0, ctx.stream>>>(off + r0, brows, rowid.p);
            DBFS_LAUNCHED();
            uint32_t *k2 = alt ? key.p : key2.p;  // free key buffer
            k_row_keys<<<blocks, 256, 0, ctx.stream>>>(sidx, rowid.p, bn, k2);
            DBFS_LAUNCHED();
            // k2 = row of each degree-ordered entry; sort (stable) by row
            bool alt2 = false;
            uint32_t *k3 = (k2 == key.p) ? key2.p : key.p;
            uint32_t *i3 = (sidx == idx.p) ? idx2.p : idx.p;
            int bits = 1;
            while (bits < 32 && ((int64_t)1 << bits) < brows) bits++;
            radix_sort_pairs(ctx, k2, sidx, k3, i3, bn, bits, &alt2);
            uint32_t *fidx = alt2 ? i3 : sidx;
            k_gather_cols<<<blocks, 256, 0, ctx.stream>>>(fidx, g.col_all.p + h[r0], 0, bn,
                                                          W.col_sorted.p + (h[r0] - h[0]));
            DBFS_LAUNCHED();
        }
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
}

// ------------------------------------------------- twin positions (pull counters by push)

// key = column, val = entry index, over one kind's entries [0, nnz)
__global__ void k_col_keys(const uint32_t *__restrict__ col, int64_t nnz, uint32_t *__restrict__ key,
                           uint32_t *__restrict__ val) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
        key[j] = col[j];
        val[j] = (uint32_t)j;
    }
}

// Sorted forward entries (by target, then source) and sorted reverse entries
// (by row, then column) pair up index by index when the kind pair is the
// reverse of itself; entry fv[t] of kind K gets the position of its source in
// the target's reverse row.  Any mismatch (not symmetric) raises *bad.
__global__ void k_twin_fill(const uint32_t *__restrict__ fv, const uint32_t *__restrict__ rv,
                            const uint32_t *__restrict__ colK, const uint32_t *__restrict__ rowK,
                            const uint32_t *__restrict__ colR, const uint32_t *__restrict__ rowR,
                            const int64_t *__restrict__ offR, int64_t n, uint32_t *__restrict__ twin,
                            unsigned *__restrict__ bad) {
    const int64_t r0 = offR[0];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = fv[t], e2 = rv[t];
        const uint32_t b = rowR[e2];
        if (colK[e] != b || rowK[e] != colR[e2]) atomicOr(bad, 1u);
        twin[e] = (uint32_t)((int64_t)e2 - (offR[b] - r0));
    }
}

// Twin positions for the kinds a BACKWARD-reported level may execute as a
// push: for every entry (u -> v) of kind K (nd, dn, dd) the
// position of u in v's row of the reverse kind R (dn, nd, dd) -- the place a
// pull of v would find u.  Alg. 1 keeps an edge and its reverse on one worker
// for these kinds, so this is per worker.  Three stable radix sorts per kind.
// A kind whose temporaries do not fit, or that is not its own reverse, keeps
// no twins (its levels always pull).
void build_twins(Graph &g) {
    Ctx &ctx = *g.ctx;
    static const int PAIR[4] = {-1, KIND_DN, KIND_ND, KIND_DD};
    DArray<unsigned> bad;
    bad.alloc(1);
    for (auto &W : g.workers) {
        for (int K = 1; K < 4; K++) {
            const int R = PAIR[K];
            const int64_t n = W.nnz[K];
            if (n == 0 || n != W.nnz[R] || n >= ((int64_t)1 << 32) || W.twin[K].n) continue;
            size_t fr = 0, tot = 0;
            DBFS_CUDA(cudaMemGetInfo(&fr, &tot));
            if ((double)n * 4.0 * 9.0 > 0.8 * (double)fr) continue;  // 8 temporaries + the twins
            const int64_t *offK = g.off_all.p + W.base[K], *offR = g.off_all.p + W.base[R];
            int64_t k0 = 0, r0 = 0;
            DBFS_CUDA(cudaMemcpy(&k0, offK, 8, cudaMemcpyDeviceToHost));
            DBFS_CUDA(cudaMemcpy(&r0, offR, 8, cudaMemcpyDeviceToHost));
            const uint32_t *colK = g.col_all.p + k0, *colR = g.col_all.p + r0;
            DArray<uint32_t> key, val, key2, val2, fv, rowK, rowR;
            key.alloc(n);
            val.alloc(n);
            key2.alloc(n);
            val2.alloc(n);
            fv.alloc(n);
            rowK.alloc(n);
            rowR.alloc(n);
            const int blocks = ctx.num_sms * 16;
            k_row_ids<<<blocks, 256, 0, ctx.stream>>>(offK, W.rows[K], rowK.p);
            DBFS_LAUNCHED();
            k_row_ids<<<blocks, 256, 0, ctx.stream>>>(offR, W.rows[R], rowR.p);
            DBFS_LAUNCHED();
            // forward entries by (target, source): CSR order is by source, one stable pass by target
            k_col_keys<<<blocks, 256, 0, ctx.stream>>>(colK, n, key.p, val.p);
            DBFS_LAUNCHED();
            bool alt = false;
            radix_sort_pairs(ctx, key.p, val.p, key2.p, val2.p, n, bits_for(W.rows[R]), &alt);
            DBFS_CUDA(cudaMemcpyAsync(fv.p, alt ? val2.p : val.p, 4 * n, cudaMemcpyDeviceToDevice, ctx.stream));
            // reverse entries by (row, column): stable by column, then stable by row
            k_col_keys<<<blocks, 256, 0, ctx.stream>>>(colR, n, key.p, val.p);
            DBFS_LAUNCHED();
            radix_sort_pairs(ctx, key.p, val.p, key2.p, val2.p, n, bits_for(W.rows[K]), &alt);
            uint32_t *sv = alt ? val2.p : val.p, *kk = alt ? key.p : key2.p;  // kk: a free key buffer
            k_row_keys<<<blocks, 256, 0, ctx.stream>>>(sv, rowR.p, n, kk);
            DBFS_LAUNCHED();
            uint32_t *k3 = kk == key.p ? key2.p : key.p, *v3 = sv == val.p ? val2.p : val.p;
            bool alt2 = false;
            radix_sort_pairs(ctx, kk, sv, k3, v3, n, bits_for(W.rows[R]), &alt2);
            const uint32_t *rv = alt2 ? v3 : sv;
            W.twin[K].alloc(n);
            DBFS_CUDA(cudaMemsetAsync(bad.p, 0, 4, ctx.stream));
            k_twin_fill<<<blocks, 256, 0, ctx.stream>>>(fv.p, rv, colK, rowK.p, colR, rowR.p, offR, n, W.twin[K].p,
                                                        bad.p);
            DBFS_LAUNCHED();
            unsigned hb = 0;
            DBFS_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, ctx.stream));
            DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
            if (hb) {
                W.twin[K].release();
                continue;
            }
            W.twin_base[K] = k0;
        }
    }
}

// ------------------------------------------------------------------ exports

void export_csr(const Graph &g, int worker, int kind, int64_t *off, void *cols) {
    const WorkerHost *W = nullptr;
    for (auto &x : g.workers)
        if (x.w == worker) W = &x;
    DBFS_CHECK(W != nullptr, DBFS_EINVAL, "worker not resident in this process");
    DBFS_CHECK(kind >= 0 && kind < 4, DBFS_EINVAL, "bad kind");
    int64_t rows = W->rows[kind];
    std::vector<int64_t> h(rows + 1);
    DBFS_CUDA(cudaMemcpy(h.data(), g.off_all.p + W->base[kind], 8 * (rows + 1), cudaMemcpyDeviceToHost));
    int64_t first = h[0];
    for (int64_t i = 0; i <= rows; i++) off[i] = h[i] - first;
    int64_t nnz = h[rows] - first;
    if (nnz == 0) return;
    if (kind == KIND_NN) {
        std::vector<uint32_t> c(nnz);
        DBFS_CUDA(cudaMemcpy(c.data(), g.col_all.p + first, 4 * nnz, cudaMemcpyDeviceToHost));
        int64_t *o = (int64_t *)cols;
        for (int64_t i = 0; i < nnz; i++) o[i] = (int64_t)c[i];
    } else {
        DBFS_CUDA(cudaMemcpy(cols, g.col_all.p + first, 4 * nnz, cudaMemcpyDeviceToHost));
    }
}

void export_sources(const Graph &g, int worker, int64_t *nd_src, uint8_t *dn, uint8_t *dd) {
    const WorkerHost *W = nullptr;
    for (auto &x : g.workers)
        if (x.w == worker) W = &x;
    DBFS_CHECK(W != nullptr, DBFS_EINVAL, "worker not resident in this process");
    auto bits = [&](int k, std::vector<uint32_t> &h) {
        h.resize(std::max<int64_t>(nwords(W->rows[k]), 1));
        DBFS_CUDA(cudaMemcpy(h.data(), W->src_bits[k].p, 4 * h.size(), cudaMemcpyDeviceToHost));
    };
    std::vector<uint32_t> h;
    if (nd_src) {
        bits(KIND_ND, h);
        int64_t c = 0;
        for (int64_t r = 0; r < W->rows[KIND_ND]; r++)
            if (h[r >> 5] >> (r & 31) & 1) nd_src[c++] = r;
    }
    if (dn) {
        bits(KIND_DN, h);
        for (int64_t r = 0; r < g.d; r++) dn[r] = h[r >> 5] >> (r & 31) & 1;
    }
    if (dd) {
        bits(KIND_DD, h);
        for (int64_t r = 0; r < g.d; r++) dd[r] = h[r >> 5] >> (r & 31) & 1;
    }
}

void export_classification(const Graph &g, int64_t *deg, int64_t *del) {
    if (deg && g.n) {
        std::vector<uint32_t> h(g.n);
        DBFS_CUDA(cudaMemcpy(h.data(), g.degree.p, 4 * g.n, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < g.n; i++) deg[i] = h[i];
    }
    if (del && g.d) DBFS_CUDA(cudaMemcpy(del, g.del_gid.p, 8 * g.d, cudaMemcpyDeviceToHost));
}

}  // namespace dbfs
