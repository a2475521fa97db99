// api.cu -- the extern "C" boundary (include/dbfs.h).  Exceptions become
// dbfs_status codes; the message is kept per thread for dbfs_last_error().
#include <cstring>
#include <string>

#include "internal.h"

namespace dbfs {
std::atomic<int64_t> g_kernel_launches{0};

void *Ctx::ensure_scratch(size_t bytes) {
    if ((size_t)scratch.n < bytes) {
        scratch.alloc((int64_t)std::max<size_t>(bytes, 4096));
        DBFS_CUDA(cudaMemset(scratch.p, 0, scratch.bytes()));
    }
    return scratch.p;
}
}  // namespace dbfs

using namespace dbfs;

struct dbfs_ctx {
    Ctx c;
};
struct dbfs_graph {
    Graph g;
};

static thread_local std::string t_err;

template <typename F>
static int32_t guard(F &&f) {
    try {
        f();
        return DBFS_OK;
    } catch (const Error &e) {
        t_err = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        t_err = "host allocation failed";
        return DBFS_ENOMEM;
    } catch (const std::exception &e) {
        t_err = e.what();
        return DBFS_EINTERNAL;
    }
}

extern "C" {

const char *dbfs_last_error(void) { return t_err.c_str(); }
int32_t dbfs_abi_version(void) { return DBFS_ABI_VERSION; }
int64_t dbfs_kernel_launch_counter(void) { return g_kernel_launches.load(); }

int32_t dbfs_device_count(int32_t *out) {
    return guard([&] {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *out = n;
    });
}

int32_t dbfs_host_alloc(int64_t bytes, void **out) {
    return guard([&] {
        *out = nullptr;
        DBFS_CUDA(cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 1), cudaHostAllocDefault));
    });
}

int32_t dbfs_host_free(void *p) {
    return guard([&] {
        if (p) DBFS_CUDA(cudaFreeHost(p));
    });
}

int32_t dbfs_ctx_flush_l2(dbfs_ctx *ctx) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(ctx->c.device));
        const size_t B = (size_t)256 << 20;
        if (ctx->c.flush.n < (int64_t)B) ctx->c.flush.alloc((int64_t)B);
        DBFS_CUDA(cudaMemsetAsync(ctx->c.flush.p, ctx->c.flush_val++ & 0xff, B, ctx->c.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

int32_t dbfs_ctx_create(int32_t device, dbfs_ctx **out) {
    return guard([&] {
        *out = nullptr;
        int n = 0;
        DBFS_CUDA(cudaGetDeviceCount(&n));
        DBFS_CHECK(device >= 0 && device < n, DBFS_EINVAL, "no such CUDA device");
        auto *c = new dbfs_ctx();
        c->c.device = device;
        DBFS_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        DBFS_CUDA(cudaGetDeviceProperties(&prop, device));
        DBFS_CHECK(prop.major >= 10, DBFS_ECUDA, "libdbfs is built for sm_100a (B200)");
        c->c.num_sms = prop.multiProcessorCount;
        DBFS_CUDA(cudaStreamCreate(&c->c.stream));  // blocking: legacy-stream cudaMemcpy orders after it
        DBFS_CUDA(cudaEventCreate(&c->c.ev0));
        DBFS_CUDA(cudaEventCreate(&c->c.ev1));
        *out = c;
    });
}

int32_t dbfs_ctx_destroy(dbfs_ctx *ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->c.device);
        nccl_destroy(ctx->c);
        ctx->c.scratch.release();
        ctx->c.flush.release();
        if (ctx->c.ev0) cudaEventDestroy(ctx->c.ev0);
        if (ctx->c.ev1) cudaEventDestroy(ctx->c.ev1);
        for (int b = 0; b < 2; b++) {
            if (ctx->c.ev_ready[b]) cudaEventDestroy(ctx->c.ev_ready[b]);
            if (ctx->c.ev_done[b]) cudaEventDestroy(ctx->c.ev_done[b]);
        }
        for (int h = 0; h < 3; h++)
            if (ctx->c.ev_hdone[h]) cudaEventDestroy(ctx->c.ev_hdone[h]);
        if (ctx->c.copy_stream) cudaStreamDestroy(ctx->c.copy_stream);
        if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
        delete ctx;
    });
}

int32_t dbfs_nccl_unique_id(uint8_t *out, int64_t len) {
    return guard([&] {
        DBFS_CHECK(len >= 128, DBFS_EINVAL, "unique id buffer must hold 128 bytes");
        nccl_unique_id(out);
    });
}

int32_t dbfs_ctx_init_dist(dbfs_ctx *ctx, const uint8_t *uid, int64_t len, int32_t nranks, int32_t rank) {
    return guard([&] {
        DBFS_CHECK(len >= 128 && nranks >= 1 && rank >= 0 && rank < nranks, DBFS_EINVAL, "bad dist args");
        nccl_init(ctx->c, uid, nranks, rank);
    });
}

int32_t dbfs_ctx_init_local_group(dbfs_ctx *ctx, const uint8_t *uid, int64_t len, int32_t nranks, int32_t rank) {
    return guard([&] {
        DBFS_CHECK(len >= 128 && nranks >= 1 && rank >= 0 && rank < nranks, DBFS_EINVAL, "bad group args");
        nccl_init(ctx->c, uid, nranks, rank);
        ctx->c.local_group = 1;
    });
}

int32_t dbfs_ctx_abort(dbfs_ctx *ctx) {
    return guard([&] { nccl_abort(ctx->c); });
}

int32_t dbfs_ctx_barrier(dbfs_ctx *ctx) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(ctx->c.device));
        if (ctx->c.comm) nccl_barrier(ctx->c);
        DBFS_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

int32_t dbfs_ctx_allreduce_max_f64(dbfs_ctx *ctx, double *inout, int64_t count) {
    return guard([&] {
        if (!ctx->c.comm || count <= 0) return;
        DBFS_CUDA(cudaSetDevice(ctx->c.device));
        DArray<double> b;
        b.alloc(count);
        DBFS_CUDA(cudaMemcpy(b.p, inout, 8 * count, cudaMemcpyHostToDevice));
        nccl_allreduce_f64_max(ctx->c, b.p, count);
        DBFS_CUDA(cudaStreamSynchronize(ctx->c.stream));
        DBFS_CUDA(cudaMemcpy(inout, b.p, 8 * count, cudaMemcpyDeviceToHost));
    });
}

int32_t dbfs_ctx_allreduce_sum_i64(dbfs_ctx *ctx, int64_t *inout, int64_t count) {
    return guard([&] {
        if (!ctx->c.comm || count <= 0) return;
        DBFS_CUDA(cudaSetDevice(ctx->c.device));
        DArray<int64_t> b;
        b.alloc(count);
        DBFS_CUDA(cudaMemcpy(b.p, inout, 8 * count, cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx->c, b.p, count, 0);
        DBFS_CUDA(cudaStreamSynchronize(ctx->c.stream));
        DBFS_CUDA(cudaMemcpy(inout, b.p, 8 * count, cudaMemcpyDeviceToHost));
    });
}

int32_t dbfs_rmat_generate(dbfs_ctx *ctx, const dbfs_rmat_params *params, int64_t begin, int64_t end,
                           int64_t *src_out, int64_t *dst_out) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(ctx->c.device));
        rmat_generate_host(ctx->c, *params, begin, end, src_out, dst_out);
    });
}

int32_t dbfs_hash_vertices(dbfs_ctx *ctx, int64_t n, uint64_t seed, const int64_t *ids_in, int64_t *ids_out,
                           int64_t count) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(ctx->c.device));
        hash_vertices_host(ctx->c, n, seed, ids_in, ids_out, count);
    });
}

static void init_graph(Graph &g, dbfs_ctx *ctx, int64_t theta, int32_t p_rank, int32_t p_gpu) {
    DBFS_CHECK(theta >= 0, DBFS_EINVAL, "theta must be >= 0");
    DBFS_CHECK(p_rank >= 1 && p_gpu >= 1, DBFS_EINVAL, "p_rank and p_gpu must be positive");
    g.ctx = &ctx->c;
    g.theta = theta;
    g.p_rank = p_rank;
    g.p_gpu = p_gpu;
    g.p = p_rank * p_gpu;
    DBFS_CHECK(g.p <= MAXW, DBFS_EINVAL, "at most 64 workers");
    g.dist = ctx->c.comm != nullptr && ctx->c.nranks > 1;
    if (g.dist) DBFS_CHECK(g.p == ctx->c.nranks, DBFS_EINVAL, "distributed graphs need p == number of ranks");
    DBFS_CUDA(cudaSetDevice(ctx->c.device));
}

int32_t dbfs_graph_build_rmat(dbfs_ctx *ctx, const dbfs_rmat_params *params, int64_t theta, int32_t p_rank,
                              int32_t p_gpu, dbfs_graph **out) {
    *out = nullptr;
    dbfs_graph *g = new dbfs_graph();
    int32_t rc = guard([&] {
        init_graph(g->g, ctx, theta, p_rank, p_gpu);
        build_graph_rmat(g->g, *params);
        g->g.symmetric = params->symmetrize != 0;
    });
    if (rc) delete g;
    else *out = g;
    return rc;
}

int32_t dbfs_graph_build_edges(dbfs_ctx *ctx, const int64_t *src, const int64_t *dst, int64_t m, int64_t n,
                               int64_t theta, int32_t p_rank, int32_t p_gpu, dbfs_graph **out) {
    *out = nullptr;
    dbfs_graph *g = new dbfs_graph();
    int32_t rc = guard([&] {
        init_graph(g->g, ctx, theta, p_rank, p_gpu);
        g->g.n = n;
        build_graph_edges(g->g, src, dst, m);
    });
    if (rc) delete g;
    else *out = g;
    return rc;
}

int32_t dbfs_graph_upload_partitioned(dbfs_ctx *ctx, int64_t n, int64_t m, int64_t theta, int32_t p_rank,
                                      int32_t p_gpu, int64_t d, const int64_t *delegate_global_ids,
                                      const int64_t *out_degree, const int64_t *const *row_offsets,
                                      const void *const *col_indices, int32_t symmetric, dbfs_graph **out) {
    *out = nullptr;
    dbfs_graph *g = new dbfs_graph();
    int32_t rc = guard([&] {
        DBFS_CHECK(n >= 0 && m >= 0 && d >= 0 && d <= n && out_degree && row_offsets && col_indices &&
                       (delegate_global_ids || d == 0),
                   DBFS_EINVAL, "bad arguments");
        init_graph(g->g, ctx, theta, p_rank, p_gpu);
        g->g.n = n;
        g->g.m = m;
        g->g.d = d;
        upload_partitioned(g->g, out_degree, delegate_global_ids, row_offsets, col_indices);
        g->g.symmetric = symmetric != 0;
    });
    if (rc) delete g;
    else *out = g;
    return rc;
}

int32_t dbfs_graph_nvls_active(const dbfs_graph *g) { return g && g->g.nvls ? 1 : 0; }

int32_t dbfs_graph_free(dbfs_graph *g) {
    return guard([&] {
        if (!g) return;
        cudaSetDevice(g->g.ctx->device);
        delete g;
    });
}

int32_t dbfs_graph_set_symmetric(dbfs_graph *g, int32_t symmetric) {
    return guard([&] { g->g.symmetric = symmetric != 0; });
}

int32_t dbfs_graph_info_get(const dbfs_graph *gg, dbfs_graph_info *out) {
    return guard([&] {
        const Graph &g = gg->g;
        memset(out, 0, sizeof(*out));
        out->n = g.n;
        out->m = g.m;
        out->d = g.d;
        out->theta = g.theta;
        out->p_rank = g.p_rank;
        out->p_gpu = g.p_gpu;
        out->p = g.p;
        out->nranks = g.ctx->nranks;
        out->rank = g.ctx->rank;
        out->n_local_workers = (int32_t)g.workers.size();
        out->first_worker = g.workers.empty() ? 0 : g.workers[0].w;
        for (int k = 0; k < 4; k++) out->kind_totals[k] = g.kind_totals[k];
        int64_t b = g.degree.bytes() + g.del_id.bytes() + g.del_gid.bytes() + g.off_all.bytes() + g.col_all.bytes();
        for (auto &W : g.workers)
            for (int k = 0; k < 4; k++) b += W.src_bits[k].bytes();
        out->device_bytes = b;
    });
}

int32_t dbfs_graph_worker_info(const dbfs_graph *gg, int32_t worker, int64_t *n_local, int64_t *rows, int64_t *nnz,
                               int64_t *n_nd_src) {
    return guard([&] {
        const Graph &g = gg->g;
        const WorkerHost *W = nullptr;
        for (auto &x : g.workers)
            if (x.w == worker) W = &x;
        DBFS_CHECK(W != nullptr, DBFS_EINVAL, "worker not resident in this process");
        if (n_local) *n_local = W->n_local;
        for (int k = 0; k < 4; k++) {
            if (rows) rows[k] = W->rows[k];
            if (nnz) nnz[k] = W->nnz[k];
        }
        if (n_nd_src) *n_nd_src = W->n_src[KIND_ND];
    });
}

int32_t dbfs_graph_export_csr(const dbfs_graph *gg, int32_t worker, int32_t kind, int64_t *row_offsets,
                              void *col_indices) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(gg->g.ctx->device));
        export_csr(gg->g, worker, kind, row_offsets, col_indices);
    });
}

int32_t dbfs_graph_export_sources(const dbfs_graph *gg, int32_t worker, int64_t *nd_source_list,
                                  uint8_t *dn_source_mask, uint8_t *dd_source_mask) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(gg->g.ctx->device));
        export_sources(gg->g, worker, nd_source_list, dn_source_mask, dd_source_mask);
    });
}

int32_t dbfs_graph_export_classification(const dbfs_graph *gg, int64_t *out_degree, int64_t *delegate_global_ids) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(gg->g.ctx->device));
        export_classification(gg->g, out_degree, delegate_global_ids);
    });
}

int32_t dbfs_bfs(dbfs_graph *gg, const dbfs_bfs_options *opts, int32_t *levels_out, int64_t *parents_out,
                 dbfs_run_stats *stats) {
    return guard([&] {
        Graph &g = gg->g;
        DBFS_CUDA(cudaSetDevice(g.ctx->device));
        run_bfs(g, *opts, stats);
        if (levels_out || parents_out) fetch_result(g, levels_out, parents_out);
        if (stats) stats->d2h_bytes += (levels_out ? 4 * g.n : 0) + (parents_out ? 8 * g.n : 0);
    });
}

int32_t dbfs_bfs_batch(dbfs_graph *gg, const dbfs_bfs_options *opts, const int64_t *roots, int64_t count,
                       int32_t *const *levels_out, int64_t *const *parents_out, int32_t local, int32_t compact,
                       dbfs_run_stats *stats) {
    return guard([&] {
        DBFS_CHECK(opts && count >= 0 && (roots || count == 0), DBFS_EINVAL, "bad arguments");
        Graph &g = gg->g;
        DBFS_CUDA(cudaSetDevice(g.ctx->device));
        run_bfs_batch(g, *opts, roots, count, levels_out, parents_out, local, compact, stats);
    });
}

int32_t dbfs_bfs_batch_output_count(const dbfs_graph *gg, int32_t local, int64_t *count) {
    return guard([&] { *count = batch_output_count(gg->g, local != 0); });
}

int32_t dbfs_fetch_result(dbfs_graph *gg, int32_t *levels_out, int64_t *parents_out) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(gg->g.ctx->device));
        fetch_result(gg->g, levels_out, parents_out);
    });
}

int32_t dbfs_bfs_iteration(const dbfs_graph *gg, int64_t it, dbfs_iteration *rec, int8_t *directions, double *bv) {
    return guard([&] {
        const Graph &g = gg->g;
        DBFS_CHECK(g.last_valid, DBFS_EINVAL, "no BFS has run");
        int64_t nrec = (int64_t)g.last_rec.size() / std::max(g.W, 1);
        DBFS_CHECK(it >= 0 && it < nrec, DBFS_ERANGE, "iteration out of range (or truncated)");
        iteration_summary(g, &g.last_rec[(size_t)it * g.W], it, g.last_la, g.last_uq, rec, directions, bv);
    });
}

int32_t dbfs_bfs_iteration_sends(const dbfs_graph *gg, int64_t it, int64_t *out) {
    return guard([&] {
        const Graph &g = gg->g;
        DBFS_CHECK(g.last_valid, DBFS_EINVAL, "no BFS has run");
        int64_t nrec = (int64_t)g.last_rec.size() / std::max(g.W, 1);
        DBFS_CHECK(it >= 0 && it < nrec, DBFS_ERANGE, "iteration out of range (or truncated)");
        for (int i = 0; i < g.W; i++)
            for (int o = 0; o < g.p; o++)
                out[(size_t)i * g.p + o] = (int64_t)g.last_rec[(size_t)it * g.W + i].send[o];
    });
}

int32_t dbfs_min_parents(dbfs_graph *gg, int64_t *parents_out) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(gg->g.ctx->device));
        min_parents(gg->g, parents_out);
    });
}

int32_t dbfs_validate(dbfs_graph *gg, int64_t root, const int32_t *levels, const int64_t *parents, int32_t *report) {
    return guard([&] {
        DBFS_CUDA(cudaSetDevice(gg->g.ctx->device));
        *report = validate(gg->g, root, levels, parents);
    });
}

int32_t dbfs_edges_text_capacity(const char *buf, int64_t len, int64_t *lines) {
    return guard([&] {
        DBFS_CHECK(len >= 0 && (buf || !len) && lines, DBFS_EINVAL, "bad buffer");
        *lines = count_text_lines(buf, len);
    });
}

int32_t dbfs_edges_parse_text(const char *buf, int64_t len, int64_t cap, int64_t *src, int64_t *dst,
                              int64_t *m_out, int64_t *header_n) {
    return guard([&] {
        DBFS_CHECK(len >= 0 && (buf || !len) && m_out && header_n, DBFS_EINVAL, "bad buffer");
        parse_edge_text(buf, len, cap, src, dst, m_out, header_n);
    });
}

int32_t dbfs_edges_write_text(const char *path, int64_t n, const int64_t *src, const int64_t *dst, int64_t m) {
    return guard([&] {
        DBFS_CHECK(path && m >= 0 && (m == 0 || (src && dst)), DBFS_EINVAL, "bad arguments");
        write_edge_text(path, n, src, dst, m);
    });
}

}  // extern "C"
