/*
 * dbfs.h -- C ABI of libdbfs.so, the B200 (sm_100a) delegate-BFS engine.
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 * The library owns all device memory; callers own host buffers.  Every entry
 * point returns a dbfs_status; dbfs_last_error() gives the message of the
 * last failure on the calling thread.
 *
 * The reference (/root/reference/pkg/src/delegate_bfs) is pure Python with no
 * FFI; these entry points replace the bodies of its public functions (the
 * Python shell in paper_1803_03922_b200/ keeps the reference signatures and
 * maps statuses onto the reference exception types):
 *
 *   dbfs_rmat_generate        <- rmat.generate_rmat / build_rmat_graph   (rmat.py:125-208)
 *   dbfs_graph_build_rmat     <- partition_graph(build_rmat_graph(...))  (partition.py:343-351)
 *   dbfs_graph_build_edges    <- partition_graph(EdgeList, theta, shape) (partition.py:343-351)
 *   dbfs_graph_upload_partitioned <- a reference PartitionedGraph as is    (partition.py:263-292)
 *   dbfs_graph_export_*       <- PartitionedGraph / WorkerGraph fields    (partition.py:263-292)
 *   dbfs_bfs                  <- engine.run_bfs                           (engine.py:98-330)
 *   dbfs_bfs_batch            <- engine.benchmark's per-source loop       (engine.py:333-364)
 *   dbfs_bfs_iteration        <- BfsRun.per_iteration records             (engine.py:291-302)
 *   dbfs_validate             <- NEW: Graph500 certificate (nearest
 *                                reference analogue is cli.cmd_verify, cli.py:159-174)
 *   dbfs_min_parents          <- NEW: min-ID parent rule
 *   dbfs_edges_parse_text     <- rmat.load_edge_list, text format         (rmat.py:232-286)
 *   dbfs_edges_write_text     <- rmat.save_edge_list, text format         (rmat.py:211-229)
 */
#ifndef DBFS_H
#define DBFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBFS_ABI_VERSION 1

typedef enum {
    DBFS_OK = 0,
    DBFS_EINVAL = 1,     /* ValueError (bad argument / mode / theta)            */
    DBFS_ERANGE = 2,     /* ValueError("source ... out of range"), engine.py:105 */
    DBFS_ECAPACITY = 3,  /* CapacityError, partition.py:308-309                  */
    DBFS_ERESOURCE = 4,  /* ResourceError, rmat.py:58-61 / device memory         */
    DBFS_ENOMEM = 5,     /* host or device allocation failed                     */
    DBFS_ECUDA = 6,      /* CUDA runtime error                                   */
    DBFS_ENCCL = 7,      /* NCCL error                                           */
    DBFS_EROUTING = 8,   /* RoutingError, comm.py:16-17                          */
    DBFS_ESTRUCT = 9,    /* StructuralError, comm.py:20-21                       */
    DBFS_ETIMEOUT = 10,  /* device watchdog fired (grid barrier)                 */
    DBFS_EINTERNAL = 11,
    DBFS_EFORMAT = 12,   /* FormatError, rmat.py:35-36 (malformed edge-list file) */
    DBFS_EIO = 13        /* OSError (file could not be opened / written)          */
} dbfs_status;

typedef struct dbfs_ctx dbfs_ctx;
typedef struct dbfs_graph dbfs_graph;

/* RmatParams (rmat.py:39-69) plus build_rmat_graph switches (rmat.py:200). */
typedef struct {
    int32_t scale;
    int32_t randomize;   /* hash_randomize_vertices(g, seed) */
    int32_t symmetrize;  /* symmetrize(g) */
    int32_t scramble;    /* this build: Feistel relabeling after the hash (balanced v mod p owners) */
    int64_t edge_factor;
    double a, b, c;      /* d = 1 - a - b - c */
    uint64_t seed;
} dbfs_rmat_params;

typedef struct {
    int64_t n, m, d, theta;
    int32_t p_rank, p_gpu, p;   /* ClusterShape (partition.py:47-76) */
    int32_t nranks, rank;       /* processes sharing the graph (1 unless NCCL) */
    int32_t n_local_workers;    /* workers resident in this process */
    int32_t first_worker;       /* global index of the first local worker */
    int32_t _pad;
    int64_t kind_totals[4];     /* nn, nd, dn, dd (partition.py:312-318) */
    int64_t device_bytes;       /* resident device bytes of the graph */
} dbfs_graph_info;

/* BfsOptions (engine.py:33-46) + parent / engine switches. */
typedef struct {
    int32_t mode;               /* 0 = "bfs", 1 = "dobfs" */
    int32_t allow_switch_back;
    int64_t source;
    double factor0[4];          /* indexed nn, nd, dn, dd (nn unused) */
    double factor1[4];
    int32_t local_all2all;      /* accounting only (comm.py:138-197) */
    int32_t uniquify;           /* accounting only */
    int32_t parent_mode;        /* 0 none, 1 any valid tree (timed), 2 min-ID tree (computed on device after
                                   the timed traversal; dbfs_bfs_batch: single-process graphs only) */
    int32_t engine;             /* 0 auto, 1 host-driven level loop, 2 persistent kernel, 3 peer (multi-GPU persistent over CUDA IPC) */
    int32_t record_iterations;  /* keep per-iteration records for dbfs_bfs_iteration */
    int32_t exec_policy;        /* 1: on symmetric graphs in dobfs mode, execute a FORWARD-reported
                                   kind as the equivalent pull, or a BACKWARD-reported kind as a
                                   counting push (twin positions recover the pull's early-exit
                                   counters), when cheaper -- reported directions and counters
                                   unchanged; 2: counting push wherever possible (tests);
                                   0: execute exactly the reported directions */
} dbfs_bfs_options;

typedef struct {
    int64_t iterations;         /* BfsRun.iterations */
    int64_t inspections[4][2];  /* [kind][forward, backward] (engine.py:143) */
    double b_measured;          /* engine.py:316-318 */
    double device_ms;           /* CUDA-event time of the traversal on device */
    int64_t reached;            /* vertices with level >= 0 */
    int64_t kernel_launches;    /* kernels launched by this call */
    int64_t wire_bytes;         /* bytes actually moved between workers */
    int64_t h2d_bytes;          /* host->device bytes copied by this call */
    int64_t d2h_bytes;          /* device->host bytes copied by this call */
    int64_t rows_touched;       /* CSR rows expanded (push) or scanned (pull), all levels */
    double init_us;             /* device time of state init + seeding */
    int64_t work_inspections;   /* inspections actually executed (<= reported when pulls replace pushes) */
    int32_t per_iteration_truncated;
    int32_t engine_used;        /* 1 host loop, 2 persistent, 3 peer */
    double total_mask_bytes;    /* CommStats.total_mask_bytes (comm.py:39-72): sum over iterations */
    int64_t total_normal_bytes; /* CommStats.total_normal_bytes */
    int64_t s_prime;            /* CommStats.s_prime: iterations with a mask reduction */
    int32_t accounting_valid;   /* 1 when the four fields above and inspections cover every iteration */
    int32_t _pad;
} dbfs_run_stats;

/* One BfsRun.per_iteration entry summed over workers (engine.py:291-302). */
typedef struct {
    int64_t iteration;
    int64_t inspections[4];
    int64_t fv[4];
    double mask_bytes;
    int64_t normal_bytes;
    int64_t message_count;
    int64_t pair_count;
    int64_t frontier_normals;   /* normals at this level (all workers) */
    int64_t frontier_delegates; /* delegates at this level */
    int64_t work[4];            /* executed inspections per kind */
    int32_t exec_dirs[4];       /* executed strategy per kind on worker 0 (0 push, 1 pull) */
    double task_avg_us[8];      /* worker 0 per-task mean warp time (T1 normal push, T2 dn push, T2 dd push,
                                   T4 dn pull, T5 nd pull, T6 dd pull, F delegates, F normals) */
    double task_max_us[8];      /* worker 0 per-task max warp time */
    double visit_us;            /* device time of the visit phase (worker 0's clock) */
    double finish_us;           /* device time of the barrier/apply phase */
    double sync_us[4];          /* persistent engines: visit compute (to the last local block), visit cross-GPU
                                   barrier wait, finish compute, finish cross-GPU wait */
    double comm_us;             /* NCCL level loop (engine 1): measured device time of the level's exchange
                                   (delegate-mask all-gather + record all-to-all), else 0 */
} dbfs_iteration;

const char *dbfs_last_error(void);
int32_t dbfs_abi_version(void);
int32_t dbfs_device_count(int32_t *out);
int64_t dbfs_kernel_launch_counter(void);

/* Pinned (page-locked) host buffers for zero-staging D2H of results. */
int32_t dbfs_host_alloc(int64_t bytes, void **out);
int32_t dbfs_host_free(void *p);

/* Contexts: one device + stream; optionally an NCCL communicator (one rank per process). */
int32_t dbfs_ctx_create(int32_t device, dbfs_ctx **out);
int32_t dbfs_ctx_destroy(dbfs_ctx *ctx);
int32_t dbfs_nccl_unique_id(uint8_t *out, int64_t len);       /* len >= 128 */
int32_t dbfs_ctx_init_dist(dbfs_ctx *ctx, const uint8_t *uid, int64_t len, int32_t nranks, int32_t rank);
/* One worker per GPU inside ONE process (the reference's ClusterShape(1, P)
 * partition_graph in one process, partition.py:47-76 / engine.py:149-164): each
 * rank is a host thread driving its own context; like dbfs_ctx_init_dist, but
 * the peers' arrays are mapped by pointer with peer access instead of CUDA IPC. */
int32_t dbfs_ctx_init_local_group(dbfs_ctx *ctx, const uint8_t *uid, int64_t len, int32_t nranks, int32_t rank);
/* Abort the context's NCCL communicator (another rank of a device group failed):
 * collectives pending on it return; the context keeps its device but no comm. */
int32_t dbfs_ctx_abort(dbfs_ctx *ctx);
int32_t dbfs_ctx_barrier(dbfs_ctx *ctx);
int32_t dbfs_ctx_flush_l2(dbfs_ctx *ctx);                     /* write 256 MB on the ctx stream, sync */                      /* NCCL all-reduce barrier + stream sync */
int32_t dbfs_ctx_allreduce_max_f64(dbfs_ctx *ctx, double *inout, int64_t count);
int32_t dbfs_ctx_allreduce_sum_i64(dbfs_ctx *ctx, int64_t *inout, int64_t count);

/* Edge generation on device, copied to host: edges [begin, end) of build_rmat_graph. */
int32_t dbfs_rmat_generate(dbfs_ctx *ctx, const dbfs_rmat_params *params, int64_t begin, int64_t end,
                           int64_t *src_out, int64_t *dst_out);

/* hash_randomize_vertices (rmat.py:153-182) on an id array; n must be a power of two. */
int32_t dbfs_hash_vertices(dbfs_ctx *ctx, int64_t n, uint64_t seed, const int64_t *ids_in, int64_t *ids_out,
                           int64_t count);

/* Graph build.  Single-process contexts build all p = p_rank*p_gpu workers on the
 * context's device.  Distributed contexts (nranks > 1) require p == nranks; rank r
 * builds worker r, and for build_edges passes the r-th contiguous slice of the edge list. */
int32_t dbfs_graph_build_rmat(dbfs_ctx *ctx, const dbfs_rmat_params *params, int64_t theta,
                              int32_t p_rank, int32_t p_gpu, dbfs_graph **out);
int32_t dbfs_graph_build_edges(dbfs_ctx *ctx, const int64_t *src, const int64_t *dst, int64_t m,
                               int64_t n, int64_t theta, int32_t p_rank, int32_t p_gpu,
                               dbfs_graph **out);
/* A partition built elsewhere -- the reference's PartitionedGraph
 * (partition.py:263-292), e.g. from its partition_graph or load_partitioned_graph
 * (partition.py:343-351, 424-464) -- uploaded as is (single process, the p
 * workers on this device): for worker w and kind k in (nn, nd, dn, dd),
 * row_offsets[w*4+k] is int64[rows+1] (rows = n_local(w) for nn/nd, d for
 * dn/dd) and col_indices[w*4+k] is int64 (nn) or uint32 (others), the
 * reference's CsrSubgraph arrays; out_degree int64[n] and the ascending
 * delegate_global_ids int64[d] are the VertexClassification.  Rows keep their
 * neighbour order (the BFS counters depend on it).  symmetric: every edge's
 * reverse is present (graphs from build_rmat_graph with symmetrize). */
int32_t dbfs_graph_upload_partitioned(dbfs_ctx *ctx, int64_t n, int64_t m, int64_t theta, int32_t p_rank,
                                      int32_t p_gpu, int64_t d, const int64_t *delegate_global_ids,
                                      const int64_t *out_degree, const int64_t *const *row_offsets,
                                      const void *const *col_indices, int32_t symmetric, dbfs_graph **out);
/* 1 when the peer engine ORs the delegate masks through an NVSwitch multicast
 * object (DBFS_NVLS=1 in a device group, nvls.cu), else 0. */
int32_t dbfs_graph_nvls_active(const dbfs_graph *g);
int32_t dbfs_graph_free(dbfs_graph *g);
/* Declare the edge multiset symmetric (every (u,v) has its (v,u)); RMAT builds with
 * symmetrize set are symmetric by construction. */
int32_t dbfs_graph_set_symmetric(dbfs_graph *g, int32_t symmetric);
int32_t dbfs_graph_info_get(const dbfs_graph *g, dbfs_graph_info *out);
/* rows[4], nnz[4] of a local worker's nn/nd/dn/dd CSRs; n_nd_src = len(nd_source_list). */
int32_t dbfs_graph_worker_info(const dbfs_graph *g, int32_t worker, int64_t *n_local, int64_t *rows,
                               int64_t *nnz, int64_t *n_nd_src);
/* row_offsets: int64[rows+1]; col_indices: int64[nnz] for nn, uint32[nnz] otherwise. */
int32_t dbfs_graph_export_csr(const dbfs_graph *g, int32_t worker, int32_t kind, int64_t *row_offsets,
                              void *col_indices);
int32_t dbfs_graph_export_sources(const dbfs_graph *g, int32_t worker, int64_t *nd_source_list,
                                  uint8_t *dn_source_mask, uint8_t *dd_source_mask);
/* out_degree: int64[n] (nullable); delegate_global_ids: int64[d] (nullable). */
int32_t dbfs_graph_export_classification(const dbfs_graph *g, int64_t *out_degree,
                                         int64_t *delegate_global_ids);

/* One BFS.  levels_out int32[n] / parents_out int64[n] are host buffers (nullable:
 * results then stay on device for dbfs_fetch_result).  In distributed contexts every
 * rank calls it; outputs are gathered on every rank. */
int32_t dbfs_bfs(dbfs_graph *g, const dbfs_bfs_options *opts, int32_t *levels_out,
                 int64_t *parents_out, dbfs_run_stats *stats);
int32_t dbfs_fetch_result(dbfs_graph *g, int32_t *levels_out, int64_t *parents_out);
/* Many roots in one call (benchmark(), Graph500's 64-root loop): root k's depth and
 * parent arrays land in levels_out[k] / parents_out[k] (host, pinned for overlap; the
 * arrays of pointers and any entry may be NULL).  The D2H of root k runs on a copy
 * stream while root k+1 traverses.  local != 0 in a distributed context: each rank
 * receives only the vertices it owns (v mod p == rank, output i = vertex rank + i*p),
 * the distributed Graph500 result; otherwise every rank gets all n.  compact != 0:
 * the depth travels as int8 (9 instead of 12 bytes per vertex over PCIe; n < 2^31)
 * and the host widens it into the caller's array on every core while later roots
 * run; a root with a depth >= 127 is re-run with full arrays.
 * Per-iteration records are not kept.  stats (nullable) receives count entries. */
int32_t dbfs_bfs_batch(dbfs_graph *g, const dbfs_bfs_options *opts, const int64_t *roots, int64_t count,
                       int32_t *const *levels_out, int64_t *const *parents_out, int32_t local, int32_t compact,
                       dbfs_run_stats *stats);
/* Entries per output array of dbfs_bfs_batch (n, or this rank's own count when local). */
int32_t dbfs_bfs_batch_output_count(const dbfs_graph *g, int32_t local, int64_t *count);
/* Per-iteration record `it` of the last dbfs_bfs; directions int8[p*4] (0 fwd, 1 bwd) and
 * bv double[p*4] (inf = None) are per worker (both nullable). */
int32_t dbfs_bfs_iteration(const dbfs_graph *g, int64_t it, dbfs_iteration *rec, int8_t *directions,
                           double *bv);
/* Min-ID parents from the last run's levels, computed on device. */
/* Send flags of iteration `it` of the last BFS: out[i * p + o] != 0 when local
 * worker i sent >= 1 normal record to worker o (comm.py:138-197 message
 * accounting across one-worker-per-GPU ranks). */
int32_t dbfs_bfs_iteration_sends(const dbfs_graph *g, int64_t it, int64_t *out);
int32_t dbfs_min_parents(dbfs_graph *g, int64_t *parents_out);
/* Graph500 certificate over the partitioned edges for the last run's
 * device-resident levels/parents, or for host arrays when given.  *report = 0 when valid,
 * else a bitmask: 1 root, 2 edge spans >1 level, 4 reached-unreached edge,
 * 8 parent level, 16 tree edge missing, 32 parent of unreached / missing parent. */
int32_t dbfs_validate(dbfs_graph *g, int64_t root, const int32_t *levels, const int64_t *parents,
                      int32_t *report);

/* Edge-list text files (rmat.py:211-286).  Host-only, no device.
 * dbfs_edges_text_capacity: upper bound on the edge count of a buffer (its line count).
 * dbfs_edges_parse_text: "u v" lines, '#' comments, "# n <count>" header (*header_n = -1
 * when absent); DBFS_EFORMAT with "<line>: ..." on a malformed line.  Ids are not range
 * checked here (the caller checks them against n, as load_edge_list does). */
int32_t dbfs_edges_text_capacity(const char *buf, int64_t len, int64_t *lines);
int32_t dbfs_edges_parse_text(const char *buf, int64_t len, int64_t cap, int64_t *src, int64_t *dst,
                              int64_t *m_out, int64_t *header_n);
/* Writes "# n <n>" then one "u v" line per edge (DBFS_EIO on failure). */
int32_t dbfs_edges_write_text(const char *path, int64_t n, const int64_t *src, const int64_t *dst, int64_t m);

#ifdef __cplusplus
}
#endif
#endif /* DBFS_H */
