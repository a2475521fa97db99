// internal.h -- host/device data structures of libdbfs.
//
// Layout in HBM (per worker w, all on the worker's device):
//   CSR  : one concatenated int64 offset array and one uint32 column array for
//          all local workers and kinds (nn | nd | dn | dd rows per worker).  A
//          kind's offsets are absolute positions into the column array, so the
//          kernels never rebase.  nn columns are global vertex ids (uint32; the
//          reference's int64 ids are restored on export), nd/dd columns are
//          delegate ids, dn columns are local normal ids (partition.py:319-326).
//   state: int32 level + int64 parent per local normal (the global arrays when
//          p == 1), int32 level + int64 parent per delegate, bitmaps
//          (1 bit/vertex) for visited / frontier / next-frontier of normals and
//          delegates, double-buffered by level parity.
#pragma once
#include <vector>

#include "common.cuh"

namespace dbfs {

// Parent ids on the device: global vertex ids as int32 (n < 2^31, checked
// when the BFS resources are set up), widened to the reference's int64 only
// where results leave the device (fetch, batch staging, validation of
// caller arrays).  Half the footprint of int64 parents keeps the scattered
// claim-time parent stores inside L2.
using parent_t = int32_t;
constexpr parent_t PARENT_MAX = 0x7fffffff;

// Per-level counters of one worker.  Slot L%3 holds the stats of the frontier
// at level L (accumulated while level L-1 ran) and the activity of level L.
struct LevelSlot {
    unsigned long long fv[4];        // FV per kind of this level's frontier (traversal.py:72)
    unsigned long long q[4];         // |queue| per kind (previsit queue sizes)
    unsigned long long nfront;       // normals in the frontier
    unsigned long long dfront;       // delegates in the frontier
    unsigned long long dpack[2];     // delegate frontier lists (dn, dd): count << View::dshift | edges
    unsigned long long insp_bwd[4];  // backward inspections at this level
    unsigned long long records;      // remote normal records sent at this level
    unsigned long long dirty;        // this worker found >= 1 new delegate (comm.py:33-36)
    unsigned long long prev_dirty;   // copy of level L-1's `dirty` (set at V(L)): dnext[(L+1)&1] may hold bits
    unsigned long long new_del;      // delegates discovered at the barrier
    unsigned long long inbox;        // records delivered to this worker
    unsigned long long pull_rows;    // reverse rows scanned by pulls at this level
    unsigned long long uq_records;   // records left after per-group uniquify (comm.py:122-127)
    unsigned long long light;        // light level: normal claims mark the touch bitmap (F folds touched chunks)
    unsigned long long prev_light;   // level L-1 was light: frontier L's chunk list is complete
    unsigned long long nchunks;      // chunks listed for this level's frontier (claims of a light level L-1)
    unsigned long long work[4];      // inspections actually executed (push: FV, pull: scanned)
    int exec_dir[4];                 // executed strategy per kind (may differ from the reported one)
    double bv[4];                    // BV per kind as the direction rule saw it (for the record)
    unsigned long long tsum[8];      // per-task warp cycles: sum over warps (T1,T2dn,T2dd,T4,T5,T6,F1,F3)
    unsigned long long tmax[8];      // per-task warp cycles: max over warps
    unsigned int sched[8];           // dynamic chunk counters: T1, T4, T6, T5, F1, F3
    unsigned long long send[MAXW];   // 1 if >= 1 record went to this destination (reference message count)
    unsigned long long sent[MAXW];   // records actually shipped (after the sender's once-per-BFS filter)
};

struct Ctl {
    LevelSlot s[3];
    int dir[2][4];                   // sticky DirectionState by level parity
    unsigned long long cumq[2][4];   // visited source counts through the level, by parity
    unsigned long long cumfv[2][4];  // sum of FV[k] over frontiers 0..L (row lengths of visited sources), by parity
    unsigned int bar_count, bar_gen; // grid barrier (persistent engine)
    unsigned int abort;              // watchdog / error flag
    int last_level;                  // iterations when the loop ended
    unsigned long long t_start, t_seeded;  // globaltimer: kernel start, after init+seed
    int cont;                        // persistent engine: termination rule of the last level (1 = go on)
    int rec_level;                   // persistent engine: last level whose record a block claimed (CAS)
};

// Per worker per level record (BfsRun.per_iteration before summing workers).
struct IterRec {
    int dir[4];
    double bv[4];
    unsigned long long fv[4];
    unsigned long long insp[4];
    unsigned long long records;
    unsigned long long dirty;
    unsigned long long messages;
    unsigned long long new_del;
    unsigned long long rows;         // rows expanded (push) + scanned (pull)
    unsigned long long uq_records;
    unsigned long long work[4];      // executed inspections
    int exec_dir[4];
    unsigned long long tsum[8], tmax[8];
    unsigned long long nfront, dfront;
    unsigned long long t[3];         // globaltimer at V start, V end, F end (persistent engine)
    unsigned long long tb[4];        // last arriver at the V / F barriers: all local blocks in, all GPUs in
    unsigned long long send[MAXW];
};

// Device-visible description of one worker (lives in device memory).
struct alignas(16) View {
    int w, W, p, p_rank, dist;       // global index, local worker count, shape
    int mode, allow_back, parents;
    int symmetric, exec_policy;      // executor may pull a FORWARD-reported kind (dobfs, symmetric graphs)
    int uniquify, local_all2all;     // comm accounting options (comm.py:138-197)
    uint32_t *uq_all[MAXW];          // per destination worker: [p staging groups][nw_n] seen-bits
    uint32_t *uq;                    // this worker's seen-bits (cleared in F)
    int64_t n_local_of_w[MAXW];      // local normal count of every worker
    const int64_t *recv_off;         // dist: first inbox index of each source rank (p+1)
    int peer;                        // dist over CUDA IPC: peers' arrays mapped, one persistent launch
    int dshift;                      // packed delegate lists: edge-count bits (count above them)
    uint32_t *sent;                  // dist: global ids already shipped to their owner this BFS (nullptr = off)
    int64_t nw_g;                    // words of `sent`
    int64_t seg_off[MAXW];           // peer: inbox segment of each source rank
    int cand_all;                    // all workers' delegate candidates readable
    int P_sources;                   // mask sources for the OR
    int rec_cap;
    int t1_dyn_min;                  // T1 claims chunks dynamically above this many pushed edges per bitmap word
    int f3_dyn;                      // F3 claims chunks dynamically on heavy levels (0: static stride)
    int pull_dyn_min;                // pulls claim chunks dynamically above this many candidates per warp
    PDiv pd;
    int64_t n, n_local, d, nw_n, nw_d;
    double f0[4], f1[4];
    unsigned long long total_src[4]; // |nd_src|, |dn_src|, |dd_src| (index by kind)
    unsigned long long nnz[4];       // edges per kind on this worker
    const int64_t *off[4];
    const uint32_t *col[4];
    const uint32_t *src_bits[4];     // rows present: [NN]/[ND] per local normal, [DN]/[DD] per delegate
    const uint32_t *deg[4];          // row lengths ([ND], [DN], [DD])
    const uint32_t *col_sorted_dd;   // dd rows reordered by neighbour degree (executor pulls only)
    const uint32_t *head[4];         // first column of every row of the kind (pull first probes; nullptr: none)
    const uint32_t *head_sorted_dd;  // first column of every sorted dd row
    const uint32_t *twin[4];         // indexed by absolute entry position (nullptr: kind has no twins)
    uint32_t *first[4];              // counting pushes: ND/DD per delegate, DN per local normal
    const int64_t *del_gid;
    const uint32_t *del_gid32;       // the same ids as uint32 (n < 2^31): half the footprint for device lookups
    int32_t *nlevel;
    parent_t *nparent;
    int32_t *dlevel;
    parent_t *dparent;
    parent_t *dcand;
    uint32_t *nvis, *nfront[2], *dvis, *dfront, *dnext[2];
    uint32_t *nseen, *dseen;         // visited(<= L) + claims of level L: the push's single test
    uint32_t *ntouch[2];             // by level parity: 1 bit per 32-word chunk holding frontier normals
    uint32_t *nchunk_list[2];        // by level parity: those chunks, listed by the claims of a light level
    int64_t ntw;                     // words of one touch bitmap
    uint32_t *nseen_all[MAXW];       // in-process: peers' seen bits (direct remote claims)
    uint32_t *coarse_d[2], *coarse_n[2];  // coarse frontier filters by level parity
    uint32_t *dlist[2][2];           // delegate frontier per push kind (0 dn, 1 dd) and parity
    int64_t *dpre[2][2];             // exclusive edge prefix of dlist rows
    uint2 *inbox[2];
    int64_t inbox_cap;
    uint2 *sendbin[MAXW];            // dist: per destination segment
    int64_t sendcap[MAXW];
    Ctl *ctl;
    Ctl *ctl_all[MAXW];              // in-process: every worker's control block
    uint32_t *nfront_all[2][MAXW];
    parent_t *nparent_all[MAXW];
    const uint32_t *mask_src[2][MAXW];
    const uint32_t *mask_mc[2];      // NVLS: multicast address of the masks (one ld_reduce.or = OR over ranks)
    const parent_t *cand_src[MAXW];
    unsigned long long *pmail;       // peer engine: this rank's barrier mailbox (arrivals by rank, abort, gen)
    unsigned long long *pmail_peer[MAXW];  // every rank's mailbox (own included)
    IterRec *rec;
    unsigned long long *trace;       // DBFS_TRACE: per level x {V start, V done, F start, F done} x block globaltimer
    int32_t *glevel;                 // global outputs when p == 1 (alias nlevel)
    parent_t *gparent;
};

template <typename T>
struct DArray {
    T *p = nullptr;
    int64_t n = 0;
    DArray() = default;
    DArray(const DArray &) = delete;
    DArray &operator=(const DArray &) = delete;
    DArray(DArray &&o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DArray &operator=(DArray &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DArray() { release(); }
    void alloc(int64_t count) {
        release();
        n = count;
        if (count <= 0) return;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * (size_t)count);
        if (e != cudaSuccess) {
            size_t fr = 0, tot = 0;
            cudaGetLastError();
            cudaMemGetInfo(&fr, &tot);
            p = nullptr;
            n = 0;
            throw Error(e == cudaErrorMemoryAllocation ? DBFS_ERESOURCE : DBFS_ECUDA,
                        std::string("device allocation of ") + std::to_string(sizeof(T) * (size_t)count) +
                            " bytes failed (" + cudaGetErrorString(e) + "; " + std::to_string(fr >> 20) +
                            " MiB free of " + std::to_string(tot >> 20) + ")");
        }
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return sizeof(T) * (size_t)n; }
};

struct Ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;  // NCCL level loop: around each level's exchange
    int nranks = 1, rank = 0;
    int local_group = 0;             // every rank is a thread of this process (one device each):
                                     // peer arrays are mapped by pointer + peer access, not CUDA IPC
    void *comm = nullptr;            // ncclComm_t
    DArray<unsigned char> scratch;   // reusable device scratch
    DArray<unsigned char> flush;     // L2 flush buffer (bench hygiene)
    cudaStream_t copy_stream = nullptr;  // non-blocking: result D2H of dbfs_bfs_batch
    cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
    cudaEvent_t ev_hdone[3] = {nullptr, nullptr, nullptr};  // compact batch: host staging set filled
    int flush_val = 1;
    void *ensure_scratch(size_t bytes);
};

struct WorkerHost {
    int w = 0;
    int64_t n_local = 0;
    int64_t base[4] = {0, 0, 0, 0};  // first offset index of each kind in off_all
    int64_t rows[4] = {0, 0, 0, 0};
    int64_t nnz[4] = {0, 0, 0, 0};
    int64_t n_src[4] = {0, 0, 0, 0}; // |nd_src| at [ND], |dn_src| at [DN], |dd_src| at [DD]
    int64_t remote_cap[MAXW];        // nn edges on this worker whose column is owned by dest
    DArray<uint32_t> src_bits[4];
    DArray<uint32_t> deg[4];         // row lengths: [ND] per local normal, [DN]/[DD] per delegate
    DArray<uint32_t> col_sorted;     // dd rows with neighbours by descending degree (executor pulls)
    DArray<uint32_t> head[4];        // [ND]/[DN]/[DD]: first column per row (0 for empty rows)
    DArray<uint32_t> head_sorted;    // first column per sorted dd row
    DArray<uint32_t> twin[4];        // [ND]/[DN]/[DD]: per entry, the source's position in the target's reverse row
    int64_t twin_base[4] = {0, 0, 0, 0};  // absolute col_all position of the kind's first entry
    DArray<uint32_t> first[4];       // per target: min twin position found by a counting push (0xffffffff = none)
    DArray<uint32_t> sentbits;       // dist: remote targets already shipped this BFS (bit per global id)
    int64_t dd_base = 0;             // absolute offset of this worker's first dd entry
    // BFS state
    DArray<int32_t> nlevel, dlevel;
    DArray<parent_t> nparent, dparent, dcand;
    DArray<uint32_t> nvis, nfront0, nfront1, dvis, dfront, dnext0, dnext1;
    DArray<uint32_t> nseen, dseen;   // visited + claims of the running level (push test)
    DArray<uint32_t> ntouch;         // 2 x ntw words: touched chunks of the frontier by parity
    DArray<uint32_t> nchunk_list;    // 2 x chunks: their lists
    DArray<uint32_t> coarse;         // 4 x 8192 words: coarse_d[0..1], coarse_n[0..1]
    DArray<uint32_t> dlist[4];       // [kind*2 + parity]
    DArray<int64_t> dpre[4];
    DArray<uint2> inbox0, inbox1, sendbuf;
    DArray<uint32_t> uq;             // uniquify seen-bits, allocated on first use
    DArray<Ctl> ctl;
    DArray<IterRec> rec;
    int64_t inbox_cap = 0;
    int64_t send_off[MAXW + 1];
};

struct Graph {
    Ctx *ctx = nullptr;
    int64_t n = 0, m = 0, d = 0, theta = 0;
    int p_rank = 1, p_gpu = 1, p = 1;
    int W = 1, first_worker = 0;
    bool dist = false;
    bool symmetric = false;          // every edge's reverse is present (build_rmat_graph / symmetrize)
    int64_t kind_totals[4] = {0, 0, 0, 0};
    DArray<uint32_t> degree;         // out-degree per global vertex
    DArray<uint32_t> del_id;         // delegate id per global vertex, 0xffffffff for normals
    DArray<int64_t> del_gid;         // delegate global ids (ascending)
    DArray<uint32_t> del_gid32;      // their uint32 copy (BFS lookups)
    DArray<int64_t> off_all;         // concatenated CSR offsets (absolute)
    DArray<uint32_t> col_all;        // concatenated CSR columns
    std::vector<WorkerHost> workers; // local workers
    // BFS engine resources (allocated on first BFS)
    bool bfs_ready = false;
    DArray<View> views;
    std::vector<View> views_h;
    DArray<int32_t> glevel;          // assembled outputs (p > 1)
    DArray<parent_t> gparent;
    DArray<int64_t> export_pv;       // int64 copy of the parents for the host (fetch, validation)
    DArray<uint32_t> mask_gather;    // dist: allgather of dnext slices
    DArray<int64_t> recv_off;        // dist: per-source inbox offsets of the current level
    DArray<unsigned long long> dist_scratch;
    Ctl *h_ctl = nullptr;            // pinned host mirrors for the distributed level loop
    int64_t *h_status = nullptr;
    int rec_cap = 0;
    double clock_ghz = 0;            // SM clock for cycle -> time conversion of task timers
    int pgrid = 0;                   // cached cooperative grid of the persistent engine
    double warps_per_worker = 0;
    // last run
    int64_t last_iterations = 0;
    int64_t last_source = -1;
    int last_parent_mode = 0;
    bool last_valid = false;
    bool assembled = true;           // dist: global outputs gathered for the last run
    bool last_truncated = false;
    std::vector<IterRec> last_rec;   // [iteration][local worker]
    std::vector<double> last_comm_us;  // NCCL level loop: measured exchange time per level
    std::vector<std::vector<unsigned long long>> last_send_matrix;
    int last_mode = 1, last_la = 0, last_uq = 0;
    // peer engine (dist): CUDA-IPC mapped peer arrays + a cross-GPU barrier
    int peer_state = 0;              // 0 untried, 1 ready, -1 unavailable
    std::vector<void *> peer_opened; // IPC mappings to close
    DArray<uint32_t> gbar_mem;       // rank 0's copy is the cross-GPU barrier
    void *gbar = nullptr;
    View peer_view_h;
    DArray<View> peer_view;
    std::vector<int64_t> cap_all;    // dist: [src][dst] remote record capacities
    std::vector<int32_t *> peer_nlevel;  // peer-mapped outputs of every rank (assembly over NVLink)
    std::vector<parent_t *> peer_nparent, peer_dparent;
    DArray<int32_t> asm_lv, asm_mylv;    // NCCL assembly buffers (kept between runs)
    DArray<parent_t> asm_pv, asm_mypv;
    DArray<unsigned long long> trace;  // DBFS_TRACE=<file>: block phase timestamps (diagnostics)
    DArray<int32_t> stage_lv[2];     // dbfs_bfs_batch: result staging, double-buffered
    DArray<int64_t> stage_pv[2];
    int8_t *hstage8[3] = {nullptr, nullptr, nullptr};   // compact batch: pinned host staging (depth int8)
    int32_t *hstage32[3] = {nullptr, nullptr, nullptr}; //   and parent int32
    int64_t hstage_n = 0;
    unsigned *hesc = nullptr;        // pinned: escape counts of the 3 host sets
    DArray<unsigned> esc;            // device escape counters (2 staging buffers)
    DArray<unsigned long long> minpar;  // min-ID parent candidates (parent_mode 2)
    void *nvls = nullptr;            // NVSwitch multicast state of the delegate masks (nvls.cu)
    DArray<IterRec> batch_drec;      // dbfs_bfs_batch scratch (grow-only): per-root records,
    IterRec *batch_hrec = nullptr;   //   their pinned host copy,
    DArray<int2> batch_info;         //   per-root (iterations, watchdog),
    std::vector<cudaEvent_t> batch_asm_evs;  // DBFS_BATCH_TRACE: assembly timing
    std::vector<cudaEvent_t> batch_evs;  // and per-root timing events
    ~Graph();
    int32_t *levels_dev();
    parent_t *parents_dev();
    const int64_t *parents_dev64();  // widened into export_pv (ctx stream)
};

// build.cu
void mem_note(const Ctx &ctx, const char *what);  // DBFS_VERBOSE=1: free device memory at build stages
void build_graph_rmat(Graph &g, const dbfs_rmat_params &prm);
void build_graph_edges(Graph &g, const int64_t *src, const int64_t *dst, int64_t m_local);
void build_twins(Graph &g);
void upload_partitioned(Graph &g, const int64_t *degree, const int64_t *dgid, const int64_t *const *off,
                        const void *const *cols);
void export_csr(const Graph &g, int worker, int kind, int64_t *off, void *cols);
void export_sources(const Graph &g, int worker, int64_t *nd_src, uint8_t *dn, uint8_t *dd);
void export_classification(const Graph &g, int64_t *deg, int64_t *del);
void hash_vertices_host(Ctx &ctx, int64_t n, uint64_t seed, const int64_t *in, int64_t *out, int64_t count);
void rmat_generate_host(Ctx &ctx, const dbfs_rmat_params &prm, int64_t begin, int64_t end,
                        int64_t *src, int64_t *dst);

// bfs.cu
void run_bfs(Graph &g, const dbfs_bfs_options &o, dbfs_run_stats *st);
void fetch_result(Graph &g, int32_t *levels, int64_t *parents);
void run_bfs_batch(Graph &g, const dbfs_bfs_options &o, const int64_t *roots, int64_t count, int32_t *const *levels,
                   int64_t *const *parents, int local, int compact, dbfs_run_stats *st);
int64_t batch_output_count(const Graph &g, bool local);
void min_parents(Graph &g, int64_t *out);
void iteration_summary(const Graph &g, const IterRec *x0, int64_t it, int last_la, int last_uq, dbfs_iteration *rec,
                       int8_t *directions, double *bv);
void run_accounting(const Graph &g, const IterRec *recs, int64_t nrec, int64_t iterations, int la, int uq,
                    dbfs_run_stats *st);
int validate(Graph &g, int64_t root, const int32_t *levels, const int64_t *parents);

// dist.cu (NCCL)
void nccl_unique_id(uint8_t *out);
void nccl_init(Ctx &ctx, const uint8_t *uid, int nranks, int rank);
void nccl_destroy(Ctx &ctx);
void nccl_abort(Ctx &ctx);
void nccl_allreduce_u32_sum(Ctx &ctx, uint32_t *dbuf, int64_t count);
void nccl_allreduce_i64(Ctx &ctx, int64_t *dbuf, int64_t count, int op);  // 0 sum, 1 min, 2 max
void nccl_allreduce_i32_min(Ctx &ctx, int32_t *dbuf, int64_t count);
void nccl_allreduce_f64_max(Ctx &ctx, double *dbuf, int64_t count);
void nccl_allgather_bytes(Ctx &ctx, const void *send, void *recv, int64_t bytes);
void nccl_alltoallv_bytes(Ctx &ctx, const void *send, const int64_t *send_off, const int64_t *send_bytes,
                          void *recv, const int64_t *recv_off, const int64_t *recv_bytes);
void nccl_barrier(Ctx &ctx);
void nccl_allreduce_async(Ctx &ctx, void *word);
void nccl_allreduce_u8_max(Ctx &ctx, uint8_t *dbuf, int64_t count);

// io.cu (host only)
int64_t count_text_lines(const char *buf, int64_t len);
void parse_edge_text(const char *buf, int64_t len, int64_t cap, int64_t *src, int64_t *dst, int64_t *m_out,
                     int64_t *header_n);
void write_edge_text(const char *path, int64_t n, const int64_t *src, const int64_t *dst, int64_t m);

// nvls.cu (NVSwitch multicast delegate masks, device groups)
bool nvls_setup(Graph &g, int64_t mask_words, uint32_t **masks, const uint32_t **mc);
void nvls_release(Graph &g);

// scan.cu helpers (device-wide exclusive scans)
void exclusive_scan_u32_to_i64(Ctx &ctx, const uint32_t *in, int64_t *out, int64_t n);  // out has n+1
void radix_sort_pairs(Ctx &ctx, uint32_t *keys, uint32_t *vals, uint32_t *keys_alt, uint32_t *vals_alt,
                      int64_t n, int bits, bool *result_in_alt);

// widen.cpp: compact batch outputs widened on the host (streaming stores)
void widen_host(const int8_t *l8, const int32_t *p32, int64_t n, int32_t *lv, int64_t *pa, int nthreads);

}  // namespace dbfs
