// bfs.cu -- BFS engines (engine.py:98-330 restated for B200).
//
//   persistent: one cooperative launch runs the whole BFS (init, seed, every
//               level's V/F phases separated by grid barriers, assembly).  No
//               host round trip per level; used whenever all workers live on
//               this device (p == 1, or the reference's simulated p workers).
//   host loop : one launch per phase with the NCCL exchange between V and F;
//               used with one worker per process (torchrun, NCCL over NVLink).
#include <algorithm>
#include <chrono>
#include <mutex>
#include <cstdio>
#include <thread>

#include <sched.h>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "bfs_device.cuh"

#ifndef DBFS_VIEW_SMEM
#define DBFS_VIEW_SMEM 1  // the block's View read from shared memory (0: from global, read-only path)
#endif
#ifndef DBFS_MINB
#define DBFS_MINB 1
#endif

namespace dbfs {

// ------------------------------------------------------------- grid barrier

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Sense-counting grid barrier with a watchdog: a block that waits > 4 s sets
// `abort`, every block then leaves the kernel (reported as DBFS_ETIMEOUT).
// With `pv` (the peer engine's view) the last local arriver also meets the
// other GPUs before releasing its GPU: it posts the barrier's generation into
// every rank's mailbox over NVLink (one release store each, no round trip)
// and then waits on its OWN mailbox until every rank's generation arrived --
// local polling, so a cross-GPU barrier costs about one NVLink latency.
// `cv`: the last arriver also evaluates the termination rule of level
// `cont_level` (over every worker's / rank's control block) once for the grid
// and publishes it in cv->ctl->cont before releasing; `ts` gets its
// local-complete / global-complete timestamps.
#ifndef DBFS_BAR_SLEEP
#define DBFS_BAR_SLEEP 64  // ns between a waiting block's polls of the barrier generation
#endif
constexpr int MAIL_ABORT = MAXW, MAIL_GEN = MAXW + 1, MAIL_WORDS = MAXW + 2;

// (the arriving thread fenced at system scope before it arrived, so the
// mailbox stores themselves can be relaxed)
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ bool grid_sync(GridBar *bar, unsigned nblocks, const View *pv = nullptr,
                                          const View *cv = nullptr, int cont_level = 0,
                                          unsigned long long *ts = nullptr) {
    __shared__ int s_ok;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned gen = ld_acquire_u32(&bar->gen);
        if (pv) __threadfence_system();
        else __threadfence();
        unsigned arrived = atomicAdd(&bar->count, 1u);
        if (arrived == nblocks - 1) {
            if (ts) ts[0] = globaltimer_ns();
            if (pv) {
                unsigned long long *mail = pv->pmail;
                const unsigned long long k = mail[MAIL_GEN] + 1;  // identical barrier sequence on every rank
                mail[MAIL_GEN] = k;
                for (int r = 0; r < pv->p; r++) st_relaxed_sys_u64(&pv->pmail_peer[r][pv->w], k);
                unsigned long long t0 = 0;
                unsigned polls = 0;
                bool aborted = false;
                for (int j = 0; j < pv->p;) {
                    if (ld_acquire_sys_u64(&mail[j]) >= k) {
                        j++;
                        continue;
                    }
                    if ((++polls & 63u) == 0) {
                        if (ld_acquire_sys_u64(&mail[MAIL_ABORT])) {
                            aborted = true;
                            break;
                        }
                        const unsigned long long t = globaltimer_ns();
                        if (t0 == 0) t0 = t;
                        else if (t - t0 > 4000000000ull) {
                            for (int r = 0; r < pv->p; r++) st_relaxed_sys_u64(&pv->pmail_peer[r][MAIL_ABORT], 1ull);
                            aborted = true;
                            break;
                        }
                    }
                }
                if (aborted) atomicExch(&bar->abort, 1u);
            }
            if (ts) ts[1] = globaltimer_ns();
            if (cv) cv->ctl->cont = level_continue(*cv, cont_level) ? 1 : 0;
            atomicExch(&bar->count, 0u);
            __threadfence();
            atomicAdd(&bar->gen, 1u);
        } else {
            unsigned long long t0 = globaltimer_ns();
            while (ld_acquire_u32(&bar->gen) == gen) {
                if (ld_acquire_u32(&bar->abort)) break;
                if (globaltimer_ns() - t0 > 4000000000ull) {
                    atomicExch(&bar->abort, 1u);
                    break;
                }
#if DBFS_BAR_SLEEP > 0
                __nanosleep(DBFS_BAR_SLEEP);
#endif
            }
        }
        if (pv) __threadfence_system();
        else __threadfence();
        s_ok = ld_acquire_u32(&bar->abort) == 0;
    }
    __syncthreads();
    return s_ok;
}

// ---------------------------------------------------------------- assembly

struct AsmArgs {
    int64_t n;
    int p;
    PDiv pd;
    const uint32_t *del_id;
    const int32_t *nlevel[MAXW];
    const parent_t *nparent[MAXW];
    int64_t stride;  // dist: gathered arrays are [p][stride]
    const int32_t *dlevel;
    const parent_t *dparent;
    const parent_t *dpar_src[MAXW];  // peer-mapped: every rank's delegate candidates (min taken here)
    int n_dpar;
    int32_t *glevel;
    parent_t *gparent;               // device-side global parents (int32)
    int64_t *gparent64;              // or: the reference's int64 parents (staging for the host)
    int parents;
    int64_t first, step, count;  // output i is vertex first + i*step (global: 0, 1, n; rank r's own: r, p, n_local)
    int8_t *glevel8;             // compact transfer form (dbfs_bfs_batch): depth as int8 from output `split` on
    int64_t split;               //   (outputs before it as int32 into glevel)
    unsigned *esc;               // depths >= 127 (escaped: the root is re-run with full arrays)
};

// Compact wire form of one depth entry (sign extension restores -1 on the host).
__device__ __forceinline__ int8_t pack_level(int32_t l, unsigned *esc) {
    if (l < 127) return (int8_t)l;
    atomicAdd(esc, 1u);
    return (int8_t)127;
}

// levels[v] for normals from worker v mod p, then delegates (engine.py:308-314).
// Output i holds vertex first + i*step: the whole graph, or (distributed) the
// vertices a rank owns, v mod p == rank -- a distributed Graph500 result.
__device__ void phase_assemble(const AsmArgs &a, int64_t tid, int64_t nth) {
    // AU outputs per thread at a time, every load of the batch issued before
    // the dependent ones: the peers' depths are NVLink round trips (~2 us), so
    // one chain per thread left the assembly latency-bound
#ifndef DBFS_AU
#define DBFS_AU 8
#endif
    constexpr int AU = DBFS_AU;
    for (int64_t o0 = tid; o0 < a.count; o0 += AU * nth) {
        uint32_t di[AU], w[AU], i[AU];
        int32_t l[AU];
        parent_t par[AU];
#pragma unroll
        for (int u = 0; u < AU; u++) {
            const int64_t o = o0 + u * nth;
            const int64_t v = a.first + (o < a.count ? o : 0) * a.step;
            di[u] = o < a.count ? a.del_id[v] : 0xfffffffeu;  // 0xfffffffe: no output
            w[u] = a.pd.mod((uint32_t)v);
            i[u] = a.pd.div((uint32_t)v);
        }
#pragma unroll
        for (int u = 0; u < AU; u++) {
            par[u] = -1;
            if (di[u] == 0xfffffffeu) continue;
            if (di[u] != 0xffffffffu) {
                l[u] = a.dlevel[di[u]];
            } else {
                l[u] = a.nlevel[w[u]][i[u]];
                if (a.parents) par[u] = a.nparent[w[u]][i[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < AU; u++) {
            const int64_t o = o0 + u * nth;
            if (di[u] == 0xfffffffeu) continue;
            if (a.parents && di[u] != 0xffffffffu && l[u] >= 0) {
                if (a.n_dpar) {
                    parent_t m = PARENT_MAX;
                    for (int s = 0; s < a.n_dpar; s++) {
                        const parent_t c = a.dpar_src[s][di[u]];
                        m = c < m ? c : m;
                    }
                    par[u] = m;
                } else {
                    par[u] = a.dparent[di[u]];
                }
            }
            if (a.glevel8 && o >= a.split) a.glevel8[o - a.split] = pack_level(l[u], a.esc);
            else a.glevel[o] = l[u];
            if (a.parents) {
                if (a.gparent64) a.gparent64[o] = par[u];
                else a.gparent[o] = par[u];
            }
        }
    }
}

// first column of every row [off[r], off[r+1]) of a kind (pull first probes)
__global__ void k_row_heads(const int64_t *__restrict__ off, int64_t rows, const uint32_t *__restrict__ col,
                            int64_t col_base, uint32_t *__restrict__ head) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = off[r];
        head[r] = b < off[r + 1] ? col[b - col_base] : 0u;
    }
}

__global__ void k_narrow_ids(const int64_t *__restrict__ in, int64_t n, uint32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// int32 device parents -> the reference's int64 (host copies, validation)
__global__ void k_widen_parents(const parent_t *__restrict__ in, int64_t n, int64_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// ----------------------------------------------------------------- kernels

__global__ void __launch_bounds__(BT, DBFS_MINB) k_bfs_persistent(const View *__restrict__ views, int W, int64_t source,
                                                       uint32_t src_del, GridBar *bar, int rec_cap,
                                                       AsmArgs asm_args, int do_assemble, GridBar *gbar,
                                                       int nranks, const uint32_t *__restrict__ del_id) {
    extern __shared__ uint4 dsm[];
    Smem &sm = *reinterpret_cast<Smem *>(dsm);
    const int wsel = blockIdx.x % W, wb = blockIdx.x / W, nb = gridDim.x / W;
    {
        static_assert(sizeof(View) % 16 == 0, "View is copied in 16-byte words");
        const uint4 *src = reinterpret_cast<const uint4 *>(&views[wsel]);
        uint4 *dst = reinterpret_cast<uint4 *>(&sm.view);
        for (int i = threadIdx.x; i < (int)(sizeof(View) / 16); i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
#if DBFS_VIEW_SMEM
    const View &V = sm.view;
#else
    const View &V = views[wsel];
#endif
    const unsigned nblocks = gridDim.x;
    const bool timer = wb == 0 && threadIdx.x == 0;
    if (timer) V.ctl->t_start = globaltimer_ns();
    // DBFS_TRACE diagnostics: every block's phase boundaries (block-uniform branch)
    auto stamp = [&](int lv, int ph) {
        if (!V.trace || lv >= 64) return;
        __syncthreads();
        if (threadIdx.x == 0) V.trace[((size_t)lv * 8 + ph) * gridDim.x + blockIdx.x] = globaltimer_ns();
    };
    phase_init(V, wb, nb);
    const View *pv = gbar ? &views[0] : nullptr;  // peer engine: cross-GPU barriers
    if (!grid_sync(bar, nblocks, pv)) return;
    if (wb == 0 && threadIdx.x == 0)  // SRC_DEL_LOOKUP: the host did not read del_id[source] (dbfs_bfs_batch)
        seed_worker(V, source, src_del == SRC_DEL_LOOKUP ? __ldg(&del_id[source]) : src_del);
    if (!grid_sync(bar, nblocks, pv)) return;
    if (timer) V.ctl->t_seeded = globaltimer_ns();
    int L = 0;
    for (;; L++) {
        if (L > 0) {
            // evaluated once by the barrier's last arriver (NVLink loads in the peer engine)
            const bool cont = __ldcg(&views[0].ctl->cont) != 0;
            if (!cont) {
                if (wb == 0 && threadIdx.x < 32 && L - 1 < rec_cap) make_record_warp(V, *V.ctl, L - 1, V.rec[L - 1]);
                break;
            }
        }
        if (timer && L < rec_cap) V.rec[L].t[0] = globaltimer_ns();
        unsigned long long *tb = L < rec_cap ? views[0].rec[L].tb : nullptr;
        stamp(L, 0);
        phase_visit(V, L, wb, nb, sm);
        // the record of level L-1 (its slot lives until F(L) ends) is made by the
        // first of the worker's blocks to finish V(L): off the critical path
        if (L > 0 && threadIdx.x < 32 && L - 1 < rec_cap) {
            int mine = 0;
            if (threadIdx.x == 0) mine = atomicCAS(&V.ctl->rec_level, L - 1, L) == L - 1;
            if (__shfl_sync(0xffffffffu, mine, 0)) make_record_warp(V, *V.ctl, L - 1, V.rec[L - 1]);
        }
        stamp(L, 5);
        if (!grid_sync(bar, nblocks, pv, nullptr, 0, tb)) return;
        if (timer && L < rec_cap) V.rec[L].t[1] = globaltimer_ns();
        stamp(L, 6);
        if (V.peer) {  // peers' records are claimed before the frontier is folded
            phase_finish(V, L, wb, nb, sm, F_DELEGATES | F_INGEST);
            if (!grid_sync(bar, nblocks)) return;
            phase_finish(V, L, wb, nb, sm, F_NORMALS);
        } else {
            phase_finish(V, L, wb, nb, sm, F_DELEGATES | F_NORMALS);
        }
        stamp(L, 7);
        if (!grid_sync(bar, nblocks, pv, &views[0], L, tb ? tb + 2 : nullptr)) return;
        if (timer && L < rec_cap) V.rec[L].t[2] = globaltimer_ns();
    }
    if (wb == 0 && threadIdx.x == 0) V.ctl->last_level = L;
    // peers read this GPU's control block until they leave the loop: nobody may
    // start the next BFS (host resets the block) before every GPU is past it
    if (gbar && !grid_sync(bar, nblocks, pv)) return;
    if (do_assemble) phase_assemble(asm_args, (int64_t)blockIdx.x * BT + threadIdx.x, (int64_t)gridDim.x * BT);
}

// dbfs_bfs_batch helpers.  Between roots the stream only runs kernels: a
// cudaMemset/cudaMemcpy would queue on a copy engine behind the previous
// root's result D2H and serialise the pipeline.
__global__ void k_batch_prep(const View *__restrict__ views, GridBar *bar) {
    static_assert(sizeof(Ctl) % 8 == 0, "Ctl is cleared in 8-byte words");
    unsigned long long *c = reinterpret_cast<unsigned long long *>(views[blockIdx.x].ctl);
    for (size_t i = threadIdx.x; i < sizeof(Ctl) / 8; i += blockDim.x) c[i] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) *bar = GridBar{0u, 0u, 0u, 0u};
}

// Per-root iteration records of a batch (dbfs_bfs_batch with record_iterations):
// the first rmax records of every worker into dst[it * W + w].
// grid (STAGE_BLOCKS, W): only the records of the iterations that ran
constexpr int STAGE_BLOCKS = 8;
__global__ void k_stage_recs(const View *__restrict__ views, int W, int rmax, IterRec *__restrict__ dst) {
    const int w = blockIdx.y;
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(views[w].rec);
    static_assert(sizeof(IterRec) % 8 == 0, "records are copied in 8-byte words");
    constexpr int NW = sizeof(IterRec) / 8;
    const int nrec = min(rmax, views[w].ctl->last_level + 1);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec * NW; i += gridDim.x * blockDim.x) {
        const int it = i / NW, j = i % NW;
        reinterpret_cast<unsigned long long *>(&dst[(size_t)it * W + w])[j] = src[i];
    }
}

__global__ void k_batch_info(const Ctl *__restrict__ ctl0, const GridBar *__restrict__ bar, int2 *info,
                             unsigned *esc) {
    *info = make_int2(ctl0->last_level, (int)bar->abort);
    if (esc) *esc = 0u;  // escape counter of this root's compact outputs
}

__global__ void k_copy_bytes(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, int64_t bytes) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t n16 = bytes >> 4;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (int64_t i = tid; i < n16; i += nth) d4[i] = __ldcs(&s4[i]);
    for (int64_t i = (n16 << 4) + tid; i < bytes; i += nth) dst[i] = src[i];
}

// Compact wire form of the whole-graph outputs (single process): 4 entries per thread.
__global__ void k_pack_result(const int32_t *__restrict__ lv, int64_t n, int8_t *__restrict__ lv8, unsigned *esc) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;  // int4 loads in flight per thread
    const int64_t nq = n >> 2;
    for (int64_t q0 = tid; q0 < nq; q0 += U * nth) {
        int4 l[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t q = q0 + u * nth;
            l[u] = q < nq ? __ldcs(reinterpret_cast<const int4 *>(lv) + q) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t q = q0 + u * nth;
            if (q >= nq) break;
            char4 c;
            c.x = pack_level(l[u].x, esc);
            c.y = pack_level(l[u].y, esc);
            c.z = pack_level(l[u].z, esc);
            c.w = pack_level(l[u].w, esc);
            reinterpret_cast<char4 *>(lv8)[q] = c;
        }
    }
    for (int64_t i = (nq << 2) + tid; i < n; i += nth) lv8[i] = pack_level(lv[i], esc);
}

__global__ void __launch_bounds__(BT) k_init(const View *__restrict__ views, int W) {
    phase_init(views[blockIdx.x % W], blockIdx.x / W, gridDim.x / W);
}

__global__ void k_seed(const View *__restrict__ views, int W, int64_t source, uint32_t src_del) {
    if (threadIdx.x == 0 && (int)blockIdx.x < W) seed_worker(views[blockIdx.x], source, src_del);
}

__global__ void __launch_bounds__(BT, DBFS_MINB) k_visit(const View *__restrict__ views, int W, int L) {
    extern __shared__ uint4 dsm[];
    Smem &sm = *reinterpret_cast<Smem *>(dsm);
    phase_visit(views[blockIdx.x % W], L, blockIdx.x / W, gridDim.x / W, sm);
}

__global__ void __launch_bounds__(BT) k_finish(const View *__restrict__ views, int W, int L, int parts) {
    extern __shared__ uint4 dsm[];
    Smem &sm = *reinterpret_cast<Smem *>(dsm);
    phase_finish(views[blockIdx.x % W], L, blockIdx.x / W, gridDim.x / W, sm, parts);
}

__global__ void __launch_bounds__(BT) k_assemble(AsmArgs a) {
    phase_assemble(a, (int64_t)blockIdx.x * BT + threadIdx.x, (int64_t)gridDim.x * BT);
}

// --------------------------------------------------------------- resources


Graph::~Graph() {
    nvls_release(*this);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (batch_hrec) cudaFreeHost(batch_hrec);
    for (cudaEvent_t e : batch_evs) cudaEventDestroy(e);
    for (cudaEvent_t e : batch_asm_evs) cudaEventDestroy(e);
    for (int h = 0; h < 3; h++) {
        if (hstage8[h]) cudaFreeHost(hstage8[h]);
        if (hstage32[h]) cudaFreeHost(hstage32[h]);
    }
    if (hesc) cudaFreeHost(hesc);
    if (h_status) cudaFreeHost(h_status);
    for (void *q : peer_opened) cudaIpcCloseMemHandle(q);
}

int32_t *Graph::levels_dev() { return (p == 1 && !dist) ? workers[0].nlevel.p : glevel.p; }
parent_t *Graph::parents_dev() { return (p == 1 && !dist) ? workers[0].nparent.p : gparent.p; }

const int64_t *Graph::parents_dev64() {
    if (export_pv.n < std::max<int64_t>(n, 1)) export_pv.alloc(std::max<int64_t>(n, 1));
    Ctx &c = *ctx;
    k_widen_parents<<<c.num_sms * 4, 256, 0, c.stream>>>(parents_dev(), n, export_pv.p);
    DBFS_LAUNCHED();
    return export_pv.p;
}

void build_sorted_dd(Graph &g);

static void ensure_resources(Graph &g) {
    if (g.bfs_ready) return;
    if (g.symmetric) build_sorted_dd(g);
    if (g.symmetric && !getenv("DBFS_NO_TWINS")) build_twins(g);
    Ctx &ctx = *g.ctx;
    DBFS_CHECK(g.n <= PARENT_MAX, DBFS_ECAPACITY, "parent ids are int32 on the device: n must be < 2^31");
    g.del_gid32.alloc(std::max<int64_t>(g.d, 1));
    if (g.d) {
        k_narrow_ids<<<g.ctx->num_sms * 4, 256, 0, g.ctx->stream>>>(g.del_gid.p, g.d, g.del_gid32.p);
        DBFS_LAUNCHED();
    }
    const int W = (int)g.workers.size();
    g.W = W;
    g.rec_cap = (int)std::min<int64_t>(std::max<int64_t>(g.n + 2, 16), 1 << 16);
    const int64_t nw_d = nwords(g.d);
    // per-destination inbox capacities
    std::vector<int64_t> inbox_cap(g.p, 0);
    if (!g.dist) {
        for (auto &W0 : g.workers)
            for (int o = 0; o < g.p; o++) inbox_cap[o] += W0.remote_cap[o];
    } else {
        // all ranks' caps towards me: all-gather the cap vectors
        DArray<int64_t> s, r;
        s.alloc(g.p);
        r.alloc((int64_t)g.p * g.p);
        std::vector<int64_t> mine(g.p);
        // peer engine: senders reserve inbox slots in chunks (SEND_CHUNK per warp,
        // bfs_device.cuh), so every non-empty segment gets one chunk per resident warp of slack
        const int64_t slack = (int64_t)ctx.num_sms * 64 * SEND_CHUNK;
        for (int o = 0; o < g.p; o++)
            mine[o] = g.workers[0].remote_cap[o] + (o != ctx.rank && g.workers[0].remote_cap[o] > 0 ? slack : 0);
        DBFS_CUDA(cudaMemcpy(s.p, mine.data(), 8 * g.p, cudaMemcpyHostToDevice));
        nccl_allgather_bytes(ctx, s.p, r.p, 8 * g.p);
        std::vector<int64_t> all((size_t)g.p * g.p);
        DBFS_CUDA(cudaMemcpy(all.data(), r.p, 8 * g.p * g.p, cudaMemcpyDeviceToHost));
        for (int src = 0; src < g.p; src++) inbox_cap[ctx.rank] += all[(size_t)src * g.p + ctx.rank];
        g.cap_all = all;
    }
    for (auto &Wk : g.workers) {
        const int64_t nl = Wk.n_local, nw_n = nwords(nl);
        Wk.nlevel.alloc(std::max<int64_t>(nl, 1));
        Wk.nparent.alloc(std::max<int64_t>(nl, 1));
        Wk.dlevel.alloc(std::max<int64_t>(g.d, 1));
        Wk.dparent.alloc(std::max<int64_t>(g.d, 1));
        Wk.dcand.alloc(std::max<int64_t>(g.d, 1));
        Wk.nvis.alloc(std::max<int64_t>(nw_n, 1));
        Wk.nseen.alloc(std::max<int64_t>(nw_n, 1));
        Wk.ntouch.alloc(2 * std::max<int64_t>(nwords(ceil_div(nw_n, 32)), 1));
        Wk.nchunk_list.alloc(2 * std::max<int64_t>(ceil_div(nw_n, 32), 1));
        Wk.dseen.alloc(std::max<int64_t>(nw_d, 1));
        Wk.nfront0.alloc(std::max<int64_t>(nw_n, 1));
        Wk.nfront1.alloc(std::max<int64_t>(nw_n, 1));
        Wk.dvis.alloc(std::max<int64_t>(nw_d, 1));
        Wk.dfront.alloc(std::max<int64_t>(nw_d, 1));
        Wk.dnext0.alloc(std::max<int64_t>(nw_d, 1));
        Wk.dnext1.alloc(std::max<int64_t>(nw_d, 1));
        Wk.coarse.alloc(4 * FW);
        for (int j = 0; j < 4; j++) {
            Wk.dlist[j].alloc(std::max<int64_t>(g.d, 1));
            Wk.dpre[j].alloc(g.d + 1);
        }
        Wk.inbox_cap = g.dist ? std::max<int64_t>(inbox_cap[Wk.w], 1) : 1;
        Wk.inbox0.alloc(Wk.inbox_cap);
        Wk.inbox1.alloc(Wk.inbox_cap);
        if (g.dist) {
            Wk.sentbits.alloc(std::max<int64_t>(nwords(g.n), 1));
            int64_t acc = 0;
            for (int o = 0; o < g.p; o++) {
                Wk.send_off[o] = acc;
                acc += Wk.remote_cap[o];
            }
            Wk.send_off[g.p] = acc;
            Wk.sendbuf.alloc(std::max<int64_t>(acc, 1));
        }
        Wk.ctl.alloc(1);
        Wk.rec.alloc(g.rec_cap);
        if (!getenv("DBFS_NO_HEADS"))  // row heads of the pulled kinds
            for (int k = 1; k < 4; k++) {
                if (Wk.rows[k] <= 0 || Wk.head[k].n) continue;
                Wk.head[k].alloc(Wk.rows[k]);
                k_row_heads<<<ctx.num_sms * 4, 256, 0, ctx.stream>>>(g.off_all.p + Wk.base[k], Wk.rows[k],
                                                                     g.col_all.p, 0, Wk.head[k].p);
                DBFS_LAUNCHED();
                if (k == KIND_DD && Wk.col_sorted.n) {
                    Wk.head_sorted.alloc(Wk.rows[k]);
                    k_row_heads<<<ctx.num_sms * 4, 256, 0, ctx.stream>>>(g.off_all.p + Wk.base[k], Wk.rows[k],
                                                                         Wk.col_sorted.p, Wk.dd_base,
                                                                         Wk.head_sorted.p);
                    DBFS_LAUNCHED();
                }
            }
        for (int k = 1; k < 4; k++)
            if (Wk.twin[k].n && !Wk.first[k].n) {
                Wk.first[k].alloc(std::max<int64_t>(k == KIND_DN ? nl : g.d, 1));
                DBFS_CUDA(cudaMemset(Wk.first[k].p, 0xff, Wk.first[k].bytes()));
            }
    }
    if (g.p > 1 || g.dist) {
        g.glevel.alloc(std::max<int64_t>(g.n, 1));
        g.gparent.alloc(std::max<int64_t>(g.n, 1));
    }
    if (g.dist) g.mask_gather.alloc(std::max<int64_t>(nw_d, 1) * g.p);
    g.recv_off.alloc(g.p + 1);
    // views
    g.views_h.assign(W, View{});
    for (int i = 0; i < W; i++) {
        WorkerHost &Wk = g.workers[i];
        View &V = g.views_h[i];
        memset(&V, 0, sizeof(View));
        V.w = Wk.w;
        V.W = W;
        V.p = g.p;
        V.p_rank = g.p_rank;
        V.dist = g.dist;
        V.cand_all = !g.dist;
        V.P_sources = g.dist ? g.p : W;
        V.rec_cap = g.rec_cap;
        V.t1_dyn_min = getenv("DBFS_T1_DYN_MIN") ? atoi(getenv("DBFS_T1_DYN_MIN")) : 4;
        V.f3_dyn = getenv("DBFS_F3_DYN") ? atoi(getenv("DBFS_F3_DYN")) : 1;
        V.pull_dyn_min = getenv("DBFS_PULL_DYN_MIN") ? atoi(getenv("DBFS_PULL_DYN_MIN")) : 32;
        {
            // one 64-bit atomic reserves list slots and edge prefixes together:
            // edge bits for this worker's dn/dd totals, count bits for d
            int cbits = 1, ebits = 1;
            while (((int64_t)1 << cbits) <= g.d) cbits++;
            const int64_t emax = std::max(Wk.nnz[KIND_DN], Wk.nnz[KIND_DD]);
            while (ebits < 63 && ((int64_t)1 << ebits) <= emax) ebits++;
            DBFS_CHECK(cbits + ebits <= 64, DBFS_ECAPACITY,
                       "delegate frontier lists: d and the dn/dd edge totals need more than 64 bits");
            V.dshift = 64 - cbits;
        }
        V.pd.init((uint32_t)g.p);
        V.n = g.n;
        V.n_local = Wk.n_local;
        V.d = g.d;
        V.nw_n = nwords(Wk.n_local);
        V.nw_d = nw_d;
        for (int o = 0; o < g.p && o < MAXW; o++) V.n_local_of_w[o] = g.n > o ? (g.n - o + g.p - 1) / g.p : 0;
        V.recv_off = g.recv_off.p;
        for (int k = 0; k < 4; k++) {
            V.off[k] = g.off_all.p + Wk.base[k];
            V.col[k] = g.col_all.p;
            V.src_bits[k] = Wk.src_bits[k].p;
            V.deg[k] = Wk.deg[k].p;
            V.total_src[k] = (unsigned long long)Wk.n_src[k];
            V.nnz[k] = (unsigned long long)Wk.nnz[k];
        }
        V.del_gid = g.del_gid.p;
        V.del_gid32 = g.del_gid32.p;
        // indexed with absolute dd offsets (the worker's copy starts at dd_base)
        V.col_sorted_dd = Wk.col_sorted.n ? Wk.col_sorted.p - Wk.dd_base : nullptr;
        for (int k = 0; k < 4; k++) V.head[k] = Wk.head[k].n ? Wk.head[k].p : nullptr;
        V.head_sorted_dd = Wk.head_sorted.n ? Wk.head_sorted.p : nullptr;
        if (V.col_sorted_dd && !V.head_sorted_dd) V.head[KIND_DD] = nullptr;  // both orders or neither
        for (int k = 1; k < 4; k++) {
            V.twin[k] = Wk.twin[k].n ? Wk.twin[k].p - Wk.twin_base[k] : nullptr;
            V.first[k] = Wk.twin[k].n ? Wk.first[k].p : nullptr;
        }
        V.nlevel = Wk.nlevel.p;
        V.nparent = Wk.nparent.p;
        V.dlevel = Wk.dlevel.p;
        V.dparent = Wk.dparent.p;
        V.dcand = Wk.dcand.p;
        V.nvis = Wk.nvis.p;
        V.nseen = Wk.nseen.p;
        V.ntw = Wk.ntouch.n / 2;
        V.ntouch[0] = Wk.ntouch.p;
        V.ntouch[1] = Wk.ntouch.p + V.ntw;
        V.nchunk_list[0] = Wk.nchunk_list.p;
        V.nchunk_list[1] = Wk.nchunk_list.p + Wk.nchunk_list.n / 2;
        V.dseen = Wk.dseen.p;
        V.nfront[0] = Wk.nfront0.p;
        V.nfront[1] = Wk.nfront1.p;
        V.dvis = Wk.dvis.p;
        V.dfront = Wk.dfront.p;
        V.dnext[0] = Wk.dnext0.p;
        V.dnext[1] = Wk.dnext1.p;
        for (int par = 0; par < 2; par++) {
            V.coarse_d[par] = Wk.coarse.p + par * FW;
            V.coarse_n[par] = Wk.coarse.p + (2 + par) * FW;
        }
        for (int kk = 0; kk < 2; kk++)
            for (int par = 0; par < 2; par++) {
                V.dlist[kk][par] = Wk.dlist[kk * 2 + par].p;
                V.dpre[kk][par] = Wk.dpre[kk * 2 + par].p;
            }
        V.inbox[0] = Wk.inbox0.p;
        V.inbox[1] = Wk.inbox1.p;
        V.inbox_cap = Wk.inbox_cap;
        V.ctl = Wk.ctl.p;
        V.rec = Wk.rec.p;
        if (g.dist) {
            for (int o = 0; o < g.p; o++) {
                V.sendbin[o] = Wk.sendbuf.p + Wk.send_off[o];
                V.sendcap[o] = Wk.remote_cap[o];
                V.mask_src[0][o] = g.mask_gather.p + (int64_t)o * std::max<int64_t>(nw_d, 1);
                V.mask_src[1][o] = V.mask_src[0][o];
            }
        } else {
            for (int j = 0; j < W; j++) {
                WorkerHost &Wj = g.workers[j];
                V.ctl_all[j] = Wj.ctl.p;
                V.nseen_all[j] = Wj.nseen.p;
                V.nfront_all[0][j] = Wj.nfront0.p;
                V.nfront_all[1][j] = Wj.nfront1.p;
                V.nparent_all[j] = Wj.nparent.p;
                V.mask_src[0][j] = Wj.dnext0.p;
                V.mask_src[1][j] = Wj.dnext1.p;
                V.cand_src[j] = Wj.dcand.p;
            }
        }
        if (g.p == 1 && !g.dist) {
            V.glevel = Wk.nlevel.p;
            V.gparent = Wk.nparent.p;
        }
    }
    g.views.alloc(W);
    DBFS_CUDA(cudaMemcpy(g.views.p, g.views_h.data(), sizeof(View) * W, cudaMemcpyHostToDevice));
    g.dist_scratch.alloc(2 * (int64_t)(g.p + 3) * (g.p + 1) + 64);
    if (!g.h_ctl) {
        DBFS_CUDA(cudaHostAlloc((void **)&g.h_ctl, sizeof(Ctl), cudaHostAllocDefault));
        DBFS_CUDA(cudaHostAlloc((void **)&g.h_status, 8 * ((size_t)(g.p + 3) * g.p + g.p + 16), cudaHostAllocDefault));
    }
    g.bfs_ready = true;
    (void)ctx;
}

// Dynamic shared-memory limits are per device: a process may drive several
// GPUs (group.py runs one host thread per device).
static void set_smem_attrs() {
    static std::mutex mu;
    static std::vector<char> done;
    int dev = 0;
    DBFS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if ((int)done.size() <= dev) done.resize(dev + 1, 0);
    if (done[dev]) return;
    DBFS_CUDA(cudaFuncSetAttribute(k_bfs_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Smem)));
    DBFS_CUDA(cudaFuncSetAttribute(k_visit, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Smem)));
    DBFS_CUDA(cudaFuncSetAttribute(k_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Smem)));
    done[dev] = 1;
}

static int persistent_grid(Graph &g, int *blocks_per_sm) {
    int occ = 0;
    set_smem_attrs();
    DBFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bfs_persistent, BT, sizeof(Smem)));
    DBFS_CHECK(occ >= 1, DBFS_EINTERNAL, "persistent kernel cannot be resident");
    *blocks_per_sm = occ;
    int grid = g.ctx->num_sms * occ;
    grid = (grid / g.W) * g.W;
    DBFS_CHECK(grid >= g.W, DBFS_EINTERNAL, "too many workers for one device");
    return grid;
}

static AsmArgs make_asm(Graph &g, bool parents) {
    AsmArgs a{};
    a.n = g.n;
    a.p = g.p;
    a.pd.init((uint32_t)g.p);
    a.del_id = g.del_id.p;
    for (auto &Wk : g.workers) {
        a.nlevel[Wk.w] = Wk.nlevel.p;
        a.nparent[Wk.w] = Wk.nparent.p;
    }
    a.dlevel = g.workers[0].dlevel.p;
    a.dparent = g.workers[0].dparent.p;
    a.glevel = g.glevel.p;
    a.gparent = g.gparent.p;
    a.parents = parents;
    a.first = 0;
    a.step = 1;
    a.count = g.n;
    return a;
}

// --------------------------------------------------------------- dist glue

__global__ void k_count_reached(const int32_t *__restrict__ lv, int64_t n, unsigned long long *out);

// Status vector of one rank at level L: records per destination (level L),
// then the termination inputs of level L-1: records(L-1), |frontier normals at
// L| (counted in F(L-1)) and the delegates found at L-1.
__global__ void k_pack_status(const Ctl *__restrict__ c, int L, int p, int64_t *__restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const LevelSlot &A = c->s[L % 3];
    for (int o = 0; o < p; o++) out[o] = (int64_t)A.sent[o];  // shipped records size the exchange
    const LevelSlot &P = c->s[(L + 2) % 3];  // level L-1
    out[p] = L > 0 ? (int64_t)P.records : 0;
    out[p + 1] = (int64_t)A.nfront;
    out[p + 2] = L > 0 ? (int64_t)P.new_del : 0;
}

// One level of the one-worker-per-process engine: a single host sync per level.
static bool dist_level(Graph &g, int L, int grid, std::vector<IterRec> &recs) {
    Ctx &ctx = *g.ctx;
    WorkerHost &Wk = g.workers[0];
    const int p = g.p, me = ctx.rank;
    const int64_t nw_d = std::max<int64_t>(nwords(g.d), 1);
    k_visit<<<grid, BT, sizeof(Smem), ctx.stream>>>(g.views.p, 1, L);
    DBFS_LAUNCHED();
    const int S = p + 3;
    int64_t *st_dev = (int64_t *)g.dist_scratch.p;
    int64_t *st_all = st_dev + S;
    k_pack_status<<<1, 32, 0, ctx.stream>>>(Wk.ctl.p, L, p, st_dev);
    DBFS_LAUNCHED();
    if (!ctx.ev_c0) {
        DBFS_CUDA(cudaEventCreate(&ctx.ev_c0));
        DBFS_CUDA(cudaEventCreate(&ctx.ev_c1));
    }
    DBFS_CUDA(cudaEventRecord(ctx.ev_c0, ctx.stream));  // the level's exchange starts
    nccl_allgather_bytes(ctx, st_dev, st_all, 8 * S);
    uint32_t *own = g.views_h[0].dnext[L & 1];  // (NVLS: the multicast-bound copy)
    nccl_allgather_bytes(ctx, own, g.mask_gather.p, nw_d * 4);
    DBFS_CUDA(cudaMemcpyAsync(g.h_status, st_all, 8 * S * p, cudaMemcpyDeviceToHost, ctx.stream));
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    const int64_t *all = g.h_status;
    if (L > 0) {
        // termination of level L-1 (engine.py:303-306), decided globally
        int64_t act = all[0 * S + p + 2];  // new delegates (identical on every rank)
        for (int r = 0; r < p; r++) act += all[r * S + p] + all[r * S + p + 1];
        IterRec rr{};
        make_record(g.views_h[0], *g.h_ctl, L - 1, rr);
        if (L - 1 < g.rec_cap) recs.push_back(rr);
        if (!act) return false;  // level L was speculative: nothing ran on an empty frontier
    }
    std::vector<int64_t> soff(p), sbytes(p), roff(p), rbytes(p);
    int64_t racc = 0;
    for (int o = 0; o < p; o++) {
        soff[o] = Wk.send_off[o] * 8;
        sbytes[o] = o == me ? 0 : all[me * S + o] * 8;
        int64_t c = o == me ? 0 : all[o * S + me];
        roff[o] = racc * 8;
        rbytes[o] = c * 8;
        racc += c;
    }
    uint2 *inbox = (L & 1) ? Wk.inbox1.p : Wk.inbox0.p;
    nccl_alltoallv_bytes(ctx, Wk.sendbuf.p, soff.data(), sbytes.data(), inbox, roff.data(), rbytes.data());
    DBFS_CUDA(cudaEventRecord(ctx.ev_c1, ctx.stream));
    {
        DBFS_CUDA(cudaEventSynchronize(ctx.ev_c1));
        float ms = 0.f;
        DBFS_CUDA(cudaEventElapsedTime(&ms, ctx.ev_c0, ctx.ev_c1));
        if ((int64_t)g.last_comm_us.size() <= L) g.last_comm_us.resize(L + 1, 0.0);
        g.last_comm_us[L] = 1e3 * ms;
    }
    g.h_status[S * p] = racc;
    DBFS_CUDA(cudaMemcpyAsync(&Wk.ctl.p->s[L % 3].inbox, &g.h_status[S * p], 8, cudaMemcpyHostToDevice, ctx.stream));
    if (g.views_h[0].uniquify) {
        for (int o = 0; o < p; o++) g.h_status[S * p + 1 + o] = roff[o] / 8;
        g.h_status[S * p + 1 + p] = racc;
        DBFS_CUDA(cudaMemcpyAsync(g.recv_off.p, &g.h_status[S * p + 1], 8 * (p + 1), cudaMemcpyHostToDevice,
                                  ctx.stream));
    }
    k_finish<<<grid, BT, sizeof(Smem), ctx.stream>>>(g.views.p, 1, L, F_DELEGATES | F_INGEST);
    DBFS_LAUNCHED();
    k_finish<<<grid, BT, sizeof(Smem), ctx.stream>>>(g.views.p, 1, L, F_NORMALS);
    DBFS_LAUNCHED();
    // the control block after F(L) is what level L's record is made from
    DBFS_CUDA(cudaMemcpyAsync(g.h_ctl, Wk.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
    return true;
}

// ------------------------------------------------------------- peer engine

// Map the peers' control blocks, delegate masks/candidates and inboxes
// through CUDA IPC (NVLink/NVSwitch), so the persistent kernel runs across all
// ranks: delegate masks are OR-ed straight from peer memory, remote records are
// stored into fixed per-sender segments of the owner's inbox, and levels are
// separated by a system-scope barrier in rank 0's memory.  Collective; every
// rank agrees on the outcome (the host-loop NCCL engine is the fallback).
static void finish_peer_setup(Graph &g, const std::vector<void *> &ptr);

static void setup_peer(Graph &g) {
    if (g.peer_state) return;
    g.peer_state = -1;
    Ctx &ctx = *g.ctx;
    const int p = g.p, me = ctx.rank;
    const char *env = getenv("DBFS_PEER");
    int ok = (!env || env[0] != '0') && p <= MAXW && g.workers.size() == 1 && (int)g.cap_all.size() == p * p;
    WorkerHost &Wk = g.workers[0];
    g.gbar_mem.alloc(2 * MAIL_WORDS);  // this rank's barrier mailbox (u64 words)
    DBFS_CUDA(cudaMemset(g.gbar_mem.p, 0, g.gbar_mem.bytes()));
    constexpr int NH = 9;
    void *bases[NH] = {Wk.ctl.p,    Wk.dnext0.p,  Wk.dnext1.p,  Wk.dcand.p,    Wk.inbox0.p,
                       Wk.nlevel.p, Wk.nparent.p, Wk.dparent.p, g.gbar_mem.p};
    if (ctx.local_group) {
        // ranks are threads of this process: exchange raw device pointers (and
        // device ordinals) and enable peer access instead of CUDA IPC
        struct Rec {
            void *ptr[NH];
            int64_t dev;
        } me_rec{}, *all_rec = nullptr;
        for (int i = 0; i < NH; i++) me_rec.ptr[i] = bases[i];
        me_rec.dev = ctx.device;
        std::vector<Rec> recs(p);
        DArray<uint8_t> hs, hr;
        hs.alloc(sizeof(Rec));
        hr.alloc(sizeof(Rec) * p);
        DBFS_CUDA(cudaMemcpy(hs.p, &me_rec, sizeof(Rec), cudaMemcpyHostToDevice));
        nccl_allgather_bytes(ctx, hs.p, hr.p, sizeof(Rec));
        DBFS_CUDA(cudaMemcpy(recs.data(), hr.p, sizeof(Rec) * p, cudaMemcpyDeviceToHost));
        all_rec = recs.data();
        int lok = ok;
        for (int j = 0; j < p && lok; j++) {
            if (j == me) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, ctx.device, (int)all_rec[j].dev) != cudaSuccess || !can) {
                cudaGetLastError();
                lok = 0;
                break;
            }
            cudaError_t e = cudaDeviceEnablePeerAccess((int)all_rec[j].dev, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) lok = 0;
            cudaGetLastError();
        }
        DArray<uint32_t> f;
        f.alloc(1);
        uint32_t h = lok ? 1u : 0u;
        DBFS_CUDA(cudaMemcpy(f.p, &h, 4, cudaMemcpyHostToDevice));
        nccl_allreduce_u32_sum(ctx, f.p, 1);
        DBFS_CUDA(cudaMemcpy(&h, f.p, 4, cudaMemcpyDeviceToHost));
        if ((int)h != p) return;
        std::vector<void *> ptr((size_t)NH * p, nullptr);
        for (int j = 0; j < p; j++)
            for (int i = 0; i < NH; i++) ptr[(size_t)j * NH + i] = all_rec[j].ptr[i];
        // NVSwitch multicast for the delegate masks (opt-in): the masks move to
        // multicast-bound memory; F reads the OR of all ranks with one load
        uint32_t *masks[2] = {nullptr, nullptr};
        const uint32_t *mc[2] = {nullptr, nullptr};
        const char *nv = getenv("DBFS_NVLS");
        const bool use_nvls = nv && nv[0] == '1' && nvls_setup(g, std::max<int64_t>(nwords(g.d), 1), masks, mc);
        if (use_nvls) {
            for (int b = 0; b < 2; b++) g.views_h[0].dnext[b] = masks[b];
            DBFS_CUDA(cudaMemcpy(g.views.p, g.views_h.data(), sizeof(View) * g.views_h.size(), cudaMemcpyHostToDevice));
        }
        finish_peer_setup(g, ptr);
        if (use_nvls)
            for (int b = 0; b < 2; b++) g.peer_view_h.mask_mc[b] = mc[b];
        return;
    }
    std::vector<cudaIpcMemHandle_t> mine(NH), all((size_t)NH * p);
    for (int i = 0; i < NH && ok; i++)
        if (cudaIpcGetMemHandle(&mine[i], bases[i]) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
        }
    const int64_t HB = (int64_t)sizeof(cudaIpcMemHandle_t) * NH;
    DArray<uint8_t> hs, hr;
    hs.alloc(HB);
    hr.alloc(HB * p);
    DBFS_CUDA(cudaMemcpy(hs.p, mine.data(), HB, cudaMemcpyHostToDevice));
    nccl_allgather_bytes(ctx, hs.p, hr.p, HB);
    DBFS_CUDA(cudaMemcpy(all.data(), hr.p, HB * p, cudaMemcpyDeviceToHost));
    auto agree = [&](int v) {
        DArray<uint32_t> f;
        f.alloc(1);
        uint32_t h = v ? 1u : 0u;
        DBFS_CUDA(cudaMemcpy(f.p, &h, 4, cudaMemcpyHostToDevice));
        nccl_allreduce_u32_sum(ctx, f.p, 1);
        DBFS_CUDA(cudaMemcpy(&h, f.p, 4, cudaMemcpyDeviceToHost));
        return (int)h == p;
    };
    if (!agree(ok)) return;
    std::vector<void *> ptr((size_t)NH * p, nullptr);
    for (int j = 0; j < p; j++)
        for (int i = 0; i < NH; i++) {
            if (j == me) {
                ptr[(size_t)j * NH + i] = bases[i];
                continue;
            }
            void *q = nullptr;
            if (ok && cudaIpcOpenMemHandle(&q, all[(size_t)j * NH + i], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
                g.peer_opened.push_back(q);
                ptr[(size_t)j * NH + i] = q;
            } else {
                cudaGetLastError();
                ok = 0;
            }
        }
    if (!agree(ok)) {
        for (void *q : g.peer_opened) cudaIpcCloseMemHandle(q);
        g.peer_opened.clear();
        return;
    }
    finish_peer_setup(g, ptr);
}

// Peer engine view from every rank's mapped arrays ptr[rank * 9 + i] (i: ctl,
// dnext0, dnext1, dcand, inbox0, nlevel, nparent, dparent, barrier).
static void finish_peer_setup(Graph &g, const std::vector<void *> &ptr) {
    Ctx &ctx = *g.ctx;
    const int p = g.p, me = ctx.rank;
    constexpr int NH = 9;
    WorkerHost &Wk = g.workers[0];
    View V = g.views_h[0];
    V.peer = 1;
    V.dist = 1;
    V.cand_all = 0;  // own candidates only; the min over ranks is taken when outputs are gathered
    V.P_sources = p;
    for (int j = 0; j < p; j++) {
        V.ctl_all[j] = (Ctl *)ptr[(size_t)j * NH + 0];
        V.mask_src[0][j] = (const uint32_t *)ptr[(size_t)j * NH + 1];
        V.mask_src[1][j] = (const uint32_t *)ptr[(size_t)j * NH + 2];
        V.cand_src[j] = (const parent_t *)ptr[(size_t)j * NH + 3];
    }
    // receiver r's inbox: segments by sender, sized by the senders' capacities towards r
    auto seg = [&](int r, int s) {
        int64_t o = 0;
        for (int t = 0; t < s; t++) o += g.cap_all[(size_t)t * p + r];
        return o;
    };
    for (int s = 0; s < p; s++) V.seg_off[s] = seg(me, s);
    for (int o = 0; o < p; o++)
        V.sendbin[o] = o == me ? nullptr : (uint2 *)ptr[(size_t)o * NH + 4] + seg(o, me);
    V.inbox[0] = V.inbox[1] = Wk.inbox0.p;
    g.peer_nlevel.assign(p, nullptr);
    g.peer_nparent.assign(p, nullptr);
    g.peer_dparent.assign(p, nullptr);
    for (int j = 0; j < p; j++) {
        g.peer_nlevel[j] = (int32_t *)ptr[(size_t)j * NH + 5];
        g.peer_nparent[j] = (parent_t *)ptr[(size_t)j * NH + 6];
        g.peer_dparent[j] = (parent_t *)ptr[(size_t)j * NH + 7];
    }
    g.gbar = ptr[NH - 1];  // non-null: the kernel runs the cross-GPU barriers (mailboxes below)
    V.pmail = reinterpret_cast<unsigned long long *>(g.gbar_mem.p);
    for (int j = 0; j < p; j++) V.pmail_peer[j] = reinterpret_cast<unsigned long long *>(ptr[(size_t)j * NH + NH - 1]);
    g.peer_view_h = V;
    g.peer_view.alloc(1);
    g.peer_state = 1;
}

// ------------------------------------------------------------------ driver

// Options of one run into the device views (uploaded on the context stream);
// returns the engine to use (1 host loop, 2 persistent, 3 peer).
static int configure_run(Graph &g, const dbfs_bfs_options &o) {
    Ctx &ctx = *g.ctx;
    ensure_resources(g);
    const int W = g.W;
    const bool parents = o.parent_mode != 0;
    // per-run options into the views
    for (auto &V : g.views_h) {
        V.mode = o.mode;
        V.allow_back = o.allow_switch_back;
        V.parents = parents;
        V.symmetric = g.symmetric;
        V.exec_policy = o.exec_policy;
        V.uniquify = o.uniquify;
        V.local_all2all = o.local_all2all;
        for (int k = 0; k < 4; k++) {
            V.f0[k] = o.factor0[k];
            V.f1[k] = o.factor1[k];
        }
    }
    if (o.uniquify && g.p > 1) {  // seen-bits: [p groups][nw_n] per worker, zeroed once, then by F
        bool fresh = false;
        for (auto &Wk : g.workers)
            if (!Wk.uq.p) {
                Wk.uq.alloc((int64_t)g.p * std::max<int64_t>(nwords(Wk.n_local), 1));
                DBFS_CUDA(cudaMemset(Wk.uq.p, 0, Wk.uq.bytes()));
                fresh = true;
            }
        if (fresh)
            for (int i = 0; i < W; i++) {
                g.views_h[i].uq = g.workers[i].uq.p;
                for (int j = 0; j < W; j++) g.views_h[i].uq_all[g.workers[j].w] = g.workers[j].uq.p;
            }
    } else {
        for (auto &V : g.views_h) V.uniquify = 0;
    }
    for (int i = 0; i < W; i++) {  // the sender-side filter hides records the uniquify accounting must see
        WorkerHost &Wk = g.workers[i];
        g.views_h[i].sent = (g.dist && !g.views_h[i].uniquify && !getenv("DBFS_NO_SEND_FILTER")) ? Wk.sentbits.p : nullptr;
        g.views_h[i].nw_g = nwords(g.n);
    }
    int engine = o.engine;
    if (g.dist) {
        // auto / persistent: one kernel across all GPUs over peer memory when every rank can map its peers
        if (engine != 1) setup_peer(g);
        engine = (engine != 1 && g.peer_state == 1) ? 3 : 1;
    } else {
        if (engine == 0 || engine == 3) engine = 2;
    }
    if (engine == 3) {
        View &P = g.peer_view_h;
        const View &B = g.views_h[0];
        P.mode = B.mode;
        P.allow_back = B.allow_back;
        P.parents = B.parents;
        P.symmetric = B.symmetric;
        P.exec_policy = B.exec_policy;
        P.uniquify = B.uniquify;
        P.uq = B.uq;
        P.sent = B.sent;
        P.nw_g = B.nw_g;
        P.local_all2all = B.local_all2all;
        for (int k = 0; k < 4; k++) {
            P.f0[k] = B.f0[k];
            P.f1[k] = B.f1[k];
        }
        DBFS_CUDA(cudaMemcpyAsync(g.peer_view.p, &P, sizeof(View), cudaMemcpyHostToDevice, ctx.stream));
    }
    DBFS_CUDA(cudaMemcpyAsync(g.views.p, g.views_h.data(), sizeof(View) * W, cudaMemcpyHostToDevice, ctx.stream));
    return engine;
}

static void dist_assemble(Graph &g);
void min_parents_device(Graph &g, int64_t root);

void run_bfs(Graph &g, const dbfs_bfs_options &o, dbfs_run_stats *st) {
    Ctx &ctx = *g.ctx;
    DBFS_CHECK(o.parent_mode >= 0 && o.parent_mode <= 2, DBFS_EINVAL, "parent_mode must be 0, 1 or 2");
    DBFS_CHECK(o.mode == 0 || o.mode == 1, DBFS_EINVAL, "mode must be one of ('bfs', 'dobfs')");
    DBFS_CHECK(0 <= o.source && o.source < g.n, DBFS_ERANGE,
               "source " + std::to_string(o.source) + " out of range [0, " + std::to_string(g.n) + ")");
    const int engine = configure_run(g, o);
    const int W = g.W;
    const bool parents = o.parent_mode != 0;
    uint32_t src_del = 0xffffffffu;
    DBFS_CUDA(cudaMemcpyAsync(&src_del, g.del_id.p + o.source, 4, cudaMemcpyDeviceToHost, ctx.stream));
    for (auto &Wk : g.workers) DBFS_CUDA(cudaMemsetAsync(Wk.ctl.p, 0, sizeof(Ctl), ctx.stream));
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));

    const int64_t launches0 = g_kernel_launches;
    g.last_comm_us.clear();
    const bool assemble = g.p > 1 && !g.dist;
    AsmArgs aa = make_asm(g, parents);
    int iterations = 0;
    bool timeout = false;

    GridBar *bar = (GridBar *)ctx.ensure_scratch(sizeof(GridBar));
    if (engine >= 2) DBFS_CUDA(cudaMemsetAsync(bar, 0, sizeof(GridBar), ctx.stream));
    // everything host-side happens before ev0: the event pair brackets only device work
    if (g.clock_ghz <= 0) {
        int khz = 0;
        cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx.device);
        g.clock_ghz = khz / 1e6;
    }
    set_smem_attrs();
    int pgrid = 0;
    if (engine >= 2) {
        if (g.pgrid <= 0) {
            int bps = 0;
            g.pgrid = persistent_grid(g, &bps);
        }
        pgrid = g.pgrid;
        g.warps_per_worker = (double)pgrid / W * WPB;
    }
    // Distributed: line the ranks up right before the launch.  The persistent
    // kernel's first grid barrier spans all GPUs, so a rank whose host reached
    // the launch early would otherwise spend the others' host skew (python,
    // driver calls: up to ~1 ms) spinning inside its own event window.
    const char *trace_path = engine >= 2 ? getenv("DBFS_TRACE") : nullptr;
    if (trace_path) {
        const int64_t tn = 64 * 8 * (int64_t)std::max(g.pgrid, 1);
        if (g.trace.n != tn) g.trace.alloc(tn);
        DBFS_CUDA(cudaMemset(g.trace.p, 0, g.trace.bytes()));
        for (auto &V : g.views_h) V.trace = g.trace.p;
        g.peer_view_h.trace = g.trace.p;
        DBFS_CUDA(cudaMemcpy(g.views.p, g.views_h.data(), sizeof(View) * W, cudaMemcpyHostToDevice));
        if (engine == 3) DBFS_CUDA(cudaMemcpy(g.peer_view.p, &g.peer_view_h, sizeof(View), cudaMemcpyHostToDevice));
    }
    if (g.dist) nccl_barrier(ctx);
    DBFS_CUDA(cudaEventRecord(ctx.ev0, ctx.stream));
    if (engine >= 2) {
        int grid = pgrid;
        const View *vp = engine == 3 ? g.peer_view.p : g.views.p;
        int64_t src = o.source;
        int rec_cap = g.rec_cap;
        int do_asm = assemble ? 1 : 0;
        GridBar *gb = engine == 3 ? (GridBar *)g.gbar : nullptr;
        int nr = engine == 3 ? g.p : 1;
        const uint32_t *dil = g.del_id.p;
        void *args[] = {(void *)&vp,      (void *)&W,  (void *)&src,    (void *)&src_del, (void *)&bar,
                        (void *)&rec_cap, (void *)&aa, (void *)&do_asm, (void *)&gb,      (void *)&nr,
                        (void *)&dil};
        DBFS_CUDA(cudaLaunchCooperativeKernel((void *)k_bfs_persistent, dim3(grid), dim3(BT), args, sizeof(Smem),
                                              ctx.stream));
        DBFS_LAUNCHED();
        DBFS_CUDA(cudaEventRecord(ctx.ev1, ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
        GridBar hb;
        DBFS_CUDA(cudaMemcpy(&hb, bar, sizeof(hb), cudaMemcpyDeviceToHost));
        timeout = hb.abort != 0;
        Ctl c0;
        DBFS_CUDA(cudaMemcpy(&c0, g.workers[0].ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
        iterations = c0.last_level;
        if (trace_path) {
            std::vector<unsigned long long> tr(g.trace.n);
            DBFS_CUDA(cudaMemcpy(tr.data(), g.trace.p, g.trace.bytes(), cudaMemcpyDeviceToHost));
            // one file per rank when several ranks share a process (device groups)
            const std::string tpath = ctx.local_group ? std::string(trace_path) + "." + std::to_string(ctx.rank)
                                                      : std::string(trace_path);
            if (FILE *f = fopen(tpath.c_str(), "a")) {
                const int nbk = g.pgrid;
                for (int lv = 0; lv < std::min(iterations, 64); lv++)
                    for (int ph = 0; ph < 8; ph++)
                        for (int b = 0; b < nbk; b++) {
                            const unsigned long long t = tr[((size_t)lv * 8 + ph) * nbk + b];
                            if (t) fprintf(f, "%d %lld %d %d %d %.3f\n", ctx.rank, (long long)o.source, lv, ph, b,
                                           (double)(t - c0.t_start) / 1e3);
                        }
                fclose(f);
            }
            for (auto &V : g.views_h) V.trace = nullptr;
            g.peer_view_h.trace = nullptr;
        }
        if (engine == 3) {
            g.assembled = false;  // outputs stay distributed until fetched (dist_assemble)
            if (timeout) g.peer_state = -1;  // barrier state unknown: later runs use the NCCL level loop
        }
    } else {
        const int grid = std::max(W, (ctx.num_sms * 4 / W) * W);
        g.warps_per_worker = (double)grid / W * WPB;
        k_init<<<grid, BT, 0, ctx.stream>>>(g.views.p, W);
        DBFS_LAUNCHED();
        k_seed<<<W, 32, 0, ctx.stream>>>(g.views.p, W, o.source, src_del);
        DBFS_LAUNCHED();
        std::vector<Ctl> hc(W);
        int L = 0;
        if (g.dist) {
            std::vector<IterRec> recs;
            for (L = 0;; L++)
                if (!dist_level(g, L, grid, recs)) break;
            iterations = L;
            for (size_t i = 0; i < recs.size(); i++)
                DBFS_CUDA(cudaMemcpyAsync(g.workers[0].rec.p + i, &recs[i], sizeof(IterRec), cudaMemcpyHostToDevice,
                                          ctx.stream));
        }
        for (; !g.dist; L++) {
            k_visit<<<grid, BT, sizeof(Smem), ctx.stream>>>(g.views.p, W, L);
            DBFS_LAUNCHED();
            {
                k_finish<<<grid, BT, sizeof(Smem), ctx.stream>>>(g.views.p, W, L, F_DELEGATES | F_NORMALS);
                DBFS_LAUNCHED();
            }
            for (int i = 0; i < W; i++)
                DBFS_CUDA(cudaMemcpyAsync(&hc[i], g.workers[i].ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx.stream));
            DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
            // per-iteration record for level L (host copy of the device rule)
            if (L < g.rec_cap) {
                for (int i = 0; i < W; i++) {
                    IterRec r{};
                    make_record(g.views_h[i], hc[i], L, r);
                    DBFS_CUDA(cudaMemcpyAsync(g.workers[i].rec.p + L, &r, sizeof(r), cudaMemcpyHostToDevice,
                                              ctx.stream));
                }
            }
            unsigned long long act = hc[0].s[L % 3].new_del;
            for (int i = 0; i < W; i++) act += hc[i].s[(L + 1) % 3].nfront + hc[i].s[L % 3].records;
            if (!act) break;
        }
        if (!g.dist) iterations = L + 1;
        if (g.dist) {
            g.assembled = false;  // outputs stay distributed until fetched (dist_assemble)
        } else if (assemble) {
            k_assemble<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(aa);
            DBFS_LAUNCHED();
        }
        DBFS_CUDA(cudaEventRecord(ctx.ev1, ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    DBFS_CUDA(cudaGetLastError());
    DBFS_CHECK(!timeout, DBFS_ETIMEOUT, "device watchdog fired in the persistent BFS kernel");
    int64_t reached = -1;
    if (!g.dist && st) {  // after ev1: not part of the timed traversal
        unsigned long long *cnt = (unsigned long long *)g.dist_scratch.p + 2 * (g.p + 3) * (g.p + 1) + 8;
        DBFS_CUDA(cudaMemsetAsync(cnt, 0, 8, ctx.stream));
        k_count_reached<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(g.levels_dev(), g.n, cnt);
        DBFS_LAUNCHED();
        unsigned long long h = 0;
        DBFS_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
        reached = (int64_t)h;
    }
    float ms = 0.f;
    DBFS_CUDA(cudaEventElapsedTime(&ms, ctx.ev0, ctx.ev1));

    // collect per-iteration records
    g.last_iterations = iterations;
    g.last_truncated = iterations > g.rec_cap;
    int nrec = std::min(iterations, g.rec_cap);
    g.last_rec.assign((size_t)nrec * W, IterRec{});
    for (int i = 0; i < W; i++) {
        std::vector<IterRec> tmp(nrec);
        if (nrec) DBFS_CUDA(cudaMemcpy(tmp.data(), g.workers[i].rec.p, sizeof(IterRec) * nrec, cudaMemcpyDeviceToHost));
        for (int L = 0; L < nrec; L++) g.last_rec[(size_t)L * W + i] = tmp[L];
    }
    g.last_source = o.source;
    g.last_parent_mode = o.parent_mode;
    g.last_valid = true;
    g.last_mode = o.mode;
    g.last_la = o.local_all2all;
    g.last_uq = o.uniquify;
    if (o.parent_mode == 2) {  // deterministic min-ID tree, after the timed traversal
        dist_assemble(g);
        min_parents_device(g, o.source);
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    if (st) {
        memset(st, 0, sizeof(*st));
        st->iterations = iterations;
        st->reached = reached;
        run_accounting(g, g.last_rec.data(), nrec, iterations, g.last_la, g.last_uq, st);
        st->device_ms = ms;
        st->kernel_launches = g_kernel_launches - launches0;
        st->per_iteration_truncated = g.last_truncated;
        st->engine_used = engine;
        int64_t wire = 0;
        for (int L = 0; L < nrec; L++)
            for (int i = 0; i < W; i++) {
                const IterRec &r = g.last_rec[(size_t)L * W + i];
                wire += (int64_t)r.records * 8;
                if (r.new_del && g.p > 1) wire += (int64_t)(g.p - 1) * nwords(g.d) * 4 / W;
            }
        st->wire_bytes = wire;
        int64_t rows = 0, work = 0;
        for (int L = 0; L < nrec; L++)
            for (int i = 0; i < W; i++) {
                const IterRec &r = g.last_rec[(size_t)L * W + i];
                rows += (int64_t)r.rows;
                for (int k = 0; k < 4; k++) work += (int64_t)r.work[k];
            }
        st->rows_touched = rows;
        st->work_inspections = work;
        // library-side copies of this call: views + options up, control block / records down
        st->h2d_bytes = (int64_t)(sizeof(View) * W);
        if (engine >= 2) {
            Ctl c0;
            DBFS_CUDA(cudaMemcpy(&c0, g.workers[0].ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
            st->init_us = (double)(c0.t_seeded - c0.t_start) / 1e3;
        }
        st->d2h_bytes = 4 + (int64_t)sizeof(Ctl) + (int64_t)(sizeof(IterRec) * nrec * W);
    }
    if (g.dist && st) {
        // inspections are per rank; sum over ranks
        DArray<int64_t> t;
        t.alloc(8);
        int64_t h[8];
        for (int k = 0; k < 4; k++) {
            h[2 * k] = st->inspections[k][0];
            h[2 * k + 1] = st->inspections[k][1];
        }
        DBFS_CUDA(cudaMemcpy(t.p, h, sizeof(h), cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx, t.p, 8, 0);
        DBFS_CUDA(cudaMemcpy(h, t.p, sizeof(h), cudaMemcpyDeviceToHost));
        for (int k = 0; k < 4; k++) {
            st->inspections[k][0] = h[2 * k];
            st->inspections[k][1] = h[2 * k + 1];
        }
        int64_t bwd = st->inspections[KIND_ND][BWD] + st->inspections[KIND_DD][BWD];
        st->b_measured = g.d ? (double)bwd / (double)(g.d * g.p) : 0.0;
    }
}

// ----------------------------------------------------------------- results

// Distributed runs keep each rank's normals local (plus the replicated
// delegates); the global depth/parent arrays are gathered only on demand.
static void dist_assemble(Graph &g) {
    if (!g.dist || g.assembled) return;
    Ctx &ctx = *g.ctx;
    const bool parents = g.last_parent_mode != 0;
    AsmArgs aa = make_asm(g, parents);
    WorkerHost &Wk = g.workers[0];
    if (g.peer_state == 1) {
        // peer-mapped: read every rank's normals and delegate candidates over NVLink,
        // then a barrier so nobody starts the next BFS while a peer still reads
        for (int w = 0; w < g.p; w++) {
            aa.nlevel[w] = g.peer_nlevel[w];
            aa.nparent[w] = g.peer_nparent[w];
            aa.dpar_src[w] = g.peer_dparent[w];
        }
        aa.n_dpar = g.p;
        k_assemble<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(aa);
        DBFS_LAUNCHED();
        nccl_barrier(ctx);
        g.assembled = true;
        return;
    }
    // delegate parents: each rank holds the candidate its own edges found (or
    // INT64_MAX) -> the tree takes the minimum over ranks
    if (parents && g.d) nccl_allreduce_i32_min(ctx, Wk.dparent.p, g.d);
    int64_t stride = ceil_div(g.n, g.p);
    DArray<int32_t> &lv = g.asm_lv, &mylv = g.asm_mylv;
    DArray<parent_t> &pv = g.asm_pv, &mypv = g.asm_mypv;
    if (lv.n != stride * g.p) {
        lv.alloc(stride * g.p);
        pv.alloc(stride * g.p);
        mylv.alloc(stride);
        mypv.alloc(stride);
    }
    DBFS_CUDA(cudaMemsetAsync(mylv.p, 0xff, 4 * stride, ctx.stream));
    DBFS_CUDA(cudaMemsetAsync(mypv.p, 0xff, sizeof(parent_t) * stride, ctx.stream));
    if (Wk.n_local) {
        DBFS_CUDA(cudaMemcpyAsync(mylv.p, Wk.nlevel.p, 4 * Wk.n_local, cudaMemcpyDeviceToDevice, ctx.stream));
        DBFS_CUDA(cudaMemcpyAsync(mypv.p, Wk.nparent.p, sizeof(parent_t) * Wk.n_local, cudaMemcpyDeviceToDevice,
                                  ctx.stream));
    }
    nccl_allgather_bytes(ctx, mylv.p, lv.p, 4 * stride);
    if (parents) nccl_allgather_bytes(ctx, mypv.p, pv.p, sizeof(parent_t) * stride);
    for (int w = 0; w < g.p; w++) {
        aa.nlevel[w] = lv.p + (int64_t)w * stride;
        aa.nparent[w] = pv.p + (int64_t)w * stride;
    }
    k_assemble<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(aa);
    DBFS_LAUNCHED();
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    g.assembled = true;
}

__global__ void k_count_reached(const int32_t *__restrict__ lv, int64_t n, unsigned long long *out) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += lv[i] >= 0;
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(out, c);
}

void fetch_result(Graph &g, int32_t *levels, int64_t *parents) {
    DBFS_CHECK(g.last_valid, DBFS_EINVAL, "no BFS result on device");
    Ctx &ctx = *g.ctx;
    dist_assemble(g);
    if (levels) DBFS_CUDA(cudaMemcpyAsync(levels, g.levels_dev(), 4 * g.n, cudaMemcpyDeviceToHost, ctx.stream));
    if (parents) {
        DBFS_CHECK(g.last_parent_mode != 0, DBFS_EINVAL, "last BFS ran without parents");
        DBFS_CUDA(cudaMemcpyAsync(parents, g.parents_dev64(), 8 * g.n, cudaMemcpyDeviceToHost, ctx.stream));
    }
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

// Pipelined roots (dbfs_bfs_batch): after root k traverses, its depth/parent
// arrays are copied device-to-device into staging buffer k%2 (a few tens of
// us at HBM speed) and then to the caller's host buffers on a non-blocking
// copy stream, so the PCIe transfer of root k overlaps the traversal of root
// k+1.  Staging buffer b is reused only after its previous D2H has finished.
static void ensure_copy_stream(Ctx &ctx) {
    if (ctx.copy_stream) return;
    DBFS_CUDA(cudaStreamCreateWithFlags(&ctx.copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
        DBFS_CUDA(cudaEventCreateWithFlags(&ctx.ev_ready[b], cudaEventDisableTiming));
        DBFS_CUDA(cudaEventCreateWithFlags(&ctx.ev_done[b], cudaEventDisableTiming));
    }
    for (int h = 0; h < 3; h++) DBFS_CUDA(cudaEventCreateWithFlags(&ctx.ev_hdone[h], cudaEventDisableTiming));
}

// Assembly arguments of the outputs a batch copies: the whole graph, or in a
// distributed graph with `local` the vertices this rank owns (v mod p == rank),
// read from the peer-mapped (or NCCL min-reduced) delegate candidates.
static AsmArgs batch_asm(Graph &g, bool parents, bool local) {
    AsmArgs aa = make_asm(g, parents);
    if (g.dist) {
        if (g.peer_state == 1) {
            for (int w = 0; w < g.p; w++) {
                aa.nlevel[w] = g.peer_nlevel[w];
                aa.nparent[w] = g.peer_nparent[w];
                aa.dpar_src[w] = g.peer_dparent[w];
            }
            aa.n_dpar = g.p;
        } else {
            WorkerHost &Wk = g.workers[0];
            aa.nlevel[Wk.w] = Wk.nlevel.p;
            aa.nparent[Wk.w] = Wk.nparent.p;
        }
    }
    if (local && g.dist) {
        aa.first = g.ctx->rank;
        aa.step = g.p;
        aa.count = g.workers[0].n_local;
    }
    return aa;
}

// Host side of the compact transfer: int8 depth / int32 parent -> the caller's
// int32 / int64 arrays (sign extension keeps -1), on every host core.
static void widen_result(const int8_t *l8, const int32_t *p32, int64_t n, int32_t *lv, int64_t *pa, int nthreads) {
    widen_host(l8, p32, n, lv, pa, nthreads);  // widen.cpp
}

// CPUs this process may run on (its affinity mask, as nproc reports; the
// machine's logical CPU count can be far larger inside a container).
static int usable_cpus() {
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, (int)CPU_COUNT(&set));
    return std::max(1, (int)std::thread::hardware_concurrency());
}

static void ensure_compact_staging(Graph &g, int64_t nout) {
    if (g.hstage_n < nout) {
        for (int h = 0; h < 3; h++) {
            if (g.hstage8[h]) cudaFreeHost(g.hstage8[h]);
            if (g.hstage32[h]) cudaFreeHost(g.hstage32[h]);
            g.hstage8[h] = nullptr;
            g.hstage32[h] = nullptr;
        }
        for (int h = 0; h < 3; h++) {
            DBFS_CUDA(cudaHostAlloc((void **)&g.hstage8[h], std::max<int64_t>(nout, 1), cudaHostAllocDefault));
            DBFS_CUDA(cudaHostAlloc((void **)&g.hstage32[h], 4 * std::max<int64_t>(nout, 1), cudaHostAllocDefault));
        }
        g.hstage_n = nout;
    }
    if (!g.hesc) DBFS_CUDA(cudaHostAlloc((void **)&g.hesc, 3 * sizeof(unsigned), cudaHostAllocDefault));
    if (g.esc.n < 2) g.esc.alloc(2);
}

int64_t batch_output_count(const Graph &g, bool local) { return (local && g.dist) ? g.workers[0].n_local : g.n; }

void run_bfs_batch(Graph &g, const dbfs_bfs_options &o0, const int64_t *roots, int64_t count, int32_t *const *levels,
                   int64_t *const *parents, int local, int compact_req, dbfs_run_stats *st) {
    Ctx &ctx = *g.ctx;
    const double tentry =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    DBFS_CHECK(o0.mode == 0 || o0.mode == 1, DBFS_EINVAL, "mode must be one of ('bfs', 'dobfs')");
    for (int64_t k = 0; k < count; k++)
        DBFS_CHECK(0 <= roots[k] && roots[k] < g.n, DBFS_ERANGE,
                   "source " + std::to_string(roots[k]) + " out of range [0, " + std::to_string(g.n) + ")");
    if (count == 0) return;
    DBFS_CHECK(o0.parent_mode >= 0 && o0.parent_mode <= 2, DBFS_EINVAL, "parent_mode must be 0, 1 or 2");
    DBFS_CHECK(o0.parent_mode != 2 || !g.dist, DBFS_EINVAL,
               "min-ID parents (parent_mode 2) are not available in distributed batches; use dbfs_bfs");
    ensure_copy_stream(ctx);
    const bool want_par = parents != nullptr && o0.parent_mode != 0;
    const int64_t nout = batch_output_count(g, local != 0);
    for (int b = 0; b < 2; b++) {
        if (levels && g.stage_lv[b].n < nout) g.stage_lv[b].alloc(std::max<int64_t>(nout, 1));
        if (want_par && g.stage_pv[b].n < nout) g.stage_pv[b].alloc(std::max<int64_t>(nout, 1));
    }
    const int engine = configure_run(g, o0);
    // root k's outputs -> staging buffer k%2 (kernels only on ctx.stream), then
    // D2H on the copy stream; staging b is reused once its previous D2H is done
    auto stage_and_copy = [&](int64_t k, const AsmArgs *asm_src) {
        const int b = (int)(k & 1);
        if (k >= 2) DBFS_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.ev_done[b], 0));
        const int blocks = ctx.num_sms * 4;
        const bool lv = levels && levels[k], pa = want_par && parents[k];
        if (asm_src) {
            AsmArgs aa = *asm_src;
            aa.glevel = g.stage_lv[b].p;
            aa.gparent = nullptr;
            aa.gparent64 = pa ? g.stage_pv[b].p : nullptr;
            aa.parents = pa;
            k_assemble<<<blocks, BT, 0, ctx.stream>>>(aa);
            DBFS_LAUNCHED();
        } else {
            if (lv) {
                k_copy_bytes<<<blocks, 256, 0, ctx.stream>>>((const uint8_t *)g.levels_dev(),
                                                             (uint8_t *)g.stage_lv[b].p, 4 * nout);
                DBFS_LAUNCHED();
            }
            if (pa) {
                k_widen_parents<<<blocks, 256, 0, ctx.stream>>>(g.parents_dev(), nout, g.stage_pv[b].p);
                DBFS_LAUNCHED();
            }
        }
        DBFS_CUDA(cudaEventRecord(ctx.ev_ready[b], ctx.stream));
        DBFS_CUDA(cudaStreamWaitEvent(ctx.copy_stream, ctx.ev_ready[b], 0));
        if (lv) DBFS_CUDA(cudaMemcpyAsync(levels[k], g.stage_lv[b].p, 4 * nout, cudaMemcpyDeviceToHost, ctx.copy_stream));
        if (pa)
            DBFS_CUDA(cudaMemcpyAsync(parents[k], g.stage_pv[b].p, 8 * nout, cudaMemcpyDeviceToHost, ctx.copy_stream));
        DBFS_CUDA(cudaEventRecord(ctx.ev_done[b], ctx.copy_stream));
        if (st) st[k].d2h_bytes += (lv ? 4 * nout : 0) + (pa ? 8 * nout : 0);
    };
    if (engine == 1) {
        // host-driven level loop: run_bfs per root (its host round trips bound
        // the overlap); delegate parents min-reduced over ranks before assembly
        for (int64_t k = 0; k < count; k++) {
            dbfs_bfs_options o = o0;
            o.source = roots[k];
            run_bfs(g, o, st ? &st[k] : nullptr);
            if (g.dist) {
                if (o0.parent_mode && g.d) nccl_allreduce_i32_min(ctx, g.workers[0].dparent.p, g.d);
                AsmArgs aa = batch_asm(g, o0.parent_mode != 0, local != 0);
                stage_and_copy(k, &aa);
                g.assembled = false;
            } else {
                stage_and_copy(k, nullptr);
            }
        }
        DBFS_CUDA(cudaStreamSynchronize(ctx.copy_stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    // Persistent engines (one GPU, or one per rank over peer memory): every
    // root is enqueued without a host round trip -- prep kernel (control
    // block, grid barrier), the traversal (the source's delegate id looked up
    // on device), an info kernel (iterations, watchdog), the assembly / staging
    // copy; the D2H runs on the copy stream.  Distributed ranks pass an NCCL
    // all-reduce (a device-side barrier) before each traversal, so no rank
    // overwrites its state while a peer still assembles from it.
    const int W = g.W;
    const bool peer = engine == 3;
    const bool compact = compact_req && levels && g.n < ((int64_t)1 << 31);
    const bool btrace = getenv("DBFS_BATCH_TRACE") != nullptr;
    auto now_ms = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double tb0 = now_ms();
    double t_wait = 0, t_widen = 0, t_asm = 0;
    if (btrace && g.batch_asm_evs.empty())
        for (int i = 0; i < 4; i++) {
            cudaEvent_t e;
            DBFS_CUDA(cudaEventCreate(&e));
            g.batch_asm_evs.push_back(e);
        }
    if (compact) ensure_compact_staging(g, nout);
    set_smem_attrs();
    if (g.pgrid <= 0) {
        int bps = 0;
        g.pgrid = persistent_grid(g, &bps);
    }
    int grid = g.pgrid;
    g.warps_per_worker = (double)grid / W * WPB;
    AsmArgs aa = make_asm(g, o0.parent_mode != 0);
    int do_asm = (!g.dist && g.p > 1) ? 1 : 0;
    AsmArgs out_asm = batch_asm(g, o0.parent_mode != 0, local != 0);
    // per-root iteration records (comm accounting / inspections of every root,
    // dbfs_run_stats.accounting_valid): staged on device after each traversal,
    // copied on the copy stream with the root's outputs
    const int rmax = std::min(g.rec_cap, 64);
    const bool want_rec = o0.record_iterations && st;
    // batch scratch is kept with the graph and only grows: cudaMalloc /
    // cudaHostAlloc / cudaFree inside the call would synchronise and stall
    DArray<IterRec> &drec = g.batch_drec;
    if (want_rec && drec.n < (int64_t)count * rmax * W) {
        drec.alloc((int64_t)count * rmax * W);
        if (g.batch_hrec) cudaFreeHost(g.batch_hrec);
        g.batch_hrec = nullptr;
        DBFS_CUDA(cudaHostAlloc((void **)&g.batch_hrec, drec.bytes(), cudaHostAllocDefault));
    }
    IterRec *const hrec = g.batch_hrec;
    auto copy_recs = [&](int64_t k) {
        if (!want_rec) return;
        const size_t per = (size_t)rmax * W;
        DBFS_CUDA(cudaMemcpyAsync(hrec + k * per, drec.p + k * per, per * sizeof(IterRec), cudaMemcpyDeviceToHost,
                                  ctx.copy_stream));
    };
    void *flag = (char *)ctx.ensure_scratch(256) + 128;  // NCCL barrier word (the grid barrier is at offset 0)
    GridBar *bar = (GridBar *)ctx.ensure_scratch(sizeof(GridBar));
    DArray<int2> &info = g.batch_info;
    if (info.n < count) info.alloc(count);
    while ((int64_t)g.batch_evs.size() < 2 * count) {
        cudaEvent_t e;
        DBFS_CUDA(cudaEventCreate(&e));
        g.batch_evs.push_back(e);
    }
    const std::vector<cudaEvent_t> &evs = g.batch_evs;
    if (peer) nccl_barrier(ctx);
    const int64_t launches0 = g_kernel_launches;
    const View *vp = peer ? g.peer_view.p : g.views.p;
    int rec_cap = g.rec_cap;
    GridBar *gb = peer ? (GridBar *)g.gbar : nullptr;
    int nr = peer ? g.p : 1;
    const uint32_t *dil = g.del_id.p;
    uint32_t sdel = SRC_DEL_LOOKUP;
    auto enqueue_root = [&](int64_t k, unsigned *esc_k) {
        int64_t src = roots[k];
        if (peer && k > 0) nccl_allreduce_async(ctx, flag);
        k_batch_prep<<<W, 256, 0, ctx.stream>>>(g.views.p, bar);
        DBFS_LAUNCHED();
        DBFS_CUDA(cudaEventRecord(evs[2 * k], ctx.stream));
        void *args[] = {(void *)&vp,      (void *)&W,  (void *)&src,    (void *)&sdel, (void *)&bar,
                        (void *)&rec_cap, (void *)&aa, (void *)&do_asm, (void *)&gb,   (void *)&nr,
                        (void *)&dil};
        DBFS_CUDA(cudaLaunchCooperativeKernel((void *)k_bfs_persistent, dim3(grid), dim3(BT), args, sizeof(Smem),
                                              ctx.stream));
        DBFS_LAUNCHED();
        DBFS_CUDA(cudaEventRecord(evs[2 * k + 1], ctx.stream));
        if (o0.parent_mode == 2) min_parents_device(g, src);  // untimed: after the traversal's end event
        if (want_rec) {
            k_stage_recs<<<dim3(STAGE_BLOCKS, W), 256, 0, ctx.stream>>>(g.views.p, W, rmax, drec.p + (size_t)k * rmax * W);
            DBFS_LAUNCHED();
        }
        if (esc_k && k >= 2) DBFS_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.ev_done[k & 1], 0));
        k_batch_info<<<1, 1, 0, ctx.stream>>>(g.workers[0].ctl.p, bar, info.p + k, esc_k);
        DBFS_LAUNCHED();
    };
    std::vector<int64_t> rerun;
    if (!compact) {
        for (int64_t k = 0; k < count; k++) {
            enqueue_root(k, nullptr);
            stage_and_copy(k, g.dist ? &out_asm : nullptr);
            copy_recs(k);  // the copy stream already waits for this root's staging
        }
    } else {
        // Compact transfers: the depth travels as int8 (9 bytes per vertex on the
        // wire instead of 12; parents go straight into the caller's int64 array)
        // and the host widens it into the caller's int32 array on every core
        // (sign extension restores -1) while the GPU runs later roots.  Three
        // pinned host staging sets: root k's D2H lands in set k%3, whose previous
        // root (k-3) the host widened one iteration earlier.  A root with a depth
        // >= 127 is re-run with full arrays after the batch.
        const int blocks = ctx.num_sms * 4;
        // the host's cores shared by the ranks on it (launchers such as torchrun
        // pin OMP_NUM_THREADS to 1, so the count is set here explicitly)
        // Whole-graph outputs in a distributed batch go to one receiving rank
        // (benchmark(), device groups: rank 0), whose host widens n depths per
        // root while the other ranks only wait on their GPUs: it takes the cores.
        const bool sole_receiver = g.dist && !local;
        const int host_threads =
            sole_receiver ? std::max(1, std::min(32, usable_cpus() - (ctx.nranks - 1)))
                          : std::max(1, std::min(16, usable_cpus() / std::max(1, g.dist ? ctx.nranks : 1)));
        // depths sent as int32 per root (rest int8): only into page-locked caller
        // arrays (a pageable destination would make the copy synchronous)
        const char *fs = getenv("DBFS_COMPACT_SPLIT");
        const double split_frac = fs ? atof(fs) : 0.0;  // widen.cpp keeps up with the GPU (s24: 0.48 vs 0.83 ms)
        std::vector<int64_t> split((size_t)count, 0);
        for (int64_t k = 0; k < count; k++) {
            if (!levels[k]) continue;
            cudaPointerAttributes pa{};
            if (cudaPointerGetAttributes(&pa, levels[k]) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if (pa.type != cudaMemoryTypeHost) continue;
            int64_t sp = (int64_t)(split_frac * (double)nout);
            sp -= sp % 64;  // keeps the int8 part 16-byte aligned for k_pack_result
            split[(size_t)k] = std::max<int64_t>(0, std::min(sp, nout));
        }
        auto split_of = [&](int64_t k) { return split[(size_t)k]; };
        for (int64_t k = 0; k < count + 2; k++) {
            if (k < count) {
                const int b = (int)(k & 1);
                enqueue_root(k, g.esc.p + b);
                int8_t *l8 = reinterpret_cast<int8_t *>(g.stage_lv[b].p);
                if (g.dist && !levels[k] && !(want_par && parents[k])) {
                    // this rank receives nothing for root k (e.g. benchmark() on ranks > 0)
                } else if (g.dist) {
                    AsmArgs ca = out_asm;
                    ca.split = split_of(k);
                    ca.glevel = g.stage_lv[b].p;
                    ca.glevel8 = l8 + 4 * ca.split;
                    ca.gparent = nullptr;  // parents travel as int64 (no host widening)
                    ca.gparent64 = want_par ? g.stage_pv[b].p : nullptr;
                    ca.parents = want_par;
                    ca.esc = g.esc.p + b;
                    if (btrace) DBFS_CUDA(cudaEventRecord(g.batch_asm_evs[2 * (k & 1)], ctx.stream));
                    k_assemble<<<blocks, BT, 0, ctx.stream>>>(ca);
                    if (btrace) {
                        DBFS_CUDA(cudaEventRecord(g.batch_asm_evs[2 * (k & 1) + 1], ctx.stream));
                        DBFS_CUDA(cudaEventSynchronize(g.batch_asm_evs[2 * (k & 1) + 1]));
                        float am = 0;
                        cudaEventElapsedTime(&am, g.batch_asm_evs[2 * (k & 1)], g.batch_asm_evs[2 * (k & 1) + 1]);
                        t_asm += am;
                    }
                    DBFS_LAUNCHED();
                } else {
                    // the first split_of(k) depths travel as int32 straight into the
                    // caller's (page-locked) array, the rest as int8 for the host to
                    // widen: PCIe and the host's memory bandwidth share the work
                    const int64_t sp = split_of(k);
                    if (sp) {
                        k_copy_bytes<<<blocks, 256, 0, ctx.stream>>>((const uint8_t *)g.levels_dev(),
                                                                     (uint8_t *)g.stage_lv[b].p, 4 * sp);
                        DBFS_LAUNCHED();
                    }
                    k_pack_result<<<blocks, 256, 0, ctx.stream>>>(g.levels_dev() + sp, nout - sp, l8 + 4 * sp,
                                                                  g.esc.p + b);
                    DBFS_LAUNCHED();
                    if (want_par) {
                        k_widen_parents<<<blocks, 256, 0, ctx.stream>>>(g.parents_dev(), nout, g.stage_pv[b].p);
                        DBFS_LAUNCHED();
                    }
                }
                DBFS_CUDA(cudaEventRecord(ctx.ev_ready[b], ctx.stream));
                // root k's D2H is queued at once: the copy engine runs back to back
                // while the host widens root k-2 (host set k%3 last held root k-3)
                const int hb = (int)(k % 3);
                DBFS_CUDA(cudaStreamWaitEvent(ctx.copy_stream, ctx.ev_ready[b], 0));
                const int64_t sp = split_of(k);
                if (sp)
                    DBFS_CUDA(cudaMemcpyAsync(levels[k], g.stage_lv[b].p, 4 * sp, cudaMemcpyDeviceToHost,
                                              ctx.copy_stream));
                if (levels[k])
                    DBFS_CUDA(cudaMemcpyAsync(g.hstage8[hb],
                                              reinterpret_cast<const int8_t *>(g.stage_lv[b].p) + 4 * sp, nout - sp,
                                              cudaMemcpyDeviceToHost, ctx.copy_stream));
                if (want_par && parents[k])  // straight into the caller's array
                    DBFS_CUDA(cudaMemcpyAsync(parents[k], g.stage_pv[b].p, 8 * nout, cudaMemcpyDeviceToHost,
                                              ctx.copy_stream));
                DBFS_CUDA(cudaMemcpyAsync(g.hesc + hb, g.esc.p + b, 4, cudaMemcpyDeviceToHost, ctx.copy_stream));
                copy_recs(k);
                DBFS_CUDA(cudaEventRecord(ctx.ev_done[b], ctx.copy_stream));
                DBFS_CUDA(cudaEventRecord(ctx.ev_hdone[hb], ctx.copy_stream));
                if (st) st[k].d2h_bytes += (levels[k] ? nout + 3 * sp : 0) + (want_par && parents[k] ? 8 * nout : 0) + 4;
            }
            if (k >= 2) {
                const int64_t j = k - 2;
                const int hb = (int)(j % 3);
                const double tw0 = btrace ? now_ms() : 0;
                DBFS_CUDA(cudaEventSynchronize(ctx.ev_hdone[hb]));
                const double tw1 = btrace ? now_ms() : 0;
                if (g.hesc[hb]) rerun.push_back(j);
                else if (levels[j]) {
                    const int64_t sp = split_of(j);
                    widen_result(g.hstage8[hb], nullptr, nout - sp, levels[j] + sp, nullptr, host_threads);
                }
                if (btrace) {
                    t_wait += tw1 - tw0;
                    t_widen += now_ms() - tw1;
                }
            }
        }
    }
    if (peer) nccl_allreduce_async(ctx, flag);  // peers may read this rank's arrays until every assembly is done
    DBFS_CUDA(cudaStreamSynchronize(ctx.copy_stream));
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    if (compact) {
        // roots with an escaped depth (>= 127) again, with full arrays; every rank
        // of a distributed run takes part in the same re-runs
        std::vector<int64_t> fl(count, 0);
        for (int64_t j : rerun) fl[j] = 1;
        if (g.dist) {
            DArray<int64_t> d;
            d.alloc(count);
            DBFS_CUDA(cudaMemcpy(d.p, fl.data(), 8 * count, cudaMemcpyHostToDevice));
            nccl_allreduce_i64(ctx, d.p, count, 0);
            DBFS_CUDA(cudaMemcpy(fl.data(), d.p, 8 * count, cudaMemcpyDeviceToHost));
        }
        for (int64_t j = 0; j < count; j++) {
            if (!fl[j]) continue;
            dbfs_bfs_options o = o0;
            o.source = roots[j];
            run_bfs(g, o, nullptr);
            if (g.dist) {
                AsmArgs fa = batch_asm(g, want_par, local != 0);
                fa.glevel = g.stage_lv[0].p;
                fa.gparent = nullptr;
                fa.gparent64 = want_par ? g.stage_pv[0].p : nullptr;
                fa.parents = want_par;
                k_assemble<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(fa);
                DBFS_LAUNCHED();
                if (peer) nccl_barrier(ctx);
                DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
                if (levels[j]) DBFS_CUDA(cudaMemcpy(levels[j], g.stage_lv[0].p, 4 * nout, cudaMemcpyDeviceToHost));
                if (want_par && parents[j])
                    DBFS_CUDA(cudaMemcpy(parents[j], g.stage_pv[0].p, 8 * nout, cudaMemcpyDeviceToHost));
                g.assembled = false;
            } else {
                fetch_result(g, levels[j], want_par ? parents[j] : nullptr);
            }
        }
    }
    if (btrace) {
        fprintf(stderr, "[batch] %lld roots: setup %.2f ms, loop+sync %.2f ms (waits %.2f, widening %.2f)\n",
                (long long)count, tb0 - tentry, now_ms() - tb0, t_wait, t_widen);
        double tb = 0, tg = 0;  // device: traversals, and what runs between them
        for (int64_t k = 0; k < count; k++) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, evs[2 * k], evs[2 * k + 1]);
            if (k + 1 < count) cudaEventElapsedTime(&b, evs[2 * k + 1], evs[2 * k + 2]);
            tb += a;
            tg += b;
        }
        fprintf(stderr, "[batch] device: traversals %.3f ms/root, between traversals %.3f ms/root (assembly %.3f)\n",
                tb / count, count > 1 ? tg / (count - 1) : 0.0, t_asm / count);
    }
    std::vector<int2> hi(count);
    DBFS_CUDA(cudaMemcpy(hi.data(), info.p, sizeof(int2) * count, cudaMemcpyDeviceToHost));
    const int64_t launches = g_kernel_launches - launches0;
    bool aborted = false;
    for (int64_t k = 0; k < count; k++) {
        aborted |= hi[k].y != 0;
        if (st) {
            float ms = 0.f;
            DBFS_CUDA(cudaEventElapsedTime(&ms, evs[2 * k], evs[2 * k + 1]));
            dbfs_run_stats &r = st[k];
            const int64_t d2h = r.d2h_bytes;
            memset(&r, 0, sizeof(r));
            r.iterations = hi[k].x;
            r.reached = -1;
            r.device_ms = ms;
            r.kernel_launches = launches / count;
            r.engine_used = engine;
            r.per_iteration_truncated = 1;  // records are not collected in batch mode
            r.h2d_bytes = k == 0 ? (int64_t)(sizeof(View) * W) : 0;
            r.d2h_bytes = d2h + (int64_t)sizeof(int2);
            if (want_rec) {
                const int64_t nrec = std::min<int64_t>(hi[k].x, rmax);
                run_accounting(g, hrec + (size_t)k * rmax * W, nrec, hi[k].x, o0.local_all2all,
                               o0.uniquify && g.p > 1, &r);
                r.d2h_bytes += (int64_t)((size_t)rmax * W * sizeof(IterRec));
                int64_t work = 0, rows = 0;
                for (int64_t it = 0; it < nrec; it++)
                    for (int i = 0; i < W; i++) {
                        const IterRec &x = hrec[((size_t)k * rmax + it) * W + i];
                        rows += (int64_t)x.rows;
                        for (int q = 0; q < 4; q++) work += (int64_t)x.work[q];
                    }
                r.rows_touched = rows;
                r.work_inspections = work;
            }
        }
    }
    if (want_rec && g.dist && !aborted) {
        // one worker per rank: inspections and normal-record bytes are per-rank
        // partial sums (mask bytes and S' follow the replicated delegate finds)
        constexpr int F = 11;
        std::vector<int64_t> h((size_t)count * F, 0);
        for (int64_t k = 0; k < count; k++) {
            const dbfs_run_stats &r = st[k];
            for (int q = 0; q < 4; q++) {
                h[k * F + 2 * q] = r.inspections[q][0];
                h[k * F + 2 * q + 1] = r.inspections[q][1];
            }
            h[k * F + 8] = r.total_normal_bytes;
            h[k * F + 9] = r.rows_touched;
            h[k * F + 10] = r.work_inspections;
        }
        DArray<int64_t> t;
        t.alloc((int64_t)h.size());
        DBFS_CUDA(cudaMemcpy(t.p, h.data(), 8 * h.size(), cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx, t.p, (int64_t)h.size(), 0);
        DBFS_CUDA(cudaMemcpy(h.data(), t.p, 8 * h.size(), cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < count; k++) {
            dbfs_run_stats &r = st[k];
            for (int q = 0; q < 4; q++) {
                r.inspections[q][0] = h[k * F + 2 * q];
                r.inspections[q][1] = h[k * F + 2 * q + 1];
            }
            r.total_normal_bytes = h[k * F + 8];
            r.rows_touched = h[k * F + 9];
            r.work_inspections = h[k * F + 10];
            const int64_t bwd = r.inspections[KIND_ND][BWD] + r.inspections[KIND_DD][BWD];
            r.b_measured = g.d ? (double)bwd / (double)(g.d * g.p) : 0.0;
            r.accounting_valid = r.iterations <= rmax ? 1 : 0;
        }
    }
    if (aborted && peer) g.peer_state = -1;
    DBFS_CHECK(!aborted, DBFS_ETIMEOUT, "device watchdog fired in the persistent BFS kernel");
    if (!rerun.empty()) {
        // a re-run root's result is what the device holds now: run_bfs set
        // last_source / last_iterations / last_parent_mode for it
        g.last_truncated = true;
        g.last_rec.clear();
        return;
    }
    if (btrace)
        fprintf(stderr, "[batch] done at %.2f ms after entry\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count() -
                    tentry);
    g.last_iterations = hi[count - 1].x;
    g.last_truncated = true;
    g.last_rec.clear();
    g.last_source = roots[count - 1];
    g.last_parent_mode = o0.parent_mode;
    g.last_valid = true;
    g.last_mode = o0.mode;
    g.last_la = o0.local_all2all;
    g.last_uq = o0.uniquify;
    g.assembled = !g.dist;
}

// ------------------------------------------------------ per-iteration records

// BfsRun.per_iteration entry `it` summed over the W local workers' records
// x[0..W) (engine.py:291-302) with the comm accounting of comm.py:75-197.
void iteration_summary(const Graph &g, const IterRec *x0, int64_t it, int last_la, int last_uq, dbfs_iteration *rec,
                       int8_t *directions, double *bv) {
    dbfs_iteration r;
    memset(&r, 0, sizeof(r));
    r.iteration = it;
    const int W = g.W;
    bool any_new = false;
    int64_t records = 0, msgs = 0, uq_records = 0;
    // send matrix [sender][dest] for message accounting
    std::vector<int64_t> cnt((size_t)g.p * g.p, 0);
    for (int i = 0; i < W; i++) {
        const IterRec &x = x0[i];
        for (int k = 0; k < 4; k++) {
            r.inspections[k] += (int64_t)x.insp[k];
            r.fv[k] += (int64_t)x.fv[k];
        }
        any_new |= x.new_del > 0;
        r.frontier_normals += (int64_t)x.nfront;
        for (int k = 0; k < 4; k++) r.work[k] += (int64_t)x.work[k];
        if (i == 0) {
            for (int k = 0; k < 4; k++) r.exec_dirs[k] = x.exec_dir[k];
            double ghz = g.clock_ghz > 0 ? g.clock_ghz : 1.9;
            double nwarps = g.warps_per_worker > 0 ? g.warps_per_worker : 1;
            for (int k = 0; k < 8; k++) {
                r.task_avg_us[k] = (double)x.tsum[k] / nwarps / (ghz * 1e3);
                r.task_max_us[k] = (double)x.tmax[k] / (ghz * 1e3);
            }
            r.frontier_delegates = (int64_t)x.dfront;
            if (x.t[1] > x.t[0]) r.visit_us = (double)(x.t[1] - x.t[0]) / 1e3;
            if (x.t[2] > x.t[1]) r.finish_us = (double)(x.t[2] - x.t[1]) / 1e3;
            if (x.tb[0] > x.t[0] && x.tb[1] >= x.tb[0] && x.tb[2] > x.t[1] && x.tb[3] >= x.tb[2]) {
                r.sync_us[0] = (double)(x.tb[0] - x.t[0]) / 1e3;
                r.sync_us[1] = (double)(x.tb[1] - x.tb[0]) / 1e3;
                r.sync_us[2] = (double)(x.tb[2] - x.t[1]) / 1e3;
                r.sync_us[3] = (double)(x.tb[3] - x.tb[2]) / 1e3;
            }
        }
        records += (int64_t)x.records;
        uq_records += (int64_t)x.uq_records;
        msgs += (int64_t)x.messages;
        int w = g.workers[i].w;
        for (int o = 0; o < g.p; o++) cnt[(size_t)w * g.p + o] = (int64_t)x.send[o];
        if (directions)
            for (int k = 0; k < 4; k++) directions[(size_t)w * 4 + k] = (int8_t)x.dir[k];
        if (bv)
            for (int k = 0; k < 4; k++) bv[(size_t)w * 4 + k] = x.bv[k];
    }
    // comm.py:75-98 / 138-197 accounting
    r.mask_bytes = any_new ? 2.0 * (double)g.d * (double)g.p_rank / 8.0 : 0.0;
    r.normal_bytes = 4 * (last_uq && g.p > 1 ? uq_records : records);
    if (last_la) {
        // local-all2all regroups (sender, dest) -> (r + p_rank * (dest / p_rank), dest)
        std::vector<int> seen((size_t)g.p * g.p, 0);
        msgs = 0;
        for (int s = 0; s < g.p; s++)
            for (int o = 0; o < g.p; o++)
                if (cnt[(size_t)s * g.p + o] > 0) {
                    int fs = (s % g.p_rank) + g.p_rank * (o / g.p_rank);
                    if (!seen[(size_t)fs * g.p + o]) {
                        seen[(size_t)fs * g.p + o] = 1;
                        msgs++;
                    }
                }
    }
    r.message_count = msgs;
    r.pair_count = last_la ? (int64_t)g.p * g.p / g.p_gpu : (int64_t)g.p * g.p;
    r.comm_us = it < (int64_t)g.last_comm_us.size() ? g.last_comm_us[it] : 0.0;
    *rec = r;
}

// Run-level accounting from the records of iterations [0, nrec): inspections
// by reported direction, b_measured (engine.py:316-318) and the CommStats
// totals (comm.py:39-72), summed in iteration order like the reference.
void run_accounting(const Graph &g, const IterRec *recs, int64_t nrec, int64_t iterations, int la, int uq,
                    dbfs_run_stats *st) {
    const int W = g.W;
    for (int k = 0; k < 4; k++) st->inspections[k][0] = st->inspections[k][1] = 0;
    st->total_mask_bytes = 0.0;
    st->total_normal_bytes = 0;
    st->s_prime = 0;
    for (int64_t it = 0; it < nrec; it++) {
        for (int i = 0; i < W; i++) {
            const IterRec &r = recs[(size_t)it * W + i];
            for (int k = 0; k < 4; k++) st->inspections[k][r.dir[k]] += (int64_t)r.insp[k];
        }
        dbfs_iteration s;
        iteration_summary(g, &recs[(size_t)it * W], it, la, uq, &s, nullptr, nullptr);
        st->total_mask_bytes += s.mask_bytes;
        st->total_normal_bytes += s.normal_bytes;
        st->s_prime += s.mask_bytes > 0;
    }
    const int64_t bwd = st->inspections[KIND_ND][BWD] + st->inspections[KIND_DD][BWD];
    st->b_measured = g.d ? (double)bwd / (double)(g.d * g.p) : 0.0;
    st->accounting_valid = (!g.dist && nrec == iterations) ? 1 : 0;
}

// ------------------------------------------------ min-ID parents (A19) / A20

struct EdgeWalk {
    const int64_t *off;
    const uint32_t *col;
    int64_t rows;
    int kind, w;
    PDiv pd;
    const int64_t *del_gid;
};

__device__ __forceinline__ int64_t row_gid(const EdgeWalk &e, int64_t r) {
    return (e.kind == KIND_NN || e.kind == KIND_ND) ? r * e.pd.p + e.w : e.del_gid[r];
}
__device__ __forceinline__ int64_t col_gid(const EdgeWalk &e, uint32_t c) {
    if (e.kind == KIND_NN) return c;
    if (e.kind == KIND_DN) return (int64_t)c * e.pd.p + e.w;
    return e.del_gid[c];
}

// parent[v] = min{u : (u->v) in E, level[u] = level[v]-1}
__global__ void k_min_parents(EdgeWalk e, const int32_t *__restrict__ lv, unsigned long long *__restrict__ par) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, TW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (int64_t r = gw; r < e.rows; r += TW) {
        int64_t u = row_gid(e, r);
        int32_t lu = lv[u];
        if (lu < 0) continue;
        for (int64_t j = e.off[r] + lane; j < e.off[r + 1]; j += 32) {
            int64_t v = col_gid(e, e.col[j]);
            if (lv[v] == lu + 1) atomicMin(&par[v], (unsigned long long)u);
        }
    }
}

__global__ void k_par_init(const int32_t *__restrict__ lv, int64_t n, unsigned long long *par) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        par[v] = lv[v] >= 0 ? 0x7fffffffffffffffull : 0xffffffffffffffffull;
}

// min-ID tree into the parent output: root -> root, unreached -> -1
__global__ void k_par_final(const unsigned long long *__restrict__ par, const int32_t *__restrict__ lv, int64_t n,
                            int64_t root, parent_t *__restrict__ out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = (parent_t)(v == root ? root : (lv[v] < 0 ? -1 : (int64_t)par[v]));
}

static EdgeWalk walk_of(Graph &g, WorkerHost &Wk, int k) {
    EdgeWalk e;
    e.off = g.off_all.p + Wk.base[k];
    e.col = g.col_all.p;
    e.rows = Wk.rows[k];
    e.kind = k;
    e.w = Wk.w;
    e.pd.init((uint32_t)g.p);
    e.del_gid = g.del_gid.p;
    return e;
}

// Replace the parent output of the last BFS (root) by the min-ID tree
// (parent_mode 2): kernels only on ctx.stream (a batch enqueues it
// between roots).  Distributed graphs min-reduce the candidates over ranks.
void min_parents_device(Graph &g, int64_t root) {
    Ctx &ctx = *g.ctx;
    DArray<unsigned long long> &par = g.minpar;
    if (par.n < std::max<int64_t>(g.n, 1)) par.alloc(std::max<int64_t>(g.n, 1));
    const int32_t *lv = g.levels_dev();
    k_par_init<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(lv, g.n, par.p);
    DBFS_LAUNCHED();
    for (auto &Wk : g.workers)
        for (int k = 0; k < 4; k++) {
            EdgeWalk e = walk_of(g, Wk, k);
            if (e.rows == 0) continue;
            k_min_parents<<<ctx.num_sms * 8, BT, 0, ctx.stream>>>(e, lv, par.p);
            DBFS_LAUNCHED();
        }
    if (g.dist) nccl_allreduce_i64(ctx, (int64_t *)par.p, g.n, 1);  // unsigned -1 stays max; reached < INT64_MAX
    k_par_final<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(par.p, lv, g.n, root, g.parents_dev());
    DBFS_LAUNCHED();
}

void min_parents(Graph &g, int64_t *out) {
    DBFS_CHECK(g.last_valid, DBFS_EINVAL, "no BFS result on device");
    DBFS_CHECK(g.last_parent_mode != 0, DBFS_EINVAL, "last BFS ran without parents");
    Ctx &ctx = *g.ctx;
    dist_assemble(g);
    if (g.last_parent_mode != 2) {
        min_parents_device(g, g.last_source);
        g.last_parent_mode = 2;
    }
    DBFS_CUDA(cudaMemcpyAsync(out, g.parents_dev64(), 8 * g.n, cudaMemcpyDeviceToHost, ctx.stream));
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

// Edge checks of the certificate.  On a symmetric graph every edge is
// undirected: both ends reached or both unreached, levels at most one apart.
// A directed graph (do_symmetrize=False, loaded edge lists) keeps only the
// directed conditions: u reached => v reached, level[v] <= level[u] + 1.
__global__ void k_validate_edges(EdgeWalk e, const int32_t *__restrict__ lv, const int64_t *__restrict__ par,
                                 uint8_t *__restrict__ ok, unsigned int *__restrict__ bad, int symmetric) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, TW = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    unsigned b = 0;
    for (int64_t r = gw; r < e.rows; r += TW) {
        int64_t u = row_gid(e, r);
        int32_t lu = lv[u];
        for (int64_t j = e.off[r] + lane; j < e.off[r + 1]; j += 32) {
            int64_t v = col_gid(e, e.col[j]);
            int32_t lvv = lv[v];
            if (symmetric) {
                if ((lu >= 0) != (lvv >= 0)) b |= 4;
                else if (lu >= 0 && (lu - lvv > 1 || lvv - lu > 1)) b |= 2;
            } else if (lu >= 0) {
                if (lvv < 0) b |= 4;
                else if (lvv - lu > 1) b |= 2;
            }
            if (lvv >= 0 && par[v] == u) ok[v] = 1;
        }
    }
    b = __reduce_or_sync(0xffffffffu, b);
    if (lane == 0 && b) atomicOr(bad, b);
}

__global__ void k_validate_vertices(const int32_t *__restrict__ lv, const int64_t *__restrict__ par,
                                    const uint8_t *__restrict__ ok, int64_t n, int64_t root,
                                    unsigned int *__restrict__ bad) {
    unsigned b = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int32_t l = lv[v];
        int64_t pv = par[v];
        if (v == root) {
            if (l != 0 || pv != root) b |= 1;
            continue;
        }
        if (l < 0) {
            if (pv != -1) b |= 32;
            continue;
        }
        if (pv < 0 || pv >= n) {
            b |= 32;
            continue;
        }
        if (lv[pv] != l - 1) b |= 8;
        if (!ok[v]) b |= 16;
    }
    b = __reduce_or_sync(0xffffffffu, b);
    if (lane_id() == 0 && b) atomicOr(bad, b);
}

int validate(Graph &g, int64_t root, const int32_t *levels, const int64_t *parents) {
    Ctx &ctx = *g.ctx;
    DBFS_CHECK(0 <= root && root < g.n, DBFS_ERANGE, "root out of range");
    DArray<int32_t> lvh;
    DArray<int64_t> pah;
    const int32_t *lv;
    const int64_t *pa;
    if (levels) {
        lvh.alloc(std::max<int64_t>(g.n, 1));
        DBFS_CUDA(cudaMemcpy(lvh.p, levels, 4 * g.n, cudaMemcpyHostToDevice));
        lv = lvh.p;
    } else {
        DBFS_CHECK(g.last_valid, DBFS_EINVAL, "no BFS result on device");
        dist_assemble(g);
        lv = g.levels_dev();
    }
    if (parents) {
        pah.alloc(std::max<int64_t>(g.n, 1));
        DBFS_CUDA(cudaMemcpy(pah.p, parents, 8 * g.n, cudaMemcpyHostToDevice));
        pa = pah.p;
    } else {
        DBFS_CHECK(g.last_valid && g.last_parent_mode != 0, DBFS_EINVAL, "no parents on device");
        dist_assemble(g);
        pa = g.parents_dev64();
    }
    DArray<uint8_t> ok;
    ok.alloc(std::max<int64_t>(g.n, 1));
    DBFS_CUDA(cudaMemsetAsync(ok.p, 0, ok.bytes(), ctx.stream));
    DArray<unsigned int> bad;
    bad.alloc(1);
    DBFS_CUDA(cudaMemsetAsync(bad.p, 0, 4, ctx.stream));
    for (auto &Wk : g.workers)
        for (int k = 0; k < 4; k++) {
            EdgeWalk e = walk_of(g, Wk, k);
            if (e.rows == 0) continue;
            k_validate_edges<<<ctx.num_sms * 8, BT, 0, ctx.stream>>>(e, lv, pa, ok.p, bad.p, g.symmetric ? 1 : 0);
            DBFS_LAUNCHED();
        }
    if (g.dist) nccl_allreduce_u8_max(ctx, ok.p, g.n);  // tree-edge marks OR-ed over ranks
    k_validate_vertices<<<ctx.num_sms * 4, BT, 0, ctx.stream>>>(lv, pa, ok.p, g.n, root, bad.p);
    DBFS_LAUNCHED();
    unsigned int hb = 0;
    if (g.dist) {  // failure bits OR-ed over ranks
        DArray<unsigned int> all;
        all.alloc(g.p);
        nccl_allgather_bytes(ctx, bad.p, all.p, 4);
        std::vector<unsigned int> h(g.p);
        DBFS_CUDA(cudaMemcpy(h.data(), all.p, 4 * g.p, cudaMemcpyDeviceToHost));
        for (unsigned x : h) hb |= x;
    } else {
        DBFS_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    return (int)hb;
}

}  // namespace dbfs
