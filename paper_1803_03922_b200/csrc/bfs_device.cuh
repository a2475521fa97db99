// bfs_device.cuh -- device phases of one BFS level (engine.py:146-306 restated
// for sm_100a).  Used both by the persistent single-launch engine (grid
// barriers between phases) and by the host-driven engine (one launch per
// phase, NCCL exchange in between).
//
// Level L of worker w runs two phases:
//   V(L)  visits (engine.py:199-263): nn push; nd/dn/dd push or pull as the
//         on-device direction rule decides (traversal.py:142-163).  Pushes
//         claim normals with atomicOr on the next-frontier bitmap and mark
//         delegates in the per-level delegate mask; pulls scan reverse rows
//         with early exit and count inspections exactly (traversal.py:111-139).
//   F(L)  barrier + apply (engine.py:265-289): OR of all workers' delegate
//         masks (comm.py:75-98), ingest of remote normal records
//         (comm.py:138-197 / engine.py:147-157), frontier bookkeeping.
//
// Pre-state rule: every test made during V(L) must see the state at the start
// of level L (the reference applies updates only after its barrier).  Hence
//   visited(<= L) normal   = nvis   (claims go to nfront[(L+1)&1], folded in F)
//   frontier L normal      = nfront[L&1]
//   visited(<= L) delegate = dvis   (finds go to dnext[L&1], folded in F)
// Discoveries are fire-and-forget (RED.OR on the next bitmap + a plain store of
// the parent; any concurrent writer's parent is a valid one; a normal's level is
// written when F folds it into visited), so no lane
// ever waits on an atomic's return value in the traversal loops.  Frontier
// statistics for the direction rule are counted from the bitmaps in F.
#pragma once
#include "internal.h"

namespace dbfs {

#ifndef DBFS_BT
#define DBFS_BT 768
#endif
constexpr int BT = DBFS_BT;    // threads per block
constexpr int WPB = BT / 32;   // warps per block
constexpr int LIST = 1024;     // per-warp compaction buffer (32 words x 32 bits)

constexpr int FW = 8192;       // words of the coarse frontier filter (32 KB, 2^18 bits)
#ifndef DBFS_FILTER
#define DBFS_FILTER 0
#endif

struct Smem {
    View view;                 // this block's worker View (global copies would be re-fetched from L2
                               // after every grid barrier's acquire)
    uint32_t list[WPB][LIST];
#if DBFS_FILTER
    uint32_t filt[FW];         // coarse filter of the pull frontier (when sparse)
#else
    uint32_t filt[1];
#endif
};

// Coarse filter: bit (x & 31) of word (x >> 10) & (FW-1) is the OR of the 32
// frontier words of x's 1024-vertex group -- a warp folds its 32 words into one
// coarse word with a shuffle OR and one atomic.
__device__ __forceinline__ bool coarse_hit(const uint32_t *filt, uint32_t x) {
    return (filt[(x >> 10) & (FW - 1)] >> (x & 31)) & 1u;
}

constexpr uint32_t SRC_DEL_LOOKUP = 0xfffffffeu;  // seed: look the source's delegate id up on device

struct GridBar {
    unsigned int count;
    unsigned int gen;
    unsigned int abort;
    unsigned int pad;
};

// ---------------------------------------------------------------- direction

__host__ __device__ inline int bitlen128(unsigned __int128 x) {
    int b = 0;
    while (x) {
        b++;
        x >>= 1;
    }
    return b;
}

// Correctly rounded N / D, i.e. Python's int / int (traversal.py:148).
__host__ __device__ inline double div_rn(unsigned __int128 N, unsigned long long D) {
    if (N == 0) return 0.0;
    if (N < ((unsigned __int128)1 << 53) && D < (1ULL << 53)) return (double)(unsigned long long)N / (double)D;
    int shift = 56 - bitlen128(N) + bitlen128(D);
    if (shift < 0) shift = 0;
    unsigned __int128 num = N << shift;
    unsigned __int128 Q = num / D;
    bool sticky = (num % D) != 0;
    int drop = bitlen128(Q) - 53;
    unsigned __int128 mant = Q >> drop;
    unsigned __int128 rem = Q & ((((unsigned __int128)1) << drop) - 1);
    unsigned __int128 half = ((unsigned __int128)1) << (drop - 1);
    if (rem > half || (rem == half && (sticky || (mant & 1)))) mant++;
    if (mant == ((unsigned __int128)1 << 53)) {
        mant >>= 1;
        drop++;
    }
    double r = (double)(unsigned long long)mant;
    int e = drop - shift;
    // exact scaling by a power of two
    while (e > 0) {
        int s = e > 60 ? 60 : e;
        r *= (double)(1ULL << s);
        e -= s;
    }
    while (e < 0) {
        int s = -e > 60 ? 60 : -e;
        r /= (double)(1ULL << s);
        e += s;
    }
    return r;
}

// estimate_backward_workload (traversal.py:142-148)
__host__ __device__ inline double bv_of(unsigned long long u, unsigned long long q, unsigned long long s) {
    if (q == 0) return (double)INFINITY;
    return div_rn((unsigned __int128)u * (unsigned __int128)(q + s), q);
}

// decide_direction (traversal.py:151-163): int FV vs float, exact.
__host__ __device__ inline int decide_dir(int dir, unsigned long long fv, double bv, double f0, double f1,
                                          int allow_back) {
    double fvd = (double)fv;  // fv <= m < 2^53
    bool fin = bv == bv && bv != (double)INFINITY;
    if (dir == FWD) return (fin && fvd > f0 * bv) ? BWD : FWD;
    return (allow_back && fvd < f1 * bv) ? FWD : BWD;
}

// U/q/s wiring of engine.py:181-189 for kind k at level L.  cum[] = visited
// source counts through level L.
__host__ __device__ inline void level_inputs(const unsigned long long *total_src, const unsigned long long *cum,
                                             const unsigned long long *q, int k, unsigned long long &U,
                                             unsigned long long &Q, unsigned long long &S) {
    unsigned long long u_nd = total_src[KIND_ND] - cum[KIND_ND];
    unsigned long long u_dn = total_src[KIND_DN] - cum[KIND_DN];
    unsigned long long u_dd = total_src[KIND_DD] - cum[KIND_DD];
    if (k == KIND_ND) {
        U = u_dn; Q = q[KIND_ND]; S = u_nd;
    } else if (k == KIND_DN) {
        U = u_nd; Q = q[KIND_DN]; S = u_dn;
    } else {
        U = u_dd; Q = q[KIND_DD]; S = u_dd;
    }
}

// Directions of level L from the sticky state of L-1 and the frontier stats.
__host__ __device__ inline void level_dirs(const View &V, const Ctl &c, int L, int dirs[4], double bv[4],
                                           unsigned long long cum[4]) {
    const LevelSlot &S = c.s[L % 3];
    const int pp = (L + 1) & 1;  // parity of L-1
    for (int k = 0; k < 4; k++) cum[k] = (L == 0 ? 0ull : c.cumq[pp][k]) + S.q[k];
    dirs[KIND_NN] = FWD;
    bv[KIND_NN] = 0.0;
    for (int k = 1; k < 4; k++) {
        unsigned long long U, Q, Sx;
        level_inputs(V.total_src, cum, S.q, k, U, Q, Sx);
        bv[k] = bv_of(U, Q, Sx);
        int prev = L == 0 ? FWD : c.dir[pp][k];
        dirs[k] = V.mode == 0 ? FWD : decide_dir(prev, S.fv[k], bv[k], V.f0[k], V.f1[k], V.allow_back);
    }
}

// Executed strategy per kind.  The reported direction (and its counter) is the
// reference rule's; when that rule says FORWARD on a symmetric graph, pushing
// the frontier's k-rows and pulling over the reverse rows of the unvisited
// k-candidates find the same vertex set, so the executor takes the cheaper one
// (estimated L2 requests: push ~4 per edge with its atomics, pull ~1.5 per
// scanned entry with hit probability FV_k / nnz_k).
//
// A BACKWARD-reported kind may run as a counting push (PUSHC): the frontier's
// k-rows are pushed and every unvisited target v keeps the minimum twin
// position (where v's reverse row holds the pushing parent), so F(L) knows the
// pull's early-exit index of every found v; the unvisited candidates' row
// lengths sum to nnz[rev] - cumfv[rev].  The pull counter is that sum minus
// (len - first - 1) per found v.  With FV_k = 0 no candidate can hit and the
// counter is the sum alone (no twins needed).  exec_policy 2 (tests) takes
// PUSHC whenever twins exist.
constexpr int PUSHC = 2;
#ifndef DBFS_PUSHC_COST
#define DBFS_PUSHC_COST 5.0  // cost units per edge of a counting push (PUSHC)
#endif
#ifndef DBFS_PUSH_COST
#define DBFS_PUSH_COST 2.0  // cost units per pushed edge in the executor model (4 -> 2: +0.7 % s24, +1.3 % s25 on 2 GPUs)
#endif

__host__ __device__ inline int rev_kind(int k) { return k == KIND_ND ? KIND_DN : (k == KIND_DN ? KIND_ND : KIND_DD); }

__host__ __device__ inline void exec_dirs(const View &V, const LevelSlot &S, const unsigned long long *cum,
                                          const int dirs[4], int ex[4]) {
    for (int k = 0; k < 4; k++) ex[k] = dirs[k];
    if (V.mode != 1 || !V.symmetric || !V.exec_policy) return;
    const unsigned long long u_nd = V.total_src[KIND_ND] - cum[KIND_ND];
    const unsigned long long u_dn = V.total_src[KIND_DN] - cum[KIND_DN];
    const unsigned long long u_dd = V.total_src[KIND_DD] - cum[KIND_DD];
    for (int k = 1; k < 4; k++) {
        if (dirs[k] == BWD) {
            if (S.fv[k] == 0) {
                ex[k] = PUSHC;
                continue;
            }
            if (!V.twin[k]) continue;
            if (V.exec_policy == 2) {
                ex[k] = PUSHC;
                continue;
            }
            const int rev = rev_kind(k);
            double U = (double)(k == KIND_ND ? u_dn : (k == KIND_DN ? u_nd : u_dd));
            double rows = (double)(V.total_src[rev] ? V.total_src[rev] : 1);
            double avg = (double)V.nnz[rev] / rows;
            double scan = (double)V.nnz[k] / (double)S.fv[k];
            if (scan > avg) scan = avg;
            double words = (double)(rev == KIND_ND ? V.nw_n : V.nw_d);
            double pull = 1.5 * U * scan + 0.25 * words;
            double push = DBFS_PUSHC_COST * (double)S.fv[k];  // push + twin load + atomicMin
            if (push < pull) ex[k] = PUSHC;
            continue;
        }
        if (V.exec_policy == 2 || S.fv[k] == 0) continue;
        // reverse kind scanned by the equivalent pull, and its candidate count
        int rev = k == KIND_ND ? KIND_DN : (k == KIND_DN ? KIND_ND : KIND_DD);
        double U = (double)(k == KIND_ND ? u_dn : (k == KIND_DN ? u_nd : u_dd));
        double rows = (double)(V.total_src[rev] ? V.total_src[rev] : 1);
        double avg = (double)V.nnz[rev] / rows;
        double scan = (double)V.nnz[k] / (double)S.fv[k];  // entries per hit, uniform model
        if (scan > avg) scan = avg;
        // hubs first: sorted rows reach a frontier hub sooner, but only when the
        // frontier holds hubs -- a small frontier far from them scans whole rows
        if (k == KIND_DD && V.col_sorted_dd) scan = scan * 0.5 > 1.0 ? scan * 0.5 : 1.0;
        double words = (double)(rev == KIND_ND ? V.nw_n : V.nw_d);
        double pull = 1.5 * U * scan + 0.25 * words;
        double push = DBFS_PUSH_COST * (double)S.fv[k];
        if (pull < push) ex[k] = BWD;
    }
}

// Per-iteration record of level L (engine.py:291-302, one worker).
// Scalar fields of the record (everything but the per-task timers and the
// per-destination message flags).
__host__ __device__ inline void make_record_core(const View &V, const Ctl &c, int L, IterRec &r) {
    const LevelSlot &S = c.s[L % 3];
    // directions and BV were published at V(L) (c.dir by parity, S.bv); nothing
    // here reads state of level L+1, so any block may make it during V(L+1)
    for (int k = 0; k < 4; k++) {
        r.dir[k] = k == KIND_NN ? FWD : c.dir[L & 1][k];
        r.bv[k] = S.bv[k];
        r.fv[k] = S.fv[k];
        r.insp[k] = r.dir[k] == FWD ? S.fv[k] : S.insp_bwd[k];
    }
    r.records = S.records;
    r.uq_records = S.uq_records;
    for (int k = 0; k < 4; k++) {
        r.work[k] = S.work[k];
        r.exec_dir[k] = S.exec_dir[k];
    }
    r.nfront = S.nfront;
    r.dfront = S.dfront;
    r.rows = S.pull_rows;
    for (int k = 0; k < 4; k++)
        if (k == KIND_NN || S.exec_dir[k] != BWD) r.rows += S.q[k];
    r.dirty = S.dirty;
    r.new_del = S.new_del;
}

__host__ __device__ inline void make_record(const View &V, const Ctl &c, int L, IterRec &r) {
    const LevelSlot &S = c.s[L % 3];
    make_record_core(V, c, L, r);
    for (int k = 0; k < 8; k++) {
        r.tsum[k] = S.tsum[k];
        r.tmax[k] = S.tmax[k];
    }
    unsigned long long msgs = 0;
    for (int o = 0; o < MAXW; o++) {
        r.send[o] = S.send[o];
        msgs += S.send[o] > 0;
    }
    r.messages = msgs;
}

// ------------------------------------------------------------------ helpers

#ifndef DBFS_UNR
#define DBFS_UNR 4
#endif
constexpr int UNR = DBFS_UNR;    // independent column loads in flight per lane (push)
#ifndef DBFS_ROWS_UNR
#define DBFS_ROWS_UNR DBFS_UNR
#endif
#ifndef DBFS_LIST_UNR
#define DBFS_LIST_UNR DBFS_UNR
#endif
constexpr int ROWS_UNR = DBFS_ROWS_UNR;  // normal-row pushes (nn, nd)
constexpr int LIST_UNR = DBFS_LIST_UNR;  // delegate-list pushes (dn, dd)
static_assert(ROWS_UNR <= UNR && LIST_UNR <= UNR, "send chunks are sized for UNR");
constexpr int PULL_U = 4;        // 32 * PULL_U columns per warp-wide pull step
#ifndef DBFS_PROBE
#define DBFS_PROBE 2
#endif
constexpr int PROBE = DBFS_PROBE;  // candidate groups whose first entry is probed together
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ bool tbit(const uint32_t *b, uint32_t i) { return (b[i >> 5] >> (i & 31)) & 1u; }

// Warp-cooperative compaction of the set bits of 32 bitmap words (one per
// lane, word index wi) into ids in `list`; returns the count (warp-uniform).
__device__ __forceinline__ unsigned warp_compact(uint32_t word, int64_t wi, uint32_t *list) {
    unsigned tot;
    unsigned off = warp_excl_scan(__popc(word), &tot);
    uint32_t basev = (uint32_t)(wi << 5);
    while (word) {
        int b = __ffs(word) - 1;
        word &= word - 1;
        list[off++] = basev + b;
    }
    __syncwarp();
    return tot;
}

__device__ __forceinline__ unsigned long long warp_excl_scan64(unsigned long long v, unsigned long long *tot) {
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(FULL, x, o);
        if (lane_id() >= (unsigned)o) x += y;
    }
    *tot = __shfl_sync(FULL, x, 31);
    return x - v;
}

// Largest lane l with key_l <= x, for keys non-decreasing over lanes and
// key_0 <= x (5 shuffle steps; all lanes must participate).
template <typename T>
__device__ __forceinline__ int owner_search(T key, T x) {
    int lo = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        int cand = lo + s;
        T v = __shfl_sync(FULL, key, cand & 31);
        if (cand < 32 && v <= x) lo = cand;
    }
    return lo;
}

// Per-warp task timer (lane 0 accumulates clock64 spans into the level slot).
#ifndef DBFS_TASK_TIMERS
#define DBFS_TASK_TIMERS 0
#endif
struct TaskTimer {
    long long t0;
    __device__ __forceinline__ void start() {
        if (DBFS_TASK_TIMERS) t0 = clock64();
    }
    __device__ __forceinline__ void stop(LevelSlot &A, int task) {
        if (!DBFS_TASK_TIMERS) return;
        long long dt = clock64() - t0;
        if (lane_id() == 0 && dt > 0) {
            atomicAdd(&A.tsum[task], (unsigned long long)dt);
            atomicMax(&A.tmax[task], (unsigned long long)dt);
        }
    }
};

// Peer engine: a warp reserves inbox slots per destination SEND_CHUNK at a time
// (lane d holds its cursor for destination d), so the per-destination counter
// sees one atomic per chunk instead of one per warp step; the unused tail of
// each chunk is filled with sentinels at the end of V (receivers skip them).
constexpr unsigned SEND_CHUNK = 256;
constexpr uint32_t REC_SKIP = 0xffffffffu;
static_assert(32 * UNR <= SEND_CHUNK, "a warp step must fit one fresh chunk");

struct VisitCounters {
    bool light;                     // light level: normal claims mark the touch bitmap
    unsigned long long fv_nn;       // FV_nn of this level's frontier (activity slot)
    unsigned long long scur, send;  // peer engine: this warp's inbox chunk for destination lane_id()
    unsigned long long records;     // remote normal records (comm accounting)
    unsigned long long uq;          // records surviving uniquify
    unsigned long long insp_bwd[4];
    unsigned long long dirty;
    unsigned long long pull_rows;
};

// Light levels: every normal claim also marks its 1024-vertex chunk in the
// next frontier's touch bitmap (1 bit per 32 bitmap words) and the first claim
// of a chunk appends it to the chunk list of frontier L+1, so F and the next
// T1 hand out the listed chunks to warps instead of sweeping all n/32 words.
// Heavy levels do not mark; their F sweeps and builds the bitmap from the fold
// (the next level then finds chunks by their touch bits).
__device__ __noinline__ void touch_chunk(const View &V, int L, uint32_t c) {
    const uint32_t chunk = c >> 10, bit = 1u << (chunk & 31);
    uint32_t *touch = V.ntouch[(L + 1) & 1];
    if (__ldcg(&touch[chunk >> 5]) & bit) return;
    if (atomicOr(&touch[chunk >> 5], bit) & bit) return;
    // first claim in this chunk: append it to the next frontier's chunk list
    const unsigned long long i = atomicAdd(&V.ctl->s[(L + 1) % 3].nchunks, 1ull);
    V.nchunk_list[(L + 1) & 1][i] = chunk;
}

// Claim normal c of worker `wv` (this worker, or an in-process peer) for
// level L+1, fire-and-forget.  `seen` is visited(<= L) plus the pushes' claims
// made so far at level L (the eager copy of the visited bitmap, see
// push_stage): one L2 test decides; a claim sets it and the next-frontier bit.
// F copies the folded visited bitmap back into it (pull finds included).
__device__ __forceinline__ void claim_on(uint32_t *__restrict__ seen, uint32_t *__restrict__ nx,
                                         parent_t *__restrict__ nparent, int parents, uint32_t c, parent_t parent) {
    const uint32_t wd = c >> 5, bit = 1u << (c & 31);
    if (__ldcg(&seen[wd]) & bit) return;  // visited, or claimed this level (possibly stale: then harmless)
    atomicOr(&seen[wd], bit);             // results unused -> RED.OR
    atomicOr(&nx[wd], bit);
    if (parents) nparent[c] = parent;     // the level is written by F3 (word order, coalesced)
}

__device__ __forceinline__ void claim_normal(const View &V, int L, uint32_t c, parent_t parent, bool light) {
    const uint32_t wd = c >> 5, bit = 1u << (c & 31);
    if (__ldcg(&V.nseen[wd]) & bit) return;
    claim_on(V.nseen, V.nfront[(L + 1) & 1], V.nparent, V.parents, c, parent);
    if (light) touch_chunk(V, L, c);
}

// Remote nn records of one warp step (engine.py:207-222 -> comm.py:138-197):
// lanes with `need` send (owner o, local c, parent).  In-process peers are
// claimed directly in their device arrays; distributed peers get an 8-byte
// record in the per-destination send bin.  One atomic per destination per warp.
// Destinations that received >= 1 record this level, per block (the
// reference's message count is the number of non-empty (sender, dest)
// pairs, comm.py:138-197); flushed once per block at the end of V.
__device__ __forceinline__ unsigned long long *block_sendmask() {
    __shared__ unsigned long long s_mask;
    return &s_mask;
}

// Remote nn targets of one warp step (U slots, engine.py:207-222 ->
// comm.py:138-197), handled as one batch so the slots' memory round trips
// overlap.  In-process peers are claimed directly in their bitmaps; a
// distributed peer gets an 8-byte record in its inbox segment, unless this
// sender already shipped that target during this BFS: a target shipped once
// was claimed by its owner at that level (or was already visited), so one
// bit per global id (test, then set) keeps each remote target to a single
// record per sender.  The reference counters see every record
// (vc.records, the destination mask).
#ifndef DBFS_SENT_WAIT
#define DBFS_SENT_WAIT 0  // 1: ship only if the returning atomic saw the bit clear (no duplicate records)
#endif
template <int U>
__device__ __forceinline__ void warp_send_batch(const View &V, int L, const bool (&need)[U], const uint32_t (&o)[U],
                                                const uint32_t (&c)[U], const uint32_t (&parent)[U],
                                                VisitCounters &vc) {
    bool any = false;
#pragma unroll
    for (int u = 0; u < U; u++) any |= need[u];
    if (!__any_sync(FULL, any)) return;
    {
        unsigned lo = 0, hi = 0;
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (need[u]) {
                vc.records++;
                if (o[u] < 32) lo |= 1u << o[u];
                else hi |= 1u << (o[u] - 32);
            }
        }
        lo = __reduce_or_sync(FULL, lo);
        if (V.p > 32) hi = __reduce_or_sync(FULL, hi);
        if (lane_id() == 0) atomicOr(block_sendmask(), ((unsigned long long)hi << 32) | lo);
    }
    if (!V.dist) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (!need[u]) continue;
            if (V.uniquify) {  // staging group of (sender, dest): comm.py:165-171
                int grp = V.local_all2all ? (V.w % V.p_rank) + V.p_rank * ((int)o[u] / V.p_rank) : V.w;
                const int64_t nwo = (V.n_local_of_w[o[u]] + 31) >> 5;
                uint32_t old = atomicOr(&V.uq_all[o[u]][(int64_t)grp * nwo + (c[u] >> 5)], 1u << (c[u] & 31));
                if (!(old & (1u << (c[u] & 31)))) vc.uq++;
            }
            claim_on(V.nseen_all[o[u]], V.nfront_all[(L + 1) & 1][o[u]], V.nparent_all[o[u]], V.parents, c[u],
                     parent[u]);
        }
        return;
    }
    bool ship[U];
    if (V.sent) {
        uint32_t w[U];
#pragma unroll
        for (int u = 0; u < U; u++) {  // all tests in flight, then all sets
            const uint32_t gv = c[u] * (uint32_t)V.p + o[u];
            w[u] = need[u] ? __ldcg(&V.sent[gv >> 5]) : 0xffffffffu;
        }
        // mark and ship without waiting for the atomic's old value: two senders
        // racing on one target may both ship it (the owner's claim is
        // idempotent; a segment holds one record per remote edge at most)
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t gv = c[u] * (uint32_t)V.p + o[u];
            const uint32_t bit = 1u << (gv & 31);
            ship[u] = need[u] && !(w[u] & bit);
#if DBFS_SENT_WAIT
            if (ship[u]) ship[u] = !(atomicOr(&V.sent[gv >> 5], bit) & bit);
#else
            if (ship[u]) atomicOr(&V.sent[gv >> 5], bit);
#endif
        }
    } else {
#pragma unroll
        for (int u = 0; u < U; u++) ship[u] = need[u];
    }
    // destinations with records to ship, then one slot reservation per destination
    unsigned long long dm = 0;
#pragma unroll
    for (int u = 0; u < U; u++)
        if (ship[u]) dm |= 1ull << o[u];
    {
        const unsigned lo = __reduce_or_sync(FULL, (unsigned)dm);
        const unsigned hi = V.p > 32 ? __reduce_or_sync(FULL, (unsigned)(dm >> 32)) : 0u;
        dm = ((unsigned long long)hi << 32) | lo;
    }
    const unsigned lt = (1u << lane_id()) - 1;
    while (dm) {
        const uint32_t dst = __ffsll(dm) - 1;
        dm &= dm - 1;
        unsigned b[U], tot = 0;
#pragma unroll
        for (int u = 0; u < U; u++) {
            b[u] = __ballot_sync(FULL, ship[u] && o[u] == dst);
            tot += __popc(b[u]);
        }
        if (V.peer && V.p <= 32) {
            // records [0, rem) finish this warp's chunk, the rest open a new one
            unsigned long long cur = __shfl_sync(FULL, vc.scur, dst), end = __shfl_sync(FULL, vc.send, dst);
            const unsigned long long rem = end - cur;
            unsigned long long nb = 0;
            if (rem < tot) {
                if (lane_id() == 0) nb = atomicAdd(&V.ctl->s[L % 3].sent[dst], (unsigned long long)SEND_CHUNK);
                nb = __shfl_sync(FULL, nb, 0);
            }
            unsigned before = 0;
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (ship[u] && o[u] == dst) {
                    const unsigned long long r = before + __popc(b[u] & lt);
                    V.sendbin[dst][r < rem ? cur + r : nb + (r - rem)] = make_uint2(c[u], parent[u]);
                }
                before += __popc(b[u]);
            }
            if (rem < tot) {
                cur = nb + (tot - rem);
                end = nb + SEND_CHUNK;
            } else {
                cur += tot;
            }
            if (lane_id() == dst) {
                vc.scur = cur;
                vc.send = end;
            }
            continue;
        }
        unsigned long long base = 0;
        if (lane_id() == 0) base = atomicAdd(&V.ctl->s[L % 3].sent[dst], (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 0);
        unsigned before = 0;
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (ship[u] && o[u] == dst)
                V.sendbin[dst][base + before + __popc(b[u] & lt)] = make_uint2(c[u], parent[u]);
            before += __popc(b[u]);
        }
    }
}

enum { ACT_NN = 0, ACT_DELEG = 1, ACT_NORMAL = 2 };

#ifndef DBFS_SEEN_L1
#define DBFS_SEEN_L1 0
#endif

// Second stage of a push step: U columns per lane are resolved with all
// status loads issued before any store (stores through the non-restrict state
// pointers would otherwise serialise one L2 round trip per edge).
template <int ACT, bool CNT, int U>
__device__ __forceinline__ void push_stage(const View &V, int L, const uint32_t (&cc)[U], const uint32_t (&pp)[U],
                                           const uint32_t (&tw)[U], uint32_t *first, const bool (&valid)[U],
                                           VisitCounters &vc) {
    const bool light = vc.light;
    // map the column to the (worker-local) vertex it names
    uint32_t tgt[U];
    bool local[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        local[u] = true;
        tgt[u] = cc[u];
        if (ACT == ACT_NN && V.p > 1) {
            local[u] = (int)V.pd.mod(cc[u]) == V.w;
            tgt[u] = V.pd.div(cc[u]);
        }
    }
    const uint32_t *vis = ACT == ACT_DELEG ? V.dvis : V.nvis;
    uint32_t *nxt = ACT == ACT_DELEG ? V.dnext[L & 1] : V.nfront[(L + 1) & 1];
    uint32_t *seen = ACT == ACT_DELEG ? V.dseen : V.nseen;
    uint32_t s[U];
    if (!CNT) {
        // one L2 test per edge: `seen` = visited(<= L) + the claims of this level
        // (kept separately from the pre-state `vis`, which pulls and counters
        // need; F leaves seen == vis for the next level)
#pragma unroll
        for (int u = 0; u < U; u++)
            s[u] = (valid[u] && local[u]) ? ((DBFS_SEEN_L1 == 1 || (DBFS_SEEN_L1 == 2 && ACT == ACT_DELEG)) ? __ldca(&seen[tgt[u] >> 5]) : __ldcg(&seen[tgt[u] >> 5]))
                                          : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ACT == ACT_DELEG && !((s[u] >> (tgt[u] & 31)) & 1u)) vc.dirty = 1;
    } else {
        // counting push: every parent of a target unvisited at level L bids its
        // twin position, claimed this level or not (the pull stops at the first)
#pragma unroll
        for (int u = 0; u < U; u++) s[u] = (valid[u] && local[u]) ? __ldca(&vis[tgt[u] >> 5]) : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < U; u++) {
            bool open = !((s[u] >> (tgt[u] & 31)) & 1u);
            if (ACT == ACT_DELEG && open) vc.dirty = 1;
            if (open) atomicMin(&first[tgt[u]], tw[u]);
            s[u] = open ? __ldcg(&seen[tgt[u] >> 5]) : 0xffffffffu;
        }
    }
    // fire-and-forget marks (RED.OR, no return value) and plain stores:
    // concurrent writers of one vertex store the same level and a valid parent.
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint32_t x = tgt[u];
        if ((s[u] >> (x & 31)) & 1u) continue;
        atomicOr(&seen[x >> 5], 1u << (x & 31));
        atomicOr(&nxt[x >> 5], 1u << (x & 31));
        if (ACT == ACT_DELEG) {
            if (V.parents) V.dcand[x] = pp[u];
        } else if (V.parents) {
            V.nparent[x] = pp[u];
        }
    }
    if (ACT != ACT_DELEG && light) {
        // light level: the claims' chunks into the touch bitmap / chunk list
#pragma unroll
        for (int u = 0; u < U; u++)
            if (!((s[u] >> (tgt[u] & 31)) & 1u)) touch_chunk(V, L, tgt[u]);
    }
    if (ACT == ACT_NN && V.p > 1) {
        bool remote[U];
        uint32_t own[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            remote[u] = valid[u] && !local[u];
            own[u] = V.pd.mod(cc[u]);
        }
        warp_send_batch(V, L, remote, own, tgt, pp, vc);
    }
}

// Expand <= 32 rows held one per lane (row start rb, length len, payload par)
// with all lanes on consecutive edges and U independent loads per lane.
template <int ACT, bool CNT = false, int U = ROWS_UNR>
__device__ __forceinline__ void warp_rows_push(const View &V, int L, const uint32_t *__restrict__ col, int64_t rb,
                                               uint32_t len, uint32_t par, VisitCounters &vc,
                                               const uint32_t *__restrict__ twin = nullptr, uint32_t *first = nullptr) {
    unsigned tot;
    unsigned excl = warp_excl_scan(len, &tot);
    const unsigned lane = lane_id();
    const int64_t delta = rb - (int64_t)excl;
    for (unsigned base = 0; base < tot; base += 32 * U) {
        uint32_t cc[U];
        uint32_t pp[U];
        uint32_t tw[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            unsigned x = base + u * 32 + lane;
            int o = owner_search<unsigned>(excl, x);
            const int64_t dl = __shfl_sync(FULL, delta, o);  // entry x at column dl + x
            pp[u] = __shfl_sync(FULL, par, o);
            cc[u] = x < tot ? __ldg(&col[dl + x]) : 0u;
            tw[u] = (CNT && x < tot) ? __ldg(&twin[dl + x]) : 0u;
        }
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; u++) valid[u] = base + u * 32 + lane < tot;
        push_stage<ACT, CNT, U>(V, L, cc, pp, tw, first, valid, vc);
    }
}

// Load-balanced push over a delegate frontier list (dlist, exclusive prefix
// dpre, `cnt` rows, `total` edges): this warp handles edges [x0, x1).
template <int ACT, bool CNT, int U = LIST_UNR>
__device__ __forceinline__ void list_push(const View &V, int L, const int64_t *__restrict__ off,
                                          const uint32_t *__restrict__ col, const uint32_t *__restrict__ list,
                                          const int64_t *__restrict__ pre, int64_t cnt, int64_t total, int64_t x0,
                                          int64_t x1, VisitCounters &vc, const uint32_t *__restrict__ twin,
                                          uint32_t *first) {
    if (x0 >= x1) return;
    const unsigned lane = lane_id();
    // 32-ary search: largest e with pre[e] <= x0
    int64_t lo = 0, hi = cnt;
    while (hi - lo > 32) {
        int64_t step = (hi - lo + 31) / 32;
        int64_t idx = lo + (int64_t)lane * step;
        bool ok = idx < hi && pre[idx] <= x0;
        unsigned m = __ballot_sync(FULL, ok);
        int l = 31 - __clz(m);
        lo = lo + (int64_t)l * step;
        hi = lo + step < hi ? lo + step : hi;
    }
    {
        int64_t idx = lo + lane;
        bool ok = idx < hi && pre[idx] <= x0;
        unsigned m = __ballot_sync(FULL, ok);
        lo += 31 - __clz(m);
    }
    int64_t i = lo;
    while (x0 < x1) {
        int64_t e = i + lane;
        int64_t pb = e < cnt ? pre[e] : total;
        uint32_t v = e < cnt ? list[e] : 0u;
        int64_t rb = e < cnt ? __ldg(&off[v]) : 0;
        uint32_t gx = e < cnt ? __ldg(&V.del_gid32[v]) : 0u;
        int64_t wend = 0;
        if (lane == 0) wend = (i + 32 < cnt) ? pre[i + 32] : total;
        wend = __shfl_sync(FULL, wend, 0);
        int64_t lim = wend < x1 ? wend : x1;
        // 32-bit keys relative to the window's first row (a window of 32 rows
        // holds < 2^32 edges): half the shuffles of the owner search; entry x
        // of the window lives at column delta(owner) + x
        const int64_t wbase = __shfl_sync(FULL, pb, 0);
        const int64_t rel = pb - wbase;
        const uint32_t pb32 = rel < 0xffffffffll ? (uint32_t)rel : 0xffffffffu;
        const int64_t delta = rb - pb;
        for (int64_t base = x0; base < lim; base += 32 * U) {
            uint32_t cc[U];
            uint32_t pp[U];
            uint32_t tw[U];
            const uint32_t b32 = (uint32_t)(base - wbase);
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t x = base + u * 32 + lane;
                const int o = owner_search<uint32_t>(pb32, b32 + (uint32_t)(u * 32) + lane);
                const int64_t dl = __shfl_sync(FULL, delta, o);
                pp[u] = __shfl_sync(FULL, gx, o);
                cc[u] = x < lim ? __ldg(&col[dl + x]) : 0u;
                tw[u] = (CNT && x < lim) ? __ldg(&twin[dl + x]) : 0u;
            }
            bool valid[U];
#pragma unroll
            for (int u = 0; u < U; u++) valid[u] = base + u * 32 + lane < lim;
            push_stage<ACT, CNT, U>(V, L, cc, pp, tw, first, valid, vc);
        }
        x0 = lim;
        i += 32;
    }
}

// ------------------------------------------------------------------- pulls
// Early-exit scan (traversal.py:111-139): the first column of row [b, e) whose
// bit is set in `front`.  A lane scans its row in geometric rounds (loads and
// bit tests of a round in flight together) and hands rows still unresolved
// after 30 entries to the whole warp (32 * PULL_U columns per step, ballot).

struct PullRes {
    int64_t pos;  // absolute index of the first hit, or -1
    uint32_t col;
};

template <int W>
__device__ __forceinline__ bool lane_round(const uint32_t *__restrict__ col, const uint32_t *__restrict__ front,
                                           const uint32_t *filt, int64_t &j, int64_t e, PullRes &r) {
    uint32_t c[W];
    bool h[W];
#pragma unroll
    for (int u = 0; u < W; u++) c[u] = j + u < e ? __ldg(&col[j + u]) : 0u;
#pragma unroll
    for (int u = 0; u < W; u++) h[u] = j + u < e && (!filt || coarse_hit(filt, c[u]));
#pragma unroll
    for (int u = 0; u < W; u++) h[u] = h[u] && tbit(front, c[u]);
#pragma unroll
    for (int u = 0; u < W; u++)
        if (h[u]) {
            r.pos = j + u;
            r.col = c[u];
            return true;
        }
    j += W;
    return false;
}

// Geometric rounds (2, 4, 8, 16 entries): a hit near the row start costs two
// tests, long scans still keep 16 loads in flight.  Returns true when resolved.
__device__ __forceinline__ bool lane_scan(const uint32_t *__restrict__ col, const uint32_t *__restrict__ front,
                                          const uint32_t *filt, int64_t b, int64_t e, int64_t &j, PullRes &r) {
    j = b;
    r.pos = -1;
    if (j < e && lane_round<2>(col, front, filt, j, e, r)) return true;
    if (j < e && lane_round<4>(col, front, filt, j, e, r)) return true;
    if (j < e && lane_round<8>(col, front, filt, j, e, r)) return true;
    if (j < e && lane_round<16>(col, front, filt, j, e, r)) return true;
    if (j >= e) {
        r.pos = -1;
        return true;
    }
    return false;
}

__device__ __forceinline__ PullRes warp_scan_row(const uint32_t *__restrict__ col, const uint32_t *__restrict__ front,
                                                 const uint32_t *filt, int64_t j, int64_t e) {
    const unsigned lane = lane_id();
    PullRes r;
    r.pos = -1;
    r.col = 0;
    for (; j < e; j += 32 * PULL_U) {
        uint32_t c[PULL_U];
        bool h[PULL_U];
#pragma unroll
        for (int u = 0; u < PULL_U; u++) {
            int64_t x = j + u * 32 + lane;
            c[u] = x < e ? __ldg(&col[x]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < PULL_U; u++) h[u] = (j + u * 32 + lane < e) && (!filt || coarse_hit(filt, c[u]));
#pragma unroll
        for (int u = 0; u < PULL_U; u++) h[u] = h[u] && tbit(front, c[u]);
#pragma unroll
        for (int u = 0; u < PULL_U; u++) {
            unsigned m = __ballot_sync(FULL, h[u]);
            if (m) {
                int l = __ffs(m) - 1;
                r.pos = j + u * 32 + l;
                r.col = __shfl_sync(FULL, c[u], l);
                return r;
            }
        }
    }
    return r;
}

// One pull kind over its candidate words.  cand(wi) gives the candidate bits
// of word wi; rows come from (off, col); `front` is the parent status bitmap;
// on_hit(candidate, hit column) records the find.
// Chunks [0, n) of 32 bitmap words over the warps of one worker: chunk gw
// first, then chunks claimed from a per-level counter, prefetched one chunk
// ahead so the atomic's latency hides behind the current chunk.  Degree skew
// makes chunk costs uneven; claiming on demand keeps warps finishing together.
#ifndef DBFS_DYN
#define DBFS_DYN 1
#endif
#ifndef DBFS_CWD
#define DBFS_CWD 8   // bitmap words per chunk over delegates (d/32 words: few, heavy)
#endif
#ifndef DBFS_CWN
#define DBFS_CWN 32  // bitmap words per chunk over normals
#endif
struct WarpChunks {
    unsigned *ctr;  // nullptr: static stride (light levels, where a claim costs more than a chunk)
    int n, TW, cur, cw;
    unsigned pend;
    __device__ __forceinline__ WarpChunks(unsigned *c, int64_t nwords, int cw_, int64_t gw, int64_t tw)
        : ctr(DBFS_DYN ? c : nullptr), n((int)((nwords + cw_ - 1) / cw_)), TW((int)tw), cur((int)gw), cw(cw_) {
        pend = (ctr && lane_id() == 0 && cur < n) ? atomicAdd(ctr, 1u) : 0u;
    }
    __device__ __forceinline__ bool valid() const { return cur < n; }
    __device__ __forceinline__ int64_t base() const { return (int64_t)cur * cw; }
    // lane's word of the chunk, or -1
    __device__ __forceinline__ int64_t word(int64_t nwords) const {
        const int64_t wi = base() + lane_id();
        return ((int)lane_id() < cw && wi < nwords) ? wi : -1;
    }
    __device__ __forceinline__ void next() {
        if (!ctr) {
            cur += TW;
            return;
        }
        cur = TW + (int)__shfl_sync(FULL, pend, 0);
        pend = (lane_id() == 0 && cur < n) ? atomicAdd(ctr, 1u) : 0u;
    }
};

#ifndef DBFS_PULL_SPLIT
#define DBFS_PULL_SPLIT 1
#endif
#ifndef DBFS_SPLIT_PROBE
#define DBFS_SPLIT_PROBE 4
#endif
constexpr int SPROBE = DBFS_SPLIT_PROBE;  // head probes of 32 candidates in flight per lane (pull_split)
// Candidates of one chunk (list[0, cnt)) in two passes: all row heads first
// (PROBE groups of 32 in flight, hits recorded at once), the misses compacted
// in place to the front of the list, then the misses' scans 32 per step, so a
// warp's lanes all scan instead of idling beside resolved heads.
template <class HitF>
__device__ __forceinline__ void pull_split(unsigned cnt, uint32_t *list, const int64_t *__restrict__ off,
                                           const uint32_t *__restrict__ col, const uint32_t *__restrict__ head,
                                           const uint32_t *__restrict__ front, const uint32_t *filt,
                                           unsigned long long &insp, HitF on_hit) {
    const unsigned lane = lane_id();
    unsigned nmiss = 0;
    for (unsigned g0 = 0; g0 < cnt; g0 += 32 * SPROBE) {
        uint32_t v[SPROBE], c0[SPROBE];
        bool ok[SPROBE], h0[SPROBE];
#pragma unroll
        for (int q = 0; q < SPROBE; q++) {
            unsigned i = g0 + q * 32 + lane;
            ok[q] = i < cnt;
            v[q] = ok[q] ? list[i] : 0u;
        }
#pragma unroll
        for (int q = 0; q < SPROBE; q++) c0[q] = ok[q] ? __ldg(&head[v[q]]) : 0u;
#pragma unroll
        for (int q = 0; q < SPROBE; q++) h0[q] = ok[q] && (!filt || coarse_hit(filt, c0[q])) && tbit(front, c0[q]);
        __syncwarp();  // this step's list entries are in registers: misses may overwrite them
#pragma unroll
        for (int q = 0; q < SPROBE; q++) {
            if (h0[q]) insp++;
            on_hit(h0[q], v[q], c0[q]);
            const bool miss = ok[q] && !h0[q];
            const unsigned m = __ballot_sync(FULL, miss);
            if (miss) list[nmiss + __popc(m & ((1u << lane) - 1u))] = v[q];
            nmiss += __popc(m);
        }
    }
    __syncwarp();
    for (unsigned g0 = 0; g0 < nmiss; g0 += 32) {
        const unsigned i = g0 + lane;
        const bool ok = i < nmiss;
        const uint32_t v = ok ? list[i] : 0u;
        const int64_t b = ok ? __ldg(&off[v]) : 0, e = ok ? __ldg(&off[v + 1]) : 0;
        PullRes r;
        r.pos = -1;
        r.col = 0;
        int64_t j = e;
        bool done = !ok || b + 1 >= e;
        if (!done) done = lane_scan(col, front, filt, b + 1, e, j, r);
        unsigned pend = __ballot_sync(FULL, !done);
        while (pend) {
            int l = __ffs(pend) - 1;
            pend &= pend - 1;
            int64_t jl = __shfl_sync(FULL, j, l), el = __shfl_sync(FULL, e, l);
            PullRes rr = warp_scan_row(col, front, filt, jl, el);
            if ((int)lane == l) r = rr;
        }
        const bool hit = ok && r.pos >= 0;
        if (ok) insp += (unsigned long long)(hit ? r.pos - b + 1 : e - b);
        on_hit(hit, v, r.col);
    }
}

template <class CandF, class HitF>
__device__ __forceinline__ void pull_kind(int64_t nw, int cw, int64_t gw, int64_t TW, unsigned *sched, uint32_t *list,
                                          const int64_t *__restrict__ off, const uint32_t *__restrict__ col,
                                          const uint32_t *__restrict__ head, const uint32_t *__restrict__ front,
                                          const uint32_t *filt, unsigned long long &insp, unsigned long long &rows,
                                          CandF cand, HitF on_hit) {
    const unsigned lane = lane_id();
    for (WarpChunks ch(sched, nw, cw, gw, TW); ch.valid(); ch.next()) {
        const int64_t wi = ch.word(nw);
        uint32_t word = wi >= 0 ? cand(wi) : 0u;
        unsigned cnt = warp_compact(word, wi, list);
        if (lane == 0) rows += cnt;
        if (DBFS_PULL_SPLIT && head) {
            pull_split(cnt, list, off, col, head, front, filt, insp, on_hit);
            __syncwarp();
            continue;
        }
        // First probe of 4 groups at once (4 independent chains per lane):
        // offsets, first column, its status bit.  Most candidates resolve here
        // at dense levels; the rest continue with the geometric lane scan.
        for (unsigned g0 = 0; g0 < cnt; g0 += 32 * PROBE) {
            uint32_t v[PROBE], c0[PROBE];
            int64_t b[PROBE], e[PROBE];
            bool ok[PROBE], h0[PROBE];
#pragma unroll
            for (int q = 0; q < PROBE; q++) {
                unsigned i = g0 + q * 32 + lane;
                ok[q] = i < cnt;
                v[q] = ok[q] ? list[i] : 0u;
            }
            if (head) {
                // row heads: a candidate's first column from a dense per-row array
                // (coalesced, no offsets, no random column sector); only the misses
                // load their offsets and scan on from the second entry.  Candidates
                // come from the rows-present bitmap, so every row has a head.
#pragma unroll
                for (int q = 0; q < PROBE; q++) c0[q] = ok[q] ? __ldg(&head[v[q]]) : 0u;
#pragma unroll
                for (int q = 0; q < PROBE; q++)
                    h0[q] = ok[q] && (!filt || coarse_hit(filt, c0[q])) && tbit(front, c0[q]);
#pragma unroll
                for (int q = 0; q < PROBE; q++) {
                    const bool need = ok[q] && !h0[q];
                    b[q] = need ? __ldg(&off[v[q]]) : 0;
                    e[q] = need ? __ldg(&off[v[q] + 1]) : (h0[q] ? 1 : 0);
                }
            } else {
#pragma unroll
                for (int q = 0; q < PROBE; q++) {
                    b[q] = ok[q] ? __ldg(&off[v[q]]) : 0;
                    e[q] = ok[q] ? __ldg(&off[v[q] + 1]) : 0;
                }
#pragma unroll
                for (int q = 0; q < PROBE; q++) c0[q] = (ok[q] && b[q] < e[q]) ? __ldg(&col[b[q]]) : 0u;
#pragma unroll
                for (int q = 0; q < PROBE; q++)
                    h0[q] = ok[q] && b[q] < e[q] && (!filt || coarse_hit(filt, c0[q])) && tbit(front, c0[q]);
            }
#pragma unroll
            for (int q = 0; q < PROBE; q++) {
                PullRes r;
                r.pos = h0[q] ? b[q] : -1;
                r.col = c0[q];
                int64_t j = e[q];
                bool done = !ok[q] || h0[q] || b[q] + 1 >= e[q];
                if (!done) done = lane_scan(col, front, filt, b[q] + 1, e[q], j, r);
                unsigned pend = __ballot_sync(FULL, !done);
                while (pend) {
                    int l = __ffs(pend) - 1;
                    pend &= pend - 1;
                    int64_t jl = __shfl_sync(FULL, j, l), el = __shfl_sync(FULL, e[q], l);
                    PullRes rr = warp_scan_row(col, front, filt, jl, el);
                    if ((int)lane == l) r = rr;
                }
                const bool hit = ok[q] && r.pos >= 0;
                if (ok[q]) insp += (unsigned long long)(hit ? r.pos - b[q] + 1 : e[q] - b[q]);
                on_hit(hit, v[q], r.col);  // warp-uniform call: marks are aggregated per word
            }
        }
        __syncwarp();
    }
}

// Warp-uniform mark of candidate v (lanes with hit): lanes of the warp hold
// near-consecutive candidates, so bits of one word are OR-ed in registers and
// the word gets one RED.OR.
__device__ __forceinline__ void warp_mark(uint32_t *bm, bool hit, uint32_t v) {
    const unsigned wkey = hit ? (v >> 5) : 0xffffffffu;
    const unsigned peers = __match_any_sync(FULL, wkey);
    const unsigned bits = __reduce_or_sync(peers, hit ? (1u << (v & 31)) : 0u);
    if (hit && (int)lane_id() == __ffs(peers) - 1) atomicOr(&bm[v >> 5], bits);
}

// Pulls of kind k are balanced dynamically when many candidates remain (the
// unvisited sources of the reverse kind), statically on light tail levels.
__device__ __forceinline__ bool dyn_pull(const View &V, const unsigned long long *cum, int k, int64_t TW) {
    unsigned long long U, Q, Sx;
    const unsigned long long q0[4] = {0, 0, 0, 0};
    level_inputs(V.total_src, cum, q0, k, U, Q, Sx);
    return U > (unsigned long long)V.pull_dyn_min * (unsigned long long)TW;
}

// The record of level L made by one whole warp (the message flags and timers
// copied lane-parallel, the scalar fields by lane 0).
__device__ __forceinline__ void make_record_warp(const View &V, const Ctl &c, int L, IterRec &r) {
    const LevelSlot &S = c.s[L % 3];
    const unsigned lane = lane_id();
    unsigned long long msgs = 0;
    for (int o = lane; o < MAXW; o += 32) {
        const unsigned long long x = S.send[o];
        r.send[o] = x;
        msgs += x > 0;
    }
    msgs = warp_sum(msgs);
    if (lane < 8) {
        r.tsum[lane] = S.tsum[lane];
        r.tmax[lane] = S.tmax[lane];
    }
    if (lane == 0) {
        make_record_core(V, c, L, r);
        r.messages = msgs;
    }
}

// Block-level counter aggregation: warps add into shared memory, then one
// global atomic per counter per block (instead of one per warp: thousands of
// same-address atomics per counter and phase otherwise).
constexpr int NACC = 16;
__device__ __forceinline__ unsigned long long *block_acc() {
    __shared__ unsigned long long s_acc[NACC];
    return s_acc;
}
__device__ __forceinline__ void block_acc_clear() {
    if (threadIdx.x < NACC) block_acc()[threadIdx.x] = 0ull;
}
__device__ __forceinline__ void warp_acc(int i, unsigned long long x) {
    const unsigned long long v = warp_sum(x);
    if (lane_id() == 0 && v) atomicAdd(&block_acc()[i], v);
}
// After a __syncthreads: thread i < n adds slot i to dst[i] (nullptr: skip).
__device__ __forceinline__ void block_acc_flush(unsigned long long *const *dst, int n) {
    if ((int)threadIdx.x < n && dst[threadIdx.x]) {
        const unsigned long long v = block_acc()[threadIdx.x];
        if (v) atomicAdd(dst[threadIdx.x], v);
    }
}

// -------------------------------------------------------------- phase V(L)

// DBFS_TRACE diagnostics: block-level timestamp of phase boundary `ph` of level
// L -- 0 V start, 1 T1 start, 2 T1 end, 3 pulls start, 4 V work end, 5 V done,
// 6 F start, 7 F done (block-uniform; adds a __syncthreads only when tracing).
__device__ __forceinline__ void trace_stamp(const View &V, int L, int ph) {
    if (!V.trace || L >= 64) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        V.trace[((size_t)L * 8 + ph) * gridDim.x + blockIdx.x] = t;
    }
}

__device__ void phase_visit(const View &V, int L, int wb, int nb, Smem &sm) {
    Ctl &C = *V.ctl;
    const LevelSlot &S = C.s[L % 3];
    int dirs[4];
    double bv[4];
    unsigned long long cum[4];
    level_dirs(V, C, L, dirs, bv, cum);
    int ex[4];
    exec_dirs(V, S, cum, dirs, ex);
    // light level: few normal claims expected (no dn pull, pushed normal-target
    // edges <= n_local/32), so claims mark the touch bitmap for F and T1
    const bool light = V.W == 1 && ex[KIND_DN] != BWD &&
                       S.fv[KIND_NN] + (ex[KIND_DN] != BWD ? S.fv[KIND_DN] : 0ull) <= (unsigned long long)V.nw_n;
    // frontier L's chunk list is complete when V(L-1) was light (level 0: the seed lists it)
    const bool prev_light = V.W == 1 && (L == 0 || C.s[(L + 2) % 3].light != 0);
    if (wb == 0 && threadIdx.x == 0) {
        unsigned long long cumfv[4];
        for (int k = 0; k < 4; k++) cumfv[k] = (L == 0 ? 0ull : C.cumfv[(L + 1) & 1][k]) + S.fv[k];
        for (int k = 0; k < 4; k++) {
            C.dir[L & 1][k] = dirs[k];
            C.cumq[L & 1][k] = cum[k];
            C.cumfv[L & 1][k] = cumfv[k];
            C.s[L % 3].exec_dir[k] = ex[k];
            if (k == 0) {
                C.s[L % 3].light = light ? 1ull : 0ull;
                C.s[L % 3].prev_light = prev_light ? 1ull : 0ull;
            }
            C.s[L % 3].bv[k] = bv[k];
            if (k == 0) C.s[L % 3].prev_dirty = L > 0 ? C.s[(L + 2) % 3].dirty : 0ull;
            if (k > 0 && ex[k] != BWD) C.s[L % 3].work[k] = S.fv[k];
            // counting push: the candidates' reverse-row lengths; F(L) takes off
            // what the early exits of the found ones skip
            if (k > 0 && ex[k] == PUSHC) atomicAdd(&C.s[L % 3].insp_bwd[k], V.nnz[rev_kind(k)] - cumfv[rev_kind(k)]);
        }
    }
    VisitCounters vc = {};
    vc.light = light;
    block_acc_clear();
    __syncthreads();
    const unsigned lane = lane_id(), warp = warp_id();
    const int64_t gw = (int64_t)wb * WPB + warp, TW = (int64_t)nb * WPB;
    uint32_t *list = sm.list[warp];
    if (V.p > 1) {
        if (threadIdx.x == 0) *block_sendmask() = 0ull;
        __syncthreads();
    }
    const int p = V.p, w = V.w;
    const uint32_t *nfront_cur = V.nfront[L & 1];

    LevelSlot &AT = C.s[L % 3];
    TaskTimer tt;
    trace_stamp(V, L, 1);
    // T1: normal frontier -- nn push (always, engine.py:207-222) + nd push.
    tt.start();
    if (S.nfront > 0) {
        const bool nd_fwd = ex[KIND_ND] != BWD && S.fv[KIND_ND] > 0;
        const bool nd_cnt = ex[KIND_ND] == PUSHC && V.first[KIND_ND];
        const uint32_t *has_nn = V.src_bits[KIND_NN], *has_nd = V.src_bits[KIND_ND];
        // claim chunks dynamically only when the rows to push, not the bitmap
        // scan, dominate (uniform frontier bits balance a static stride)
        const unsigned long long t1_edges = S.fv[KIND_NN] + (nd_fwd ? S.fv[KIND_ND] : 0ull);
        const bool t1_dyn = S.nfront > (unsigned long long)TW && t1_edges > (unsigned long long)V.t1_dyn_min * V.nw_n;
        const uint32_t *touch = V.ntouch[L & 1];
        // one 32-word chunk of the frontier: compaction, then 32 rows per warp step
        auto push_chunk = [&](int64_t chunk) {
            const int64_t wi = chunk * 32 + lane;
            // only frontier vertices with an nn row (or an nd row when nd pushes)
            uint32_t word = wi < V.nw_n ? (nfront_cur[wi] & (has_nn[wi] | (nd_fwd ? has_nd[wi] : 0u))) : 0u;
            unsigned cnt = warp_compact(word, wi < V.nw_n ? wi : 0, list);
            for (unsigned g0 = 0; g0 < cnt; g0 += 32) {
                unsigned i = g0 + lane;
                bool ok = i < cnt;
                uint32_t u = ok ? list[i] : 0u;
                uint32_t gid = u * (uint32_t)p + (uint32_t)w;
                int64_t b = ok ? __ldg(&V.off[KIND_NN][u]) : 0, e = ok ? __ldg(&V.off[KIND_NN][u + 1]) : 0;
                vc.fv_nn += (unsigned long long)(e - b);
                warp_rows_push<ACT_NN>(V, L, V.col[KIND_NN], b, (uint32_t)(e - b), gid, vc);
                if (nd_fwd) {
                    int64_t b2 = ok ? __ldg(&V.off[KIND_ND][u]) : 0, e2 = ok ? __ldg(&V.off[KIND_ND][u + 1]) : 0;
                    if (nd_cnt)
                        warp_rows_push<ACT_DELEG, true>(V, L, V.col[KIND_ND], b2, (uint32_t)(e2 - b2), gid, vc,
                                                        V.twin[KIND_ND], V.first[KIND_ND]);
                    else
                        warp_rows_push<ACT_DELEG>(V, L, V.col[KIND_ND], b2, (uint32_t)(e2 - b2), gid, vc);
                }
            }
            __syncwarp();
        };
        if (prev_light) {
            // frontier listed by the claims of a light V(L-1): a listed chunk per warp
            const int64_t nl = (int64_t)S.nchunks;
            for (int64_t i = gw; i < nl; i += TW) push_chunk(V.nchunk_list[L & 1][i]);
        } else {
            for (WarpChunks ch(t1_dyn ? &AT.sched[0] : nullptr, V.nw_n, DBFS_CWN, gw, TW); ch.valid(); ch.next()) {
                // chunks without frontier vertices are skipped
                if (!((__ldcg(&touch[ch.cur >> 5]) >> (ch.cur & 31)) & 1u)) continue;
                push_chunk(ch.cur);
            }
        }
    }

    tt.stop(AT, 0);
    trace_stamp(V, L, 2);
    // T2: delegate frontier -- dn / dd push, load balanced over the level's
    // edge space (engine.py:238-263).
    tt.start();
    const unsigned long long EM = (1ull << V.dshift) - 1;  // packed list: count << dshift | edges
    if (ex[KIND_DN] != BWD && (S.dpack[0] & EM)) {
        int64_t cnt = (int64_t)(S.dpack[0] >> V.dshift), total = (int64_t)(S.dpack[0] & EM);
        int64_t x0 = gw * total / TW, x1 = (gw + 1) * total / TW;
        if (ex[KIND_DN] == PUSHC && V.first[KIND_DN])
            list_push<ACT_NORMAL, true>(V, L, V.off[KIND_DN], V.col[KIND_DN], V.dlist[0][L & 1], V.dpre[0][L & 1], cnt,
                                        total, x0, x1, vc, V.twin[KIND_DN], V.first[KIND_DN]);
        else
            list_push<ACT_NORMAL, false>(V, L, V.off[KIND_DN], V.col[KIND_DN], V.dlist[0][L & 1], V.dpre[0][L & 1],
                                         cnt, total, x0, x1, vc, nullptr, nullptr);
    }
    tt.stop(AT, 1);
    tt.start();
    if (ex[KIND_DD] != BWD && (S.dpack[1] & EM)) {
        int64_t cnt = (int64_t)(S.dpack[1] >> V.dshift), total = (int64_t)(S.dpack[1] & EM);
        int64_t x0 = gw * total / TW, x1 = (gw + 1) * total / TW;
        if (ex[KIND_DD] == PUSHC && V.first[KIND_DD])
            list_push<ACT_DELEG, true>(V, L, V.off[KIND_DD], V.col[KIND_DD], V.dlist[1][L & 1], V.dpre[1][L & 1], cnt,
                                       total, x0, x1, vc, V.twin[KIND_DD], V.first[KIND_DD]);
        else
            list_push<ACT_DELEG, false>(V, L, V.off[KIND_DD], V.col[KIND_DD], V.dlist[1][L & 1], V.dpre[1][L & 1],
                                        cnt, total, x0, x1, vc, nullptr, nullptr);
    }
    tt.stop(AT, 2);

    trace_stamp(V, L, 3);
    // Pull frontiers that are sparse relative to the 2^18-bit coarse filter
    // are tested in shared memory first (block-uniform decisions).
    const bool dpull = ex[KIND_DN] == BWD || ex[KIND_DD] == BWD;
    const bool dfilt = DBFS_FILTER && dpull && (double)S.dfront < 0.7 * FW * 32;
    const bool nfilt = false;  // (the normal frontier has no coarse filter: light levels list their chunks)
    if (dfilt) {
        __syncthreads();
        const uint32_t *src = V.coarse_d[L & 1];
        for (int i = threadIdx.x; i < FW; i += BT) sm.filt[i] = __ldcg(&src[i]);
        __syncthreads();
    }
    const uint32_t *filt = dfilt ? sm.filt : nullptr;

    // T4: dn pull -- unvisited nd-source normals scan nd rows for frontier
    // delegates (engine.py:242-248).
    tt.start();
    if (ex[KIND_DN] == BWD) {
        const uint32_t *srcb = V.src_bits[KIND_ND];
        const uint32_t *nvis = V.nvis;
        pull_kind(V.nw_n, DBFS_CWN, gw, TW, dyn_pull(V, cum, KIND_DN, TW) ? &AT.sched[1] : nullptr, list, V.off[KIND_ND], V.col[KIND_ND], V.head[KIND_ND], V.dfront, filt, vc.insp_bwd[KIND_DN], vc.pull_rows,
                  [&](int64_t wi) { return srcb[wi] & ~nvis[wi]; },
                  [&](bool hit, uint32_t c, uint32_t x) {
                      warp_mark(V.nfront[(L + 1) & 1], hit, c);
                      if (hit && V.parents) V.nparent[c] = (parent_t)__ldg(&V.del_gid32[x]);
                  });
    }
    tt.stop(AT, 3);
    // T6: dd pull -- unvisited dd-source delegates scan dd rows (engine.py:257-261).
    tt.start();
    if (ex[KIND_DD] == BWD) {
        const uint32_t *srcb = V.src_bits[KIND_DD];
        const uint32_t *dvis = V.dvis;
        // reported FORWARD: any scan order finds the same set, so use the rows
        // sorted by neighbour degree (hubs first); reported BACKWARD: the
        // reference order, whose early-exit position is the counter.
        const bool sorted = dirs[KIND_DD] == FWD && V.col_sorted_dd;
        const uint32_t *cdd = sorted ? V.col_sorted_dd : V.col[KIND_DD];
        const uint32_t *hdd = sorted ? V.head_sorted_dd : V.head[KIND_DD];
        pull_kind(V.nw_d, DBFS_CWD, gw, TW, dyn_pull(V, cum, KIND_DD, TW) ? &AT.sched[2] : nullptr, list, V.off[KIND_DD], cdd, hdd, V.dfront, filt, vc.insp_bwd[KIND_DD], vc.pull_rows,
                  [&](int64_t wi) { return srcb[wi] & ~dvis[wi]; },
                  [&](bool hit, uint32_t x, uint32_t y) {
                      warp_mark(V.dnext[L & 1], hit, x);
                      if (hit) {
                          vc.dirty = 1;
                          if (V.parents) V.dcand[x] = (parent_t)__ldg(&V.del_gid32[y]);
                      }
                  });
    }
    tt.stop(AT, 5);
    if (nfilt) {
        __syncthreads();
        const uint32_t *src = V.coarse_n[L & 1];
        for (int i = threadIdx.x; i < FW; i += BT) sm.filt[i] = __ldcg(&src[i]);
        __syncthreads();
    }
    // T5: nd pull -- unvisited dn-source delegates scan dn rows for frontier
    // normals (engine.py:229-233).
    tt.start();
    if (ex[KIND_ND] == BWD) {
        const uint32_t *srcb = V.src_bits[KIND_DN];
        const uint32_t *dvis = V.dvis;
        pull_kind(V.nw_d, DBFS_CWD, gw, TW, dyn_pull(V, cum, KIND_ND, TW) ? &AT.sched[3] : nullptr, list, V.off[KIND_DN], V.col[KIND_DN], V.head[KIND_DN], nfront_cur, nfilt ? sm.filt : nullptr,
                  vc.insp_bwd[KIND_ND], vc.pull_rows,
                  [&](int64_t wi) { return srcb[wi] & ~dvis[wi]; },
                  [&](bool hit, uint32_t x, uint32_t c) {
                      warp_mark(V.dnext[L & 1], hit, x);
                      if (hit) {
                          vc.dirty = 1;
                          if (V.parents) V.dcand[x] = (parent_t)(c * (uint32_t)p + (uint32_t)w);
                      }
                  });
    }
    tt.stop(AT, 4);
    trace_stamp(V, L, 4);
    if (V.peer && V.p <= 32) {  // sentinel-fill the unused tails of this warp's inbox chunks
        for (int dst = 0; dst < V.p; dst++) {
            const unsigned long long cur = __shfl_sync(FULL, vc.scur, dst), end = __shfl_sync(FULL, vc.send, dst);
            for (unsigned long long i = cur + lane; i < end; i += 32) V.sendbin[dst][i] = make_uint2(REC_SKIP, 0u);
        }
    }
    // flush: warps into shared slots, one global atomic per counter per block
    LevelSlot &A = C.s[L % 3];
    warp_acc(0, vc.fv_nn);
    warp_acc(1, vc.records);
    warp_acc(2, vc.uq);
    warp_acc(3, vc.dirty);
    warp_acc(4, vc.pull_rows);
    for (int k = 1; k < 4; k++) warp_acc(4 + k, vc.insp_bwd[k]);
    __syncthreads();
    {
        unsigned long long *dst[11] = {&A.fv[KIND_NN], &A.records, &A.uq_records, nullptr, &A.pull_rows,
                                       dirs[KIND_ND] == BWD ? &A.insp_bwd[KIND_ND] : nullptr,
                                       dirs[KIND_DN] == BWD ? &A.insp_bwd[KIND_DN] : nullptr,
                                       dirs[KIND_DD] == BWD ? &A.insp_bwd[KIND_DD] : nullptr,
                                       &A.work[KIND_ND], &A.work[KIND_DN], &A.work[KIND_DD]};
        if (threadIdx.x >= 8 && threadIdx.x < 11) block_acc()[threadIdx.x] = block_acc()[threadIdx.x - 3];
        // work[k] of an executed pull = its inspections (slots 5..7 mirrored to 8..10)
        block_acc_flush(dst, 11);
        if (threadIdx.x == 11 && block_acc()[0]) atomicAdd(&A.work[KIND_NN], block_acc()[0]);
        if (threadIdx.x == 12 && block_acc()[3]) atomicOr(&A.dirty, 1ull);
    }
    if (V.p > 1) {
        const unsigned long long dm = *block_sendmask();
        for (int i = threadIdx.x; i < V.p; i += BT)
            if ((dm >> i) & 1) atomicOr(&A.send[i], 1ull);
    }
}

// ------------------------------------------------------------ phase F(L)

struct FinishCounters {
    unsigned long long dfv_dn, dq_dn, dfv_dd, dq_dd, new_del;
    unsigned long long nfv_nd, nq_nd, ncount;
    unsigned long long skip[4];  // counting pushes: sum over found targets of (len - first - 1)
};

constexpr uint32_t NO_FIRST = 0xffffffffu;

// Counting push of kind k at level L found target x (reverse-row length len):
// the pull would have stopped after first+1 entries.  Resets the slot.
__device__ __forceinline__ void take_first(uint32_t *first, uint32_t x, uint64_t len, unsigned long long &skip) {
    const uint32_t f = first[x];
    if (f != NO_FIRST) {
        skip += len - f - 1;
        first[x] = NO_FIRST;
    }
}

// Delegate state of new delegate x (lane-held): level, parent, global output.
// gx = its global id (loaded when the global outputs are written here), par =
// its parent when the caller already has it (one in-process worker), else
// the minimum over the candidates of the workers that found it.
#ifndef DBFS_NB
#define DBFS_NB 4
#endif
constexpr int NB_DEL = DBFS_NB;  // new vertices per lane whose loads are in flight together (F1, F3)

__device__ __forceinline__ void new_delegate(const View &V, int L, uint32_t x, int64_t gx, parent_t par_known) {
    const uint32_t xw = x >> 5, xb = x & 31;
    V.dlevel[x] = L + 1;
    parent_t par = PARENT_MAX;
    if (V.parents) {
        if (V.cand_all && V.P_sources == 1) {
            par = par_known;
        } else if (V.cand_all) {
            for (int s = 0; s < V.P_sources; s++)
                if ((__ldcg(&V.mask_src[L & 1][s][xw]) >> xb) & 1u) {
                    const parent_t c = __ldcg(&V.cand_src[s][x]);
                    par = c < par ? c : par;
                }
        } else if ((V.dnext[L & 1][xw] >> xb) & 1u) {
            par = V.dcand[x];
        }
        V.dparent[x] = par;
    }
    if (V.glevel) {
        V.glevel[gx] = L + 1;
        if (V.parents) V.gparent[gx] = par;
    }
}

#ifndef DBFS_F1_FEW
#define DBFS_F1_FEW 1
#endif

// F1: delegate mask OR-reduction (comm.py:75-98) -> delegates of level L+1,
// their state, and the push lists of level L+1 (one packed atomic per warp
// batch and kind keeps list positions and edge prefixes consistent).
__device__ void finish_delegates(const View &V, int L, int64_t gw, int64_t TW, uint32_t *list, FinishCounters &fc) {
    const unsigned lane = lane_id();
    uint32_t *next_mask = V.dnext[(L + 1) & 1];
    LevelSlot &N = V.ctl->s[(L + 1) % 3];
    // sources that found delegates this level (a clean source's mask is all
    // zero): the others' masks -- NVLink reads in the peer engine -- are skipped
    __shared__ unsigned long long s_src;
    if (threadIdx.x == 0) s_src = 0ull;
    __syncthreads();
    {
        // one thread per source reads its dirty flag (NVLink loads in the peer engine run in parallel)
        const bool flags = V.peer || !V.dist;  // control blocks of every source are mapped
        const int s = threadIdx.x;
        if (s < V.P_sources && (!flags || __ldcg(&V.ctl_all[s]->s[L % 3].dirty))) atomicOr(&s_src, 1ull << s);
    }
    __syncthreads();
    const unsigned long long src = s_src;
    // delegates were found: new-delegate work to balance, unless this lone
    // worker's level can have found only a few (every find took at least one
    // executed nd / dd inspection): then a static sweep without claims
    const LevelSlot &SW = V.ctl->s[L % 3];
    const bool few = DBFS_F1_FEW && V.P_sources == 1 &&
                     __ldcg(&SW.work[KIND_ND]) + __ldcg(&SW.work[KIND_DD]) < (unsigned long long)V.nw_d;
    const bool dyn = src != 0 && !few;
    // remote masks: 32-word chunks, so every lane has a word and its sources'
    // loads are in flight together (8 per batch) -- NVLink latency, not bandwidth
    // (light levels -- nothing found -- sweep with a static stride: 32-word
    // chunks there, a quarter of the iterations of the balanced 8-word ones)
    const int cw = (!dyn || (V.peer && __popcll(src) > 1)) ? 32 : DBFS_CWD;
    const LevelSlot &SL = V.ctl->s[L % 3];
    // nothing found anywhere, no delegate frontier to clear, and this worker's
    // mask of level L-1 (cleared here for level L+1) is already zero: no-op
    if (src == 0 && SL.dfront == 0 && SL.prev_dirty == 0) return;
    uint32_t *cnt_nd = SL.exec_dir[KIND_ND] == PUSHC ? V.first[KIND_ND] : nullptr;
    uint32_t *cnt_dd = SL.exec_dir[KIND_DD] == PUSHC ? V.first[KIND_DD] : nullptr;
    for (WarpChunks ch(dyn ? &V.ctl->s[L % 3].sched[4] : nullptr, V.nw_d, cw, gw, TW); ch.valid(); ch.next()) {
        const int64_t base = ch.base();
        const int64_t wi = ch.word(V.nw_d);
        uint32_t nw = 0u;
        if (wi >= 0 && V.mask_mc[L & 1]) {
            // NVLS: the NVSwitch returns the OR of every rank's copy of the word
            uint32_t r;
            asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b32 %0, [%1];"
                         : "=r"(r)
                         : "l"(V.mask_mc[L & 1] + wi)
                         : "memory");
            uint32_t dv = V.dvis[wi];
            nw = r & ~dv;
            next_mask[wi] = 0u;
            V.dfront[wi] = nw;
            if (nw) {
                V.dvis[wi] = dv | nw;
                V.dseen[wi] = dv | nw;
            }
        } else if (wi >= 0) {
            uint32_t r = 0;
            for (int s0 = 0; s0 < V.P_sources; s0 += 8) {
                uint32_t t[8];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int s = s0 + j;
                    t[j] = (s < V.P_sources && ((src >> s) & 1)) ? __ldcg(&V.mask_src[L & 1][s][wi]) : 0u;
                }
#pragma unroll
                for (int j = 0; j < 8; j++) r |= t[j];
            }
            uint32_t dv = V.dvis[wi];
            nw = r & ~dv;
            next_mask[wi] = 0u;
            V.dfront[wi] = nw;
            if (nw) {
                V.dvis[wi] = dv | nw;
                V.dseen[wi] = dv | nw;  // + the other workers' finds (own claims are in it already)
            }
        }
        {
            uint32_t fold = nw;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) fold |= __shfl_xor_sync(FULL, fold, o);
            if (lane == 0 && fold) atomicOr(&V.coarse_d[(L + 1) & 1][(base >> 5) & (FW - 1)], fold);
        }
        unsigned cnt = warp_compact(nw, wi, list);
        if (!cnt) continue;
        // pass A: state + totals, NB delegates per lane at a time with every
        // load of the batch issued before any store (stores through the state
        // pointers would otherwise keep the compiler from overlapping them)
        unsigned long long cdn = 0, edn = 0, cdd = 0, edd = 0;
        for (unsigned g0 = 0; g0 < cnt; g0 += 32 * NB_DEL) {
            uint32_t x[NB_DEL], ldn[NB_DEL], ldd[NB_DEL];
            int64_t gx[NB_DEL];
            parent_t par[NB_DEL];
            bool ok[NB_DEL];
#pragma unroll
            for (int u = 0; u < NB_DEL; u++) {
                const unsigned i = g0 + u * 32 + lane;
                ok[u] = i < cnt;
                x[u] = ok[u] ? list[i] : 0u;
            }
#pragma unroll
            for (int u = 0; u < NB_DEL; u++) {
                ldn[u] = ok[u] ? __ldg(&V.deg[KIND_DN][x[u]]) : 0u;
                ldd[u] = ok[u] ? __ldg(&V.deg[KIND_DD][x[u]]) : 0u;
                gx[u] = (ok[u] && V.glevel) ? (int64_t)__ldg(&V.del_gid32[x[u]]) : 0;
                // a lone in-process worker's new delegates all come from its own mask
                par[u] = (ok[u] && V.parents && V.cand_all && V.P_sources == 1) ? V.dcand[x[u]] : 0;
            }
#pragma unroll
            for (int u = 0; u < NB_DEL; u++) {
                if (!ok[u]) continue;
                new_delegate(V, L, x[u], gx[u], par[u]);
                if (cnt_nd) take_first(cnt_nd, x[u], ldn[u], fc.skip[KIND_ND]);
                if (cnt_dd) take_first(cnt_dd, x[u], ldd[u], fc.skip[KIND_DD]);
                cdn += ldn[u] > 0;
                edn += ldn[u];
                cdd += ldd[u] > 0;
                edd += ldd[u];
                fc.new_del++;
            }
        }
        fc.dfv_dn += edn;
        fc.dq_dn += cdn;
        fc.dfv_dd += edd;
        fc.dq_dd += cdd;
        unsigned long long tdn = warp_sum(cdn), tedn = warp_sum(edn), tdd = warp_sum(cdd), tedd = warp_sum(edd);
        unsigned long long bdn = 0, bdd = 0;
        if (lane == 0) {
            if (tdn) bdn = atomicAdd(&N.dpack[0], (tdn << V.dshift) + tedn);
            if (tdd) bdd = atomicAdd(&N.dpack[1], (tdd << V.dshift) + tedd);
        }
        bdn = __shfl_sync(FULL, bdn, 0);
        bdd = __shfl_sync(FULL, bdd, 0);
        // pass B: list entries in batch order
        const unsigned long long EM = (1ull << V.dshift) - 1;
        unsigned long long pdn = bdn >> V.dshift, qdn = bdn & EM, pdd = bdd >> V.dshift, qdd = bdd & EM;
        uint32_t *ldn_list = V.dlist[0][(L + 1) & 1], *ldd_list = V.dlist[1][(L + 1) & 1];
        int64_t *ldn_pre = V.dpre[0][(L + 1) & 1], *ldd_pre = V.dpre[1][(L + 1) & 1];
        for (unsigned g0 = 0; g0 < cnt; g0 += 32) {
            unsigned i = g0 + lane;
            uint32_t x = i < cnt ? list[i] : 0u;
            uint64_t a = i < cnt ? (uint64_t)__ldg(&V.deg[KIND_DN][x]) : 0;
            uint64_t b = i < cnt ? (uint64_t)__ldg(&V.deg[KIND_DD][x]) : 0;
            unsigned t1, t2;
            unsigned long long e1, e2;
            unsigned p1 = warp_excl_scan(a > 0 ? 1u : 0u, &t1);
            unsigned long long s1 = warp_excl_scan64(a, &e1);
            unsigned p2 = warp_excl_scan(b > 0 ? 1u : 0u, &t2);
            unsigned long long s2 = warp_excl_scan64(b, &e2);
            if (a > 0) {
                ldn_list[pdn + p1] = x;
                ldn_pre[pdn + p1] = (int64_t)(qdn + s1);
            }
            if (b > 0) {
                ldd_list[pdd + p2] = x;
                ldd_pre[pdd + p2] = (int64_t)(qdd + s2);
            }
            pdn += t1;
            qdn += e1;
            pdd += t2;
            qdd += e2;
        }
        __syncwarp();
    }
}

// F2 (distributed only): ingest remote records (engine.py:147-157).
__device__ void finish_ingest(const View &V, int L, int64_t tid, int64_t nth) {
    const bool light = V.ctl->s[L % 3].light != 0;
    if (V.peer) {  // senders stored into fixed segments of this inbox over NVLink
        __shared__ unsigned long long s_cnt[MAXW];
        if (threadIdx.x < V.p) s_cnt[threadIdx.x] = __ldcg(&V.ctl_all[threadIdx.x]->s[L % 3].sent[V.w]);
        __syncthreads();
        unsigned long long uq = 0;
        for (int s = 0; s < V.p; s++) {
            if (s == V.w) continue;
            const unsigned long long cnt = s_cnt[s];
            const uint2 *seg = V.inbox[0] + V.seg_off[s];
            const int grp = V.local_all2all ? (s % V.p_rank) + V.p_rank * (V.w / V.p_rank) : s;
            for (int64_t i = tid; i < (int64_t)cnt; i += nth) {
                uint2 rec = __ldcg(&seg[i]);
                if (rec.x == REC_SKIP) continue;  // unused tail of a sender's chunk
                if (V.uniquify) {
                    uint32_t old = atomicOr(&V.uq[(int64_t)grp * V.nw_n + (rec.x >> 5)], 1u << (rec.x & 31));
                    if (!(old & (1u << (rec.x & 31)))) uq++;
                }
                claim_normal(V, L, rec.x, (parent_t)rec.y, light);
            }
        }
        uq = warp_sum(uq);
        if (lane_id() == 0 && uq) atomicAdd(&V.ctl->s[L % 3].uq_records, uq);
        return;
    }
    const unsigned long long nin = V.ctl->s[L % 3].inbox;
    const uint2 *inbox = V.inbox[L & 1];
    unsigned long long uq = 0;
    for (int64_t i = tid; i < (int64_t)nin; i += nth) {
        uint2 rec = inbox[i];
        if (V.uniquify) {  // records arrive grouped by source rank: recover it
            int s = 0;
            while (s + 1 < V.p && V.recv_off[s + 1] <= i) s++;
            int grp = V.local_all2all ? (s % V.p_rank) + V.p_rank * (V.w / V.p_rank) : s;
            uint32_t old = atomicOr(&V.uq[(int64_t)grp * V.nw_n + (rec.x >> 5)], 1u << (rec.x & 31));
            if (!(old & (1u << (rec.x & 31)))) uq++;
        }
        claim_normal(V, L, rec.x, (parent_t)rec.y, light);
    }
    uq = warp_sum(uq);
    if (lane_id() == 0 && uq) atomicAdd(&V.ctl->s[L % 3].uq_records, uq);
}

// Fold one 32-word chunk of the new normal frontier (chunk index ch, lane =
// word): visited |= next, the new vertices' levels and previsit statistics;
// clears the old frontier's words when clear_cur.  Returns true when the
// chunk holds new vertices.
__device__ __forceinline__ bool fold_chunk(const View &V, int L, int64_t ch, bool clear_cur, uint32_t *list,
                                           FinishCounters &fc, uint32_t *cnt_dn) {
    uint32_t *cur = V.nfront[L & 1];
    const uint32_t *nxt = V.nfront[(L + 1) & 1];
    const int64_t wi = ch * 32 + lane_id();
    uint32_t nw = 0u;
    if (wi < V.nw_n) {
        if (clear_cur && cur[wi]) cur[wi] = 0u;
        nw = nxt[wi];
        if (nw) {
            const uint32_t vis = V.nvis[wi] | nw;
            V.nvis[wi] = vis;
            V.nseen[wi] = vis;  // + the pulls' finds (pulls do not mark seen: a push claiming the
                                // same vertex again only repeats an idempotent mark)
        }
    }
    if (!__any_sync(FULL, nw != 0u)) return false;
    unsigned cnt = warp_compact(nw, wi < V.nw_n ? wi : 0, list);
    // NB_DEL new vertices per lane at a time: their row-length loads in flight together
    for (unsigned g0 = 0; g0 < cnt; g0 += 32 * NB_DEL) {
        uint32_t c[NB_DEL], dnd[NB_DEL];
#pragma unroll
        for (int u = 0; u < NB_DEL; u++) {
            const unsigned i = g0 + u * 32 + lane_id();
            c[u] = i < cnt ? list[i] : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < NB_DEL; u++) dnd[u] = c[u] != 0xffffffffu ? __ldg(&V.deg[KIND_ND][c[u]]) : 0u;
#pragma unroll
        for (int u = 0; u < NB_DEL; u++) {
            if (c[u] == 0xffffffffu) continue;
            V.nlevel[c[u]] = L + 1;  // every claim of level L+1 (push, pull, remote record) lands here
            if (cnt_dn) take_first(cnt_dn, c[u], (uint64_t)dnd[u], fc.skip[KIND_DN]);
            fc.nfv_nd += (unsigned long long)dnd[u];
            fc.nq_nd += dnd[u] > 0;
            fc.ncount++;
        }
    }
    __syncwarp();
    return true;
}

// F3: fold the new normal frontier into visited, clear the old one, and count
// the new frontier's previsit statistics (FV_nd, q_nd, |frontier|).  After a
// light level V(L) the new frontier's chunks are those listed by its claims;
// the old frontier's chunks come from its list (V(L-1) light) or its touch
// bits.  After a heavy level every word is swept and the touch bitmap of
// frontier L+1 is built from the fold.  Either way touch[(L+1)&1] marks
// exactly the non-empty chunks of frontier L+1 and touch[L&1] ends zero.
__device__ void finish_normals(const View &V, int L, int64_t gw, int64_t TW, uint32_t *list, FinishCounters &fc) {
    const unsigned lane = lane_id();
    const LevelSlot &A = V.ctl->s[L % 3];
    uint32_t *cnt_dn = A.exec_dir[KIND_DN] == PUSHC ? V.first[KIND_DN] : nullptr;
    uint32_t *t_old = V.ntouch[L & 1], *t_new = V.ntouch[(L + 1) & 1];
    const int64_t nch = (V.nw_n + 31) >> 5;
    if (A.light) {
        uint32_t *cur = V.nfront[L & 1];
        auto clear_old = [&](int64_t ch) {
            const int64_t wi = ch * 32 + lane;
            if (wi < V.nw_n && cur[wi]) cur[wi] = 0u;
            if (lane == 0) atomicAnd(&t_old[ch >> 5], ~(1u << (ch & 31)));
        };
        if (A.prev_light) {  // old frontier listed by the claims of V(L-1)
            const int64_t no = (int64_t)A.nchunks;
            for (int64_t i = gw; i < no; i += TW) clear_old(V.nchunk_list[L & 1][i]);
        } else {
            for (int64_t ch = gw; ch < nch; ch += TW)
                if ((__ldcg(&t_old[ch >> 5]) >> (ch & 31)) & 1u) clear_old(ch);
        }
        const int64_t nn = (int64_t)__ldcg(&V.ctl->s[(L + 1) % 3].nchunks);
        for (int64_t i = gw; i < nn; i += TW) fold_chunk(V, L, V.nchunk_list[(L + 1) & 1][i], false, list, fc, cnt_dn);
        return;
    }
    const int64_t tid = gw * 32 + lane, nth = TW * 32;
    for (int64_t i = tid; i < V.ntw; i += nth) t_old[i] = 0u;
    const bool dyn = V.f3_dyn && A.nfront + A.dfront > (unsigned long long)TW;  // heavy level: large next frontier likely
    for (WarpChunks ch(dyn ? &V.ctl->s[L % 3].sched[5] : nullptr, V.nw_n, DBFS_CWN, gw, TW); ch.valid(); ch.next()) {
        if (fold_chunk(V, L, ch.cur, true, list, fc, cnt_dn) && lane == 0)
            atomicOr(&t_new[ch.cur >> 5], 1u << (ch.cur & 31));
    }
    (void)nch;
}

__device__ void flush_finish(const View &V, int L, FinishCounters &fc, int wb, bool zero_slot) {
    Ctl &C = *V.ctl;
    LevelSlot &A = C.s[L % 3];
    LevelSlot &N = C.s[(L + 1) % 3];
    warp_acc(0, fc.nfv_nd);
    warp_acc(1, fc.nq_nd);
    warp_acc(2, fc.ncount);
    warp_acc(3, fc.dfv_dn);
    warp_acc(4, fc.dq_dn);
    warp_acc(5, fc.dfv_dd);
    warp_acc(6, fc.dq_dd);
    warp_acc(7, fc.new_del);
    for (int k = 1; k < 4; k++) warp_acc(8 + k, fc.skip[k]);
    __syncthreads();
    {
        unsigned long long *dst[9] = {&N.fv[KIND_ND], &N.q[KIND_ND], &N.nfront, &N.fv[KIND_DN], &N.q[KIND_DN],
                                      &N.fv[KIND_DD], &N.q[KIND_DD], &N.dfront, &A.new_del};
        if (threadIdx.x == 8) block_acc()[8] = block_acc()[7];  // new delegates: next frontier and this level
        block_acc_flush(dst, 9);
        const int k = (int)threadIdx.x - 8;  // counting pushes: V(L) added the full row lengths
        if (k >= 1 && k < 4 && block_acc()[8 + k]) atomicAdd(&A.insp_bwd[k], 0ull - block_acc()[8 + k]);
    }
    if (zero_slot && wb == 0) {
        // slot (L+2)%3 is idle during level L: clear it for level L+2
        unsigned long long *z = (unsigned long long *)&C.s[(L + 2) % 3];
        for (size_t i = threadIdx.x; i < sizeof(LevelSlot) / 8; i += BT) z[i] = 0ull;
    }
}

enum { F_DELEGATES = 1, F_INGEST = 2, F_NORMALS = 4 };

__device__ void phase_finish(const View &V, int L, int wb, int nb, Smem &sm, int parts) {
    FinishCounters fc = {};
    block_acc_clear();
    __syncthreads();
    const int64_t gw = (int64_t)wb * WPB + warp_id(), TW = (int64_t)nb * WPB;
    const int64_t tid = (int64_t)wb * BT + threadIdx.x, nth = (int64_t)nb * BT;
    uint32_t *list = sm.list[warp_id()];
    TaskTimer tt;
    if (parts & F_DELEGATES) {
        for (int64_t i = tid; i < FW; i += nth) V.coarse_d[L & 1][i] = 0u;
        tt.start();
        finish_delegates(V, L, gw, TW, list, fc);
        tt.stop(V.ctl->s[L % 3], 6);
    }
    if (parts & F_INGEST) finish_ingest(V, L, tid, nth);
    if ((parts & F_NORMALS) && V.uniquify)
        for (int64_t i = tid; i < (int64_t)V.p * V.nw_n; i += nth) V.uq[i] = 0u;
    if (parts & F_NORMALS) {
        tt.start();
        finish_normals(V, L, gw, TW, list, fc);
        tt.stop(V.ctl->s[L % 3], 7);
    }
    flush_finish(V, L, fc, wb, (parts & F_DELEGATES) != 0);
}

// ------------------------------------------------------------ init / seed

__device__ void phase_init(const View &V, int wb, int nb) {
    const int64_t tid = (int64_t)wb * BT + threadIdx.x, nth = (int64_t)nb * BT;
    for (int64_t i = tid; i < V.n_local; i += nth) {
        V.nlevel[i] = -1;
        if (V.parents) V.nparent[i] = -1;
    }
    for (int64_t i = tid; i < V.d; i += nth) V.dlevel[i] = -1;
    for (int64_t i = tid; i < V.nw_n; i += nth) {
        V.nvis[i] = 0u;
        V.nseen[i] = 0u;
        V.nfront[0][i] = 0u;
        V.nfront[1][i] = 0u;
    }
    for (int64_t i = tid; i < FW; i += nth) {
        V.coarse_d[0][i] = 0u;
        V.coarse_d[1][i] = 0u;
        V.coarse_n[0][i] = 0u;
        V.coarse_n[1][i] = 0u;
    }
    if (V.sent)
        for (int64_t i = tid; i < V.nw_g; i += nth) V.sent[i] = 0u;
    for (int64_t i = tid; i < 2 * V.ntw; i += nth) V.ntouch[0][i] = 0u;  // both parities (contiguous)
    for (int64_t i = tid; i < V.nw_d; i += nth) {
        V.dvis[i] = 0u;
        V.dseen[i] = 0u;
        V.dfront[i] = 0u;
        V.dnext[0][i] = 0u;
        V.dnext[1][i] = 0u;
    }
}

// engine.py:131-139: the source is a delegate (replicated) or a normal owned
// by source mod p.  del_id = delegate id of the source or 0xffffffff.
__device__ void seed_worker(const View &V, int64_t source, uint32_t del_id) {
    LevelSlot &S = V.ctl->s[0];
    if (del_id != 0xffffffffu) {
        uint32_t x = del_id;
        V.dlevel[x] = 0;
        V.dvis[x >> 5] |= 1u << (x & 31);
        V.dseen[x >> 5] |= 1u << (x & 31);
        V.dfront[x >> 5] |= 1u << (x & 31);
        V.coarse_d[0][(x >> 10) & (FW - 1)] |= 1u << (x & 31);
        if (V.parents) V.dparent[x] = (parent_t)source;
        if (V.glevel) {
            V.glevel[source] = 0;
            if (V.parents) V.gparent[source] = (parent_t)source;
        }
        int64_t ddn = V.off[KIND_DN][x + 1] - V.off[KIND_DN][x];
        int64_t ddd = V.off[KIND_DD][x + 1] - V.off[KIND_DD][x];
        S.fv[KIND_DN] = ddn;
        S.q[KIND_DN] = ddn > 0;
        S.fv[KIND_DD] = ddd;
        S.q[KIND_DD] = ddd > 0;
        S.dfront = 1;
        if (ddn > 0) {
            V.dlist[0][0][0] = x;
            V.dpre[0][0][0] = 0;
            S.dpack[0] = (1ull << V.dshift) | (unsigned long long)ddn;
        }
        if (ddd > 0) {
            V.dlist[1][0][0] = x;
            V.dpre[1][0][0] = 0;
            S.dpack[1] = (1ull << V.dshift) | (unsigned long long)ddd;
        }
    } else if ((int)(source % V.p) == V.w) {
        uint32_t c = (uint32_t)(source / V.p);
        V.nlevel[c] = 0;
        if (V.parents) V.nparent[c] = (parent_t)source;
        V.nfront[0][c >> 5] |= 1u << (c & 31);
        V.nvis[c >> 5] |= 1u << (c & 31);
        V.nseen[c >> 5] |= 1u << (c & 31);
        V.ntouch[0][(c >> 10) >> 5] |= 1u << ((c >> 10) & 31);
        V.nchunk_list[0][0] = c >> 10;
        S.nchunks = 1;
        int64_t dnd = V.off[KIND_ND][c + 1] - V.off[KIND_ND][c];
        S.fv[KIND_ND] = dnd;
        S.q[KIND_ND] = dnd > 0;
        S.nfront = 1;
    }
}

// Continue after level L?  engine.py:303-306: new local normals, new
// delegates, or any record in flight (over all in-process workers).
__device__ __forceinline__ bool level_continue(const View &V, int L) {
    if (V.ctl->s[L % 3].new_del) return true;
    // a peer GPU's block in the peer engine: the loads of 8 sources are in flight together
    unsigned long long any = 0;
    for (int i0 = 0; i0 < V.P_sources; i0 += 8) {
        unsigned long long t[16];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int i = i0 + j;
            const Ctl *c = V.ctl_all[i < V.P_sources ? i : 0];
            t[2 * j] = i < V.P_sources ? __ldcg(&c->s[(L + 1) % 3].nfront) : 0ull;
            t[2 * j + 1] = i < V.P_sources ? __ldcg(&c->s[L % 3].records) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 16; j++) any |= t[j];
    }
    return any != 0;
}

}  // namespace dbfs
