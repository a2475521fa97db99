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
//   visited(<= L) normal  = nvis | nfront[L&1]   (claims go to nfront[(L+1)&1])
//   visited(<= L) delegate= dvis                 (finds go to dnext[L&1])
#pragma once
#include "internal.h"

namespace dbfs {

constexpr int BT = 256;        // threads per block
constexpr int WPB = BT / 32;   // warps per block
constexpr int LIST = 1024;     // per-warp compaction buffer (32 words x 32 bits)

struct Smem {
    uint32_t list[WPB][LIST];
};

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

// Per-iteration record of level L (engine.py:291-302, one worker).
__host__ __device__ inline void make_record(const View &V, const Ctl &c, int L, IterRec &r) {
    const LevelSlot &S = c.s[L % 3];
    unsigned long long cum[4];
    int dirs[4];
    double bv[4];
    // directions were published at V(L); recompute bv from the same inputs
    level_dirs(V, c, L, dirs, bv, cum);
    for (int k = 0; k < 4; k++) {
        r.dir[k] = k == KIND_NN ? FWD : c.dir[L & 1][k];
        r.bv[k] = bv[k];
        r.fv[k] = S.fv[k];
        r.insp[k] = r.dir[k] == FWD ? S.fv[k] : S.insp_bwd[k];
    }
    r.records = S.records;
    r.rows = S.pull_rows;
    for (int k = 0; k < 4; k++)
        if (k == KIND_NN || r.dir[k] == FWD) r.rows += S.q[k];
    r.dirty = S.dirty;
    r.new_del = S.new_del;
    unsigned long long msgs = 0;
    for (int o = 0; o < MAXW; o++) {
        r.send[o] = S.send[o];
        msgs += S.send[o] > 0;
    }
    r.messages = msgs;
}

// ------------------------------------------------------------------ helpers

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

struct VisitCounters {
    unsigned long long fv_nn;       // FV_nn of this level's frontier (activity slot)
    unsigned long long nfv_nd, nq_nd, ncount;  // next frontier (normals)
    unsigned long long local_claims, records;
    unsigned long long insp_bwd[4];
    unsigned long long dirty;
    unsigned long long pull_rows;
};

struct FinishCounters {
    unsigned long long nfv_nd, nq_nd, ncount;
    unsigned long long dfv_dn, dq_dn, dfv_dd, dq_dd, dcount, new_del;
};

// Claim local normal c for level L+1 (pre-state unvisited already checked or
// checked here).  The atomicOr winner is the unique discoverer.
__device__ __forceinline__ void claim_normal(const View &V, int L, uint32_t c, int64_t parent, bool check,
                                             VisitCounters &vc) {
    const uint32_t wd = c >> 5, bit = 1u << (c & 31);
    if (check) {
        if ((V.nvis[wd] | V.nfront[L & 1][wd]) & bit) return;
    }
    uint32_t *nx = V.nfront[(L + 1) & 1];
    if (nx[wd] & bit) return;
    uint32_t old = atomicOr(&nx[wd], bit);
    if (old & bit) return;
    V.nlevel[c] = L + 1;
    if (V.parents) V.nparent[c] = parent;
    int64_t dnd = V.off[KIND_ND][c + 1] - V.off[KIND_ND][c];
    vc.local_claims++;
    vc.ncount++;
    vc.nfv_nd += dnd;
    vc.nq_nd += dnd > 0;
}

// Mark delegate x found at level L by this worker (delegate mask, comm.py:33-36).
__device__ __forceinline__ void find_delegate(const View &V, int L, uint32_t x, int64_t parent,
                                              unsigned long long &dirty) {
    const uint32_t wd = x >> 5, bit = 1u << (x & 31);
    uint32_t *dn = V.dnext[L & 1];
    if (dn[wd] & bit) return;
    uint32_t old = atomicOr(&dn[wd], bit);
    if (old & bit) return;
    if (V.parents) V.dcand[x] = parent;
    dirty = 1;
}

__device__ __forceinline__ void send_record(const View &V, int L, uint32_t owner, uint32_t local, int64_t parent,
                                            VisitCounters &vc) {
    vc.records++;
    uint2 rec = make_uint2(local, (uint32_t)parent);
    if (V.dist) {
        unsigned long long pos = atomicAdd(&V.ctl->s[L % 3].send[owner], 1ull);
        V.sendbin[owner][pos] = rec;
    } else {
        atomicAdd(&V.ctl->s[L % 3].send[owner], 1ull);
        unsigned long long pos = atomicAdd(&V.ctl_all[owner]->s[L % 3].inbox, 1ull);
        V.inbox_all[L & 1][owner][pos] = rec;
    }
}

// -------------------------------------------------------------- phase V(L)

__device__ void phase_visit(const View &V, int L, int wb, int nb, Smem &sm) {
    Ctl &C = *V.ctl;
    const LevelSlot &S = C.s[L % 3];
    int dirs[4];
    double bv[4];
    unsigned long long cum[4];
    level_dirs(V, C, L, dirs, bv, cum);
    if (wb == 0 && threadIdx.x == 0) {
        for (int k = 0; k < 4; k++) {
            C.dir[L & 1][k] = dirs[k];
            C.cumq[L & 1][k] = cum[k];
        }
    }
    VisitCounters vc = {};
    const unsigned lane = lane_id(), warp = warp_id();
    const int64_t gw = (int64_t)wb * WPB + warp, TW = (int64_t)nb * WPB;
    uint32_t *list = sm.list[warp];
    const int p = V.p, w = V.w;
    const uint32_t *nfront_cur = V.nfront[L & 1];
    const int64_t *off_nn = V.off[KIND_NN], *off_nd = V.off[KIND_ND], *off_dn = V.off[KIND_DN],
                  *off_dd = V.off[KIND_DD];
    const uint32_t *col_nn = V.col[KIND_NN], *col_nd = V.col[KIND_ND], *col_dn = V.col[KIND_DN],
                   *col_dd = V.col[KIND_DD];

    // T1: normal frontier -- nn push (always, engine.py:207-222) + nd push.
    if (S.nfront > 0) {
        const bool nd_fwd = dirs[KIND_ND] == FWD;
        for (int64_t base = gw * 32; base < V.nw_n; base += TW * 32) {
            int64_t wi = base + lane;
            uint32_t word = wi < V.nw_n ? nfront_cur[wi] : 0u;
            unsigned cnt = warp_compact(word, base + lane, list);
            // warp_compact uses each lane's own wi; ids are absolute
            for (unsigned i = lane; i < cnt; i += 32) {
                uint32_t u = list[i];
                int64_t gid_u = (int64_t)u * p + w;
                int64_t b = __ldg(&off_nn[u]), e = __ldg(&off_nn[u + 1]);
                vc.fv_nn += e - b;
                for (int64_t j = b; j < e; j++) {
                    uint32_t g = __ldg(&col_nn[j]);
                    if (p == 1) {
                        claim_normal(V, L, g, gid_u, true, vc);
                    } else {
                        uint32_t o = V.pd.mod(g), c = V.pd.div(g);
                        if ((int)o == w) claim_normal(V, L, c, gid_u, true, vc);
                        else send_record(V, L, o, c, gid_u, vc);
                    }
                }
                if (nd_fwd) {
                    int64_t b2 = __ldg(&off_nd[u]), e2 = __ldg(&off_nd[u + 1]);
                    for (int64_t j = b2; j < e2; j++) {
                        uint32_t x = __ldg(&col_nd[j]);
                        if (!tbit(V.dvis, x)) find_delegate(V, L, x, gid_u, vc.dirty);
                    }
                }
            }
            __syncwarp();
        }
    }

    // T2: delegate frontier, non-hub rows -- dn / dd push (engine.py:238-263).
    const bool dn_fwd = dirs[KIND_DN] == FWD, dd_fwd = dirs[KIND_DD] == FWD;
    if (S.dfront > 0 && (dn_fwd || dd_fwd)) {
        for (int64_t base = gw * 32; base < V.nw_d; base += TW * 32) {
            int64_t wi = base + lane;
            uint32_t word = wi < V.nw_d ? V.dfront[wi] : 0u;
            unsigned cnt = warp_compact(word, wi, list);
            for (unsigned i = 0; i < cnt; i++) {
                uint32_t x = list[i];
                int64_t gx = __ldg(&V.del_gid[x]);
                if (dn_fwd) {
                    int64_t b = __ldg(&off_dn[x]), e = __ldg(&off_dn[x + 1]);
                    if (e - b <= V.hub)
                        for (int64_t j = b + lane; j < e; j += 32) claim_normal(V, L, __ldg(&col_dn[j]), gx, true, vc);
                }
                if (dd_fwd) {
                    int64_t b = __ldg(&off_dd[x]), e = __ldg(&off_dd[x + 1]);
                    if (e - b <= V.hub)
                        for (int64_t j = b + lane; j < e; j += 32) {
                            uint32_t y = __ldg(&col_dd[j]);
                            if (!tbit(V.dvis, y)) find_delegate(V, L, y, gx, vc.dirty);
                        }
                }
            }
            __syncwarp();
        }
    }

    // T3: hub rows of the delegate frontier, split into fixed-size chunks.
    if (S.chunks > 0 && (dn_fwd || dd_fwd)) {
        const uint64_t *ch = V.chunks[L & 1];
        const int64_t nch = (int64_t)S.chunks < V.chunk_cap ? (int64_t)S.chunks : V.chunk_cap;
        for (int64_t ci = gw; ci < nch; ci += TW) {
            uint64_t ent = ch[ci];
            uint32_t x = (uint32_t)(ent >> 32);
            int kind = (ent & 1) ? KIND_DD : KIND_DN;
            if ((kind == KIND_DN && !dn_fwd) || (kind == KIND_DD && !dd_fwd)) continue;
            int64_t idx = (int64_t)((ent >> 1) & 0x7fffffffu);
            const int64_t *off = V.off[kind];
            int64_t b0 = __ldg(&off[x]), e0 = __ldg(&off[x + 1]);
            int64_t b = b0 + idx * V.chunk, e = b + V.chunk < e0 ? b + V.chunk : e0;
            int64_t gx = __ldg(&V.del_gid[x]);
            if (kind == KIND_DN) {
                for (int64_t j = b + lane; j < e; j += 32) claim_normal(V, L, __ldg(&col_dn[j]), gx, true, vc);
            } else {
                for (int64_t j = b + lane; j < e; j += 32) {
                    uint32_t y = __ldg(&col_dd[j]);
                    if (!tbit(V.dvis, y)) find_delegate(V, L, y, gx, vc.dirty);
                }
            }
        }
    }

    // T4: dn pull -- unvisited nd-source normals scan nd rows for frontier
    // delegates (engine.py:242-248, traversal.py:111-139).
    if (dirs[KIND_DN] == BWD) {
        const uint32_t *srcb = V.src_bits[KIND_ND];
        for (int64_t base = gw * 32; base < V.nw_n; base += TW * 32) {
            int64_t wi = base + lane;
            uint32_t word = wi < V.nw_n ? (srcb[wi] & ~(V.nvis[wi] | nfront_cur[wi])) : 0u;
            unsigned cnt = warp_compact(word, wi, list);
            if (lane == 0) vc.pull_rows += cnt;
            for (unsigned i = lane; i < cnt; i += 32) {
                uint32_t c = list[i];
                int64_t b = __ldg(&off_nd[c]), e = __ldg(&off_nd[c + 1]);
                int64_t j = b;
                uint32_t x = 0;
                for (; j < e; j++) {
                    x = __ldg(&col_nd[j]);
                    if (tbit(V.dfront, x)) break;
                }
                if (j < e) {
                    vc.insp_bwd[KIND_DN] += j - b + 1;
                    claim_normal(V, L, c, __ldg(&V.del_gid[x]), false, vc);
                } else {
                    vc.insp_bwd[KIND_DN] += e - b;
                }
            }
            __syncwarp();
        }
    }

    // T5: nd pull -- unvisited dn-source delegates scan dn rows for frontier
    // normals (engine.py:229-233).
    if (dirs[KIND_ND] == BWD) {
        const uint32_t *srcb = V.src_bits[KIND_DN];
        for (int64_t base = gw * 32; base < V.nw_d; base += TW * 32) {
            int64_t wi = base + lane;
            uint32_t word = wi < V.nw_d ? (srcb[wi] & ~V.dvis[wi]) : 0u;
            unsigned cnt = warp_compact(word, wi, list);
            if (lane == 0) vc.pull_rows += cnt;
            for (unsigned i = lane; i < cnt; i += 32) {
                uint32_t x = list[i];
                int64_t b = __ldg(&off_dn[x]), e = __ldg(&off_dn[x + 1]);
                int64_t j = b;
                uint32_t c = 0;
                for (; j < e; j++) {
                    c = __ldg(&col_dn[j]);
                    if (tbit(nfront_cur, c)) break;
                }
                if (j < e) {
                    vc.insp_bwd[KIND_ND] += j - b + 1;
                    find_delegate(V, L, x, (int64_t)c * p + w, vc.dirty);
                } else {
                    vc.insp_bwd[KIND_ND] += e - b;
                }
            }
            __syncwarp();
        }
    }

    // T6: dd pull -- unvisited dd-source delegates scan dd rows (engine.py:257-261).
    if (dirs[KIND_DD] == BWD) {
        const uint32_t *srcb = V.src_bits[KIND_DD];
        for (int64_t base = gw * 32; base < V.nw_d; base += TW * 32) {
            int64_t wi = base + lane;
            uint32_t word = wi < V.nw_d ? (srcb[wi] & ~V.dvis[wi]) : 0u;
            unsigned cnt = warp_compact(word, wi, list);
            if (lane == 0) vc.pull_rows += cnt;
            for (unsigned i = lane; i < cnt; i += 32) {
                uint32_t x = list[i];
                int64_t b = __ldg(&off_dd[x]), e = __ldg(&off_dd[x + 1]);
                int64_t j = b;
                uint32_t y = 0;
                for (; j < e; j++) {
                    y = __ldg(&col_dd[j]);
                    if (tbit(V.dfront, y)) break;
                }
                if (j < e) {
                    vc.insp_bwd[KIND_DD] += j - b + 1;
                    find_delegate(V, L, x, __ldg(&V.del_gid[y]), vc.dirty);
                } else {
                    vc.insp_bwd[KIND_DD] += e - b;
                }
            }
            __syncwarp();
        }
    }

    // flush: one atomic per warp per counter
    LevelSlot &A = C.s[L % 3];
    LevelSlot &N = C.s[(L + 1) % 3];
    unsigned long long v;
    v = warp_sum(vc.fv_nn);
    if (lane == 0) atomic_add_u64(&A.fv[KIND_NN], v);
    v = warp_sum(vc.nfv_nd);
    if (lane == 0) atomic_add_u64(&N.fv[KIND_ND], v);
    v = warp_sum(vc.nq_nd);
    if (lane == 0) atomic_add_u64(&N.q[KIND_ND], v);
    v = warp_sum(vc.ncount);
    if (lane == 0) atomic_add_u64(&N.nfront, v);
    v = warp_sum(vc.local_claims);
    if (lane == 0) atomic_add_u64(&A.local_claims, v);
    v = warp_sum(vc.records);
    if (lane == 0) atomic_add_u64(&A.records, v);
    for (int k = 1; k < 4; k++) {
        v = warp_sum(vc.insp_bwd[k]);
        if (lane == 0) atomic_add_u64(&A.insp_bwd[k], v);
    }
    v = warp_sum(vc.dirty);
    if (lane == 0 && v) atomicOr(&A.dirty, 1ull);
    v = warp_sum(vc.pull_rows);
    if (lane == 0) atomic_add_u64(&A.pull_rows, v);
}

// -------------------------------------------------------------- phase F(L)

__device__ __forceinline__ void append_chunks(const View &V, int L, uint32_t x, int kind, int64_t deg) {
    int64_t nch = (deg + V.chunk - 1) / V.chunk;
    unsigned long long pos = atomicAdd(&V.ctl->s[(L + 1) % 3].chunks, (unsigned long long)nch);
    uint64_t *ch = V.chunks[(L + 1) & 1];
    for (int64_t i = 0; i < nch && (int64_t)pos + i < V.chunk_cap; i++)
        ch[pos + i] = ((uint64_t)x << 32) | ((uint64_t)i << 1) | (kind == KIND_DD ? 1ull : 0ull);
}

__device__ void phase_finish(const View &V, int L, int wb, int nb) {
    Ctl &C = *V.ctl;
    LevelSlot &A = C.s[L % 3];
    LevelSlot &N = C.s[(L + 1) % 3];
    FinishCounters fc = {};
    VisitCounters vc = {};
    const int64_t tid = (int64_t)wb * BT + threadIdx.x, nth = (int64_t)nb * BT;
    const uint32_t *own_mask = V.dnext[L & 1];
    uint32_t *next_mask = V.dnext[(L + 1) & 1];

    // F1: delegate mask OR-reduction (comm.py:75-98) -> new delegates at L+1
    for (int64_t wi = tid; wi < V.nw_d; wi += nth) {
        uint32_t r = 0;
        for (int s = 0; s < V.P_sources; s++) r |= V.mask_src[L & 1][s][wi];
        uint32_t nw = r & ~V.dvis[wi];
        next_mask[wi] = 0u;
        V.dfront[wi] = nw;
        if (!nw) continue;
        V.dvis[wi] |= nw;
        uint32_t own = own_mask[wi];
        while (nw) {
            int b = __ffs(nw) - 1;
            nw &= nw - 1;
            uint32_t x = (uint32_t)(wi << 5) + b;
            V.dlevel[x] = L + 1;
            int64_t par = 0x7fffffffffffffffLL;
            if (V.parents) {
                if (V.cand_all) {
                    for (int s = 0; s < V.P_sources; s++)
                        if ((V.mask_src[L & 1][s][wi] >> b) & 1u) {
                            int64_t c = V.cand_src[s][x];
                            par = c < par ? c : par;
                        }
                } else if ((own >> b) & 1u) {
                    par = V.dcand[x];
                }
                V.dparent[x] = par;
            }
            if (V.glevel) {
                int64_t gx = V.del_gid[x];
                V.glevel[gx] = L + 1;
                if (V.parents) V.gparent[gx] = par;
            }
            int64_t ddn = V.off[KIND_DN][x + 1] - V.off[KIND_DN][x];
            int64_t ddd = V.off[KIND_DD][x + 1] - V.off[KIND_DD][x];
            fc.dfv_dn += ddn;
            fc.dq_dn += ddn > 0;
            fc.dfv_dd += ddd;
            fc.dq_dd += ddd > 0;
            fc.dcount++;
            fc.new_del++;
            if (ddn > V.hub) append_chunks(V, L, x, KIND_DN, ddn);
            if (ddd > V.hub) append_chunks(V, L, x, KIND_DD, ddd);
        }
    }

    // F2: ingest remote records (engine.py:147-157): first claim wins.
    const unsigned long long nin = A.inbox;
    const uint2 *inbox = V.inbox[L & 1];
    for (int64_t i = tid; i < (int64_t)nin; i += nth) {
        uint2 rec = inbox[i];
        int32_t lv = V.nlevel[rec.x];
        if ((uint32_t)lv <= (uint32_t)L) continue;  // visited at <= L
        claim_normal(V, L, rec.x, (int64_t)rec.y, false, vc);
    }

    // F3: fold this level's frontier into visited and clear it for reuse.
    uint32_t *cur = V.nfront[L & 1];
    for (int64_t wi = tid; wi < V.nw_n; wi += nth) {
        uint32_t x = cur[wi];
        if (x) {
            V.nvis[wi] |= x;
            cur[wi] = 0u;
        }
    }

    const unsigned lane = lane_id();
    unsigned long long v;
    v = warp_sum(vc.nfv_nd + fc.nfv_nd);
    if (lane == 0) atomic_add_u64(&N.fv[KIND_ND], v);
    v = warp_sum(vc.nq_nd + fc.nq_nd);
    if (lane == 0) atomic_add_u64(&N.q[KIND_ND], v);
    v = warp_sum(vc.ncount + fc.ncount);
    if (lane == 0) atomic_add_u64(&N.nfront, v);
    v = warp_sum(fc.dfv_dn);
    if (lane == 0) atomic_add_u64(&N.fv[KIND_DN], v);
    v = warp_sum(fc.dq_dn);
    if (lane == 0) atomic_add_u64(&N.q[KIND_DN], v);
    v = warp_sum(fc.dfv_dd);
    if (lane == 0) atomic_add_u64(&N.fv[KIND_DD], v);
    v = warp_sum(fc.dq_dd);
    if (lane == 0) atomic_add_u64(&N.q[KIND_DD], v);
    v = warp_sum(fc.dcount);
    if (lane == 0) atomic_add_u64(&N.dfront, v);
    v = warp_sum(fc.new_del);
    if (lane == 0) atomic_add_u64(&A.new_del, v);
    if (wb == 0 && threadIdx.x == 0) {
        // slot (L+2)%3 is idle during level L: clear it for level L+2
        LevelSlot &Z = C.s[(L + 2) % 3];
        unsigned long long *z = (unsigned long long *)&Z;
        for (size_t i = 0; i < sizeof(LevelSlot) / 8; i++) z[i] = 0ull;
    }
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
        V.nfront[0][i] = 0u;
        V.nfront[1][i] = 0u;
    }
    for (int64_t i = tid; i < V.nw_d; i += nth) {
        V.dvis[i] = 0u;
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
        V.dfront[x >> 5] |= 1u << (x & 31);
        if (V.parents) V.dparent[x] = source;
        if (V.glevel) {
            V.glevel[source] = 0;
            if (V.parents) V.gparent[source] = source;
        }
        int64_t ddn = V.off[KIND_DN][x + 1] - V.off[KIND_DN][x];
        int64_t ddd = V.off[KIND_DD][x + 1] - V.off[KIND_DD][x];
        S.fv[KIND_DN] = ddn;
        S.q[KIND_DN] = ddn > 0;
        S.fv[KIND_DD] = ddd;
        S.q[KIND_DD] = ddd > 0;
        S.dfront = 1;
        if (ddn > V.hub) append_chunks(V, -1, x, KIND_DN, ddn);
        if (ddd > V.hub) append_chunks(V, -1, x, KIND_DD, ddd);
    } else if ((int)(source % V.p) == V.w) {
        uint32_t c = (uint32_t)(source / V.p);
        V.nlevel[c] = 0;
        if (V.parents) V.nparent[c] = source;
        V.nfront[0][c >> 5] |= 1u << (c & 31);
        int64_t dnd = V.off[KIND_ND][c + 1] - V.off[KIND_ND][c];
        S.fv[KIND_ND] = dnd;
        S.q[KIND_ND] = dnd > 0;
        S.nfront = 1;
    }
}

// Continue after level L?  engine.py:303-306: local news, new delegates, or
// any record in flight (over all in-process workers).
__device__ __forceinline__ bool level_continue(const View *views, int W, int L) {
    const LevelSlot &A0 = views[0].ctl->s[L % 3];
    if (A0.new_del) return true;
    for (int i = 0; i < W; i++) {
        const LevelSlot &A = views[i].ctl->s[L % 3];
        if (A.local_claims || A.records) return true;
    }
    return false;
}

}  // namespace dbfs
