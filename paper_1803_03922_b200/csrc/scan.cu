// scan.cu -- device-wide exclusive scan and a stable LSD radix sort (key/value
// uint32 pairs).  Used by the graph build to reproduce the reference's stable
// (worker, kind, row) ordering (partition.py:132-137, 295-301).
#include <algorithm>

#include "internal.h"

namespace dbfs {

static constexpr int SCAN_THREADS = 256;
static constexpr int SCAN_ITEMS = 16;
static constexpr int64_t SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__global__ void k_tile_sums(const T *__restrict__ in, int64_t n, int64_t *__restrict__ sums) {
    __shared__ int64_t red[SCAN_THREADS / 32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int64_t s = 0;
#pragma unroll 4
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t idx = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
        if (idx < n) s += (int64_t)in[idx];
    }
    s = warp_sum(s);
    if (lane_id() == 0) red[warp_id()] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int i = 0; i < SCAN_THREADS / 32; i++) t += red[i];
        sums[blockIdx.x] = t;
    }
}

// Exclusive scan of one tile with a carried-in offset; thread t owns items
// [t*ITEMS, (t+1)*ITEMS) so the scan is item-contiguous.
template <typename T>
__global__ void k_tile_scan(const T *__restrict__ in, int64_t n, const int64_t *__restrict__ tile_off,
                            int64_t *__restrict__ out) {
    __shared__ int64_t wsum[SCAN_THREADS / 32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t idx = base + i;
        v[i] = idx < n ? (int64_t)in[idx] : 0;
        s += v[i];
    }
    // block exclusive scan of s
    int64_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane_id() >= (unsigned)o) x += y;
    }
    if (lane_id() == 31) wsum[warp_id()] = x;
    __syncthreads();
    int64_t woff = 0;
    for (unsigned i = 0; i < warp_id(); i++) woff += wsum[i];
    int64_t run = tile_off[blockIdx.x] + woff + x - s;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t idx = base + i;
        if (idx < n) out[idx] = run;
        run += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1) out[n] = run;
}

__global__ void k_single_scan_i64(int64_t *a, int64_t n) {
    // tiny fallback for <= SCAN_TILE elements: sequential in one thread block
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t run = 0;
        for (int64_t i = 0; i < n; i++) {
            int64_t t = a[i];
            a[i] = run;
            run += t;
        }
    }
}

// out[0..n] = exclusive scan of in[0..n), out[n] = total.
template <typename T>
static void exclusive_scan_impl(Ctx &ctx, const T *in, int64_t *out, int64_t n) {
    if (n == 0) {
        DBFS_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), ctx.stream));
        return;
    }
    int64_t tiles = ceil_div(n, SCAN_TILE);
    DArray<int64_t> sums;
    sums.alloc(tiles + 1);
    k_tile_sums<T><<<(unsigned)tiles, SCAN_THREADS, 0, ctx.stream>>>(in, n, sums.p);
    DBFS_LAUNCHED();
    if (tiles <= 64) {
        k_single_scan_i64<<<1, 32, 0, ctx.stream>>>(sums.p, tiles);
        DBFS_LAUNCHED();
    } else {
        DArray<int64_t> sums2;
        sums2.alloc(tiles + 1);
        exclusive_scan_impl<int64_t>(ctx, sums.p, sums2.p, tiles);
        DBFS_CUDA(cudaMemcpyAsync(sums.p, sums2.p, sizeof(int64_t) * tiles, cudaMemcpyDeviceToDevice,
                                  ctx.stream));
        DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    k_tile_scan<T><<<(unsigned)tiles, SCAN_THREADS, 0, ctx.stream>>>(in, n, sums.p, out);
    DBFS_LAUNCHED();
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

void exclusive_scan_u32_to_i64(Ctx &ctx, const uint32_t *in, int64_t *out, int64_t n) {
    exclusive_scan_impl<uint32_t>(ctx, in, out, n);
}

// ---------------------------------------------------------------- radix sort

static constexpr int RS_THREADS = 256;
static constexpr int RS_ITEMS = 16;
static constexpr int64_t RS_TILE = RS_THREADS * RS_ITEMS;
static constexpr int RS_WARPS = RS_THREADS / 32;

__global__ void k_rs_hist(const uint32_t *__restrict__ keys, int64_t n, int shift, int rbits,
                          int64_t tiles, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    int radix = 1 << rbits;
    for (int i = threadIdx.x; i < radix; i += RS_THREADS) h[i] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
    uint32_t mask = radix - 1;
#pragma unroll 4
    for (int i = 0; i < RS_ITEMS; i++) {
        int64_t idx = base + (int64_t)i * RS_THREADS + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & mask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < radix; i += RS_THREADS) hist[(int64_t)i * tiles + blockIdx.x] = h[i];
}

// Stable scatter: the tile's elements are ranked in index order, 256 at a time
// (thread t of round r holds element r*256+t).  Within a warp, __match_any_sync
// groups equal digits; across warps a per-digit prefix over warp counts keeps
// warp order, and the running per-digit offset carries the order across rounds.
__global__ void k_rs_scatter(const uint32_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                             uint32_t *__restrict__ okeys, uint32_t *__restrict__ ovals, int64_t n,
                             int shift, int rbits, int64_t tiles, const int64_t *__restrict__ offs) {
    __shared__ int64_t run[256];
    __shared__ uint32_t wcnt[RS_WARPS][256];
    __shared__ int64_t wpos[RS_WARPS][256];
    const int radix = 1 << rbits;
    const uint32_t mask = radix - 1;
    for (int i = threadIdx.x; i < radix; i += RS_THREADS) {
        run[i] = offs[(int64_t)i * tiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < RS_WARPS; w++) wcnt[w][i] = 0;
    }
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const unsigned lane = lane_id(), wid = warp_id();
    for (int r = 0; r < RS_ITEMS; r++) {
        int64_t idx = base + (int64_t)r * RS_THREADS + threadIdx.x;
        bool valid = idx < n;
        uint32_t k = valid ? keys[idx] : 0;
        uint32_t v = valid ? vals[idx] : 0;
        uint32_t dg = valid ? ((k >> shift) & mask) : 0xffffffffu;
        unsigned peers = __match_any_sync(0xffffffffu, dg);
        unsigned rank = __popc(peers & ((1u << lane) - 1));
        if (valid && rank == 0) wcnt[wid][dg] = __popc(peers);
        __syncthreads();
        for (int i = threadIdx.x; i < radix; i += RS_THREADS) {
            int64_t acc = run[i];
#pragma unroll
            for (int w = 0; w < RS_WARPS; w++) {
                wpos[w][i] = acc;
                acc += wcnt[w][i];
                wcnt[w][i] = 0;
            }
            run[i] = acc;
        }
        __syncthreads();
        if (valid) {
            int64_t pos = wpos[wid][dg] + rank;
            okeys[pos] = k;
            ovals[pos] = v;
        }
    }
}

// Stable LSD radix sort of (key, value) pairs on the low `bits` key bits.
void radix_sort_pairs(Ctx &ctx, uint32_t *keys, uint32_t *vals, uint32_t *keys_alt, uint32_t *vals_alt,
                      int64_t n, int bits, bool *result_in_alt) {
    *result_in_alt = false;
    if (n <= 1 || bits <= 0) return;
    int passes = (bits + 7) / 8;
    int rbits = (bits + passes - 1) / passes;
    int64_t tiles = ceil_div(n, RS_TILE);
    int radix = 1 << rbits;
    DArray<uint32_t> hist;
    DArray<int64_t> offs;
    hist.alloc((int64_t)radix * tiles);
    offs.alloc((int64_t)radix * tiles + 1);
    uint32_t *ik = keys, *iv = vals, *ok = keys_alt, *ov = vals_alt;
    for (int ps = 0; ps < passes; ps++) {
        int shift = ps * rbits;
        int rb = std::min(rbits, bits - shift);
        k_rs_hist<<<(unsigned)tiles, RS_THREADS, 0, ctx.stream>>>(ik, n, shift, rb, tiles, hist.p);
        DBFS_LAUNCHED();
        exclusive_scan_u32_to_i64(ctx, hist.p, offs.p, (int64_t)(1 << rb) * tiles);
        k_rs_scatter<<<(unsigned)tiles, RS_THREADS, 0, ctx.stream>>>(ik, iv, ok, ov, n, shift, rb, tiles,
                                                                     offs.p);
        DBFS_LAUNCHED();
        std::swap(ik, ok);
        std::swap(iv, ov);
        *result_in_alt = !*result_in_alt;
    }
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace dbfs
