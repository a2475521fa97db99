// common.cuh -- shared helpers for libdbfs (sm_100a).
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/dbfs.h"

namespace dbfs {

// Exception carrying a dbfs_status; converted to a status at the C-ABI boundary.
struct Error : std::runtime_error {
    int32_t code;
    Error(int32_t c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define DBFS_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess)                                                              \
            throw ::dbfs::Error(_e == cudaErrorMemoryAllocation ? DBFS_ERESOURCE : DBFS_ECUDA, \
                                std::string(#call) + ": " + cudaGetErrorString(_e) + " @" + \
                                    __FILE__ + ":" + std::to_string(__LINE__));             \
    } while (0)

#define DBFS_CHECK(cond, code, msg)                         \
    do {                                                    \
        if (!(cond)) throw ::dbfs::Error((code), (msg));    \
    } while (0)

// Every kernel launch in the library goes through this counter so callers can
// report how many of *our* kernels ran (bench.py "gpu_launches").
extern std::atomic<int64_t> g_kernel_launches;  // several host threads may launch (group.py)
inline void note_launch(int64_t k = 1) { g_kernel_launches += k; }
#define DBFS_LAUNCHED()                          \
    do {                                         \
        ::dbfs::note_launch();                   \
        DBFS_CUDA(cudaGetLastError());           \
    } while (0)

constexpr int KIND_NN = 0, KIND_ND = 1, KIND_DN = 2, KIND_DD = 3;
constexpr int FWD = 0, BWD = 1;
constexpr int MAXW = 64;  // maximum workers (p) supported per graph

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t nwords(int64_t bits) { return (bits + 31) >> 5; }

// Fast divide by the worker count p (owner = v mod p, local = v div p).
struct PDiv {
    uint32_t p, shift, mul;  // mul: magic for non powers of two
    bool pow2;
    __host__ void init(uint32_t pp) {
        p = pp;
        pow2 = (pp & (pp - 1)) == 0;
        shift = 0;
        while ((1u << shift) < pp) shift++;
        mul = 0;
    }
    __host__ __device__ __forceinline__ uint32_t div(uint32_t v) const { return pow2 ? (v >> shift) : v / p; }
    __host__ __device__ __forceinline__ uint32_t mod(uint32_t v) const { return pow2 ? (v & (p - 1)) : v % p; }
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void atomic_add_u64(unsigned long long *p, unsigned long long v) {
    if (v) atomicAdd(p, v);
}

// Warp-level exclusive prefix sum of a 32-bit value; returns the exclusive part, total in *tot.
__device__ __forceinline__ unsigned warp_excl_scan(unsigned v, unsigned *tot) {
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane_id() >= (unsigned)o) x += y;
    }
    *tot = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

}  // namespace dbfs
