// Host-side widening of compact batch outputs (int8 depth -> int32), see
// run_bfs_batch in bfs.cu.  The destination is the caller's page-locked
// array, written once and not read back here: streaming (non-temporal)
// stores skip the read-for-ownership of every destination line, so a
// vertex costs 1 byte read + 4 bytes written of host memory instead of 9.
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cstdint>

namespace dbfs {

__attribute__((target("avx2"))) static void widen_avx2(const int8_t *src, int32_t *dst, int64_t n) {
    int64_t i = 0;
    // scalar head up to a 32-byte aligned destination
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
        dst[i] = src[i];
        i++;
    }
    for (; i + 32 <= n; i += 32) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
        const __m128i lo = _mm256_castsi256_si128(v), hi = _mm256_extracti128_si256(v, 1);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), _mm256_cvtepi8_epi32(lo));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 8), _mm256_cvtepi8_epi32(_mm_srli_si128(lo, 8)));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 16), _mm256_cvtepi8_epi32(hi));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 24), _mm256_cvtepi8_epi32(_mm_srli_si128(hi, 8)));
    }
    for (; i < n; i++) dst[i] = src[i];
    _mm_sfence();
}

// int8 -> int32 (sign extension restores -1) and int32 -> int64 on nthreads cores
void widen_host(const int8_t *l8, const int32_t *p32, int64_t n, int32_t *lv, int64_t *pa, int nthreads) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    const int64_t CH = 1 << 16, nch = (n + CH - 1) / CH;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t c = 0; c < nch; c++) {
        const int64_t b = c * CH, e = std::min(n, b + CH);
        if (lv) {
            if (avx2) widen_avx2(l8 + b, lv + b, e - b);
            else
                for (int64_t i = b; i < e; i++) lv[i] = l8[i];
        }
        if (pa)
            for (int64_t i = b; i < e; i++) pa[i] = p32[i];
    }
}

}  // namespace dbfs
