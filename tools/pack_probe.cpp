// Host-side probe (development aid): can the host cores pack an int32 (m,2)
// edge array into 3-byte IDs faster than PCIe moves the 4-byte one?
//   g++ -O3 -mssse3 -pthread tools/pack_probe.cpp -o /tmp/pack_probe && /tmp/pack_probe [threads]
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <thread>
#include <vector>

static void pack24(const uint32_t* in, uint8_t* out, size_t nvals) {
    const __m128i shuf = _mm_setr_epi8(0, 1, 2, 4, 5, 6, 8, 9, 10, 12, 13, 14, -1, -1, -1, -1);
    size_t i = 0;
    for (; i + 16 <= nvals; i += 16) {
        __m128i a = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(in + i)), shuf);
        __m128i b = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(in + i + 4)), shuf);
        __m128i c = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(in + i + 8)), shuf);
        __m128i d = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(in + i + 12)), shuf);
        // 4 x 12 bytes -> 48 bytes = 3 x 16
        __m128i o0 = _mm_or_si128(a, _mm_slli_si128(b, 12));
        __m128i o1 = _mm_or_si128(_mm_srli_si128(b, 4), _mm_slli_si128(c, 8));
        __m128i o2 = _mm_or_si128(_mm_srli_si128(c, 8), _mm_slli_si128(d, 4));
        _mm_storeu_si128((__m128i*)(out + 3 * i), o0);
        _mm_storeu_si128((__m128i*)(out + 3 * i + 16), o1);
        _mm_storeu_si128((__m128i*)(out + 3 * i + 32), o2);
    }
    for (; i < nvals; ++i) memcpy(out + 3 * i, in + i, 3);
}

template <typename F>
static double timed(int threads, size_t n, F f) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t)
        ts.emplace_back([&, t] {
            size_t lo = n * t / threads / 16 * 16, hi = t == threads - 1 ? n : n * (t + 1) / threads / 16 * 16;
            f(lo, hi);
        });
    for (auto& x : ts) x.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main(int argc, char** argv) {
    const int threads = argc > 1 ? atoi(argv[1]) : (int)std::thread::hardware_concurrency();
    const size_t n = (size_t)1 << 28;  // 2^28 uint32 = 1 GiB (RMAT-22 symmetrised, int32 AoS)
    uint32_t* in = (uint32_t*)aligned_alloc(64, n * 4);
    uint8_t* out = (uint8_t*)aligned_alloc(64, n * 4);
    timed(threads, n, [&](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; ++i) in[i] = (uint32_t)((i * 2654435761u) & 0x3FFFFF);
        memset(out + 3 * lo, 0, 3 * (hi - lo));
    });
    for (int rep = 0; rep < 3; ++rep) {
        double tc = timed(threads, n, [&](size_t lo, size_t hi) {
            memcpy(out + 4 * lo, in + lo, 4 * (hi - lo));
        });
        double tp = timed(threads, n, [&](size_t lo, size_t hi) { pack24(in + lo, out + 3 * lo, hi - lo); });
        printf("threads=%d memcpy 1 GiB: %.2f ms (%.1f GB/s)  pack24: %.2f ms (%.1f GB/s of input)\n",
               threads, tc * 1e3, n * 4 / tc / 1e9, tp * 1e3, n * 4 / tp / 1e9);
    }
    // check
    for (size_t i = 0; i < 1000; ++i) {
        uint32_t v = 0;
        memcpy(&v, out + 3 * i, 3);
        if (v != in[i]) { printf("MISMATCH at %zu\n", i); return 1; }
    }
    return 0;
}
