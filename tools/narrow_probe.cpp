// Host memory bandwidth of the pageable-int64 staging path (DESIGN 5.20):
// 16 threads narrowing int64 pairs to uint32 (scalar / AVX-512, streaming
// stores), against plain read and memcpy bandwidth.
//   g++ -O3 -march=native -pthread tools/narrow_probe.cpp -o /tmp/np && /tmp/np 16
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <chrono>
#include <thread>
#include <vector>

static void par(int T, int64_t n, void (*f)(int64_t, int64_t, void*), void* a) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back([=] { f(n * t / T, n * (t + 1) / T, a); });
    for (auto& x : th) x.join();
}
struct Args { const int64_t* in; uint32_t* out; uint64_t* sink; };
static void scalar(int64_t lo, int64_t hi, void* p) {
    Args* a = (Args*)p;
    for (int64_t i = lo; i < hi; i += 4)
        _mm_stream_si128((__m128i*)(a->out + i), _mm_set_epi32((int)a->in[i + 3], (int)a->in[i + 2],
                                                               (int)a->in[i + 1], (int)a->in[i]));
    _mm_sfence();
}
static void avx512(int64_t lo, int64_t hi, void* p) {
    Args* a = (Args*)p;
    const __m512i zero = _mm512_setzero_si512(), top = _mm512_set1_epi64(0xFFFFFFFFll),
                  ones = _mm512_set1_epi64(-1);
    for (int64_t i = lo; i < hi; i += 16) {
        __m512i x = _mm512_loadu_si512(a->in + i), y = _mm512_loadu_si512(a->in + i + 8);
        x = _mm512_mask_mov_epi64(x, _mm512_cmplt_epi64_mask(x, zero) | _mm512_cmpgt_epi64_mask(x, top), ones);
        y = _mm512_mask_mov_epi64(y, _mm512_cmplt_epi64_mask(y, zero) | _mm512_cmpgt_epi64_mask(y, top), ones);
        _mm512_stream_si512((__m512i*)(a->out + i), _mm512_inserti64x4(
            _mm512_castsi256_si512(_mm512_cvtepi64_epi32(x)), _mm512_cvtepi64_epi32(y), 1));
    }
    _mm_sfence();
}
static void avx512_plain(int64_t lo, int64_t hi, void* p) {
    Args* a = (Args*)p;
    for (int64_t i = lo; i < hi; i += 16) {
        __m512i x = _mm512_loadu_si512(a->in + i), y = _mm512_loadu_si512(a->in + i + 8);
        _mm512_storeu_si512((__m512i*)(a->out + i), _mm512_inserti64x4(
            _mm512_castsi256_si512(_mm512_cvtepi64_epi32(x)), _mm512_cvtepi64_epi32(y), 1));
    }
}
static void readonly(int64_t lo, int64_t hi, void* p) {
    Args* a = (Args*)p;
    __m512i acc = _mm512_setzero_si512();
    for (int64_t i = lo; i < hi; i += 8) acc = _mm512_add_epi64(acc, _mm512_loadu_si512(a->in + i));
    a->sink[lo % 64] += _mm512_reduce_add_epi64(acc);
}
static void cpy(int64_t lo, int64_t hi, void* p) {
    Args* a = (Args*)p;
    memcpy(a->out + lo, (const uint32_t*)a->in + lo, (hi - lo) * 4);
}
int main(int argc, char** argv) {
    const int T = argc > 1 ? atoi(argv[1]) : 16;
    const int64_t n = (int64_t)1 << 31;  // int64 values: 16 GB in, 8 GB out
    int64_t* in = (int64_t*)aligned_alloc(64, n * 8);
    uint32_t* out = (uint32_t*)aligned_alloc(64, n * 4);
    uint64_t sink[64] = {0};
    Args a{in, out, sink};
    par(T, n, [](int64_t lo, int64_t hi, void* p) {
        Args* a = (Args*)p;
        for (int64_t i = lo; i < hi; ++i) ((int64_t*)a->in)[i] = i & 0xFFFFFFF;
        memset(a->out + lo, 0, (hi - lo) * 4);
    }, &a);
    struct { const char* name; void (*f)(int64_t, int64_t, void*); double in_b, out_b; } cases[] = {
        {"read", readonly, 8.0, 0}, {"memcpy", cpy, 4.0, 4.0},
        {"narrow_scalar", scalar, 8.0, 4.0}, {"narrow_avx512", avx512, 8.0, 4.0},
        {"narrow_avx512_plainstore", avx512_plain, 8.0, 4.0}};
    for (auto& c : cases) {
        double best = 1e9;
        for (int r = 0; r < 3; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            par(T, n, c.f, &a);
            best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        printf("{\"case\": \"%s\", \"threads\": %d, \"s\": %.3f, \"read_GBps\": %.1f, \"write_GBps\": %.1f}\n",
               c.name, T, best, n * c.in_b / best / 1e9, n * c.out_b / best / 1e9);
    }
    return (int)(sink[0] & 1);
}
