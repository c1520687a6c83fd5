// Host-side probe (development aid): narrowing int64 (m, 2) rows to uint32
// pairs vs packing them to 7-byte rows (u | v << 28) for the PCIe link, into
// small rotating output sub-chunks as the staging pipeline does.
//   g++ -O3 -march=native -pthread tools/link_probe.cpp -o /tmp/link_probe && /tmp/link_probe [threads]
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <algorithm>
#include <thread>
#include <vector>

static void narrow(const int64_t* in, uint8_t* out8, int64_t lo, int64_t hi) {
    uint32_t* out = (uint32_t*)out8;
    int64_t i = 2 * lo;
    const int64_t e = 2 * hi;
    for (; i + 16 <= e; i += 16) {
        __m512i a = _mm512_loadu_si512(in + i), b = _mm512_loadu_si512(in + i + 8);
        __m256i la = _mm512_cvtepi64_epi32(a), lb = _mm512_cvtepi64_epi32(b);
        _mm512_storeu_si512(out + i, _mm512_inserti64x4(_mm512_castsi256_si512(la), lb, 1));
    }
    for (; i < e; ++i) out[i] = (uint32_t)in[i];
}

template <int MODE>  // 0 masked store, 1 overlapping full stores + masked last
static void pack7(const int64_t* in, uint8_t* out, int64_t lo, int64_t hi) {
    const int R = 7, b = 28;
    const __m512i iu = _mm512_set_epi64(14, 12, 10, 8, 6, 4, 2, 0);
    const __m512i iv = _mm512_set_epi64(15, 13, 11, 9, 7, 5, 3, 1);
    const __m512i vm = _mm512_set1_epi64((1ll << b) - 1);
    alignas(64) uint8_t idx[64];
    for (int j = 0; j < 64; ++j) idx[j] = (uint8_t)(j < 8 * R ? (j / R) * 8 + j % R : 0);
    const __m512i bi = _mm512_load_si512(idx);
    const __mmask64 sm = (1ull << 56) - 1;
    int64_t i = lo;
    __mmask8 bad = 0;
    for (; i + 8 <= hi; i += 8) {
        __m512i a = _mm512_loadu_si512(in + 2 * i), c = _mm512_loadu_si512(in + 2 * i + 8);
        __m512i u = _mm512_permutex2var_epi64(a, iu, c), v = _mm512_permutex2var_epi64(a, iv, c);
        bad |= _mm512_test_epi64_mask(_mm512_or_si512(u, v), _mm512_set1_epi64(~((1ll << b) - 1)));
        __m512i x = _mm512_or_si512(_mm512_and_si512(u, vm), _mm512_slli_epi64(_mm512_and_si512(v, vm), b));
        __m512i p = _mm512_permutexvar_epi8(bi, x);
        if (MODE == 0 || i + 16 > hi) _mm512_mask_storeu_epi8(out + i * R, sm, p);
        else _mm512_storeu_si512(out + i * R, p);
    }
    for (; i < hi; ++i) {
        uint64_t x = (uint64_t)in[2 * i] | ((uint64_t)in[2 * i + 1] << b);
        memcpy(out + i * R, &x, R);
    }
    if (bad) fprintf(stderr, "bad\n");
}

int main(int argc, char** argv) {
    const int threads = argc > 1 ? atoi(argv[1]) : 16;
    const int64_t m = 1ll << 27;  // 2 GiB of int64 pairs
    const int64_t sub = 1 << 20;
    int64_t* in = (int64_t*)aligned_alloc(64, m * 16);
    for (int64_t i = 0; i < 2 * m; ++i) in[i] = (i * 2654435761ll) & ((1 << 28) - 1);
    auto run = [&](const char* name, auto fn, int rb) {
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> ts;
            for (int t = 0; t < threads; ++t)
                ts.emplace_back([&, t] {
                    // per thread: its part of the rows, in 64 K-row pieces written
                    // into 4 rotating private buffers (LLC-sized, as the pipeline's)
                    std::vector<uint8_t*> outs(4);
                    for (auto& o : outs) o = (uint8_t*)aligned_alloc(64, (sub / 16) * 8 + 64);
                    const int64_t lo = m * t / threads / 16 * 16;
                    const int64_t hi = t == threads - 1 ? m : m * (t + 1) / threads / 16 * 16;
                    int k = 0;
                    for (int64_t a = lo; a < hi; a += sub / 16, ++k) {
                        const int64_t e = std::min<int64_t>(hi, a + sub / 16);
                        fn(in + 2 * a, outs[k & 3], 0, e - a);
                    }
                    for (auto& o : outs) free(o);
                });
            for (auto& x : ts) x.join();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            printf("%-22s threads=%d read %.1f GB/s  out %.1f GB/s  (%.3f s)\n", name, threads,
                   m * 16 / s / 1e9, m * rb / s / 1e9, s);
        }
    };
    run("narrow_uint32_pairs", narrow, 8);
    run("pack7_masked_store", pack7<0>, 7);
    run("pack7_overlap_store", pack7<1>, 7);
    return 0;
}
