// Host-side (multi-threaded C++) generators for the seeded synthetic inputs.
// Same definitions as the device generator and as oracle/gen.py.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "contour.h"
#include "gen_rng.cuh"

namespace {

template <typename F>
void parallel_for(int64_t total, int threads, F&& f) {
    if (threads < 1) threads = 1;
    if (total < 65536) threads = 1;
    if (threads == 1) { f(0, total, 0); return; }
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = total * t / threads, hi = total * (t + 1) / threads;
        th.emplace_back([&f, lo, hi, t] { f(lo, hi, t); });
    }
    for (auto& x : th) x.join();
}

inline void put(void* out, int eb, int64_t row, uint64_t u, uint64_t v) {
    if (eb == 4) {
        ((int32_t*)out)[2 * row] = (int32_t)(uint32_t)u;
        ((int32_t*)out)[2 * row + 1] = (int32_t)(uint32_t)v;
    } else {
        ((int64_t*)out)[2 * row] = (int64_t)u;
        ((int64_t*)out)[2 * row + 1] = (int64_t)v;
    }
}

}  // namespace

extern "C" {

int cc_gen_rmat_host(int scale, int ef, uint64_t seed, uint32_t tA, uint32_t tAB, uint32_t tABC,
                     int symmetrize, int permute, int64_t lo, int64_t hi, void* out, int eb,
                     int threads) {
    if (scale < 1 || scale > 32 || ef < 1 || (eb != 4 && eb != 8) || !out) return CC_EINVAL;
    const int64_t n = (int64_t)1 << scale;
    const int64_t M = (int64_t)ef * n;
    const int64_t rows = symmetrize ? 2 * M : M;
    if (lo < 0 || hi > rows || lo > hi) return CC_EINVAL;
    ccgen::RmatParams rp{ccgen::key(seed, ccgen::STREAM_RMAT), (uint32_t)scale, tA, tAB, tABC};
    ccgen::Perm pm = ccgen::perm_init((uint64_t)n, ccgen::key(seed, ccgen::STREAM_PERM));
    parallel_for(hi - lo, threads, [&](int64_t a, int64_t b, int) {
        for (int64_t k = a; k < b; ++k) {
            const int64_t r = lo + k;
            const bool back = symmetrize && r >= M;
            uint64_t u, v;
            ccgen::rmat_edge(rp, back ? (uint64_t)(r - M) : (uint64_t)r, u, v);
            if (permute) { u = ccgen::perm_apply(pm, u); v = ccgen::perm_apply(pm, v); }
            put(out, eb, k, back ? v : u, back ? u : v);
        }
    });
    return CC_OK;
}

int cc_gen_grid_host(int64_t rows, int64_t cols, uint32_t thr, uint64_t seed, int permute,
                     void* out, int eb, int64_t* m_out, int threads) {
    if (rows < 0 || cols < 0 || (eb != 4 && eb != 8) || !m_out) return CC_EINVAL;
    const int64_t n = rows * cols;
    const int64_t nh = rows * std::max<int64_t>(cols - 1, 0);
    const int64_t nv = std::max<int64_t>(rows - 1, 0) * cols;
    const int64_t nb = nh + nv;
    const uint64_t k = ccgen::key(seed, ccgen::STREAM_GRID);
    ccgen::Perm pm = ccgen::perm_init((uint64_t)n, ccgen::key(seed, ccgen::STREAM_PERM));
    if (threads < 1) threads = 1;
    if (nb < 65536) threads = 1;
    std::vector<int64_t> cnt(threads + 1, 0);
    parallel_for(nb, threads, [&](int64_t a, int64_t b, int t) {
        int64_t c = 0;
        for (int64_t i = a; i < b; ++i) c += (uint32_t)(ccgen::rnd(k, (uint64_t)i) >> 32) < thr;
        cnt[t + 1] = c;
    });
    for (int t = 0; t < threads; ++t) cnt[t + 1] += cnt[t];
    *m_out = cnt[threads];
    if (!out) return CC_OK;
    parallel_for(nb, threads, [&](int64_t a, int64_t b, int t) {
        int64_t row = cnt[t];
        for (int64_t i = a; i < b; ++i) {
            if ((uint32_t)(ccgen::rnd(k, (uint64_t)i) >> 32) >= thr) continue;
            uint64_t u, v;
            if (i < nh) {
                u = (uint64_t)((i / (cols - 1)) * cols + i % (cols - 1));
                v = u + 1;
            } else {
                u = (uint64_t)(i - nh);
                v = u + (uint64_t)cols;
            }
            if (permute) { u = ccgen::perm_apply(pm, u); v = ccgen::perm_apply(pm, v); }
            put(out, eb, row++, u, v);
        }
    });
    return CC_OK;
}

int cc_gen_er_host(int64_t n, int64_t pairs, uint64_t seed, void* out, int eb, int64_t* m_out) {
    if (n < 1 || pairs < 0 || (eb != 4 && eb != 8) || !m_out) return CC_EINVAL;
    const uint64_t k = ccgen::key(seed, ccgen::STREAM_ER);
    int64_t row = 0;
    for (int64_t i = 0; i < pairs; ++i) {
        const uint64_t d = ccgen::rnd(k, (uint64_t)i);
        const uint64_t u = (d & 0xFFFFFFFFull) % (uint64_t)n, v = (d >> 32) % (uint64_t)n;
        if (u == v) continue;
        if (out) put(out, eb, row, u, v);
        ++row;
    }
    *m_out = row;
    return CC_OK;
}

int cc_gen_forest_host(const int64_t* sizes, int64_t comps, int64_t n, uint64_t seed, void* out,
                       int eb, int64_t* m_out, int threads) {
    if (comps < 0 || n < 0 || (eb != 4 && eb != 8) || !m_out || (comps && !sizes)) return CC_EINVAL;
    std::vector<int64_t> off(comps + 1, 0);
    for (int64_t c = 0; c < comps; ++c) {
        if (sizes[c] < 1) return CC_EINVAL;
        off[c + 1] = off[c] + sizes[c];
    }
    if (off[comps] > n) return CC_EINVAL;
    *m_out = off[comps] - comps;
    if (!out) return CC_OK;
    const uint64_t kt = ccgen::key(seed, ccgen::STREAM_FTREE);
    ccgen::Perm pm = ccgen::perm_init((uint64_t)n, ccgen::key(seed, ccgen::STREAM_PERM));
    parallel_for(comps, comps >= 65536 ? threads : 1, [&](int64_t a, int64_t b, int) {
        for (int64_t c = a; c < b; ++c) {
            const int64_t o = off[c], s = sizes[c];
            int64_t row = o - c;
            for (int64_t j = 1; j < s; ++j) {
                uint64_t par = (c % 2 == 0) ? (uint64_t)(j - 1)
                                            : ccgen::rnd(kt, (uint64_t)(o + j)) % (uint64_t)j;
                const uint64_t u = ccgen::perm_apply(pm, (uint64_t)o + par);
                const uint64_t v = ccgen::perm_apply(pm, (uint64_t)(o + j));
                put(out, eb, row++, u, v);
            }
        }
    });
    return CC_OK;
}

}  // extern "C"
