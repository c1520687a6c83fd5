// Counter-based generators for the seeded synthetic inputs (host + device).
//
// Bit-for-bit the same definitions as the numpy specification in
// oracle/gen.py (checked by tests/test_gen.py): a splitmix64 finaliser keyed
// by (seed, stream, index), a keyed 4-round multiply/xorshift bijection on
// [0, 2^k) with cycle walking for [0, n).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CC_HD __host__ __device__ __forceinline__
#else
#define CC_HD inline
#endif

namespace ccgen {

constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull;
constexpr uint64_t M1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t M2 = 0x94D049BB133111EBull;
enum : uint64_t { STREAM_RMAT = 1, STREAM_PERM = 2, STREAM_GRID = 3, STREAM_ER = 4,
                  STREAM_FSIZE = 5, STREAM_FTREE = 6 };

CC_HD uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * M1;
    z = (z ^ (z >> 27)) * M2;
    return z ^ (z >> 31);
}
CC_HD uint64_t key(uint64_t seed, uint64_t stream) { return mix(seed * GOLD + stream + 1); }
CC_HD uint64_t rnd(uint64_t k, uint64_t idx) { return mix(k + (idx + 1) * GOLD); }

// Keyed bijection on [0, 2^bits), round keys precomputed by perm_init.
struct Perm {
    uint64_t n;      // domain size (cycle walking bound)
    uint64_t mask;   // 2^bits - 1
    uint32_t bits;
    uint32_t shift;  // (bits + 1) / 2
    uint64_t rk[4];
};

CC_HD uint32_t perm_bits(uint64_t n) {
    uint32_t b = 0;
    if (n <= 1) return 0;
    uint64_t x = n - 1;
    while (x) { ++b; x >>= 1; }
    return b;
}

CC_HD Perm perm_init(uint64_t n, uint64_t pkey) {
    Perm p;
    p.n = n;
    p.bits = perm_bits(n);
    p.mask = p.bits >= 64 ? ~0ull : ((1ull << p.bits) - 1);
    p.shift = (p.bits + 1) / 2;
    for (int r = 0; r < 4; ++r) p.rk[r] = rnd(pkey, (uint64_t)r) & p.mask;
    return p;
}

CC_HD uint64_t perm_pow2(const Perm& p, uint64_t x) {
    if (p.bits == 0) return 0;
    const uint64_t odd[4] = {0x9E3779B97F4A7C15ull, 0xBF58476D1CE4E5B9ull,
                             0x94D049BB133111EBull, 0xD6E8FEB86659FD93ull};
    x &= p.mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        x = (x * odd[r] + p.rk[r]) & p.mask;
        x ^= x >> p.shift;
    }
    return x;
}

CC_HD uint64_t perm_apply(const Perm& p, uint64_t x) {
    uint64_t y = perm_pow2(p, x);
    while (y >= p.n) y = perm_pow2(p, y);
    return y;
}

// RMAT edge `i` (pre-permutation endpoints), levels MSB first.
struct RmatParams {
    uint64_t key;
    uint32_t scale;
    uint32_t tA, tAB, tABC;
};

CC_HD void rmat_edge(const RmatParams& rp, uint64_t i, uint64_t& u, uint64_t& v) {
    const uint64_t D = (rp.scale + 1) / 2;
    uint64_t d = 0;
    u = 0;
    v = 0;
    for (uint32_t l = 0; l < rp.scale; ++l) {
        uint32_t r;
        if ((l & 1) == 0) {
            d = rnd(rp.key, i * D + (l >> 1));
            r = (uint32_t)(d & 0xFFFFFFFFull);
        } else {
            r = (uint32_t)(d >> 32);
        }
        uint64_t ub = r >= rp.tAB;
        uint64_t vb = ((r >= rp.tA) && (r < rp.tAB)) || (r >= rp.tABC);
        u = (u << 1) | ub;
        v = (v << 1) | vb;
    }
}

}  // namespace ccgen
