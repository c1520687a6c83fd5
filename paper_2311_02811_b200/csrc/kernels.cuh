// Device side of the Contour hot path for sm_100a.
//
// Semantics follow the reference sweep kernel sweep_edges
// (/root/reference/pkg/src/minmapcc/_kernels.py:35-102):
//   per edge (w, v), w != v: walk both label chains x0 = w, x_{j+1} = L[x_j]
//   for up to `order` steps, stopping at a fixed point; z = min of the two
//   h-fold values; lower every chain cell t to z if L[t] > z.
// Labels are uint32 (every vertex ID < n <= 2^32-1), edges packed uint32 SoA.
//
// Layout / bytes per edge for the order-2 asynchronous sweep (the hot path):
//   edge stream  : 8 B/edge, read once with 128-bit streaming loads (ld.global.cs)
//   label gathers: L[u], L[v], then L[L[u]], L[L[v]] (4 x 4 B random, L2-resident
//                  when 4n bytes fit the 126 MB L2) -- predicated off at fixed points
//   label stores : <= 4 conditional 4 B lowerings, only where a cell is lowered
//                  (red.global.min after an L2 re-check of hot cells by default,
//                  plain stores for atomic=False schedules; see the store modes)
// Kernels here: k_sweep (flat rows, any order), k_sweep_o2_peers (fused
// multi-GPU exchange), k_sweep_slice / k_sweep_bucketed[_tma] (dst labels in
// shared memory, dst-bucketed rows), k_check_slice (early check on those
// rows), k_sweep_first (load-free identity sweep).
// The "something was lowered" bit is a per-thread bool folded by
// __syncthreads_or and published with ONE plain store per block (no atomics).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

#include <type_traits>

namespace cck {

typedef uint32_t lab_t;

constexpr int kThreads = 256;
constexpr int kChainBuf = 16;  // buffered chain cells per endpoint for order >= 3

// Store modes for lowering cell t to z (the caller already saw L[t] > z):
//   0 plain store (the reference's non-atomic mode, _kernels.py:94-102)
//   1 fire-and-forget atomic min, red.global.min.u32 (the reference's CAS
//     mode, _kernels.py:79-93, and every synchronous sweep)
//   2 re-check the L2 copy (ld.global.cg) and store plainly only if still > z
//   3 re-check, then red.min
// Modes 2/3 trade one L2 load for skipping stores that a concurrent thread
// already made redundant -- on hot cells those stores invalidate L1 lines
// that every SM is reading.
//   4 re-check EVERY target cell, then red.min: synchronous sweeps, where the
//     target is the shadow array that many edges lower at once (the result,
//     the min over all proposals, is unchanged by skipping provable no-ops)
enum { kStorePlain = 0, kStoreRed = 1, kStoreCheckPlain = 2, kStoreCheckRed = 3,
       kStoreCheckAllRed = 4 };

// HOT marks chain cells past the endpoint (L[w], L[v], ...): those are the
// shared parents many edges lower at once; endpoint cells are random and
// rarely contended, so the re-check modes 2/3 only re-check HOT cells.
template <int SM, bool HOT>
__device__ __forceinline__ void lower(lab_t* T, lab_t t, lab_t z) {
    constexpr bool check =
        SM == kStoreCheckAllRed || (HOT && (SM == kStoreCheckPlain || SM == kStoreCheckRed));
    constexpr bool red = SM == kStoreRed || SM == kStoreCheckRed || SM == kStoreCheckAllRed;
    if (check && __ldcg(T + t) <= z) return;
    if (red) {
        atomicMin(T + t, z);
    } else {
        T[t] = z;
    }
}

// ---- order 1 (C-1 sweeps): z = min(L[w], L[v]); targets w, v -------------
template <int NE, int SM>
__device__ __forceinline__ bool batch_o1(const lab_t* R, lab_t* T, const lab_t (&u)[NE],
                                         const lab_t (&v)[NE]) {
    lab_t lu[NE], lv[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const bool live = u[k] != v[k];
        lu[k] = live ? R[u[k]] : 0u;
        lv[k] = live ? R[v[k]] : 0u;
    }
    bool wrote = false;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        if (u[k] == v[k]) continue;  // self-loop inert (_kernels.py:55-56)
        const lab_t z = min(lu[k], lv[k]);
        if (lu[k] > z) { lower<SM, false>(T, u[k], z); wrote = true; }
        if (lv[k] > z) { lower<SM, false>(T, v[k], z); wrote = true; }
    }
    return wrote;
}

// ---- order 2 (C-2 / C-Syn): z = min(L[L[w]], L[L[v]]); targets w, L[w], v, L[v]
// All four target cells' current values were read while walking the chains
// (L[w]=lu, L[L[w]]=zu, ...), so the conditional stores need no re-read.
// Cache-hint flags OR-ed into the order-2 store-mode parameter (launch_o2
// variants 6/7), for label arrays far beyond L2 (l2_tiled layout): the
// src-side endpoint gathers L[u] hit random lines over all n labels and are
// loaded evict-first, so they do not push the tile's dst window (kHintDstKeep:
// loaded evict-last) out of L2.
// kHintEdgeFirst: the edge stream is loaded L1::no_allocate with an L2
// evict-first policy; kHintSrcKeep: src-side gathers evict-last.
// kHintDstCg: dst gathers bypass L1 (ld.global.cg; they almost never hit it).
// kHintPipe: software-pipelined edge stream (the next iteration's rows are
// loaded before this iteration's gathers; k_sweep only).
constexpr int kStoreMask = 7, kHintSrcStream = 8, kHintDstKeep = 16, kHintEdgeFirst = 32,
              kHintSrcKeep = 64, kHintDstCg = 128, kHintPipe = 256;

__device__ __forceinline__ lab_t ld_evict_last(const lab_t* p) {
    uint64_t pol;
    lab_t r;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

// the same, bypassing L1 (ld.global.cg): random gathers that rarely hit L1
__device__ __forceinline__ lab_t ld_cg_evict_last(const lab_t* p) {
    uint64_t pol;
    lab_t r;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ uint4 ld_edges_evict_first(const uint4* p) {
    uint64_t pol;
    uint4 r;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

template <int NE, int SMH>
__device__ __forceinline__ bool batch_o2(const lab_t* R, lab_t* T, const lab_t (&u)[NE],
                                         const lab_t (&v)[NE]) {
    constexpr int SM = SMH & kStoreMask;
    lab_t lu[NE], lv[NE], zu[NE], zv[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const bool live = u[k] != v[k];
        if (SMH & kHintSrcStream) lu[k] = live ? __ldcs(R + u[k]) : u[k];
        else if (SMH & kHintSrcKeep) lu[k] = live ? ld_evict_last(R + u[k]) : u[k];
        else lu[k] = live ? R[u[k]] : u[k];
        if ((SMH & kHintDstKeep) && (SMH & kHintDstCg))
            lv[k] = live ? ld_cg_evict_last(R + v[k]) : v[k];
        else if (SMH & kHintDstKeep) lv[k] = live ? ld_evict_last(R + v[k]) : v[k];
        else if (SMH & kHintDstCg) lv[k] = live ? __ldcg(R + v[k]) : v[k];
        else lv[k] = live ? R[v[k]] : v[k];
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        // second hop only off a fixed point (early stop, _kernels.py:63-65)
        zu[k] = (lu[k] != u[k]) ? R[lu[k]] : lu[k];
        zv[k] = (lv[k] != v[k]) ? R[lv[k]] : lv[k];
    }
    bool wrote = false;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        if (u[k] == v[k]) continue;
        const lab_t z = min(zu[k], zv[k]);
        if (lu[k] > z) { lower<SM, false>(T, u[k], z); wrote = true; }
        if (lu[k] != u[k] && zu[k] > z) { lower<SM, true>(T, lu[k], z); wrote = true; }
        if (lv[k] > z) { lower<SM, false>(T, v[k], z); wrote = true; }
        if (lv[k] != v[k] && zv[k] > z) { lower<SM, true>(T, lv[k], z); wrote = true; }
    }
    return wrote;
}

// ---- fused sweep + exchange (multi-GPU) ------------------------------------
// Every lowering of the local replica is also sent, as a fire-and-forget
// red.global.min, to the label replicas of the peer GPUs (their buffers
// mapped into this process through CUDA IPC; stores to them travel over
// NVLink / NVSwitch).  The exchange overlaps the sweep edge by edge and its
// volume is the number of lowerings, not 4n bytes per sweep as with an
// allreduce.  After a host barrier every replica holds the min over all
// lowerings of all ranks, i.e. the replicas are identical again.
constexpr int kMaxPeers = 7;
struct PeerSet {
    lab_t* p[kMaxPeers];
    int n;
};

template <int SM, bool HOT>
__device__ __forceinline__ void lower_bcast(lab_t* T, const PeerSet& ps, lab_t t, lab_t z) {
    constexpr bool check = HOT && (SM == kStoreCheckPlain || SM == kStoreCheckRed);
    // a local value already <= z came from a lowering that was broadcast too
    if (check && __ldcg(T + t) <= z) return;
    // always an atomic min locally: peers red.min into this replica at any
    // time, and a plain store could overwrite a smaller value a peer just
    // wrote -- the replicas would then diverge for good (the peer's min was
    // already sent, so nothing would bring it back).  Atomic min is one legal
    // interleaving of the plain-store schedule (atomic=False) too.
    atomicMin(T + t, z);
    for (int i = 0; i < ps.n; ++i) atomicMin(ps.p[i] + t, z);
}

template <int SM>
__global__ void __launch_bounds__(kThreads) k_sweep_o2_peers(const lab_t* __restrict__ src,
                                                             const lab_t* __restrict__ dst,
                                                             int64_t m, lab_t* L, PeerSet ps,
                                                             int* __restrict__ flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool wrote = false;
    const int64_t nvec = m >> 2;
    const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
    const uint4* __restrict__ d4 = reinterpret_cast<const uint4*>(dst);
    auto edge = [&](lab_t u, lab_t v) {
        if (u == v) return;
        const lab_t lu = L[u], lv = L[v];
        const lab_t zu = (lu != u) ? L[lu] : lu;
        const lab_t zv = (lv != v) ? L[lv] : lv;
        const lab_t z = min(zu, zv);
        if (lu > z) { lower_bcast<SM, false>(L, ps, u, z); wrote = true; }
        if (lu != u && zu > z) { lower_bcast<SM, true>(L, ps, lu, z); wrote = true; }
        if (lv > z) { lower_bcast<SM, false>(L, ps, v, z); wrote = true; }
        if (lv != v && zv > z) { lower_bcast<SM, true>(L, ps, lv, z); wrote = true; }
    };
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
        const uint4 a = __ldcs(s4 + i), b = __ldcs(d4 + i);
        edge(a.x, b.x);
        edge(a.y, b.y);
        edge(a.z, b.z);
        edge(a.w, b.w);
    }
    for (int64_t e = (nvec << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += stride)
        edge(src[e], dst[e]);
    if (__syncthreads_or(wrote) && threadIdx.x == 0) *flag = 1;
}

// ---- generic order h (C-m, C-11mm, C-1m1m high sweeps) --------------------
// Walk both chains buffering up to kChainBuf (cell, value) pairs each, then
// lower the buffered cells.  Cells beyond the buffer (chains longer than 16
// hops before a fixed point -- rare) are re-walked from the last buffered
// successor; re-walking is safe under races because a store needs
// L[t] > z, and t >= L[t] > z keeps the forest invariant.
template <int SM>
__device__ __forceinline__ bool edge_oh(const lab_t* R, lab_t* T, lab_t w, lab_t v, int order) {
    if (w == v) return false;
    lab_t cw[kChainBuf], vw[kChainBuf], cv[kChainBuf], vv[kChainBuf];
    int nw = 0, nv = 0;
    lab_t c = w;
    for (int j = 0; j < order; ++j) {
        const lab_t nxt = R[c];
        if (nw < kChainBuf) { cw[nw] = c; vw[nw] = nxt; }
        ++nw;
        if (nxt == c) break;
        c = nxt;
    }
    const lab_t zw = c;
    c = v;
    for (int j = 0; j < order; ++j) {
        const lab_t nxt = R[c];
        if (nv < kChainBuf) { cv[nv] = c; vv[nv] = nxt; }
        ++nv;
        if (nxt == c) break;
        c = nxt;
    }
    const lab_t zv = c;
    const lab_t z = min(zw, zv);
    bool wrote = false;
    const int bw = nw < kChainBuf ? nw : kChainBuf;
    if (vw[0] > z) { lower<SM, false>(T, cw[0], z); wrote = true; }
    for (int i = 1; i < bw; ++i)
        if (vw[i] > z) { lower<SM, true>(T, cw[i], z); wrote = true; }
    if (nw > kChainBuf) {
        lab_t x = vw[kChainBuf - 1];
        for (int j = kChainBuf; j < nw; ++j) {
            const lab_t nxt = R[x];
            if (nxt > z) { lower<SM, true>(T, x, z); wrote = true; }
            if (nxt == x) break;
            x = nxt;
        }
    }
    const int bv = nv < kChainBuf ? nv : kChainBuf;
    if (vv[0] > z) { lower<SM, false>(T, cv[0], z); wrote = true; }
    for (int i = 1; i < bv; ++i)
        if (vv[i] > z) { lower<SM, true>(T, cv[i], z); wrote = true; }
    if (nv > kChainBuf) {
        lab_t x = vv[kChainBuf - 1];
        for (int j = kChainBuf; j < nv; ++j) {
            const lab_t nxt = R[x];
            if (nxt > z) { lower<SM, true>(T, x, z); wrote = true; }
            if (nxt == x) break;
            x = nxt;
        }
    }
    return wrote;
}

// ---- generic order h, register chains (the bulk sweeps) --------------------
// Same update as edge_oh, but the first kRegChain cells of each chain live in
// registers (fully unrolled, no local memory) and the first hop of all NE
// edges is loaded up front; chains that run longer (before a fixed point and
// within `order` steps) are finished by walking/re-walking as in edge_oh.
constexpr int kRegChain = 4;

struct RegChain {
    lab_t c[kRegChain], val[kRegChain];
    int len;  // cells walked (may exceed kRegChain)
    lab_t z;  // the order-fold value
};

__device__ __forceinline__ void walk_reg(const lab_t* R, lab_t x, lab_t lx, int order,
                                         RegChain& ch) {
    lab_t c = x, nxt = lx;
    int j = 0;
    bool done = false;
#pragma unroll
    for (int s = 0; s < kRegChain; ++s) {
        if (!done) {
            if (s > 0) nxt = R[c];
            ch.c[s] = c;
            ch.val[s] = nxt;
            ++j;
            if (nxt == c) {
                done = true;
            } else {
                c = nxt;
                if (j == order) done = true;
            }
        }
    }
    if (!done) {
        for (;;) {
            const lab_t n2 = R[c];
            ++j;
            if (n2 == c) break;
            c = n2;
            if (j == order) break;
        }
    }
    ch.len = j;
    ch.z = c;
}

template <int SM>
__device__ __forceinline__ bool lower_reg(const lab_t* R, lab_t* T, const RegChain& ch, lab_t z) {
    bool wrote = false;
#pragma unroll
    for (int s = 0; s < kRegChain; ++s) {
        if (s < ch.len && ch.val[s] > z) {
            if (s == 0) lower<SM, false>(T, ch.c[s], z);
            else lower<SM, true>(T, ch.c[s], z);
            wrote = true;
        }
    }
    if (ch.len > kRegChain) {
        lab_t x = ch.val[kRegChain - 1];
        for (int j = kRegChain; j < ch.len; ++j) {
            const lab_t nxt = R[x];
            if (nxt > z) { lower<SM, true>(T, x, z); wrote = true; }
            if (nxt == x) break;
            x = nxt;
        }
    }
    return wrote;
}

// Order >= 3.  The first three hops of every chain are loaded for all NE
// edges at once (ILP 2*NE per hop, as in the order-2 batch); after a sweep or
// two almost every chain reaches a fixed point within those hops (vertex ->
// parent -> root), and such an edge is finished from registers.  Edges whose
// chain is still moving after three hops (with order > 3) take the general
// register-chain walk.
template <int NE, int SM>
__device__ __forceinline__ bool batch_oh(const lab_t* R, lab_t* T, const lab_t (&u)[NE],
                                         const lab_t (&v)[NE], int order) {
    lab_t lu[NE], lv[NE], zu[NE], zv[NE], gu[NE], gv[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const bool live = u[k] != v[k];
        lu[k] = live ? R[u[k]] : u[k];
        lv[k] = live ? R[v[k]] : v[k];
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        zu[k] = (lu[k] != u[k]) ? R[lu[k]] : lu[k];
        zv[k] = (lv[k] != v[k]) ? R[lv[k]] : lv[k];
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        gu[k] = (zu[k] != lu[k]) ? R[zu[k]] : zu[k];
        gv[k] = (zv[k] != lv[k]) ? R[zv[k]] : zv[k];
    }
    bool wrote = false;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        if (u[k] == v[k]) continue;
        // chain ends within three cells: at a fixed point, or after exactly
        // three steps when order == 3 (then the third successor is z)
        const bool short_u = lu[k] == u[k] || zu[k] == lu[k] || gu[k] == zu[k] || order == 3;
        const bool short_v = lv[k] == v[k] || zv[k] == lv[k] || gv[k] == zv[k] || order == 3;
        if (short_u && short_v) {
            const lab_t eu = lu[k] == u[k] ? u[k] : (zu[k] == lu[k] ? lu[k] : gu[k]);
            const lab_t ev = lv[k] == v[k] ? v[k] : (zv[k] == lv[k] ? lv[k] : gv[k]);
            const lab_t z = min(eu, ev);
            if (lu[k] > z) { lower<SM, false>(T, u[k], z); wrote = true; }
            if (lu[k] != u[k] && zu[k] > z) { lower<SM, true>(T, lu[k], z); wrote = true; }
            if (lu[k] != u[k] && zu[k] != lu[k] && gu[k] > z) {
                lower<SM, true>(T, zu[k], z);
                wrote = true;
            }
            if (lv[k] > z) { lower<SM, false>(T, v[k], z); wrote = true; }
            if (lv[k] != v[k] && zv[k] > z) { lower<SM, true>(T, lv[k], z); wrote = true; }
            if (lv[k] != v[k] && zv[k] != lv[k] && gv[k] > z) {
                lower<SM, true>(T, zv[k], z);
                wrote = true;
            }
        } else {
            RegChain cu, cv;
            walk_reg(R, u[k], lu[k], order, cu);
            walk_reg(R, v[k], lv[k], order, cv);
            const lab_t z = min(cu.z, cv.z);
            wrote |= lower_reg<SM>(R, T, cu, z);
            wrote |= lower_reg<SM>(R, T, cv, z);
        }
    }
    return wrote;
}

template <int OK, int NE, int SM>
__device__ __forceinline__ bool batch_other(const lab_t* R, lab_t* T, const lab_t (&u)[NE],
                                            const lab_t (&v)[NE], int order) {
    if (OK == 1) return batch_o1<NE, SM>(R, T, u, v);
    if (SM == kStoreCheckAllRed) {
        // synchronous sweeps (the only users of mode 4): labels do not move
        // within the sweep, chains stay long, so walk each edge's chains
        // directly instead of batching three hops first
        bool wrote = false;
#pragma unroll 1
        for (int k = 0; k < NE; ++k) {
            if (u[k] == v[k]) continue;
            RegChain cu, cv;
            walk_reg(R, u[k], R[u[k]], order, cu);
            walk_reg(R, v[k], R[v[k]], order, cv);
            const lab_t z = min(cu.z, cv.z);
            wrote |= lower_reg<SM>(R, T, cu, z);
            wrote |= lower_reg<SM>(R, T, cv, z);
        }
        return wrote;
    }
    return batch_oh<NE, SM>(R, T, u, v, order);
}

// SM: store mode, plus the kHint* bits for the order-2 batch.
template <int OK, int NE, int SM>
__device__ __forceinline__ bool batch(const lab_t* R, lab_t* T, const lab_t (&u)[NE],
                                      const lab_t (&v)[NE], int order) {
    if (OK == 2) return batch_o2<NE, SM>(R, T, u, v);
    return batch_other<OK, NE, SM & kStoreMask>(R, T, u, v, order);
}

// Exact single-edge form for cc_mm_order (16-cell buffers: every golden
// chain is buffered before any store, as the reference does).
template <int OK, int SM>
__device__ __forceinline__ bool single_edge(const lab_t* R, lab_t* T, lab_t w, lab_t v,
                                            int order) {
    lab_t u1[1] = {w}, v1[1] = {v};
    if (OK == 1) return batch_o1<1, SM>(R, T, u1, v1);
    if (OK == 2) return batch_o2<1, SM>(R, T, u1, v1);
    return edge_oh<SM>(R, T, w, v, order);
}

// One sweep over edges [0, m) of the SoA arrays (16-byte aligned).
// OK: 1, 2 or 0 (generic order).  Sync sweeps pass R = labels, T = shadow
// with SM = kStoreRed; async sweeps R == T (in place).  SM: store mode.  NV: uint4 vectors per
// array per thread per iteration (4*NV edges in flight per thread).
// d_order != nullptr (graph-captured loop): the order of this sweep is read
// from device memory and the launch is a no-op unless it matches OK, so a
// captured body holds one launch per order kind the schedule can use.
template <int OK, int SM, int NV, int MINB = 1>
__global__ void __launch_bounds__(kThreads, MINB) k_sweep(const lab_t* __restrict__ src,
                                                    const lab_t* __restrict__ dst, int64_t m,
                                                    const lab_t* R, lab_t* T, int order,
                                                    int* __restrict__ flag,
                                                    const int* __restrict__ d_order) {
    if (d_order) {
        order = *d_order;
        if ((OK == 1) != (order == 1) || (OK == 2) != (order == 2)) return;
    }
    const int64_t nvec = m >> 2;
    const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
    const uint4* __restrict__ d4 = reinterpret_cast<const uint4*>(dst);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool wrote = false;
    auto load = [&](int64_t i, uint4& a, uint4& b) {
        a = make_uint4(0, 0, 0, 0);
        b = make_uint4(0, 0, 0, 0);
        if (i < nvec) {
            if (SM & kHintEdgeFirst) {
                a = ld_edges_evict_first(s4 + i);
                b = ld_edges_evict_first(d4 + i);
            } else {
                a = __ldcs(s4 + i);
                b = __ldcs(d4 + i);
            }
        }
    };
    if constexpr ((SM & kHintPipe) != 0) {
        uint4 a[NV], b[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) load(tid + (int64_t)q * stride, a[q], b[q]);
        for (int64_t base = tid; base < nvec; base += stride * NV) {
            lab_t u[4 * NV], v[4 * NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                u[4 * q + 0] = a[q].x; u[4 * q + 1] = a[q].y; u[4 * q + 2] = a[q].z;
                u[4 * q + 3] = a[q].w;
                v[4 * q + 0] = b[q].x; v[4 * q + 1] = b[q].y; v[4 * q + 2] = b[q].z;
                v[4 * q + 3] = b[q].w;
                load(base + stride * NV + (int64_t)q * stride, a[q], b[q]);
            }
            wrote |= batch<OK, 4 * NV, SM>(R, T, u, v, order);
        }
    } else {
        for (int64_t base = tid; base < nvec; base += stride * NV) {
            lab_t u[4 * NV], v[4 * NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                uint4 a, b;
                load(base + (int64_t)q * stride, a, b);
                u[4 * q + 0] = a.x; u[4 * q + 1] = a.y; u[4 * q + 2] = a.z; u[4 * q + 3] = a.w;
                v[4 * q + 0] = b.x; v[4 * q + 1] = b.y; v[4 * q + 2] = b.z; v[4 * q + 3] = b.w;
            }
            wrote |= batch<OK, 4 * NV, SM>(R, T, u, v, order);
        }
    }
    for (int64_t e = (nvec << 2) + tid; e < m; e += stride) {
        lab_t u[1] = {src[e]}, v[1] = {dst[e]};
        wrote |= batch<OK, 1, SM>(R, T, u, v, order);
    }
    if (__syncthreads_or(wrote) && threadIdx.x == 0) *flag = 1;
}

// ---- dst-bucketed order-2 sweep ---------------------------------------------
// Layout (cc_reorder_edges mode 3): rows grouped by dst bucket
// [b*B, (b+1)*B) and sorted by src inside each bucket.  A work item is a
// row range inside one bucket.  The CTA copies the bucket's B labels into
// shared memory, so the random L[dst] gather becomes a shared-memory load
// (no L1->L2 request), and src-sorted rows make the L[src] gathers of a warp
// coalesce.  A lowering of the dst cell goes to shared memory (so later rows
// of the item see it) AND through to global memory with store mode SM, so
// other CTAs see it as early as with the plain kernel; every other cell is
// read and lowered in global memory.  Slice reads may be stale w.r.t. other
// CTAs -- a legal asynchronous interleaving; a sweep that decides no
// lowering anywhere saw unchanged labels everywhere, so the ballot/OR flag
// stays exact.
struct BucketItem {
    int64_t start, end;  // row range
    uint32_t base, len;  // label slice [base, base+len)
};

template <int SM, int NE>
__device__ __forceinline__ bool bucket_rows(lab_t* L, const lab_t* sl, lab_t base, lab_t len,
                                            const lab_t (&u)[NE], const lab_t (&v)[NE]) {
    lab_t lu[NE], lv[NE], zu[NE], zv[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const bool live = u[k] != v[k];
        lv[k] = live ? ((v[k] - base < len) ? sl[v[k] - base] : L[v[k]]) : v[k];
        lu[k] = live ? L[u[k]] : u[k];
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        zu[k] = (lu[k] != u[k]) ? L[lu[k]] : lu[k];
        zv[k] = (lv[k] != v[k]) ? ((lv[k] - base < len) ? sl[lv[k] - base] : L[lv[k]]) : lv[k];
    }
    bool wrote = false;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        if (u[k] == v[k]) continue;
        const lab_t z = min(zu[k], zv[k]);
        // z <= zu <= lu and z <= zv <= lv (every stored label is <= its
        // cell's index), so nothing is lowered iff max(lu, lv) == z: one
        // test on the common path of a converging sweep
        if (max(lu[k], lv[k]) == z) continue;
        if (lu[k] > z) { lower<SM, false>(L, u[k], z); wrote = true; }
        if (lu[k] != u[k] && zu[k] > z) { lower<SM, true>(L, lu[k], z); wrote = true; }
        if (lv[k] > z) {
            if (v[k] - base < len) atomicMin((lab_t*)sl + (v[k] - base), z);
            lower<SM, false>(L, v[k], z);
            wrote = true;
        }
        if (lv[k] != v[k] && zv[k] > z) {
            if (lv[k] - base < len) atomicMin((lab_t*)sl + (lv[k] - base), z);
            lower<SM, true>(L, lv[k], z);
            wrote = true;
        }
    }
    return wrote;
}

// NV uint4 vectors (4 rows each) per array per thread per iteration.
template <int SM, int NV>
__global__ void __launch_bounds__(1024)
    k_sweep_bucketed(const lab_t* __restrict__ src, const lab_t* __restrict__ dst, lab_t* L,
                     const BucketItem* __restrict__ items, int n_items, int* __restrict__ flag,
                     const int* __restrict__ d_order) {
    extern __shared__ lab_t sl[];
    if (d_order && *d_order != 2) return;
    bool wrote = false;
    const int T = blockDim.x;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const BucketItem w = items[it];
        const lab_t base = w.base, len = w.len;
        for (lab_t i = threadIdx.x; i < len; i += T) sl[i] = __ldcg(L + base + i);
        __syncthreads();
        // [start, a0) scalar head, [a0, a1) uint4 body, [a1, end) scalar tail
        const int64_t a0 = min((w.start + 3) & ~(int64_t)3, w.end);
        const int64_t a1 = max(a0, w.end & ~(int64_t)3);
        for (int64_t r = w.start + threadIdx.x; r < a0; r += T) {
            lab_t u[1] = {src[r]}, v[1] = {dst[r]};
            wrote |= bucket_rows<SM, 1>(L, sl, base, len, u, v);
        }
        const uint4* s4 = reinterpret_cast<const uint4*>(src + a0);
        const uint4* d4 = reinterpret_cast<const uint4*>(dst + a0);
        const int64_t nvec = (a1 - a0) >> 2;
        for (int64_t q0 = threadIdx.x; q0 < nvec; q0 += (int64_t)T * NV) {
            lab_t u[4 * NV], v[4 * NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int64_t i = q0 + (int64_t)q * T;
                uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
                if (i < nvec) { a = __ldcs(s4 + i); b = __ldcs(d4 + i); }
                u[4 * q + 0] = a.x; u[4 * q + 1] = a.y; u[4 * q + 2] = a.z; u[4 * q + 3] = a.w;
                v[4 * q + 0] = b.x; v[4 * q + 1] = b.y; v[4 * q + 2] = b.z; v[4 * q + 3] = b.w;
            }
            // padding rows (i >= nvec) are u == v == 0: inert, and 0 is never
            // read from the slice because live rows only are looked up
            wrote |= bucket_rows<SM, 4 * NV>(L, sl, base, len, u, v);
        }
        for (int64_t r = a1 + threadIdx.x; r < w.end; r += T) {
            lab_t u[1] = {src[r]}, v[1] = {dst[r]};
            wrote |= bucket_rows<SM, 1>(L, sl, base, len, u, v);
        }
        __syncthreads();  // the next item overwrites the slice
    }
    if (__syncthreads_or(wrote) && threadIdx.x == 0) *flag = 1;
}

// ---- dst-bucketed order-2 sweep, bulk-copy pipelined ------------------------
// Same layout, items and semantics as k_sweep_bucketed, restructured for
// latency: the ncu profile of k_sweep_bucketed shows it latency-bound (1 CTA
// of 32 warps per SM, "long scoreboard" the top stall: every thread waits on
// its own edge loads before it can issue its gathers).  Here one thread
// streams the item's rows into an NS-deep ring of shared-memory stages with
// cp.async.bulk (TMA bulk copies, completion on an mbarrier), and the slice
// itself arrives the same way, so the threads only issue label gathers and
// stores.  Every dst endpoint v of an item lies in its slice by construction
// (rows are grouped by dst bucket), so the first-hop dst gather is an
// unconditional shared-memory load; the second hops read global memory.
constexpr int kBT = 1024;             // threads per CTA
constexpr int kStageRows = 4 * kBT;   // rows per pipeline stage (4 per thread)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes,
                                         uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_addr(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_addr(b))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_addr(b);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}

__device__ __forceinline__ lab_t lds_u32(uint32_t addr) {
    lab_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
}

// Shared-memory address of slice entry v is sadj + 4 v, sadj = smem(sl) -
// 4 base (mod 2^32): one IMAD per gather, and the compiler no longer
// re-derives the shared window base (S2R SR_CgaCtaId + LEA) per batch.
__device__ __forceinline__ uint32_t slice_adj(const lab_t* sl, lab_t base) {
    return smem_addr(sl) - 4u * base;
}

// Rows (u[k], v[k]) with v[k] in the slice [base, base+len); u == v rows are
// inert (self loops and the masked rows of a partial stage).
template <int SM, int NE>
__device__ __forceinline__ bool slice_rows(lab_t* L, lab_t* sl, lab_t base, lab_t len,
                                           const lab_t (&u)[NE], const lab_t (&v)[NE]) {
    const uint32_t sadj = slice_adj(sl, base);
    lab_t lu[NE], lv[NE], zu[NE], zv[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const bool live = u[k] != v[k];
        lv[k] = live ? lds_u32(sadj + 4u * v[k]) : v[k];
        lu[k] = live ? L[u[k]] : u[k];
    }
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        zu[k] = (lu[k] != u[k]) ? L[lu[k]] : lu[k];
        zv[k] = (lv[k] != v[k]) ? L[lv[k]] : lv[k];
    }
    bool wrote = false;
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        if (u[k] == v[k]) continue;
        const lab_t z = min(zu[k], zv[k]);
        // z <= zu <= lu and z <= zv <= lv (every stored label is <= its
        // cell's index), so nothing is lowered iff max(lu, lv) == z: one
        // test on the common path of a converging sweep
        if (max(lu[k], lv[k]) == z) continue;
        if (lu[k] > z) { lower<SM, false>(L, u[k], z); wrote = true; }
        if (lu[k] != u[k] && zu[k] > z) { lower<SM, true>(L, lu[k], z); wrote = true; }
        if (lv[k] > z) {
            atomicMin(sl + (v[k] - base), z);
            lower<SM, false>(L, v[k], z);
            wrote = true;
        }
        if (lv[k] != v[k] && zv[k] > z) {
            if (lv[k] - base < len) atomicMin(sl + (lv[k] - base), z);
            lower<SM, true>(L, lv[k], z);
            wrote = true;
        }
    }
    return wrote;
}

// Dst column of a bucketed row range: absolute uint32 vertex IDs, or (DT =
// uint16_t, the compact hybrid copy) 16-bit offsets into the item's slice
// [base, base + 2^bucket_shift), 2 B per row instead of 4.
template <typename DT>
__device__ __forceinline__ void load_dst4(const DT* __restrict__ d, int64_t q, lab_t base,
                                          lab_t (&v)[4]) {
    if constexpr (sizeof(DT) == 4) {
        const uint4 b = __ldcs(reinterpret_cast<const uint4*>(d) + q);
        v[0] = b.x; v[1] = b.y; v[2] = b.z; v[3] = b.w;
    } else {
        const uint2 b = __ldcs(reinterpret_cast<const uint2*>(d) + q);
        v[0] = base + (b.x & 0xFFFFu); v[1] = base + (b.x >> 16);
        v[2] = base + (b.y & 0xFFFFu); v[3] = base + (b.y >> 16);
    }
}
template <typename DT>
__device__ __forceinline__ lab_t load_dst1(const DT* __restrict__ d, int64_t r, lab_t base) {
    if constexpr (sizeof(DT) == 4) return d[r];
    else return base + (lab_t)d[r];
}

// Lean form of k_sweep_bucketed for items with a slice (len > 0): the
// first-hop dst gather is an unconditional (predicated) shared-memory load
// and the second hops are predicated global loads -- no divergent branches
// around the loads, so a thread's gathers issue back to back.  Warps run
// independently inside an item (no barrier per row batch).  PF: the next
// batch's edge vectors are loaded before the current batch is processed.
template <int SM, bool PF, typename DT = lab_t>
__global__ void __launch_bounds__(kBT, 1)
    k_sweep_slice(const lab_t* __restrict__ src, const DT* __restrict__ dst, lab_t* L,
                  const BucketItem* __restrict__ items, int n_items, int* __restrict__ flag,
                  const int* __restrict__ d_order) {
    extern __shared__ __align__(128) lab_t sl[];
    __shared__ __align__(8) uint64_t sbar;
    if (d_order && *d_order != 2) return;
    bool wrote = false;
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&sbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t par = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const BucketItem w = items[it];
        const lab_t base = w.base, len = w.len;
        // the slice arrives as ONE bulk copy (a per-thread load loop is 32
        // dependent L2 round trips per thread: ~13 us per item, measured)
        const lab_t lenb = len & ~3u;
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sbar, lenb * 4u);
            if (lenb) bulk_g2s(sl, L + base, lenb * 4u, &sbar);
        }
        if (tid < len - lenb) sl[lenb + tid] = __ldcg(L + base + lenb + tid);
        mbar_wait(&sbar, par);
        par ^= 1u;
        __syncthreads();
        const int64_t a0 = min((w.start + 3) & ~(int64_t)3, w.end);
        const int64_t a1 = max(a0, w.end & ~(int64_t)3);
        if (tid < a0 - w.start) {  // <= 3 head rows
            lab_t u[1] = {src[w.start + tid]}, v[1] = {load_dst1(dst, w.start + tid, base)};
            wrote |= slice_rows<SM, 1>(L, sl, base, len, u, v);
        }
        if (tid < w.end - a1) {  // <= 3 tail rows
            lab_t u[1] = {src[a1 + tid]}, v[1] = {load_dst1(dst, a1 + tid, base)};
            wrote |= slice_rows<SM, 1>(L, sl, base, len, u, v);
        }
        const uint4* s4 = reinterpret_cast<const uint4*>(src + a0);
        const DT* d0 = dst + a0;
        const int64_t nvec = (a1 - a0) >> 2;
        // masked rows are inert (u == v): u = base pairs with a zero offset
        // (compact copy) and u = 0 with a zero vertex ID
        const lab_t uf = sizeof(DT) == 2 ? base : 0u;
        const uint4 fill = make_uint4(uf, uf, uf, uf);
        if (PF) {
            // ping-pong: batch q's rows in (u0, v0) while q + kBT's load into
            // (u1, v1) and the other way round -- no register moves per batch
            lab_t u0[4] = {uf, uf, uf, uf}, v0[4] = {0, 0, 0, 0}, u1[4], v1[4];
            if (sizeof(DT) == 2) { v0[0] = v0[1] = v0[2] = v0[3] = base; }
            int64_t q = tid;
            if (q < nvec) {
                const uint4 a = __ldcs(s4 + q);
                u0[0] = a.x; u0[1] = a.y; u0[2] = a.z; u0[3] = a.w;
                load_dst4(d0, q, base, v0);
            }
            for (; q < nvec; q += 2 * kBT) {
                uint4 a = fill;
                if (q + kBT < nvec) { a = __ldcs(s4 + q + kBT); load_dst4(d0, q + kBT, base, v1); }
                else { v1[0] = v1[1] = v1[2] = v1[3] = uf; }
                u1[0] = a.x; u1[1] = a.y; u1[2] = a.z; u1[3] = a.w;
                wrote |= slice_rows<SM, 4>(L, sl, base, len, u0, v0);
                if (q + kBT >= nvec) break;
                a = fill;
                if (q + 2 * kBT < nvec) { a = __ldcs(s4 + q + 2 * kBT); load_dst4(d0, q + 2 * kBT, base, v0); }
                else { v0[0] = v0[1] = v0[2] = v0[3] = uf; }
                u0[0] = a.x; u0[1] = a.y; u0[2] = a.z; u0[3] = a.w;
                wrote |= slice_rows<SM, 4>(L, sl, base, len, u1, v1);
            }
        } else {
            for (int64_t q = tid; q < nvec; q += kBT) {
                const uint4 a = __ldcs(s4 + q);
                lab_t u[4] = {a.x, a.y, a.z, a.w}, v[4];
                load_dst4(d0, q, base, v);
                wrote |= slice_rows<SM, 4>(L, sl, base, len, u, v);
            }
        }
        __syncthreads();  // the next item overwrites the slice
    }
    if (__syncthreads_or(wrote) && threadIdx.x == 0) *flag = 1;
}

// Edge-agreement half of the early convergence check (engine.py:331-348)
// on the dst-bucketed layout: L[v] comes from the item's slice in shared
// memory, so the only global gathers are the src-sorted (coalescing) L[u].
// Nothing is written during a check, so the slice equals global memory.
// Same guards as the flat check: return at once when the sweep wrote
// nothing or the check already failed; poll the failure word every 16 row
// batches (one load per warp).
// NV uint4 row vectors per thread per iteration (4*NV independent gathers).
template <int NV, typename DT = lab_t>
__global__ void __launch_bounds__(kBT, 1)
    k_check_slice(const lab_t* __restrict__ src, const DT* __restrict__ dst,
                  const lab_t* __restrict__ L, const BucketItem* __restrict__ items, int n_items,
                  int* flags, int wrote_idx, int check_idx) {
    extern __shared__ __align__(128) lab_t sl[];
    __shared__ __align__(8) uint64_t sbar;
    volatile int* vf = flags;
    const int tid = threadIdx.x;
    // the skip decision must be uniform across the CTA: another CTA can set
    // the failure word while this one's threads read it, and a thread that
    // left early could be the one that issues the slice copy the others wait
    // for (mbarrier) -- a hang, seen once in ~50 test runs
    if (__syncthreads_or(tid == 0 && (!vf[wrote_idx] || vf[check_idx]))) return;
    if (tid == 0) {
        mbar_init(&sbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t par = 0;
    bool bad = false;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const BucketItem w = items[it];
        const lab_t base = w.base, len = w.len;
        const lab_t lenb = len & ~3u;
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sbar, lenb * 4u);
            if (lenb) bulk_g2s(sl, L + base, lenb * 4u, &sbar);
        }
        if (tid < len - lenb) sl[lenb + tid] = L[base + lenb + tid];
        mbar_wait(&sbar, par);
        par ^= 1u;
        __syncthreads();
        const int64_t a0 = min((w.start + 3) & ~(int64_t)3, w.end);
        const int64_t a1 = max(a0, w.end & ~(int64_t)3);
        if (tid < a0 - w.start)
            bad |= L[src[w.start + tid]] != sl[load_dst1(dst, w.start + tid, base) - base];
        if (tid < w.end - a1) bad |= L[src[a1 + tid]] != sl[load_dst1(dst, a1 + tid, base) - base];
        const uint32_t sadj = slice_adj(sl, base);
        const uint4* s4 = reinterpret_cast<const uint4*>(src + a0);
        const DT* d0 = dst + a0;
        const int64_t nvec = (a1 - a0) >> 2;
        int k = 0;
        for (int64_t q = tid; q < nvec && !bad; q += (int64_t)kBT * NV) {
            if ((++k & 7) == 0 && vf[check_idx]) break;
            uint4 a[NV];
            lab_t b[NV][4];
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int64_t i = q + (int64_t)j * kBT;
                if (i < nvec) { a[j] = __ldcs(s4 + i); load_dst4(d0, i, base, b[j]); }
            }
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                if (q + (int64_t)j * kBT < nvec)
                    bad |= (L[a[j].x] != lds_u32(sadj + 4u * b[j][0])) |
                           (L[a[j].y] != lds_u32(sadj + 4u * b[j][1])) |
                           (L[a[j].z] != lds_u32(sadj + 4u * b[j][2])) |
                           (L[a[j].w] != lds_u32(sadj + 4u * b[j][3]));
            }
        }
        if (bad) vf[check_idx] = 1;
        // uniform exit decision (the slice is reused by the next item)
        if (__syncthreads_or(bad || (tid == 0 && vf[check_idx]))) return;
    }
}

// Dynamic shared memory: NS stages x (src, dst) x kStageRows labels, then the
// slice of up to 2^bucket_shift labels.  Items must have len > 0.
template <int SM, int NS>
__global__ void __launch_bounds__(kBT, 1)
    k_sweep_bucketed_tma(const lab_t* __restrict__ src, const lab_t* __restrict__ dst, lab_t* L,
                         const BucketItem* __restrict__ items, int n_items,
                         int* __restrict__ flag, const int* __restrict__ d_order) {
    extern __shared__ __align__(128) lab_t smem[];
    __shared__ __align__(8) uint64_t full[NS + 1];  // [NS] = slice barrier
    if (d_order && *d_order != 2) return;
    lab_t* sl = smem + NS * 2 * kStageRows;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s <= NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t par = 0;  // parity bit per barrier, identical in every thread
    bool wrote = false;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const BucketItem w = items[it];
        const lab_t base = w.base, len = w.len;
        const int64_t a0 = w.start & ~(int64_t)3;
        const int64_t a1 = max(a0, w.end & ~(int64_t)3);
        const int64_t nst = (a1 - a0 + kStageRows - 1) / kStageRows;
        const lab_t lenb = len & ~3u;  // bulk part of the slice (16-byte multiple)
        if (tid == 0) {
            // order this CTA's earlier generic-proxy writes of the slice and
            // stages (made visible by the __syncthreads) before the bulk writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lenb) {
                mbar_expect_tx(&full[NS], lenb * 4u);
                bulk_g2s(sl, L + base, lenb * 4u, &full[NS]);
            } else {
                mbar_expect_tx(&full[NS], 0u);
            }
            for (int64_t k = 0; k < (nst < NS ? nst : (int64_t)NS); ++k) {
                const int64_t r0 = a0 + k * kStageRows;
                const uint32_t bytes = (uint32_t)(min((int64_t)kStageRows, a1 - r0) * 4);
                lab_t* st = smem + k * 2 * kStageRows;
                mbar_expect_tx(&full[k], 2u * bytes);
                bulk_g2s(st, src + r0, bytes, &full[k]);
                bulk_g2s(st + kStageRows, dst + r0, bytes, &full[k]);
            }
        }
        for (lab_t i = lenb + tid; i < len; i += kBT) sl[i] = __ldcg(L + base + i);
        mbar_wait(&full[NS], (par >> NS) & 1u);
        par ^= 1u << NS;
        __syncthreads();  // slice tail stores visible
        for (int64_t k = 0; k < nst; ++k) {
            const int s = (int)(k % NS);
            mbar_wait(&full[s], (par >> s) & 1u);
            par ^= 1u << s;
            const int64_t r = a0 + k * kStageRows + 4 * tid;
            const lab_t* st = smem + s * 2 * kStageRows;
            lab_t u[4] = {0, 0, 0, 0}, v[4] = {0, 0, 0, 0};
            if (r < a1) {
                const uint4 a = reinterpret_cast<const uint4*>(st)[tid];
                const uint4 b = reinterpret_cast<const uint4*>(st + kStageRows)[tid];
                u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w;
                v[0] = b.x; v[1] = b.y; v[2] = b.z; v[3] = b.w;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (r + j < w.start) v[j] = u[j];  // head rows of the previous item
            }
            wrote |= slice_rows<SM, 4>(L, sl, base, len, u, v);
            __syncthreads();  // stage s consumed by every thread
            if (tid == 0 && k + NS < nst) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const int64_t r0 = a0 + (k + NS) * kStageRows;
                const uint32_t bytes = (uint32_t)(min((int64_t)kStageRows, a1 - r0) * 4);
                lab_t* sp = smem + s * 2 * kStageRows;
                mbar_expect_tx(&full[s], 2u * bytes);
                bulk_g2s(sp, src + r0, bytes, &full[s]);
                bulk_g2s(sp + kStageRows, dst + r0, bytes, &full[s]);
            }
        }
        for (int64_t r = max(a1, w.start) + tid; r < w.end; r += kBT) {
            lab_t u[1] = {src[r]}, v[1] = {dst[r]};
            wrote |= slice_rows<SM, 1>(L, sl, base, len, u, v);
        }
        __syncthreads();  // the next item overwrites the slice
    }
    if (__syncthreads_or(wrote) && threadIdx.x == 0) *flag = 1;
}

// First sweep from freshly initialised labels (L[x] = x for all x).
// Every chain is a single fixed point, so for any order h the operator on
// edge (u, v) is z = min(u, v) with targets u and v: only the cell max(u, v)
// can be lowered, to min(u, v).  Reading the start-of-sweep (identity)
// values instead of gathering them is a legal asynchronous interleaving, and
// the store is an atomic min (never loses a lowering), so the sweep needs
// NO label loads: one fire-and-forget red.global.min.u32 per edge.  In sync
// mode T is the shadow and the result is exactly the reference's sweep 1
// (shadow = element-wise min over all proposals).
template <int NV>
__global__ void __launch_bounds__(kThreads) k_sweep_first(const lab_t* __restrict__ src,
                                                          const lab_t* __restrict__ dst, int64_t m,
                                                          lab_t* T, int* __restrict__ flag) {
    const int64_t nvec = m >> 2;
    const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
    const uint4* __restrict__ d4 = reinterpret_cast<const uint4*>(dst);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool wrote = false;
    for (int64_t base = tid; base < nvec; base += stride * NV) {
        uint4 a[NV], b[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int64_t i = base + (int64_t)q * stride;
            a[q] = make_uint4(0, 0, 0, 0);
            b[q] = a[q];
            if (i < nvec) { a[q] = __ldcs(s4 + i); b[q] = __ldcs(d4 + i); }
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const lab_t u[4] = {a[q].x, a[q].y, a[q].z, a[q].w};
            const lab_t v[4] = {b[q].x, b[q].y, b[q].z, b[q].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (u[k] != v[k]) {
                    atomicMin(T + max(u[k], v[k]), min(u[k], v[k]));
                    wrote = true;
                }
            }
        }
    }
    for (int64_t e = (nvec << 2) + tid; e < m; e += stride) {
        const lab_t u = src[e], v = dst[e];
        if (u != v) { atomicMin(T + max(u, v), min(u, v)); wrote = true; }
    }
    if (__syncthreads_or(wrote) && threadIdx.x == 0) *flag = 1;
}

}  // namespace cck
