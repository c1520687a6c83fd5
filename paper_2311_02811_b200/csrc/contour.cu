// libcontour.so -- B200 (sm_100a) implementation of the Contour hot path behind
// the C-ABI declared in include/contour.h.
//
// The host driver below restates the reference driver loop run_contour
// (/root/reference/pkg/src/minmapcc/engine.py:248-328) over device kernels:
// labels live in HBM as uint32 (4n B), edges as packed uint32 SoA (8m B),
// each sweep is one kernel launch over all edges, and convergence is decided
// from a one-word device flag instead of an n-sized label diff.
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <thread>
#include <vector>

#include "contour.h"
#include "gen_rng.cuh"
#include "kernels.cuh"

using cck::lab_t;
using cck::kThreads;

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define CUDA_TRY(x)                                                                        \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            return fail(CC_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_),     \
                        __FILE__, __LINE__);                                               \
    } while (0)

#define CC_TRY(x)                \
    do {                         \
        int rc_ = (x);           \
        if (rc_ != CC_OK) return rc_; \
    } while (0)

// ------------------------------------------------------------------ kernels
namespace {

constexpr int kFlagWrote = 0;    // any lowering in the current sweep (ballot/OR)
constexpr int kFlagBad = 1;      // early check / staging range violation
constexpr int kFlagCompress = 2; // compress round changed something
constexpr int kFlagLe = 3;      // cc_verify: forest invariant violated
constexpr int kFlagCheck = 4;   // device-side early check failed (graph loop)
constexpr int kNumFlags = 5;

__global__ void k_iota(lab_t* L, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        L[i] = (lab_t)i;
}

__device__ __forceinline__ unsigned long long block_sum(unsigned long long x) {
    __shared__ unsigned long long part[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = x;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;  // valid in thread 0
}

// Synchronous commit (engine.py:309-311): count cells where the shadow was
// lowered, copy them into the labels.  Sets the wrote flag if any changed.
__global__ void __launch_bounds__(kThreads) k_commit(lab_t* L, const lab_t* S, int64_t n,
                                                     unsigned long long* count, int* flags) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const lab_t s = S[i];
        if (s != L[i]) { L[i] = s; ++c; }
    }
    c = block_sum(c);
    if (threadIdx.x == 0 && c) { atomicAdd(count, c); flags[kFlagWrote] = 1; }
}

// changed = count_nonzero(target != before) (engine.py:309), async mode.
__global__ void __launch_bounds__(kThreads) k_diff(const lab_t* L, const lab_t* B, int64_t n,
                                                   unsigned long long* count) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        c += (L[i] != B[i]);
    c = block_sum(c);
    if (threadIdx.x == 0 && c) atomicAdd(count, c);
}

// early_convergence_check (engine.py:331-348): idempotence, then agreement.
__global__ void k_check_idem(const lab_t* L, int64_t n, int* flags) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const lab_t l = L[i];
        bad |= (L[l] != l);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[kFlagBad] = 1;
}

__global__ void k_check_edges(const lab_t* __restrict__ src, const lab_t* __restrict__ dst,
                              int64_t m, const lab_t* L, int* flags) {
    if (*(volatile int*)&flags[kFlagBad]) return;  // idempotence already failed
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= (L[__ldcs(src + e)] != L[__ldcs(dst + e)]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[kFlagBad] = 1;
}

// The same check inside the graph loop (engine.py:318-320: run after every
// sweep that changed something).  Both kernels return at once when the sweep
// wrote nothing (the loop then stops on the change flag); the edge pass also
// returns when idempotence already failed, and polls the failure word every
// 16 iterations (one load per warp), so a failing check -- the common case
// before convergence -- costs a small fraction of a pass.
// Launched after the edge half (which fails fast before convergence), so it
// mostly returns at once; the CTA-wide skip decision is uniform (the flag can
// be set by another CTA meanwhile) because the pass ends in a barrier.
__global__ void __launch_bounds__(kThreads) k_gcheck_idem(const lab_t* __restrict__ L, int64_t n,
                                                          int* flags) {
    volatile int* vf = flags;
    if (__syncthreads_or(threadIdx.x == 0 && (!vf[kFlagWrote] || vf[kFlagCheck]))) return;
    bool bad = false;
    int it = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n && !bad;
         i += (int64_t)gridDim.x * blockDim.x) {
        if ((++it & 15) == 0 && vf[kFlagCheck]) break;
        const lab_t l = L[i];
        bad = (L[l] != l);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[kFlagCheck] = 1;
}

__global__ void __launch_bounds__(kThreads) k_gcheck_edges(const lab_t* __restrict__ src,
                                                           const lab_t* __restrict__ dst,
                                                           int64_t m, const lab_t* __restrict__ L,
                                                           int* flags) {
    volatile int* vf = flags;
    if (!vf[kFlagWrote] || vf[kFlagCheck]) return;
    const int64_t nvec = m >> 2;
    const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
    const uint4* __restrict__ d4 = reinterpret_cast<const uint4*>(dst);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int it = 0;
    for (int64_t i = tid; i < nvec; i += stride) {
        if ((++it & 15) == 0 && vf[kFlagCheck]) return;
        const uint4 a = __ldcs(s4 + i), b = __ldcs(d4 + i);
        const bool bad = (L[a.x] != L[b.x]) | (L[a.y] != L[b.y]) | (L[a.z] != L[b.z]) |
                         (L[a.w] != L[b.w]);
        if (bad) {
            vf[kFlagCheck] = 1;
            return;
        }
    }
    for (int64_t e = (nvec << 2) + tid; e < m; e += stride)
        if (L[src[e]] != L[dst[e]]) vf[kFlagCheck] = 1;
}

// Forest invariant L[x] <= x -- part of cc_verify.
__global__ void k_check_le(const lab_t* L, int64_t n, int* flags) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= ((int64_t)L[i] > i);
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[kFlagLe] = 1;
}

// Pointer-jumping compress L[v] = L[L[v]] (north-star step 4; the semantic
// model is normalize_labels, baselines.py:146-152).
// Four labels per thread per iteration (one uint4 load, four independent
// gathers): the pass is bound by the dependent, random L[L[x]] load, so ILP
// is what makes it fast.  Lowerings
// use red.min: L[L[x]] <= L[x] always, and a concurrent writer (a peer GPU's
// fused exchange) can never be overwritten by a larger value.
// gate != nullptr: return at once if *gate == 0 (the graph loop's shortcut
// after a sweep that wrote nothing, and its final pass after a loop that
// ended on a no-write order >= 2 sweep or a passed early check -- the labels
// are idempotent then).
__global__ void __launch_bounds__(kThreads) k_compress(lab_t* L, int64_t n, int* flags,
                                                       const int* gate = nullptr) {
    if (gate && *(volatile const int*)gate == 0) return;
    bool ch = false;
    const int64_t nv = n >> 2;
    const uint4* L4 = reinterpret_cast<const uint4*>(L);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t q = tid; q < nv; q += stride) {
        const uint4 l = L4[q];
        const lab_t a = L[l.x], b = L[l.y], c = L[l.z], d = L[l.w];
        lab_t* p = L + 4 * q;
        if (a != l.x) { atomicMin(p + 0, a); ch = true; }
        if (b != l.y) { atomicMin(p + 1, b); ch = true; }
        if (c != l.z) { atomicMin(p + 2, c); ch = true; }
        if (d != l.w) { atomicMin(p + 3, d); ch = true; }
    }
    for (int64_t i = (nv << 2) + tid; i < n; i += stride) {
        const lab_t l = L[i];
        const lab_t ll = L[l];
        if (ll != l) { atomicMin(L + i, ll); ch = true; }
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0) flags[kFlagCompress] = 1;
}

// labels[n] = wrote ? 0 : 1, flag cleared: folds "did any rank write" into
// an allreduce-min over n+1 elements.
__global__ void k_fold(lab_t* L, int64_t n, int* flags, int first) {
    const lab_t f = flags[kFlagWrote] ? 0u : 1u;
    L[n] = first ? f : min(L[n], f);
    flags[kFlagWrote] = 0;
}

// Staging: (m,2) AoS int32/int64 rows -> packed uint32 SoA + range check
// (graph.py:73-79).
template <typename T>
__global__ void k_stage(const T* __restrict__ aos, int64_t rows, int64_t n, lab_t* src, lab_t* dst,
                        int* flags) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows;
         e += (int64_t)gridDim.x * blockDim.x) {
        const T a = aos[2 * e], b = aos[2 * e + 1];
        const bool out = (a < 0) | (b < 0) | ((int64_t)a >= n) | ((int64_t)b >= n);
        bad |= out;
        // an out-of-range row fails the staging call; until then it is an
        // inert self loop, so a sweep streamed behind the copy never indexes
        // outside the label array
        src[e] = out ? 0u : (lab_t)a;
        dst[e] = out ? 0u : (lab_t)b;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[kFlagBad] = 1;
}

// Layout 3 keys: ((dst bucket * runs + run) << sbits) | src, where run is
// the row's original position in `runs` equal slices -> bucket-major, then
// `runs` src-sorted runs per bucket.
// run_major: ((run * nb + dst bucket) << sbits) | src instead -> run-major.
template <typename K>
__global__ void k_make_keys(const lab_t* __restrict__ src, const lab_t* __restrict__ dst,
                            int64_t m, int bshift, int sbits, int runs, int64_t nb,
                            int run_major, K* keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const K run = (K)((i * runs) / m);
        const K b = (K)(dst[i] >> bshift);
        const K g = run_major ? run * (K)nb + b : b * (K)runs + run;
        keys[i] = (g << sbits) | (K)src[i];
    }
}

template <typename K>
__global__ void k_unkey(const K* __restrict__ keys, int64_t m, K mask, lab_t* src) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        src[i] = (lab_t)(keys[i] & mask);
}

// starts[b] = first row whose bucket >= b (lower bound on the sorted keys).
template <typename K>
__global__ void k_bucket_starts(const K* __restrict__ keys, int64_t m, int64_t nb, int sbits,
                                int runs, int64_t* starts) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
         b += (int64_t)gridDim.x * blockDim.x) {
        const K target = ((K)b * (K)runs) << sbits;
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        starts[b] = lo;
    }
}

// Layout 4 partition: rows -> P = ceil(n / 2^shift) dst buckets (P <= 1024).
constexpr int kMaxTiles = 1024;
constexpr int64_t kPartRows = 1 << 16;  // rows per partition block

__global__ void __launch_bounds__(kThreads) k_tile_hist(const lab_t* __restrict__ dst, int64_t m,
                                                        int shift, int P,
                                                        unsigned long long* counts) {
    __shared__ unsigned int h[kMaxTiles];
    for (int i = threadIdx.x; i < P; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * kPartRows;
    const int64_t hi = min(lo + kPartRows, m);
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) atomicAdd(&h[dst[e] >> shift], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        if (h[i]) atomicAdd(counts + i, (unsigned long long)h[i]);
}

// Each block reserves one slice per bucket (one global atomic per bucket),
// then scatters its rows into the reservations.
__global__ void __launch_bounds__(kThreads) k_tile_scatter(const lab_t* __restrict__ src,
                                                           const lab_t* __restrict__ dst,
                                                           int64_t m, int shift, int P,
                                                           unsigned long long* cursor,
                                                           lab_t* osrc, lab_t* odst) {
    __shared__ unsigned int h[kMaxTiles];
    __shared__ unsigned long long basep[kMaxTiles];
    for (int i = threadIdx.x; i < P; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * kPartRows;
    const int64_t hi = min(lo + kPartRows, m);
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) atomicAdd(&h[dst[e] >> shift], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        basep[i] = h[i] ? atomicAdd(cursor + i, (unsigned long long)h[i]) : 0ull;
        h[i] = 0;
    }
    __syncthreads();
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        const lab_t d = dst[e];
        const int b = (int)(d >> shift);
        const unsigned long long pos = basep[b] + atomicAdd(&h[b], 1u);
        osrc[pos] = src[e];
        odst[pos] = d;
    }
}

// ---- FastSV baseline (baselines.py:81-131) ------------
// One synchronous iteration = hooking proposals from every edge into a copy
// of the parent array by atomic min (order-independent, so per-iteration
// results equal the reference's numpy np.minimum.at exactly), then
// shortcutting against the grandparents.
__global__ void __launch_bounds__(kThreads) k_fastsv_hook(const lab_t* __restrict__ src,
                                                          const lab_t* __restrict__ dst,
                                                          int64_t m, const lab_t* P,
                                                          const lab_t* G, lab_t* N) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const lab_t w = __ldcs(src + e), v = __ldcs(dst + e);
        const lab_t gw = G[w], gv = G[v], pw = P[w], pv = P[v];
        // N starts as a copy of P and only decreases, so a proposal that is
        // not below the target's P value is a no-op; G = P[P] gives P[pw] = gw
        // and P[pv] = gv for free.  Skipping provable no-ops keeps the result
        // (the min over all proposals) exact and keeps every edge from
        // serialising on the hot root cells.
        if (gv < gw) atomicMin(N + pw, gv);  // stochastic hooking (baselines.py:109-110)
        if (gw < gv) atomicMin(N + pv, gw);
        if (gv < pw) atomicMin(N + w, gv);   // aggressive hooking (baselines.py:111-112)
        if (gw < pv) atomicMin(N + v, gw);
    }
}

// N = min(N, G) (shortcutting, :113); count N != P (:114).
__global__ void __launch_bounds__(kThreads) k_fastsv_shortcut(lab_t* N, const lab_t* G,
                                                              const lab_t* P, int64_t n,
                                                              unsigned long long* count) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const lab_t x = min(N[i], G[i]);
        N[i] = x;
        c += (x != P[i]);
    }
    c = block_sum(c);
    if (threadIdx.x == 0 && c) atomicAdd(count, c);
}

// G2 = P[P] (:116); flag if G2 != G (:121).
__global__ void __launch_bounds__(kThreads) k_fastsv_grand(const lab_t* P, const lab_t* G,
                                                           lab_t* G2, int64_t n, int* flags) {
    bool diff = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const lab_t g = P[P[i]];
        G2[i] = g;
        diff |= (g != G[i]);
    }
    if (__syncthreads_or(diff) && threadIdx.x == 0) flags[kFlagBad] = 1;
}

__global__ void k_widen(const lab_t* L, int64_t n, int64_t* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)L[i];
}

// Caller labels (int64 or int32/uint32 as T) -> device labels, with the
// range check 0 <= x < n (kFlagBad).
template <typename T>
__global__ void k_labels_in(const T* in, int64_t n, lab_t* L, int* flags) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const T x = in[i];
        const bool out = (int64_t)x < 0 || (int64_t)x >= n;
        bad |= out;
        L[i] = out ? (lab_t)i : (lab_t)x;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[kFlagBad] = 1;
}

__global__ void k_from64(const int64_t* in, int64_t n, lab_t* L) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        L[i] = (lab_t)in[i];
}

// Single-edge operator through the same device routines as the sweeps.
__global__ void k_single_edge(const lab_t* R, lab_t* T, lab_t w, lab_t v, int order, int inplace,
                              int* changed) {
    constexpr int P = cck::kStorePlain, A = cck::kStoreRed;
    if (inplace) {
        bool c;
        if (order == 1) c = cck::single_edge<1, P>(T, T, w, v, order);
        else if (order == 2) c = cck::single_edge<2, P>(T, T, w, v, order);
        else c = cck::single_edge<0, P>(T, T, w, v, order);
        *changed = c;
    } else {  // sync form: atomic lowering of a separate target (host diffs it)
        if (order == 1) cck::single_edge<1, A>(R, T, w, v, order);
        else if (order == 2) cck::single_edge<2, A>(R, T, w, v, order);
        else cck::single_edge<0, A>(R, T, w, v, order);
    }
}

// ---- device-side convergence loop (CUDA graph with a conditional WHILE node)
// Body per iteration: order-guarded k_sweep launches -> k_loop_control,
// which reads and clears the ballot/OR flag, records (wrote, globaltimer),
// and sets the WHILE condition.  No host round trip between sweeps.
struct LoopState {
    long long sweep;      // sweeps completed
    int order;            // operator order of the next sweep
    int converged;        // last sweep lowered nothing
    int capped;           // sweep cap reached while still changing
    int by_check;         // stopped by the early check (not the change flag)
    int need_compress;    // the final pointer-jumping pass can change something
    int order_first;      // layout 5 guards: the next sweep's order if it is sweep 1, else 0
    int order_rest;       // ... if it is a later sweep, else 0
    unsigned long long t0;
};
struct SweepRec {
    int wrote;
    int pad;
    unsigned long long t;
};
constexpr int kMaxRec = 4096;
constexpr int kEagerRec = 64;  // records copied back with every graph run

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int order_for_dev(const cc_schedule& s, long long sweep) {
    switch (s.variant) {  // engine.py:61-74
        case CC_VAR_C2:
        case CC_VAR_CSYN: return 2;
        case CC_VAR_C1: return 1;
        case CC_VAR_CM: return s.high_order;
        case CC_VAR_C11MM: return sweep <= s.warmup ? 1 : s.high_order;
        default: return (sweep % 2 == 1) ? 1 : s.high_order;
    }
}

// start: sweeps already done before the loop (1 after cc_run_host's
// streamed first sweep, else 0).
__global__ void k_loop_init(LoopState* st, int* flags, cc_schedule s, long long start) {
    st->sweep = start;
    st->order = order_for_dev(s, start + 1);
    st->order_first = start == 0 ? st->order : 0;
    st->order_rest = start == 0 ? 0 : st->order;
    st->converged = 0;
    st->capped = 0;
    st->by_check = 0;
    st->need_compress = 1;
    flags[kFlagWrote] = 0;
    flags[kFlagCheck] = 0;
    flags[kFlagCompress] = 0;
    st->t0 = globaltimer();
}

__global__ void k_loop_control(LoopState* st, SweepRec* rec, int* flags, cc_schedule s,
                               long long cap, int check, cudaGraphConditionalHandle h) {
    const int wrote = flags[kFlagWrote];
    const int bad = flags[kFlagCheck];
    flags[kFlagWrote] = 0;
    flags[kFlagCheck] = 0;
    flags[kFlagCompress] = 0;  // only the post-loop compress pass reports to the host
    const long long k = ++st->sweep;
    if (k <= kMaxRec) {
        rec[k - 1].wrote = wrote;
        rec[k - 1].t = globaltimer();
    }
    if (!wrote) {
        st->converged = 1;
        // after a no-write sweep of any order every edge has L[u] == L[v], so
        // each component holds one common value, a member whose label is
        // itself: the labels are final
        st->need_compress = 0;
        cudaGraphSetConditional(h, 0);
    } else if (check && !bad) {  // engine.py:318-320
        st->converged = 1;
        st->by_check = 1;
        st->need_compress = 0;  // the check proved L[L[x]] == L[x]
        cudaGraphSetConditional(h, 0);
    } else if (k >= cap) {
        st->capped = 1;
        cudaGraphSetConditional(h, 0);
    } else {
        st->order = order_for_dev(s, k + 1);
        st->order_first = 0;
        st->order_rest = st->order;
        cudaGraphSetConditional(h, 1);
    }
}

// RMAT rows [lo, hi) of the symmetrised list (rows >= M are (v,u) of row-M).
__global__ void k_gen_rmat(ccgen::RmatParams rp, ccgen::Perm pm, int permute, int64_t M,
                           int symmetrize, int64_t lo, int64_t hi, lab_t* src, lab_t* dst) {
    for (int64_t r = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < hi;
         r += (int64_t)gridDim.x * blockDim.x) {
        const bool back = symmetrize && r >= M;
        const uint64_t i = back ? (uint64_t)(r - M) : (uint64_t)r;
        uint64_t u, v;
        ccgen::rmat_edge(rp, i, u, v);
        if (permute) { u = ccgen::perm_apply(pm, u); v = ccgen::perm_apply(pm, v); }
        src[r - lo] = (lab_t)(back ? v : u);
        dst[r - lo] = (lab_t)(back ? u : v);
    }
}

}  // namespace

// ------------------------------------------------------------------ context
struct cc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    bool own_stream = false;
    int sm_count = 148;
    int64_t n = 0, m = 0;
    lab_t* src = nullptr;
    lab_t* dst = nullptr;
    int64_t edge_cap = 0;
    bool own_edges = false;
    lab_t* labels = nullptr;  // n + 1
    int64_t label_cap = 0;
    bool own_labels = false;
    int64_t* wide = nullptr;  // cached int64 label buffer for copy_out
    int64_t wide_cap = 0;
    lab_t* shadow = nullptr;
    lab_t* before = nullptr;
    int64_t aux_cap = 0;
    int* dflags = nullptr;
    unsigned long long* dcount = nullptr;
    int* hflags = nullptr;                // pinned mirror of dflags
    unsigned long long* hcount = nullptr; // pinned
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs = nullptr, eve = nullptr;
    int store_mode_plain = cck::kStorePlain;  // async, Schedule.atomic == False
    int store_mode_atomic = cck::kStoreCheckRed;  // async, Schedule.atomic == True
    int64_t sort_chunk = (int64_t)1 << 23;    // rows per chunk (staging, layout mode 2)
    int layout = 0;                           // current row order (cc_reorder_edges modes)
    int bucket_shift = 15;                    // layout 3: B = 2^shift labels per bucket
    int tile_shift = 24;                      // layout 4: 2^shift labels (64 MB) per L2 window
    int shortcut = 1;  // pointer-jumping passes after every async sweep (fast path)
    int tile_split = 2;  // layout 4: independently sorted runs per L2 window
    int bucket_nosmem = 0;  // layout 3 experiment: gather dst labels from global memory
    int sweep_variant = 12;  // order-2 kernel tuning variant (launch_o2): 12 = auto
    cck::PeerSet peers = {};  // peer label replicas for the fused sweep + exchange
    int64_t item_rows = (int64_t)1 << 18;     // layout 3: rows per work item
    int bucket_threads = 1024;
    int bucket_pipe = 2;  // layout 3/5 kernel (launch_bucketed): lean + edge prefetch
    int item_order = 0;   // layout 3: 0 bucket-major items, 1 run-major (see reorder_bucketed)
    cck::BucketItem* items = nullptr;         // layout 3/5 work items (device)
    lab_t* bsrc = nullptr;                    // layout 5: dst-bucketed copy of the rows
    lab_t* bdst = nullptr;
    int64_t bcap = 0;
    int n_items = 0;
    int stage_layout = 0;                     // layout applied by cc_stage_edges*
    lab_t* sort_ks = nullptr;                 // cached radix-sort scratch
    lab_t* sort_vs = nullptr;
    void* sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int64_t sort_rows_cap = 0;
    void* stage_buf[2] = {nullptr, nullptr};  // cached H2D staging buffers
    size_t stage_buf_bytes = 0;
    cudaEvent_t copied[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    cudaEvent_t spec_ready = nullptr, spec_done = nullptr;  // speculative label read-back
    // graph-captured convergence loop (built lazily, rebuilt when its key changes)
    cudaStream_t cap_stream = nullptr, body_stream = nullptr;
    cudaGraph_t loop_graph = nullptr;
    cudaGraphExec_t loop_exec = nullptr;
    LoopState* dstate = nullptr;
    SweepRec* drec = nullptr;
    LoopState* hstate = nullptr;  // pinned
    SweepRec* hrec = nullptr;     // pinned
    struct {
        const void *src, *dst, *labels;
        int64_t m, n, cap;
        cc_schedule s;
        int sm;
        int shortcut;
        int layout;
        int check;
        const void* items;
        int n_items;
        int resume;
        const void* bsrc;
    } loop_key = {};
    std::mutex mu;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int grid_for(const cc_ctx* c, int64_t work, int per_sm = 8) {
    int64_t b = (work + kThreads - 1) / kThreads;
    int64_t cap = (int64_t)c->sm_count * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// Launch context of one sweep: the stream, for graph capture the device
// word holding the order (nullptr: use the host value), and optionally a row
// window [off, off + rows) of the staged edges (rows < 0: all m rows; the
// flat k_sweep path only -- the streamed first sweep of cc_run_host).
struct SweepLaunch {
    cudaStream_t stream;
    const int* d_order;
    int64_t off = 0;
    int64_t rows = -1;
};

// Rows the bucketed kernels walk: the rows themselves (layout 3) or the
// dst-bucketed copy kept next to the chunk-sorted rows (layout 5).
const lab_t* bucket_src(const cc_ctx* c) { return c->layout == 5 ? c->bsrc : c->src; }
const lab_t* bucket_dst(const cc_ctx* c) { return c->layout == 5 ? c->bdst : c->dst; }
bool has_buckets(const cc_ctx* c) { return (c->layout == 3 || c->layout == 5) && c->items; }

template <int OK, int SM, int NV, int MINB = 1>
int launch_sweep_t(cc_ctx* c, const lab_t* R, lab_t* T, int order, SweepLaunch sl) {
    static int occ = 0;
    if (occ == 0) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cck::k_sweep<OK, SM, NV, MINB>,
                                                      kThreads, 0);
        occ = o > 0 ? o : 1;
    }
    const int64_t m = sl.rows < 0 ? c->m : sl.rows;
    const int64_t units = (m + 4 * NV - 1) / (4 * NV);
    const int blocks = grid_for(c, units, occ);
    cck::k_sweep<OK, SM, NV, MINB><<<blocks, kThreads, 0, sl.stream>>>(
        c->src + sl.off, c->dst + sl.off, m, R, T, order, c->dflags + kFlagWrote, sl.d_order);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

// H: cck::kHint* cache-hint bits (order 2 only).
template <int OK, int NV, int MINB = 1, int H = 0>
int launch_store_mode(cc_ctx* c, const lab_t* R, lab_t* T, int order, int sm, SweepLaunch sl) {
    switch (sm) {
        case cck::kStorePlain:
            return launch_sweep_t<OK, cck::kStorePlain | H, NV, MINB>(c, R, T, order, sl);
        case cck::kStoreRed:
            return launch_sweep_t<OK, cck::kStoreRed | H, NV, MINB>(c, R, T, order, sl);
        case cck::kStoreCheckPlain:
            return launch_sweep_t<OK, cck::kStoreCheckPlain | H, NV, MINB>(c, R, T, order, sl);
        case cck::kStoreCheckAllRed:
            return launch_sweep_t<OK, cck::kStoreCheckAllRed | H, NV, MINB>(c, R, T, order, sl);
        default:
            return launch_sweep_t<OK, cck::kStoreCheckRed | H, NV, MINB>(c, R, T, order, sl);
    }
}

// The order-2 sweep in one of its tuning variants (CC_OPT_SWEEP_VARIANT):
// 0 = 8 rows/thread (default), 1 = 4 rows/thread, 2 = 8 rows/thread capped
// at 64 registers (4 blocks/SM), 3 = 16 rows/thread.
template <int SM>
int launch_o2_peers(cc_ctx* c, lab_t* L, SweepLaunch sl) {
    static int occ = 0;
    if (occ == 0) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cck::k_sweep_o2_peers<SM>, kThreads, 0);
        occ = o > 0 ? o : 1;
    }
    const int blocks = grid_for(c, (c->m + 3) / 4, occ);
    cck::k_sweep_o2_peers<SM><<<blocks, kThreads, 0, sl.stream>>>(c->src, c->dst, c->m, L,
                                                                  c->peers, c->dflags + kFlagWrote);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

int launch_o2(cc_ctx* c, const lab_t* R, lab_t* T, int sm, SweepLaunch sl) {
    if (c->peers.n > 0 && R == T && !sl.d_order) {  // fused sweep + peer exchange (async only)
        switch (sm) {
            case cck::kStorePlain: return launch_o2_peers<cck::kStorePlain>(c, T, sl);
            case cck::kStoreRed: return launch_o2_peers<cck::kStoreRed>(c, T, sl);
            case cck::kStoreCheckPlain: return launch_o2_peers<cck::kStoreCheckPlain>(c, T, sl);
            default: return launch_o2_peers<cck::kStoreCheckRed>(c, T, sl);
        }
    }
    // 12 (auto): on L2-window tiles the cache hints of variant 11 -- there the
    // edge stream and the src gathers would evict the tile's dst window from
    // L2 (RMAT-28: 84 ms vs 122 ms per run with tile split 2, measured); for a
    // sparse graph (m < 4n, the forest: DRAM-latency-bound random gathers,
    // 1.7 % issue) with 16 rows per thread (variant 13: 682 vs 773 ms; the
    // same on RMAT-28, L2-request-bound, costs 3.7x); elsewhere variant 1
    const int variant = c->sweep_variant != 12 ? c->sweep_variant
                        : c->layout != 4       ? 1
                        : c->m < 4 * c->n      ? 13
                                               : 11;
    switch (variant) {
        case 1: return launch_store_mode<2, 1>(c, R, T, 2, sm, sl);
        case 2: return launch_store_mode<2, 2, 4>(c, R, T, 2, sm, sl);
        case 3: return launch_store_mode<2, 4>(c, R, T, 2, sm, sl);
        case 4: return launch_store_mode<2, 1, 6>(c, R, T, 2, sm, sl);
        case 5: return launch_store_mode<2, 1, 8>(c, R, T, 2, sm, sl);
        case 6: return launch_store_mode<2, 1, 1, cck::kHintSrcStream>(c, R, T, 2, sm, sl);
        case 7:
            return launch_store_mode<2, 1, 1, cck::kHintSrcStream | cck::kHintDstKeep>(c, R, T,
                                                                                       2, sm, sl);
        case 8: return launch_store_mode<2, 1, 1, cck::kHintDstKeep>(c, R, T, 2, sm, sl);
        case 9: return launch_store_mode<2, 1, 1, cck::kHintEdgeFirst>(c, R, T, 2, sm, sl);
        case 10:
            return launch_store_mode<2, 1, 1,
                                     cck::kHintEdgeFirst | cck::kHintDstKeep | cck::kHintSrcKeep>(
                c, R, T, 2, sm, sl);
        case 11:
            return launch_store_mode<2, 1, 1, cck::kHintEdgeFirst | cck::kHintDstKeep>(c, R, T, 2,
                                                                                       sm, sl);
        case 13:
            return launch_store_mode<2, 4, 1, cck::kHintEdgeFirst | cck::kHintDstKeep>(c, R, T, 2,
                                                                                       sm, sl);
        case 14:
            return launch_store_mode<2, 4, 2, cck::kHintEdgeFirst | cck::kHintDstKeep>(c, R, T, 2,
                                                                                       sm, sl);
        case 15:
            return launch_store_mode<2, 2, 3, cck::kHintEdgeFirst | cck::kHintDstKeep>(c, R, T, 2,
                                                                                       sm, sl);
        case 16: return launch_store_mode<2, 1, 1, cck::kHintDstCg>(c, R, T, 2, sm, sl);
        case 17:
            return launch_store_mode<2, 1, 1, cck::kHintDstCg | cck::kHintEdgeFirst>(c, R, T, 2,
                                                                                     sm, sl);
        default: return launch_store_mode<2, 2>(c, R, T, 2, sm, sl);
    }
}

// Order-specialised sweep: order 1 and 2 get unrolled batch kernels, any
// other order the buffered chain walker.
int launch_order_sl(cc_ctx* c, const lab_t* R, lab_t* T, int order, int sm, SweepLaunch sl) {
    if (order == 1) return launch_store_mode<1, 2>(c, R, T, order, sm, sl);
    if (order == 2) return launch_o2(c, R, T, sm, sl);
    return launch_store_mode<0, 1>(c, R, T, order, sm, sl);
}

int launch_order(cc_ctx* c, const lab_t* R, lab_t* T, int order, int sm) {
    return launch_order_sl(c, R, T, order, sm, SweepLaunch{c->stream, nullptr});
}

int ensure_aux(cc_ctx* c, bool need_shadow, bool need_before) {
    if (c->aux_cap < c->n) {
        if (c->shadow) cudaFree(c->shadow);
        if (c->before) cudaFree(c->before);
        c->shadow = c->before = nullptr;
        c->aux_cap = c->n;
    }
    if (need_shadow && !c->shadow) CUDA_TRY(cudaMalloc(&c->shadow, sizeof(lab_t) * (c->n + 1)));
    if (need_before && !c->before) CUDA_TRY(cudaMalloc(&c->before, sizeof(lab_t) * (c->n + 1)));
    return CC_OK;
}

int ensure_labels(cc_ctx* c) {
    if (c->labels && (c->label_cap >= c->n + 1 || !c->own_labels)) return CC_OK;
    if (c->labels && c->own_labels) cudaFree(c->labels);
    CUDA_TRY(cudaMalloc(&c->labels, sizeof(lab_t) * (c->n + 1)));
    c->label_cap = c->n + 1;
    c->own_labels = true;
    return CC_OK;
}

int ensure_edges(cc_ctx* c, int64_t m) {
    if (c->own_edges && c->edge_cap >= m && c->src) return CC_OK;
    if (c->own_edges) {
        if (c->src) cudaFree(c->src);
        if (c->dst) cudaFree(c->dst);
    }
    c->src = c->dst = nullptr;
    c->edge_cap = 0;
    const int64_t cap = m > 0 ? m : 4;
    CUDA_TRY(cudaMalloc(&c->src, sizeof(lab_t) * cap));
    CUDA_TRY(cudaMalloc(&c->dst, sizeof(lab_t) * cap));
    c->edge_cap = cap;
    c->own_edges = true;
    return CC_OK;
}

int set_graph(cc_ctx* c, int64_t m, int64_t n) {
    if (n < 0 || m < 0) return fail(CC_EINVAL, "vertex and edge counts must be non-negative");
    if (n > (int64_t)0xFFFFFFFFll)
        return fail(CC_EINVAL, "n=%lld exceeds the uint32 vertex-ID range", (long long)n);
    if (m > 0 && n == 0) return fail(CC_EINVAL, "edge endpoint out of range: n=0");
    c->n = n;
    c->m = m;
    c->layout = 0;  // a new edge set: any bucketed work items are stale
    c->n_items = 0;
    // the captured loop stays valid: its key (build_loop) holds every value
    // the capture baked in, so restaging a same-shaped graph into the same
    // buffers (the end-to-end path) reuses it
    return ensure_labels(c);
}

int read_flags(cc_ctx* c) {
    CUDA_TRY(cudaMemcpyAsync(c->hflags, c->dflags, sizeof(int) * kNumFlags,
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->hcount, c->dcount, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return CC_OK;
}

int order_for(const cc_schedule* s, int64_t sweep) {  // engine.py:61-74
    switch (s->variant) {
        case CC_VAR_C2:
        case CC_VAR_CSYN: return 2;
        case CC_VAR_C1: return 1;
        case CC_VAR_CM: return s->high_order;
        case CC_VAR_C11MM: return sweep <= s->warmup ? 1 : s->high_order;
        case CC_VAR_C1M1M: return (sweep % 2 == 1) ? 1 : s->high_order;
    }
    return -1;
}

// Enqueue one sweep; flag word (and count for sync) left on device.
template <int SM, int U>
int launch_bucketed_t(cc_ctx* c, SweepLaunch sl) {
    const size_t smem = sizeof(lab_t) * ((size_t)1 << c->bucket_shift);
    static size_t smem_set = 0;
    if (smem_set != smem) {
        CUDA_TRY(cudaFuncSetAttribute(cck::k_sweep_bucketed<SM, U>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cck::k_sweep_bucketed<SM, U>,
                                                  c->bucket_threads, smem);
    if (occ < 1) occ = 1;
    const int blocks = std::min<int64_t>(c->n_items, (int64_t)c->sm_count * occ);
    cck::k_sweep_bucketed<SM, U><<<std::max(blocks, 1), c->bucket_threads, smem, sl.stream>>>(
        bucket_src(c), bucket_dst(c), c->labels, c->items, c->n_items, c->dflags + kFlagWrote,
        sl.d_order);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

template <int U>
int launch_bucketed_u(cc_ctx* c, int sm, SweepLaunch sl) {
    switch (sm) {
        case cck::kStorePlain: return launch_bucketed_t<cck::kStorePlain, U>(c, sl);
        case cck::kStoreRed: return launch_bucketed_t<cck::kStoreRed, U>(c, sl);
        case cck::kStoreCheckPlain: return launch_bucketed_t<cck::kStoreCheckPlain, U>(c, sl);
        default: return launch_bucketed_t<cck::kStoreCheckRed, U>(c, sl);
    }
}

constexpr int kCheckNV = 4;  // 16 rows per thread per iteration of the slice check (8 spills)

int launch_check_slice(cc_ctx* c, cudaStream_t st) {
    const size_t smem = sizeof(lab_t) * ((size_t)1 << c->bucket_shift);
    static size_t smem_set = 0;
    if (smem_set != smem) {
        CUDA_TRY(cudaFuncSetAttribute(cck::k_check_slice<kCheckNV>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    const int blocks = (int)std::min<int64_t>(c->n_items, (int64_t)c->sm_count);
    cck::k_check_slice<kCheckNV><<<std::max(blocks, 1), cck::kBT, smem, st>>>(
        bucket_src(c), bucket_dst(c), c->labels, c->items, c->n_items, c->dflags, kFlagWrote,
        kFlagCheck);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

template <int SM, int NS>
int launch_bucketed_pipe_t(cc_ctx* c, SweepLaunch sl) {
    const size_t smem = sizeof(lab_t) * ((size_t)NS * 2 * cck::kStageRows +
                                         ((size_t)1 << c->bucket_shift));
    static size_t smem_set = 0;
    if (smem_set != smem) {
        CUDA_TRY(cudaFuncSetAttribute(cck::k_sweep_bucketed_tma<SM, NS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    const int blocks = (int)std::min<int64_t>(c->n_items, (int64_t)c->sm_count);
    cck::k_sweep_bucketed_tma<SM, NS><<<std::max(blocks, 1), cck::kBT, smem, sl.stream>>>(
        bucket_src(c), bucket_dst(c), c->labels, c->items, c->n_items, c->dflags + kFlagWrote,
        sl.d_order);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

template <int NS>
int launch_bucketed_pipe(cc_ctx* c, int sm, SweepLaunch sl) {
    switch (sm) {
        case cck::kStorePlain: return launch_bucketed_pipe_t<cck::kStorePlain, NS>(c, sl);
        case cck::kStoreRed: return launch_bucketed_pipe_t<cck::kStoreRed, NS>(c, sl);
        case cck::kStoreCheckPlain: return launch_bucketed_pipe_t<cck::kStoreCheckPlain, NS>(c, sl);
        default: return launch_bucketed_pipe_t<cck::kStoreCheckRed, NS>(c, sl);
    }
}

// PF: 0 lean, 1 lean + edge prefetch
template <int SM, int PF>
int launch_slice_t(cc_ctx* c, SweepLaunch sl) {
    const size_t smem = sizeof(lab_t) * ((size_t)1 << c->bucket_shift);
    auto kern = cck::k_sweep_slice<SM, PF == 1>;
    static size_t smem_set = 0;
    if (smem_set != smem) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        smem_set = smem;
    }
    const int blocks = (int)std::min<int64_t>(c->n_items, (int64_t)c->sm_count);
    kern<<<std::max(blocks, 1), cck::kBT, smem, sl.stream>>>(
        bucket_src(c), bucket_dst(c), c->labels, c->items, c->n_items, c->dflags + kFlagWrote,
        sl.d_order);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

template <int PF>
int launch_slice(cc_ctx* c, int sm, SweepLaunch sl) {
    switch (sm) {
        case cck::kStorePlain: return launch_slice_t<cck::kStorePlain, PF>(c, sl);
        case cck::kStoreRed: return launch_slice_t<cck::kStoreRed, PF>(c, sl);
        case cck::kStoreCheckPlain: return launch_slice_t<cck::kStoreCheckPlain, PF>(c, sl);
        default: return launch_slice_t<cck::kStoreCheckRed, PF>(c, sl);
    }
}

// bucket_pipe (CC_OPT_BUCKET_PIPE): 1 lean slice kernel, 2 lean + edge
// prefetch, 3 bulk-copy pipelined kernel; 0 the general kernel with
// U = 4 rows per thread at up to 1024 threads, or 8 at up to 512.
int launch_bucketed(cc_ctx* c, int sm, SweepLaunch sl) {
    if (c->bucket_pipe > 0 && !c->bucket_nosmem) {
        if (c->bucket_pipe == 1) return launch_slice<0>(c, sm, sl);
        if (c->bucket_pipe == 2) return launch_slice<1>(c, sm, sl);
        return launch_bucketed_pipe<3>(c, sm, sl);
    }
    return c->bucket_threads > 512 ? launch_bucketed_u<1>(c, sm, sl)
                                   : launch_bucketed_u<2>(c, sm, sl);
}

int launch_first(cc_ctx* c, lab_t* T) {
    static int occ = 0;
    if (occ == 0) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, cck::k_sweep_first<2>, kThreads, 0);
        occ = o > 0 ? o : 1;
    }
    const int64_t units = (c->m + 7) / 8;
    cck::k_sweep_first<2><<<grid_for(c, units, occ), kThreads, 0, c->stream>>>(
        c->src, c->dst, c->m, T, c->dflags + kFlagWrote);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

// first: labels are the identity (sweep 1 after init) -> load-free scatter.
// sweep_no: 1-based sweep index (layout 5 runs sweep 1 on the chunk-sorted
// rows and later order-2 sweeps on the bucketed copy); 0 = unknown.
int enqueue_sweep(cc_ctx* c, int order, int sync, int atomic, bool count_changes,
                  bool first = false, int64_t sweep_no = 0) {
    if (order < 1) return fail(CC_EINVAL, "operator order must be >= 1");
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 0, sizeof(int), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dcount, 0, sizeof(unsigned long long), c->stream));
    if (c->m == 0) return CC_OK;
    if (sync) {
        CC_TRY(ensure_aux(c, true, false));
        const lab_t* R = c->labels;
        lab_t* T = c->shadow;
        int rc = first ? launch_first(c, T)
                       : launch_order(c, R, T, order, cck::kStoreCheckAllRed);
        if (rc) return rc;
        CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 0, sizeof(int), c->stream));
        k_commit<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->shadow, c->n,
                                                                c->dcount, c->dflags);
        CUDA_TRY(cudaGetLastError());
        return CC_OK;
    }
    if (count_changes) {
        CC_TRY(ensure_aux(c, false, true));
        CUDA_TRY(cudaMemcpyAsync(c->before, c->labels, sizeof(lab_t) * c->n,
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    lab_t* L = c->labels;
    const int sm = atomic ? c->store_mode_atomic : c->store_mode_plain;
    int rc;
    if (first) {
        rc = launch_first(c, L);
    } else if (order == 2 && has_buckets(c) && (c->layout == 3 || sweep_no > 1)) {
        rc = launch_bucketed(c, sm, SweepLaunch{c->stream, nullptr});
    } else {
        rc = launch_order(c, L, L, order, sm);
    }
    if (rc) return rc;
    if (count_changes) {
        k_diff<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->before, c->n,
                                                              c->dcount);
        CUDA_TRY(cudaGetLastError());
    }
    return CC_OK;
}

int enqueue_init(cc_ctx* c, bool sync) {
    if (c->n == 0) return CC_OK;
    k_iota<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n);
    CUDA_TRY(cudaGetLastError());
    if (sync) {
        CC_TRY(ensure_aux(c, true, false));
        CUDA_TRY(cudaMemcpyAsync(c->shadow, c->labels, sizeof(lab_t) * c->n,
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    return CC_OK;
}

int early_check(cc_ctx* c, int* ok) {  // engine.py:331-348
    if (c->n == 0) { *ok = 1; return CC_OK; }
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
    k_check_idem<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n, c->dflags);
    CUDA_TRY(cudaGetLastError());
    if (c->m > 0) {
        k_check_edges<<<grid_for(c, c->m), kThreads, 0, c->stream>>>(c->src, c->dst, c->m,
                                                                     c->labels, c->dflags);
        CUDA_TRY(cudaGetLastError());
    }
    CC_TRY(read_flags(c));
    *ok = c->hflags[kFlagBad] == 0;
    return CC_OK;
}

int compress(cc_ctx* c, int* rounds) {
    int r = 0;
    if (c->n > 0) {
        for (int it = 0; it < 70; ++it) {
            CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagCompress, 0, sizeof(int), c->stream));
            k_compress<<<grid_for(c, (c->n + 3) / 4), kThreads, 0, c->stream>>>(c->labels, c->n, c->dflags);
            CUDA_TRY(cudaGetLastError());
            CC_TRY(read_flags(c));
            if (!c->hflags[kFlagCompress]) break;
            ++r;
        }
    }
    if (rounds) *rounds = r;
    return CC_OK;
}

// Capture one order-guarded sweep launch per order kind the schedule can
// use (order 1, order 2, generic); at run time only the launch matching the
// device-side order does any work.
int launch_guarded(cc_ctx* c, const cc_schedule* s, int sm, cudaStream_t st) {
    bool need1 = false, need2 = false, needh = false;
    auto mark = [&](int order) {
        if (order == 1) need1 = true;
        else if (order == 2) need2 = true;
        else needh = true;
    };
    switch (s->variant) {
        case CC_VAR_C2:
        case CC_VAR_CSYN: mark(2); break;
        case CC_VAR_C1: mark(1); break;
        case CC_VAR_CM: mark(s->high_order); break;
        default: mark(1); mark(s->high_order); break;
    }
    const SweepLaunch sl{st, &c->dstate->order};
    lab_t* L = c->labels;
    if (need2 && c->layout == 5 && c->items) {
        // sweep 1 on the chunk-sorted rows, later sweeps on the bucketed copy
        CC_TRY(launch_o2(c, L, L, sm, SweepLaunch{st, &c->dstate->order_first}));
        CC_TRY(launch_bucketed(c, sm, SweepLaunch{st, &c->dstate->order_rest}));
    } else if (need2 && c->layout == 3 && c->items) {
        CC_TRY(launch_bucketed(c, sm, sl));
    } else if (need2) {
        CC_TRY(launch_o2(c, L, L, sm, sl));
    }
    if (need1) CC_TRY((launch_store_mode<1, 2>(c, L, L, 1, sm, sl)));
    if (needh) CC_TRY((launch_store_mode<0, 1>(c, L, L, s->high_order, sm, sl)));
    return CC_OK;
}

bool same_schedule(const cc_schedule& a, const cc_schedule& b) {
    return a.variant == b.variant && a.high_order == b.high_order && a.warmup == b.warmup &&
           a.sync == b.sync && a.atomic == b.atomic;
}

// Capture iota -> loop_init -> WHILE{ guarded sweeps -> loop_control } -> compress
// into one executable graph.
int build_loop(cc_ctx* c, const cc_schedule* s, int64_t cap, int sm, int check, int resume) {
    auto& k = c->loop_key;
    if (c->loop_exec && k.src == c->src && k.dst == c->dst && k.labels == c->labels &&
        k.m == c->m && k.n == c->n && k.cap == cap && same_schedule(k.s, *s) && k.sm == sm &&
        k.shortcut == c->shortcut && k.layout == c->layout && k.check == check &&
        k.items == c->items && k.n_items == c->n_items && k.resume == resume &&
        k.bsrc == c->bsrc)
        return CC_OK;
    if (c->loop_exec) cudaGraphExecDestroy(c->loop_exec);
    if (c->loop_graph) cudaGraphDestroy(c->loop_graph);
    c->loop_exec = nullptr;
    c->loop_graph = nullptr;
    if (!c->dstate) {
        CUDA_TRY(cudaMalloc(&c->dstate, sizeof(LoopState)));
        CUDA_TRY(cudaMalloc(&c->drec, sizeof(SweepRec) * kMaxRec));
        CUDA_TRY(cudaHostAlloc(&c->hstate, sizeof(LoopState), cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc(&c->hrec, sizeof(SweepRec) * kMaxRec, cudaHostAllocDefault));
    }
    cudaStream_t cs = c->cap_stream;
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    if (!resume) k_iota<<<grid_for(c, c->n), kThreads, 0, cs>>>(c->labels, c->n);
    k_loop_init<<<1, 1, 0, cs>>>(c->dstate, c->dflags, *s, resume ? 1 : 0);
    cudaStreamCaptureStatus status;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CUDA_TRY(cudaStreamGetCaptureInfo(cs, &status, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h;
    CUDA_TRY(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CUDA_TRY(cudaGraphAddNode(&cn, g, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CUDA_TRY(cudaStreamUpdateCaptureDependencies(cs, &cn, 1, cudaStreamSetCaptureDependencies));
    CUDA_TRY(cudaStreamBeginCaptureToGraph(c->body_stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    CC_TRY(launch_guarded(c, s, sm, c->body_stream));
    for (int j = 0; j < c->shortcut; ++j)
        k_compress<<<grid_for(c, (c->n + 3) / 4), kThreads, 0, c->body_stream>>>(
            c->labels, c->n, c->dflags, c->dflags + kFlagWrote);
    if (check) {  // edge half first: it fails within microseconds before convergence
        if (c->m > 0 && has_buckets(c) && !c->bucket_nosmem)
            CC_TRY(launch_check_slice(c, c->body_stream));
        else if (c->m > 0)
            k_gcheck_edges<<<grid_for(c, (c->m + 3) / 4), kThreads, 0, c->body_stream>>>(
                c->src, c->dst, c->m, c->labels, c->dflags);
        k_gcheck_idem<<<grid_for(c, c->n), kThreads, 0, c->body_stream>>>(c->labels, c->n,
                                                                          c->dflags);
    }
    k_loop_control<<<1, 1, 0, c->body_stream>>>(c->dstate, c->drec, c->dflags, *s, cap, check,
                                                h);
    CUDA_TRY(cudaGetLastError());
    cudaGraph_t body_out = nullptr;
    CUDA_TRY(cudaStreamEndCapture(c->body_stream, &body_out));
    k_compress<<<grid_for(c, (c->n + 3) / 4), kThreads, 0, cs>>>(c->labels, c->n, c->dflags,
                                                                 &c->dstate->need_compress);
    // the loop state, the first records and the flags come back inside the
    // graph (memcpy nodes into pinned memory): run_graph then needs one
    // launch and one synchronisation, no further API calls per run
    CUDA_TRY(cudaMemcpyAsync(c->hstate, c->dstate, sizeof(LoopState), cudaMemcpyDeviceToHost,
                             cs));
    CUDA_TRY(cudaMemcpyAsync(c->hrec, c->drec, sizeof(SweepRec) * kEagerRec,
                             cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaMemcpyAsync(c->hflags, c->dflags, sizeof(int) * kNumFlags,
                             cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaStreamEndCapture(cs, &c->loop_graph));
    CUDA_TRY(cudaGraphInstantiate(&c->loop_exec, c->loop_graph, 0));
    k = {c->src, c->dst,   c->labels, c->m,     c->n,       cap,   *s,
         sm,     c->shortcut, c->layout, check, c->items, c->n_items, resume, c->bsrc};
    return CC_OK;
}

int copy_out(cc_ctx* c, void* out, int eb);

// The fast path of cc_run: async sweeps, no per-sweep counting or early
// check -- the whole convergence loop is one graph launch.
// resume = 1: sweep 1 already ran (cc_run_host); the loop starts at sweep 2
// and leaves the stats entries of sweep 1 to the caller.
int run_graph(cc_ctx* c, const cc_schedule* s, int64_t cap, void* labels_out, int out_eb,
              cc_stats* st, int check, int resume = 0) {
    const int sm = s->atomic ? c->store_mode_atomic : c->store_mode_plain;
    CC_TRY(build_loop(c, s, cap, sm, check, resume));
    CUDA_TRY(cudaEventRecord(c->evs, c->stream));
    CUDA_TRY(cudaGraphLaunch(c->loop_exec, c->stream));
    CUDA_TRY(cudaEventRecord(c->eve, c->stream));
    // one synchronisation: state, flags and the first records were copied
    // back by the graph itself (build_loop)
    const bool want_rec = st && (st->changed_per_sweep || st->sweep_seconds);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const long long k = c->hstate->sweep;
    if (c->hstate->capped)
        return fail(CC_ECAP, "no convergence after %lld sweeps on n=%lld, m=%lld",
                    (long long)cap, (long long)c->n, (long long)c->m);
    const long long nrec = std::min<long long>(k, kMaxRec);
    if (want_rec && nrec > 0) {
        if (nrec > kEagerRec) {
            CUDA_TRY(cudaMemcpyAsync(c->hrec, c->drec, sizeof(SweepRec) * nrec,
                                     cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaStreamSynchronize(c->stream));
        }
        unsigned long long prev = c->hstate->t0;
        for (long long i = resume; i < nrec && i < st->capacity; ++i) {
            if (st->changed_per_sweep) st->changed_per_sweep[i] = c->hrec[i].wrote ? -1 : 0;
            if (st->sweep_seconds) st->sweep_seconds[i] = (c->hrec[i].t - prev) * 1e-9;
            prev = c->hrec[i].t;
        }
    }
    int rounds = 0;
    // the post-loop pass is gated off (final labels after a no-write sweep or
    // a passed check); should it ever change something, finish on the host
    if (c->hflags[kFlagCompress]) {
        CC_TRY(compress(c, &rounds));
        ++rounds;
    }
    float total_ms = 0.f;
    cudaEventElapsedTime(&total_ms, c->evs, c->eve);
    if (st) {
        st->sweeps_executed = k;
        // engine.py:313-320: a sweep passing the early check was still a
        // changing sweep
        const int by_check = c->hstate->by_check;
        st->sweeps_until_stable = by_check ? k : k - 1;
        st->converged_by = by_check ? 1 : 0;
        st->compress_rounds = rounds;
        st->converge_seconds = total_ms * 1e-3;
    }
    return copy_out(c, labels_out, out_eb);
}

// Enqueue the label read-back on stream st (int32/uint32 or int64 host array).
int copy_labels_async(cc_ctx* c, void* out, int eb, cudaStream_t st) {
    if (c->n == 0 || !out) return CC_OK;
    if (eb == 4) {
        CUDA_TRY(cudaMemcpyAsync(out, c->labels, sizeof(lab_t) * c->n, cudaMemcpyDeviceToHost,
                                 st));
        return CC_OK;
    }
    if (eb != 8) return fail(CC_EINVAL, "label element size must be 4 or 8");
    if (c->wide_cap < c->n) {
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
        cudaFree(c->wide);
        c->wide = nullptr;
        c->wide_cap = 0;
        CUDA_TRY(cudaMalloc((void**)&c->wide, sizeof(int64_t) * c->n));
        c->wide_cap = c->n;
    }
    k_widen<<<grid_for(c, c->n), kThreads, 0, st>>>(c->labels, c->n, c->wide);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, c->wide, sizeof(int64_t) * c->n, cudaMemcpyDeviceToHost, st));
    return CC_OK;
}

int copy_out(cc_ctx* c, void* out, int eb) {
    if (c->n == 0 || !out) return CC_OK;
    if (eb == 4) {
        CUDA_TRY(cudaMemcpyAsync(out, c->labels, sizeof(lab_t) * c->n, cudaMemcpyDeviceToHost,
                                 c->stream));
    } else if (eb == 8) {
        // a cached device buffer: a per-call stream-ordered allocation of 8n
        // bytes re-maps pool memory every call (~0.8 ms at n = 2^22, measured)
        if (c->wide_cap < c->n) {
            cudaFree(c->wide);
            c->wide = nullptr;
            c->wide_cap = 0;
            CUDA_TRY(cudaMalloc((void**)&c->wide, sizeof(int64_t) * c->n));
            c->wide_cap = c->n;
        }
        k_widen<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n, c->wide);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(out, c->wide, sizeof(int64_t) * c->n, cudaMemcpyDeviceToHost,
                                 c->stream));
    } else {
        return fail(CC_EINVAL, "label element size must be 4 or 8");
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return CC_OK;
}

// Radix-sort rows [off, off+len) of the SoA arrays by src, in place (CUB
// onesweep into the context's cached scratch, then copied back).  len must
// not exceed c->sort_chunk.
int sort_rows(cc_ctx* c, int64_t off, int64_t len) {
    if (len < 2) return CC_OK;
    const int bits = std::max<int>(1, (int)ccgen::perm_bits((uint64_t)c->n));
    const int64_t cap = std::max<int64_t>(len, c->sort_rows_cap);
    if (!c->sort_ks || c->sort_rows_cap < len) {
        cudaFree(c->sort_ks);
        cudaFree(c->sort_vs);
        cudaFree(c->sort_tmp);
        c->sort_ks = c->sort_vs = nullptr;
        c->sort_tmp = nullptr;
        CUDA_TRY(cudaMalloc(&c->sort_ks, sizeof(lab_t) * cap));
        CUDA_TRY(cudaMalloc(&c->sort_vs, sizeof(lab_t) * cap));
        c->sort_tmp_bytes = 0;
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, c->sort_tmp_bytes, c->src, c->sort_ks,
                                                 c->dst, c->sort_vs, (int)cap, 0, 32, c->stream));
        CUDA_TRY(cudaMalloc(&c->sort_tmp, c->sort_tmp_bytes));
        c->sort_rows_cap = cap;
    }
    size_t tb = c->sort_tmp_bytes;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->sort_tmp, tb, c->src + off, c->sort_ks,
                                             c->dst + off, c->sort_vs, (int)len, 0, bits,
                                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->src + off, c->sort_ks, sizeof(lab_t) * len,
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->dst + off, c->sort_vs, sizeof(lab_t) * len,
                             cudaMemcpyDeviceToDevice, c->stream));
    return CC_OK;
}

// ss != nullptr (cc_run_host): labels are initialised first and sweep 1 of
// schedule ss runs chunk by chunk right behind the copy -- each chunk's rows
// are swept as soon as they are staged, while the next chunk is in flight.
// Sweeping the chunks one after another is one asynchronous sweep over all
// rows in staging order (the grid-stride sweep visits rows in that order
// too), so it is sweep 1 of the run, overlapped with the transfer.
template <typename T>
int stage_impl(cc_ctx* c, const T* edges, int64_t m, bool host,
               const cc_schedule* ss = nullptr, bool ss_check = false, void* spec_out = nullptr,
               int spec_eb = 8) {
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
    const int ssm = ss ? (ss->atomic ? c->store_mode_atomic : c->store_mode_plain) : 0;
    if (ss) {
        k_iota<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemsetAsync(c->dflags, 0, sizeof(int) * kNumFlags, c->stream));
        CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    }
    const bool chunk_sort = c->stage_layout == 2;
    const int64_t chunk = std::min<int64_t>(c->sort_chunk, std::max<int64_t>(m, 1));
    if (m > 0) {
        if (!host) {
            k_stage<T><<<grid_for(c, m), kThreads, 0, c->stream>>>(edges, m, c->n, c->src, c->dst,
                                                                   c->dflags);
            CUDA_TRY(cudaGetLastError());
            if (chunk_sort)
                for (int64_t off = 0; off < m; off += chunk)
                    CC_TRY(sort_rows(c, off, std::min<int64_t>(chunk, m - off)));
        } else {
            // double-buffered H2D chunks on copy_stream, overlapped with the
            // AoS->SoA conversion (+ optional chunk sort) on the compute stream
            const size_t need = sizeof(T) * 2 * chunk;
            if (c->stage_buf_bytes < need) {
                cudaFree(c->stage_buf[0]);
                cudaFree(c->stage_buf[1]);
                c->stage_buf[0] = c->stage_buf[1] = nullptr;
                CUDA_TRY(cudaMalloc(&c->stage_buf[0], need));
                CUDA_TRY(cudaMalloc(&c->stage_buf[1], need));
                c->stage_buf_bytes = need;
            }
            for (int b = 0; b < 2; ++b) CUDA_TRY(cudaEventRecord(c->freed[b], c->stream));
            int64_t k = 0, swept = 0;
            for (int64_t off = 0; off < m; off += chunk, ++k) {
                const int b = (int)(k & 1);
                T* buf = (T*)c->stage_buf[b];
                const int64_t rows = std::min<int64_t>(chunk, m - off);
                CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->freed[b], 0));
                CUDA_TRY(cudaMemcpyAsync(buf, edges + 2 * off, sizeof(T) * 2 * rows,
                                         cudaMemcpyHostToDevice, c->copy_stream));
                CUDA_TRY(cudaEventRecord(c->copied[b], c->copy_stream));
                CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copied[b], 0));
                k_stage<T><<<grid_for(c, rows), kThreads, 0, c->stream>>>(
                    buf, rows, c->n, c->src + off, c->dst + off, c->dflags);
                CUDA_TRY(cudaGetLastError());
                CUDA_TRY(cudaEventRecord(c->freed[b], c->stream));
                if (chunk_sort) CC_TRY(sort_rows(c, off, rows));
                if (ss) {
                    // sweep windows start 16-byte aligned (the sweep's uint4 edge
                    // loads): a chunk's last rows mod 4 wait for the next chunk
                    const int64_t hi = off + rows == m ? m : (off + rows) & ~(int64_t)3;
                    if (hi > swept)
                        CC_TRY(launch_order_sl(c, c->labels, c->labels, order_for(ss, 1), ssm,
                                               SweepLaunch{c->stream, nullptr, swept, hi - swept}));
                    swept = hi;
                }
            }
        }
    }
    if (ss) CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    if (ss) {
        // sweep 1's shortcut and early check, in the same synchronisation
        for (int j = 0; j < c->shortcut; ++j)
            k_compress<<<grid_for(c, (c->n + 3) / 4), kThreads, 0, c->stream>>>(c->labels, c->n,
                                                                      c->dflags);
        if (spec_out) {
            // speculative read-back of the labels after sweep 1 on the copy
            // stream, overlapped with the check / confirming sweep: it is the
            // answer whenever nothing changes after this point
            // (cc_run_host decides, spec_valid)
            CUDA_TRY(cudaEventRecord(c->spec_ready, c->stream));
            CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->spec_ready, 0));
            CC_TRY(copy_labels_async(c, spec_out, spec_eb, c->copy_stream));
            CUDA_TRY(cudaEventRecord(c->spec_done, c->copy_stream));
        }
        if (ss_check) {
            if (m > 0)
                k_gcheck_edges<<<grid_for(c, (m + 3) / 4), kThreads, 0, c->stream>>>(
                    c->src, c->dst, m, c->labels, c->dflags);
            k_gcheck_idem<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n,
                                                                          c->dflags);
        }
        CUDA_TRY(cudaGetLastError());
    }
    const int rc = read_flags(c);
    if (spec_out && (rc || c->hflags[kFlagBad]))
        cudaEventSynchronize(c->spec_done);  // no read-back in flight after a failure
    if (rc) return rc;
    if (c->hflags[kFlagBad]) return fail(CC_EINVAL, "edge endpoint out of range (n=%lld)",
                                         (long long)c->n);
    return CC_OK;
}

int stage(cc_ctx* c, const void* edges, int eb, int64_t m, int64_t n, bool host,
          const cc_schedule* ss = nullptr, bool ss_check = false, void* spec_out = nullptr,
          int spec_eb = 8) {
    if (eb != 4 && eb != 8) return fail(CC_EINVAL, "edge element size must be 4 or 8");
    if (m > 0 && !edges) return fail(CC_EINVAL, "null edge buffer");
    CC_TRY(set_graph(c, m, n));
    CC_TRY(ensure_edges(c, m));
    if (eb == 4)
        return stage_impl<int32_t>(c, (const int32_t*)edges, m, host, ss, ss_check, spec_out,
                                   spec_eb);
    return stage_impl<int64_t>(c, (const int64_t*)edges, m, host, ss, ss_check, spec_out,
                               spec_eb);
}

}  // namespace

// ------------------------------------------------------------------ C-ABI
extern "C" {

const char* cc_last_error(void) { return g_err; }
int cc_version(void) { return 1; }

int cc_create(int device, void* stream, cc_ctx** out) {
    if (!out) return fail(CC_EINVAL, "null output pointer");
    *out = nullptr;
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(CC_EINVAL, "device %d out of range (%d devices)", device, ndev);
    DeviceGuard g(device);
    cc_ctx* c = new cc_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (stream) {
        c->stream = (cudaStream_t)stream;
    } else {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaMalloc(&c->dflags, sizeof(int) * kNumFlags));
    CUDA_TRY(cudaMemset(c->dflags, 0, sizeof(int) * kNumFlags));
    CUDA_TRY(cudaMalloc(&c->dcount, sizeof(unsigned long long)));
    CUDA_TRY(cudaHostAlloc(&c->hflags, sizeof(int) * kNumFlags, cudaHostAllocDefault));
    CUDA_TRY(cudaHostAlloc(&c->hcount, sizeof(unsigned long long), cudaHostAllocDefault));
    CUDA_TRY(cudaEventCreate(&c->ev0));
    CUDA_TRY(cudaEventCreate(&c->ev1));
    CUDA_TRY(cudaEventCreate(&c->evs));
    CUDA_TRY(cudaEventCreate(&c->eve));
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(cudaEventCreateWithFlags(&c->copied[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->freed[b], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&c->spec_ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->spec_done, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->body_stream, cudaStreamNonBlocking));
    *out = c;
    return CC_OK;
}

void cc_destroy(cc_ctx* c) {
    if (!c) return;
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->own_edges) { cudaFree(c->src); cudaFree(c->dst); }
    cudaFree(c->bsrc);
    cudaFree(c->bdst);
    if (c->own_labels) cudaFree(c->labels);
    cudaFree(c->wide);
    cudaFree(c->shadow);
    cudaFree(c->before);
    cudaFree(c->dflags);
    cudaFree(c->dcount);
    cudaFreeHost(c->hflags);
    cudaFreeHost(c->hcount);
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    cudaEventDestroy(c->evs);
    cudaEventDestroy(c->eve);
    for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(c->copied[b]);
        cudaEventDestroy(c->freed[b]);
        cudaFree(c->stage_buf[b]);
    }
    cudaEventDestroy(c->spec_ready);
    cudaEventDestroy(c->spec_done);
    cudaFree(c->sort_ks);
    cudaFree(c->sort_vs);
    cudaFree(c->sort_tmp);
    cudaFree(c->items);
    if (c->loop_exec) cudaGraphExecDestroy(c->loop_exec);
    if (c->loop_graph) cudaGraphDestroy(c->loop_graph);
    cudaFree(c->dstate);
    cudaFree(c->drec);
    cudaFreeHost(c->hstate);
    cudaFreeHost(c->hrec);
    cudaStreamDestroy(c->cap_stream);
    cudaStreamDestroy(c->body_stream);
    cudaStreamDestroy(c->copy_stream);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

int cc_stage_edges(cc_ctx* c, const void* edges, int eb, int64_t m, int64_t n) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return stage(c, edges, eb, m, n, true);
}

int cc_stage_edges_device(cc_ctx* c, const void* edges, int eb, int64_t m, int64_t n) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return stage(c, edges, eb, m, n, false);
}

int cc_attach_soa(cc_ctx* c, uint32_t* src, uint32_t* dst, int64_t m, int64_t n) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (m > 0 && (!src || !dst)) return fail(CC_EINVAL, "null edge arrays");
    if (((uintptr_t)src | (uintptr_t)dst) & 15)
        return fail(CC_EINVAL, "SoA edge arrays must be 16-byte aligned");
    if (c->own_edges) { cudaFree(c->src); cudaFree(c->dst); }
    c->src = src;
    c->dst = dst;
    c->own_edges = false;
    c->edge_cap = m;
    return set_graph(c, m, n);
}

int cc_attach_labels(cc_ctx* c, uint32_t* labels) {
    if (!c || !labels) return fail(CC_EINVAL, "null argument");
    if ((uintptr_t)labels & 15) return fail(CC_EINVAL, "label buffer must be 16-byte aligned");
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->own_labels && c->labels) cudaFree(c->labels);
    c->labels = labels;
    c->own_labels = false;
    c->label_cap = c->n + 1;
    return CC_OK;
}

int cc_labels_device(cc_ctx* c, uint32_t** out) {
    if (!c || !out) return fail(CC_EINVAL, "null argument");
    *out = c->labels;
    return CC_OK;
}

int cc_init_labels(cc_ctx* c) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return enqueue_init(c, false);
}

int cc_sweep(cc_ctx* c, int order, int sync, int atomic, int first, int* wrote_out) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (sync) {
        CC_TRY(ensure_aux(c, true, false));
        CUDA_TRY(cudaMemcpyAsync(c->shadow, c->labels, sizeof(lab_t) * c->n,
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    CC_TRY(enqueue_sweep(c, order, sync, atomic, false, first != 0));
    if (wrote_out) {
        CC_TRY(read_flags(c));
        *wrote_out = c->hflags[kFlagWrote] != 0;
    }
    return CC_OK;
}

int cc_fold_flag(cc_ctx* c, int first) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    k_fold<<<1, 1, 0, c->stream>>>(c->labels, c->n, c->dflags, first);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

int cc_shortcut(cc_ctx* c, int passes) {
    if (!c) return fail(CC_EINVAL, "null context");
    if (passes < 0) return fail(CC_EINVAL, "passes must be >= 0");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    for (int j = 0; j < passes && c->n > 0; ++j)
        k_compress<<<grid_for(c, (c->n + 3) / 4), kThreads, 0, c->stream>>>(c->labels, c->n, c->dflags);
    CUDA_TRY(cudaGetLastError());
    return CC_OK;
}

int cc_compress(cc_ctx* c, int* rounds) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return compress(c, rounds);
}

int cc_early_check(cc_ctx* c, int* ok) {
    if (!c || !ok) return fail(CC_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return early_check(c, ok);
}

// Size-independent certificate of a final labelling (used where the host
// oracle cannot run): bit 0 some edge has L[u] != L[v], bit 1 some label is
// not a root (L[L[x]] != L[x]), bit 2 some L[x] > x.  0 = every component
// carries one root label <= all its vertex IDs.
int cc_verify(cc_ctx* c, int* result) {
    if (!c || !result) return fail(CC_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    *result = 0;
    if (c->n == 0) return CC_OK;
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dflags + 3, 0, sizeof(int), c->stream));
    k_check_idem<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n, c->dflags);
    k_check_le<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->n, c->dflags);
    CUDA_TRY(cudaGetLastError());
    CC_TRY(read_flags(c));
    const int idem_bad = c->hflags[kFlagBad], le_bad = c->hflags[kFlagLe];
    int edge_bad = 0;
    if (c->m > 0) {
        CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
        k_check_edges<<<grid_for(c, c->m), kThreads, 0, c->stream>>>(c->src, c->dst, c->m,
                                                                     c->labels, c->dflags);
        CUDA_TRY(cudaGetLastError());
        CC_TRY(read_flags(c));
        edge_bad = c->hflags[kFlagBad];
    }
    *result = (edge_bad ? 1 : 0) | (idem_bad ? 2 : 0) | (le_bad ? 4 : 0);
    return CC_OK;
}

int cc_write_labels(cc_ctx* c, const void* in, int eb) {
    if (!c || (!in && c->n > 0)) return fail(CC_EINVAL, "null argument");
    if (eb != 4 && eb != 8) return fail(CC_EINVAL, "label element size must be 4 or 8");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (c->n == 0) return CC_OK;
    CC_TRY(ensure_labels(c));
    if (c->wide_cap < c->n) {  // staging buffer: the int64 read-back buffer
        cudaFree(c->wide);
        c->wide = nullptr;
        c->wide_cap = 0;
        CUDA_TRY(cudaMalloc((void**)&c->wide, sizeof(int64_t) * c->n));
        c->wide_cap = c->n;
    }
    CUDA_TRY(cudaMemcpyAsync(c->wide, in, (size_t)eb * c->n, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
    if (eb == 8)
        k_labels_in<int64_t><<<grid_for(c, c->n), kThreads, 0, c->stream>>>(
            (const int64_t*)c->wide, c->n, c->labels, c->dflags);
    else
        k_labels_in<int32_t><<<grid_for(c, c->n), kThreads, 0, c->stream>>>(
            (const int32_t*)c->wide, c->n, c->labels, c->dflags);
    CUDA_TRY(cudaGetLastError());
    CC_TRY(read_flags(c));
    if (c->hflags[kFlagBad]) return fail(CC_EINVAL, "labels reference vertices outside 0..n-1");
    return CC_OK;
}

int cc_read_labels(cc_ctx* c, void* out, int eb) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return copy_out(c, out, eb);
}

int cc_synchronize(cc_ctx* c) {
    if (!c) return fail(CC_EINVAL, "null context");
    DeviceGuard g(c->device);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return CC_OK;
}

}  // extern "C"

namespace {

int check_run_args(cc_ctx* c, const cc_schedule* s, void* labels_out, int out_eb) {
    if (!c || !s) return fail(CC_EINVAL, "null argument");
    if (s->variant < CC_VAR_CSYN || s->variant > CC_VAR_C1M1M)
        return fail(CC_EINVAL, "unknown variant code %d", s->variant);
    if (labels_out && out_eb != 4 && out_eb != 8)
        return fail(CC_EINVAL, "label element size must be 4 or 8");
    return CC_OK;
}

// run_contour (engine.py:248-328) over the device kernels; caller holds c->mu.
int run_impl(cc_ctx* c, const cc_schedule* s, int flags, int64_t cap, void* labels_out,
             int out_eb, cc_stats* st) {
    const bool sync = s->sync != 0;
    const bool count = (flags & CC_RUN_COUNT_CHANGES) != 0;
    const bool check = (flags & CC_RUN_EARLY_CHECK) != 0;
    const bool times = (flags & CC_RUN_SWEEP_TIMES) != 0;
    const bool first_scatter = (flags & CC_RUN_FIRST_SCATTER) != 0;
    if (!sync && !count && !first_scatter && !(flags & CC_RUN_HOST_LOOP) && c->n > 0 &&
        c->peers.n == 0)
        return run_graph(c, s, cap, labels_out, out_eb, st, check ? 1 : 0);
    CUDA_TRY(cudaEventRecord(c->evs, c->stream));
    CC_TRY(enqueue_init(c, sync));
    int64_t sweep = 0, until_stable = 0;
    int converged_by = 0;
    while (true) {
        ++sweep;
        if (sweep > cap)
            return fail(CC_ECAP, "no convergence after %lld sweeps on n=%lld, m=%lld",
                        (long long)cap, (long long)c->n, (long long)c->m);
        const int order = order_for(s, sweep);
        if (times) CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
        CC_TRY(enqueue_sweep(c, order, sync, s->atomic, count, sweep == 1 && first_scatter,
                             sweep));
        if (!sync && !count)
            for (int j = 0; j < c->shortcut; ++j)
                k_compress<<<grid_for(c, (c->n + 3) / 4), kThreads, 0, c->stream>>>(c->labels, c->n,
                                                                          c->dflags);
        if (times) CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
        CC_TRY(read_flags(c));
        const bool wrote = c->hflags[kFlagWrote] != 0;
        const int64_t changed = (sync || count) ? (int64_t)*c->hcount : (wrote ? -1 : 0);
        if (st && st->changed_per_sweep && sweep <= st->capacity)
            st->changed_per_sweep[sweep - 1] = changed;
        if (st && st->sweep_seconds && sweep <= st->capacity) {
            float ms = 0.f;
            if (times) cudaEventElapsedTime(&ms, c->ev0, c->ev1);
            st->sweep_seconds[sweep - 1] = ms * 1e-3;
        }
        if (!wrote && changed == 0) { converged_by = 0; break; }
        until_stable = sweep;
        if (check) {
            int ok = 0;
            CC_TRY(early_check(c, &ok));
            if (ok) { converged_by = 1; break; }
        }
    }
    int rounds = 0;
    CC_TRY(compress(c, &rounds));
    CUDA_TRY(cudaEventRecord(c->eve, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->eve));
    float total_ms = 0.f;
    cudaEventElapsedTime(&total_ms, c->evs, c->eve);
    if (st) {
        st->sweeps_executed = sweep;
        st->sweeps_until_stable = until_stable;
        st->converged_by = converged_by;
        st->compress_rounds = rounds;
        st->converge_seconds = total_ms * 1e-3;
    }
    return copy_out(c, labels_out, out_eb);
}

// The streamed path of cc_run_host: applies to asynchronous runs without
// exact counting / first scatter / host loop / peers, staged in input or
// chunk-sorted order (the orders a sweep can follow while rows arrive).
bool streamable(const cc_ctx* c, const cc_schedule* s, int flags) {
    return !s->sync && !(flags & (CC_RUN_COUNT_CHANGES | CC_RUN_FIRST_SCATTER | CC_RUN_HOST_LOOP)) &&
           c->peers.n == 0 && (c->stage_layout == 0 || c->stage_layout == 2);
}

}  // namespace

extern "C" {

int cc_run(cc_ctx* c, const cc_schedule* s, int flags, int64_t cap, void* labels_out, int out_eb,
           cc_stats* st) {
    CC_TRY(check_run_args(c, s, labels_out, out_eb));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return run_impl(c, s, flags, cap, labels_out, out_eb, st);
}

// Stage host edges AND run (run_contour(g, ...) for a graph in host memory):
// sweep 1 streams behind the host-to-device copy (stage_impl), then its
// shortcut pass and early check decide whether the device-side loop must
// continue from sweep 2.
int cc_run_host(cc_ctx* c, const void* edges_host, int elem_bytes, int64_t m, int64_t n,
                const cc_schedule* s, int flags, int64_t cap, void* labels_out, int out_eb,
                cc_stats* st) {
    CC_TRY(check_run_args(c, s, labels_out, out_eb));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (!streamable(c, s, flags) || n == 0 || cap < 1) {
        CC_TRY(stage(c, edges_host, elem_bytes, m, n, true));
        return run_impl(c, s, flags, cap, labels_out, out_eb, st);
    }
    const bool check = (flags & CC_RUN_EARLY_CHECK) != 0;
    CC_TRY(stage(c, edges_host, elem_bytes, m, n, true, s, check, labels_out, out_eb));
    const bool wrote = c->hflags[kFlagWrote] != 0;
    const bool passed = check && wrote && c->hflags[kFlagCheck] == 0;
    float sweep1_ms = 0.f;
    cudaEventElapsedTime(&sweep1_ms, c->ev0, c->ev1);
    int64_t k = 1, until_stable = wrote ? 1 : 0;
    int by = passed ? 1 : 0;
    double seconds = sweep1_ms * 1e-3;
    int rounds = 0;
    if (wrote && !passed) {  // not converged after sweep 1: the loop from sweep 2
        CUDA_TRY(cudaMemsetAsync(c->dflags, 0, sizeof(int) * kNumFlags, c->stream));
        cc_stats local = {};
        cc_stats* gs = st ? st : &local;
        const int rc = run_graph(c, s, cap, nullptr, out_eb, gs, check ? 1 : 0, 1);
        if (rc) {  // (e.g. the cap) -- no read-back may still be writing the caller's buffer
            if (labels_out) cudaEventSynchronize(c->spec_done);
            return rc;
        }
        k = gs->sweeps_executed;
        until_stable = gs->sweeps_until_stable;
        by = gs->converged_by;
        rounds = gs->compress_rounds;
        seconds += gs->converge_seconds;
    } else if (!passed) {
        const int rc = compress(c, &rounds);  // (a passed check already proved idempotence)
        if (rc) {
            if (labels_out) cudaEventSynchronize(c->spec_done);
            return rc;
        }
    }
    // the speculative read-back (stage_impl) holds the final labels iff nothing
    // changed after sweep 1's shortcut: converged at sweep 1, or sweep 2 was a
    // no-write sweep (its shortcut and the final compress are then gated off)
    // and no compress round changed anything
    const bool spec_valid = rounds == 0 && (k == 1 || (k == 2 && by == 0));
    if (labels_out && c->n > 0) {
        CUDA_TRY(cudaEventSynchronize(c->spec_done));  // before the buffer is reused
        if (spec_valid) labels_out = nullptr;
    }
    if (st) {
        st->sweeps_executed = k;
        st->sweeps_until_stable = until_stable;
        st->converged_by = by;
        st->compress_rounds = rounds;
        st->converge_seconds = seconds;
        if (st->capacity >= 1) {
            if (st->changed_per_sweep) st->changed_per_sweep[0] = wrote ? -1 : 0;
            if (st->sweep_seconds) st->sweep_seconds[0] = sweep1_ms * 1e-3;
        }
    }
    return copy_out(c, labels_out, out_eb);
}

// ---- fused multi-GPU exchange: peer replicas over CUDA IPC -----------------
int cc_ipc_get_handle(cc_ctx* c, void* handle_out) {
    if (!c || !handle_out) return fail(CC_EINVAL, "null argument");
    if (!c->own_labels || !c->labels)
        return fail(CC_EINVAL, "IPC export needs the context's own label buffer");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, c->labels));
    memcpy(handle_out, &h, sizeof(h));
    return CC_OK;
}

int cc_ipc_open(cc_ctx* c, const void* handle, uint64_t* ptr_out) {
    if (!c || !handle || !ptr_out) return fail(CC_EINVAL, "null argument");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr_out = (uint64_t)(uintptr_t)p;
    return CC_OK;
}

int cc_ipc_close(cc_ctx* c, uint64_t ptr) {
    if (!c) return fail(CC_EINVAL, "null context");
    DeviceGuard g(c->device);
    CUDA_TRY(cudaIpcCloseMemHandle((void*)(uintptr_t)ptr));
    return CC_OK;
}

int cc_set_peers(cc_ctx* c, const uint64_t* ptrs, int npeers) {
    if (!c || (npeers > 0 && !ptrs)) return fail(CC_EINVAL, "null argument");
    if (npeers < 0 || npeers > cck::kMaxPeers)
        return fail(CC_EINVAL, "peer count must be 0..%d", cck::kMaxPeers);
    std::lock_guard<std::mutex> lk(c->mu);
    c->peers.n = npeers;
    for (int i = 0; i < npeers; ++i) c->peers.p[i] = (lab_t*)(uintptr_t)ptrs[i];
    c->loop_key.m = -1;
    return CC_OK;
}

// FastSV baseline (baselines.py:81-131) on the staged edges: synchronous
// hooking + shortcutting until the grandparent array stops changing.
// stats: changed_per_sweep = cells changed per iteration (exact, equal to the
// reference's), converged_by = 2 ("grandparent-stable").
int cc_fastsv(cc_ctx* c, int64_t cap, void* labels_out, int out_eb, cc_stats* st, int flags) {
    if (!c) return fail(CC_EINVAL, "null context");
    if (labels_out && out_eb != 4 && out_eb != 8)
        return fail(CC_EINVAL, "label element size must be 4 or 8");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    const int64_t n = c->n;
    const bool times = (flags & CC_RUN_SWEEP_TIMES) != 0;
    CC_TRY(ensure_aux(c, true, false));
    lab_t *G2 = nullptr, *N = nullptr;
    CUDA_TRY(cudaMalloc(&G2, sizeof(lab_t) * (n + 1)));
    CUDA_TRY(cudaMalloc(&N, sizeof(lab_t) * (n + 1)));
    lab_t* const n_alloc = N;
    lab_t* const g2_alloc = G2;
    lab_t* P = c->labels;
    lab_t* G = c->shadow;
    CUDA_TRY(cudaEventRecord(c->evs, c->stream));
    if (n > 0) {
        k_iota<<<grid_for(c, n), kThreads, 0, c->stream>>>(P, n);
        CUDA_TRY(cudaMemcpyAsync(G, P, sizeof(lab_t) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
    int64_t it = 0, until = 0;
    int rc = CC_OK;
    while (true) {
        ++it;
        if (it > cap) {
            rc = fail(CC_ECAP, "fastsv did not converge in %lld iterations", (long long)cap);
            break;
        }
        if (times) CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
        CUDA_TRY(cudaMemsetAsync(c->dcount, 0, sizeof(unsigned long long), c->stream));
        CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
        if (n > 0) {
            CUDA_TRY(cudaMemcpyAsync(N, P, sizeof(lab_t) * n, cudaMemcpyDeviceToDevice, c->stream));
            if (c->m > 0)
                k_fastsv_hook<<<grid_for(c, c->m, 16), kThreads, 0, c->stream>>>(c->src, c->dst,
                                                                                 c->m, P, G, N);
            k_fastsv_shortcut<<<grid_for(c, n), kThreads, 0, c->stream>>>(N, G, P, n, c->dcount);
            std::swap(P, N);
            k_fastsv_grand<<<grid_for(c, n), kThreads, 0, c->stream>>>(P, G, G2, n, c->dflags);
            CUDA_TRY(cudaGetLastError());
        }
        if (times) CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
        CC_TRY(read_flags(c));
        const int64_t changed = (int64_t)*c->hcount;
        if (st && st->changed_per_sweep && it <= st->capacity) st->changed_per_sweep[it - 1] = changed;
        if (st && st->sweep_seconds && it <= st->capacity) {
            float ms = 0.f;
            if (times) cudaEventElapsedTime(&ms, c->ev0, c->ev1);
            st->sweep_seconds[it - 1] = ms * 1e-3;
        }
        if (changed) until = it;
        if (!c->hflags[kFlagBad]) break;
        std::swap(G, G2);
    }
    if (rc == CC_OK && n > 0 && P != c->labels)
        CUDA_TRY(cudaMemcpyAsync(c->labels, P, sizeof(lab_t) * n, cudaMemcpyDeviceToDevice,
                                 c->stream));
    // the local pointers rotated; the two scratch allocations are freed by
    // their original addresses (c->labels / c->shadow stay owned by the ctx)
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    cudaFree(n_alloc);
    cudaFree(g2_alloc);
    if (rc != CC_OK) return rc;
    int rounds = 0;
    CC_TRY(compress(c, &rounds));
    CUDA_TRY(cudaEventRecord(c->eve, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->eve));
    float total_ms = 0.f;
    cudaEventElapsedTime(&total_ms, c->evs, c->eve);
    if (st) {
        st->sweeps_executed = it;
        st->sweeps_until_stable = until;
        st->converged_by = 2;
        st->compress_rounds = rounds;
        st->converge_seconds = total_ms * 1e-3;
    }
    return copy_out(c, labels_out, out_eb);
}

int cc_set_option(cc_ctx* c, int option, int64_t value) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    switch (option) {
        case CC_OPT_STORE_MODE_PLAIN:
        case CC_OPT_STORE_MODE_ATOMIC:
            if (value < cck::kStorePlain || value > cck::kStoreCheckRed)
                return fail(CC_EINVAL, "store mode must be 0..3");
            // a non-atomic schedule may use any mode (atomic min is one legal
            // interleaving of plain stores); an atomic one must never lose a
            // lowering, so it only accepts the red.min modes
            if (option == CC_OPT_STORE_MODE_ATOMIC &&
                (value == cck::kStorePlain || value == cck::kStoreCheckPlain))
                return fail(CC_EINVAL, "atomic schedules need store mode 1 or 3");
            (option == CC_OPT_STORE_MODE_PLAIN ? c->store_mode_plain : c->store_mode_atomic) =
                (int)value;
            return CC_OK;
        case CC_OPT_SORT_CHUNK:
            if (value < 1 || value >= ((int64_t)1 << 31))
                return fail(CC_EINVAL, "sort chunk must be in [1, 2^31)");
            c->sort_chunk = value;
            return CC_OK;
        case CC_OPT_STAGE_LAYOUT:
            if (value != 0 && value != 2)
                return fail(CC_EINVAL, "staging layout must be 0 (input) or 2 (chunk-sorted)");
            c->stage_layout = (int)value;
            return CC_OK;
        case CC_OPT_BUCKET_SHIFT:
            if (value < 8 || value > 15)
                return fail(CC_EINVAL, "bucket shift must be in [8, 15] (<= 128 KB of labels)");
            c->bucket_shift = (int)value;
            return CC_OK;
        case CC_OPT_ITEM_ROWS:
            if (value < 1024) return fail(CC_EINVAL, "item rows must be >= 1024");
            c->item_rows = value;
            return CC_OK;
        case CC_OPT_SHORTCUT:
            if (value < 0 || value > 8) return fail(CC_EINVAL, "shortcut passes must be 0..8");
            c->shortcut = (int)value;
            return CC_OK;
        case CC_OPT_SWEEP_VARIANT:
            if (value < 0 || value > 17) return fail(CC_EINVAL, "sweep variant must be 0..17");
            c->sweep_variant = (int)value;
            c->loop_key.m = -1;
            return CC_OK;
        case CC_OPT_BUCKET_NOSMEM:
            c->bucket_nosmem = value != 0;
            c->loop_key.m = -1;
            return CC_OK;
        case CC_OPT_BUCKET_PIPE:
            if (value < 0 || value > 3) return fail(CC_EINVAL, "bucket kernel must be 0..3");
            c->bucket_pipe = (int)value;
            c->loop_key.m = -1;
            return CC_OK;
        case CC_OPT_ITEM_ORDER:
            if (value < 0 || value > 2)
                return fail(CC_EINVAL, "item order must be 0 (bucket-major), 1 (run-major) or "
                                       "2 (run-major, staggered)");
            c->item_order = (int)value;
            return CC_OK;
        case CC_OPT_TILE_SPLIT:
            if (value < 1 || value > 1024) return fail(CC_EINVAL, "tile split must be 1..1024");
            c->tile_split = (int)value;
            return CC_OK;
        case CC_OPT_TILE_SHIFT:
            if (value < 10 || value > 30) return fail(CC_EINVAL, "tile shift must be in [10, 30]");
            c->tile_shift = (int)value;
            return CC_OK;
        case CC_OPT_BUCKET_THREADS:
            if (value != 256 && value != 512 && value != 1024)
                return fail(CC_EINVAL, "bucket threads must be 256, 512 or 1024");
            c->bucket_threads = (int)value;
            return CC_OK;
    }
    return fail(CC_EINVAL, "unknown option %d", option);
}

}  // extern "C"

namespace {

template <typename K>
// Output rows go to (osrc, odst): the row arrays themselves (layout 3) or
// the bucketed copy (layout 5); the input rows are read from c->src/c->dst.
int reorder_bucketed_t(cc_ctx* c, int sbits, int total_bits, int64_t nb, int runs,
                       int run_major, lab_t* osrc, lab_t* odst, int layout) {
    const int64_t m = c->m;
    K *kin = nullptr, *kout = nullptr;
    lab_t* vout = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CUDA_TRY(cudaMalloc(&kin, sizeof(K) * m));
    CUDA_TRY(cudaMalloc(&kout, sizeof(K) * m));
    CUDA_TRY(cudaMalloc(&vout, sizeof(lab_t) * m));
    k_make_keys<K><<<grid_for(c, m, 16), kThreads, 0, c->stream>>>(
        c->src, c->dst, m, c->bucket_shift, sbits, runs, nb, run_major, kin);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, c->dst, vout, (int)m, 0,
                                             total_bits, c->stream));
    CUDA_TRY(cudaMalloc(&tmp, tb));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, c->dst, vout, (int)m, 0,
                                             total_bits, c->stream));
    k_unkey<K><<<grid_for(c, m, 16), kThreads, 0, c->stream>>>(kout, m,
                                                                (K)(((K)1 << sbits) - 1), osrc);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(odst, vout, sizeof(lab_t) * m, cudaMemcpyDeviceToDevice,
                             c->stream));
    // group g = bucket (bucket-major) or run * nb + bucket (run-major)
    const int64_t ng = nb * runs;
    int64_t* dstarts = nullptr;
    CUDA_TRY(cudaMalloc(&dstarts, sizeof(int64_t) * (ng + 1)));
    k_bucket_starts<K><<<grid_for(c, ng), kThreads, 0, c->stream>>>(kout, m, ng, sbits, 1,
                                                                     dstarts);
    CUDA_TRY(cudaGetLastError());
    std::vector<int64_t> starts(ng + 1);
    CUDA_TRY(cudaMemcpyAsync(starts.data(), dstarts, sizeof(int64_t) * ng,
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    starts[ng] = m;
    cudaFree(kin);
    cudaFree(kout);
    cudaFree(vout);
    cudaFree(tmp);
    cudaFree(dstarts);
    // work items: each group's (src-sorted) rows cut into pieces of <=
    // item_rows, in group order.  Run-major groups make the CTAs running at
    // the same time cover the same src range of every bucket of one run, so
    // the whole GPU walks each run's src range in increasing order, as the
    // grid-stride sweep does on chunk-sorted rows (the order that propagates
    // the smallest labels furthest per sweep).
    // item_order 2 staggers the items of one run: item j of bucket b's k
    // items is keyed ((j / k + b / nb) mod 1), so the CTAs running at the same
    // time read different src ranges (run-major lockstep makes every SM
    // gather the same src labels at once) while the runs stay ordered.
    struct Keyed {
        int64_t run;
        double key;
        cck::BucketItem it;
    };
    std::vector<Keyed> keyed;
    const int64_t B = (int64_t)1 << c->bucket_shift;
    for (int64_t g = 0; g < ng; ++g) {
        const int64_t b = run_major ? g % nb : g;
        const uint32_t base = (uint32_t)(b * B);
        const uint32_t len = (uint32_t)std::min<int64_t>(B, c->n - b * B);
        const int64_t k = (starts[g + 1] - starts[g] + c->item_rows - 1) / c->item_rows;
        int64_t j = 0;
        for (int64_t r = starts[g]; r < starts[g + 1]; r += c->item_rows, ++j) {
            double key = (double)keyed.size();
            if (c->item_order == 2) {
                key = (double)j / (double)k + (double)b / (double)nb;
                key -= (double)(int64_t)key;
            }
            keyed.push_back({run_major ? g / nb : 0, key,
                             {r, std::min<int64_t>(r + c->item_rows, starts[g + 1]), base,
                              c->bucket_nosmem ? 0u : len}});
        }
    }
    std::stable_sort(keyed.begin(), keyed.end(), [](const Keyed& a, const Keyed& b) {
        return a.run != b.run ? a.run < b.run : a.key < b.key;
    });
    std::vector<cck::BucketItem> items;
    items.reserve(keyed.size());
    for (auto& k : keyed) items.push_back(k.it);
    if (items.size() >= ((size_t)1 << 31)) return fail(CC_EINVAL, "too many bucket work items");
    cudaFree(c->items);
    c->items = nullptr;
    c->n_items = (int)items.size();
    if (!items.empty()) {
        CUDA_TRY(cudaMalloc(&c->items, sizeof(cck::BucketItem) * items.size()));
        CUDA_TRY(cudaMemcpy(c->items, items.data(), sizeof(cck::BucketItem) * items.size(),
                            cudaMemcpyHostToDevice));
    }
    c->layout = layout;
    return CC_OK;
}

// Layout 3: rows grouped by dst bucket, src-sorted inside (one global sort).
// item_order 1: rows first cut, in their current order, into runs of
// sort_chunk rows; groups are (run, bucket).
// layout 5 (hybrid): the rows keep their order (sweep 1 runs on them) and a
// dst-bucketed copy is built next to them for the later sweeps / checks.
int reorder_bucketed(cc_ctx* c, int layout = 3) {
    if (c->m >= ((int64_t)1 << 31)) return fail(CC_EINVAL, "bucketed layout needs m < 2^31");
    lab_t *osrc = c->src, *odst = c->dst;
    if (layout == 5) {
        if (c->bcap < c->m) {
            cudaFree(c->bsrc);
            cudaFree(c->bdst);
            c->bsrc = c->bdst = nullptr;
            c->bcap = 0;
            CUDA_TRY(cudaMalloc(&c->bsrc, sizeof(lab_t) * c->m));
            CUDA_TRY(cudaMalloc(&c->bdst, sizeof(lab_t) * c->m));
            c->bcap = c->m;
        }
        osrc = c->bsrc;
        odst = c->bdst;
    }
    const int sbits = std::max<int>(1, (int)ccgen::perm_bits((uint64_t)c->n));
    const int64_t B = (int64_t)1 << c->bucket_shift;
    const int64_t nb = (c->n + B - 1) / B;
    const int run_major = c->item_order >= 1;
    const int runs =
        run_major ? (int)std::max<int64_t>(1, (c->m + c->sort_chunk - 1) / c->sort_chunk) : 1;
    const int bbits = std::max<int>(1, (int)ccgen::perm_bits((uint64_t)(nb * runs)));
    if (sbits + bbits <= 32)
        return reorder_bucketed_t<uint32_t>(c, sbits, sbits + bbits, nb, runs, run_major, osrc,
                                            odst, layout);
    return reorder_bucketed_t<unsigned long long>(c, sbits, sbits + bbits, nb, runs, run_major,
                                                  osrc, odst, layout);
}

// Layout 4: rows partitioned by dst into L2-window buckets of 2^tile_shift
// vertices (default 2^23: 32 MB of labels), then sorted by src inside each
// bucket.  A grid-stride sweep walks the buckets in order, so at any time
// the gathered dst labels come from one 32 MB window that stays in L2 and
// the src gathers of consecutive rows coalesce.  Scales past 2^31 rows
// (partition kernels + per-bucket CUB sorts); needs 8m bytes of scratch.
int reorder_l2tiles(cc_ctx* c) {
    const int64_t m = c->m;
    const int shift = c->tile_shift;
    const int64_t P = (c->n + ((int64_t)1 << shift) - 1) >> shift;
    if (P > kMaxTiles) return fail(CC_EINVAL, "too many L2 tiles (%lld); raise tile shift",
                                   (long long)P);
    unsigned long long* dcnt = nullptr;
    CUDA_TRY(cudaMalloc(&dcnt, sizeof(unsigned long long) * P));
    CUDA_TRY(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * P, c->stream));
    const int64_t nblk = (m + kPartRows - 1) / kPartRows;
    k_tile_hist<<<(unsigned)nblk, kThreads, 0, c->stream>>>(c->dst, m, shift, (int)P, dcnt);
    CUDA_TRY(cudaGetLastError());
    std::vector<unsigned long long> cnt(P), start(P + 1, 0);
    CUDA_TRY(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(unsigned long long) * P,
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int64_t b = 0; b < P; ++b) start[b + 1] = start[b] + cnt[b];
    CUDA_TRY(cudaMemcpyAsync(dcnt, start.data(), sizeof(unsigned long long) * P,
                             cudaMemcpyHostToDevice, c->stream));
    lab_t *os = nullptr, *od = nullptr;
    CUDA_TRY(cudaMalloc(&os, sizeof(lab_t) * m));
    CUDA_TRY(cudaMalloc(&od, sizeof(lab_t) * m));
    k_tile_scatter<<<(unsigned)nblk, kThreads, 0, c->stream>>>(c->src, c->dst, m, shift, (int)P,
                                                                dcnt, os, od);
    CUDA_TRY(cudaGetLastError());
    // per-bucket sort by src, out of the scratch copy straight back into src/dst
    const int bits = std::max<int>(1, (int)ccgen::perm_bits((uint64_t)c->n));
    int64_t maxb = 0;
    for (int64_t b = 0; b < P; ++b) maxb = std::max<int64_t>(maxb, (int64_t)cnt[b]);
    if (maxb >= ((int64_t)1 << 31)) {
        cudaFree(os);
        cudaFree(od);
        cudaFree(dcnt);
        return fail(CC_EINVAL, "an L2 tile holds >= 2^31 rows; lower the tile shift");
    }
    void* tmp = nullptr;
    size_t tb = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, os, c->src, od, c->dst,
                                             (int)std::max<int64_t>(maxb, 1), 0, bits,
                                             c->stream));
    CUDA_TRY(cudaMalloc(&tmp, tb));
    // each window is sorted as tile_split independent runs: a sweep then
    // crosses the src range tile_split times per window, which propagates
    // labels further within one sweep (fewer sweeps) at a small cost in
    // src-gather coalescing
    for (int64_t b = 0; b < P; ++b) {
        const int64_t off = (int64_t)start[b], len = (int64_t)cnt[b];
        const int64_t k = std::max<int64_t>(1, std::min<int64_t>(c->tile_split, len));
        for (int64_t r = 0; r < k; ++r) {
            const int64_t lo = off + len * r / k, hi = off + len * (r + 1) / k;
            if (hi <= lo) continue;
            size_t t2 = tb;
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, t2, os + lo, c->src + lo, od + lo,
                                                     c->dst + lo, (int)(hi - lo), 0, bits,
                                                     c->stream));
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    cudaFree(tmp);
    cudaFree(os);
    cudaFree(od);
    cudaFree(dcnt);
    c->layout = 4;
    return CC_OK;
}

}  // namespace

extern "C" {

int cc_reorder_edges(cc_ctx* c, int mode) {
    if (!c) return fail(CC_EINVAL, "null context");
    if (mode == 0) return CC_OK;
    if (mode < 1 || mode > 5) return fail(CC_EINVAL, "unknown edge layout mode %d", mode);
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (c->m < 2) return CC_OK;
    if (mode == 3 || mode == 5) return reorder_bucketed(c, mode);
    if (mode == 4) return reorder_l2tiles(c);
    c->layout = mode;
    // mode 1: one global sort by src; mode 2: independent sorts of
    // consecutive chunks of c->sort_chunk rows (each chunk's label gathers
    // coalesce almost as well, and chunks can be sorted while later chunks
    // are still being copied in).
    const int64_t chunk = mode == 1 ? c->m : std::min<int64_t>(c->sort_chunk, c->m);
    if (chunk >= ((int64_t)1 << 31)) return fail(CC_EINVAL, "edge reorder needs chunks < 2^31 rows");
    for (int64_t off = 0; off < c->m; off += chunk)
        CC_TRY(sort_rows(c, off, std::min<int64_t>(chunk, c->m - off)));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return CC_OK;
}

int cc_mm_order(const int64_t* read, int64_t* target, int64_t n, int64_t w, int64_t v, int order,
                int inplace, int* changed_out) {
    if (order < 1) return fail(CC_EINVAL, "operator order must be >= 1");
    if (!read || !target || n <= 0 || w < 0 || v < 0 || w >= n || v >= n)
        return fail(CC_EINVAL, "bad single-edge arguments");
    int64_t* d64 = nullptr;
    lab_t *R = nullptr, *T = nullptr;
    int* dch = nullptr;
    CUDA_TRY(cudaMalloc(&d64, sizeof(int64_t) * n));
    CUDA_TRY(cudaMalloc(&R, sizeof(lab_t) * n));
    CUDA_TRY(cudaMalloc(&T, sizeof(lab_t) * n));
    CUDA_TRY(cudaMalloc(&dch, sizeof(int)));
    CUDA_TRY(cudaMemset(dch, 0, sizeof(int)));
    CUDA_TRY(cudaMemcpy(d64, read, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    k_from64<<<1, 256>>>(d64, n, R);
    CUDA_TRY(cudaMemcpy(d64, inplace ? read : target, sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    k_from64<<<1, 256>>>(d64, n, T);
    k_single_edge<<<1, 1>>>(R, T, (lab_t)w, (lab_t)v, order, inplace, dch);
    CUDA_TRY(cudaGetLastError());
    k_widen<<<1, 256>>>(T, n, d64);
    std::vector<int64_t> before(target, target + n);
    if (inplace) before.assign(read, read + n);
    CUDA_TRY(cudaMemcpy(target, d64, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    int ch = 0;
    CUDA_TRY(cudaMemcpy(&ch, dch, sizeof(int), cudaMemcpyDeviceToHost));
    if (!inplace) {
        ch = 0;
        for (int64_t i = 0; i < n; ++i) ch |= (target[i] != before[i]);
    }
    if (changed_out) *changed_out = ch;
    cudaFree(d64);
    cudaFree(R);
    cudaFree(T);
    cudaFree(dch);
    return CC_OK;
}

int cc_gen_rmat_device(cc_ctx* c, int scale, int ef, uint64_t seed, uint32_t tA, uint32_t tAB,
                       uint32_t tABC, int symmetrize, int permute, int64_t lo, int64_t hi) {
    if (!c) return fail(CC_EINVAL, "null context");
    if (scale < 1 || scale > 32 || ef < 1) return fail(CC_EINVAL, "bad RMAT scale/edgefactor");
    const int64_t n = (int64_t)1 << scale;
    const int64_t M = (int64_t)ef * n;
    const int64_t rows = symmetrize ? 2 * M : M;
    if (lo < 0 || hi > rows || lo > hi) return fail(CC_EINVAL, "bad RMAT row range");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    CC_TRY(set_graph(c, hi - lo, n));
    CC_TRY(ensure_edges(c, hi - lo));
    ccgen::RmatParams rp{ccgen::key(seed, ccgen::STREAM_RMAT), (uint32_t)scale, tA, tAB, tABC};
    ccgen::Perm pm = ccgen::perm_init((uint64_t)n, ccgen::key(seed, ccgen::STREAM_PERM));
    if (hi > lo) {
        k_gen_rmat<<<grid_for(c, hi - lo, 16), kThreads, 0, c->stream>>>(rp, pm, permute, M, symmetrize,
                                                                         lo, hi, c->src, c->dst);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return CC_OK;
}

}  // extern "C"
