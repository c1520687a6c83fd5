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
#include <emmintrin.h>
#include <immintrin.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <tuple>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

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

// NVTX ranges around the C-ABI entry points (SURVEY §5 tracing): visible to
// ncu --nvtx / nsys; a no-op without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

#include "device_aux.inc"

#include "hostpool.inc"

#include "ctx.inc"

#include "launch.inc"

#include "loop.inc"

#include "staging.inc"

#include "relabel.inc"

#include "ingest.inc"

// ------------------------------------------------------------------ C-ABI
extern "C" {

const char* cc_last_error(void) { return g_err; }
int cc_version(void) { return 1; }

int cc_layout_info(cc_ctx* c, int64_t* out, int count) {
    if (!c || !out || count < 1) return fail(CC_EINVAL, "cc_layout_info: invalid argument");
    std::lock_guard<std::mutex> lk(c->mu);
    // sweep 1's split as the last run (or the next caller-driven sweep) takes it
    const int P = std::max(0, (int)c->win_start.size() - 1);
    int k = 0, parts = 0;
    if (split_sweep1(c)) {
        k = split_k(c);
        if (c->split_mask) {
            parts = __builtin_popcountll(c->split_mask >> k);
        } else {
            const int r = split_r(c) > 0 ? split_r(c) : P;
            parts = (P - k + r - 1) / r;
        }
    }
    const int64_t v[14] = {c->layout, c->layout == 6 ? (c->check_dp ? 2 : c->check_sbits ? 1 : 0) : -1,
                           c->layout == 6 ? c->check_bytes : 0, c->n_items, c->m,
                           c->citems ? c->canon_rows : 0, c->citems ? c->canon_bytes : 0,
                           c->canon_status, c->citems ? c->canon_side_groups : 0,
                           P, k, parts, c->unite_run ? 1 : 0,
                           (k > 0 && canon_sweep(c, true)) ? 1 : 0};
    for (int i = 0; i < count && i < 14; ++i) out[i] = v[i];
    return CC_OK;
}

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
    CUDA_TRY(cudaHostAlloc(&c->hflags, sizeof(int) * kNumFlags, cudaHostAllocMapped));
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
    cudaFree(c->bdst16);
    cudaFree(c->bits);
    cudaFree(c->cgbase);
    cudaFree(c->cwords);
    cudaFree(c->cgb);
    cudaFree(c->cside);
    cudaFree(c->citems);
    cudaFree(c->dr0);
    cudaFree(c->rlab);
    cudaFree(c->rorig);
    cudaFree(c->rmin);
    for (int b = 0; b < kNSub; ++b) {
        cudaFreeHost(c->hsub[b]);
        if (c->subdone[b]) cudaEventDestroy(c->subdone[b]);
    }
    cudaFreeHost(c->hlab);
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
    NvtxRange nvtx_("cc_stage_edges");
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return stage(c, edges, eb, m, n, true);
}

int cc_stage_edges_device(cc_ctx* c, const void* edges, int eb, int64_t m, int64_t n) {
    NvtxRange nvtx_("cc_stage_edges_device");
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
    NvtxRange nvtx_("cc_sweep");
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    c->unite_run = false;  // (caller-driven sweeps: the caller's check decides)
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

// An asynchronous sweep that knows its place in the run (1-based): on layout
// 6 sweep 1 is the split sweep and later order-2 sweeps the bitmap sweep over
// the check copy, as in cc_run -- for drivers that loop on the host (the
// multi-GPU CheckedShardedContour).
int cc_sweep_numbered(cc_ctx* c, int order, int atomic, int64_t sweep_no, int* wrote_out) {
    NvtxRange nvtx_("cc_sweep_numbered");
    if (!c) return fail(CC_EINVAL, "null context");
    if (sweep_no < 1) return fail(CC_EINVAL, "sweep number must be >= 1");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    c->unite_run = false;
    CC_TRY(enqueue_sweep(c, order, 0, atomic, false, false, sweep_no));
    if (wrote_out) {
        CC_TRY(read_flags(c));
        *wrote_out = c->hflags[kFlagWrote] != 0;
    }
    return CC_OK;
}

// Synchronous sweep split in two for the multi-GPU sync mode (SURVEY 8(e)
// last bullet): phase 1 lowers a shadow copy of the labels from this
// context's edge shard (read L, atomic min into the shadow); the caller then
// all-reduces the shadows with MIN across ranks -- min is associative, so
// the result is the single-device synchronous sweep's shadow exactly -- and
// phase 2 commits it (count cells changed, L = shadow; engine.py:309-311).
int cc_sync_sweep(cc_ctx* c, int order, int* wrote_out) {
    NvtxRange nvtx_("cc_sync_sweep");
    if (!c) return fail(CC_EINVAL, "null context");
    if (order < 1) return fail(CC_EINVAL, "operator order must be >= 1");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    CC_TRY(ensure_aux(c, true, false));
    if (c->n > 0)
        CUDA_TRY(cudaMemcpyAsync(c->shadow, c->labels, sizeof(lab_t) * c->n,
                                 cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 0, sizeof(int), c->stream));
    if (c->m > 0) CC_TRY(launch_order(c, c->labels, c->shadow, order, cck::kStoreCheckAllRed));
    if (wrote_out) {
        CC_TRY(read_flags(c));
        *wrote_out = c->hflags[kFlagWrote] != 0;
    }
    return CC_OK;
}

int cc_sync_commit(cc_ctx* c, int64_t* changed_out) {
    if (!c) return fail(CC_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    CC_TRY(ensure_aux(c, true, false));
    CUDA_TRY(cudaMemsetAsync(c->dcount, 0, sizeof(unsigned long long), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 0, sizeof(int), c->stream));
    if (c->n > 0) {
        k_commit<<<grid_for(c, c->n), kThreads, 0, c->stream>>>(c->labels, c->shadow, c->n,
                                                                c->dcount, c->dflags);
        CUDA_TRY(cudaGetLastError());
    }
    CC_TRY(read_flags(c));
    if (changed_out) *changed_out = (int64_t)*c->hcount;
    return CC_OK;
}

int cc_shadow_device(cc_ctx* c, uint32_t** out) {
    if (!c || !out) return fail(CC_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    CC_TRY(ensure_aux(c, true, false));
    *out = c->shadow;
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

// The early check exactly as the convergence loop runs it after a changing
// sweep (layout-aware halves: shared-memory slices on bucketed layouts,
// cache-hinted few-CTA pass on L2-window tiles) on the current labels.
int cc_loop_check(cc_ctx* c, int* ok) {
    if (!c || !ok) return fail(CC_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    *ok = 1;
    if (c->n == 0) return CC_OK;
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagCheck, 0, sizeof(int), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 1, 1, c->stream));  // "the sweep changed"
    CC_TRY(enqueue_loop_check(c, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 0, sizeof(int), c->stream));
    CC_TRY(read_flags(c));
    *ok = c->hflags[kFlagCheck] == 0;
    return CC_OK;
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
    const bool pageable = host_pageable(in);
    if (pageable) {  // narrowed by the context's threads into pinned memory (hostpool.inc)
        CC_TRY(ensure_hlab(c));
        uint32_t* h = c->hlab;
        ensure_pool(c)->run(c->n, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) {
                const int64_t x = eb == 8 ? ((const int64_t*)in)[i] : ((const int32_t*)in)[i];
                h[i] = (x < 0 || x > 0xFFFFFFFFll) ? 0xFFFFFFFFu : (uint32_t)x;
            }
        });
        CUDA_TRY(cudaMemcpyAsync(c->wide, h, sizeof(uint32_t) * c->n, cudaMemcpyHostToDevice,
                                 c->stream));
    } else {
        CUDA_TRY(cudaMemcpyAsync(c->wide, in, (size_t)eb * c->n, cudaMemcpyHostToDevice,
                                 c->stream));
    }
    CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagBad, 0, sizeof(int), c->stream));
    if (pageable)
        k_labels_in<uint32_t><<<grid_for(c, c->n), kThreads, 0, c->stream>>>(
            (const uint32_t*)c->wide, c->n, c->labels, c->dflags);
    else if (eb == 8)
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

}  // extern "C"

namespace {

// The staged rows back in host memory, in their current device order, as the
// reference's (m, 2) pair array: device AoS conversion per chunk, then the
// copy engine into pinned buffers that the context's threads hand over to a
// pageable destination while the next chunk is in flight (or straight into
// a pinned destination).
template <typename T>
int read_edges_impl(cc_ctx* c, T* out, int64_t lo, int64_t hi) {
    const int64_t chunk = (int64_t)1 << 23;
    const bool pageable = host_pageable(out);
    T* dbuf[2] = {nullptr, nullptr};
    T* hbuf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc = CC_OK;
    auto cleanup = [&]() {
        for (int b = 0; b < 2; ++b) {
            if (ev[b]) { cudaEventSynchronize(ev[b]); cudaEventDestroy(ev[b]); }
            cudaFree(dbuf[b]);
            cudaFreeHost(hbuf[b]);
        }
    };
    auto step = [&]() -> int {
        for (int b = 0; b < 2; ++b) {
            CUDA_TRY(cudaMalloc(&dbuf[b], sizeof(T) * 2 * chunk));
            if (pageable) CUDA_TRY(cudaHostAlloc(&hbuf[b], sizeof(T) * 2 * chunk, cudaHostAllocDefault));
            CUDA_TRY(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
        }
        int64_t prev_off = -1, prev_rows = 0;
        int k = 0;
        for (int64_t off = lo; off < hi; off += chunk, ++k) {
            const int b = k & 1;
            const int64_t rows = std::min<int64_t>(chunk, hi - off);
            k_unstage<T><<<grid_for(c, rows), kThreads, 0, c->stream>>>(c->src + off, c->dst + off,
                                                                        rows, dbuf[b]);
            CUDA_TRY(cudaGetLastError());
            T* target = pageable ? hbuf[b] : out + 2 * (off - lo);
            CUDA_TRY(cudaMemcpyAsync(target, dbuf[b], sizeof(T) * 2 * rows, cudaMemcpyDeviceToHost,
                                     c->stream));
            CUDA_TRY(cudaEventRecord(ev[b], c->stream));
            if (pageable && prev_off >= 0) {  // hand over the previous chunk meanwhile
                CUDA_TRY(cudaEventSynchronize(ev[b ^ 1]));
                const T* h = hbuf[b ^ 1];
                T* o = out + 2 * (prev_off - lo);
                ensure_pool(c)->run(prev_rows, [&](int64_t a, int64_t e) {
                    memcpy(o + 2 * a, h + 2 * a, sizeof(T) * 2 * (e - a));
                });
            }
            prev_off = off;
            prev_rows = rows;
        }
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (pageable && prev_off >= 0) {
            const T* h = hbuf[(k - 1) & 1];
            T* o = out + 2 * (prev_off - lo);
            ensure_pool(c)->run(prev_rows, [&](int64_t a, int64_t e) {
                memcpy(o + 2 * a, h + 2 * a, sizeof(T) * 2 * (e - a));
            });
        }
        return CC_OK;
    };
    rc = step();
    cleanup();
    return rc;
}

}  // namespace

extern "C" {

int cc_read_edges(cc_ctx* c, void* out, int eb, int64_t lo, int64_t hi) {
    NvtxRange nvtx_("cc_read_edges");
    if (!c) return fail(CC_EINVAL, "null context");
    if (eb != 4 && eb != 8) return fail(CC_EINVAL, "edge element size must be 4 or 8");
    std::lock_guard<std::mutex> lk(c->mu);
    if (lo < 0 || hi > c->m || lo > hi) return fail(CC_EINVAL, "bad row range");
    if (hi > lo && !out) return fail(CC_EINVAL, "null output buffer");
    if (hi == lo) return CC_OK;
    DeviceGuard g(c->device);
    if (eb == 4) return read_edges_impl<int32_t>(c, (int32_t*)out, lo, hi);
    return read_edges_impl<int64_t>(c, (int64_t*)out, lo, hi);
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
// start > 0: sweeps 1..start already ran (cc_run_host's streamed, counted
// sweep 1) and changed something; the host loop continues from start + 1.
int run_impl(cc_ctx* c, const cc_schedule* s, int flags, int64_t cap, void* labels_out,
             int out_eb, cc_stats* st, int64_t start = 0) {
    const bool sync = s->sync != 0;
    const bool count = (flags & CC_RUN_COUNT_CHANGES) != 0;
    const bool check = (flags & CC_RUN_EARLY_CHECK) != 0;
    const bool times = (flags & CC_RUN_SWEEP_TIMES) != 0;
    const bool first_scatter = (flags & CC_RUN_FIRST_SCATTER) != 0;
    // asynchronous C-2 runs without exact counts end on the uniting check
    // (sweep 1's split then follows it, launch.inc: split_k)
    c->unite_run = check && !sync && !count && !first_scatter && c->peers.n == 0 &&
                   unite_schedule(c, s);
    // layout 7: asynchronous runs without exact counts on the relabeled rows
    // (the dynamics differ from the original IDs', so parity modes use the
    // original rows in input order)
    if (c->layout == 7 && c->rlab && !sync && !count && !first_scatter && c->peers.n == 0 &&
        start == 0)
        return run_relabeled(c, s, flags, cap, labels_out, out_eb, st);
    if (!sync && !count && !first_scatter && !(flags & CC_RUN_HOST_LOOP) && c->n > 0 &&
        c->peers.n == 0 && start == 0)
        return run_graph(c, s, cap, labels_out, out_eb, st, check ? 1 : 0);
    CUDA_TRY(cudaEventRecord(c->evs, c->stream));
    if (start == 0) CC_TRY(enqueue_init(c, sync));
    int64_t sweep = start, until_stable = start;
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
        if (check) {  // the graph loop's check kernels (same layout-aware halves)
            CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagCheck, 0, sizeof(int), c->stream));
            // the check kernels skip when the wrote word is 0; this sweep changed
            // labels (sync / count modes tell it by the diff count)
            CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagWrote, 1, 1, c->stream));
            // (asynchronous runs without exact counts may unite disagreeing rows
            // instead of failing, as the graph loop does: the check then always
            // ends the loop and compress() below finishes the labels)
            const bool unite = c->unite_run;
            CUDA_TRY(cudaMemsetAsync(c->dflags + kFlagUnite, 0, sizeof(int), c->stream));
            CC_TRY(enqueue_loop_check(c, c->stream, unite));
            CC_TRY(read_flags(c));
            if (!c->hflags[kFlagCheck]) { converged_by = 1; break; }
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
    return !s->sync && !(flags & (CC_RUN_FIRST_SCATTER | CC_RUN_HOST_LOOP)) &&
           c->peers.n == 0 && (c->stage_layout == 0 || c->stage_layout == 2);
}

}  // namespace

extern "C" {

int cc_run(cc_ctx* c, const cc_schedule* s, int flags, int64_t cap, void* labels_out, int out_eb,
           cc_stats* st) {
    NvtxRange nvtx_("cc_run");
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
    NvtxRange nvtx_("cc_run_host");
    CC_TRY(check_run_args(c, s, labels_out, out_eb));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (!streamable(c, s, flags) || n == 0 || cap < 1) {
        CC_TRY(stage(c, edges_host, elem_bytes, m, n, true));
        return run_impl(c, s, flags, cap, labels_out, out_eb, st);
    }
    const bool check = (flags & CC_RUN_EARLY_CHECK) != 0;
    const bool count = (flags & CC_RUN_COUNT_CHANGES) != 0;
    CC_TRY(stage(c, edges_host, elem_bytes, m, n, true, s, check, labels_out, out_eb, count));
    const bool wrote = c->hflags[kFlagWrote] != 0;
    const int64_t changed1 = count ? (int64_t)*c->hcount : (wrote ? -1 : 0);
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
        const int rc = count ? run_impl(c, s, flags, cap, nullptr, out_eb, gs, 1)
                             : run_graph(c, s, cap, nullptr, out_eb, gs, check ? 1 : 0, 1);
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
        if (spec_valid) {
            if (c->pend_out) finish_pageable(c, c->pend_out, c->pend_eb);  // pinned -> caller
            c->pend_out = nullptr;
            labels_out = nullptr;
        }
    }
    if (st) {
        st->sweeps_executed = k;
        st->sweeps_until_stable = until_stable;
        st->converged_by = by;
        st->compress_rounds = rounds;
        st->converge_seconds = seconds;
        if (st->capacity >= 1) {
            if (st->changed_per_sweep) st->changed_per_sweep[0] = changed1;
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
    NvtxRange nvtx_("cc_fastsv");
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
    // any option but the staging layout may change what the captured graph loop launches
    if (option != CC_OPT_STAGE_LAYOUT) ++c->opt_epoch;
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
            if (value < 0 || value > 22) return fail(CC_EINVAL, "sweep variant must be 0..22");
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
            if (value < 0 || value > 3)
                return fail(CC_EINVAL, "item order must be 0 (bucket-major), 1 (run-major), "
                                       "2 (run-major, staggered) or 3 (src-major)");
            c->item_order = (int)value;
            return CC_OK;
        case CC_OPT_TILE_SPLIT:
            if (value < 1 || value > 1024) return fail(CC_EINVAL, "tile split must be 1..1024");
            c->tile_split = (int)value;
            return CC_OK;
        case CC_OPT_TILE_SHIFT:
            if (value < 10 || value > 30) return fail(CC_EINVAL, "tile shift must be in [10, 30]");
            c->tile_shift = (int)value;
            c->tile_shift_auto = false;
            return CC_OK;
        case CC_OPT_SWEEP_CTAS:
            if (value < 0 || value > 32) return fail(CC_EINVAL, "sweep CTAs per SM must be 0..32");
            c->sweep_ctas = (int)value;
            c->loop_key.m = -1;
            return CC_OK;
        case CC_OPT_FLAT_BITS:
            if (value < 0 || value > 2) return fail(CC_EINVAL, "flat bits must be 0, 1 or 2");
            c->flat_bits = (int)value;
            c->loop_key.m = -1;
            return CC_OK;
        case CC_OPT_RELABEL_INTERLEAVE:
            if (value < 0 || value > 4096) return fail(CC_EINVAL, "interleave must be 0..4096");
            c->relabel_interleave = (int)value;
            return CC_OK;
        case CC_OPT_RELABEL_BLOCK:
            if (value < 10 || value > 30) return fail(CC_EINVAL, "relabel block must be 10..30");
            c->relabel_block = (int)value;
            return CC_OK;
        case CC_OPT_CANON_GROUP_WINDOWS:
            if (value < 0 || value > 64) return fail(CC_EINVAL, "group windows must be 0..64");
            c->canon_group_windows = (int)value;
            return CC_OK;
        case CC_OPT_CANON_SPAN_BITS:
            if (value < 0 || value > 31) return fail(CC_EINVAL, "span bits must be 0..31");
            c->canon_span_bits = (int)value;
            return CC_OK;
        case CC_OPT_CANON_CHECK:
            c->canon_check = value != 0;
            return CC_OK;
        case CC_OPT_SPLIT_SHORTCUT:
            if (value < 0 || value > 4) return fail(CC_EINVAL, "split shortcut must be 0..4");
            c->split_shortcut = (int)value;
            return CC_OK;
        case CC_OPT_SPLIT_MASK:
            c->split_mask = (uint64_t)value;
            return CC_OK;
        case CC_OPT_SPLIT_REBUILD:
            if (value < -1 || value > kMaxTiles) return fail(CC_EINVAL, "split rebuild out of range");
            c->split_rebuild = (int)value;
            return CC_OK;
        case CC_OPT_SPLIT_SWEEP:
            if (value < -1 || value > kMaxTiles) return fail(CC_EINVAL, "split windows out of range");
            c->split_windows = (int)value;
            return CC_OK;
        case CC_OPT_LINK_PACK:
            c->link_pack = value != 0;
            return CC_OK;
        case CC_OPT_CHECK_PACK:
            if (value < 0 || value > 2) return fail(CC_EINVAL, "check pack must be 0..2");
            c->check_pack = (int)value;
            return CC_OK;
        case CC_OPT_HOST_SUB:
            if (value < 4096 || value > ((int64_t)1 << 26))
                return fail(CC_EINVAL, "host sub-chunk must be in [4096, 2^26] rows");
            c->host_sub = value & ~(int64_t)15;
            return CC_OK;
        case CC_OPT_HOST_NT:
            c->host_nt = value != 0;
            return CC_OK;
        case CC_OPT_CHECK_SHIFT:
            if (value < 7 || value > 20)
                return fail(CC_EINVAL, "check shift must be in [7, 20] (<= 128 KB of bits)");
            c->check_shift = (int)value;
            c->check_shift_auto = false;
            return CC_OK;
        case CC_OPT_CANON_SWEEP:
            if (value < -1 || value > 2)
                return fail(CC_EINVAL, "canon sweep must be -1 (auto), 0, 1 or 2");
            c->canon_sweep = (int)value;
            return CC_OK;
        case CC_OPT_BITS_DEFER:
            if (value < -1 || value > 4) return fail(CC_EINVAL, "bits defer must be in -1..4");
            c->bits_defer = (int)value;
            return CC_OK;
        case CC_OPT_CHECK_UNITE:
            c->check_unite = value != 0;
            return CC_OK;
        case CC_OPT_BITS_PUBLISH:
            if (value < 0 || value > 2) return fail(CC_EINVAL, "bits publish must be 0, 1 or 2");
            c->bits_publish = (int)value;
            return CC_OK;
        case CC_OPT_WARP_TRANSPOSE:
            c->warp_transpose = value != 0;
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


extern "C" {

int cc_reorder_edges(cc_ctx* c, int mode) {
    NvtxRange nvtx_("cc_reorder_edges");
    if (!c) return fail(CC_EINVAL, "null context");
    if (mode == 0) return CC_OK;
    if (mode < 1 || mode > 7) return fail(CC_EINVAL, "unknown edge layout mode %d", mode);
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (c->m < 2) return CC_OK;
    if (mode == 3 || mode == 5) return reorder_bucketed(c, mode);
    if (mode == 4 || mode == 6) {
        // Window and bucket sizes left to the library: 2^24-vertex L2 windows
        // (64 MB of labels) and 2^20-vertex buckets, except on a dense graph
        // (m >= 4n, where sweep 1 is split) with fewer than 2^28 vertices --
        // there n/16-vertex windows, so that mid-size graphs get RMAT-28's
        // sweep-1 schedule too (one window on the tiles, the rest as a bitmap
        // part: RMAT-24 2.87 -> 1.38 ms per run, RMAT-25 5.83 -> 2.72, RMAT-26
        // 6.07 -> 4.70, RMAT-27 9.9 -> 9.3; DESIGN 5.35)
        if (c->tile_shift_auto) {
            int lg = 0;
            while (((int64_t)1 << lg) < c->n) ++lg;
            const bool dense = mode == 6 && c->m >= 4 * c->n;
            c->tile_shift = dense ? std::min(24, std::max(16, lg - 4)) : 24;
        }
        if (c->check_shift_auto) c->check_shift = std::min(20, c->tile_shift);
        return reorder_l2tiles(c, mode);
    }
    if (mode == 7) return reorder_relabel(c);
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
