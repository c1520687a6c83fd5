/*
 * contour.h -- C-ABI of the B200-native Contour connected-components hot path
 * (libcontour.so, built from paper_2311_02811_b200/csrc/ for sm_100a).
 *
 * The reference (minmapcc, /root/reference/pkg) is a Python package whose hot
 * path is reached through these Python call sites; each entry point below
 * names the reference interface it replaces.  Plain pointers and sizes only:
 * no torch / CUDA types appear in the signatures (streams and device buffers
 * travel as void* / uint32_t*).
 *
 * Error convention: every int-returning function returns
 *   CC_OK 0, CC_EINVAL 1 (-> ValueError), CC_ECAP 2 (-> IterationCapExceeded,
 *   errors.py:12-13), CC_ECUDA 3 (-> RuntimeError).  cc_last_error() gives
 *   the thread-local message of the last failure on the calling thread.
 *
 * Threading: a context serialises calls on itself (internal mutex); use one
 * context per caller thread for concurrency (SPEC.md:212 reentrancy).
 */
#ifndef CONTOUR_H
#define CONTOUR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_OK 0
#define CC_EINVAL 1
#define CC_ECAP 2
#define CC_ECUDA 3

/* Variant codes, in the order of VARIANTS (engine.py:46). */
#define CC_VAR_CSYN 0
#define CC_VAR_C1 1
#define CC_VAR_C2 2
#define CC_VAR_CM 3
#define CC_VAR_C11MM 4
#define CC_VAR_C1M1M 5

/* Schedule (engine.py:51-74): order_for(k) is evaluated per sweep. */
typedef struct cc_schedule {
    int32_t variant;
    int32_t high_order;
    int32_t warmup;
    int32_t sync;   /* 1: read L, lower a shadow, commit after the sweep (engine.py:288-291,310-311) */
    int32_t atomic; /* 1: lowering never lost (CAS loop, _kernels.py:79-93) -> red.global.min */
} cc_schedule;

/* cc_run flags */
#define CC_RUN_EARLY_CHECK 1   /* early_convergence_check after each changing sweep (engine.py:318-320) */
#define CC_RUN_COUNT_CHANGES 2 /* exact changed_per_sweep by label diff (engine.py:293,309) */
#define CC_RUN_SWEEP_TIMES 4   /* per-sweep device times (IterationStats.sweep_seconds) */
#define CC_RUN_FIRST_SCATTER 8 /* run sweep 1 as the load-free identity scatter (see cc_sweep) */
#define CC_RUN_HOST_LOOP 16    /* drive sweeps from the host even when the device-side
                                  loop applies.  Without COUNT_CHANGES / EARLY_CHECK /
                                  FIRST_SCATTER and in async mode, cc_run otherwise runs the
                                  whole convergence loop as ONE CUDA-graph launch (a
                                  conditional WHILE node around sweep + control kernels). */

/* Output of cc_run, the IterationStats contract (engine.py:77-90). */
typedef struct cc_stats {
    int64_t sweeps_executed;
    int64_t sweeps_until_stable;
    int32_t converged_by;      /* 0 "change-flag", 1 "early-check" */
    int32_t compress_rounds;   /* pointer-jumping rounds that changed something (0 after a correct run) */
    int64_t capacity;          /* entries available in the two caller arrays below */
    int64_t* changed_per_sweep;/* caller-owned or NULL; -1 = "changed, count not requested" */
    double* sweep_seconds;     /* caller-owned or NULL */
    double converge_seconds;   /* device time: label init -> compressed labels */
} cc_stats;

typedef struct cc_ctx cc_ctx;

/* Context on CUDA device `device`.  `stream` is a cudaStream_t (e.g. torch's
 * current stream) or NULL to create a private non-blocking stream. */
int cc_create(int device, void* stream, cc_ctx** out);
void cc_destroy(cc_ctx* ctx);
const char* cc_last_error(void);
int cc_version(void);
/* Staged-layout facts for measurement (bench.py's rooflines): out[0] layout
 * code, out[1] check-copy format (-1 none, 0 8-byte rows, 1 6-byte rows, 2
 * delta-packed groups), out[2] bytes one pass over the check copy streams,
 * out[3] work items, out[4] staged rows, out[5] / out[6] rows and bytes of the
 * canonical check copy (0 if none), out[7] its build status (0 built, 1 off or not
 * applicable, 2 a window beyond 2^31 rows, 3 no memory, 4 not under 55 % of the rows,
 * 5 side table full), out[8] its groups kept with raw sources (side table);
 * out[9] L2 windows of layout 4/6, out[10] windows sweep 1 runs on the tiles when it
 * is split (0 = not split), out[11] the bitmap parts that follow them, out[12] 1 if the
 * last cc_run ended on the uniting check (CC_OPT_CHECK_UNITE), out[13] 1 if the split
 * parts walk the canonical copy -- out[10..13] describe the last run (or, before any
 * run, a caller-driven cc_sweep); the first `count` entries are written. */
int cc_layout_info(cc_ctx* ctx, int64_t* out, int count);

/* ---- staging: the Graph input contract (graph.py:57-90, engine.py:268-270) ----
 * edges: (m, 2) row-major pairs, elem_bytes 4 (int32) or 8 (int64), as the
 * reference's g.edges.  Converted on device to packed uint32 SoA src[]/dst[]
 * with the endpoint range check of graph.py:73-79 (-> CC_EINVAL).
 * Host variant: the buffer is borrowed for the call only.  Pinned memory is
 * read by the copy engine directly; pageable memory (a numpy array) is
 * narrowed to uint32 pairs by the context's host threads into pinned staging
 * chunks, pipelined with the copy.  Device variant: device pointer. */
int cc_stage_edges(cc_ctx* ctx, const void* edges_host, int elem_bytes, int64_t m, int64_t n);
int cc_stage_edges_device(cc_ctx* ctx, const void* edges_dev, int elem_bytes, int64_t m, int64_t n);
/* Borrow caller-owned device SoA arrays (must outlive their use). */
int cc_attach_soa(cc_ctx* ctx, uint32_t* src_dev, uint32_t* dst_dev, int64_t m, int64_t n);
/* Borrow a caller-owned device label buffer of n+1 uint32 (slot n = exchange flag). */
int cc_attach_labels(cc_ctx* ctx, uint32_t* labels_dev);
int cc_labels_device(cc_ctx* ctx, uint32_t** labels_dev);

/* ---- the hot path: run_contour(g, schedule, threads, seed) (engine.py:248-328) ----
 * Initialise labels = arange(n), sweep with order_for(k) until a sweep
 * lowers nothing (ballot/OR flag) or the early check passes, then
 * pointer-jump compress.  cap: sweeps allowed (the reference uses n+2,
 * engine.py:275) -> CC_ECAP.  labels_out: host buffer of n elements of
 * out_elem_bytes (4 or 8), or NULL to leave labels on device (a pageable
 * buffer is filled from a pinned read-back buffer by the context's threads). */
int cc_run(cc_ctx* ctx, const cc_schedule* sched, int flags, int64_t cap,
           void* labels_out, int out_elem_bytes, cc_stats* stats);

/* Stage host edges (as cc_stage_edges) AND run (as cc_run) in one call --
 * run_contour(g, ...) for a graph in host memory.  Asynchronous runs without
 * FIRST_SCATTER / HOST_LOOP, staged in input or chunk-sorted
 * order (CC_OPT_STAGE_LAYOUT 0 or 2), run sweep 1 chunk by chunk right behind
 * the host-to-device copy (each chunk is swept as soon as it is staged, while
 * the next one is in flight), then its shortcut pass and early check, then
 * the device-side loop from sweep 2 if needed; sweep_seconds[0] is the span
 * of the streamed sweep.  With COUNT_CHANGES, sweep 1's exact count is the
 * number of cells it moved off the identity (no shortcut pass then) and the
 * counted host loop continues from sweep 2.  Every other case stages, then
 * runs. */
int cc_run_host(cc_ctx* ctx, const void* edges_host, int elem_bytes, int64_t m, int64_t n,
                const cc_schedule* sched, int flags, int64_t cap, void* labels_out,
                int out_elem_bytes, cc_stats* stats);

/* ---- building blocks (multi-GPU driver, tests) ---- */
int cc_init_labels(cc_ctx* ctx);
/* One sweep over the staged edges: sweep_edges(read, target, edges, 0, m, 0,
 * order, use_cas) (_kernels.py:35-102).  first=1 asserts the labels are the
 * identity (right after cc_init_labels): the sweep is then the load-free
 * scatter L[max(u,v)] min= min(u,v), identical to the reference's sweep 1 in
 * sync mode and a legal interleaving of it in async mode.  Leaves the
 * "wrote" flag on device; if wrote_out != NULL it is synchronously read back. */
int cc_sweep(cc_ctx* ctx, int order, int sync, int atomic, int first, int* wrote_out);
/* Asynchronous sweep number sweep_no (>= 1) of a host-driven run: on layout 6
 * sweep 1 runs split (CC_OPT_SPLIT_SWEEP) and later order-2 sweeps as bitmap
 * sweeps over the check copy, as inside cc_run. */
int cc_sweep_numbered(cc_ctx* ctx, int order, int atomic, int64_t sweep_no, int* wrote_out);
/* Staging-time edge layout (the analogue of the reference's CSR build at
 * Graph construction, graph.py:80,109-122): mode 0 keeps the input order,
 * mode 1 stably sorts all rows by src (radix sort on device, m < 2^31),
 * mode 2 sorts each consecutive chunk of CC_OPT_SORT_CHUNK rows by src, so
 * label gathers of consecutive rows coalesce; mode 3 groups all rows by dst
 * bucket (2^CC_OPT_BUCKET_SHIFT vertices) and sorts them by src inside each
 * bucket (one device radix sort, m < 2^31): order-2 async sweeps then hold
 * the bucket's labels in shared memory (the dst-bucketed sweep kernel);
 * mode 4 partitions rows by dst into L2-sized windows of 2^CC_OPT_TILE_SHIFT
 * vertices and sorts each window's rows by src (any m; 8m bytes scratch), so
 * a grid-stride sweep gathers dst labels from one L2-resident window at a
 * time -- for label arrays larger than L2 (RMAT-28: 1 GB); mode 5 (hybrid)
 * keeps the current row order for sweep 1 and builds a mode-3 copy of the
 * rows (8m more bytes) that the later order-2 sweeps and checks walk with
 * shared-memory dst slices; mode 6 is mode 4 plus a copy of the rows for the
 * early check (8m more bytes): inside each L2 window the rows regrouped by
 * 2^CC_OPT_CHECK_SHIFT-vertex dst buckets and src-sorted, walked with a
 * component bitmap (one bit per vertex: "labelled like the giant
 * component") whose dst part sits in shared memory -- the check then
 * streams rows instead of gathering labels; mode 7 relabels the vertices
 * that appear in edges by first appearance in the row order and keeps a copy
 * of the rows in those IDs (sparse graphs whose labels exceed L2, e.g. a
 * forest written tree by tree: the rows a sweep processes together then touch
 * nearby labels); asynchronous runs without exact counts sweep the copy and
 * map the labels back to the minimum original ID per component, every other
 * run uses the rows in input order; without locality in the input order the
 * build falls back to mode 4. */
int cc_reorder_edges(cc_ctx* ctx, int mode);

/* Tuning knobs of a context.  Store modes for async sweeps:
 * 0 plain store, 1 red.global.min, 2 L2 re-check then plain store,
 * 3 L2 re-check then red.min (atomic schedules accept only 1 and 3). */
#define CC_OPT_STORE_MODE_PLAIN 1  /* Schedule.atomic == False (default 0) */
#define CC_OPT_STORE_MODE_ATOMIC 2 /* Schedule.atomic == True (default 3) */
#define CC_OPT_SORT_CHUNK 3        /* rows per chunk of layout mode 2 (default 2^23) */
#define CC_OPT_BUCKET_SHIFT 5      /* layout 3: 2^shift labels per dst bucket (8..15, default 15) */
#define CC_OPT_ITEM_ROWS 6         /* layout 3: rows per work item (default 2^18) */
#define CC_OPT_BUCKET_THREADS 7    /* layout 3: threads per CTA (256/512/1024, default 1024) */
#define CC_OPT_TILE_SHIFT 8        /* layouts 4/6: 2^shift labels per L2 window.  Unset: 24 (64 MB),
                                      except layout 6 on a dense graph (m >= 4n) below 2^28
                                      vertices: n/16-vertex windows (>= 2^16), so that sweep 1
                                      splits there too; the buckets of CC_OPT_CHECK_SHIFT then
                                      default to min(20, this) */
#define CC_OPT_SHORTCUT 9          /* pointer-jumping passes L[v]=L[L[v]] after every async sweep
                                      without exact counting (0..8, default 1) */
#define CC_OPT_TILE_SPLIT 10       /* layout 4: independently src-sorted runs per window (default 2) */
#define CC_OPT_BUCKET_NOSMEM 11    /* layout 3: 1 = gather dst labels from global memory (experiment) */
#define CC_OPT_SWEEP_VARIANT 12    /* order-2 kernel: 0 8 rows/thread, 1 4 rows, 2 8 rows <=64 regs,
                                      3 16 rows, 4 4 rows <=40 regs, 5 4 rows <=32 regs,
                                      6 4 rows + evict-first src gathers, 7 = 6 + evict-last dst
                                      gathers, 8 4 rows + evict-last dst gathers, 9 4 rows +
                                      evict-first edge stream, 10 = 9 + evict-last src and dst
                                      gathers, 11 = 9 + evict-last dst gathers, 12 auto: on
                                      layout 4 13 if m < 4n else 18, elsewhere 1 (default 12),
                                      13 = 11 with 16 rows/thread, 14 = 13 capped at 128 regs
                                      (2 blocks/SM), 15 = 11 with 8 rows/thread, 3 blocks/SM,
                                      16 L1-bypassing dst gathers, 17 = 16 + evict-first edges,
                                      18 = 11 + evict-first src gathers */
#define CC_OPT_BUCKET_PIPE 13      /* layout 3/5 sweep kernel: 0 general, 1 lean slice kernel,
                                      2 lean + edge prefetch (default), 3 bulk-copy (TMA)
                                      pipelined, 3-stage ring */
#define CC_OPT_ITEM_ORDER 14       /* layout 3: 0 bucket-major work items (default), 1 run-major:
                                      rows cut into sort_chunk runs in input order, items ordered
                                      (run, bucket) so the GPU walks each run's src range in order,
                                      2 run-major with the items of a run staggered over src */
#define CC_OPT_WARP_TRANSPOSE 15   /* sorted layouts: store each 128-row block transposed so a
                                      warp's k-th gather reads 32 consecutive sorted rows (default
                                      1; applied when the layout is built) */
#define CC_OPT_SWEEP_CTAS 16       /* flat order-1/2/h sweeps: CTAs per SM (0 = auto, default:
                                      3 on dense L2-window tiles, else the occupancy limit) */
#define CC_OPT_CHECK_SHIFT 17      /* layout 6: 2^shift-vertex dst buckets of the check copy
                                      (7..20, default 20 = 128 KB of bitmap per CTA) */
#define CC_OPT_FLAT_BITS 18        /* early check on flat rows with the component bitmap:
                                      0 never, 1 always, 2 auto (default: labels beyond L2
                                      and m >= 4n, e.g. one-shot RMAT-28) */
#define CC_OPT_HOST_SUB 19         /* pageable host edges: rows narrowed per pinned sub-chunk
                                      (default 2^20; small enough to stay in the host's LLC
                                      until the copy engine reads it) */
#define CC_OPT_HOST_NT 20          /* 1: streaming (non-temporal) stores into the pinned
                                      sub-chunks (default 0: cached stores) */
#define CC_OPT_CHECK_PACK 21       /* layout 6 check copy: 2 (default) = delta-packed groups of
                                      128 rows (source offset from the group's first source in
                                      32 - shift bits | dst offset, 4.03 B/row) when they fit,
                                      else 1 = 6-byte rows (uint32 src + high offset bits, uint16
                                      low offset bits) when log2(n) + shift - 16 <= 32, else
                                      0 = 8-byte rows */
#define CC_OPT_SPLIT_SWEEP 23       /* layout 6, order-2 sweep 1: the first k L2 windows on the
                                      tiles, then the bitmap sweep over the check copy of the
                                      rest (0 = off: all windows on the tiles; -1 = auto, the
                                      default: a quarter of the windows on dense graphs) */
#define CC_OPT_SPLIT_REBUILD 24     /* split sweep 1: L2 windows per component bitmap (the bitmap
                                      is rebuilt from the current labels before every group of
                                      that many windows; 0 = one bitmap for all; -1 = auto,
                                      the default: 3/16 of the windows) */
#define CC_OPT_SPLIT_MASK 26        /* split sweep 1, explicit schedule: bit w set = a bitmap part
                                      starts at L2 window w (the lowest set bit ends the tiled
                                      part); 0 (default) = use the two options above */
#define CC_OPT_CANON_CHECK 27       /* layout 6: 1 (default) = also build a copy with each
                                      undirected pair once (canonical, de-duplicated; kept only
                                      if under 55 % of the rows) for the early check, which then
                                      runs on its own instead of folded into a bitmap sweep */
#define CC_OPT_CANON_SPAN_BITS 28   /* tests: canonical-copy groups whose source span reaches
                                      2^bits keep raw sources (side table); 0 (default) = only
                                      spans beyond the 32 - check_shift offset bits */
#define CC_OPT_CANON_GROUP_WINDOWS 29 /* tests: L2 windows per build group of the canonical copy
                                        (default 0 = up to 64, fewer if over 2^30 rows) */
#define CC_OPT_RELABEL_INTERLEAVE 30 /* layout 7: rows of each 2^block-row block of the relabeled
                                       copy interleaved with this stride (0 = off) */
#define CC_OPT_RELABEL_BLOCK 31      /* layout 7: log2 rows per interleave block (default 24) */
#define CC_OPT_SPLIT_SHORTCUT 32    /* split sweep 1: pointer-jumping passes before each bitmap
                                      part (more rows decided by the bitmap) */
#define CC_OPT_CANON_SWEEP 33      /* layout 6, when the canonical copy was built: 1 = the
                                      whole-graph bitmap sweeps (sweep 2 on) walk it, each
                                      undirected pair once; 2 = the split sweep 1's bitmap parts
                                      too; 0 = every bitmap sweep walks the dst-bucketed check
                                      copy (every row); -1 (default) = 2 in runs that end on
                                      the uniting check, else 1 */
#define CC_OPT_BITS_DEFER 36       /* publishing bitmap sweeps: every lane parks up to this many
                                      (0..4; 0 = off) undecided rows and the warp runs them as
                                      one batch when a list would overflow or the item ends;
                                      -1 (default) = 4 in runs that end on the uniting check,
                                      else 0 (late rows cost the plain check its one-sweep
                                      convergence) */
#define CC_OPT_CHECK_UNITE 35      /* layout 6 with a delta-packed copy, asynchronous C-2 runs
                                      (cc_run with CC_RUN_EARLY_CHECK, without exact counts):
                                      1 (default) = the early check after a changing sweep
                                      unites the trees of every row whose labels differ (the
                                      larger root lowered to the smaller, a conditional min
                                      assignment on the root cell) instead of failing, and
                                      pointer jumping finishes the labels -- the check pass is
                                      the last pass over the rows (DESIGN 5.32); sweep 1 then
                                      splits after a sixteenth of the windows with one bitmap;
                                      0 = the plain check (sweeps until it passes) */
#define CC_OPT_BITS_PUBLISH 34     /* layout 6, delta-packed copies: the bitmap sweeps set a
                                      vertex's bit as soon as a row leaves it at the root label
                                      (later rows of that vertex are decided by the bitmap
                                      again): 1 (default) = in the split sweep 1's parts, 2 = in
                                      every bitmap sweep, 0 = the bitmap stays as built */
#define CC_OPT_LINK_PACK 22        /* pageable host edges: 1 (default) = rows cross PCIe as
                                      ceil(2 log2(n) / 8) in {6, 7} bytes (u | v << log2 n)
                                      when that is under 8; 0 = uint32 pairs */
#define CC_OPT_STAGE_LAYOUT 4     /* layout applied while staging: 0 input order (default),
                                      2 chunk-sorted, each chunk sorted as soon as it lands,
                                      overlapped with the next chunk's host->device copy */
int cc_set_option(cc_ctx* ctx, int option, int64_t value);
/* Fold the wrote flag into label slot n for an allreduce-min exchange
 * (SURVEY 8(e)): first=1: labels[n] = wrote ? 0 : 1; first=0:
 * labels[n] = min(labels[n], wrote ? 0 : 1).  Clears the flag. */
int cc_fold_flag(cc_ctx* ctx, int first);
int cc_compress(cc_ctx* ctx, int* rounds_out);
/* Deterministic multi-GPU synchronous sweeps (last bullet),
 * replacing engine.py:288-291,309-311 across devices: cc_sync_sweep copies
 * labels -> shadow and lowers the shadow from this context's edges (read the
 * labels, atomic min into the shadow); the caller all-reduces the n shadow
 * entries with MIN over all ranks (cc_shadow_device gives the buffer, n+1
 * uint32); cc_sync_commit then counts the cells that changed and copies the
 * shadow into the labels.  Every sweep equals the single-device synchronous
 * sweep, so changed_per_sweep equals the reference's. */
int cc_sync_sweep(cc_ctx* ctx, int order, int* wrote_out);
int cc_sync_commit(cc_ctx* ctx, int64_t* changed_out);
int cc_shadow_device(cc_ctx* ctx, uint32_t** shadow_dev);
/* `passes` pointer-jumping passes L[v] = L[L[v]] without reading back (the
 * between-sweep shortcut of CC_OPT_SHORTCUT for drivers using cc_sweep). */
int cc_shortcut(cc_ctx* ctx, int passes);
/* early_convergence_check(g, labels) (engine.py:331-365) on device. */
int cc_early_check(cc_ctx* ctx, int* ok_out);
/* The same check as the device convergence loop runs it after a changing
 * sweep (layout-aware: shared-memory slices on the bucketed layouts, the
 * cache-hinted pass on L2-window tiles) on the current device labels. */
int cc_loop_check(cc_ctx* ctx, int* ok_out);
/* Size-independent certificate of the device labels: *result bit 0 = some
 * edge has L[u] != L[v], bit 1 = some L[L[x]] != L[x], bit 2 = some
 * L[x] > x; 0 means every component carries one root label <= its IDs. */
int cc_verify(cc_ctx* ctx, int* result);
int cc_read_labels(cc_ctx* ctx, void* out_host, int elem_bytes);
/* The staged rows [row_lo, row_hi) back to host memory as (rows, 2) pairs of
 * elem_bytes (4 or 8), in their current device order (input order until a
 * layout is applied; with layout 3 the bucketed order).  The inverse of
 * cc_stage_edges -- e.g. to hand a graph generated on the device
 * (cc_gen_rmat_device) to host-side callers such as the reference's own
 * Graph type.  Pageable destinations are filled by the context's threads
 * from pinned chunks, overlapped with the next chunk's copy. */
int cc_read_edges(cc_ctx* ctx, void* out_host, int elem_bytes, int64_t row_lo, int64_t row_hi);
/* Load caller labels (n int64 or int32 host values, each in 0..n-1, else
 * CC_EINVAL) as the device labels -- e.g. before cc_early_check on labels
 * from elsewhere (early_convergence_check(g, labels), engine.py:331-348). */
int cc_write_labels(cc_ctx* ctx, const void* labels_host, int elem_bytes);
int cc_synchronize(cc_ctx* ctx);

/* Single-edge operator mm_order(target, read, w, v, order, atomic)
 * (engine.py:209-231) run by the device edge routines on a private copy:
 * inplace=1 -> target is read (async form), else target is separate
 * (sync form).  Arrays are int64 host arrays of length n. */
int cc_mm_order(const int64_t* read, int64_t* target, int64_t n, int64_t w, int64_t v,
                int order, int inplace, int* changed_out);

/* ---- seeded synthetic inputs (definitions: oracle/gen.py) ---- */
/* RMAT rows [row_lo, row_hi) of the (symmetrised) edge list, generated on
 * device straight into the context's SoA arrays (a shard for multi-GPU). */
int cc_gen_rmat_device(cc_ctx* ctx, int scale, int edgefactor, uint64_t seed, uint32_t tA,
                       uint32_t tAB, uint32_t tABC, int symmetrize, int permute,
                       int64_t row_lo, int64_t row_hi);
/* Host generators writing (m,2) AoS rows of elem_bytes; out may be NULL to
 * count; *m_out receives the row count. */
int cc_gen_rmat_host(int scale, int edgefactor, uint64_t seed, uint32_t tA, uint32_t tAB,
                     uint32_t tABC, int symmetrize, int permute, int64_t row_lo, int64_t row_hi,
                     void* out, int elem_bytes, int threads);
int cc_gen_grid_host(int64_t rows, int64_t cols, uint32_t keep_thr, uint64_t seed, int permute,
                     void* out, int elem_bytes, int64_t* m_out, int threads);
int cc_gen_er_host(int64_t n, int64_t pairs, uint64_t seed, void* out, int elem_bytes,
                   int64_t* m_out);
int cc_gen_forest_host(const int64_t* sizes, int64_t components, int64_t n, uint64_t seed,
                       void* out, int elem_bytes, int64_t* m_out, int threads);

/* ---- fused sweep + exchange for multi-GPU runs ----
 * Instead of an allreduce-min of the n labels after every sweep, each
 * order-2 sweep sends every lowering it makes, as red.global.min, to the
 * label replicas of up to 7 peer GPUs (mapped with CUDA IPC, stores over
 * NVLink).  After a host barrier all replicas hold the min over all ranks'
 * lowerings; a round where no rank lowered anything is converged.
 * cc_ipc_get_handle: 64-byte cudaIpcMemHandle_t of the context's own label
 * buffer; cc_ipc_open/close: map/unmap a peer's handle; cc_set_peers: the
 * peer label pointers (device addresses valid in this context). */
int cc_ipc_get_handle(cc_ctx* ctx, void* handle_out);
int cc_ipc_open(cc_ctx* ctx, const void* handle, uint64_t* ptr_out);
int cc_ipc_close(cc_ctx* ctx, uint64_t ptr);
int cc_set_peers(cc_ctx* ctx, const uint64_t* ptrs, int npeers);

/* ---- FastSV baseline: fastsv(g) (baselines.py:81-131) on
 * the staged edges.  Synchronous hooking + shortcutting with atomic-min
 * proposals, so every iteration equals the reference's; stats as cc_run with
 * converged_by = 2 ("grandparent-stable"); flags: CC_RUN_SWEEP_TIMES. */
int cc_fastsv(cc_ctx* ctx, int64_t cap, void* labels_out, int out_elem_bytes, cc_stats* stats,
              int flags);

/* ---- ingestion: multi-threaded text parsers ----
 * Line semantics of load_edge_list (graph.py:149-197, mode 0: '#'/'%'
 * comments, exactly two integer tokens >= 0) and of the Matrix Market entry
 * lines (graph.py:203-274, mode 1: '%' comments, >= 2 tokens, first two
 * integers).  Rows go to out as int64 pairs in file order (out may be NULL
 * to count); on a malformed line returns CC_EINVAL with *err_line (1-based),
 * *err_code (CC_PARSE_*), *err_tokens (token count of that line) and
 * err_vals[0..1] (its two integers).  mode 1 with bound != 0 also rejects
 * entries outside 1..bound (CC_PARSE_RANGE; bound < 0 rejects every entry),
 * in file order with the other errors. */
#define CC_PARSE_TOKENS (-1)
#define CC_PARSE_NONINT (-2)
#define CC_PARSE_NEGATIVE (-3)
#define CC_PARSE_RANGE (-4)
int cc_parse_edges(const char* buf, int64_t len, int mode, int64_t* out, int64_t cap,
                   int64_t* m_out, int64_t* err_line, int* err_code, int* err_tokens,
                   int threads, int64_t bound, int64_t* err_vals);

/* ---- ingestion on the device ----
 * The reference loaders load_edge_list (graph.py:149-197) and the Matrix
 * Market body of load_matrix_market (graph.py:252-274) with the text moved to
 * HBM once: newline split, tokenising (the line semantics of cc_parse_edges,
 * one shared definition), canonical (min, max) rows, densification by
 * ascending original ID (np.unique + np.searchsorted, graph.py:186-194) and
 * sorted de-duplication (np.unique(axis=0), graph.py:142-146) run on the
 * device.  A handle owns its device buffers; results stay valid until the
 * next parse on it or cc_ingest_destroy.  Calls on one handle serialise. */
typedef struct cc_ingest cc_ingest;
int cc_ingest_create(int device, cc_ingest** out);
void cc_ingest_destroy(cc_ingest* h);
/* Parse host text buf[0, len) (pageable or pinned); errors as cc_parse_edges
 * (first malformed line in file order, 1-based).  canonical != 0 stores every
 * row as (min, max) (graph.py:133-139); mode 1 rows are made 0-based
 * (graph.py:267).  *m_out = rows kept. */
int cc_ingest_parse(cc_ingest* h, const char* buf, int64_t len, int mode, int64_t bound,
                    int canonical, int64_t* m_out, int64_t* err_line, int* err_code,
                    int* err_tokens, int64_t* err_vals);
/* The same for text already in device memory (on the handle's device). */
int cc_ingest_parse_device(cc_ingest* h, const char* text_dev, int64_t len, int mode,
                           int64_t bound, int canonical, int64_t* m_out, int64_t* err_line,
                           int* err_code, int* err_tokens, int64_t* err_vals);
/* remap != 0: densify IDs (*has_map = 1 when the IDs were not already 0..k-1);
 * dedupe != 0: sorted unique rows.  n_given >= 0 fixes n (Matrix Market
 * size line); else n = #distinct IDs (remap) or max ID + 1 (0 when empty). */
int cc_ingest_finish(cc_ingest* h, int remap, int dedupe, int64_t n_given, int64_t* n_out,
                     int64_t* m_out, int* has_map);
/* Device pointers of the result: edges (m, 2) int64, id map (n) int64 or NULL. */
int cc_ingest_result(cc_ingest* h, const int64_t** edges_dev, const int64_t** id_map_dev);
/* Copy the result to host or device memory (either pointer may be NULL). */
int cc_ingest_copy(cc_ingest* h, int64_t* edges_out, int64_t* id_map_out);

#ifdef __cplusplus
}
#endif

#endif /* CONTOUR_H */
