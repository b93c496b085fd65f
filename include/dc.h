/*
 * dc.h — C ABI of libdc: the B200 (sm_100a) calling-context-tree (CCT) aggregation path of
 * arXiv 2411.02797 ("DeepContext": a context-aware cross-platform profiler).
 *
 * PAPER.md below is the paper text; "§4.2" etc. are its sections.
 * DESIGN.md "Readings" R1..R21 resolve every place where the paper is silent or ambiguous.
 *
 * Conventions (all calls):
 *  - Every call returns dc_status. No exception or abort crosses the ABI; dc_last_error()
 *    gives a message for the last failing call on a context.
 *  - One dc_ctx = one CUDA device + one CUDA stream; a context is not thread-safe.
 *  - Device-pointer arguments ("dev") are caller-owned device memory (e.g. torch tensors);
 *    they must stay valid until the context's stream has passed the call. Host-pointer
 *    arguments ("host") are read or written before the call returns.
 *  - Calls are stream-ordered. Some calls read small counts back to the host to size their
 *    outputs and therefore synchronize the stream; each call says so. Argument errors
 *    (NULL where not allowed, zero sizes where not allowed, bad enums) are returned
 *    synchronously as DC_ERR_ARG. Data errors found on the device (frame id >= n_frames,
 *    raw key with kind == 0xFFFFFFFF, path deeper than DC_MAX_DEPTH, launch_leaf entry not a
 *    node of the tree) raise a device flag that dc_ctx_sync() — and every synchronizing call
 *    — reports as DC_ERR_TRACE. Lenient data conditions (bad launch index, bad stall id,
 *    zero sample count, empty path) are dropped/handled and counted in dc_diag (reading R16,
 *    SPEC.md:359 lenient correlation policy).
 *  - Opaque handles dc_cct / dc_dict / dc_comm are library-owned and freed by *_free.
 *    dc_cct_view_get() returns BORROWED device pointers valid until the handle is freed or
 *    mutated by a later call.
 *  - Integer results are exact. Metrics are u64 (reading R17: the caller guarantees that
 *    per-metric sums fit in 64 bits; sums of squares are kept in 128 bits).
 */
#ifndef DC_H
#define DC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DC_OK = 0,
  DC_ERR_ARG = 1,        /* invalid argument (synchronous) */
  DC_ERR_OOM = 2,        /* device allocation failed */
  DC_ERR_CUDA = 3,       /* CUDA runtime error */
  DC_ERR_NCCL = 4,       /* NCCL error */
  DC_ERR_CAPACITY = 5,   /* a size limit of this implementation was exceeded (message says which) */
  DC_ERR_TRACE = 6,      /* malformed trace data detected on the device */
  DC_ERR_COLLISION = 7,  /* cross-rank path-hash collision detected (merge) */
  DC_ERR_STATE = 8       /* call not allowed in the handle's current state */
} dc_status;

#define DC_MAX_DEPTH 1024u          /* longest call path accepted by dc_cct_build */
#define DC_MAX_STALL 32u            /* n_stall limit of dc_pc_sample_attribute */
#define DC_NO_NODE 0xFFFFFFFFu      /* parent of the root; frame of the root */
#define DC_METRIC_SAMPLES 0xFFFFFFFFu /* metric selector for the PC-sample count column */

/* Frame kinds (the identity rule of each kind is PAPER.md:344-346, §4.2). */
enum { DC_KIND_PY = 0, DC_KIND_OP = 1, DC_KIND_NATIVE = 2, DC_KIND_API = 3, DC_KIND_KERNEL = 4, DC_KIND_INSTR = 5 };

typedef struct dc_ctx dc_ctx;
typedef struct dc_cct dc_cct;
typedef struct dc_dict dc_dict;
typedef struct dc_comm dc_comm;

/* Cumulative per-context diagnostics (host copy). */
typedef struct {
  uint64_t empty_paths;          /* records with an empty call path (attributed to the root, R10) */
  uint64_t samples_bad_launch;   /* PC samples with launch >= n_launch (dropped, R16) */
  uint64_t samples_bad_stall;    /* PC samples with stall >= n_stall (dropped) */
  uint64_t samples_zero_count;   /* PC samples with count == 0 (dropped) */
  uint64_t collisions_detected;  /* path-hash collisions resolved exactly (build) or reported (merge) */
  uint64_t levels_built;         /* tree levels constructed */
  uint64_t max_depth_seen;       /* deepest call path seen */
  uint64_t bytes_moved_est;      /* algorithmic bytes of the calls so far */
} dc_diag;

/* ---------------------------------------------------------------------------- context */
/* device: CUDA ordinal. cuda_stream: the cudaStream_t every call of this context runs on,
   used as given (NULL = the legacy default stream); inputs produced and outputs consumed on
   that stream need no further synchronization. */
dc_status dc_ctx_create(int device, void* cuda_stream, dc_ctx** out);
/* Waits for the stream; returns DC_ERR_TRACE if a device data-error flag is set. */
dc_status dc_ctx_sync(dc_ctx* ctx);
/* Synchronizes, then copies the cumulative diagnostics to *out_h (host). */
dc_status dc_ctx_diag(dc_ctx* ctx, dc_diag* out_h);
void dc_ctx_destroy(dc_ctx* ctx);
const char* dc_last_error(const dc_ctx* ctx);
/* Number of kernels this library has launched on the context (bench evidence). */
uint64_t dc_ctx_launch_count(const dc_ctx* ctx);
/* Measurement support: with timing on, every call records CUDA events on the context stream
   around each stage ("intern", "build", "attribute", "pc", "rollup", "topk") and around the
   dominant single kernel launches ("k:<kernel>"). dc_ctx_timer_report synchronizes, writes
   "name count total_ms\n" lines (summed per name since the last report) into buf (host,
   len bytes, NUL-terminated) and resets the timers. */
dc_status dc_ctx_set_timing(dc_ctx* ctx, int on);
dc_status dc_ctx_timer_report(dc_ctx* ctx, char* buf, size_t len);
/* Grows the context's private stream-ordered memory pool (created by dc_ctx_create; every
   scratch and handle allocation of the library comes from it; its release threshold is
   infinity, which affects no other allocator of the process) to hold at least `bytes` by allocating
   and freeing one block on the context stream, then synchronizes. Later calls then carve their
   buffers from memory that is already mapped, instead of mapping new physical memory (a
   millisecond-scale stall) the first time a call needs more than any earlier one. Optional;
   results never depend on it. DC_ERR_OOM if the pool cannot grow that far. */
dc_status dc_ctx_reserve(dc_ctx* ctx, uint64_t bytes);
/* Synchronizes, then returns the context pool's cached free memory to the device down to
   keep_bytes (cudaMemPoolTrimTo). Memory held by live handles is unaffected. The pool itself is
   destroyed by dc_ctx_destroy (deferred until the last handle made on the context is freed). */
dc_status dc_ctx_trim(dc_ctx* ctx, uint64_t keep_bytes);

/* ------------------------------------------------------------------- a1: interning */
/* Raw frame key, 16 B. Identity: Python (PY, file string id, line);
   framework op (OP, operator-name string id, 0); C/C++ / GPU API / kernel / instruction
   (kind, library string id, module-relative PC) (R3-R5). kind == 0xFFFFFFFF is reserved. */
typedef struct { uint32_t kind; uint32_t str_id; uint64_t addr; } dc_frame_key;

/* dc_intern_frames — frame unification (§4.2 "collapsing frames that
   refer to the same locations").
   keys     dev  [n] raw keys, 16-B aligned.
   out_ids  dev  [n] u32: out_ids[j] = rank of keys[j] among the DISTINCT keys in
                 lexicographic (kind, str_id, addr) order (canonical frame id, R2).
   out_dict host: receives a new dictionary handle (the D distinct keys in rank order +
                 their kinds), used by dc_cct_build for kind masks and by the merge.
   n may be 0 (empty dictionary). Synchronizes (reads D). */
dc_status dc_intern_frames(dc_ctx* ctx, const dc_frame_key* keys, uint64_t n, uint32_t* out_ids, dc_dict** out_dict);
/* Builds a dictionary from D keys that are already distinct and sorted (pre-interned traces). */
dc_status dc_dict_from_sorted(dc_ctx* ctx, const dc_frame_key* keys, uint64_t D, dc_dict** out_dict);
uint64_t dc_dict_size(const dc_dict* d);
/* Borrowed device pointers: keys [D] (16 B each) and kinds [D] (u8). */
dc_status dc_dict_arrays(const dc_dict* d, const dc_frame_key** keys_dev, const uint8_t** kinds_dev);

/* --------------------------------------------------------------- a2/a3: CCT build */
/* A trace of R records in CSR form: record r's call path (root-most frame first) is
   frames[offsets[r] .. offsets[r+1]), each entry a canonical frame id < n_frames. */
typedef struct {
  uint64_t n_records;
  const uint64_t* offsets;  /* dev [R+1], offsets[0] == 0, non-decreasing */
  const uint32_t* frames;   /* dev [offsets[R]] */
} dc_paths;

/* dc_cct_build — CCT construction by inserting every call path and collapsing equal
   frames (Fig. "calling context"). The result has a root (id 0, frame
   DC_NO_NODE, depth 0, R1) plus one node per distinct non-empty path prefix; node ids are
   canonical: ordered by (depth, lexicographic frame-id path), i.e. breadth-first with
   children in ascending frame id (R2). Children of a node are contiguous.
   dict      may be NULL (then kind masks in views are ignored); else its size must be n_frames.
   out_leaf  dev [R] or NULL: node id of each record's full path (root for an empty path).
   out       host: receives the new handle, state BUILT. Synchronizes (reads sizes). */
dc_status dc_cct_build(dc_ctx* ctx, const dc_paths* paths, const dc_dict* dict, uint32_t n_frames,
                       uint32_t* out_leaf, dc_cct** out);

/* ------------------------------------------------- a4: exclusive metric attribution */
/* dc_cct_attribute_metrics — GPU metrics joined to their call path through the correlation
   id are aggregated at the path's bottom node "by sum, minimum, average,
   and standard deviation": per node the exact count, and per metric the
   exact sum, minimum and 128-bit sum of squares of the values whose record ends there.
   leaf     dev [n_records] node ids (from dc_cct_build's out_leaf).
   metrics  dev column-major [M][ld] u64: metric m of record r is metrics[m*ld + r].
   Accumulates (may be called repeatedly with further record chunks); M is fixed by the
   first call. State -> DIRTY. Asynchronous. */
dc_status dc_cct_attribute_metrics(dc_ctx* ctx, dc_cct* cct, const uint32_t* leaf, uint64_t n_records,
                                   const uint64_t* metrics, uint32_t M, uint64_t ld);

/* ---------------------------------------------------------- a5: inclusive rollup */
/* dc_cct_rollup — "once a metric has been updated at the bottom of a call path, it is
   propagated to the root node ... updating the metric along the entire call path"
   (PAPER.md:348): incl(n) = excl(n) (+) the excl of every descendant, with (+) = (+count,
   +sum, min, +sumsq) and the same for the PC-sample columns. Recomputes from the exclusive
   columns (idempotent). State -> ROLLED. Asynchronous. */
dc_status dc_cct_rollup(dc_ctx* ctx, dc_cct* cct);

/* ---------------------------------------------------- a6: PC-sampling attribution */
/* One instruction sample (CUPTI-style), 16 B. */
typedef struct { uint32_t launch, pc_off; uint16_t stall, flags; uint32_t count; } dc_pc_sample;

/* dc_pc_sample_attribute — instruction samples "extend the call path by inserting the PC of
   each instruction collected", with per-instruction stall reasons
   (PAPER.md:414-416). Sample s with launch < n_launch, stall < n_stall and count > 0 adds
   count to bin (ctx, pc_off, stall), ctx = launch_leaf[launch] (the kernel-launch record's
   node); checks in that order, each failure dropped and counted in dc_diag. The PC nodes are
   the distinct (ctx, pc_off) pairs, numbered n_nodes + rank in (ctx, pc_off) order (R15);
   bins are kept sorted by (pc node, stall). Each ctx's exclusive `samples` / `stall[s]`
   columns get the totals of its PC children (rolled up by dc_cct_rollup).
   s                 dev [n] samples.
   launch_leaf       dev [n_launch] node ids.
   launch_sample_off dev [n_launch+1] or NULL: if given, samples of launch l are exactly
                     s[off[l] .. off[l+1]) (as delivered per kernel activity buffer,
                     PAPER.md:355-356) and the context-owner histogram schedule is used; a
                     sample whose launch field disagrees with its segment is still
                     attributed by its own launch field. NULL: samples in any order; with
                     n_launch <= 49,152 they are first partitioned by launch on the device (a
                     scratch copy of the samples, n x 16 B) and the context-owner schedule runs
                     on the copy; with more launches an L2 hash-table schedule is used. Same
                     results either way.
   n_stall           <= DC_MAX_STALL; fixed by the first call on a handle (DC_ERR_ARG if a
                     later call differs).
   Accumulates: may be called repeatedly, e.g. once per chunk / activity buffer of samples
   (the paper "flushes the metrics" per buffer). A later call's bins and PC
   nodes are merged exactly with the earlier ones (counts of equal (ctx, pc, stall) added, PC
   nodes renumbered over the union), so any split of the samples into calls gives the same
   tree as one call. On error the earlier results are kept. DC_ERR_STATE on a merged
   partition. Synchronizes (reads bin counts). State -> DIRTY. */
dc_status dc_pc_sample_attribute(dc_ctx* ctx, dc_cct* cct, const dc_pc_sample* s, uint64_t n,
                                 const uint32_t* launch_leaf, uint64_t n_launch,
                                 const uint64_t* launch_sample_off, uint32_t n_stall);

/* ------------------------------------------------------------------- a7: views */
typedef enum {
  DC_VIEW_INCLUSIVE = 0,  /* hotspot identification ① on inclusive values */
  DC_VIEW_EXCLUSIVE = 1,  /* same candidates ranked by exclusive values */
  DC_VIEW_BOTTOM_UP = 2,  /* per frame: sum of exclusive values over all nodes with that frame
                             ("aggregates individual metrics at the same node across different
                             call paths"); id = frame id */
  DC_VIEW_STALL = 3       /* stall reasons of node stall_node ranked by inclusive sample count
                             (analysis ④ topk(stalls)); id = stall id */
} dc_view;

typedef struct { uint32_t id; uint32_t _pad; uint64_t value; double fraction; } dc_topk_entry;

/* dc_hotspots_topk — for INCLUSIVE/EXCLUSIVE the candidates are the non-root nodes whose
   frame kind is in kind_mask (bit k = kind k; ignored when the tree has no dictionary);
   value = the metric's inclusive/exclusive sum (metric < M, or DC_METRIC_SAMPLES);
   fraction = (double)value / (double)total with total = the root's inclusive value
   ("total_time = call_tree.root.time"); for STALL, value = istall[s][node] and
   total = isamples[node]. Entries with fraction > threshold (strict, R12) are ordered by
   (value desc, id asc) and the first k are copied to out_h (host, room for k entries);
   *n_out_h = their number. total == 0 gives an empty list. Requires state ROLLED.
   Synchronizes. */
dc_status dc_hotspots_topk(dc_ctx* ctx, const dc_cct* cct, dc_view view, uint32_t metric, uint32_t kind_mask,
                           double threshold, uint32_t k, uint32_t stall_node, dc_topk_entry* out_h,
                           uint32_t* n_out_h);

/* a8: derived floats — "average, and standard deviation", population std
   (R7): mean = (double)sum / (double)count; std = sqrt(RN(count*sumsq - sum^2)) / (double)count
   with the radicand formed exactly in 256-bit and rounded once (R18); count == 0 gives 0, 0
   (R11). out_mean / out_std dev [n_nodes] f64. incl != 0 selects inclusive aggregates
   (requires ROLLED). Asynchronous. */
dc_status dc_cct_derived(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, int incl, double* out_mean,
                         double* out_std);

/* ------------------------------------------------------------- analyzer rules (NEXT-2)
   The example analyses of §4.3 as device predicates over a complete, rolled-up tree.
   Ratios are binary64 with single roundings; thresholds are the caller's (the paper fixes
   none except the ratio 2 of ③). */
typedef enum {
  DC_RULE_SMALL_KERNELS = 2, /* ② kernel fusion: node n (not the root)
                                qualifies if launches(n) > 0 and
                                (double)isum[metric_a](n) / (double)launches(n) < threshold,
                                launches(n) = xcnt summed over the nodes of n's subtree whose
                                frame kind is in kind_mask (records ending at kernel frames) */
  DC_RULE_BWD_FWD = 3,       /* ③ forward/backward: n (frame kind in kind_mask,
                                normally operators) qualifies if fwd = isum[metric_b](n) > 0, fwd >=
                                floor (the epsilon guard) and (double)isum[metric_a] / (double)fwd >
                                threshold (the paper's ratio 2); per node, no ancestor suppression
                                (SPEC.md analyze_fwd_bwd, reading R25). metric_a / metric_b are the
                                backward / forward time columns (a record's time goes to the column of
                                its direction; paths integrated with dc_seq_associate) */
  DC_RULE_CPU_LATENCY = 5    /* ⑤ CPU latency: n qualifies if
                                isum[metric_a](n) > floor and
                                (double)isum[metric_a] / (double)max(isum[metric_b], 1) > threshold
                                (SPEC.md analyze_cpu_latency: max(.,1) guard, absolute floor) */
} dc_rule;
typedef struct {
  uint32_t metric_a, metric_b, kind_mask, _pad;
  double threshold;
  uint64_t floor;
} dc_rule_params;

/* dc_analyze_flags — ids of the flagged nodes in breadth-first (= ascending id) order. For ② and
   ⑤ a node is flagged if it qualifies and no ancestor (the root excluded) qualifies — children
   of a flagged frame are not re-flagged (SPEC.md analyze_kernel_fusion / analyze_cpu_latency,
   reading R22); for ③ every qualifying node is flagged. Writes the first min(total, cap) ids to out_ids_h (host) and *n_out_h = total.
   Requires state ROLLED and a complete (not partitioned) tree. Synchronizes. */
dc_status dc_analyze_flags(dc_ctx* ctx, const dc_cct* cct, dc_rule rule, const dc_rule_params* params,
                           uint32_t* out_ids_h, uint32_t cap, uint32_t* n_out_h);

typedef struct { uint32_t node, stall; uint64_t count; } dc_stall_issue;

/* dc_analyze_stalls — analysis ④ (SPEC.md analyze_stalls): hotspots =
   dc_hotspots_topk(INCLUSIVE, metric, kind_mask, hot_threshold, all); for each hotspot n in
   that order, its instruction (PC) children c with (double)samples(c) / (double)isamples(n) >
   stall_threshold; per stall reason s, the sum of bin(c, s) over those children; the non-zero
   reasons ordered by (count desc, s asc), first k (<= 32) per hotspot, as {n, s, count}
   entries. Writes the first min(total, cap) entries to out_h; *n_out_h = total. Requires
   ROLLED. Synchronizes. */
dc_status dc_analyze_stalls(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, uint32_t kind_mask, double hot_threshold,
                            double stall_threshold, uint32_t k, dc_stall_issue* out_h, uint32_t cap,
                            uint32_t* n_out_h);

/* dc_export_folded — flame-graph folded stacks (SPEC.md export_folded;
   PAPER.md:444-447): one line per non-root node whose exclusive sum of `metric` is non-zero, in
   canonical (breadth-first) order: node_h[i], value_h[i] (the exclusive value), and its path =
   frames_h[off_h[i] .. off_h[i] + depth) (frame ids, outermost first; labels are the caller's).
   *n_lines_h / *n_frames_h receive the totals; when they exceed cap_lines / cap_frames nothing
   else is written (call again with room). Host buffers. The root's exclusive value (empty
   paths) has no stack and no line (reading R24). Requires metrics. Synchronizes. */
dc_status dc_export_folded(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, uint32_t* node_h, uint64_t* value_h,
                           uint64_t* off_h, uint32_t* frames_h, uint64_t cap_lines, uint64_t cap_frames,
                           uint64_t* n_lines_h, uint64_t* n_frames_h);

/* dc_cct_invert — SURVEY §8(f) NEXT-3, the bottom-up (caller-inverted) tree behind the paper's
   "switchable top-down and bottom-up views" (§4.4). Every non-root node n of
   cct whose exclusive value x(n) of `metric` (DC_METRIC_SAMPLES: PC samples) is non-zero
   contributes x(n) along its call path read innermost first: its own frame, its caller's, ...,
   the outermost frame (reading R27). *out receives a new ROLLED tree (library-owned, free with
   dc_cct_free) whose nodes are the distinct such reversed prefixes, in canonical (depth,
   lexicographic) order: its roots are the frames where the cost is spent (each root's inclusive
   value = that frame's DC_VIEW_BOTTOM_UP sum), their children the callers. Its single metric
   (index 0) holds, per inverted node q, the exact aggregate over the contributing nodes'
   values: isum = their sum, icnt = their number, imin / isq the minimum / square sum; the
   exclusive columns hold the nodes whose whole path reversed ends at q. The frame kinds are
   carried over (kind masks in views apply). cct must hold exclusive values (state DIRTY or
   ROLLED) and be complete (DC_ERR_STATE otherwise). Synchronizes. */
dc_status dc_cct_invert(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, dc_cct** out);

/* dc_cpu_intervals — CPU-sample interval attribution (PAPER.md:359-363
   "subtract the previous timestamp from it, and use the result as the interval between two
   samples"; SPEC.md attribute_cpu_sample). Samples in trace order: thread[n] (u32), kind[n]
   (u8: CPU_TIME / REAL_TIME / ...), ts[n] (u64, ns). For each (thread, kind) stream the first
   sample is the baseline (out_valid 0, out_interval 0); every later one gets ts - ts of the
   previous sample of its stream (out_valid 1). The intervals of the valid samples are then
   attributed to their call paths with dc_cct_attribute_metrics. Timestamps decreasing inside a
   stream are a trace error (DC_ERR_TRACE at the next synchronisation). Device pointers;
   asynchronous. */
dc_status dc_cpu_intervals(dc_ctx* ctx, const uint32_t* thread, const uint8_t* kind, const uint64_t* ts, uint64_t n,
                           uint64_t* out_interval, uint8_t* out_valid);

/* dc_seq_associate — forward/backward operator association (
   SPEC.md associate_backward): the forward registry is fwd_seq[nf] (sequence ids; < 0 = none,
   not registered) with the forward ops' Python + framework path prefixes (CSR fwd_off[nf+1],
   fwd_frames); it is a map, so a later entry with the same id replaces an earlier one. Each
   backward record r (bwd_seq[r], its own native/kernel path CSR bwd_off / bwd_frames) gets the
   integrated path = the registered forward prefix of its sequence id followed by its own
   frames; a record without a sequence id (< 0) keeps its path; an id missing from the registry
   keeps its path and is counted in *n_unmatched_h. out_off (device, [nb+1]) receives the
   integrated offsets; out_frames (device, cap_frames) the frames when *n_frames_h <= cap_frames
   (otherwise only the offsets: call again with room). Synchronizes. */
dc_status dc_seq_associate(dc_ctx* ctx, const int64_t* fwd_seq, const uint64_t* fwd_off, const uint32_t* fwd_frames,
                           uint64_t nf, const int64_t* bwd_seq, const uint64_t* bwd_off, const uint32_t* bwd_frames,
                           uint64_t nb, uint64_t* out_off, uint32_t* out_frames, uint64_t cap_frames, uint64_t* n_frames_h,
                           uint64_t* n_unmatched_h);

/* ------------------------------------------------------------- borrowed view */
typedef struct {
  uint64_t n_nodes, n_pc_nodes, n_bins, n_records;
  uint32_t n_metrics, n_stall, max_depth, n_frames;
  const uint32_t *parent, *frame;  /* [n_nodes] */
  const uint16_t* depth;           /* [n_nodes] */
  const uint32_t* level_off;       /* [max_depth+2]: nodes of depth d are [level_off[d], level_off[d+1]) */
  const uint64_t *xcnt, *icnt;     /* [n_nodes] */
  const uint64_t *xsum, *xmin, *xsq_lo, *xsq_hi, *isum, *imin, *isq_lo, *isq_hi; /* [n_metrics][n_nodes] */
  const uint64_t *xsamples, *isamples;  /* [n_nodes] */
  const uint64_t *xstall, *istall;      /* [n_stall][n_nodes] */
  const uint32_t *pc_ctx, *pc_off;      /* [n_pc_nodes] */
  const uint32_t* bin_pcnode;           /* [n_bins] */
  const uint16_t* bin_stall;            /* [n_bins] */
  const uint64_t* bin_count;            /* [n_bins] */
  int state;                            /* 0 BUILT, 1 DIRTY, 2 ROLLED */
} dc_cct_view;
/* dc_cct_view_get — fills *out_h with the handle's sizes and borrowed device pointers.
   The inclusive columns (icnt, isum, imin, isq_lo, isq_hi, isamples, istall) are defined only
   after dc_cct_rollup: in state BUILT or DIRTY they are returned as NULL and the call returns
   DC_ERR_STATE (every other field is still filled, so structure and exclusive columns can be
   read before the rollup). DC_OK in state ROLLED. */
dc_status dc_cct_view_get(const dc_cct* cct, dc_cct_view* out_h);
void dc_cct_free(dc_cct* cct);
void dc_dict_free(dc_dict* d);

/* ------------------------------------------------------- a9: cross-rank merge */
/* NCCL plumbing: rank 0 calls dc_nccl_unique_id and broadcasts the 128 bytes (e.g. with
   torch.distributed); every rank then calls dc_comm_create (collective). */
dc_status dc_nccl_unique_id(uint8_t out_h[128]);
/* dc_merge_plan — the exchange plan of dc_cct_merge_ranks step 4 (host only, no device work;
   exported so the multi-process host logic is testable without GPUs): given this rank's record
   counts per destination send_counts[P][2] (node records, bin records) and the counts every
   source sends to it recv_counts[P][2] (the all-to-all of send_counts), writes the offset of
   each destination's slab in the send buffer send_off[P][2], the offset at which each source's
   records land in the receive buffer recv_off[P][2] (sources in rank order) and the received
   totals recv_total[2]. All arrays are host memory, counts in records. */
dc_status dc_merge_plan(uint32_t P, const uint64_t* send_counts, const uint64_t* recv_counts, uint64_t* send_off,
                        uint64_t* recv_off, uint64_t* recv_total);
dc_status dc_comm_create(dc_ctx* ctx, const uint8_t uid[128], int nranks, int rank, dc_comm** out);
void dc_comm_destroy(dc_comm* comm);

/* dc_cct_merge_ranks — collective. Merged CCT == the CCT of the concatenation of every
   rank's records (R19; not in the paper). Dictionaries are unified into a global sorted
   dictionary (frame id = global rank), every node gets a 128-bit full-path hash, nodes are
   hash-partitioned across ranks and exchanged with NCCL over NVLink, and each rank reduces
   the nodes it owns. Collisions are detected exactly ((parent hash, frame, depth) must agree
   within a run) and reported as DC_ERR_COLLISION. local must be ROLLED; the output partition
   is ROLLED and holds only this rank's share (its ids are partition-local).
   Synchronizes. */
dc_status dc_cct_merge_ranks(dc_ctx* ctx, dc_comm* comm, const dc_cct* local, const dc_dict* local_dict,
                             dc_cct** out_partition, dc_dict** out_global_dict);
/* Gathers the partitions at `root` and canonicalizes them into one CCT (parity/views only):
   on `root` *out_canonical is a ROLLED tree in canonical (depth, lexicographic) order over the
   global dictionary; NULL on the other ranks. Collective; synchronizes. */
dc_status dc_cct_gather(dc_ctx* ctx, dc_comm* comm, const dc_cct* part, int root, dc_cct** out_canonical);
/* Single-GPU emulation of merge_ranks + gather for P logical ranks (loopback exchange through
   device copies instead of NCCL; same partition/reduce/verify/canonicalise kernels).
   locals[p] (ROLLED) with dicts[p]; returns the canonical merged tree and global dictionary.
   With P = 2 it is also the fold step of chunked / online aggregation:
   merge(CCT of chunks 0..k-1, CCT of chunk k) = CCT of chunks 0..k (reading R19). */
dc_status dc_cct_merge_local(dc_ctx* ctx, uint32_t P, dc_cct* const* locals, dc_dict* const* dicts, dc_cct** out_canonical,
                             dc_dict** out_global_dict);

#ifdef __cplusplus
}
#endif
#endif /* DC_H */
