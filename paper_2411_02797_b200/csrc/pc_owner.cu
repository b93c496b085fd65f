// pc_owner.cu — a6, context-owner schedule of the (context, pc, stall) histogram.
//
// When samples arrive contiguous per launch (launch_sample_off given, "flushes the metrics"
// per activity buffer), launches are ordered by their context node and the
// resulting ctx-ordered virtual sample stream is cut into num_SMs equal ranges of stages, one
// persistent CTA per SM; a CTA that finishes its range steals stages from the back of the
// range with the most unclaimed stages (per-CTA claim words), so the slowest range does not
// set the kernel time:
//   * the producer warp streams each stage's launch segments (32-sample rows, see the stage
//     plan below) into shared memory with TMA bulk copies (cp.async.bulk + mbarrier, 3 x 40 KB
//     stages) and decides the flush points;
//   * 20 consumer warps aggregate (pc_off, stall) -> count in an 11,776-slot shared-memory
//     hash table probed in 4-slot buckets (one 16-B load settles a hit; predicated
//     red.shared.add); misses are queued per warp and probed 32 at a time; warps run free
//     (no per-stage CTA barrier) and only meet at flushes;
//   * on a context change (or at 2/3 table load) the table is flushed once to a partial list
//     in HBM: each bin is written once per (CTA, context) segment — no global atomics on
//     bins, no L2 hash table.
// The global-bitmap reduce (k_br_*) then adds the partial entries into their final, canonical
// (pc, stall) slots (the per-context shared-memory sort reduce, k_own_reduce, takes contexts
// whose PC range is too wide for the bitmap).
// Any sample this schedule cannot take (a valid launch that disagrees with its segment,
// pc_off >= 2^27, a context whose partial list cannot be chunked into shared memory) makes
// the call fall back to the generic schedule (pc.cu) for the whole input — same result.
#include <stdlib.h>
#include <algorithm>
#include <vector>

#include "prim.cuh"

namespace dc {

#ifndef DC_OW_WARPS
#define DC_OW_WARPS 20
#endif
#ifndef DC_OW_CPS
#define DC_OW_CPS 1
#endif
constexpr int OW_CONS_WARPS = DC_OW_WARPS;  // consumer warps per CTA (A/B builds: others)
constexpr int OW_CPS = DC_OW_CPS;           // k_pc_owner CTAs per SM (A/B builds: 2)
constexpr int OW_CONS = 32 * OW_CONS_WARPS;   // 512 consumer threads
constexpr int OW_THREADS = OW_CONS + 32;      // + producer warp
#ifndef DC_OW_NOBR
#define DC_OW_NOBR 1  // branch-free hit / miss bookkeeping: 0.449 -> 0.435 ms (same-box A/B)
#endif
#ifndef DC_OW_PSTORE
#define DC_OW_PSTORE 1  // predicated miss-queue store: 0.385 -> 0.381 ms (same-box A/B)
#endif
#ifndef DC_OW_DYN
#define DC_OW_DYN 1  // consumer row groups by ticket: 0.424 -> 0.413 ms (same-box A/B)
#endif
#ifndef DC_OW_HINT
#define DC_OW_HINT 0  // preferred-slot lookup (A/B builds)
#endif
#ifndef DC_OW_STAGES
#define DC_OW_STAGES 3
#endif
constexpr int OW_STAGES = DC_OW_STAGES;  // (A/B builds: other counts)
constexpr int OW_PER_LANE = 4;                // samples per lane per stage
constexpr int OW_ROUND = 32 * OW_PER_LANE;    // samples per warp per stage
constexpr int OW_STAGE = OW_CONS_WARPS * OW_ROUND;  // 2560 samples per stage (40 KB)
#ifndef DC_OW_TAB
#define DC_OW_TAB 11776
#endif
constexpr int OW_TAB = DC_OW_TAB;             // shared hash table slots (92 KB)
constexpr int OW_PEND = OW_ROUND + 32;        // per-warp queue of missed keys (probed 32 at a time)
// a flush is requested at 2/3 load; past OW_SPILL_AT distinct keys new keys are not inserted
// but appended to the CTA's spill region in HBM (kept as partial entries), so the table can
// never overflow whatever the key cardinality. `distinct` lags by at most one round per warp.
#ifndef DC_OW_FLUSH_PCT
#define DC_OW_FLUSH_PCT 75
#endif
constexpr uint32_t OW_FLUSH_REQ = OW_TAB * DC_OW_FLUSH_PCT / 100;  // (A/B builds: other loads)
constexpr uint32_t OW_SPILL_AT = OW_TAB - OW_CONS_WARPS * OW_PEND - 1;
constexpr uint32_t OW_MISS = 0xFFFFFFFEu;
constexpr uint32_t OW_SPILL_CAP = 4096;       // spill chunk (entries); the first per CTA is preallocated
constexpr uint32_t OW_SP_RING = 8;            // spill chunk bases kept (by generation)
constexpr uint32_t OW_CLAIM = 8;              // stages claimed from the own range at a time
constexpr uint32_t OW_STEAL = 16;             // at most this many stages stolen at a time
constexpr uint32_t EMPTY32 = 0xFFFFFFFFu;
constexpr uint32_t OW_DONE = 0xFFFFFFFFu;

enum { OWF_FALLBACK = 1, OWF_OVERFLOW = 2 };

constexpr int OW_ROWS = OW_STAGE / 32;        // 32-sample rows per stage
struct __align__(16) OwMeta {
  uint32_t ctx, count, flush, epoch;  // epoch: flushes up to and including this stage (DC_OW_DYN)
  uint32_t row_launch[OW_ROWS];  // launch of each 32-sample row (pieces start on row boundaries)
  uint8_t row_valid[OW_ROWS];    // valid samples in the row (a launch's tail row is partial)
};

struct OwnSmem {
  uint4 stage[OW_STAGES][OW_STAGE];
  uint32_t key[OW_TAB];
  uint32_t cnt[OW_TAB + OW_CONS_WARPS];  // + one dummy counter per consumer warp (never read)
  uint32_t pend[OW_CONS_WARPS][OW_PEND + 1];  // + a dummy tail slot (never read)
  unsigned long long full[OW_STAGES], empty[OW_STAGES];
  OwMeta meta[OW_STAGES];
  uint32_t distinct;
  // counts above 1 added to the table since the last flush (aggregated records): a flush is
  // requested past OW_EXTRA_FLUSH so no 32-bit counter can wrap (see own_hot)
  uint32_t extra;
  uint32_t flush_req;
  // spill allocator: word = generation << 20 | entries taken in the generation's chunk; a full
  // chunk is closed as a segment and replaced by one from the global entry pool (sp_lock)
  uint32_t sp_word, sp_seg, sp_lock;  // sp_seg: entries of the current chunk already in a segment
  unsigned long long sp_base[OW_SP_RING];
  uint32_t warp_cnt[OW_CONS_WARPS];
  uint32_t warp_mx[OW_CONS_WARPS], warp_or[OW_CONS_WARPS];  // flush: per-warp key range of the segment
  uint32_t seg_si;
  unsigned long long seg_base;
  uint32_t ticket;  // DC_OW_DYN: next row group of the stage stream
};
static_assert(OW_CPS * (sizeof(OwnSmem) + 1024) <= 233472, "k_pc_owner shared memory past the SM");
static_assert(sizeof(OwnSmem) <= 232448, "k_pc_owner shared memory past the 227 KB opt-in limit");

__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(OW_CONS) : "memory"); }

// ---------------------------------------------------------------- prep kernels
__global__ void k_own_check(const uint64_t* __restrict__ off, uint64_t n_launch, uint64_t n, uint32_t* bad) { DC_PDL_ENTER();
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < n_launch; l += (uint64_t)gridDim.x * blockDim.x)
    if (off[l + 1] < off[l]) atomicOr(bad, 1u);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n_launch] != n)) atomicOr(bad, 1u);
}

__global__ void k_own_keys(const uint32_t* __restrict__ leaf, uint64_t n_launch, uint64_t N, uint64_t* __restrict__ key,
                           uint32_t* __restrict__ val) { DC_PDL_ENTER();
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < n_launch; l += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = leaf[l];
    key[l] = c < N ? c : N;
    val[l] = (uint32_t)l;
  }
}

// Launches ordered by context with a counting sort over the context ids (the order inside a
// context is irrelevant to the result): histogram with the offsets check fused in, a scan of the
// N + 1 counters, a scatter through atomic cursors. Three launches instead of check + keys + a
// multi-pass radix sort.
__global__ void k_own_hist(const uint32_t* __restrict__ leaf, const uint64_t* __restrict__ off, uint64_t n_launch, uint64_t n,
                           uint64_t N, uint32_t* __restrict__ hist, uint32_t* bad) { DC_PDL_ENTER();
  bool b = false;
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < n_launch; l += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = leaf[l];
    atomicAdd(&hist[c < N ? c : (uint32_t)N], 1u);
    b |= off[l + 1] < off[l];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n_launch] != n)) b = true;
  if (b) atomicOr(bad, 1u);
}
__global__ void k_own_scatter(const uint32_t* __restrict__ leaf, uint64_t n_launch, uint64_t N, uint32_t* __restrict__ cursor,
                              uint64_t* __restrict__ key, uint32_t* __restrict__ val) { DC_PDL_ENTER();
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < n_launch; l += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c0 = leaf[l], c = c0 < N ? c0 : (uint32_t)N;
    const uint32_t pos = atomicAdd(&cursor[c], 1u);
    key[pos] = c;
    val[pos] = (uint32_t)l;
  }
}

// ---- stage plan. The ctx-ordered launches are laid out as a stream of 32-sample rows: launch i
// takes rows_i = ceil(cnt_i / 32) rows (its last row partial), the launches of one context are
// contiguous and every context starts on a stage boundary (OW_ROWS rows), so a stage holds one
// context and every row one launch. Per row the plan stores the launch id and the number of
// valid samples (0 for padding); per stage, its first launch and context.
__global__ void k_plan_launch(const uint64_t* __restrict__ off, const uint32_t* __restrict__ order,
                              const uint64_t* __restrict__ lkey, uint64_t n_launch, uint64_t* __restrict__ lrow,
                              uint32_t* __restrict__ lflag, uint64_t* __restrict__ lsrc, uint64_t* __restrict__ lcnt) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_launch; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t l = order[i];
    const uint64_t b = off[l], e = off[l + 1];
    const uint64_t c = e > b ? e - b : 0;  // inconsistent offsets are rejected before the main kernel
    lrow[i] = (c + 31) / 32;
    lflag[i] = (i == 0 || lkey[i] != lkey[i - 1]) ? 1u : 0u;
    lsrc[i] = b;
    lcnt[i] = c;
  }
}

// gfirst[g] = first sorted launch of context group g; gfirst[NG] = n_launch
__global__ void k_plan_gfirst(const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ gx, const uint32_t* ng,
                              uint64_t n_launch, uint32_t* __restrict__ gfirst) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_launch; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i == 0 || lkey[i] != lkey[i - 1]) gfirst[gx[i]] = (uint32_t)i;
    if (i == n_launch - 1) gfirst[*ng] = (uint32_t)n_launch;
  }
}

// stages per group (0 past the last group, so the scan can run over the n_launch bound)
__global__ void k_plan_gstages(const uint64_t* __restrict__ E, const uint32_t* __restrict__ gfirst, const uint32_t* ng,
                               uint64_t n_launch, uint64_t* __restrict__ gst) { DC_PDL_ENTER();
  const uint32_t NG = *ng;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n_launch; g += (uint64_t)gridDim.x * blockDim.x)
    gst[g] = g < NG ? (E[gfirst[g + 1]] - E[gfirst[g]] + OW_ROWS - 1) / OW_ROWS : 0;
}

// one warp per launch: row position, row meta, stage starts
__global__ void k_plan_rows(const uint64_t* __restrict__ E, const uint32_t* __restrict__ gx,
                            const uint32_t* __restrict__ gfirst, const uint64_t* __restrict__ SB,
                            const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ order,
                            const uint64_t* __restrict__ lcnt, uint64_t n_launch, uint64_t row_cap,
                            uint64_t* __restrict__ rowpos, uint32_t* __restrict__ row_launch, uint8_t* __restrict__ row_valid,
                            uint32_t* __restrict__ st_first, uint32_t* __restrict__ st_ctx) { DC_PDL_ENTER();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = wid; i < n_launch; i += nw) {
    const uint32_t flag = (i == 0 || lkey[i] != lkey[i - 1]) ? 1u : 0u;
    const uint32_t g = gx[i] + flag - 1;
    const uint64_t rp = OW_ROWS * SB[g] + E[i] - E[gfirst[g]];
    const uint64_t rows = E[i + 1] - E[i], c = lcnt[i];
    const uint32_t l = order[i], ctx = (uint32_t)lkey[i];
    if (lane == 0) rowpos[i] = rp;
    for (uint64_t k = lane; k < rows; k += 32) {
      const uint64_t R = rp + k;
      if (R < row_cap) {
        row_launch[R] = l;
        row_valid[R] = (uint8_t)(c - 32 * k < 32 ? c - 32 * k : 32);
      }
    }
    if (rows > 0) {  // stages whose first row lies in this launch
      const uint64_t s_lo = (rp + OW_ROWS - 1) / OW_ROWS, s_hi = (rp + rows - 1) / OW_ROWS;
      for (uint64_t st = s_lo + lane; st <= s_hi; st += 32)
        if (OW_ROWS * st < row_cap) {
          st_first[st] = (uint32_t)i;
          st_ctx[st] = ctx;
        }
    }
  }
}

// Per stage, the TMA pieces the producer issues, precomputed so the producer warp does no
// dependent loads per stage: 4 x uint4 = {ctx, pieces, first launch, 0} and up to OW_DPIECES
// pieces {source sample lo, hi, samples, destination sample in the stage}. A stage with more
// pieces (more than OW_DPIECES launches) keeps its count and is cut by the producer itself.
constexpr uint32_t OW_DPIECES = 3;
__global__ void k_plan_pieces(const uint64_t* __restrict__ rowpos, const uint64_t* __restrict__ lsrc, const uint64_t* __restrict__ lcnt,
                              const uint32_t* __restrict__ st_first, const uint32_t* __restrict__ st_ctx,
                              const uint64_t* __restrict__ st_total, uint64_t n_launch, uint4* __restrict__ desc) { DC_PDL_ENTER();
  const uint64_t ST = *st_total;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < ST; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t R0 = OW_ROWS * s, R1 = R0 + OW_ROWS;
    const uint32_t f = st_first[s];
    uint32_t np = 0;
    for (uint64_t li = f; li < n_launch; ++li) {
      const uint64_t rp = rowpos[li], cnt = lcnt[li], rows = (cnt + 31) / 32;
      if (rp >= R1) break;
      if (rows == 0 || rp + rows <= R0) continue;
      const uint64_t r_lo = rp > R0 ? rp : R0, r_hi = rp + rows < R1 ? rp + rows : R1;
      const uint64_t lo = 32 * (r_lo - rp), hi = 32 * (r_hi - rp) < cnt ? 32 * (r_hi - rp) : cnt;
      const uint64_t src = lsrc[li] + lo;
      if (np < OW_DPIECES) desc[4 * s + 1 + np] = make_uint4((uint32_t)src, (uint32_t)(src >> 32), (uint32_t)(hi - lo), (uint32_t)(32 * (r_lo - R0)));
      ++np;
    }
    desc[4 * s] = make_uint4(st_ctx[s], np, f, 0u);
  }
}

// ---------------------------------------------------------------- main kernel
struct OwnArgs {
  const dc_pc_sample* smp;
  // stage plan (k_plan_*), per ctx-sorted launch i: first row, first sample, sample count
  const uint64_t* rowpos;
  const uint64_t* lsrc;
  const uint64_t* lcnt;
  const uint32_t* st_first;    // per stage: first launch, context
  const uint4* desc;           // per stage: TMA pieces (k_plan_pieces)
  const uint32_t* st_ctx;
  const uint32_t* row_launch;  // per row: launch id, valid samples
  const uint8_t* row_valid;
  const uint64_t* st_total;    // number of stages (device)
  uint64_t n_launch, N;
  uint32_t S;
  uint32_t* pkey;              // partial entries: key
  unsigned long long* pcnt;    //                  count
  uint64_t cap_entries;
  uint4* seg;                  // {ctx, n, base_lo, base_hi}
  uint2* seg_meta;             // per segment {max key + 1, OR of pc_off}: table flushes; {~0, 0} = unknown (spills)
  uint32_t cap_segs;
  unsigned long long* g_entries;
  unsigned int* g_segs;
  uint32_t* g_flags;
  uint32_t* trace_flags;       // ctx->d_flags (DC_ERR_TRACE conditions)
  unsigned long long* ldiag;
  uint64_t spill_base0;        // CTA b spills into pkey/pcnt[spill_base0 + b * OW_SPILL_CAP ...]
  uint32_t probe_mode;         // measurement only (DC_OWN_MODE): 1 = stream + keys, no table
  uint32_t* sink;
  const uint32_t* bad;         // launch_sample_off inconsistent (k_own_check): do nothing, generic schedule
  unsigned long long* claim;   // [gridDim.x] stage claim words, zeroed by the host
};

// all consumer threads; the caller has synchronised the consumers (every insert is done)
__device__ __forceinline__ void own_flush(OwnSmem& sm, const OwnArgs& a, uint32_t ctx, uint32_t ctid) {
  const uint32_t n = sm.distinct;
  const uint32_t w = ctid >> 5, lane = ctid & 31;
  if (ctid == 0) {
    unsigned long long base = ~0ull;
    if (n > 0) {
      base = atomicAdd(a.g_entries, (unsigned long long)n);
      const unsigned si = atomicAdd(a.g_segs, 1u);
      if (si < a.cap_segs && base + n <= a.cap_entries) {
        a.seg[si] = make_uint4(ctx, n, (uint32_t)base, (uint32_t)(base >> 32));
        sm.seg_si = si;
      } else {
        atomicOr(a.g_flags, (uint32_t)OWF_OVERFLOW);
        base = ~0ull;
      }
    }
    sm.seg_base = base;
    // this context's entries of the current spill chunk form their own segment
    const uint32_t wv = *(volatile uint32_t*)&sm.sp_word;
    const uint32_t sp_hi = min(wv & 0xFFFFFu, OW_SPILL_CAP);
    if (sp_hi > sm.sp_seg) {
      const uint64_t sb = sm.sp_base[(wv >> 20) % OW_SP_RING] + sm.sp_seg;
      const unsigned si2 = atomicAdd(a.g_segs, 1u);
      if (si2 < a.cap_segs) {
        a.seg[si2] = make_uint4(ctx, sp_hi - sm.sp_seg, (uint32_t)sb, (uint32_t)(sb >> 32));
        a.seg_meta[si2] = make_uint2(0xFFFFFFFFu, 0u);  // spill entries: range unknown
      } else {
        atomicOr(a.g_flags, (uint32_t)OWF_OVERFLOW);
      }
      sm.sp_seg = sp_hi;
    }
  }
  constexpr uint32_t PER_WARP = (OW_TAB / 32 + OW_CONS_WARPS - 1) / OW_CONS_WARPS * 32;  // 416 slots, multiple of 32
  const uint32_t s_lo = w * PER_WARP, s_hi = min((uint32_t)OW_TAB, s_lo + PER_WARP);
  uint32_t c = 0, mk = 0, orp = 0;
  for (uint32_t s = s_lo + lane; s < s_hi; s += 32) {
    const uint32_t k = sm.key[s];
    const bool occ = k != EMPTY32;
    c += __popc(__ballot_sync(0xffffffffu, occ));
    if (occ) {
      mk = max(mk, k + 1);
      orp |= k >> 5;
    }
  }
  mk = __reduce_max_sync(0xffffffffu, mk);
  orp = __reduce_or_sync(0xffffffffu, orp);
  if (lane == 0) {
    sm.warp_cnt[w] = c;
    sm.warp_mx[w] = mk;
    sm.warp_or[w] = orp;
  }
  cons_sync();
  if (ctid == 0 && n > 0 && sm.seg_base != ~0ull) {  // the segment's key range (k_ctx_hist skips a pass)
    uint32_t m2 = 0, o2 = 0;
    for (int ww = 0; ww < OW_CONS_WARPS; ++ww) {
      m2 = max(m2, sm.warp_mx[ww]);
      o2 |= sm.warp_or[ww];
    }
    a.seg_meta[sm.seg_si] = make_uint2(m2, o2);
  }
  const unsigned long long base = sm.seg_base;
  uint32_t pos = 0;
  for (uint32_t ww = 0; ww < w; ++ww) pos += sm.warp_cnt[ww];
  for (uint32_t s0 = s_lo; s0 < s_hi; s0 += 32) {
    const uint32_t s = s0 + lane;
    const uint32_t k = sm.key[s];
    const bool occ = k != EMPTY32;
    const uint32_t m = __ballot_sync(0xffffffffu, occ);
    if (occ && base != ~0ull) {
      const unsigned long long o = base + pos + __popc(m & lanemask_lt());
      a.pkey[o] = k;
      a.pcnt[o] = sm.cnt[s];
    }
    pos += __popc(m);
    sm.key[s] = EMPTY32;
    sm.cnt[s] = 0;
  }
  cons_sync();
  if (ctid == 0) {
    sm.distinct = 0;
    sm.extra = 0;
  }
  cons_sync();
}

// The table is probed in OW_BW-slot buckets (4: one 16-B shared load compares a key with a whole
// bucket, so a key displaced from its home slot usually still costs a single load; 2: 8-B loads,
// fewer bank-conflict wavefronts per warp, more displaced keys — A/B builds).
#ifndef DC_OW_BW
#define DC_OW_BW 1
#endif
#ifndef DC_OW_GW
#define DC_OW_GW 1  // width 1: misses walk aligned 4-slot groups (16-B loads) after the home slot
#endif
constexpr uint32_t OW_BW = DC_OW_BW;
static_assert(OW_BW == 1 || OW_BW == 2 || OW_BW == 4, "bucket width 1, 2 or 4");
constexpr uint32_t OW_NB = OW_TAB / OW_BW;
__device__ __forceinline__ uint32_t own_bucket(uint32_t key) { return __umulhi(key * 0x9E3779B1u, OW_NB); }
// preferred slot of a key within its home bucket (independent bits): new keys take it when it is
// free, so most lookups settle with one 4-B load of that slot instead of a 16-B bucket load
__device__ __forceinline__ uint32_t own_hint(uint32_t key) { return OW_BW == 1 ? 0u : (key * 0x27D4EB2Fu) >> (OW_BW == 4 ? 30 : 31); }
// a bucket's keys as a uint4 (width 2: .z / .w are never a key and never EMPTY: slot words only)
__device__ __forceinline__ uint4 bkt_ld(const uint32_t* p) {
  if (OW_BW == 4) return *reinterpret_cast<const uint4*>(p);
  if (OW_BW == 1) return make_uint4(*p, OW_MISS, OW_MISS, OW_MISS);
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  return make_uint4(v.x, v.y, OW_MISS, OW_MISS);
}
__device__ __forceinline__ int bucket_match(const uint4 v, uint32_t key) {
  return v.x == key ? 0 : (OW_BW >= 2 && v.y == key) ? 1 : (OW_BW == 4 && v.z == key) ? 2 : (OW_BW == 4 && v.w == key) ? 3 : -1;
}
__device__ __forceinline__ uint4 ld_shared_v4_volatile(const uint32_t* p) {
  uint4 v;
  if (OW_BW == 4) {
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
  } else if (OW_BW == 2) {
    asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
    v.z = v.w = OW_MISS;
  } else {
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v.x) : "r"(smem_u32(p)));
    v.y = v.z = v.w = OW_MISS;
  }
  return v;
}

// branch-free bucket lookup: keys are unique in the table, so at most one compare holds
__device__ __forceinline__ uint32_t bucket_slot(const uint4 v, uint32_t key, uint32_t b) {
  if (OW_BW == 1) return v.x == key ? b : (uint32_t)OW_MISS;
  if (OW_BW == 2) return (v.x == key) | (v.y == key) ? 2 * b + (v.y == key ? 1u : 0u) : (uint32_t)OW_MISS;
  const uint32_t j = (v.y == key ? 1u : 0u) | (v.z == key ? 2u : 0u) | (v.w == key ? 3u : 0u);
  return (v.x == key) | (j != 0u) ? 4 * b + j : (uint32_t)OW_MISS;
}
__device__ __forceinline__ void red_shared_inc_if(uint32_t* p, bool pred) {  // predicated, no branch
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.u32 p, %1, 0;\n@p red.shared.add.u32 [%0], 1;\n}\n" ::"r"(smem_u32(p)), "r"((uint32_t)pred)
      : "memory");
}

// Shared addresses as (base of the CTA's shared block, computed once) + offset: a generic ->
// shared conversion per use (smem_u32) costs a uniform S2UR / ULEA sequence in the hot loop.
__device__ __forceinline__ uint32_t s_off(const OwnSmem& sm, const void* p, uint32_t sb) {
  return sb + (uint32_t)((const unsigned char*)p - (const unsigned char*)&sm);
}
__device__ __forceinline__ uint32_t s_ld32v(uint32_t a) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 s_ld128v(uint32_t a) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t s_cas32(uint32_t a, uint32_t cmp, uint32_t val) {
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t s_inc32(uint32_t a, uint32_t lim) {
  uint32_t old;
  asm volatile("atom.shared.inc.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(lim) : "memory");
  return old;
}
__device__ __forceinline__ void s_mbar_wait(uint32_t a, uint32_t parity) {
  for (uint64_t i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (i > DC_SPIN_LIMIT) __trap();
  }
}
__device__ __forceinline__ void s_mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// slow path: the key is not in its home bucket (new key, or displaced). Returns the slot, or
// OW_TAB when the table is near full (the sample then goes to the spill region).
// returns slot | (1 << 31 if this call inserted the key)
#ifndef DC_OW_PROBE_CALL  // inlined: 0.454 -> 0.450 ms (same-box A/B); DC_OW_PROBE_CALL: A/B builds
__device__ __forceinline__
#else
__device__ __noinline__
#endif
uint32_t own_probe(OwnSmem& sm, uint32_t key, uint32_t b, uint32_t sb) {
  // `distinct` is refreshed once per warp round (not per insert), hence the margin in OW_SPILL_AT
  const bool full = *(volatile uint32_t*)&sm.distinct >= OW_SPILL_AT;
#if DC_OW_BW == 1 && DC_OW_GW
  {
    // Group walk: the home slot first (the fast path's 4-B lookup), then the aligned 4-slot
    // groups from the home slot's group on, one 16-B load each; a new key takes the home slot or
    // else the first empty slot in that order. Slots are never freed between flushes, so a group
    // with an empty slot ends the walk. (One slot per step measured ~8 steps per miss at 75 % load.)
    const uint32_t kb = s_off(sm, &sm.key[0], sb);
    const uint32_t k0 = s_ld32v(kb + 4 * b);
    if (k0 == key) return b;
    if (k0 == EMPTY32) {
      if (full) return OW_TAB;
      const uint32_t old = s_cas32(kb + 4 * b, EMPTY32, key);
      if (old == EMPTY32) return b | 0x80000000u;
      if (old == key) return b;
    }
    uint32_t g = b & ~3u;
    for (uint32_t walked = 0;; ++walked) {
      if (walked > OW_TAB / 4 + 1) return OW_TAB;  // cannot happen below OW_SPILL_AT; spill rather than spin
      const uint4 v = s_ld128v(kb + 4 * g);
      const uint32_t hit = (v.x == key ? 1u : 0u) | (v.y == key ? 2u : 0u) | (v.z == key ? 4u : 0u) | (v.w == key ? 8u : 0u);
      if (hit) return g + __ffs(hit) - 1;
      uint32_t empt = (v.x == EMPTY32 ? 1u : 0u) | (v.y == EMPTY32 ? 2u : 0u) | (v.z == EMPTY32 ? 4u : 0u) | (v.w == EMPTY32 ? 8u : 0u);
      if (empt && full) return OW_TAB;
      while (empt) {
        const uint32_t q = __ffs(empt) - 1;
        empt &= empt - 1;
        const uint32_t old = s_cas32(kb + 4 * (g + q), EMPTY32, key);
        if (old == EMPTY32) return (g + q) | 0x80000000u;
        if (old == key) return g + q;
      }
      // every slot of the group taken (possibly just now by other keys): the next group. A slot
      // whose CAS lost to another key cannot hold this key, so re-reading the group is not needed.
      g = g + 4 == (uint32_t)OW_TAB ? 0u : g + 4;
    }
  }
#else
  for (uint32_t walked = 0;; ++walked) {
    if (walked > 2 * OW_NB) return OW_TAB;  // cannot happen below OW_SPILL_AT; spill rather than spin
    const uint4 v = ld_shared_v4_volatile(&sm.key[OW_BW * b]);
    const int j = bucket_match(v, key);
    if (j >= 0) return OW_BW * b + j;
    uint32_t empt = (v.x == EMPTY32 ? 1u : 0u) | (OW_BW >= 2 && v.y == EMPTY32 ? 2u : 0u) |
                    (OW_BW == 4 ? (v.z == EMPTY32 ? 4u : 0u) | (v.w == EMPTY32 ? 8u : 0u) : 0u);
    if (empt && full) return OW_TAB;
    if (DC_OW_HINT && walked == 0) {  // home bucket: the key's preferred slot first
      const uint32_t hq = own_hint(key);
      if ((empt >> hq) & 1u) {
        const uint32_t old = atomicCAS(&sm.key[OW_BW * b + hq], EMPTY32, key);
        if (old == EMPTY32) return (OW_BW * b + hq) | 0x80000000u;
        if (old == key) return OW_BW * b + hq;
        empt &= ~(1u << hq);
      }
    }
    while (empt) {
      const uint32_t q = __ffs(empt) - 1;
      empt &= empt - 1;
      const uint32_t old = atomicCAS(&sm.key[OW_BW * b + q], EMPTY32, key);
      if (old == EMPTY32) return (OW_BW * b + q) | 0x80000000u;
      if (old == key) return OW_BW * b + q;
    }
    b = b + 1 == OW_NB ? 0u : b + 1;
  }
#endif
}

// One exact partial entry outside the table (table full, or a sample whose count is not 1).
// Entries go to the CTA's current spill chunk; the thread that finds the chunk full (and wins
// sp_lock) closes it as a segment of the current context (all consumers are in one context
// between flushes), takes a fresh chunk from the global entry pool and opens the next
// generation; the others wait for it and retry. Entries never exceed the samples, so the pool
// (n + 1 + one chunk per CTA) cannot run out.
__device__ __noinline__ void own_spill(OwnSmem& sm, const OwnArgs& a, uint32_t key, uint32_t count, uint32_t ctx) {
  for (uint32_t spin = 0;; ++spin) {
    if (spin > DC_SPIN_LIMIT) __trap();
    const uint32_t wv = atomicAdd(&sm.sp_word, 1u);
    const uint32_t gen = wv >> 20, i = wv & 0xFFFFFu;
    if (i < OW_SPILL_CAP) {
      const uint64_t o = *(volatile unsigned long long*)&sm.sp_base[gen % OW_SP_RING] + i;
      a.pkey[o] = key;
      a.pcnt[o] = count;
      return;
    }
    if (atomicCAS(&sm.sp_lock, 0u, 1u) == 0u) {
      if ((*(volatile uint32_t*)&sm.sp_word >> 20) == gen) {  // nobody replaced the chunk yet
        const uint64_t cb = sm.sp_base[gen % OW_SP_RING];
        if (OW_SPILL_CAP > sm.sp_seg) {
          const uint64_t sb = cb + sm.sp_seg;
          const unsigned si = atomicAdd(a.g_segs, 1u);
          if (si < a.cap_segs) {
            a.seg[si] = make_uint4(ctx, OW_SPILL_CAP - sm.sp_seg, (uint32_t)sb, (uint32_t)(sb >> 32));
            a.seg_meta[si] = make_uint2(0xFFFFFFFFu, 0u);  // spill entries: range unknown
          } else {
            atomicOr(a.g_flags, (uint32_t)OWF_OVERFLOW);
          }
        }
        const unsigned long long nb = atomicAdd(a.g_entries, (unsigned long long)OW_SPILL_CAP);
        if (nb + OW_SPILL_CAP > a.cap_entries) atomicOr(a.g_flags, (uint32_t)OWF_OVERFLOW);  // cannot happen
        *(volatile unsigned long long*)&sm.sp_base[(gen + 1) % OW_SP_RING] =
            nb + OW_SPILL_CAP > a.cap_entries ? a.spill_base0 + (uint64_t)blockIdx.x * OW_SPILL_CAP : nb;
        *(volatile uint32_t*)&sm.sp_seg = 0;
        __threadfence_block();
        atomicExch(&sm.sp_word, ((gen + 1) & 0xFFFu) << 20);
      }
      __threadfence_block();
      atomicExch(&sm.sp_lock, 0u);
    } else {
      while ((*(volatile uint32_t*)&sm.sp_word >> 20) == gen && (*(volatile uint32_t*)&sm.sp_word & 0xFFFFFu) >= OW_SPILL_CAP) {
      }
    }
  }
}

__device__ __forceinline__ void own_add(OwnSmem& sm, const OwnArgs& a, uint32_t key, uint32_t h, uint32_t add, uint32_t ctx) {
  if (h == (uint32_t)OW_TAB) {  // table full: one exact partial entry in the spill chunk
    own_spill(sm, a, key, add, ctx);
    return;
  }
  // Fire-and-forget shared reduction. Only samples with count == 1 reach the table (others
  // go to the spill region), so a counter gains at most one per sample of the CTA between
  // flushes and cannot wrap below 2^32 samples per CTA.
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(&sm.cnt[h])), "r"(add) : "memory");
}

struct OwCounters {
  uint32_t bad_l, bad_s, zero, fallback;
};

// rare path: classify a sample that failed the fused validity test (same order of checks as
// the generic schedule: launch, stall, count)
__device__ __noinline__ uint32_t own_reject(uint32_t launch, uint32_t stall, uint32_t count, uint32_t seg_launch, uint64_t n_launch,
                                            uint32_t S, bool ctx_ok, uint32_t* trace_flags) {
  // returns the counter to bump: 0 bad launch, 1 bad stall, 2 zero count, 3 fallback, 4 none
  if (launch >= n_launch) return 0;
  if (launch != seg_launch) return 3;  // misplaced sample: generic schedule
  if (stall >= S) return 1;
  if (count == 0) return 2;
  if (!ctx_ok) {
    atomicOr(trace_flags, (uint32_t)FLAG_BAD_LEAF);
    return 4;
  }
  return 3;  // pc_off >= 2^27 - 1 (key would not fit 32 bits)
}

// Hot path: a raw sample (count 1) of its row's launch with a valid stall -> key (pc_off << 5 |
// stall). Everything else takes own_cold: invalid samples are classified and counted, samples
// with count > 1 (aggregated records) are kept exactly as partial entries in the spill region.
// Counts 2 .. 2^16 - 1 (per-PC aggregated records, as CUPTI's PC-sampling API delivers them)
// take the cold path but are added in the table too when their key is in its home bucket
// (else an exact spill entry): a slot's counter then gains at most (samples of the CTA between
// flushes) + (counts above 1 since the last flush); the second term is kept below
// OW_EXTRA_FLUSH + the stages already in flight (4 x 2,048 x 65,535 < 2^30) by a flush request,
// so a counter stays below 2^32 for fewer than 2^31 samples per CTA between flushes. The fast
// path itself handles count == 1 only (a count test there cost 4 % of the kernel).
constexpr uint32_t OW_MAX_HOT_COUNT = 65535u;
constexpr uint32_t OW_EXTRA_FLUSH = 1u << 30;
__device__ __forceinline__ bool own_hot(const uint4 q, uint32_t row_launch, uint32_t S) {
  return (q.x == row_launch) & ((q.z & 0xFFFFu) < S) & (q.w == 1u) & (q.y < (1u << 27) - 1u);
}
// returns 1 when this call inserted a new key into the table (the caller publishes it)
__device__ __noinline__ uint32_t own_cold(const uint4 q, uint32_t seg_launch, const OwnArgs& a, bool ctx_ok, OwCounters& k,
                                          OwnSmem& sm, uint32_t ctx) {
  const uint32_t stall = q.z & 0xFFFFu;
  const bool ok = (q.x == seg_launch) & (stall < a.S) & (q.w != 0) & (q.y < (1u << 27) - 1u) & ctx_ok & (q.x < a.n_launch);
  if (ok) {  // valid sample with count > 1
    const uint32_t key = (q.y << 5) | stall;
    if (q.w <= OW_MAX_HOT_COUNT) {  // the table path, with the counts-above-1 budget
      const uint32_t before = atomicAdd(&sm.extra, q.w - 1u);
      if (before < OW_EXTRA_FLUSH && before + (q.w - 1u) >= OW_EXTRA_FLUSH) *(volatile uint32_t*)&sm.flush_req = 1u;
      const uint32_t bb = own_bucket(key);
      const uint4 v = ld_shared_v4_volatile(&sm.key[OW_BW * bb]);
      uint32_t sl = bucket_slot(v, key, bb);
      uint32_t ins = 0;
      if (sl == OW_MISS) {  // new or displaced key: probe, inserting it (round 2: per-PC aggregated
                            // records used to spill every key not yet in the table)
        const uint32_t r = own_probe(sm, key, bb, smem_u32(&sm));
        ins = r >> 31;
        sl = r & 0x7FFFFFFFu;
      }
      if (sl != (uint32_t)OW_TAB) {
        atomicAdd(&sm.cnt[sl], q.w);
        return ins;
      }
    }
    own_spill(sm, a, key, q.w, ctx);  // table full, or a count past 2^16
    return 0;
  }
  const uint32_t r = own_reject(q.x, stall, q.w, seg_launch, a.n_launch, a.S, ctx_ok, a.trace_flags);
  k.bad_l += r == 0;
  k.bad_s += r == 1;
  k.zero += r == 2;
  k.fallback |= r == 3;
  return 0;
}

template <int MODE>  // 0 = the product; 1, 2, 3, 4, 9 = measurement variants (DC_OWN_MODE)
__global__ void __launch_bounds__(OW_THREADS, OW_CPS) k_pc_owner(OwnArgs a) { DC_PDL_WAIT();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  OwnSmem& sm = *reinterpret_cast<OwnSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  if (*a.bad) return;  // the stage plan is meaningless; the host reruns the generic schedule
  // range of this CTA: stages [s0, s1) of the plan
  const uint64_t G = gridDim.x, ST = *a.st_total;
  const uint64_t s0 = ST * blockIdx.x / G, s1 = ST * (blockIdx.x + 1) / G;
  for (uint32_t s = tid; s < OW_TAB; s += OW_THREADS) {
    sm.key[s] = EMPTY32;
    sm.cnt[s] = 0;
  }
  if (tid == 0) {
    for (int s = 0; s < OW_STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], OW_CONS_WARPS);
    }
    sm.distinct = 0;
    sm.extra = 0;
    sm.flush_req = 0;
    sm.sp_word = 0;
    sm.sp_seg = 0;
    sm.sp_lock = 0;
    sm.ticket = 0;
    sm.sp_base[0] = a.spill_base0 + (uint64_t)blockIdx.x * OW_SPILL_CAP;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < 32) {
    // ------------------------------------------------ producer warp
    // Per stage s the plan gives the first launch f; lane j cuts launch f + j to the stage's rows
    // [OW_ROWS s, OW_ROWS (s + 1)) and issues its own TMA bulk copy, lane 0 copies the row meta.
    // The launch fields of stage s + 1 are loaded while stage s is issued (and the per-stage
    // first-launch / context words 32 stages at a time, one batch ahead).
    const uint32_t lane = tid;
    uint32_t st = 0, ph = 0, prev_ctx = OW_DONE, epoch = 0;  // epoch: lane 0's flush count
    volatile uint32_t* freq = &sm.flush_req;
    const bool prof = MODE == 2 || MODE == 9;  // measurement only
    long long p_wait = 0, p_comp = 0, p_stages = 0, p_pieces = 0;
    const long long p_t0 = prof ? clock64() : 0;
    // ---- stage source. The CTA's own range [s0, s1) is claimed from the front, OW_CLAIM stages
    // at a time (claim word: stages taken from the front | from the back << 32). When it is
    // exhausted the CTA steals from the back of the range with the most unclaimed stages (at
    // most OW_STEAL at a time), so CTAs whose contexts cost more per sample (more distinct keys,
    // more flushes) do not set the kernel time. Any stage is processed by exactly one CTA.
    unsigned long long* const claim = a.claim;
    uint64_t c_lo = 0, c_hi = 0;    // claimed, not yet handed out
    unsigned long long w_pend = 0;  // lane 0: result of the outstanding front claim
    bool own = true;
    if (lane == 0) w_pend = atomicAdd(claim + blockIdx.x, (unsigned long long)OW_CLAIM);
    auto next_stage = [&]() -> uint64_t {
      if (c_lo < c_hi) return c_lo++;
      if (own) {
        const unsigned long long w = __shfl_sync(0xffffffffu, w_pend, 0);
        const uint64_t lo = s0 + (uint32_t)w, hi_all = s1 - (w >> 32);
        const uint64_t hi = lo + OW_CLAIM < hi_all ? lo + OW_CLAIM : hi_all;
        if (lo < hi) {
          c_lo = lo + 1;
          c_hi = hi;
          if (lane == 0) w_pend = atomicAdd(claim + blockIdx.x, (unsigned long long)OW_CLAIM);  // used at the next call
          return lo;
        }
        own = false;
      }
      for (uint32_t tries = 0;; ++tries) {
        if (tries > (1u << 20)) __trap();  // bounded: every failed CAS means another CTA progressed
        uint64_t best = 0;
        uint32_t bv = 0;
        unsigned long long bw = 0;
        for (uint32_t v = lane; v < G; v += 32) {
          const unsigned long long w = ld_relaxed_u64(claim + v);
          const uint64_t lo = ST * v / G + (uint32_t)w, hi = ST * (v + 1) / G - (w >> 32);
          const uint64_t rem = hi > lo ? hi - lo : 0;
          if (rem > best) {
            best = rem;
            bv = v;
            bw = w;
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
          const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const unsigned long long ow = __shfl_xor_sync(0xffffffffu, bw, o);
          if (ob > best || (ob == best && ov < bv)) {
            best = ob;
            bv = ov;
            bw = ow;
          }
        }
        if (best == 0) return ~0ull;  // nothing left anywhere
        uint64_t t = (best + 1) / 2;
        if (t > OW_STEAL) t = OW_STEAL;
        uint32_t got = 0;
        if (lane == 0) got = atomicCAS(claim + bv, bw, bw + (t << 32)) == bw;
        if (__shfl_sync(0xffffffffu, got, 0)) {
          const uint64_t hi = ST * (bv + 1) / G - (bw >> 32);
          c_lo = hi - t + 1;
          c_hi = hi;
          return hi - t;
        }
      }
    };
    // software pipeline over the stage stream: stage A is issued now, the piece descriptors of
    // B and C are in flight (lane j < 4 holds uint4 j of a stage's descriptor)
    auto load_desc = [&](uint64_t sx) {
      uint4 d = make_uint4(0, 0, 0, 0);
      if (sx != ~0ull && lane < 4) d = a.desc[4 * sx + lane];
      return d;
    };
    uint64_t sA = next_stage(), sB = sA != ~0ull ? next_stage() : ~0ull;
    uint4 dA = load_desc(sA), dB = load_desc(sB);
    while (sA != ~0ull) {
      const long long pc0 = prof ? clock64() : 0;
      const uint64_t s = sA;
      const uint4 d = dA;
      const uint64_t sC = sB != ~0ull ? next_stage() : ~0ull;
      const uint4 dC = load_desc(sC);
      sA = sB;
      dA = dB;
      sB = sC;
      dB = dC;
      const uint32_t ctx = __shfl_sync(0xffffffffu, d.x, 0), npc = __shfl_sync(0xffffffffu, d.y, 0);
      if (lane == 0) mbar_wait(&sm.empty[st], ph ^ 1u);  // the slot (and its meta) is free
      __syncwarp();
      const long long pc1 = prof ? clock64() : 0;
      const uint64_t R0 = OW_ROWS * s, R1 = R0 + OW_ROWS;
      if (lane == 0) {
        uint32_t flush = ctx != prev_ctx && MODE != 4 ? 1u : 0u;  // MODE 4 (measurement only): no context flushes
        if (*freq) {
          *freq = 0u;
          flush = 1u;
        }
        sm.meta[st].ctx = ctx;
        sm.meta[st].flush = flush;
        epoch += flush;
        sm.meta[st].epoch = epoch;
      }
      uint32_t npieces = 0;
      if (npc <= OW_DPIECES) {  // precomputed pieces: lane j in [1, npc] issues piece j - 1
        const bool in = lane >= 1 && lane <= npc;
        const uint32_t bytes = __reduce_add_sync(0xffffffffu, in ? d.z * 16u : 0u);
        // expect_tx before the arrive (below) keeps the phase open however early a copy lands
        if (lane == 0 && bytes)
          asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.full[st])), "r"(bytes) : "memory");
        __syncwarp();
        if (in) tma_bulk_g2s(&sm.stage[st][d.w], a.smp + (((uint64_t)d.y << 32) | d.x), d.z * 16u, &sm.full[st]);
        npieces = npc;
      } else {  // rare: a stage with more than OW_DPIECES launches, cut here 32 launches at a time
        const uint32_t f = __shfl_sync(0xffffffffu, d.z, 0);
        for (uint64_t base = f;; base += 32) {
          const uint64_t li = base + lane;
          uint64_t rp = ~0ull, src = 0, cnt = 0;
          if (li < a.n_launch) {
            rp = a.rowpos[li];
            src = a.lsrc[li];
            cnt = a.lcnt[li];
          }
          const uint64_t rows = (cnt + 31) / 32;
          const bool in = rp != ~0ull && rp < R1 && rp + rows > R0 && rows > 0;
          uint64_t lo = 0, len = 0, dst = 0;
          if (in) {
            const uint64_t r_lo = rp > R0 ? rp : R0;
            const uint64_t r_hi = rp + rows < R1 ? rp + rows : R1;
            lo = 32 * (r_lo - rp);
            const uint64_t hi = 32 * (r_hi - rp) < cnt ? 32 * (r_hi - rp) : cnt;
            len = hi - lo;
            dst = 32 * (r_lo - R0);
          }
          const uint32_t bytes = __reduce_add_sync(0xffffffffu, (uint32_t)len * 16u);
          const uint32_t m = __ballot_sync(0xffffffffu, in);
          if (lane == 0 && bytes)
            asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.full[st])), "r"(bytes) : "memory");
          __syncwarp();
          if (in) tma_bulk_g2s(&sm.stage[st][dst], a.smp + src + lo, (uint32_t)len * 16u, &sm.full[st]);
          npieces += __popc(m);
          // the batch's last launch ends inside the stage: more launches may follow
          const bool more = (rp != ~0ull) & (rp + rows < R1) & (base + 32 < a.n_launch);
          if (!__shfl_sync(0xffffffffu, more, 31)) break;
        }
      }
      if (lane == 0) {  // row meta; the arrive releases the ctx / flush words written above
        mbar_expect_tx(&sm.full[st], (uint32_t)(OW_ROWS * 5));
        tma_bulk_g2s(sm.meta[st].row_launch, a.row_launch + R0, OW_ROWS * 4, &sm.full[st]);
        tma_bulk_g2s(sm.meta[st].row_valid, a.row_valid + R0, OW_ROWS, &sm.full[st]);
      }
      __syncwarp();
      if (prof) {
        p_wait += pc1 - pc0;
        p_comp += clock64() - pc1;
        ++p_stages;
        p_pieces += npieces;
      }
      prev_ctx = ctx;
      if (++st == OW_STAGES) {
        st = 0;
        ph ^= 1u;
      }
    }
    if (lane == 0) {
      mbar_wait(&sm.empty[st], ph ^ 1u);
      sm.meta[st].ctx = OW_DONE;
      sm.meta[st].count = 0;
      sm.meta[st].flush = 1;
      sm.meta[st].epoch = epoch + 1;
      mbar_arrive(&sm.full[st]);
    }
    if (prof && lane == 0) {
      unsigned long long* dbg = reinterpret_cast<unsigned long long*>(a.sink) + 8 * ((uint64_t)gridDim.x * OW_CONS_WARPS + blockIdx.x);
      dbg[0] = p_wait;
      dbg[1] = p_comp;
      dbg[2] = p_stages;
      dbg[3] = p_pieces;
      dbg[4] = clock64() - p_t0;
    }
    return;
  }
  // -------------------------------------------------- consumer warps
  // warp w takes samples [w*OW_ROUND, (w+1)*OW_ROUND) of every stage (OW_STAGE = 16 rounds),
  // loads them into registers, releases the stage, then aggregates them
  const uint32_t ctid = tid - 32, lane = ctid & 31, w = ctid >> 5;
  // shared address of the block, pinned in a register (a volatile move: the compiler would
  // otherwise rematerialise the conversion in the loop); hot-loop addresses are sb + offset
  uint32_t sb;
  asm volatile("mov.u32 %0, %1;" : "=r"(sb) : "r"(smem_u32(&sm)));
  const uint32_t a_full = s_off(sm, &sm.full[0], sb), a_empty = s_off(sm, &sm.empty[0], sb);
  const uint32_t a_cnt = s_off(sm, &sm.cnt[0], sb), a_pend = s_off(sm, &sm.pend[w][0], sb);
  uint32_t cur_ctx = OW_DONE, st = 0, ph = 0;
  OwCounters k{0, 0, 0, 0};
  uint32_t sinkv = 0;
  long long t_wait = 0, t_flush = 0, t_work = 0, n_stage = 0, t_key = 0, t_bucket = 0, t_add = 0, n_miss = 0, since_flush = 0;  // MODE 9 only
  uint32_t np = 0;        // queued misses of this warp (warp-uniform)
  uint32_t inserted = 0;  // keys this lane inserted since the last publish
  auto probe_add = [&](uint32_t key, uint32_t add) {
    const uint32_t r = own_probe(sm, key, own_bucket(key), sb);
    inserted += r >> 31;
    own_add(sm, a, key, r & 0x7FFFFFFFu, add, cur_ctx);
  };
  auto probe_one = [&](uint32_t key) { probe_add(key, 1u); };
  // one `distinct` update per warp round (flush request when it crosses OW_FLUSH_REQ)
  auto publish = [&]() {
    const uint32_t ins = __reduce_add_sync(0xffffffffu, inserted);
    inserted = 0;
    if (lane == 0 && ins) {
      const uint32_t before = atomicAdd(&sm.distinct, ins);
      if (before < OW_FLUSH_REQ && before + ins >= OW_FLUSH_REQ) *(volatile uint32_t*)&sm.flush_req = 1u;
    }
  };
  uint32_t my_epoch = 0, grp = w;  // DC_OW_DYN: flushes this warp took part in; row group of the stage
  while (true) {
    const long long c_0 = MODE == 9 ? clock64() : 0;
    if (DC_OW_DYN) {
      // Row groups by ticket: the next group of the stage stream goes to whichever warp asks, so
      // no warp runs ahead of the others (a slot is refilled once all its groups are taken). At
      // most one ticket per warp is outstanding, so the tickets taken while a flush barrier waits
      // all lie in the flush stage (groups per stage = warps): the ring cannot deadlock.
      // The ticket counts modulo one ring period (groups x stages x 2 phases): slot, phase and
      // group come from a small quotient, and the wrapping increment is one shared atomic (a
      // plain atomicAdd under `lane == 0` compiles to the warp-aggregated sequence).
      constexpr uint32_t TK_PERIOD = (uint32_t)OW_CONS_WARPS * OW_STAGES * 2;
      uint32_t tk = 0;
      if (lane == 0) tk = s_inc32(s_off(sm, &sm.ticket, sb), TK_PERIOD - 1);
      tk = __shfl_sync(0xffffffffu, tk, 0);
      const uint32_t kst = tk / (uint32_t)OW_CONS_WARPS;  // < 2 * OW_STAGES
      grp = tk - kst * (uint32_t)OW_CONS_WARPS;
      ph = kst >= (uint32_t)OW_STAGES ? 1u : 0u;
      st = kst - ph * (uint32_t)OW_STAGES;
    }
    s_mbar_wait(a_full + 8 * st, ph);
    const long long c_1 = MODE == 9 ? clock64() : 0;
    const uint32_t mctx = sm.meta[st].ctx;
    const uint32_t flush = DC_OW_DYN ? (sm.meta[st].epoch != my_epoch ? 1u : 0u) : sm.meta[st].flush;
    if (DC_OW_DYN) my_epoch = sm.meta[st].epoch;
    if (flush) {  // uniform: every consumer sees the same meta
      if (np) {  // this warp's queued misses belong to the table being flushed
        if (lane < np) probe_one(sm.pend[w][lane]);
        np = 0;
        publish();
      }
      cons_sync();  // every consumer finished all previous stages
      // always entered by every consumer (its barriers are uniform); empty tables emit nothing.
      own_flush(sm, a, cur_ctx, ctid);
    }
    if (MODE == 9) {
      t_wait += c_1 - c_0;
      t_flush += clock64() - c_1;
      // measurement split: waits in the first ring-worth of stages after a flush (bucket slot)
      // and the final wait for the DONE marker (miss slot)
      if (flush) since_flush = 0;
      if (mctx == OW_DONE) n_miss = c_1 - c_0;
      else if (since_flush++ < OW_STAGES) t_bucket += c_1 - c_0;
    }
    if (mctx == OW_DONE) break;
    cur_ctx = mctx;
    const bool ctx_ok = mctx < a.N;
    if (MODE == 2) {  // measurement only: the TMA pipeline alone (stage released unread)
      __syncwarp();
      if (lane == 0) s_mbar_arrive(a_empty + 8 * st);
      if (!DC_OW_DYN && ++st == OW_STAGES) {
        st = 0;
        ph ^= 1u;
      }
      continue;
    }
    uint4 q[OW_PER_LANE];
    uint32_t lch[OW_PER_LANE];
    bool vld[OW_PER_LANE];
#pragma unroll
    for (int i = 0; i < OW_PER_LANE; ++i) {
      const uint32_t row = grp * OW_PER_LANE + i;  // rows [4g, 4g+4) of the stage (g = w, or by ticket)
      lch[i] = sm.meta[st].row_launch[row];      // row-uniform: one broadcast load
      vld[i] = lane < sm.meta[st].row_valid[row];
      q[i] = vld[i] ? sm.stage[st][32 * row + lane] : make_uint4(0, 0, 0, 0);
    }
    uint32_t t[OW_PER_LANE], b[OW_PER_LANE];
    bool cold = false;
#pragma unroll
    for (int i = 0; i < OW_PER_LANE; ++i) {
      const bool hot = vld[i] & own_hot(q[i], lch[i], a.S) & ctx_ok;
      t[i] = hot ? (q[i].y << 5) | (q[i].z & 0xFFFFu) : EMPTY32;
      cold |= vld[i] & !hot;
    }
    const bool any_cold = __any_sync(0xffffffffu, cold);
    if (any_cold) {  // rare: spills and invalid samples
#pragma unroll
      for (int i = 0; i < OW_PER_LANE; ++i)
        if (vld[i] && t[i] == EMPTY32) inserted += own_cold(q[i], lch[i], a, ctx_ok, k, sm, mctx);
    }
    const long long c_2 = MODE == 9 ? clock64() : 0;
    if (MODE == 9) t_key += c_2 - c_1;
    // the stage's samples and row meta are in registers: release the slot to the producer now,
    // before the table work (one more stage of prefetch in flight)
    __syncwarp();
    if (lane == 0) s_mbar_arrive(a_empty + 8 * st);
    if (MODE == 1) {  // measurement: data movement + classification only
#pragma unroll
      for (int i = 0; i < OW_PER_LANE; ++i) sinkv ^= t[i] * (2 * i + 1);
    } else {
      uint32_t slot[OW_PER_LANE];
      const long long c_3 = MODE == 9 ? clock64() : 0;
#pragma unroll
      for (int i = 0; i < OW_PER_LANE; ++i) b[i] = own_bucket(t[i]);
      if (DC_OW_HINT) {  // the preferred slot (4-B load), then the whole bucket for the rest
        uint32_t hs[OW_PER_LANE], k1[OW_PER_LANE];
#pragma unroll
        for (int i = 0; i < OW_PER_LANE; ++i) hs[i] = OW_BW * b[i] + own_hint(t[i]);
#pragma unroll
        for (int i = 0; i < OW_PER_LANE; ++i) k1[i] = sm.key[hs[i]];
#pragma unroll
        for (int i = 0; i < OW_PER_LANE; ++i) {
          slot[i] = hs[i];
          if (k1[i] != t[i] && t[i] != EMPTY32) {
            const uint4 v = bkt_ld(&sm.key[OW_BW * b[i]]);  // home bucket
            slot[i] = bucket_slot(v, t[i], b[i]);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < OW_PER_LANE; ++i) {
          const uint4 v = bkt_ld(&sm.key[OW_BW * b[i]]);  // home bucket
          slot[i] = bucket_slot(v, t[i], b[i]);
        }
      }
      // Hits are added directly. Misses (new or displaced keys, a few % of the samples) are
      // queued per warp and probed 32 at a time, so the slow path runs with all lanes busy.
      // (Claiming new keys inline with a CAS, or draining the queue every stage, cut the
      // misses but measured slower: 0.61 / 0.72 ms vs 0.51 ms on config 3.)
#pragma unroll
      for (int i = 0; i < OW_PER_LANE; ++i) {
        const bool miss = t[i] != EMPTY32 && slot[i] == OW_MISS;
        if (DC_OW_NOBR) {  // branch-free: lanes without a hit add into the warp's dummy counter and
                           // lanes without a miss store into the queue's dummy tail slot
          const uint32_t cs = t[i] != EMPTY32 && !miss ? slot[i] : (uint32_t)OW_TAB + w;
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a_cnt + 4 * cs) : "memory");
          const uint32_t mm = __ballot_sync(0xffffffffu, miss);
#if DC_OW_PSTORE
          // predicated store (no dummy-slot wavefront when no lane missed)
          asm volatile("{\n.reg .pred p;\nsetp.ne.u32 p, %2, 0;\n@p st.shared.u32 [%0], %1;\n}\n" ::"r"(
                           a_pend + 4 * (np + __popc(mm & lanemask_lt()))),
                       "r"(t[i]), "r"((uint32_t)miss)
                       : "memory");
#else
          sm.pend[w][miss ? np + __popc(mm & lanemask_lt()) : (uint32_t)OW_PEND] = t[i];
#endif
          np += __popc(mm);
        } else {
          red_shared_inc_if(&sm.cnt[slot[i] & 0x7FFFFFFFu], t[i] != EMPTY32 && !miss);  // hit: never the spill slot
          const uint32_t mm = __ballot_sync(0xffffffffu, miss);
          if (miss) sm.pend[w][np + __popc(mm & lanemask_lt())] = t[i];
          np += __popc(mm);
        }
      }
      if (MODE == 3) np = 0;  // measurement only: misses dropped
        __syncwarp();
      // new keys are inserted only by the miss probes and the cold path: publish after those
      const bool pub = any_cold || np >= 32;
      while (np >= 32) {
        np -= 32;
        probe_one(sm.pend[w][np + lane]);
      }
      __syncwarp();
      if (pub) publish();
      if (MODE == 9) t_add += clock64() - c_3;
    }
    if (MODE == 9) {
      t_work += clock64() - c_1;
      ++n_stage;
    }
    if (!DC_OW_DYN && ++st == OW_STAGES) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (MODE == 9 && lane == 0) {  // measurement: per-warp cycle split (wait / flush / work)
    unsigned long long* dbg = reinterpret_cast<unsigned long long*>(a.sink) + 8 * (blockIdx.x * OW_CONS_WARPS + w);
    dbg[0] = t_wait;
    dbg[1] = t_flush;
    dbg[2] = t_work - t_flush;
    dbg[3] = n_stage;
    dbg[4] = t_key;
    dbg[5] = t_bucket;
    dbg[6] = t_add;
    dbg[7] = n_miss;
  }
  uint32_t bad_l = k.bad_l, bad_s = k.bad_s, zero = k.zero, fallback = k.fallback;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad_l += __shfl_xor_sync(0xffffffffu, bad_l, o);
    bad_s += __shfl_xor_sync(0xffffffffu, bad_s, o);
    zero += __shfl_xor_sync(0xffffffffu, zero, o);
    fallback |= __shfl_xor_sync(0xffffffffu, fallback, o);
  }
  if (lane == 0) {
    if (bad_l) atomicAdd(a.ldiag + DG_BAD_LAUNCH, (unsigned long long)bad_l);
    if (bad_s) atomicAdd(a.ldiag + DG_BAD_STALL, (unsigned long long)bad_s);
    if (zero) atomicAdd(a.ldiag + DG_ZERO, (unsigned long long)zero);
    if (fallback) atomicOr(a.g_flags, (uint32_t)OWF_FALLBACK);
    if (MODE && sinkv == 0x12345678u) a.sink[0] = sinkv;
  }
}

// ---------------------------------------------------------------- global bitmap reduce
// The data-parallel reduce used whenever every context's PC range is small enough (always for
// real kernels). Per context c, with pc' = pc_off >> (common trailing zero bits of c's PCs),
// key (pc', stall) is bit (pc' << 5 | stall) of c's slice of one global presence bitmap; one
// 32-bit word per PC. Because contexts (then PCs, then stalls) are laid out in canonical order,
// an exclusive scan over the words' popcounts is each bin's final index and a scan over
// non-zero words each PC node's index: the partial entries are reduced by global atomics into
// their final slots, without sorting.
constexpr uint32_t BR_MAX_WORDS = 1u << 20;   // per context (larger PC ranges: per-group reduce)
constexpr uint64_t BR_MAX_TOTAL = 1ull << 27;  // whole bitmap (512 MB)
// segment kernels: one warp per (segment, chunk of BR_CH entries)
constexpr uint32_t BR_CH = 256;
constexpr uint32_t BR_MAXCH = ((OW_TAB > (int)OW_SPILL_CAP ? OW_TAB : OW_SPILL_CAP) + BR_CH - 1) / BR_CH;
#define BR_FOR_CHUNKS(seg, n_segs, N)                                                                          \
  for (uint64_t item = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; item < (uint64_t)n_segs * BR_MAXCH; \
       item += ((uint64_t)gridDim.x * blockDim.x) >> 5)                                                        \
    if (const uint4 sg = seg[item / BR_MAXCH]; sg.x < N && (item % BR_MAXCH) * BR_CH < sg.y)

// runs before the host has read the segment count: it takes the device counter (clamped)
__global__ void k_br_range(const uint4* __restrict__ seg, const unsigned int* __restrict__ d_nsegs, uint32_t cap_segs,
                           const uint32_t* __restrict__ pkey, uint64_t N, uint32_t* __restrict__ cmax, uint32_t* __restrict__ cor,
                           const uint32_t* __restrict__ g_flags) { DC_PDL_ENTER();
  const uint32_t lane = threadIdx.x & 31;
  if (*g_flags) return;  // fallback / overflow: the host reruns the generic schedule
  const uint32_t n_segs = min(*d_nsegs, cap_segs);
  BR_FOR_CHUNKS(seg, n_segs, N) {
    const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
    const uint32_t j0 = (uint32_t)(item % BR_MAXCH) * BR_CH, j1 = min(sg.y, j0 + BR_CH);
    uint32_t mk = 0, orp = 0;
#pragma unroll 4
    for (uint32_t j = j0 + lane; j < j1; j += 32) {
      const uint32_t kk = pkey[base + j];
      mk = max(mk, kk + 1);  // 0 = no entry
      orp |= kk >> 5;
    }
    mk = __reduce_max_sync(0xffffffffu, mk);
    orp = __reduce_or_sync(0xffffffffu, orp);
    if (lane == 0) {
      atomicMax(cmax + sg.x, mk);
      atomicOr(cor + sg.x, orp);
    }
  }
}

__global__ void k_br_words(const uint32_t* __restrict__ cmax, const uint32_t* __restrict__ cor, uint64_t N,
                           uint64_t* __restrict__ cw, uint8_t* __restrict__ csh, uint32_t* too_wide) { DC_PDL_ENTER();
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < N; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t m = cmax[c], o = cor[c];
    const int sh = o ? __ffs(o) - 1 : 0;
    const uint64_t words = m ? (uint64_t)(((m - 1) >> 5) >> sh) + 1 : 0;
    if (words > BR_MAX_WORDS) atomicOr(too_wide, 1u);
    cw[c] = words;
    csh[c] = (uint8_t)sh;
  }
}

__global__ void k_br_bits(const uint4* __restrict__ seg, uint32_t n_segs, const uint32_t* __restrict__ pkey, uint64_t N,
                          const uint64_t* __restrict__ wbase, const uint8_t* __restrict__ csh, uint32_t* __restrict__ bm) { DC_PDL_ENTER();
  BR_FOR_CHUNKS(seg, n_segs, N) {
    const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
    const uint32_t j0 = (uint32_t)(item % BR_MAXCH) * BR_CH, j1 = min(sg.y, j0 + BR_CH);
    const uint64_t wb = wbase[sg.x];
    const int sh = csh[sg.x];
#pragma unroll 4
    for (uint32_t j = j0 + (threadIdx.x & 31); j < j1; j += 32) {
      const uint32_t kk = pkey[base + j];
      atomicOr(bm + wb + ((kk >> 5) >> sh), 1u << (kk & 31u));
    }
  }
}

// packed per-word counts: bins (popcount) in the high half, PC nodes (word != 0) in the low half
__global__ void k_br_pop(const uint32_t* __restrict__ bm, uint64_t W, uint64_t* __restrict__ pk) { DC_PDL_ENTER();
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = bm[w];
    pk[w] = ((uint64_t)__popc(b) << 32) | (b != 0u ? 1u : 0u);
  }
}

// one thread per bitmap word: its PC node and bins (counts are zeroed by the caller). The word's
// context is found by binary search over the word bases (empty contexts share their base with
// the next context, so the last base <= w is the owning, non-empty one).
__global__ void k_br_emit(const uint32_t* __restrict__ bm, const uint64_t* __restrict__ pre, uint64_t W,
                          const uint64_t* __restrict__ wbase, const uint8_t* __restrict__ csh, uint64_t N,
                          uint32_t* __restrict__ pc_ctx, uint32_t* __restrict__ pc_off, uint32_t* __restrict__ bin_pcnode,
                          uint16_t* __restrict__ bin_stall) { DC_PDL_ENTER();
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t bits = bm[w];
    if (!bits) continue;
    uint64_t lo = 0, hi = N - 1;  // last c with wbase[c] <= w
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (wbase[mid] <= w) lo = mid;
      else hi = mid - 1;
    }
    const uint64_t c = lo;
    const uint64_t pr = pre[w];
    const uint32_t p = (uint32_t)pr;  // PC node rank
    uint64_t r = pr >> 32;            // first bin
    pc_ctx[p] = (uint32_t)c;
    pc_off[p] = (uint32_t)((w - wbase[c]) << csh[c]);
    while (bits) {
      const uint32_t b = __ffs(bits) - 1;
      bits &= bits - 1;
      bin_pcnode[r] = (uint32_t)(N + p);
      bin_stall[r] = (uint16_t)b;
      ++r;
    }
  }
}

// one warp per segment chunk: counts into their final bins; per-stall totals of the segment's
// context summed in shared memory (exact: 32-bit halves with carry) and added once per chunk
constexpr int BR_WARPS = 8;
__global__ void __launch_bounds__(32 * BR_WARPS) k_br_count(
    const uint4* __restrict__ seg, uint32_t n_segs, const uint32_t* __restrict__ pkey,
    const unsigned long long* __restrict__ pcnt, uint64_t N, uint32_t S, const uint32_t* __restrict__ bm,
    const uint64_t* __restrict__ pre, const uint64_t* __restrict__ wbase, const uint8_t* __restrict__ csh,
    unsigned long long* __restrict__ bin_count, unsigned long long* __restrict__ xsamples,
    unsigned long long* __restrict__ xstall) { DC_PDL_ENTER();
  __shared__ uint32_t lo[BR_WARPS][32], hi[BR_WARPS][32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  lo[w][lane] = 0;
  hi[w][lane] = 0;
  __syncwarp();
  BR_FOR_CHUNKS(seg, n_segs, N) {
    const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
    const uint32_t j0 = (uint32_t)(item % BR_MAXCH) * BR_CH, j1 = min(sg.y, j0 + BR_CH);
    const uint64_t wb = wbase[sg.x];
    const int sh = csh[sg.x];
    // all BR_CH / 32 entries of the lane in flight at once: entry loads, then the bitmap word /
    // prefix loads, then the updates (one latency round each instead of one per entry pair)
    constexpr int U = BR_CH / 32;
    uint32_t kk[U];
    unsigned long long cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + lane + 32 * u;
      kk[u] = j < j1 ? pkey[base + j] : 0u;
      cv[u] = j < j1 ? pcnt[base + j] : 0ull;
    }
    uint64_t pr[U];
    uint32_t bw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + lane + 32 * u;
      const uint64_t wd = wb + ((kk[u] >> 5) >> sh);
      pr[u] = j < j1 ? pre[wd] : 0ull;
      bw[u] = j < j1 ? bm[wd] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + lane + 32 * u;
      if (j >= j1) continue;
      const uint32_t b = kk[u] & 31u;
      const uint64_t r = (pr[u] >> 32) + __popc(bw[u] & ((1u << b) - 1u));
      atomicAdd(bin_count + r, cv[u]);
      const uint32_t c32 = (uint32_t)cv[u];
      const uint32_t old = atomicAdd(&lo[w][b], c32);
      const uint32_t carry = old + c32 < old ? 1u : 0u;
      if (carry + (uint32_t)(cv[u] >> 32)) atomicAdd(&hi[w][b], carry + (uint32_t)(cv[u] >> 32));
    }
    __syncwarp();
    const unsigned long long t = ((unsigned long long)hi[w][lane] << 32) | lo[w][lane];
    lo[w][lane] = 0;
    hi[w][lane] = 0;
    if (t && lane < S) atomicAdd(xstall + (uint64_t)lane * N + sg.x, t);
    unsigned long long tot = lane < S ? t : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0 && tot) atomicAdd(xsamples + sg.x, tot);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- context reduce (default)
// Three small launches and a scan, no sort, no waiting between contexts:
//  k_ctx_order: one CTA sums each context group's partial entries (segment headers) and orders
//    the groups largest first (log2 buckets: longest-processing-time-first over the CTAs);
//  k_ctx_hist: persistent CTAs take the groups in that order by ticket. For its context a CTA
//    gathers the segments' partial entries, builds the (pc', stall) presence bitmap in shared
//    memory (pc' = pc_off >> the common trailing zero bits of the context's PCs; one 32-bit word
//    per PC), ranks the keys by the word popcount prefix (bin index within the context) and sums
//    the counts per bin in shared memory (exact u64 as 32-bit halves), adds the context's
//    per-stall totals into its sample columns, and writes per word (bits, bin prefix, PC-node
//    prefix, group) and the per-bin counts into bump-allocated scratch, with the context's
//    (bins, PC nodes);
//  an exclusive scan over the groups (ascending context id = canonical order) gives every
//    context its global bin / PC-node bases;
//  k_ctx_emit: one thread per scratch word (whole grid, coalesced) writes the word's PC node,
//    its bins and their counts at their global positions.
// A context whose PC range or segment count does not fit shared memory (or scratch that is too
// small) raises CR_WIDE: the host takes the k_br_* path; outputs past the allocated capacity
// are not written (the host sees more bins than the capacity, reallocates and reruns k_ctx_emit only).
#ifndef DC_CR_THREADS
#define DC_CR_THREADS 1024
#endif
#ifndef DC_CR_WORDS
#define DC_CR_WORDS 8192
#endif
#ifndef DC_CR_BINS
#define DC_CR_BINS 12288
#endif
#ifndef DC_CR_SEGS
#define DC_CR_SEGS 4096
#endif
#ifndef DC_CR_CPS
#define DC_CR_CPS 1
#endif
constexpr int CR_THREADS = DC_CR_THREADS;
constexpr int CR_NW = CR_THREADS / 32;     // warps per CTA
constexpr int CR_CPS = DC_CR_CPS;          // CTAs per SM
constexpr uint32_t CR_WORDS = DC_CR_WORDS;  // PCs per context (pc' range)
constexpr uint32_t CR_BINS = DC_CR_BINS;    // bins per context counted in shared memory
constexpr uint32_t CR_SEGS = DC_CR_SEGS;    // segments per context
constexpr uint32_t CR_USEGS = 1024;    // of which with an unknown key range (more: pass A walks all)
constexpr uint32_t CR_ORDER_MAX = 8192;   // groups ordered by size (more: ascending order; static smem)
enum { CR_WIDE = 1, CR_OVER = 2 };
struct CtxRedSmem {
  uint32_t bm[CR_WORDS];
  uint32_t bpre[CR_WORDS];   // bins before word w (within the context)
  // u64 sums as 32-bit halves with an exact carry (native 32-bit shared atomics; a 64-bit
  // shared atomic add is a CAS loop)
  uint32_t cnt_lo[CR_BINS], cnt_hi[CR_BINS];
  uint32_t wst_lo[CR_THREADS / 32][32], wst_hi[CR_THREADS / 32][32];  // per-warp stall totals
  uint32_t segs[CR_SEGS];
  uint32_t useg[CR_USEGS];  // segments whose key range is unknown (spill chunks): walked by pass A
  uint32_t nseg, nuseg, g, maxk, orp;
  unsigned long long ow, ob;
};
struct __align__(16) CtxWord {  // scratch per bitmap word
  uint32_t bits, bpre, ppre, g;
};
struct __align__(16) CtxRec {  // scratch per group
  unsigned long long ow, ob;   // first scratch word, first scratch count
  uint32_t ctx, sh;
};

// Walks the context's entries: chunks of 32 x CR_U entries, chunk k of the concatenated
// segments to warp k mod CR_NW; every lane has CR_U independent loads in flight (one memory
// latency per chunk instead of one per entry). fn(key, count) for every valid entry.
constexpr uint32_t CR_U = 8;
template <bool WITH_CNT, class F>
__device__ __forceinline__ void cr_for_entries(const uint32_t* segs, const uint4* __restrict__ seg, const uint32_t* __restrict__ pkey,
                                               const unsigned long long* __restrict__ pcnt, uint32_t ns, F fn) {
  constexpr uint32_t CH = 32 * CR_U;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t kbase = 0;
  for (uint32_t q = 0; q < ns; ++q) {
    const uint4 sg = seg[segs[q]];
    const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
    const uint32_t nch = (sg.y + CH - 1) / CH;
    for (uint32_t ch = (w + CR_NW - kbase % CR_NW) % CR_NW; ch < nch; ch += CR_NW) {
      uint32_t kk[CR_U];
      unsigned long long cv[CR_U];
#pragma unroll
      for (uint32_t u = 0; u < CR_U; ++u) {
        const uint32_t j = ch * CH + u * 32 + lane;
        kk[u] = j < sg.y ? __ldcg(pkey + base + j) : 0u;
        if (WITH_CNT) cv[u] = j < sg.y ? __ldcg(pcnt + base + j) : 0ull;
      }
#pragma unroll
      for (uint32_t u = 0; u < CR_U; ++u)
        if (ch * CH + u * 32 + lane < sg.y) fn(kk[u], WITH_CNT ? cv[u] : 0ull);
    }
    kbase += nch;
  }
}

// one CTA: group g's partial-entry total, groups ordered by descending log2 size (LPT)
__global__ void __launch_bounds__(1024) k_ctx_order(const uint4* __restrict__ seg, const unsigned int* __restrict__ d_nsegs,
                                                    uint32_t cap_segs, const uint64_t* __restrict__ lkey,
                                                    const uint32_t* __restrict__ gfirst, const uint32_t* __restrict__ d_ng,
                                                    uint32_t* __restrict__ order) { DC_PDL_ENTER();
  __shared__ uint32_t size[CR_ORDER_MAX];
  __shared__ uint32_t bucket[33];
  const uint32_t NG = *d_ng, n_segs = min(*d_nsegs, cap_segs), tid = threadIdx.x;
  if (NG > CR_ORDER_MAX) {  // plain ascending order
    for (uint32_t g = tid; g < NG; g += blockDim.x) order[g] = g;
    return;
  }
  for (uint32_t g = tid; g < NG; g += blockDim.x) size[g] = 0;
  if (tid < 33) bucket[tid] = 0;
  __syncthreads();
  for (uint32_t i = tid; i < n_segs; i += blockDim.x) {
    const uint4 sg = seg[i];
    if (!sg.y) continue;
    uint32_t lo = 0, hi = NG;  // group of context sg.x: groups are in ascending context order
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (lkey[gfirst[mid]] < sg.x) lo = mid + 1;
      else hi = mid;
    }
    if (lo < NG && lkey[gfirst[lo]] == sg.x) atomicAdd(&size[lo], sg.y);
  }
  __syncthreads();
  for (uint32_t g = tid; g < NG; g += blockDim.x) atomicAdd(&bucket[size[g] ? 32 - __clz(size[g]) : 0], 1u);
  __syncthreads();
  if (tid == 0) {  // descending buckets: start of bucket b = groups in buckets > b
    uint32_t run = 0;
    for (int b = 32; b >= 0; --b) {
      const uint32_t c = bucket[b];
      bucket[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (uint32_t g = tid; g < NG; g += blockDim.x) order[atomicAdd(&bucket[size[g] ? 32 - __clz(size[g]) : 0], 1u)] = g;
}

__global__ void __launch_bounds__(CR_THREADS, CR_CPS) k_ctx_hist(
    const uint4* __restrict__ seg, const uint2* __restrict__ seg_meta, const unsigned int* __restrict__ d_nsegs, uint32_t cap_segs, const uint32_t* __restrict__ pkey,
    const unsigned long long* __restrict__ pcnt, const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ gfirst,
    const uint32_t* __restrict__ d_ng, const uint32_t* __restrict__ order, uint64_t N, uint32_t S, const uint32_t* __restrict__ g_flags,
    unsigned long long* __restrict__ ctl,  // [0] ticket, [1] status, [2] scratch words used, [3] scratch bins used
    CtxWord* __restrict__ wscr, uint64_t wcap, unsigned long long* __restrict__ bscr, uint64_t bcap, CtxRec* __restrict__ rec,
    uint64_t* __restrict__ gnb, uint64_t* __restrict__ gnp, unsigned long long* __restrict__ xsamples,
    unsigned long long* __restrict__ xstall) { DC_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char cr_raw[];
  CtxRedSmem& sm = *reinterpret_cast<CtxRedSmem*>(cr_raw);
  if (*g_flags) return;  // the owner pass fell back: the host reruns the generic schedule
  const uint32_t tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const uint32_t NG = *d_ng, n_segs = min(*d_nsegs, cap_segs);
  for (;;) {
    if (tid == 0) {
      const uint32_t t = (uint32_t)atomicAdd(ctl, 1ull);
      sm.g = t < NG ? order[t] : 0xFFFFFFFFu;
      sm.nseg = 0;
      sm.nuseg = 0;
      sm.maxk = 0;
      sm.orp = 0;
      sm.ow = 0;
      sm.ob = 0;
    }
    __syncthreads();
    const uint32_t g = sm.g;
    if (g == 0xFFFFFFFFu) break;
    const uint64_t ctx = lkey[gfirst[g]];
    bool ok = ctx < N;  // launches with an invalid leaf: no bins (flagged by the plan)
    uint32_t W = 0, nb = 0, np = 0, ns = 0;
    int sh = 0;
    if (ok) {
      uint32_t mk = 0, orp = 0;
      // this context's segments (headers scanned 8 per thread in flight)
      for (uint32_t i0 = 0; i0 < n_segs; i0 += 8 * CR_THREADS) {
        uint32_t cx[8], cn[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t i = i0 + u * CR_THREADS + tid;
          const uint2 h = i < n_segs ? __ldcg(reinterpret_cast<const uint2*>(seg + i)) : make_uint2(0xFFFFFFFFu, 0u);
          cx[u] = h.x;
          cn[u] = h.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (cx[u] == ctx && cn[u]) {
            const uint32_t si = i0 + u * CR_THREADS + tid;
            const uint32_t q = atomicAdd(&sm.nseg, 1u);
            if (q < CR_SEGS) sm.segs[q] = si;
            // pass A, folded in: key range (max key + 1, OR of the PCs). A table-flush segment
            // carries it (seg_meta, written by k_pc_owner's flush); only the spill segments'
            // entries are walked below
            const uint2 m = __ldcg(seg_meta + si);
            if (m.x == 0xFFFFFFFFu) {
              const uint32_t uu = atomicAdd(&sm.nuseg, 1u);
              if (uu < CR_USEGS) sm.useg[uu] = si;
            } else {
              mk = max(mk, m.x);
              orp |= m.y;
            }
          }
      }
      __syncthreads();
      ns = min(sm.nseg, CR_SEGS);
      if (sm.nuseg > CR_USEGS) {  // too many spill segments to list: walk every segment
        cr_for_entries<false>(sm.segs, seg, pkey, pcnt, ns, [&](uint32_t kk, unsigned long long) {
          mk = max(mk, kk + 1);
          orp |= kk >> 5;
        });
      } else if (sm.nuseg) {
        cr_for_entries<false>(sm.useg, seg, pkey, pcnt, sm.nuseg, [&](uint32_t kk, unsigned long long) {
          mk = max(mk, kk + 1);
          orp |= kk >> 5;
        });
      }
      mk = __reduce_max_sync(0xffffffffu, mk);
      orp = __reduce_or_sync(0xffffffffu, orp);
      if (lane == 0) {
        atomicMax(&sm.maxk, mk);
        atomicOr(&sm.orp, orp);
      }
      __syncthreads();
      sh = sm.orp ? __ffs(sm.orp) - 1 : 0;
      W = sm.maxk ? (((sm.maxk - 1) >> 5) >> sh) + 1 : 0;
      if (W > CR_WORDS || sm.nseg > CR_SEGS) {
        if (tid == 0) atomicOr(ctl + 1, (unsigned long long)CR_WIDE);
        ok = false;
      }
    }
    if (ok) {
      // pass B: presence bits
      for (uint32_t w = tid; w < W; w += CR_THREADS) sm.bm[w] = 0;
      __syncthreads();
      cr_for_entries<false>(sm.segs, seg, pkey, pcnt, ns, [&](uint32_t kk, unsigned long long) {
        atomicOr(&sm.bm[(kk >> 5) >> sh], 1u << (kk & 31u));
      });
      __syncthreads();
      // word prefixes: thread t owns words [t * WP, (t + 1) * WP)
      constexpr uint32_t WP = CR_WORDS / CR_THREADS;
      uint32_t bsum = 0, psum = 0;
#pragma unroll
      for (uint32_t i = 0; i < WP; ++i) {
        const uint32_t w = tid * WP + i;
        const uint32_t b = w < W ? sm.bm[w] : 0u;
        bsum += __popc(b);
        psum += b != 0u;
      }
      // both prefixes in one block scan: bins (< 2^18 per context) low, PC nodes high
      unsigned long long tot2 = 0;
      const unsigned long long ex2 =
          block_excl_scan<unsigned long long, CR_THREADS>((unsigned long long)bsum | ((unsigned long long)psum << 32), &tot2);
      uint32_t bex = (uint32_t)ex2, pex = (uint32_t)(ex2 >> 32);
      nb = (uint32_t)tot2;
      np = (uint32_t)(tot2 >> 32);
      if (tid == 0) {
        sm.ow = atomicAdd(ctl + 2, (unsigned long long)W);
        sm.ob = atomicAdd(ctl + 3, (unsigned long long)nb);
        if (sm.ow + W > wcap || sm.ob + nb > bcap) {  // scratch too small: the host takes the k_br_* path
          atomicOr(ctl + 1, (unsigned long long)CR_WIDE);
          sm.ow = ~0ull;
        }
      }
      __syncthreads();
      const unsigned long long ow = sm.ow;
#pragma unroll
      for (uint32_t i = 0; i < WP; ++i) {
        const uint32_t w = tid * WP + i;
        if (w < W) {
          const uint32_t b = sm.bm[w];
          sm.bpre[w] = bex;
          if (ow != ~0ull) wscr[ow + w] = CtxWord{b, bex, pex, g};
          bex += __popc(b);
          pex += b != 0u;
        }
      }
      if (ow == ~0ull) ok = false;
    }
    const bool in_smem = nb <= CR_BINS;
    for (uint32_t i = tid; i < CR_NW * 32; i += CR_THREADS) {
      (&sm.wst_lo[0][0])[i] = 0;
      (&sm.wst_hi[0][0])[i] = 0;
    }
    if (ok && in_smem)
      for (uint32_t i = tid; i < nb; i += CR_THREADS) {
        sm.cnt_lo[i] = 0;
        sm.cnt_hi[i] = 0;
      }
    const unsigned long long ob = sm.ob;
    if (ok && !in_smem)
      for (uint32_t i = tid; i < nb; i += CR_THREADS) bscr[ob + i] = 0;
    __syncthreads();
    if (ok) {
      // pass C: counts into their bins; per-stall totals
      cr_for_entries<true>(sm.segs, seg, pkey, pcnt, ns, [&](uint32_t kk, unsigned long long cv) {
        const uint32_t w = (kk >> 5) >> sh, b = kk & 31u;
        const uint32_t r = sm.bpre[w] + __popc(sm.bm[w] & ((1u << b) - 1u));
        const uint32_t lo = (uint32_t)cv, hi = (uint32_t)(cv >> 32);
        if (in_smem) {
          const uint32_t old = atomicAdd(&sm.cnt_lo[r], lo);
          const uint32_t up = hi + (old + lo < old ? 1u : 0u);
          if (up) atomicAdd(&sm.cnt_hi[r], up);
        } else {
          atomicAdd(bscr + ob + r, cv);
        }
        const uint32_t old = atomicAdd(&sm.wst_lo[wp][b], lo);
        const uint32_t up = hi + (old + lo < old ? 1u : 0u);
        if (up) atomicAdd(&sm.wst_hi[wp][b], up);
      });
      __syncthreads();
      if (in_smem)
        for (uint32_t i = tid; i < nb; i += CR_THREADS) bscr[ob + i] = ((unsigned long long)sm.cnt_hi[i] << 32) | sm.cnt_lo[i];
      if (tid < 32) {
        unsigned long long t = 0;
        for (int w2 = 0; w2 < CR_THREADS / 32; ++w2) t += ((unsigned long long)sm.wst_hi[w2][tid] << 32) | sm.wst_lo[w2][tid];
        if (tid < S && t) xstall[(uint64_t)tid * N + ctx] += t;
        unsigned long long tot = tid < S ? t : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (tid == 0 && tot) xsamples[ctx] += tot;
      }
    }
    if (tid == 0) {
      rec[g] = CtxRec{ok ? sm.ow : 0ull, ob, (uint32_t)ctx, (uint32_t)sh};
      gnb[g] = ok ? nb : 0;
      gnp[g] = ok ? np : 0;
    }
    __syncthreads();
  }
}

// Per scratch word (grid-stride over the words used): its PC node, bins and counts.
// DC_CE_WARP: a warp takes 32 consecutive words; each lane writes its word's PC node, then the
// warp writes the words' bins together — bin j of the warp's list goes to lane j % 32, which finds
// its word by a binary search over the lanes' inclusive bin counts and its stall as the k-th set
// bit of the word — so consecutive lanes store consecutive bins (the words of one context are
// contiguous in the output). Otherwise one thread writes all bins of its word.
#ifndef DC_CE_WARP
#define DC_CE_WARP 1
#endif
__global__ void k_ctx_emit(const CtxWord* __restrict__ wscr, const unsigned long long* __restrict__ ctl, const CtxRec* __restrict__ rec,
                           const uint64_t* __restrict__ bbase, const uint64_t* __restrict__ pbase,
                           const unsigned long long* __restrict__ bscr, uint64_t N, uint64_t cap, unsigned long long* __restrict__ status,
                           uint32_t* __restrict__ pc_ctx, uint32_t* __restrict__ pc_off, uint32_t* __restrict__ bin_pcnode,
                           uint16_t* __restrict__ bin_stall, uint64_t* __restrict__ bin_count, const uint32_t* __restrict__ g_flags) { DC_PDL_ENTER();
  if (*g_flags || (ctl[1] & CR_WIDE)) return;
  const uint64_t total = ctl[2];
#if DC_CE_WARP
  {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wg = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = wg * 32; base < total; base += nw * 32) {  // warp-uniform
      const uint64_t i = base + lane;
      uint32_t bits = 0, cnt = 0;
      uint64_t q = 0, src = 0, pn = 0;
      if (i < total) {
        const CtxWord cw = wscr[i];
        bits = cw.bits;
        if (bits) {
          const CtxRec r = rec[cw.g];
          const uint64_t p = pbase[cw.g] + cw.ppre;
          q = bbase[cw.g] + cw.bpre;
          cnt = __popc(bits);
          if (q + cnt > cap) {
            atomicOr(status, (unsigned long long)CR_OVER);
            bits = 0;
            cnt = 0;
          } else {
            pc_ctx[p] = r.ctx;
            pc_off[p] = (uint32_t)(i - r.ow) << r.sh;
            src = r.ob + cw.bpre;
            pn = N + p;
          }
        }
      }
      const uint32_t incl = warp_incl_scan<uint32_t>(cnt);
      const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t j0 = 0; j0 < T; j0 += 32) {  // warp-uniform trip count
        const uint32_t j = j0 + lane;
        uint32_t L = 0;  // owner lane: the number of lanes whose inclusive count is <= j
#pragma unroll
        for (uint32_t st = 16; st; st >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, L + st - 1);
          if (v <= j) L += st;
        }
        L = L > 31 ? 31 : L;
        const uint32_t incl_L = __shfl_sync(0xffffffffu, incl, L), cnt_L = __shfl_sync(0xffffffffu, cnt, L);
        const uint32_t bits_L = __shfl_sync(0xffffffffu, bits, L);
        const uint64_t q_L = __shfl_sync(0xffffffffu, q, L), src_L = __shfl_sync(0xffffffffu, src, L),
                       pn_L = __shfl_sync(0xffffffffu, pn, L);
        if (j < T) {
          const uint32_t k = j - (incl_L - cnt_L);
          bin_pcnode[q_L + k] = (uint32_t)pn_L;
          bin_stall[q_L + k] = (uint16_t)__fns(bits_L, 0, (int)k + 1);
          bin_count[q_L + k] = bscr[src_L + k];
        }
      }
    }
  }
#else
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const CtxWord cw = wscr[i];
    uint32_t bits = cw.bits;
    if (!bits) continue;
    const CtxRec r = rec[cw.g];
    const uint64_t p = pbase[cw.g] + cw.ppre;
    uint64_t q = bbase[cw.g] + cw.bpre;
    if (q + __popc(bits) > cap) {
      atomicOr(status, (unsigned long long)CR_OVER);
      continue;
    }
    pc_ctx[p] = r.ctx;
    pc_off[p] = (uint32_t)(i - r.ow) << r.sh;
    const unsigned long long* src = bscr + r.ob + cw.bpre;
    uint32_t k = 0;
    while (bits) {
      const uint32_t b = __ffs(bits) - 1;
      bits &= bits - 1;
      bin_pcnode[q] = (uint32_t)(N + p);
      bin_stall[q] = (uint16_t)b;
      bin_count[q] = src[k++];
      ++q;
    }
  }
#endif
}

// ---------------------------------------------------------------- per-context reduce
// One CTA per context. Its partial entries (all segments of the context: several CTAs of the
// main kernel and several flushes) are processed in key-range chunks of at most RD_CAP
// entries (one chunk for almost every context); each chunk is gathered into shared memory,
// stably radix-sorted, reduced (equal keys summed) and appended, so the output is sorted.
constexpr int RD_THREADS = 1024;
constexpr uint32_t RD_CAP = 10240;  // entries sorted in shared memory at once
constexpr int RD_BUCKETS = 4096;

// Bitmap path: with pc' = pc_off >> (common trailing zero bits of the context's PCs), every
// (pc', stall) key is bit (pc' << 5 | stall) and every PC is exactly one 32-bit word, so a
// presence bitmap + word prefix sums give each distinct key its rank in (pc, stall) order
// directly — no sort. Used whenever the context's pc' range fits BM_WORDS words.
constexpr uint32_t BM_WORDS = 16384;  // 2^19 key bits, PCs with pc' < 16384
struct RedSmem {
  union {
    struct {
      uint32_t k[2][RD_CAP];
      uint32_t v[2][RD_CAP];
      uint32_t wcnt[32][256];
      uint32_t hist[RD_BUCKETS];
      uint16_t bchunk[RD_BUCKETS];
    } r;
    struct {
      uint32_t bm[BM_WORDS];
      uint32_t pre[BM_WORDS];
    } b;
  };
  unsigned long long wstall[32][32];  // [warp][stall]
  uint32_t fill, maxkey, prev_key, total, bad, orpc;
};

__global__ void __launch_bounds__(RD_THREADS, 1) k_own_reduce(
    const uint4* __restrict__ seg, const uint32_t* __restrict__ seg_order, const uint32_t* __restrict__ grp_start,
    uint32_t n_groups, const uint64_t* __restrict__ grp_out, const uint32_t* __restrict__ pkey,
    const unsigned long long* __restrict__ pcnt, uint64_t N, uint32_t* __restrict__ okey,
    unsigned long long* __restrict__ ocnt, uint32_t* __restrict__ g_nbins, uint32_t* __restrict__ g_npcs,
    uint32_t* __restrict__ g_ctx, unsigned long long* __restrict__ xsamples, unsigned long long* __restrict__ xstall,
    uint32_t S, uint32_t* g_flags) { DC_PDL_ENTER();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RedSmem& sm = *reinterpret_cast<RedSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  constexpr uint32_t HALF = RD_CAP / 2;
  for (uint32_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const uint32_t gs = grp_start[g], ge = grp_start[g + 1];
    const uint32_t ctx = seg[seg_order[gs]].x;
    unsigned long long stall_acc = 0;  // this lane's stall (= lane id) total over its warp's heads
    if (tid == 0) {
      sm.maxkey = 0;
      sm.orpc = 0;
      sm.bad = 0;
      sm.prev_key = 0xFFFFFFFFu;
      uint32_t tot = 0;
      for (uint32_t si = gs; si < ge; ++si) tot += seg[seg_order[si]].y;
      sm.total = tot;
    }
    __syncthreads();
    const uint32_t E = sm.total;
    // key range (sort width)
    uint32_t mk = 0, orp = 0;
    for (uint32_t si = gs; si < ge; ++si) {
      const uint4 sg = seg[seg_order[si]];
      const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
      for (uint32_t j = tid; j < sg.y; j += RD_THREADS) {
        const uint32_t kk = pkey[base + j];
        mk = max(mk, kk);
        orp |= kk >> 5;
      }
    }
    mk = __reduce_max_sync(0xffffffffu, mk);
    orp = __reduce_or_sync(0xffffffffu, orp);
    if (lane == 0) {
      atomicMax(&sm.maxkey, mk);
      atomicOr(&sm.orpc, orp);
    }
    __syncthreads();
    const uint64_t obase = grp_out[g];
    uint32_t n_out = 0, n_pc = 0;
    const int pshift = sm.orpc ? __ffs(sm.orpc) - 1 : 0;  // common trailing zero bits of the PCs
    const uint32_t nwords = ((sm.maxkey >> 5) >> pshift) + 1;
    if (nwords <= BM_WORDS) {
      // ---------------- bitmap path: bit (pc' << 5 | stall), one word per PC
      for (uint32_t wd = tid; wd < nwords; wd += RD_THREADS) sm.b.bm[wd] = 0;
      __syncthreads();
      for (uint32_t si = gs; si < ge; ++si) {
        const uint4 sg = seg[seg_order[si]];
        const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
        for (uint32_t j = tid; j < sg.y; j += RD_THREADS) {
          const uint32_t kk = pkey[base + j];
          atomicOr(&sm.b.bm[(kk >> 5) >> pshift], 1u << (kk & 31u));
        }
      }
      __syncthreads();
      // word prefix sums (rank of the first key of each PC) and PC count
      constexpr uint32_t WPT = BM_WORDS / RD_THREADS;  // 16 words per thread
      uint32_t cnt = 0, npc_t = 0;
#pragma unroll
      for (uint32_t q = 0; q < WPT; ++q) {
        const uint32_t wd = tid * WPT + q;
        const uint32_t bits = wd < nwords ? sm.b.bm[wd] : 0u;
        cnt += __popc(bits);
        npc_t += bits != 0;
      }
      uint32_t tot_bins, tot_pcs;
      uint32_t run = block_excl_scan<uint32_t, RD_THREADS>(cnt, &tot_bins);
      block_excl_scan<uint32_t, RD_THREADS>(npc_t, &tot_pcs);
      for (uint32_t q = 0; q < WPT; ++q) {
        const uint32_t wd = tid * WPT + q;
        if (wd >= nwords) break;
        uint32_t bits = sm.b.bm[wd];
        sm.b.pre[wd] = run;
        while (bits) {  // emit the PC's keys in stall order; counts start at 0
          const uint32_t b = __ffs(bits) - 1;
          bits &= bits - 1;
          okey[obase + run] = ((wd << pshift) << 5) | b;
          ocnt[obase + run] = 0;
          ++run;
        }
      }
      __syncthreads();  // orders the zeroing above before the atomics below (same CTA)
      for (uint32_t si = gs; si < ge; ++si) {
        const uint4 sg = seg[seg_order[si]];
        const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
        for (uint32_t j0 = 0; j0 < sg.y; j0 += RD_THREADS) {  // warp-uniform trip count
          const uint32_t j = j0 + tid;
          const bool ok = j < sg.y;
          const uint32_t kk = ok ? pkey[base + j] : 0;
          const unsigned long long cv = ok ? pcnt[base + j] : 0;
          if (ok) {
            const uint32_t wd = (kk >> 5) >> pshift, b = kk & 31u;
            const uint32_t rank = sm.b.pre[wd] + __popc(sm.b.bm[wd] & ((1u << b) - 1u));
            atomicAdd(&ocnt[obase + rank], cv);
          }
          const uint32_t my_stall = ok ? (kk & 31u) : 32u;
#pragma unroll 4
          for (int src = 0; src < 32; ++src) {
            const uint32_t st = __shfl_sync(0xffffffffu, my_stall, src);
            const unsigned long long sv = __shfl_sync(0xffffffffu, cv, src);
            if (st == lane) stall_acc += sv;
          }
        }
      }
      n_out = tot_bins;
      n_pc = tot_pcs;
    } else {
    const int kb = sm.maxkey ? 32 - __clz(sm.maxkey) : 1;
    const int bshift = kb > 12 ? kb - 12 : 0;
    uint32_t nchunks = 1;
    if (E > RD_CAP) {
      // chunk c holds the buckets whose exclusive prefix lies in [c*HALF, (c+1)*HALF): with every
      // bucket <= HALF, a chunk holds <= RD_CAP entries
      for (uint32_t b = tid; b < RD_BUCKETS; b += RD_THREADS) sm.r.hist[b] = 0;
      __syncthreads();
      for (uint32_t si = gs; si < ge; ++si) {
        const uint4 sg = seg[seg_order[si]];
        const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
        for (uint32_t j = tid; j < sg.y; j += RD_THREADS) atomicAdd(&sm.r.hist[pkey[base + j] >> bshift], 1u);
      }
      __syncthreads();
      uint32_t h4[4], s4 = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        h4[q] = sm.r.hist[tid * 4 + q];
        s4 += h4[q];
        if (h4[q] > HALF) sm.bad = 1;
      }
      uint32_t ex = block_excl_scan<uint32_t, RD_THREADS>(s4, nullptr);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sm.r.bchunk[tid * 4 + q] = (uint16_t)(ex / HALF);
        ex += h4[q];
      }
      __syncthreads();
      if (sm.bad) {
        if (tid == 0) atomicOr(g_flags, (uint32_t)OWF_FALLBACK);
        __syncthreads();
        continue;
      }
      nchunks = (E - 1) / HALF + 1;
    }
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
      if (tid == 0) sm.fill = 0;
      __syncthreads();
      for (uint32_t si = gs; si < ge; ++si) {
        const uint4 sg = seg[seg_order[si]];
        const uint64_t base = (uint64_t)sg.z | ((uint64_t)sg.w << 32);
        for (uint32_t j0 = 0; j0 < sg.y; j0 += RD_THREADS) {  // warp-uniform trip count
          const uint32_t j = j0 + tid;
          const uint32_t kk = j < sg.y ? pkey[base + j] : 0;
          const bool take = j < sg.y && (nchunks == 1 || sm.r.bchunk[kk >> bshift] == ch);
          const uint32_t m = __ballot_sync(0xffffffffu, take);
          uint32_t wbase = 0;
          if (lane == 0 && m) wbase = atomicAdd(&sm.fill, (uint32_t)__popc(m));  // one atomic per warp
          wbase = __shfl_sync(0xffffffffu, wbase, 0);
          if (take) {
            const uint32_t slot = wbase + __popc(m & lanemask_lt());
            sm.r.k[0][slot] = kk;
            sm.r.v[0][slot] = (uint32_t)(base + j);
          }
        }
      }
      __syncthreads();
      const uint32_t n = sm.fill;
      // stable LSD radix sort of (key, global index) over kb bits (equal keys are summed, so
      // their relative order does not matter)
      int cur = 0;
      const uint32_t per_warp = (n + 31) / 32;
      for (int shift = 0; shift < kb; shift += 8) {
        const int nb = kb - shift < 8 ? kb - shift : 8;
        const uint32_t mask = (1u << nb) - 1u;
        for (int i = tid; i < 32 * 256; i += RD_THREADS) (&sm.r.wcnt[0][0])[i] = 0;
        __syncthreads();
        const uint32_t b0 = w * per_warp, b1 = min(n, b0 + per_warp);
        for (uint32_t bs = b0; bs < b1; bs += 32) {
          const uint32_t j = bs + lane;
          const bool ok = j < b1;
          const uint32_t d = ok ? (sm.r.k[cur][j] >> shift) & mask : 0xFFFFFFFFu;
          const uint32_t peers = __match_any_sync(0xffffffffu, d);
          if (ok && (peers & lanemask_lt()) == 0) sm.r.wcnt[w][d] += __popc(peers);
          __syncwarp();
        }
        __syncthreads();
        uint32_t tot = 0;
        if (tid < 256)
          for (int ww = 0; ww < 32; ++ww) tot += sm.r.wcnt[ww][tid];
        const uint32_t ex = block_excl_scan<uint32_t, RD_THREADS>(tid < 256 ? tot : 0u, nullptr);
        if (tid < 256) {
          uint32_t run = ex;
          for (int ww = 0; ww < 32; ++ww) {
            const uint32_t c = sm.r.wcnt[ww][tid];
            sm.r.wcnt[ww][tid] = run;
            run += c;
          }
        }
        __syncthreads();
        for (uint32_t bs = b0; bs < b1; bs += 32) {
          const uint32_t j = bs + lane;
          const bool ok = j < b1;
          const uint32_t kk = ok ? sm.r.k[cur][j] : 0, vv = ok ? sm.r.v[cur][j] : 0;
          const uint32_t d = ok ? (kk >> shift) & mask : 0xFFFFFFFFu;
          const uint32_t peers = __match_any_sync(0xffffffffu, d);
          const uint32_t pos = ok ? sm.r.wcnt[w][d] + __popc(peers & lanemask_lt()) : 0;
          __syncwarp();
          if (ok && (peers & lanemask_lt()) == 0) sm.r.wcnt[w][d] += __popc(peers);
          __syncwarp();
          if (ok) {
            sm.r.k[cur ^ 1][pos] = kk;
            sm.r.v[cur ^ 1][pos] = vv;
          }
        }
        __syncthreads();
        cur ^= 1;
      }
      // reduce runs of equal keys; PC-node heads continue across chunk boundaries
      const uint32_t prev = sm.prev_key;
      for (uint32_t bs = 0; bs < n; bs += RD_THREADS) {
        const uint32_t j = bs + tid;
        const bool ok = j < n;
        const uint32_t kk = ok ? sm.r.k[cur][j] : 0;
        const uint32_t pk = j == 0 ? prev : (ok ? sm.r.k[cur][j - 1] : 0);
        const uint32_t head = ok && (pk != kk) ? 1u : 0u;
        const uint32_t pchead = ok && (pk == 0xFFFFFFFFu || (pk >> 5) != (kk >> 5)) ? 1u : 0u;
        uint32_t tot_h, tot_p;
        const uint32_t ex = block_excl_scan<uint32_t, RD_THREADS>(head, &tot_h);
        block_excl_scan<uint32_t, RD_THREADS>(pchead, &tot_p);
        unsigned long long s = 0;
        if (head) {
          for (uint32_t t = j; t < n && sm.r.k[cur][t] == kk; ++t) s += pcnt[sm.r.v[cur][t]];
          okey[obase + n_out + ex] = kk;
          ocnt[obase + n_out + ex] = s;
        }
        // per-stall totals without shared atomics: lane q of each warp collects stall q
        const uint32_t my_stall = head ? (kk & 31u) : 32u;
#pragma unroll 4
        for (int src = 0; src < 32; ++src) {
          const uint32_t st = __shfl_sync(0xffffffffu, my_stall, src);
          const unsigned long long sv = __shfl_sync(0xffffffffu, s, src);
          if (st == lane) stall_acc += sv;
        }
        n_out += tot_h;
        n_pc += tot_p;
        __syncthreads();
      }
      if (tid == 0 && n) sm.prev_key = sm.r.k[cur][n - 1];
      __syncthreads();
    }
    }  // radix path
    if (tid == 0) {
      g_nbins[g] = n_out;
      g_npcs[g] = n_pc;
      g_ctx[g] = ctx;
    }
    sm.wstall[w][lane] = stall_acc;
    __syncthreads();
    if (w == 0) {
      unsigned long long t = 0;
      for (int ww = 0; ww < RD_THREADS / 32; ++ww) t += sm.wstall[ww][lane];
      if (lane < S && ctx < N) xstall[(uint64_t)lane * N + ctx] = t;
      unsigned long long tot = lane < S ? t : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (lane == 0 && ctx < N) xsamples[ctx] = tot;
    }
    __syncthreads();
  }
}

// final SoA: one block per group
__global__ void k_own_place(const uint64_t* __restrict__ grp_out, const uint32_t* __restrict__ g_nbins,
                            const uint32_t* __restrict__ bin_base, const uint32_t* __restrict__ pc_base,
                            const uint32_t* __restrict__ g_ctx, uint32_t n_groups, const uint32_t* __restrict__ okey,
                            const unsigned long long* __restrict__ ocnt, uint64_t N, uint32_t* __restrict__ pc_ctx,
                            uint32_t* __restrict__ pc_off, uint32_t* __restrict__ bin_pcnode, uint16_t* __restrict__ bin_stall,
                            uint64_t* __restrict__ bin_count) { DC_PDL_ENTER();
  for (uint32_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const uint64_t ib = grp_out[g];
    const uint32_t nb = g_nbins[g], ob = bin_base[g], pb = pc_base[g], ctx = g_ctx[g];
    uint32_t run = 0;  // pc index carried across chunks
    for (uint32_t base = 0; base < nb; base += blockDim.x) {
      const uint32_t j = base + threadIdx.x;
      const bool ok = j < nb;
      const uint32_t kk = ok ? okey[ib + j] : 0;
      const uint32_t pchead = ok && (j == 0 || (okey[ib + j - 1] >> 5) != (kk >> 5)) ? 1u : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<uint32_t, 256>(pchead, &tot);
      if (ok) {
        const uint32_t pidx = pb + run + ex + pchead - 1u;
        if (pchead) {
          pc_ctx[pidx] = ctx;
          pc_off[pidx] = kk >> 5;
        }
        bin_pcnode[ob + j] = (uint32_t)(N + pidx);
        bin_stall[ob + j] = (uint16_t)(kk & 31u);
        bin_count[ob + j] = ocnt[ib + j];
      }
      run += tot;
    }
  }
}

__global__ void k_own_groups(const uint64_t* __restrict__ skey, uint32_t n, uint32_t* __restrict__ head) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    head[i] = (i == 0 || skey[i - 1] != skey[i]) ? 1u : 0u;
}
__global__ void k_own_gstart(const uint32_t* __restrict__ head, const uint32_t* __restrict__ hex, uint32_t n,
                             uint32_t* __restrict__ grp_start, uint32_t n_groups) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (head[i]) grp_start[hex[i]] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) grp_start[n_groups] = n;
}
__global__ void k_own_segkeys(const uint4* __restrict__ seg, uint32_t n, uint64_t* __restrict__ key, uint32_t* __restrict__ val) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    key[i] = seg[i].x;
    val[i] = i;
  }
}
__global__ void k_own_gsize(const uint4* __restrict__ seg, const uint32_t* __restrict__ order, const uint32_t* __restrict__ grp_start,
                            uint32_t n_groups, uint64_t* __restrict__ gsz) { DC_PDL_ENTER();
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_groups; g += gridDim.x * blockDim.x) {
    uint64_t s = 0;
    for (uint32_t i = grp_start[g]; i < grp_start[g + 1]; ++i) s += seg[order[i]].y;
    gsz[g] = s;
  }
}

dc_status pc_owner_hist(Ctx* c, dc_cct* t, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf,
                        uint64_t n_launch, const uint64_t* launch_off, uint32_t S, FillList& fl,
                        uint64_t* n_bins_out, int* handled) {
  *handled = 0;
  if (n == 0 || n_launch == 0 || n_launch >= (1ull << 31)) return DC_OK;
  const uint64_t N = t->N;
  const uint32_t G = (uint32_t)c->num_sms * OW_CPS;  // k_pc_owner CTAs (claims, spill chunks)
  const uint32_t Gs = (uint32_t)c->num_sms;          // one CTA per SM: the reduce kernels
  Buf<uint32_t> bad;
  Buf<uint64_t> k0, k1;
  Buf<uint32_t> v0, v1;
  // stage plan
  Buf<uint64_t> lrow, lsrc, lcnt, gst, rowpos, tot;
  Buf<uint32_t> lflag, gx, gfirst, row_launch, st_first, st_ctx;
  Buf<uint4> desc;
  Buf<uint8_t> row_valid;
  // rows: sum ceil(cnt/32) <= n/32 + n_launch; context padding < OW_ROWS rows per context (<= n_launch)
  const uint64_t st_cap = (n / 32 + n_launch + OW_ROWS - 1) / OW_ROWS + n_launch + 1;
  const uint64_t row_cap = OW_ROWS * st_cap;
  if (st_cap >= (1ull << 32)) return DC_OK;  // stage claims count in 32 bits
  const uint64_t* lkey_out = nullptr;  // launches' contexts in ascending order (the stage plan's sort)
  // every zeroed scratch of the schedule (and the caller's column fills) in one fill launch
  const bool counting_sort = N < (1ull << 31) && !getenv("DC_TEST_OWN_RADIX");
  Buf<uint32_t> hist;
  Buf<unsigned long long> ctr, ldiag, ctl;
  Buf<uint32_t> flags;
  const uint64_t ctl_n = 4 + 2 * (n_launch + 1);  // ctl[4] and the group (bins, pcs) arrays of the context reduce
  DC_TRY(alloc_fill(c, fl, bad, 1));
  if (counting_sort) DC_TRY(alloc_fill(c, fl, hist, N + 1));
  DC_TRY(alloc_fill(c, fl, row_valid, row_cap));
  DC_TRY(alloc_fill(c, fl, ctr, 2 + (uint64_t)G));  // entry / segment counters + per-CTA stage claims
  DC_TRY(alloc_fill(c, fl, flags, 2));
  DC_TRY(alloc_fill(c, fl, ldiag, DG_N));
  DC_TRY(alloc_fill(c, fl, ctl, ctl_n));
  DC_TRY(fill_flush(c, fl));
  {
    Region rp(c, "pc:prep");
    // launches ordered by context
    DC_TRY(alloc(c, k0, n_launch));
    DC_TRY(alloc(c, k1, n_launch));
    DC_TRY(alloc(c, v0, n_launch));
    DC_TRY(alloc(c, v1, n_launch));
    bool in1 = false;
    if (counting_sort) {
      Region rs(c, "prep:sort");
      dc_launch(k_own_hist, grid_for(c, n_launch, 256), 256, 0, c->stream, launch_leaf, launch_off, n_launch, n, N, hist.p, bad.p);
      DC_LAUNCHED(c);
      DC_TRY(excl_scan<uint32_t>(c, hist.p, hist.p, N + 1, nullptr));
      dc_launch(k_own_scatter, grid_for(c, n_launch, 256), 256, 0, c->stream, launch_leaf, n_launch, N, hist.p, k0.p, v0.p);
      DC_LAUNCHED(c);
    } else {
      dc_launch(k_own_check, grid_for(c, n_launch, 256), 256, 0, c->stream, launch_off, n_launch, n, bad.p);
      DC_LAUNCHED(c);
      dc_launch(k_own_keys, grid_for(c, n_launch, 256), 256, 0, c->stream, launch_leaf, n_launch, N, k0.p, v0.p);
      DC_LAUNCHED(c);
      Region rs(c, "prep:sort");
      DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, n_launch, 0, bits_for(N), &in1));
    }
    Region rpl(c, "prep:plan");
    const uint64_t* lkey = in1 ? k1.p : k0.p;
    lkey_out = lkey;
    const uint32_t* order = in1 ? v1.p : v0.p;
    DC_TRY(alloc(c, lrow, n_launch + 1));
    DC_TRY(alloc(c, lsrc, n_launch));
    DC_TRY(alloc(c, lcnt, n_launch));
    DC_TRY(alloc(c, lflag, n_launch + 1));
    DC_TRY(alloc(c, gx, n_launch + 1));
    DC_TRY(alloc(c, gfirst, n_launch + 1));
    DC_TRY(alloc(c, gst, n_launch + 1));
    DC_TRY(alloc(c, rowpos, n_launch));
    DC_TRY(alloc(c, tot, 1));
    DC_TRY(alloc(c, row_launch, row_cap));
    DC_TRY(alloc(c, st_first, st_cap));
    DC_TRY(alloc(c, st_ctx, st_cap));
    dc_launch(k_plan_launch, grid_for(c, n_launch, 256), 256, 0, c->stream, launch_off, order, lkey, n_launch, lrow.p, lflag.p,
                                                                    lsrc.p, lcnt.p);
    DC_LAUNCHED(c);
    // E: first row within the stream; group index (NG at gx[n])
    DC_TRY((excl_scan_pair<uint64_t, uint32_t>(c, lrow.p, lrow.p, lrow.p + n_launch, lflag.p, gx.p, gx.p + n_launch, n_launch)));
    dc_launch(k_plan_gfirst, grid_for(c, n_launch, 256), 256, 0, c->stream, lkey, gx.p, gx.p + n_launch, n_launch, gfirst.p);
    DC_LAUNCHED(c);
    dc_launch(k_plan_gstages, grid_for(c, n_launch, 256), 256, 0, c->stream, lrow.p, gfirst.p, gx.p + n_launch, n_launch, gst.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint64_t>(c, gst.p, gst.p, n_launch, tot.p));  // first stage per group, total stages
    dc_launch(k_plan_rows, grid_for(c, n_launch * 32, 256), 256, 0, c->stream, lrow.p, gx.p, gfirst.p, gst.p, lkey, order, lcnt.p,
                                                                       n_launch, row_cap, rowpos.p, row_launch.p,
                                                                       row_valid.p, st_first.p, st_ctx.p);
    DC_LAUNCHED(c);
    DC_TRY(alloc(c, desc, 4 * st_cap));
    dc_launch(k_plan_pieces, grid_for(c, st_cap, 256), 256, 0, c->stream, rowpos.p, lsrc.p, lcnt.p, st_first.p, st_ctx.p, tot.p,
              n_launch, desc.p);
    DC_LAUNCHED(c);
  }
  // partial outputs
  // entry pool: table flushes + spill chunks after each CTA's first (at most n entries, plus a
  // partly used last chunk per CTA); the first chunks sit after the pool
  const uint64_t cap_entries = n + 1 + (uint64_t)G * OW_SPILL_CAP;
  const uint32_t cap_segs = (uint32_t)(n_launch + 4ull * G + n / 4096 + n / OW_SPILL_CAP + 1024);
  Buf<uint32_t> pkey, cm, wide;
  Buf<uint64_t> cw;
  Buf<uint8_t> csh;
  uint64_t hw[2] = {0, 0};
  Buf<unsigned long long> pcnt;
  Buf<uint4> seg;
  Buf<uint2> seg_meta;
  uint64_t hc[2];
  uint32_t hf[2];
  {
    Region rp(c, "pc:main");
    DC_TRY(alloc(c, pkey, cap_entries + (uint64_t)G * OW_SPILL_CAP));
    DC_TRY(alloc(c, pcnt, cap_entries + (uint64_t)G * OW_SPILL_CAP));
    DC_TRY(alloc(c, seg, cap_segs));
    DC_TRY(alloc(c, seg_meta, cap_segs));
    OwnArgs a;
    a.smp = s;
    a.rowpos = rowpos.p;
    a.lsrc = lsrc.p;
    a.lcnt = lcnt.p;
    a.st_first = st_first.p;
    a.desc = desc.p;
    a.st_ctx = st_ctx.p;
    a.row_launch = row_launch.p;
    a.row_valid = row_valid.p;
    a.st_total = tot.p;
    a.n_launch = n_launch;
    a.N = N;
    a.S = S;
    a.pkey = pkey.p;
    a.pcnt = pcnt.p;
    a.cap_entries = cap_entries;
    a.seg = seg.p;
    a.seg_meta = seg_meta.p;
    a.cap_segs = cap_segs;
    a.g_entries = ctr.p;
    a.g_segs = (unsigned int*)(ctr.p + 1);
    a.g_flags = flags.p;
    a.trace_flags = c->d_flags;
    a.ldiag = ldiag.p;
    a.spill_base0 = cap_entries;
    a.probe_mode = 0;
    a.sink = flags.p;
    a.bad = bad.p;
    a.claim = ctr.p + 2;
    if (const char* pm = getenv("DC_OWN_MODE")) a.probe_mode = (uint32_t)atoi(pm);  // measurement only
    Buf<unsigned long long> dbg;
    if (a.probe_mode == 9 || a.probe_mode == 2) {
      DC_TRY(alloc_zero(c, dbg, (uint64_t)G * (OW_CONS_WARPS + 1) * 8));
      a.sink = reinterpret_cast<uint32_t*>(dbg.p);
    }
    const size_t smem = sizeof(OwnSmem);
    void (*kern)(OwnArgs) = k_pc_owner<0>;
    switch (a.probe_mode) {  // measurement variants only
      case 1: kern = k_pc_owner<1>; break;
      case 2: kern = k_pc_owner<2>; break;
      case 3: kern = k_pc_owner<3>; break;
      case 4: kern = k_pc_owner<4>; break;
      case 9: kern = k_pc_owner<9>; break;
      default: a.probe_mode = 0;
    }
    DC_SMEM_OPTIN(c, kern);
    {
      Region rk(c, "k:pc_owner");
      dc_launch(kern, G, OW_THREADS, smem, c->stream, a);
      DC_LAUNCHED(c);
    }
    if (a.probe_mode == 9 || a.probe_mode == 2) {  // measurement only: print the cycle splits
      std::vector<unsigned long long> hp((size_t)G * 8);
      DC_TRY(readback(c, dbg.p + (size_t)G * OW_CONS_WARPS * 8, hp.size() * 8, hp.data()));
      double ps[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pmax = 0;
      for (size_t i = 0; i < hp.size(); ++i) ps[i % 8] += (double)hp[i];
      for (uint32_t g = 0; g < G; ++g) pmax = std::max(pmax, (double)hp[8 * g + 4]);
      fprintf(stderr,
              "{\"own_producer\": {\"wait_empty_cyc\": %.0f, \"compose_cyc\": %.0f, \"stages\": %.1f, \"pieces\": %.1f, "
              "\"total_cyc\": %.0f, \"max_total_cyc\": %.0f}}\n",
              ps[0] / G, ps[1] / G, ps[2] / G, ps[3] / G, ps[4] / G, pmax);
    }
    if (a.probe_mode == 9) {  // measurement only: print the consumer cycle split
      std::vector<unsigned long long> h((size_t)G * OW_CONS_WARPS * 8);
      DC_TRY(readback(c, dbg.p, h.size() * 8, h.data()));
      double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (size_t i = 0; i < h.size(); ++i) s[i % 8] += (double)h[i];
      const double nw = (double)G * OW_CONS_WARPS;
      fprintf(stderr,
              "{\"own_split\": {\"wait_cyc\": %.0f, \"flush_cyc\": %.0f, \"work_cyc\": %.0f, \"stages\": %.1f, "
              "\"key_cyc\": %.0f, \"wait_after_flush_cyc\": %.0f, \"add_cyc\": %.0f, \"wait_done_cyc\": %.0f}}\n",
              s[0] / nw, s[1] / nw, s[2] / nw, s[3] / nw, s[4] / nw, s[5] / nw, s[6] / nw, s[7] / nw);
    }
    uint32_t hbad = 0;
    if (!getenv("DC_TEST_PC_BR")) {
      // ------------------------------------------------ context reduce (k_ctx_order, k_ctx_hist, scan, k_ctx_emit)
      Region rr(c, "pc:creduce");
      uint64_t cap = c->pc_bins_hint > (1ull << 20) ? c->pc_bins_hint : (1ull << 20);
      if (cap > n) cap = n ? n : 1;
      if (getenv("DC_TEST_PC_CAP")) cap = 1;  // test only: force the reallocate-and-rerun path
      const uint64_t wcap = std::max<uint64_t>(c->pc_words_hint, 4ull << 20);
      const uint64_t bcap = std::max<uint64_t>(c->pc_bins_hint, 4ull << 20);
      Buf<unsigned long long> bscr;
      Buf<CtxWord> wscr;
      Buf<CtxRec> rec;
      Buf<uint32_t> order;
      Buf<uint64_t> gbase;  // [bin base | pc base] (n_launch + 1 each)
      uint64_t* gn = reinterpret_cast<uint64_t*>(ctl.p + 4);  // [gnb | gnp] per group, zeroed with the counters
      DC_TRY(alloc(c, wscr, wcap));
      DC_TRY(alloc(c, bscr, bcap));
      DC_TRY(alloc(c, rec, n_launch));
      DC_TRY(alloc(c, order, n_launch));
      DC_TRY(alloc(c, gbase, 2 * (n_launch + 1)));
      auto outputs = [&](uint64_t k) -> dc_status {
        DC_TRY(palloc(c, t->pc_ctx, k));
        DC_TRY(palloc(c, t->pc_off, k));
        DC_TRY(palloc(c, t->bin_pcnode, k));
        DC_TRY(palloc(c, t->bin_stall, k));
        return palloc(c, t->bin_count, k);
      };
      auto drop_outputs = [&]() {
        void* q[] = {t->pc_ctx, t->pc_off, t->bin_pcnode, t->bin_stall, t->bin_count};
        for (void* x : q)
          if (x) cudaFreeAsync(x, c->stream);
        t->pc_ctx = t->pc_off = t->bin_pcnode = nullptr;
        t->bin_stall = nullptr;
        t->bin_count = nullptr;
      };
      auto clear_cols = [&]() -> dc_status {
        FillList f2;
        DC_TRY(fill_add(c, f2, t->xsamples, N * 8));
        DC_TRY(fill_add(c, f2, t->xstall, (uint64_t)S * N * 8));
        return fill_flush(c, f2);
      };
      DC_TRY(outputs(cap));
      dc_launch(k_ctx_order, 1, 1024, 0, c->stream, seg.p, a.g_segs, cap_segs, lkey_out, gfirst.p, gx.p + n_launch, order.p);
      DC_LAUNCHED(c);
      const size_t csmem = sizeof(CtxRedSmem);
      DC_SMEM_OPTIN(c, k_ctx_hist);
      {
        Region rk(c, "k:ctx_hist");
        // groups past NG keep zero (bins, pcs) for the scan over the n_launch bound: k_ctx_hist
        // writes every group < NG; the rest are cleared with the counters
        dc_launch(k_ctx_hist, Gs * CR_CPS, CR_THREADS, csmem, c->stream, seg.p, seg_meta.p, a.g_segs, cap_segs, pkey.p, pcnt.p, lkey_out, gfirst.p,
                  gx.p + n_launch, order.p, N, S, flags.p, ctl.p, wscr.p, wcap, bscr.p, bcap, rec.p, gn, gn + n_launch + 1,
                  (unsigned long long*)t->xsamples, (unsigned long long*)t->xstall);
        DC_LAUNCHED(c);
      }
      DC_TRY((excl_scan_pair<uint64_t, uint64_t>(c, gn, gbase.p, gbase.p + n_launch, gn + n_launch + 1,
                                                 gbase.p + n_launch + 1, gbase.p + 2 * n_launch + 1, n_launch)));
      auto emit = [&](uint64_t k) -> dc_status {
        Region rk(c, "k:ctx_emit");
        dc_launch(k_ctx_emit, grid_for(c, std::max<uint64_t>(c->pc_words_hint, 1ull << 16), 256), 256, 0, c->stream, wscr.p, ctl.p,
                  rec.p, gbase.p, gbase.p + n_launch + 1, bscr.p, N, k, ctl.p + 1, t->pc_ctx, t->pc_off, t->bin_pcnode,
                  t->bin_stall, t->bin_count, flags.p);
        DC_LAUNCHED(c);
        return DC_OK;
      };
      // split-phase: everything the host decides on is known after the scan, so the emission
      // runs while the host reads it back (no host turnaround between the scan and the kernels
      // that follow the call); a bin count past the capacity guess is seen on the host (nb > cap)
      uint64_t hst[3] = {0, 0, 0}, htot[2] = {0, 0};
      DC_TRY(readback_begin(c, {{flags.p, 8, hf}, {bad.p, 4, &hbad}, {ctl.p + 1, 24, hst}, {gbase.p + n_launch, 8, &htot[0]},
                                {gbase.p + 2 * n_launch + 1, 8, &htot[1]}, {ctr.p, 16, hc}}));
      DC_TRY(emit(cap));
      DC_TRY(readback_end(c));
      if (getenv("DC_PC_STATS"))  // measurement only
        fprintf(stderr, "{\"pc_stats\": {\"entries\": %llu, \"segments\": %llu, \"bins\": %llu, \"pcs\": %llu, \"status\": %llu, "
                "\"words\": %llu, \"scratch_bins\": %llu}}\n", (unsigned long long)hc[0], (unsigned long long)(hc[1] & 0xFFFFFFFFu),
                (unsigned long long)htot[0], (unsigned long long)htot[1], (unsigned long long)hst[0], (unsigned long long)hst[1],
                (unsigned long long)hst[2]);
      c->pc_words_hint = hst[1] + hst[1] / 8;
      if (hbad || hf[0]) {  // offsets inconsistent / owner fallback: generic schedule
        drop_outputs();
        if (hf[0] && !hbad && getenv("DC_TEST_OWNER_STRICT"))
          return fail(c, DC_ERR_STATE, "test: owner schedule fell back (flags 0x%x)", hf[0]);
        return DC_OK;
      }
      if (!(hst[0] & CR_WIDE)) {
        const uint64_t nb = htot[0], npc = htot[1];
        if (nb > cap) {  // more bins than the capacity guess: exact outputs, emit again
          drop_outputs();
          DC_TRY(outputs(nb));
          DC_TRY(emit(nb));
        }
        t->Npc = npc;
        t->Nbins = nb;
        c->pc_bins_hint = nb + nb / 8;
        DC_TRY(add_diag(c, ldiag.p));
        *n_bins_out = nb;
        *handled = 1;
        return DC_OK;
      }
      c->pc_bins_hint = std::max<uint64_t>(hst[2] + hst[2] / 8, c->pc_bins_hint);
      // a context too wide for shared memory: the global-bitmap reduce below (from scratch)
      drop_outputs();
      DC_TRY(clear_cols());
    }
    // the reduce's first kernels run on the device counts, before the one host round trip
    DC_TRY(alloc_zero(c, cm, 2 * N));  // cmax | cor
    DC_TRY(alloc(c, cw, N + 1));
    DC_TRY(alloc(c, csh, N));
    DC_TRY(alloc_zero(c, wide, 1));
    {
      Region rk(c, "k:br_range");
      dc_launch(k_br_range, grid_for(c, (uint64_t)cap_segs * BR_MAXCH * 32, 256), 256, 0, c->stream, seg.p, a.g_segs, cap_segs, pkey.p,
                N, cm.p, cm.p + N, flags.p);
      DC_LAUNCHED(c);
    }
    {
      Region rk(c, "k:br_words");
      dc_launch(k_br_words, grid_for(c, N, 256), 256, 0, c->stream, cm.p, cm.p + N, N, cw.p, csh.p, wide.p);
      DC_LAUNCHED(c);
    }
    DC_TRY(excl_scan<uint64_t>(c, cw.p, cw.p, N, cw.p + N));  // word base per context, W at cw[N]
    DC_TRY(readback_multi(c, {{ctr.p, 16, hc}, {flags.p, 8, hf}, {bad.p, 4, &hbad}, {cw.p + N, 8, &hw[0]},
                              {wide.p, 4, &hw[1]}}));
    if (hbad) return DC_OK;  // offsets inconsistent: generic schedule
    if (a.probe_mode == 9)
      fprintf(stderr, "{\"own_out\": {\"entries\": %llu, \"segments\": %llu}}\n", (unsigned long long)hc[0],
              (unsigned long long)(hc[1] & 0xFFFFFFFFu));
  }
  if (hf[0]) {  // fallback / overflow -> generic schedule (diag of this pass discarded)
    if (getenv("DC_TEST_OWNER_STRICT")) return fail(c, DC_ERR_STATE, "test: owner schedule fell back (flags 0x%x)", hf[0]);
    return DC_OK;
  }
  const uint32_t n_segs = (uint32_t)(hc[1] & 0xFFFFFFFFu);
  {
    // ------------------------------------------------ global bitmap reduce (see k_br_*)
    HostRegion hr(c, "br");
    Region rb(c, "pc:breduce");
    const int segs_grid = grid_for(c, (uint64_t)n_segs * BR_MAXCH * 32, 256);
    const uint64_t W = hw[0];
    if (!(hw[1] & 0xFFFFFFFFu) && W <= BR_MAX_TOTAL) {
      Buf<uint32_t> bm;
      Buf<uint64_t> pk;
      DC_TRY(alloc_zero(c, bm, W));
      DC_TRY(alloc(c, pk, W + 1));
      {
        Region rk(c, "k:br_bits");
        dc_launch(k_br_bits, segs_grid, 256, 0, c->stream, seg.p, n_segs, pkey.p, N, cw.p, csh.p, bm.p);
        DC_LAUNCHED(c);
      }
      {
        Region rk(c, "k:br_pop");
        dc_launch(k_br_pop, grid_for(c, W, 256), 256, 0, c->stream, bm.p, W, pk.p);
        DC_LAUNCHED(c);
      }
      // output arrays sized by the partial-entry count (every bin has at least one entry, every
      // PC node at least one bin) and allocated before the one round trip, so only the two
      // launches follow it
      const uint64_t nb_cap = hc[0] + (uint64_t)G * OW_SPILL_CAP;
      DC_TRY(palloc(c, t->pc_ctx, nb_cap));
      DC_TRY(palloc(c, t->pc_off, nb_cap));
      DC_TRY(palloc(c, t->bin_pcnode, nb_cap));
      DC_TRY(palloc(c, t->bin_stall, nb_cap));
      DC_TRY(palloc(c, t->bin_count, nb_cap));
      DC_TRY(excl_scan<uint64_t>(c, pk.p, pk.p, W, pk.p + W));
      uint64_t ht = 0;
      DC_TRY(readback(c, pk.p + W, 8, &ht));
      const uint64_t nb = ht >> 32, npc = ht & 0xFFFFFFFFu;
      if (nb > nb_cap) return fail(c, DC_ERR_STATE, "internal: %llu bins > %llu partial entries", (unsigned long long)nb,
                                   (unsigned long long)nb_cap);
      t->Npc = npc;
      t->Nbins = nb;
      DC_CUDA(c, cudaMemsetAsync(t->bin_count, 0, (nb ? nb : 1) * 8, c->stream));
      if (nb) {
        {
          Region rk(c, "k:br_emit");
          dc_launch(k_br_emit, grid_for(c, W, 256), 256, 0, c->stream, bm.p, pk.p, W, cw.p, csh.p, N, t->pc_ctx, t->pc_off,
                                                                t->bin_pcnode, t->bin_stall);
          DC_LAUNCHED(c);
        }
        {
          Region rk(c, "k:br_count");
          dc_launch(k_br_count, grid_for(c, (uint64_t)n_segs * BR_MAXCH * 32, 32 * BR_WARPS), 32 * BR_WARPS, 0, c->stream, seg.p, n_segs, pkey.p, pcnt.p, N, S, bm.p, pk.p, cw.p, csh.p, (unsigned long long*)t->bin_count,
              (unsigned long long*)t->xsamples, (unsigned long long*)t->xstall);
          DC_LAUNCHED(c);
        }
      }
      DC_TRY(add_diag(c, ldiag.p));
      *n_bins_out = nb;
      *handled = 1;
      return DC_OK;
    }
  }
  Region rr(c, "pc:reduce");
  // group segments by context
  Buf<uint64_t> sk0, sk1;
  Buf<uint32_t> sv0, sv1, head, hex, grp_start;
  DC_TRY(alloc(c, sk0, n_segs));
  DC_TRY(alloc(c, sk1, n_segs));
  DC_TRY(alloc(c, sv0, n_segs));
  DC_TRY(alloc(c, sv1, n_segs));
  DC_TRY(alloc(c, head, n_segs));
  DC_TRY(alloc(c, hex, n_segs));
  dc_launch(k_own_segkeys, grid_for(c, n_segs, 256), 256, 0, c->stream, seg.p, n_segs, sk0.p, sv0.p);
  DC_LAUNCHED(c);
  bool sin1 = false;
  DC_TRY(radix_sort_pairs(c, sk0.p, sv0.p, sk1.p, sv1.p, n_segs, 0, bits_for(N), &sin1));
  uint64_t* ssk = sin1 ? sk1.p : sk0.p;
  uint32_t* sso = sin1 ? sv1.p : sv0.p;
  dc_launch(k_own_groups, grid_for(c, n_segs, 256), 256, 0, c->stream, ssk, n_segs, head.p);
  DC_LAUNCHED(c);
  Buf<uint32_t> ng;
  DC_TRY(alloc(c, ng, 1));
  DC_TRY(excl_scan<uint32_t>(c, head.p, hex.p, n_segs, ng.p));
  uint32_t n_groups = 0;
  DC_TRY(readback(c, ng.p, 4, &n_groups));
  if (n_groups == 0) {  // no valid sample: no PC nodes, no bins
    t->Npc = t->Nbins = 0;
    DC_TRY(palloc(c, t->pc_ctx, 1));
    DC_TRY(palloc(c, t->pc_off, 1));
    DC_TRY(palloc(c, t->bin_pcnode, 1));
    DC_TRY(palloc(c, t->bin_stall, 1));
    DC_TRY(palloc(c, t->bin_count, 1));
    DC_TRY(add_diag(c, ldiag.p));
    *n_bins_out = 0;
    *handled = 1;
    return DC_OK;
  }
  DC_TRY(alloc(c, grp_start, n_groups + 1));
  dc_launch(k_own_gstart, grid_for(c, n_segs, 256), 256, 0, c->stream, head.p, hex.p, n_segs, grp_start.p, n_groups);
  DC_LAUNCHED(c);
  Buf<uint64_t> gsz, gout;
  DC_TRY(alloc(c, gsz, n_groups));
  DC_TRY(alloc(c, gout, n_groups + 1));
  dc_launch(k_own_gsize, grid_for(c, n_groups, 128), 128, 0, c->stream, seg.p, sso, grp_start.p, n_groups, gsz.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint64_t>(c, gsz.p, gout.p, n_groups, gout.p + n_groups));
  // per-context reduce
  Buf<uint32_t> okey, gnb, gnp, gctx, bbase, pbase;
  Buf<unsigned long long> ocnt;
  Buf<uint32_t> tots;
  DC_TRY(alloc(c, okey, hc[0] + (uint64_t)G * OW_SPILL_CAP));  // table entries + spills
  DC_TRY(alloc(c, ocnt, hc[0] + (uint64_t)G * OW_SPILL_CAP));
  DC_TRY(alloc(c, gnb, n_groups));
  DC_TRY(alloc(c, gnp, n_groups));
  DC_TRY(alloc(c, gctx, n_groups));
  DC_TRY(alloc(c, bbase, n_groups));
  DC_TRY(alloc(c, pbase, n_groups));
  DC_TRY(alloc(c, tots, 2));
  const size_t rsmem = sizeof(RedSmem);
  DC_SMEM_OPTIN(c, k_own_reduce);  // per device
  {
    Region rk(c, "k:own_reduce");
    dc_launch(k_own_reduce, n_groups < Gs ? n_groups : Gs, RD_THREADS, rsmem, c->stream, seg.p, sso, grp_start.p, n_groups, gout.p, pkey.p, pcnt.p, N, okey.p, ocnt.p, gnb.p, gnp.p, gctx.p,
        (unsigned long long*)t->xsamples, (unsigned long long*)t->xstall, S, flags.p);
    DC_LAUNCHED(c);
  }
  DC_TRY(readback(c, flags.p, 4, hf));
  if (hf[0]) {  // a context that cannot be chunked into shared memory: generic schedule
    DC_CUDA(c, cudaMemsetAsync(t->xsamples, 0, N * 8, c->stream));
    DC_CUDA(c, cudaMemsetAsync(t->xstall, 0, (uint64_t)S * N * 8, c->stream));
    return DC_OK;
  }
  DC_TRY(excl_scan<uint32_t>(c, gnb.p, bbase.p, n_groups, tots.p));
  DC_TRY(excl_scan<uint32_t>(c, gnp.p, pbase.p, n_groups, tots.p + 1));
  uint32_t ht[2];
  DC_TRY(readback(c, tots.p, 8, ht));
  const uint64_t nb = ht[0], npc = ht[1];
  t->Npc = npc;
  t->Nbins = nb;
  DC_TRY(palloc(c, t->pc_ctx, npc));
  DC_TRY(palloc(c, t->pc_off, npc));
  DC_TRY(palloc(c, t->bin_pcnode, nb));
  DC_TRY(palloc(c, t->bin_stall, nb));
  DC_TRY(palloc(c, t->bin_count, nb));
  dc_launch(k_own_place, n_groups < 4u * Gs ? (n_groups ? n_groups : 1) : 4 * Gs, 256, 0, c->stream, gout.p, gnb.p, bbase.p, pbase.p, gctx.p, n_groups, okey.p, ocnt.p, N, t->pc_ctx, t->pc_off, t->bin_pcnode,
      t->bin_stall, t->bin_count);
  DC_LAUNCHED(c);
  DC_TRY(add_diag(c, ldiag.p));
  *n_bins_out = nb;
  *handled = 1;
  return DC_OK;
}

}  // namespace dc
