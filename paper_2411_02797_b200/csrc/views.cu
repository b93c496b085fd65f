// views.cu — a7: analyzer views over the rolled-up CCT.
//   INCLUSIVE / EXCLUSIVE: hotspot identification ①: candidates = nodes of
//     the masked frame kinds, fraction = value / root inclusive value, strict > threshold,
//     order (value desc, id asc), first k.
//   BOTTOM_UP: the same frame aggregated across call paths, exclusive values.
//   STALL: stall-reason top-k of one node (analysis ④).
// Candidates are compacted in id order and stably radix-sorted by ~value, which yields
// (value desc, id asc) without a comparison sort.
#include <stdlib.h>
#include <vector>

#include "prim.cuh"

namespace dc {

__device__ __forceinline__ bool kind_ok(const uint8_t* fk, uint32_t n_frames, uint32_t f, uint32_t mask) {
  if (!fk) return true;
  if (f >= n_frames) return false;
  uint32_t k = fk[f];
  return k < 32 && ((mask >> k) & 1u);
}

__device__ __forceinline__ double frac_of(uint64_t v, uint64_t total) {
  return __ddiv_rn(__ull2double_rn(v), __ull2double_rn(total));
}

// flag[i] for candidates i in [0, n) of the view; value[i]
__global__ void k_view_nodes(const uint64_t* __restrict__ val, const uint32_t* __restrict__ frame, const uint8_t* __restrict__ fk,
                             uint32_t n_frames, uint32_t mask, uint64_t N, const uint64_t* __restrict__ total_p, double threshold,
                             uint32_t* __restrict__ flag) { DC_PDL_ENTER();
  const uint64_t total = *total_p;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
    bool ok = i > 0 && total > 0 && kind_ok(fk, n_frames, frame[i], mask) && frac_of(val[i], total) > threshold;
    flag[i] = ok ? 1u : 0u;
  }
}

__global__ void k_bu_accum(const uint64_t* __restrict__ xval, const uint32_t* __restrict__ frame, const uint8_t* __restrict__ fk,
                           uint32_t n_frames, uint32_t mask, uint64_t N, unsigned long long* __restrict__ byf,
                           uint32_t* __restrict__ seen) { DC_PDL_ENTER();
  for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t f = frame[i];
    if (f >= n_frames || !kind_ok(fk, n_frames, f, mask)) continue;
    uint64_t v = xval[i];
    if (v) atomicAdd(byf + f, (unsigned long long)v);
    seen[f] = 1u;
  }
}

__global__ void k_view_frames(const uint64_t* __restrict__ byf, const uint32_t* __restrict__ seen, uint32_t n_frames,
                              const uint64_t* __restrict__ total_p, double threshold, uint32_t* __restrict__ flag) { DC_PDL_ENTER();
  const uint64_t total = *total_p;
  for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < n_frames; f += gridDim.x * blockDim.x)
    flag[f] = (seen[f] && total > 0 && frac_of(byf[f], total) > threshold) ? 1u : 0u;
}

__global__ void k_view_compact(const uint64_t* __restrict__ val, const uint32_t* __restrict__ flag,
                               const uint32_t* __restrict__ pos, uint64_t n, uint64_t* __restrict__ key, uint32_t* __restrict__ id) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      key[pos[i]] = ~val[i];  // ascending ~value == descending value; stable keeps id order
      id[pos[i]] = (uint32_t)i;
    }
}

__global__ void k_view_emit(const uint64_t* __restrict__ key, const uint32_t* __restrict__ id, uint32_t k,
                            const uint64_t* __restrict__ total_p, dc_topk_entry* __restrict__ out) { DC_PDL_ENTER();
  const uint64_t total = *total_p;
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    uint64_t v = ~key[i];
    dc_topk_entry e;
    e.id = id[i];
    e._pad = 0;
    e.value = v;
    e.fraction = frac_of(v, total);
    out[i] = e;
  }
}

// one warp: rank S <= 32 stall counts by (count desc, stall asc), keep fraction > threshold
__global__ void k_view_stall(const uint64_t* __restrict__ istall, const uint64_t* __restrict__ isamples, uint64_t N,
                             uint32_t S, uint32_t node, double threshold, uint32_t k, dc_topk_entry* __restrict__ out,
                             uint32_t* __restrict__ n_out) { DC_PDL_ENTER();
  const uint32_t s = lane_id();
  const uint64_t total = isamples[node];
  uint64_t v = s < S ? istall[(uint64_t)s * N + node] : 0;
  bool ok = s < S && total > 0 && frac_of(v, total) > threshold;
  uint32_t okmask = __ballot_sync(0xffffffffu, ok);
  uint32_t rank = 0;
  for (uint32_t o = 0; o < 32; ++o) {
    uint64_t vo = __shfl_sync(0xffffffffu, v, o);
    if (((okmask >> o) & 1u) && (vo > v || (vo == v && o < s))) ++rank;
  }
  if (ok && rank < k) {
    dc_topk_entry e;
    e.id = s;
    e._pad = 0;
    e.value = v;
    e.fraction = frac_of(v, total);
    out[rank] = e;
  }
  if (s == 0) *n_out = min((uint32_t)__popc(okmask), k);
}

// ---------------------------------------------------------------- one-CTA top-k (small trees)
// Candidates are compacted into shared memory; the k-th largest composite key (value, ~id) —
// unique per candidate, so "larger" is exactly the (value desc, id asc) order — is found by a
// 12-digit radix select (8-bit digits, most significant first), the k keys >= it are gathered
// and placed by rank. The result count (or an overflow flag: more candidates than fit) is the
// header entry out[0], so the host reads the whole answer with ONE copy.
constexpr int TK_THREADS = 1024;
constexpr uint32_t TK_CAP = 8192;        // candidates held in shared memory
constexpr uint32_t TK_FRAMES = 8192;     // frames accumulated in shared memory (bottom-up)
constexpr uint32_t TK_MAXK = 1024;
constexpr uint64_t TK_MAX_NODES = 1ull << 18;
struct TopkSmem {
  uint64_t v[TK_CAP];
  uint32_t id[TK_CAP];
  unsigned long long byf[TK_FRAMES];
  uint32_t seen[TK_FRAMES / 32];
  uint32_t hist[256];
  uint64_t sel_v[TK_MAXK];
  uint32_t sel_id[TK_MAXK];
  uint32_t cnt, nsel, digit, rem, overflow;
  uint64_t total;
};

__device__ __forceinline__ uint32_t tk_digit(uint64_t v, uint32_t id, int p) {  // p = 0 (top) .. 11
  return p < 8 ? (uint32_t)(v >> (56 - 8 * p)) & 0xFFu : (uint32_t)((~id) >> (24 - 8 * (p - 8))) & 0xFFu;
}
__device__ __forceinline__ bool tk_greater(uint64_t va, uint32_t ia, uint64_t vb, uint32_t ib) {
  return va > vb || (va == vb && ia < ib);
}

__global__ void __launch_bounds__(TK_THREADS, 1) k_topk_one(const uint64_t* __restrict__ val, const uint32_t* __restrict__ frame,
                                                           const uint8_t* __restrict__ fk, uint32_t n_frames, uint32_t mask,
                                                           uint64_t N, const uint64_t* __restrict__ total_p, double threshold,
                                                           uint32_t k, int bottom_up, dc_topk_entry* __restrict__ out) { DC_PDL_ENTER();
  extern __shared__ __align__(16) unsigned char tk_raw[];
  TopkSmem& sm = *reinterpret_cast<TopkSmem*>(tk_raw);
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    sm.cnt = 0;
    sm.nsel = 0;
    sm.overflow = 0;
    sm.total = *total_p;
  }
  if (bottom_up) {
    for (uint32_t f = tid; f < n_frames; f += TK_THREADS) sm.byf[f] = 0;
    for (uint32_t w = tid; w < (n_frames + 31) / 32; w += TK_THREADS) sm.seen[w] = 0;
  }
  __syncthreads();
  const uint64_t total = sm.total;
  if (bottom_up) {  // same frame across call paths: exclusive values summed per frame
    for (uint64_t i = 1 + tid; i < N; i += TK_THREADS) {
      const uint32_t f = frame[i];
      if (f >= n_frames || !kind_ok(fk, n_frames, f, mask)) continue;
      const uint64_t v = val[i];
      if (v) atomicAdd(&sm.byf[f], (unsigned long long)v);
      atomicOr(&sm.seen[f >> 5], 1u << (f & 31));
    }
    __syncthreads();
    if (total > 0)
      for (uint32_t f = tid; f < n_frames; f += TK_THREADS) {
        const uint64_t v = sm.byf[f];
        if (((sm.seen[f >> 5] >> (f & 31)) & 1u) && frac_of(v, total) > threshold) {
          const uint32_t q = atomicAdd(&sm.cnt, 1u);
          if (q < TK_CAP) {
            sm.v[q] = v;
            sm.id[q] = f;
          }
        }
      }
  } else if (total > 0) {
    for (uint64_t i = 1 + tid; i < N; i += TK_THREADS) {
      if (!kind_ok(fk, n_frames, frame[i], mask)) continue;
      const uint64_t v = val[i];
      if (frac_of(v, total) > threshold) {
        const uint32_t q = atomicAdd(&sm.cnt, 1u);
        if (q < TK_CAP) {
          sm.v[q] = v;
          sm.id[q] = (uint32_t)i;
        }
      }
    }
  }
  __syncthreads();
  if (sm.cnt > TK_CAP) {  // more candidates than shared memory holds: the host takes the general path
    if (tid == 0) {
      dc_topk_entry h = {};
      h._pad = 1;
      out[0] = h;
    }
    return;
  }
  const uint32_t c = sm.cnt, kk = min(k, c);
  if (c <= (uint32_t)TK_THREADS) {
    // few candidates (the usual case: the threshold keeps a handful of hotspots): every
    // candidate's rank among all of them directly, one pass instead of up to 12 radix passes
    if (tid < c) {
      const uint64_t v = sm.v[tid];
      const uint32_t id = sm.id[tid];
      uint32_t rank = 0;
      for (uint32_t o = 0; o < c; ++o) rank += tk_greater(sm.v[o], sm.id[o], v, id) ? 1u : 0u;
      if (rank < kk) {
        dc_topk_entry en;
        en.id = id;
        en._pad = 0;
        en.value = v;
        en.fraction = frac_of(v, total);
        out[1 + rank] = en;
      }
    }
    if (tid == 0) {
      dc_topk_entry h = {};
      h.id = kk;
      out[0] = h;
    }
    return;
  }
  // radix select of the kk-th largest (value, ~id); every candidate key is distinct
  uint64_t pv = 0;   // prefix of the value digits found so far
  uint32_t pid = 0;  // prefix of the ~id digits
  if (tid == 0) sm.rem = kk;
  for (int p = 0; p < 12 && kk < c; ++p) {
    if (tid < 256) sm.hist[tid] = 0;
    __syncthreads();
    for (uint32_t q = tid; q < c; q += TK_THREADS) {
      const uint64_t v = sm.v[q];
      const uint32_t ni = ~sm.id[q];
      bool match;
      if (p < 8) match = p == 0 || (v >> (64 - 8 * p)) == (pv >> (64 - 8 * p));
      else match = v == pv && (p == 8 || (ni >> (32 - 8 * (p - 8))) == (pid >> (32 - 8 * (p - 8))));
      if (match) atomicAdd(&sm.hist[tk_digit(v, sm.id[q], p)], 1u);
    }
    __syncthreads();
    if (tid < 32) {  // largest digit d with (count of digits >= d) >= rem
      const uint32_t rem = sm.rem;
      uint32_t above = 0;
      uint32_t d = 0, cnt_above = 0;
      for (int g = 7; g >= 0; --g) {  // 8 groups of 32 digits, top down
        const uint32_t dg = (uint32_t)g * 32 + tid;
        const uint32_t h = sm.hist[dg];
        // inclusive suffix sum within the group (digits >= dg)
        uint32_t suf = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u = __shfl_down_sync(0xffffffffu, suf, o);
          if (tid + o < 32) suf += u;
        }
        const uint32_t hit = __ballot_sync(0xffffffffu, above + suf >= rem);
        if (hit) {
          const int l = 31 - __clz(hit);  // largest digit in the group reaching rem
          d = (uint32_t)g * 32 + l;
          const uint32_t suf_l = __shfl_sync(0xffffffffu, suf, l);
          const uint32_t h_l = __shfl_sync(0xffffffffu, h, l);
          cnt_above = above + suf_l - h_l;
          break;
        }
        above += __shfl_sync(0xffffffffu, suf, 0);
      }
      if (tid == 0) {
        sm.digit = d;
        sm.rem = rem - cnt_above;
      }
    }
    __syncthreads();
    const uint32_t d = sm.digit;
    if (p < 8) pv |= (uint64_t)d << (56 - 8 * p);
    else pid |= d << (24 - 8 * (p - 8));
  }
  // gather the kk largest: key >= (pv, ~pid) (all candidates when kk == c)
  const uint32_t kid = ~pid;
  for (uint32_t q = tid; q < c; q += TK_THREADS) {
    const uint64_t v = sm.v[q];
    const uint32_t id = sm.id[q];
    if (kk == c || v > pv || (v == pv && id <= kid)) {
      const uint32_t s = atomicAdd(&sm.nsel, 1u);
      if (s < TK_MAXK) {
        sm.sel_v[s] = v;
        sm.sel_id[s] = id;
      }
    }
  }
  __syncthreads();
  const uint32_t ns = min(sm.nsel, kk);
  for (uint32_t e = tid; e < ns; e += TK_THREADS) {
    const uint64_t v = sm.sel_v[e];
    const uint32_t id = sm.sel_id[e];
    uint32_t rank = 0;
    for (uint32_t o = 0; o < ns; ++o) rank += tk_greater(sm.sel_v[o], sm.sel_id[o], v, id) ? 1u : 0u;
    dc_topk_entry en;
    en.id = id;
    en._pad = 0;
    en.value = v;
    en.fraction = frac_of(v, total);
    out[1 + rank] = en;
  }
  if (tid == 0) {
    dc_topk_entry h = {};
    h.id = ns;
    out[0] = h;
  }
}

dc_status hotspots_topk(Ctx* c, const dc_cct* t, dc_view view, uint32_t metric, uint32_t kind_mask, double threshold, uint32_t k,
                        uint32_t stall_node, dc_topk_entry* out_h, uint32_t* n_out_h) {
  *n_out_h = 0;
  if (t->state != 2) return fail(c, DC_ERR_STATE, "dc_hotspots_topk needs a rolled-up tree (call dc_cct_rollup)");
  if (k == 0) return DC_OK;
  Buf<dc_topk_entry> out;
  DC_TRY(alloc(c, out, k));
  if (view == DC_VIEW_STALL) {
    if (stall_node >= t->N) return fail(c, DC_ERR_ARG, "stall_node %u >= n_nodes", stall_node);
    if (!t->xsamples) return DC_OK;
    const uint32_t ks = k < 32 ? k : 32;  // at most 32 stall reasons
    DC_TRY(alloc(c, out, ks + 1));
    dc_launch(k_view_stall, 1, 32, 0, c->stream, t->istall, t->isamples, t->N, t->S, stall_node, threshold, ks, out.p + 1,
              (uint32_t*)out.p);
    DC_LAUNCHED(c);
    std::vector<dc_topk_entry> h(ks + 1);
    DC_TRY(readback(c, out.p, (ks + 1) * sizeof(dc_topk_entry), h.data()));
    const uint32_t nh = h[0].id;
    for (uint32_t i = 0; i < nh; ++i) out_h[i] = h[1 + i];
    *n_out_h = nh;
    return DC_OK;
  }
  const uint64_t *ival, *xval;
  if (metric == DC_METRIC_SAMPLES) {
    if (!t->xsamples) return DC_OK;
    ival = t->isamples;
    xval = t->xsamples;
  } else {
    if (metric >= t->M) return fail(c, DC_ERR_ARG, "metric %u >= M = %u", metric, t->M);
    ival = t->col(C_ISUM, metric);
    xval = t->col(C_XSUM, metric);
  }
  const uint64_t* total_p = ival;  // root = node 0
  const bool bu = view == DC_VIEW_BOTTOM_UP;
  if ((view == DC_VIEW_INCLUSIVE || view == DC_VIEW_EXCLUSIVE || bu) && t->N <= TK_MAX_NODES && k <= TK_MAXK &&
      (!bu || t->n_frames <= TK_FRAMES) && !getenv("DC_TEST_TOPK_GENERAL")) {
    Buf<dc_topk_entry> o1;
    DC_TRY(alloc(c, o1, k + 1));
    DC_SMEM_OPTIN(c, k_topk_one);
    dc_launch(k_topk_one, 1, TK_THREADS, sizeof(TopkSmem), c->stream, view == DC_VIEW_INCLUSIVE ? ival : xval, t->frame,
              t->frame_kind, t->n_frames, kind_mask, t->N, total_p, threshold, k, bu ? 1 : 0, o1.p);
    DC_LAUNCHED(c);
    std::vector<dc_topk_entry> h(k + 1);
    DC_TRY(readback(c, o1.p, (k + 1) * sizeof(dc_topk_entry), h.data()));
    if (!h[0]._pad) {  // else: more candidates than the one-CTA path holds, general path below
      const uint32_t nh = h[0].id;
      for (uint32_t i = 0; i < nh; ++i) out_h[i] = h[1 + i];
      *n_out_h = nh;
      c->bytes_host += 8 * t->N;
      return DC_OK;
    }
  }
  uint64_t n = 0;
  const uint64_t* val = nullptr;
  Buf<unsigned long long> byf;
  Buf<uint32_t> seen, flag, pos;
  Buf<uint32_t> cnt;
  DC_TRY(alloc(c, cnt, 1));
  if (view == DC_VIEW_INCLUSIVE || view == DC_VIEW_EXCLUSIVE) {
    n = t->N;
    val = view == DC_VIEW_INCLUSIVE ? ival : xval;
    DC_TRY(alloc(c, flag, n));
    dc_launch(k_view_nodes, grid_for(c, n, 256), 256, 0, c->stream, val, t->frame, t->frame_kind, t->n_frames, kind_mask, n, total_p,
                                                             threshold, flag.p);
    DC_LAUNCHED(c);
  } else if (view == DC_VIEW_BOTTOM_UP) {
    n = t->n_frames;
    DC_TRY(alloc_zero(c, byf, n));
    DC_TRY(alloc_zero(c, seen, n));
    DC_TRY(alloc(c, flag, n));
    dc_launch(k_bu_accum, grid_for(c, t->N, 256), 256, 0, c->stream, xval, t->frame, t->frame_kind, t->n_frames, kind_mask, t->N,
                                                              byf.p, seen.p);
    DC_LAUNCHED(c);
    dc_launch(k_view_frames, grid_for(c, n, 256), 256, 0, c->stream, (const uint64_t*)byf.p, seen.p, (uint32_t)n, total_p, threshold,
                                                              flag.p);
    DC_LAUNCHED(c);
    val = (const uint64_t*)byf.p;
  } else {
    return fail(c, DC_ERR_ARG, "unknown view %d", (int)view);
  }
  DC_TRY(alloc(c, pos, n));
  DC_TRY(excl_scan<uint32_t>(c, flag.p, pos.p, n, cnt.p));
  uint32_t nc = 0;
  DC_TRY(readback(c, cnt.p, 4, &nc));
  if (nc == 0) return DC_OK;
  Buf<uint64_t> k0, k1;
  Buf<uint32_t> i0, i1;
  DC_TRY(alloc(c, k0, nc));
  DC_TRY(alloc(c, k1, nc));
  DC_TRY(alloc(c, i0, nc));
  DC_TRY(alloc(c, i1, nc));
  dc_launch(k_view_compact, grid_for(c, n, 256), 256, 0, c->stream, val, flag.p, pos.p, n, k0.p, i0.p);
  DC_LAUNCHED(c);
  bool in1 = false;
  DC_TRY(radix_sort_pairs(c, k0.p, i0.p, k1.p, i1.p, nc, 0, 64, &in1));
  uint32_t kk = nc < k ? nc : k;
  dc_launch(k_view_emit, 1, 256, 0, c->stream, in1 ? k1.p : k0.p, in1 ? i1.p : i0.p, kk, total_p, out.p);
  DC_LAUNCHED(c);
  DC_TRY(readback(c, out.p, kk * sizeof(dc_topk_entry), out_h));
  *n_out_h = kk;
  c->bytes_host += 8 * t->N;
  return DC_OK;
}

}  // namespace dc
