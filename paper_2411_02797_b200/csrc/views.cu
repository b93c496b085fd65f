// views.cu — a7: analyzer views over the rolled-up CCT.
//   INCLUSIVE / EXCLUSIVE: hotspot identification ①: candidates = nodes of
//     the masked frame kinds, fraction = value / root inclusive value, strict > threshold,
//     order (value desc, id asc), first k.
//   BOTTOM_UP: the same frame aggregated across call paths, exclusive values.
//   STALL: stall-reason top-k of one node (analysis ④).
// Candidates are compacted in id order and stably radix-sorted by ~value, which yields
// (value desc, id asc) without a comparison sort.
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
    Buf<uint32_t> nout;
    DC_TRY(alloc(c, nout, 1));
    dc_launch(k_view_stall, 1, 32, 0, c->stream, t->istall, t->isamples, t->N, t->S, stall_node, threshold, k, out.p, nout.p);
    DC_LAUNCHED(c);
    uint32_t h = 0;
    DC_TRY(readback(c, nout.p, 4, &h));
    if (h) DC_TRY(readback(c, out.p, h * sizeof(dc_topk_entry), out_h));
    *n_out_h = h;
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
