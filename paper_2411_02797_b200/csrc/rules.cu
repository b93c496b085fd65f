// rules.cu — SURVEY §8(f) NEXT-2: the analyzer's rule predicates as device kernels over the
// rolled-up CCT (readings R22-R24).
//   ② small kernels (SPEC.md analyze_kernel_fusion): breadth-first over the
//      frame nodes, n qualifies if launches(n) > 0 and gpu_time(n) / launches(n) < threshold,
//      launches(n) = records in n's subtree that end at a frame of the kernel kind mask,
//      gpu_time(n) = inclusive sum of the time metric; a qualifying node is flagged unless an
//      ancestor qualifies ("children of a flagged node are not re-flagged").
//   ⑤ CPU latency (SPEC.md analyze_cpu_latency): n qualifies if
//      cpu(n) / max(gpu(n), 1) > threshold and cpu(n) > floor; same ancestor suppression.
//   ④ stalls (SPEC.md analyze_stalls): for every hotspot (view ①), its
//      instruction (PC) children whose samples / the hotspot's samples > stall_threshold; their
//      stall counts summed per reason; top-k reasons by (count desc, reason asc).
// Ratios are formed in binary64 with single roundings (__ddiv_rn), as in the oracle.
#include "prim.cuh"

namespace dc {

dc_status hotspots_topk(Ctx* c, const dc_cct* t, dc_view view, uint32_t metric, uint32_t kind_mask, double threshold, uint32_t k,
                        uint32_t stall_node, dc_topk_entry* out_h, uint32_t* n_out_h);

__device__ __forceinline__ bool rule_kind_ok(const uint8_t* fk, uint32_t n_frames, uint32_t f, uint32_t mask) {
  if (!fk) return true;
  if (f >= n_frames) return false;
  const uint32_t k = fk[f];
  return k < 32 && ((mask >> k) & 1u);
}
__device__ __forceinline__ double rdiv(uint64_t a, uint64_t b) { return __ddiv_rn(__ull2double_rn(a), __ull2double_rn(b)); }

// launches(n) = sum of xcnt over masked-kind nodes of n's subtree: own value + push to ancestors
__global__ void k_rule_launches(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ frame,
                                const uint8_t* __restrict__ fk, uint32_t n_frames, uint32_t mask,
                                const uint64_t* __restrict__ xcnt, uint64_t N, unsigned long long* __restrict__ il) { DC_PDL_ENTER();
  for (uint64_t n = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = rule_kind_ok(fk, n_frames, frame[n], mask) ? xcnt[n] : 0;
    if (!v) continue;
    atomicAdd(il + n, (unsigned long long)v);
    for (uint32_t a = parent[n], prev = (uint32_t)n; a < prev && a != 0; prev = a, a = parent[a]) atomicAdd(il + a, (unsigned long long)v);
  }
}

__global__ void k_rule_kind_gate(const uint32_t* __restrict__ frame, const uint8_t* __restrict__ fk, uint32_t n_frames,
                                 uint32_t mask, uint64_t N, unsigned long long* __restrict__ gate) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x)
    gate[n] = (n > 0 && rule_kind_ok(fk, n_frames, frame[n], mask)) ? 1ull : 0ull;
}

__global__ void k_rule_qualify(int rule, uint64_t N, const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                               const uint64_t* __restrict__ il, double threshold, uint64_t floor, uint8_t* __restrict__ q) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x) {
    bool ok = false;
    if (n > 0) {
      if (rule == DC_RULE_SMALL_KERNELS) {
        const uint64_t l = il[n];
        ok = l > 0 && rdiv(a[n], l) < threshold;
      } else if (rule == DC_RULE_BWD_FWD) {  // kind gate applied by the caller through il (0/1)
        const uint64_t bwd = a[n], fwd = b[n];
        ok = il[n] != 0 && fwd > 0 && fwd >= floor && rdiv(bwd, fwd) > threshold;
      } else {
        const uint64_t cpu = a[n], gpu = b[n];
        ok = cpu > floor && rdiv(cpu, gpu > 0 ? gpu : 1) > threshold;
      }
    }
    q[n] = ok ? 1 : 0;
  }
}

// flagged = qualifies and no proper (non-root) ancestor qualifies
__global__ void k_rule_suppress(const uint32_t* __restrict__ parent, uint64_t N, const uint8_t* __restrict__ q,
                                uint32_t* __restrict__ flag, int suppress) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x) {
    bool f = q[n] != 0;
    if (f && suppress)
      for (uint32_t a = parent[n], prev = (uint32_t)n; a < prev && a != 0; prev = a, a = parent[a])
        if (q[a]) {
          f = false;
          break;
        }
    flag[n] = f ? 1u : 0u;
  }
}

__global__ void k_rule_emit(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, uint64_t N, uint32_t cap,
                            uint32_t* __restrict__ out) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x)
    if (flag[n] && pos[n] < cap) out[pos[n]] = (uint32_t)n;
}

dc_status analyze_flags(Ctx* c, const dc_cct* t, dc_rule rule, const dc_rule_params* p, uint32_t* out_h, uint32_t cap,
                        uint32_t* n_out_h) {
  *n_out_h = 0;
  if (t->state != 2) return fail(c, DC_ERR_STATE, "dc_analyze_flags needs a rolled-up tree (call dc_cct_rollup)");
  if (t->partition) return fail(c, DC_ERR_STATE, "dc_analyze_flags needs a complete tree (gather the partitions first)");
  if (rule != DC_RULE_SMALL_KERNELS && rule != DC_RULE_CPU_LATENCY && rule != DC_RULE_BWD_FWD)
    return fail(c, DC_ERR_ARG, "unknown rule %d", (int)rule);
  if (p->metric_a >= t->M || (rule != DC_RULE_SMALL_KERNELS && p->metric_b >= t->M))
    return fail(c, DC_ERR_ARG, "metric out of range (M = %u)", t->M);
  const uint64_t N = t->N;
  Buf<unsigned long long> il;
  Buf<uint8_t> q;
  Buf<uint32_t> flag, pos, cnt, out;
  if (rule == DC_RULE_SMALL_KERNELS) {
    DC_TRY(alloc_zero(c, il, N));
    dc_launch(k_rule_launches, grid_for(c, N, 256), 256, 0, c->stream, t->parent, t->frame, t->frame_kind, t->n_frames, p->kind_mask,
                                                               t->xcnt, N, il.p);
    DC_LAUNCHED(c);
  } else if (rule == DC_RULE_BWD_FWD) {  // operator nodes: the kind gate as a 0/1 column
    DC_TRY(alloc(c, il, N));
    dc_launch(k_rule_kind_gate, grid_for(c, N, 256), 256, 0, c->stream, t->frame, t->frame_kind, t->n_frames, p->kind_mask, N, il.p);
    DC_LAUNCHED(c);
  }
  DC_TRY(alloc(c, q, N));
  DC_TRY(alloc(c, flag, N));
  DC_TRY(alloc(c, pos, N));
  DC_TRY(alloc(c, cnt, 1));
  DC_TRY(alloc(c, out, cap ? cap : 1));
  dc_launch(k_rule_qualify, grid_for(c, N, 256), 256, 0, c->stream, (int)rule, N, t->col(C_ISUM, p->metric_a),
                                                             rule != DC_RULE_SMALL_KERNELS ? t->col(C_ISUM, p->metric_b) : nullptr,
                                                             (const uint64_t*)il.p, p->threshold, p->floor, q.p);
  DC_LAUNCHED(c);
  // ② and ⑤ report the highest qualifying frame; ③ is per operator node (no suppression)
  dc_launch(k_rule_suppress, grid_for(c, N, 256), 256, 0, c->stream, t->parent, N, q.p, flag.p, rule == DC_RULE_BWD_FWD ? 0 : 1);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint32_t>(c, flag.p, pos.p, N, cnt.p));
  dc_launch(k_rule_emit, grid_for(c, N, 256), 256, 0, c->stream, flag.p, pos.p, N, cap, out.p);
  DC_LAUNCHED(c);
  uint32_t nf = 0;
  DC_TRY(readback(c, cnt.p, 4, &nf));
  const uint32_t m = nf < cap ? nf : cap;
  if (m) DC_TRY(readback(c, out.p, (size_t)m * 4, out_h));
  *n_out_h = nf;  // total flagged; the first min(nf, cap) ids (ascending = breadth-first) are written
  return DC_OK;
}

// ---- ④: one block per hotspot node
constexpr int ST_THREADS = 256;
__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint64_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(ST_THREADS) k_stall_issues(const uint32_t* __restrict__ hot, uint64_t N, uint64_t Npc,
                                                             uint64_t Nb, uint32_t S, const uint32_t* __restrict__ pc_ctx,
                                                             const uint32_t* __restrict__ bin_pcnode,
                                                             const uint16_t* __restrict__ bin_stall,
                                                             const uint64_t* __restrict__ bin_count,
                                                             const uint64_t* __restrict__ isamples, double stall_threshold,
                                                             uint32_t k, unsigned long long* __restrict__ pc_tot,
                                                             dc_stall_issue* __restrict__ out, uint32_t* __restrict__ n_out) { DC_PDL_ENTER();
  __shared__ unsigned long long ss[32];
  const uint32_t node = hot[blockIdx.x];
  if (threadIdx.x < 32) ss[threadIdx.x] = 0;
  const uint64_t plo = lower_bound_u32(pc_ctx, Npc, node), phi = lower_bound_u32(pc_ctx, Npc, (uint64_t)node + 1);
  const uint64_t blo = lower_bound_u32(bin_pcnode, Nb, N + plo), bhi = lower_bound_u32(bin_pcnode, Nb, N + phi);
  const uint64_t total = isamples[node];
  __syncthreads();
  // per-instruction sample totals (this block's PC nodes are its own: disjoint slices of pc_tot)
  for (uint64_t b = blo + threadIdx.x; b < bhi; b += ST_THREADS)
    atomicAdd(pc_tot + (bin_pcnode[b] - N), (unsigned long long)bin_count[b]);
  __syncthreads();
  for (uint64_t b = blo + threadIdx.x; b < bhi; b += ST_THREADS) {
    const uint64_t pt = pc_tot[bin_pcnode[b] - N];
    if (total > 0 && rdiv(pt, total) > stall_threshold && bin_stall[b] < 32)
      atomicAdd(&ss[bin_stall[b]], (unsigned long long)bin_count[b]);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // rank the reasons: (count desc, reason asc), non-zero only
    const uint32_t s = threadIdx.x;
    const uint64_t v = s < S ? ss[s] : 0;
    const bool ok = v > 0;
    const uint32_t okm = __ballot_sync(0xffffffffu, ok);
    uint32_t rank = 0;
    for (uint32_t o = 0; o < 32; ++o) {
      const uint64_t vo = __shfl_sync(0xffffffffu, v, o);
      if (((okm >> o) & 1u) && (vo > v || (vo == v && o < s))) ++rank;
    }
    if (ok && rank < k) {
      dc_stall_issue e;
      e.node = node;
      e.stall = s;
      e.count = v;
      out[(uint64_t)blockIdx.x * k + rank] = e;
    }
    if (s == 0) n_out[blockIdx.x] = min((uint32_t)__popc(okm), k);
  }
}

dc_status analyze_stalls(Ctx* c, const dc_cct* t, uint32_t metric, uint32_t kind_mask, double hot_threshold,
                         double stall_threshold, uint32_t k, dc_stall_issue* out_h, uint32_t cap, uint32_t* n_out_h) {
  *n_out_h = 0;
  if (t->state != 2) return fail(c, DC_ERR_STATE, "dc_analyze_stalls needs a rolled-up tree (call dc_cct_rollup)");
  if (t->partition) return fail(c, DC_ERR_STATE, "dc_analyze_stalls needs a complete tree (gather the partitions first)");
  if (k > 32) k = 32;
  if (k == 0 || !t->xsamples || t->Nbins == 0) return DC_OK;
  // hotspots (analysis ①), every one above the threshold, in (value desc, id asc) order
  std::vector<dc_topk_entry> hs((size_t)t->N);
  uint32_t nh = 0;
  DC_TRY(hotspots_topk(c, t, DC_VIEW_INCLUSIVE, metric, kind_mask, hot_threshold, (uint32_t)t->N, 0, hs.data(), &nh));
  if (nh == 0) return DC_OK;
  std::vector<uint32_t> hid(nh);
  for (uint32_t i = 0; i < nh; ++i) hid[i] = hs[i].id;
  Buf<uint32_t> dhot, dn;
  Buf<unsigned long long> pc_tot;
  Buf<dc_stall_issue> dout;
  DC_TRY(alloc(c, dhot, nh));
  DC_TRY(alloc(c, dn, nh));
  DC_TRY(alloc_zero(c, pc_tot, t->Npc));
  DC_TRY(alloc(c, dout, (uint64_t)nh * k));
  DC_CUDA(c, cudaMemcpyAsync(dhot.p, hid.data(), nh * 4, cudaMemcpyHostToDevice, c->stream));
  dc_launch(k_stall_issues, nh, ST_THREADS, 0, c->stream, dhot.p, t->N, t->Npc, t->Nbins, t->S, t->pc_ctx, t->bin_pcnode, t->bin_stall,
                                                   t->bin_count, t->isamples, stall_threshold, k, pc_tot.p, dout.p, dn.p);
  DC_LAUNCHED(c);
  std::vector<uint32_t> hn(nh);
  std::vector<dc_stall_issue> ho((size_t)nh * k);
  DC_TRY(readback(c, dn.p, nh * 4, hn.data()));
  DC_TRY(readback(c, dout.p, ho.size() * sizeof(dc_stall_issue), ho.data()));
  uint32_t w = 0, total = 0;
  for (uint32_t i = 0; i < nh; ++i)
    for (uint32_t r = 0; r < hn[i]; ++r, ++total)
      if (w < cap) out_h[w++] = ho[(size_t)i * k + r];
  *n_out_h = total;
  return DC_OK;
}

}  // namespace dc

// ---------------------------------------------------------------- NEXT-3: folded flame-graph stacks
// One line per non-root node with a non-zero exclusive value of the metric (SPEC.md
// export_folded, PAPER.md:444-447 flame graphs): the node's path (frame ids, root excluded,
// outermost first) and its exclusive value, in canonical (breadth-first) node order. Labels are
// the caller's (strings are not part of the device data).
namespace dc {
__global__ void k_fold_flags(const uint64_t* __restrict__ x, const uint16_t* __restrict__ depth, uint64_t N,
                             uint32_t* __restrict__ flag, uint64_t* __restrict__ dep) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x) {
    const bool f = n > 0 && x[n] != 0;
    flag[n] = f ? 1u : 0u;
    dep[n] = f ? depth[n] : 0;
  }
}
__global__ void k_fold_emit(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, const uint64_t* __restrict__ poff,
                            const uint32_t* __restrict__ parent, const uint32_t* __restrict__ frame, const uint16_t* __restrict__ depth,
                            const uint64_t* __restrict__ x, uint64_t N, uint32_t* __restrict__ node_out, uint64_t* __restrict__ val_out,
                            uint64_t* __restrict__ off_out, uint32_t* __restrict__ frames_out) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x) {
    if (!flag[n]) continue;
    const uint32_t i = pos[n];
    const uint64_t o = poff[n];
    node_out[i] = (uint32_t)n;
    val_out[i] = x[n];
    off_out[i] = o;
    uint64_t k = depth[n];
    for (uint32_t a = (uint32_t)n; a != 0 && k > 0; a = parent[a]) frames_out[o + --k] = frame[a];
  }
}
}  // namespace dc

namespace dc {
dc_status export_folded(Ctx* c, const dc_cct* t, uint32_t metric, uint32_t* node_h, uint64_t* value_h, uint64_t* off_h,
                        uint32_t* frames_h, uint64_t cap_lines, uint64_t cap_frames, uint64_t* n_lines_h, uint64_t* n_frames_h) {
  *n_lines_h = *n_frames_h = 0;
  if (t->state == 0) return fail(c, DC_ERR_STATE, "dc_export_folded needs metrics (call dc_cct_attribute_metrics)");
  if (t->partition) return fail(c, DC_ERR_STATE, "dc_export_folded needs a complete tree (gather the partitions first)");
  if (metric >= t->M) return fail(c, DC_ERR_ARG, "metric %u >= M = %u", metric, t->M);
  const uint64_t N = t->N;
  Buf<uint32_t> flag, pos, tot32;
  Buf<uint64_t> dep, poff, tot64;
  DC_TRY(alloc(c, flag, N));
  DC_TRY(alloc(c, pos, N));
  DC_TRY(alloc(c, dep, N));
  DC_TRY(alloc(c, poff, N));
  DC_TRY(alloc(c, tot32, 1));
  DC_TRY(alloc(c, tot64, 1));
  dc_launch(k_fold_flags, grid_for(c, N, 256), 256, 0, c->stream, t->col(C_XSUM, metric), t->depth, N, flag.p, dep.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint32_t>(c, flag.p, pos.p, N, tot32.p));
  DC_TRY(excl_scan<uint64_t>(c, dep.p, poff.p, N, tot64.p));
  uint32_t nl = 0;
  uint64_t nf = 0;
  DC_TRY(readback_multi(c, {{tot32.p, 4, &nl}, {tot64.p, 8, &nf}}));
  *n_lines_h = nl;
  *n_frames_h = nf;
  if (nl > cap_lines || nf > cap_frames) return DC_OK;  // sizes only: the caller retries with room
  Buf<uint32_t> nodes, frames;
  Buf<uint64_t> vals, offs;
  DC_TRY(alloc(c, nodes, nl));
  DC_TRY(alloc(c, vals, nl));
  DC_TRY(alloc(c, offs, nl));
  DC_TRY(alloc(c, frames, nf));
  dc_launch(k_fold_emit, grid_for(c, N, 256), 256, 0, c->stream, flag.p, pos.p, poff.p, t->parent, t->frame, t->depth,
                                                          t->col(C_XSUM, metric), N, nodes.p, vals.p, offs.p, frames.p);
  DC_LAUNCHED(c);
  if (nl) {
    DC_TRY(readback(c, nodes.p, (size_t)nl * 4, node_h));
    DC_TRY(readback(c, vals.p, (size_t)nl * 8, value_h));
    DC_TRY(readback(c, offs.p, (size_t)nl * 8, off_h));
  }
  if (nf) DC_TRY(readback(c, frames.p, (size_t)nf * 4, frames_h));
  return DC_OK;
}

// ---------------------------------------------------------------- NEXT-3: bottom-up caller inversion
// The bottom-up view ("switchable top-down and bottom-up views"): every
// non-root node n with a non-zero exclusive value x(n) contributes x(n) along its call path read
// innermost first (its own frame, then its caller's, ... up to the outermost), so the inverted
// tree's roots are the frames where cost is spent and their children the callers (reading R27).
// In bulk this IS a CCT build: the selected nodes become records whose paths are their reversed
// call paths and whose metric is x(n); dc_cct_build + dc_cct_attribute_metrics + dc_cct_rollup
// then give the inverted tree with canonical ids, inclusive value / count / min / square sum.
__global__ void k_inv_emit(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, const uint64_t* __restrict__ poff,
                           const uint32_t* __restrict__ parent, const uint32_t* __restrict__ frame, const uint16_t* __restrict__ depth,
                           const uint64_t* __restrict__ x, uint64_t N, uint32_t nl, uint64_t nf, uint64_t* __restrict__ off_out,
                           uint64_t* __restrict__ val_out, uint32_t* __restrict__ frames_out) { DC_PDL_ENTER();
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < N; n += (uint64_t)gridDim.x * blockDim.x) {
    if (n == 0) off_out[nl] = nf;
    if (!flag[n]) continue;
    const uint32_t i = pos[n];
    const uint64_t o = poff[n];
    off_out[i] = o;
    val_out[i] = x[n];
    uint64_t k = 0;
    const uint64_t L = depth[n];
    for (uint32_t a = (uint32_t)n; a != 0 && k < L; a = parent[a]) frames_out[o + k++] = frame[a];
  }
}

dc_status cct_build(Ctx* c, const dc_paths* p, const dc_dict* dict, uint32_t n_frames, uint32_t* out_leaf, dc_cct** out);
dc_status attribute_metrics(Ctx* c, dc_cct* t, const uint32_t* leaf, uint64_t R, const uint64_t* X, uint32_t M, uint64_t ld);
dc_status rollup(Ctx* c, dc_cct* t);

dc_status cct_invert(Ctx* c, const dc_cct* t, uint32_t metric, dc_cct** out) {
  *out = nullptr;
  if (t->state == 0) return fail(c, DC_ERR_STATE, "dc_cct_invert needs exclusive values (attribute metrics / samples first)");
  if (t->partition) return fail(c, DC_ERR_STATE, "dc_cct_invert needs a complete tree (gather the partitions first)");
  const uint64_t* x;
  if (metric == DC_METRIC_SAMPLES) {
    if (!t->xsamples) return fail(c, DC_ERR_STATE, "no PC samples attributed");
    x = t->xsamples;
  } else {
    if (metric >= t->M) return fail(c, DC_ERR_ARG, "metric %u >= M = %u", metric, t->M);
    x = t->col(C_XSUM, metric);
  }
  const uint64_t N = t->N;
  Buf<uint32_t> flag, pos, tot32;
  Buf<uint64_t> dep, poff, tot64;
  DC_TRY(alloc(c, flag, N));
  DC_TRY(alloc(c, pos, N));
  DC_TRY(alloc(c, dep, N));
  DC_TRY(alloc(c, poff, N));
  DC_TRY(alloc(c, tot32, 1));
  DC_TRY(alloc(c, tot64, 1));
  dc_launch(k_fold_flags, grid_for(c, N, 256), 256, 0, c->stream, x, t->depth, N, flag.p, dep.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint32_t>(c, flag.p, pos.p, N, tot32.p));
  DC_TRY(excl_scan<uint64_t>(c, dep.p, poff.p, N, tot64.p));
  uint32_t nl = 0;
  uint64_t nf = 0;
  DC_TRY(readback_multi(c, {{tot32.p, 4, &nl}, {tot64.p, 8, &nf}}));
  Buf<uint64_t> off, val;
  Buf<uint32_t> frames, leaf;
  DC_TRY(alloc(c, off, (uint64_t)nl + 1));
  DC_TRY(alloc(c, val, nl));
  DC_TRY(alloc(c, frames, nf));
  DC_TRY(alloc(c, leaf, nl));
  dc_launch(k_inv_emit, grid_for(c, N, 256), 256, 0, c->stream, flag.p, pos.p, poff.p, t->parent, t->frame, t->depth, x, N, nl, nf,
            off.p, val.p, frames.p);
  DC_LAUNCHED(c);
  dc_paths ip{nl, off.p, nf ? frames.p : nullptr};
  dc_dict kinds;  // carries the frame kinds into the inverted tree (views with kind masks)
  kinds.D = t->n_frames;
  kinds.kinds = t->frame_kind;
  dc_cct* inv = nullptr;
  DC_TRY(cct_build(c, &ip, t->frame_kind ? &kinds : nullptr, t->n_frames, leaf.p, &inv));
  HandleGuard<dc_cct, dc_cct_free> guard{inv};
  if (nl) DC_TRY(attribute_metrics(c, inv, leaf.p, nl, val.p, 1, nl));
  else DC_TRY(attribute_metrics(c, inv, nullptr, 0, nullptr, 1, 0));
  DC_TRY(rollup(c, inv));
  guard.h = nullptr;
  *out = inv;
  return DC_OK;
}
}  // namespace dc

// ---------------------------------------------------------------- NEXT-4: CPU-sample intervals
// on each CPU_TIME / REAL_TIME sample the profiler "subtract[s] the previous
// timestamp from it, and use[s] the result as the interval between two samples"; SPEC.md
// attribute_cpu_sample: per (thread, kind), the first sample is the baseline and attributes
// nothing. In bulk: a stable radix sort of the samples by (thread, kind) keeps trace order inside
// each stream, then a segmented adjacent difference, scattered back to trace order.
namespace dc {
__global__ void k_iv_keys(const uint32_t* __restrict__ thread, const uint8_t* __restrict__ kind, uint64_t n,
                          uint64_t* __restrict__ key, uint32_t* __restrict__ val) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    key[i] = (uint64_t)thread[i] << 8 | kind[i];
    val[i] = (uint32_t)i;
  }
}
__global__ void k_iv_diff(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val, const uint64_t* __restrict__ ts,
                          uint64_t n, uint64_t* __restrict__ interval, uint8_t* __restrict__ valid, uint32_t* d_flags) { DC_PDL_ENTER();
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = val[j];
    uint64_t iv = 0;
    uint8_t ok = 0;
    if (j > 0 && key[j - 1] == key[j]) {
      const uint64_t t0 = ts[val[j - 1]], t1 = ts[i];
      if (t1 >= t0) {
        iv = t1 - t0;
        ok = 1;
      } else {
        atomicOr(d_flags, FLAG_BAD_OFFSETS);  // timestamps not monotone within a (thread, kind) stream
      }
    }
    interval[i] = iv;
    valid[i] = ok;
  }
}

dc_status cpu_intervals(Ctx* c, const uint32_t* thread, const uint8_t* kind, const uint64_t* ts, uint64_t n,
                        uint64_t* out_interval, uint8_t* out_valid) {
  if (n == 0) return DC_OK;
  if (n >= (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "dc_cpu_intervals: n >= 2^31 samples");
  Buf<uint64_t> k0, k1;
  Buf<uint32_t> v0, v1;
  DC_TRY(alloc(c, k0, n));
  DC_TRY(alloc(c, k1, n));
  DC_TRY(alloc(c, v0, n));
  DC_TRY(alloc(c, v1, n));
  dc_launch(k_iv_keys, grid_for(c, n, 256), 256, 0, c->stream, thread, kind, n, k0.p, v0.p);
  DC_LAUNCHED(c);
  bool in1 = false;
  DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, n, 0, 40, &in1));
  dc_launch(k_iv_diff, grid_for(c, n, 256), 256, 0, c->stream, in1 ? k1.p : k0.p, in1 ? v1.p : v0.p, ts, n, out_interval, out_valid,
                                                         c->d_flags);
  DC_LAUNCHED(c);
  return DC_OK;
}
}  // namespace dc

// ---------------------------------------------------------------- NEXT-4: forward/backward association
// backward threads lose the Python / framework context; "the backward thread
// looks up the forward CPU thread, fetches the Python and framework call path of the
// corresponding forward operator [same sequence ID], and integrates it with the native call path
// of the backward operator". SPEC.md associate_backward: forward prefix root-ward of the backward
// frames; an unknown sequence id keeps the backward path (and is counted); the registry is a map
// (a later forward entry with the same id replaces an earlier one).
namespace dc {
constexpr uint64_t SQ_EMPTY = ~0ull;
__device__ __forceinline__ uint64_t sq_slot(uint64_t seq, uint64_t mask) { return (mix64(seq) >> 7) & mask; }

__global__ void k_seq_insert(const int64_t* __restrict__ fseq, uint64_t nf, unsigned long long* key, unsigned long long* idx,
                             uint64_t mask, unsigned int* overflow) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nf; i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t s = fseq[i];
    if (s < 0) continue;  // only forward ops carrying a sequence id are registered
    uint64_t q = sq_slot((uint64_t)s, mask);
    bool done = false;
    for (uint64_t p = 0; p <= mask && !done; ++p, q = (q + 1) & mask) {
      const unsigned long long old = atomicCAS(key + q, SQ_EMPTY, (unsigned long long)s);
      if (old == SQ_EMPTY || old == (unsigned long long)s) {
        atomicMax(idx + q, (unsigned long long)i);  // the map keeps the last entry
        done = true;
      }
    }
    if (!done) atomicOr(overflow, 1u);
  }
}

// per backward record: its forward entry (or none) and integrated length
__global__ void k_seq_lookup(const int64_t* __restrict__ bseq, uint64_t nb, const uint64_t* __restrict__ boff,
                             const uint64_t* __restrict__ foff, const unsigned long long* __restrict__ key,
                             const unsigned long long* __restrict__ idx, uint64_t mask, uint64_t* __restrict__ fwd_of,
                             uint64_t* __restrict__ len, unsigned long long* unmatched) { DC_PDL_ENTER();
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nb; r += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t s = bseq[r];
    uint64_t f = SQ_EMPTY;
    if (s >= 0) {
      uint64_t q = sq_slot((uint64_t)s, mask);
      for (uint64_t p = 0; p <= mask; ++p, q = (q + 1) & mask) {
        const unsigned long long k = key[q];
        if (k == (unsigned long long)s) {
          f = idx[q];
          break;
        }
        if (k == SQ_EMPTY) break;
      }
      if (f == SQ_EMPTY) atomicAdd(unmatched, 1ull);
    }
    fwd_of[r] = f;
    len[r] = (f == SQ_EMPTY ? 0 : foff[f + 1] - foff[f]) + (boff[r + 1] - boff[r]);
  }
}

// warp per backward record: forward prefix then the record's own frames
__global__ void k_seq_copy(uint64_t nb, const uint64_t* __restrict__ fwd_of, const uint64_t* __restrict__ foff,
                           const uint32_t* __restrict__ ffr, const uint64_t* __restrict__ boff, const uint32_t* __restrict__ bfr,
                           const uint64_t* __restrict__ ooff, uint32_t* __restrict__ ofr) { DC_PDL_ENTER();
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = warp; r < nb; r += nw) {
    const uint64_t f = fwd_of[r], o = ooff[r];
    uint64_t pl = 0;
    if (f != SQ_EMPTY) {
      const uint64_t a = foff[f];
      pl = foff[f + 1] - a;
      for (uint64_t j = lane; j < pl; j += 32) ofr[o + j] = ffr[a + j];
    }
    const uint64_t b = boff[r], bl = boff[r + 1] - b;
    for (uint64_t j = lane; j < bl; j += 32) ofr[o + pl + j] = bfr[b + j];
  }
}

dc_status seq_associate(Ctx* c, const int64_t* fseq, const uint64_t* foff, const uint32_t* ffr, uint64_t nf, const int64_t* bseq,
                        const uint64_t* boff, const uint32_t* bfr, uint64_t nb, uint64_t* out_off, uint32_t* out_frames,
                        uint64_t cap_frames, uint64_t* n_frames_h, uint64_t* n_unmatched_h) {
  *n_frames_h = 0;
  *n_unmatched_h = 0;
  if (nb == 0) {
    DC_CUDA(c, cudaMemsetAsync(out_off, 0, 8, c->stream));
    return DC_OK;
  }
  uint64_t cap = 1024;
  while (cap < 2 * nf) cap <<= 1;
  Buf<unsigned long long> key, idx, unm;
  Buf<unsigned int> ovf;
  Buf<uint64_t> fwd_of, len;
  DC_TRY(alloc(c, key, cap));
  DC_TRY(alloc_zero(c, idx, cap));
  DC_TRY(alloc_zero(c, unm, 1));
  DC_TRY(alloc_zero(c, ovf, 1));
  DC_TRY(alloc(c, fwd_of, nb));
  DC_TRY(alloc(c, len, nb));
  DC_CUDA(c, cudaMemsetAsync(key.p, 0xFF, cap * 8, c->stream));
  if (nf) {
    dc_launch(k_seq_insert, grid_for(c, nf, 256), 256, 0, c->stream, fseq, nf, key.p, idx.p, cap - 1, ovf.p);
    DC_LAUNCHED(c);
  }
  dc_launch(k_seq_lookup, grid_for(c, nb, 256), 256, 0, c->stream, bseq, nb, boff, foff, key.p, idx.p, cap - 1, fwd_of.p, len.p, unm.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint64_t>(c, len.p, out_off, nb, out_off + nb));
  uint64_t tot = 0, un = 0;
  uint32_t of = 0;
  DC_TRY(readback_multi(c, {{out_off + nb, 8, &tot}, {unm.p, 8, &un}, {ovf.p, 4, &of}}));
  if (of) return fail(c, DC_ERR_CAPACITY, "dc_seq_associate: registry table overflow");
  *n_frames_h = tot;
  *n_unmatched_h = un;
  if (tot > cap_frames) return DC_OK;  // offsets only: the caller retries with room
  dc_launch(k_seq_copy, grid_for(c, nb * 32, 256), 256, 0, c->stream, nb, fwd_of.p, foff, ffr, boff, bfr, out_off, out_frames);
  DC_LAUNCHED(c);
  return DC_OK;
}
}  // namespace dc
