// pc.cu — a6: PC-sampling attribution ("extend the call path by inserting the
// PC of each instruction collected"; stall reasons PAPER.md:414-416).
//
// Output: PC nodes = distinct (ctx, pc_off), ids N + rank in (ctx, pc_off) order; bins
// (pc node, stall, count) sorted; per-ctx exclusive samples / stall[s] columns.
//
// Generic schedule (any sample order): every valid sample updates its (ctx, pc, stall) bin
// in an L2-resident open-addressing table (16-B keys, u64 counts, read-first probing). The
// distinct bins are then compacted, radix-sorted into canonical order and run-length
// encoded into PC nodes. The context-owner schedule (pc_owner.cu) replaces the table pass
// when per-launch sample offsets are given.
#include <algorithm>

#include "prim.cuh"

namespace dc {

dc_status pc_owner_hist(Ctx* c, dc_cct* t, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf,
                        uint64_t n_launch, const uint64_t* launch_off, uint32_t S, FillList& fl, uint64_t* n_bins_out,
                        int* handled);

__device__ __forceinline__ void block_diag_add(unsigned long long* d_diag, uint32_t bad_l, uint32_t bad_s, uint32_t zero) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad_l += __shfl_xor_sync(0xffffffffu, bad_l, o);
    bad_s += __shfl_xor_sync(0xffffffffu, bad_s, o);
    zero += __shfl_xor_sync(0xffffffffu, zero, o);
  }
  if (lane_id() == 0) {
    if (bad_l) atomicAdd(d_diag + DG_BAD_LAUNCH, (unsigned long long)bad_l);
    if (bad_s) atomicAdd(d_diag + DG_BAD_STALL, (unsigned long long)bad_s);
    if (zero) atomicAdd(d_diag + DG_ZERO, (unsigned long long)zero);
  }
}

// key layout in the table: x = (ctx << 32) | pc_off, y = stall; EMPTY = all ones
__global__ void k_pc_table(const dc_pc_sample* __restrict__ smp, uint64_t n, const uint32_t* __restrict__ launch_leaf,
                           uint64_t n_launch, uint32_t S, uint64_t N, ulonglong2* table, unsigned long long* tcnt,
                           uint64_t mask, unsigned int* d_distinct, unsigned int* d_overflow, unsigned long long* d_diag,
                           uint32_t* d_flags) { DC_PDL_ENTER();
  uint32_t bad_l = 0, bad_s = 0, zero = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(smp) + j);  // {launch, pc_off, stall|flags<<16, count}
    const uint32_t launch = q.x, pc = q.y, stall = q.z & 0xFFFFu, count = q.w;
    if (launch >= n_launch) { ++bad_l; continue; }
    if (stall >= S) { ++bad_s; continue; }
    if (count == 0) { ++zero; continue; }
    const uint32_t ctx = __ldg(launch_leaf + launch);
    if (ctx >= N) { atomicOr(d_flags, FLAG_BAD_LEAF); continue; }
    const uint64_t kx = ((uint64_t)ctx << 32) | pc, ky = stall;
    uint64_t s = mix64(kx * 0x9E3779B97F4A7C15ull + ky) & mask;
    bool done = false;
    // a probe run this long means the table is (nearly) full: report overflow (the host retries
    // with a table sized by the distinct bins) instead of walking the whole table per sample
    const uint64_t max_probe = mask < 4096 ? mask : 4096;
    for (uint64_t probe = 0; probe <= max_probe; ++probe, s = (s + 1) & mask) {
      ulonglong2 cur = ld_relaxed_v2(table + s);
      if (cur.x == kx && cur.y == ky) { done = true; break; }
      if (cur.x != ~0ull && cur.y != ~0ull) continue;
      unsigned __int128 expect = ~(unsigned __int128)0;
      unsigned __int128 want = ((unsigned __int128)ky << 64) | kx;
      unsigned __int128 old = atomicCAS(reinterpret_cast<unsigned __int128*>(table + s), expect, want);
      if (old == expect) { atomicAdd(d_distinct, 1u); done = true; break; }
      if (old == want) { done = true; break; }
    }
    if (!done) { atomicOr(d_overflow, 1u); continue; }
    atomicAdd(tcnt + s, (unsigned long long)count);
  }
  block_diag_add(d_diag, bad_l, bad_s, zero);
}

// compact the table into (sort key, count) with key = ((ctx << pcb | pc) << 5) | stall
__global__ void k_pc_compact(const ulonglong2* __restrict__ table, const unsigned long long* __restrict__ tcnt, uint64_t cap,
                             int pcb, uint64_t* __restrict__ keys, uint64_t* __restrict__ cnts, unsigned int* d_pos) { DC_PDL_ENTER();
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    ulonglong2 cur = table[s];
    if (cur.x == ~0ull) continue;
    unsigned p = atomicAdd(d_pos, 1u);
    uint64_t ctx = cur.x >> 32, pc = cur.x & 0xFFFFFFFFull;
    keys[p] = (((ctx << pcb) | pc) << 5) | cur.y;
    cnts[p] = tcnt[s];
  }
}

__global__ void k_pc_maxpc(const ulonglong2* __restrict__ table, uint64_t cap, unsigned int* d_max) { DC_PDL_ENTER();
  uint32_t m = 0;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    ulonglong2 cur = table[s];
    if (cur.x != ~0ull) m = max(m, (uint32_t)cur.x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(d_max, m);
}

__global__ void k_iota32(uint32_t* a, uint64_t n) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] = (uint32_t)i;
}

// heads of (ctx, pc) runs among sorted bins
__global__ void k_pc_heads(const uint64_t* __restrict__ keys, uint64_t nb, uint32_t* __restrict__ head) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (keys[i - 1] >> 5) != (keys[i] >> 5)) ? 1u : 0u;
}

__global__ void k_pc_emit(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ order, const uint64_t* __restrict__ cnts,
                          uint64_t nb, int pcb, const uint32_t* __restrict__ head, const uint32_t* __restrict__ run_excl,
                          uint64_t N, uint64_t S, uint32_t* __restrict__ pc_ctx, uint32_t* __restrict__ pc_off,
                          uint32_t* __restrict__ bin_pcnode, uint16_t* __restrict__ bin_stall, uint64_t* __restrict__ bin_count,
                          unsigned long long* __restrict__ xsamples, unsigned long long* __restrict__ xstall) { DC_PDL_ENTER();
  const uint64_t pcmask = (1ull << pcb) - 1ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    uint32_t stall = (uint32_t)(k & 31u);
    uint64_t cp = k >> 5;
    uint32_t ctx = (uint32_t)(cp >> pcb), pc = (uint32_t)(cp & pcmask);
    uint32_t pidx = run_excl[i] + head[i] - 1u;
    if (head[i]) {
      pc_ctx[pidx] = ctx;
      pc_off[pidx] = pc;
    }
    uint64_t cnt = cnts[order ? order[i] : i];
    bin_pcnode[i] = (uint32_t)(N + pidx);
    bin_stall[i] = (uint16_t)stall;
    bin_count[i] = cnt;
    atomicAdd(xsamples + ctx, (unsigned long long)cnt);
    atomicAdd(xstall + (uint64_t)stall * N + ctx, (unsigned long long)cnt);
  }
}

static uint64_t np2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

// ---------------------------------------------------------------- repeated calls (chunks)
// A later call's bins and PC nodes are merged exactly with the earlier ones: both bin lists are
// in canonical (ctx, pc, stall) order with unique keys, so after one sort of their union an
// equal key occurs at most twice (adjacent); the first of a run emits the bin with both counts.
__global__ void k_pc_binkeys(const uint32_t* __restrict__ pc_ctx, const uint32_t* __restrict__ pc_off,
                             const uint32_t* __restrict__ bin_pcnode, const uint16_t* __restrict__ bin_stall,
                             const uint64_t* __restrict__ bin_count, uint64_t nb, uint64_t N, int pcb,
                             uint64_t* __restrict__ keys, uint64_t* __restrict__ cnts) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = bin_pcnode[i] - N;
    keys[i] = ((((uint64_t)pc_ctx[p] << pcb) | pc_off[p]) << 5) | bin_stall[i];
    cnts[i] = bin_count[i];
  }
}

__global__ void k_pc_maxoff(const uint32_t* __restrict__ a, uint64_t n, unsigned int* d_max) { DC_PDL_ENTER();
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) m = max(m, a[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(d_max, m);
}

// hb = first of an equal-key run (a bin), hp = first bin of a (ctx, pc) run (a PC node)
__global__ void k_pc_mheads(const uint64_t* __restrict__ k, uint64_t nb, uint32_t* __restrict__ hb, uint32_t* __restrict__ hp) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x) {
    const bool b = i == 0 || k[i - 1] != k[i];
    hb[i] = b;
    hp[i] = b && (i == 0 || (k[i - 1] >> 5) != (k[i] >> 5));
  }
}

__global__ void k_pc_memit(const uint64_t* __restrict__ k, const uint32_t* __restrict__ ord, const uint64_t* __restrict__ cnts,
                           uint64_t nb, int pcb, const uint32_t* __restrict__ hb, const uint32_t* __restrict__ hp,
                           const uint32_t* __restrict__ bidx, const uint32_t* __restrict__ pidx, uint64_t N,
                           uint32_t* __restrict__ pc_ctx, uint32_t* __restrict__ pc_off, uint32_t* __restrict__ bin_pcnode,
                           uint16_t* __restrict__ bin_stall, uint64_t* __restrict__ bin_count) { DC_PDL_ENTER();
  const uint64_t pcmask = (1ull << pcb) - 1ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!hb[i]) continue;
    const uint64_t key = k[i], cp = key >> 5;
    const uint32_t p = pidx[i] + hp[i] - 1u, b = bidx[i];
    if (hp[i]) {
      pc_ctx[p] = (uint32_t)(cp >> pcb);
      pc_off[p] = (uint32_t)(cp & pcmask);
    }
    uint64_t cnt = cnts[ord[i]];
    if (i + 1 < nb && k[i + 1] == key) cnt += cnts[ord[i + 1]];
    bin_pcnode[b] = (uint32_t)(N + p);
    bin_stall[b] = (uint16_t)(key & 31u);
    bin_count[b] = cnt;
  }
}

__global__ void k_add_u64(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src, uint64_t n) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) dst[i] += src[i];
}

struct PcPrev {  // the tree's PC results before a repeated call
  uint64_t *xsamples = nullptr, *xstall = nullptr, *bin_count = nullptr;
  uint32_t *pc_ctx = nullptr, *pc_off = nullptr, *bin_pcnode = nullptr;
  uint16_t* bin_stall = nullptr;
  uint64_t Npc = 0, Nbins = 0;
};

static dc_status pc_merge_prev(Ctx* c, dc_cct* t, const PcPrev& o) {
  const uint64_t N = t->N, S = t->S;
  dc_launch(k_add_u64, grid_for(c, N, 256), 256, 0, c->stream, t->xsamples, o.xsamples, N);
  DC_LAUNCHED(c);
  dc_launch(k_add_u64, grid_for(c, S * N, 256), 256, 0, c->stream, t->xstall, o.xstall, S * N);
  DC_LAUNCHED(c);
  const uint64_t na = o.Nbins, nbn = t->Nbins, nb = na + nbn;
  if (nb >= (1ull << 32)) return fail(c, DC_ERR_CAPACITY, "more than 2^32 PC bins");
  Buf<unsigned int> mx;
  DC_TRY(alloc_zero(c, mx, 1));
  if (o.Npc) {
    dc_launch(k_pc_maxoff, grid_for(c, o.Npc, 256), 256, 0, c->stream, o.pc_off, o.Npc, mx.p);
    DC_LAUNCHED(c);
  }
  if (t->Npc) {
    dc_launch(k_pc_maxoff, grid_for(c, t->Npc, 256), 256, 0, c->stream, t->pc_off, t->Npc, mx.p);
    DC_LAUNCHED(c);
  }
  uint32_t hmax = 0;
  DC_TRY(readback(c, mx.p, 4, &hmax));
  int pcb = bits_for(hmax);
  if (pcb == 0) pcb = 1;
  const int kbits = bits_for(N > 1 ? N - 1 : 1) + pcb + 5;
  if (kbits > 64) return fail(c, DC_ERR_CAPACITY, "PC bin sort key exceeds 64 bits");
  Buf<uint64_t> k0, k1, cnts;
  Buf<uint32_t> v0, v1, hb, hp, bidx, pidx, tot;
  DC_TRY(alloc(c, k0, nb));
  DC_TRY(alloc(c, k1, nb));
  DC_TRY(alloc(c, cnts, nb));
  DC_TRY(alloc(c, v0, nb));
  DC_TRY(alloc(c, v1, nb));
  if (na) {
    dc_launch(k_pc_binkeys, grid_for(c, na, 256), 256, 0, c->stream, o.pc_ctx, o.pc_off, o.bin_pcnode, o.bin_stall, o.bin_count, na,
              N, pcb, k0.p, cnts.p);
    DC_LAUNCHED(c);
  }
  if (nbn) {
    dc_launch(k_pc_binkeys, grid_for(c, nbn, 256), 256, 0, c->stream, t->pc_ctx, t->pc_off, t->bin_pcnode, t->bin_stall,
              t->bin_count, nbn, N, pcb, k0.p + na, cnts.p + na);
    DC_LAUNCHED(c);
  }
  dc_launch(k_iota32, grid_for(c, nb, 256), 256, 0, c->stream, v0.p, nb);
  DC_LAUNCHED(c);
  bool in1 = false;
  DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, nb, 0, kbits, &in1));
  const uint64_t* sk = in1 ? k1.p : k0.p;
  const uint32_t* so = in1 ? v1.p : v0.p;
  DC_TRY(alloc(c, hb, nb));
  DC_TRY(alloc(c, hp, nb));
  DC_TRY(alloc(c, bidx, nb));
  DC_TRY(alloc(c, pidx, nb));
  DC_TRY(alloc_zero(c, tot, 2));
  if (nb) {
    dc_launch(k_pc_mheads, grid_for(c, nb, 256), 256, 0, c->stream, sk, nb, hb.p, hp.p);
    DC_LAUNCHED(c);
    DC_TRY((excl_scan_pair<uint32_t, uint32_t>(c, hb.p, bidx.p, tot.p, hp.p, pidx.p, tot.p + 1, nb)));
  }
  uint32_t ht[2] = {0, 0};
  DC_TRY(readback(c, tot.p, 8, ht));
  void* stale[] = {t->pc_ctx, t->pc_off, t->bin_pcnode, t->bin_stall, t->bin_count};
  t->pc_ctx = t->pc_off = t->bin_pcnode = nullptr;
  t->bin_stall = nullptr;
  t->bin_count = nullptr;
  for (void* q : stale) cudaFreeAsync(q, c->stream);
  t->Nbins = ht[0];
  t->Npc = ht[1];
  DC_TRY(palloc(c, t->pc_ctx, t->Npc));
  DC_TRY(palloc(c, t->pc_off, t->Npc));
  DC_TRY(palloc(c, t->bin_pcnode, t->Nbins));
  DC_TRY(palloc(c, t->bin_stall, t->Nbins));
  DC_TRY(palloc(c, t->bin_count, t->Nbins));
  if (nb) {
    dc_launch(k_pc_memit, grid_for(c, nb, 256), 256, 0, c->stream, sk, so, cnts.p, nb, pcb, hb.p, hp.p, bidx.p, pidx.p, N, t->pc_ctx,
              t->pc_off, t->bin_pcnode, t->bin_stall, t->bin_count);
    DC_LAUNCHED(c);
  }
  return DC_OK;
}

static dc_status pc_attribute_once(Ctx* c, dc_cct* t, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf,
                                   uint64_t n_launch, const uint64_t* launch_off, uint32_t S, FillList& fl);

dc_status pc_attribute(Ctx* c, dc_cct* t, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf, uint64_t n_launch,
                       const uint64_t* launch_off, uint32_t S) {
  const uint64_t N = t->N;
  if (!t->pc_done) {  // first call: the tree's sample columns, zeroed
    t->S = S;
    DC_TRY(palloc(c, t->xsamples, N));
    DC_TRY(palloc(c, t->isamples, N));
    DC_TRY(palloc(c, t->xstall, (uint64_t)S * N));
    DC_TRY(palloc(c, t->istall, (uint64_t)S * N));
    // (the inclusive columns are written whole by dc_cct_rollup and unreadable before it)
    FillList fl;
    DC_TRY(fill_add(c, fl, t->xsamples, N * 8));
    DC_TRY(fill_add(c, fl, t->xstall, (uint64_t)S * N * 8));
    return pc_attribute_once(c, t, s, n, launch_leaf, n_launch, launch_off, S, fl);
  }
  // a later call (e.g. the next chunk of samples, "flushes the metrics" per
  // buffer): this call's bins and exclusive columns are computed on their own, then merged
  PcPrev o;
  o.xsamples = t->xsamples;
  o.xstall = t->xstall;
  o.pc_ctx = t->pc_ctx;
  o.pc_off = t->pc_off;
  o.bin_pcnode = t->bin_pcnode;
  o.bin_stall = t->bin_stall;
  o.bin_count = t->bin_count;
  o.Npc = t->Npc;
  o.Nbins = t->Nbins;
  t->xsamples = t->xstall = t->bin_count = nullptr;
  t->pc_ctx = t->pc_off = t->bin_pcnode = nullptr;
  t->bin_stall = nullptr;
  t->Npc = t->Nbins = 0;
  dc_status st = palloc(c, t->xsamples, N);
  if (st == DC_OK) st = palloc(c, t->xstall, (uint64_t)S * N);
  FillList fl;
  if (st == DC_OK) st = fill_add(c, fl, t->xsamples, N * 8);
  if (st == DC_OK) st = fill_add(c, fl, t->xstall, (uint64_t)S * N * 8);
  if (st == DC_OK) st = pc_attribute_once(c, t, s, n, launch_leaf, n_launch, launch_off, S, fl);
  if (st == DC_OK) st = pc_merge_prev(c, t, o);
  if (st != DC_OK) {  // keep the earlier results: the handle stays valid, this call had no effect
    void* cur[] = {t->xsamples, t->xstall, t->pc_ctx, t->pc_off, t->bin_pcnode, t->bin_stall, t->bin_count};
    for (void* q : cur) if (q) cudaFreeAsync(q, c->stream);
    t->xsamples = o.xsamples;
    t->xstall = o.xstall;
    t->pc_ctx = o.pc_ctx;
    t->pc_off = o.pc_off;
    t->bin_pcnode = o.bin_pcnode;
    t->bin_stall = o.bin_stall;
    t->bin_count = o.bin_count;
    t->Npc = o.Npc;
    t->Nbins = o.Nbins;
    return st;
  }
  void* prev[] = {o.xsamples, o.xstall, o.pc_ctx, o.pc_off, o.bin_pcnode, o.bin_stall, o.bin_count};
  for (void* q : prev) if (q) cudaFreeAsync(q, c->stream);
  t->state = 1;
  return DC_OK;
}

// -------- launch partition (round 2): samples in any order, no per-launch offsets. When the
// launches are few enough for a per-CTA shared-memory histogram, the samples are first
// partitioned by launch (a counting sort: per-CTA histograms, one scan in launch-major order,
// a scatter through shared cursors; the order inside a launch is irrelevant to the bins) and
// the context-owner schedule runs on the partitioned copy with the offsets the scan gives —
// three passes over the samples instead of one L2-atomic table update per sample. Samples whose
// launch is out of range go to a last bucket and are counted as DG_BAD_LAUNCH, as in k_pc_table.
constexpr uint64_t LP_MAX = 49152;  // launches (+1 bucket) in a CTA's shared-memory histogram
constexpr int LP_THREADS = 1024;
__global__ void __launch_bounds__(LP_THREADS) k_lp_count(const dc_pc_sample* __restrict__ smp, uint64_t n, uint32_t n_launch,
                                                         uint32_t* __restrict__ gh) { DC_PDL_ENTER();
  extern __shared__ uint32_t lh[];
  const uint32_t G = gridDim.x, b = blockIdx.x;
  for (uint32_t l = threadIdx.x; l <= n_launch; l += LP_THREADS) lh[l] = 0;
  __syncthreads();
  const uint64_t lo = n * b / G, hi = n * (b + 1) / G;
  const uint32_t* lf = reinterpret_cast<const uint32_t*>(smp);  // launch = word 0 of each 16-B sample
  for (uint64_t j = lo + threadIdx.x; j < hi; j += LP_THREADS) {
    const uint32_t l = __ldg(lf + 4 * j);
    atomicAdd(&lh[l < n_launch ? l : n_launch], 1u);
  }
  __syncthreads();
  for (uint32_t l = threadIdx.x; l <= n_launch; l += LP_THREADS) gh[(uint64_t)l * G + b] = lh[l];  // launch-major
}
__global__ void k_lp_offsets(const uint32_t* __restrict__ gh, uint32_t n_launch, uint32_t G, uint64_t n,
                             uint64_t* __restrict__ loff, unsigned long long* __restrict__ ldiag) { DC_PDL_ENTER();
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l <= n_launch; l += gridDim.x * blockDim.x) {
    loff[l] = gh[(uint64_t)l * G];
    if (l == n_launch) ldiag[DG_BAD_LAUNCH] = n - gh[(uint64_t)l * G];
  }
}
__global__ void __launch_bounds__(LP_THREADS) k_lp_scatter(const dc_pc_sample* __restrict__ smp, uint64_t n, uint32_t n_launch,
                                                           const uint32_t* __restrict__ gh, uint4* __restrict__ out) { DC_PDL_ENTER();
  extern __shared__ uint32_t cur[];
  const uint32_t G = gridDim.x, b = blockIdx.x;
  for (uint32_t l = threadIdx.x; l <= n_launch; l += LP_THREADS) cur[l] = gh[(uint64_t)l * G + b];
  __syncthreads();
  const uint64_t lo = n * b / G, hi = n * (b + 1) / G;
  const uint4* q = reinterpret_cast<const uint4*>(smp);
  for (uint64_t j = lo + threadIdx.x; j < hi; j += LP_THREADS) {
    const uint4 v = __ldg(q + j);
    const uint32_t pos = atomicAdd(&cur[v.x < n_launch ? v.x : n_launch], 1u);
    out[pos] = v;
  }
}

static dc_status pc_attribute_once(Ctx* c, dc_cct* t, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf,
                                   uint64_t n_launch, const uint64_t* launch_off, uint32_t S, FillList& fl) {
  const uint64_t N = t->N;
  // -------- histogram into (sort key, count) pairs
  Buf<uint64_t> keys, cnts, keys2;
  uint64_t nb = 0;
  int pcb = 32;
  int handled = 0;
  Buf<ulonglong2> table;
  Buf<unsigned long long> tcnt;
  if (launch_off) {
    // context-owner schedule (pc_owner.cu); handled == 0 means "not applicable, use generic"
    DC_TRY(pc_owner_hist(c, t, s, n, launch_leaf, n_launch, launch_off, S, fl, &nb, &handled));
    if (handled) {
      t->pc_done = true;
      t->state = 1;
      c->bytes_host += 16 * n + 16 * nb + 8 * t->Npc;
      return DC_OK;
    }
  } else if (n && n_launch && n_launch <= LP_MAX && n < (1ull << 32) && !getenv("DC_TEST_PC_GENERIC")) {
    // launch partition, then the context-owner schedule on the partitioned copy
    const uint32_t G = (uint32_t)c->num_sms * 2;
    const size_t lsm = ((size_t)n_launch + 1) * 4;
    Buf<uint32_t> gh;
    Buf<uint64_t> loff;
    Buf<uint4> part;
    Buf<unsigned long long> pdiag;
    DC_TRY(alloc(c, gh, ((uint64_t)n_launch + 1) * G));
    DC_TRY(alloc(c, loff, (uint64_t)n_launch + 1));
    DC_TRY(alloc(c, part, n));
    DC_TRY(alloc_zero(c, pdiag, DG_N));
    {
      Region rk(c, "pc:partition");
      DC_SMEM_OPTIN(c, k_lp_count);
      DC_SMEM_OPTIN(c, k_lp_scatter);
      dc_launch(k_lp_count, G, LP_THREADS, lsm, c->stream, s, n, (uint32_t)n_launch, gh.p);
      DC_LAUNCHED(c);
      DC_TRY(excl_scan<uint32_t>(c, gh.p, gh.p, ((uint64_t)n_launch + 1) * G, nullptr));
      dc_launch(k_lp_offsets, grid_for(c, n_launch + 1, 256), 256, 0, c->stream, gh.p, (uint32_t)n_launch, G, n, loff.p, pdiag.p);
      DC_LAUNCHED(c);
      dc_launch(k_lp_scatter, G, LP_THREADS, lsm, c->stream, s, n, (uint32_t)n_launch, gh.p, part.p);
      DC_LAUNCHED(c);
    }
    uint64_t n_valid = 0;
    DC_TRY(readback(c, loff.p + n_launch, 8, &n_valid));
    DC_TRY(pc_owner_hist(c, t, reinterpret_cast<const dc_pc_sample*>(part.p), n_valid, launch_leaf, n_launch, loff.p, S, fl, &nb,
                         &handled));
    if (handled) {
      DC_TRY(add_diag(c, pdiag.p));  // out-of-range launches (counted once: the generic path did not run)
      t->pc_done = true;
      t->state = 1;
      c->bytes_host += 3 * 16 * n + 16 * nb + 8 * t->Npc;
      return DC_OK;
    }
  }
  DC_TRY(fill_flush(c, fl));  // pending column fills (the owner schedule did not run / flush them)
  if (!handled) {
    // table sized for twice the bins of the last generic call (or 2 x min(n, 4M)); an overflow
    // (distinct bins past half load, or a probe run past 4,096) retries with 4x the slots
    uint64_t guess = c->pc_generic_hint ? c->pc_generic_hint : (n < (1ull << 22) ? n : (1ull << 22));
    if (guess > n) guess = n;
    uint64_t cap = np2(2 * guess);
    if (cap < 1024) cap = 1024;
    Buf<unsigned int> ctr;
    Buf<unsigned long long> ldiag;  // this call's diag counts (a retry recounts every sample)
    for (int attempt = 0;; ++attempt) {
      FillList f2;
      DC_TRY(alloc_fill(c, f2, table, cap, 0xFF));
      DC_TRY(alloc_fill(c, f2, tcnt, cap));
      DC_TRY(alloc_fill(c, f2, ctr, 4));
      DC_TRY(alloc_fill(c, f2, ldiag, DG_N));
      DC_TRY(fill_flush(c, f2));
      {
        Region rk(c, "k:pc_table");
        dc_launch(k_pc_table, grid_for(c, n, 256, 16), 256, 0, c->stream, s, n, launch_leaf, n_launch, S, N, table.p, tcnt.p,
                                                                    cap - 1, ctr.p, ctr.p + 1, ldiag.p, c->d_flags);
      DC_LAUNCHED(c);
      }
      uint32_t h[2];
      DC_TRY(readback(c, ctr.p, 8, h));
      if (!h[1] && (uint64_t)h[0] * 2 <= cap) {
        nb = h[0];
        c->pc_generic_hint = nb;
        break;
      }
      if (attempt == 4 || cap >= (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "PC bin table overflow (%u distinct bins)", h[0]);
      cap = std::max<uint64_t>(4 * cap, np2(4 * (uint64_t)h[0]));
      if (cap > (1ull << 31)) cap = 1ull << 31;
    }
    DC_TRY(add_diag(c, ldiag.p));
    Buf<unsigned int> mx;
    DC_TRY(alloc_zero(c, mx, 2));
    dc_launch(k_pc_maxpc, grid_for(c, cap, 256), 256, 0, c->stream, table.p, cap, mx.p);
    DC_LAUNCHED(c);
    uint32_t hm[2];
    DC_TRY(readback(c, mx.p, 8, hm));
    pcb = bits_for(hm[0]);
    if (pcb == 0) pcb = 1;
    if (bits_for(N > 1 ? N - 1 : 1) + pcb + 5 > 64)
      return fail(c, DC_ERR_CAPACITY, "PC bin sort key exceeds 64 bits");
    DC_TRY(alloc(c, keys, nb));
    DC_TRY(alloc(c, cnts, nb));
    dc_launch(k_pc_compact, grid_for(c, cap, 256), 256, 0, c->stream, table.p, tcnt.p, cap, pcb, keys.p, cnts.p, mx.p + 1);
    DC_LAUNCHED(c);
    table.release();
    tcnt.release();
  } else {
    return fail(c, DC_ERR_STATE, "internal: context-owner output not wired");
  }
  // -------- canonical order: sort bins by (ctx, pc, stall)
  Buf<uint32_t> ord0, ord1, head, runs;
  DC_TRY(alloc(c, keys2, nb));
  DC_TRY(alloc(c, ord0, nb));
  DC_TRY(alloc(c, ord1, nb));
  dc_launch(k_iota32, grid_for(c, nb, 256), 256, 0, c->stream, ord0.p, nb);
  DC_LAUNCHED(c);
  bool in1 = false;
  const int kbits = bits_for(N > 1 ? N - 1 : 1) + pcb + 5;
  DC_TRY(radix_sort_pairs(c, keys.p, ord0.p, keys2.p, ord1.p, nb, 0, kbits, &in1));
  uint64_t* sk = in1 ? keys2.p : keys.p;
  uint32_t* so = in1 ? ord1.p : ord0.p;
  DC_TRY(alloc(c, head, nb));
  DC_TRY(alloc(c, runs, nb));
  dc_launch(k_pc_heads, grid_for(c, nb, 256), 256, 0, c->stream, sk, nb, head.p);
  DC_LAUNCHED(c);
  Buf<uint32_t> npc;
  DC_TRY(alloc(c, npc, 1));
  DC_TRY(excl_scan<uint32_t>(c, head.p, runs.p, nb, npc.p));
  uint32_t hnpc = 0;
  DC_TRY(readback(c, npc.p, 4, &hnpc));
  t->Npc = hnpc;
  t->Nbins = nb;
  DC_TRY(palloc(c, t->pc_ctx, hnpc));
  DC_TRY(palloc(c, t->pc_off, hnpc));
  DC_TRY(palloc(c, t->bin_pcnode, nb));
  DC_TRY(palloc(c, t->bin_stall, nb));
  DC_TRY(palloc(c, t->bin_count, nb));
  if (nb) {
    dc_launch(k_pc_emit, grid_for(c, nb, 256), 256, 0, c->stream, sk, so, cnts.p, nb, pcb, head.p, runs.p, N, S, t->pc_ctx,
                                                           t->pc_off, t->bin_pcnode, t->bin_stall, t->bin_count,
                                                           (unsigned long long*)t->xsamples, (unsigned long long*)t->xstall);
    DC_LAUNCHED(c);
  }
  t->pc_done = true;
  t->state = 1;
  c->bytes_host += 16 * n + 16 * nb + 8 * hnpc;
  return DC_OK;
}

}  // namespace dc
