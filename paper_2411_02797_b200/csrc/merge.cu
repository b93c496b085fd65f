// merge.cu — a9: cross-rank merge of per-rank CCTs (north_star; not in the paper).
//
// Merged CCT == CCT of the concatenation of every rank's records (reading R19): inclusive
// and exclusive aggregates are additive (and min-combinable) across disjoint record shards,
// so nodes with equal full paths are simply combined.
//   1. dictionary unify: all-gather the per-rank sorted dictionaries; every rank interns the
//      union (same kernels as dc_intern_frames) -> identical global ranks; local -> global map.
//   2. 128-bit full-path hash per node, level by level: h(root) = H0, h(n) = mix(h(parent), gframe).
//   3. partition: owner(n) = floor(h_hi * P / 2^64); counting-sort node records into per-owner
//      slabs (PC bins travel as (h_ctx, pc, stall, count), owner from (h_ctx, pc)).
//   4. exchange: NCCL all-to-all of counts, grouped ncclSend/ncclRecv of the slabs (NVLink).
//   5. reduce: sort received records by h, combine runs (+ / min), and VERIFY that every run
//      agrees on (parent hash, global frame, depth): by induction from the fixed root hash a
//      hash collision between different paths always shows up as such a mismatch
//      (DC_ERR_COLLISION), so the merge is exact or fails loudly.
//   6. (parity / views) gather: partitions to a root rank, canonicalised level by level into
//      the (depth, lexicographic) node order — the same canonical CCT the single-GPU build gives.
// dc_cct_merge_local runs steps 1-6 for P logical ranks on ONE GPU with a loopback exchange
// (device copies instead of NCCL) — the emulated-rank test path.
#include <memory>
#include <vector>

#include "prim.cuh"
#if DC_HAVE_NCCL
#include <nccl.h>
#endif

namespace dc {
dc_status intern_frames(Ctx* c, const dc_frame_key* keys, uint64_t n, uint32_t* out_ids, dc_dict** out, uint64_t d_hint = 0);
dc_status ensure_metric_cols(Ctx* c, dc_cct* t, uint32_t M);

// record layout, in u64 words
//  0 h_lo  1 h_hi  2 hp_lo  3 hp_hi  4 gframe | depth << 32  5 xcnt  6 icnt
//  7 + 8m .. : xsum xmin xsqlo xsqhi isum imin isqlo isqhi     (m < M)
//  7 + 8M    : xsamples isamples, then per stall s: xstall istall (when the tree has PC data)
struct RecFmt {
  uint32_t M, S, has_pc, W;
};
static RecFmt rec_fmt(uint32_t M, uint32_t S, bool has_pc) {
  RecFmt f{M, S, has_pc ? 1u : 0u, 0};
  f.W = 7 + 8 * M + (has_pc ? 2 + 2 * S : 0);
  return f;
}
constexpr int BIN_W = 4;  // h_lo, h_hi, pc | stall << 32, count

__device__ __forceinline__ void mix128(uint64_t& lo, uint64_t& hi, uint32_t f) {
  uint64_t a = mix64(lo ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull) ^ 0x243F6A8885A308D3ull);
  uint64_t b = mix64(hi + ((uint64_t)f << 17) + lo * 0xC2B2AE3D27D4EB4Full + 0x13198A2E03707344ull);
  lo = a;
  hi = b ^ (a >> 7);
}
constexpr uint64_t H0_LO = 0x6A09E667F3BCC908ull, H0_HI = 0xBB67AE8584CAA73Bull;

__global__ void k_hash_root(uint64_t* h) { DC_PDL_ENTER();
  h[0] = H0_LO;
  h[1] = H0_HI;
}
// nodes [a, b): h[2n..2n+1] from the parent's
__global__ void k_hash_level(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ frame,
                             const uint32_t* __restrict__ l2g, uint32_t a, uint32_t b, uint64_t* __restrict__ h,
                             uint64_t mask) { DC_PDL_ENTER();
  for (uint32_t n = a + blockIdx.x * blockDim.x + threadIdx.x; n < b; n += gridDim.x * blockDim.x) {
    uint32_t p = parent[n];
    uint64_t lo = h[2ull * p], hi = h[2ull * p + 1];
    mix128(lo, hi, l2g ? l2g[frame[n]] : frame[n]);
    lo &= mask;
    hi &= mask;
    h[2ull * n] = lo;
    h[2ull * n + 1] = hi;
  }
}

// small trees: every level in one CTA (a barrier per level instead of a launch per level)
__global__ void __launch_bounds__(1024) k_hash_levels_one(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ frame,
                                                          const uint32_t* __restrict__ l2g, const uint32_t* __restrict__ level_off,
                                                          uint32_t maxd, uint64_t* h, uint64_t mask) { DC_PDL_ENTER();
  if (threadIdx.x == 0) {
    h[0] = H0_LO;
    h[1] = H0_HI;
  }
  __syncthreads();
  for (uint32_t d = 1; d <= maxd; ++d) {
    const uint32_t a = level_off[d], b = level_off[d + 1];
    for (uint32_t n = a + threadIdx.x; n < b; n += blockDim.x) {
      const uint32_t p = parent[n];
      uint64_t lo = __ldcg(h + 2ull * p), hi = __ldcg(h + 2ull * p + 1);
      mix128(lo, hi, l2g ? l2g[frame[n]] : frame[n]);
      h[2ull * n] = lo & mask;
      h[2ull * n + 1] = hi & mask;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ uint32_t owner_of(uint64_t hi, uint32_t P) { return (uint32_t)__umul64hi(hi, (uint64_t)P); }

// Block-cooperative slab slots: every thread of the block holds an owner o < P (or is idle);
// ranks within the block come from shared-memory counters, then one global atomic per owner
// per block tile (instead of one per record on P hot addresses). Returns the thread's slot in
// its owner's slab (count_only: only adds the tile's counts). P <= PART_MAXP.
constexpr uint32_t PART_MAXP = 1024;
__device__ __forceinline__ uint64_t part_slot(uint32_t o, bool valid, uint32_t P, unsigned long long* cursor, bool count_only) {
  __shared__ uint32_t s_cnt[PART_MAXP];
  __shared__ unsigned long long s_base[PART_MAXP];
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint32_t r = valid ? atomicAdd(&s_cnt[o], 1u) : 0u;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
    const uint32_t k = s_cnt[i];
    s_base[i] = k ? atomicAdd(cursor + i, (unsigned long long)k) : 0ull;
  }
  __syncthreads();
  const uint64_t slot = valid && !count_only ? s_base[o] + r : 0ull;
  __syncthreads();
  return slot;
}

__global__ void k_part_count(const uint64_t* __restrict__ h, uint64_t N, uint32_t P, unsigned long long* cnt) { DC_PDL_ENTER();
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < N; b += (uint64_t)gridDim.x * blockDim.x) {  // block-uniform
    const uint64_t n = b + threadIdx.x;
    part_slot(n < N ? owner_of(h[2 * n + 1], P) : 0u, n < N, P, cnt, true);
  }
}

// write node records into per-owner slabs (order inside a slab is irrelevant)
__global__ void k_part_nodes(const uint64_t* __restrict__ h, const uint32_t* __restrict__ parent, const uint32_t* __restrict__ frame,
                             const uint16_t* __restrict__ depth, const uint32_t* __restrict__ l2g, const uint64_t* __restrict__ xcnt,
                             const uint64_t* __restrict__ icnt, const uint64_t* __restrict__ mcols, const uint64_t* __restrict__ xs,
                             const uint64_t* __restrict__ is, const uint64_t* __restrict__ xst, const uint64_t* __restrict__ ist,
                             uint64_t N, RecFmt f, uint32_t P, unsigned long long* cursor, uint64_t* __restrict__ out) { DC_PDL_ENTER();
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < N; b += (uint64_t)gridDim.x * blockDim.x) {  // block-uniform
    const uint64_t n = b + threadIdx.x;
    const uint64_t slot = part_slot(n < N ? owner_of(h[2 * n + 1], P) : 0u, n < N, P, cursor, false);
    if (n >= N) continue;
    uint64_t* r = out + slot * f.W;
    r[0] = h[2 * n];
    r[1] = h[2 * n + 1];
    const uint32_t p = n ? parent[n] : 0;
    r[2] = n ? h[2ull * p] : 0;
    r[3] = n ? h[2ull * p + 1] : 0;
    const uint32_t gf = n ? (l2g ? l2g[frame[n]] : frame[n]) : DC_NO_NODE;
    r[4] = (uint64_t)gf | ((uint64_t)depth[n] << 32);
    r[5] = xcnt[n];
    r[6] = icnt[n];
    for (uint32_t m = 0; m < f.M; ++m)
      for (uint32_t w = 0; w < 8; ++w) r[7 + 8 * m + w] = mcols[((uint64_t)w * f.M + m) * N + n];
    if (f.has_pc) {
      uint64_t* q = r + 7 + 8 * f.M;
      q[0] = xs[n];
      q[1] = is[n];
      for (uint32_t s = 0; s < f.S; ++s) {
        q[2 + 2 * s] = xst[(uint64_t)s * N + n];
        q[3 + 2 * s] = ist[(uint64_t)s * N + n];
      }
    }
  }
}

__device__ __forceinline__ uint32_t bin_owner(uint64_t hlo, uint64_t hi, uint32_t pc, uint32_t P) {
  return owner_of(mix64(hi ^ hlo ^ ((uint64_t)pc * 0xD1B54A32D192ED03ull)), P);
}

// bins of a local tree -> (h_ctx, pc | stall << 32, count) records, per owner
__global__ void k_part_bins(const uint64_t* __restrict__ h, const uint32_t* __restrict__ bin_pcnode, const uint16_t* __restrict__ bin_stall,
                            const uint64_t* __restrict__ bin_count, const uint32_t* __restrict__ pc_ctx,
                            const uint32_t* __restrict__ pc_off, uint64_t N, uint64_t nb, uint32_t P, int count_only,
                            unsigned long long* cnt_or_cursor, uint64_t* __restrict__ out) { DC_PDL_ENTER();
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x; b < nb; b += (uint64_t)gridDim.x * blockDim.x) {  // block-uniform
    const uint64_t i = b + threadIdx.x;
    const bool valid = i < nb;
    uint32_t o = 0, pc = 0;
    uint64_t lo = 0, hi = 0;
    if (valid) {
      const uint32_t pn = bin_pcnode[i] - (uint32_t)N;
      const uint32_t ctx = pc_ctx[pn];
      pc = pc_off[pn];
      lo = h[2ull * ctx];
      hi = h[2ull * ctx + 1];
      o = bin_owner(lo, hi, pc, P);
    }
    const uint64_t slot = part_slot(o, valid, P, cnt_or_cursor, count_only != 0);
    if (count_only || !valid) continue;
    uint64_t* r = out + slot * BIN_W;
    r[0] = lo;
    r[1] = hi;
    r[2] = (uint64_t)pc | ((uint64_t)bin_stall[i] << 32);
    r[3] = bin_count[i];
  }
}

// ---------------------------------------------------------------- reduce received records
// Hash combine, no sort: every received record inserts its 128-bit key into an L2 hash table
// (nodes: the full-path hash; bins: a 128-bit mix of (context hash, pc, stall)); the first
// inserter of a key is its representative (its record index is published in the slot after the
// key, release / acquire). Representatives are numbered by a scan over the records (output
// order = receive order of the representatives); every record then adds / min-s its aggregate
// words into the output record with global atomics, after checking its identity words against
// the representative's: nodes (parent hash, global frame, depth), bins (the full key). Any
// mismatch is a hash collision (DC_ERR_COLLISION): the merge is exact or fails loudly. A key
// occurs at most once per source rank, so the atomics see at most P contributions per address.
constexpr uint32_t KV_EMPTY = 0xFFFFFFFFu;

__device__ __forceinline__ ulonglong2 kv_key(const uint64_t* r, bool bins) {
  if (!bins) return make_ulonglong2(r[0], r[1]);
  return make_ulonglong2(mix64(r[0] ^ (r[2] * 0x9E3779B97F4A7C15ull)), r[1] + mix64(r[2] + 0x632BE59BD9B4E019ull));
}

__global__ void k_kv_insert(const uint64_t* __restrict__ rec, uint32_t W, uint64_t n, bool bins, ulonglong2* tab, uint32_t* tval,
                            uint64_t mask, uint32_t* __restrict__ slot_of, uint32_t* d_flag) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2 k = kv_key(rec + i * W, bins);
    uint64_t s = mix64(k.x ^ k.y) & mask;
    for (uint64_t probe = 0;; ++probe, s = (s + 1) & mask) {
      if (probe > mask) {  // cannot happen: the table holds 2x the records
        atomicOr(d_flag, 2u);
        slot_of[i] = KV_EMPTY;
        break;
      }
      const ulonglong2 cur = ld_relaxed_v2(tab + s);
      bool mine = cur.x == k.x && cur.y == k.y;
      if (!mine) {
        if (cur.x != ~0ull || cur.y != ~0ull) continue;
        const unsigned __int128 expect = ~(unsigned __int128)0;
        const unsigned __int128 want = ((unsigned __int128)k.y << 64) | k.x;
        const unsigned __int128 old = atomicCAS(reinterpret_cast<unsigned __int128*>(tab + s), expect, want);
        if (old == expect) {  // representative: publish the record index
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(tval + s), "r"((uint32_t)i) : "memory");
          slot_of[i] = (uint32_t)s;
          break;
        }
        mine = old == want;
        if (!mine) continue;
      }
      slot_of[i] = (uint32_t)s;
      break;
    }
  }
}

__device__ __forceinline__ uint32_t kv_rep(const uint32_t* tval, uint32_t s) {
  uint32_t v;
  for (uint64_t spin = 0;; ++spin) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(tval + s) : "memory");
    if (v != KV_EMPTY) return v;
    if (spin > DC_SPIN_LIMIT) __trap();
  }
}

__global__ void k_kv_heads(const uint32_t* __restrict__ slot_of, const uint32_t* tval, uint64_t n, uint32_t* __restrict__ head) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = slot_of[i];
    head[i] = s != KV_EMPTY && kv_rep(tval, s) == (uint32_t)i ? 1u : 0u;
  }
}

// representatives: output index into the slot's value (after the heads pass) + identity record
__global__ void k_kv_init(const uint64_t* __restrict__ rec, uint32_t W, uint64_t n, bool bins, RecFmt f,
                          const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ head, const uint32_t* __restrict__ ridx,
                          uint32_t* tidx, uint64_t* __restrict__ out) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    const uint32_t o = ridx[i];
    tidx[slot_of[i]] = o;
    const uint64_t* a = rec + i * W;
    uint64_t* r = out + (uint64_t)o * W;
    if (bins) {
      r[0] = a[0];
      r[1] = a[1];
      r[2] = a[2];
      r[3] = 0;
      continue;
    }
    for (uint32_t w = 0; w < 5; ++w) r[w] = a[w];
    for (uint32_t w = 5; w < W; ++w) r[w] = 0;
    for (uint32_t m = 0; m < f.M; ++m) {
      r[7 + 8 * m + 1] = ~0ull;  // xmin
      r[7 + 8 * m + 5] = ~0ull;  // imin
    }
  }
}

__global__ void k_kv_combine(const uint64_t* __restrict__ rec, uint32_t W, uint64_t n, bool bins, RecFmt f,
                             const uint32_t* __restrict__ slot_of, const uint32_t* tval, const uint32_t* __restrict__ tidx,
                             unsigned long long* __restrict__ out, uint32_t* d_collision) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = slot_of[i];
    if (s == KV_EMPTY) continue;
    const uint64_t* b = rec + i * W;
    const uint64_t* a = rec + (uint64_t)kv_rep(tval, s) * W;
    unsigned long long* o = out + (uint64_t)tidx[s] * W;
    if (bins) {
      if (a[0] != b[0] || a[1] != b[1] || a[2] != b[2]) atomicOr(d_collision, 1u);
      atomicAdd(o + 3, (unsigned long long)b[3]);
      continue;
    }
    if (a[2] != b[2] || a[3] != b[3] || a[4] != b[4]) atomicOr(d_collision, 1u);
    if (b[5]) atomicAdd(o + 5, (unsigned long long)b[5]);
    if (b[6]) atomicAdd(o + 6, (unsigned long long)b[6]);
    for (uint32_t m = 0; m < f.M; ++m) {
      unsigned long long* om = o + 7 + 8 * m;
      const uint64_t* bm = b + 7 + 8 * m;
      if (bm[0]) atomicAdd(om, (unsigned long long)bm[0]);
      if (bm[1] != ~0ull) atomicMin(om + 1, (unsigned long long)bm[1]);
      if (bm[2] | bm[3]) atomic_add_u128(om + 2, om + 3, bm[2], bm[3]);
      if (bm[4]) atomicAdd(om + 4, (unsigned long long)bm[4]);
      if (bm[5] != ~0ull) atomicMin(om + 5, (unsigned long long)bm[5]);
      if (bm[6] | bm[7]) atomic_add_u128(om + 6, om + 7, bm[6], bm[7]);
    }
    if (f.has_pc)
      for (uint32_t w = 7 + 8 * f.M; w < W; ++w)
        if (b[w]) atomicAdd(o + w, (unsigned long long)b[w]);
  }
}

// received node records (W words) and bin records (BIN_W) -> unique records; one host round trip
static dc_status reduce_received(Ctx* c, const uint64_t* rn_p, uint64_t rn, const uint64_t* rb_p, uint64_t rb, const RecFmt& f,
                                 Buf<uint64_t>& out_n, uint64_t* n_out, Buf<uint64_t>& out_b, uint64_t* b_out, uint32_t* d_collision,
                                 bool owned /* outputs handed to a partition handle: pool memory */) {
  struct Side {
    const uint64_t* rec;
    uint64_t n;
    uint32_t W;
    bool bins;
    uint64_t cap;
    Buf<ulonglong2> tab;
    Buf<uint32_t> tval, tidx, slot, head, ridx;
  } side[2] = {{rn_p, rn, f.W, false, 0, {}, {}, {}, {}, {}, {}}, {rb_p, rb, (uint32_t)BIN_W, true, 0, {}, {}, {}, {}, {}, {}}};
  Buf<uint32_t> tot;
  DC_TRY(alloc_zero(c, tot, 3));  // [0] nodes, [1] bins, [2] table overflow flag
  for (int k = 0; k < 2; ++k) {
    Side& sd = side[k];
    if (!sd.n) continue;
    if (sd.n >= (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "merge: %llu received records", (unsigned long long)sd.n);
    sd.cap = 1024;
    while (sd.cap < 2 * sd.n) sd.cap <<= 1;
    DC_TRY(alloc(c, sd.tab, sd.cap));
    DC_TRY(alloc(c, sd.tval, sd.cap));
    DC_TRY(alloc(c, sd.tidx, sd.cap));
    DC_TRY(alloc(c, sd.slot, sd.n));
    DC_TRY(alloc(c, sd.head, sd.n));
    DC_TRY(alloc(c, sd.ridx, sd.n));
    {  // one fill kernel (a DMA memset between PDL-chained kernels costs a full launch latency)
      FillList fl;
      DC_TRY(fill_add(c, fl, sd.tab.p, sd.cap * 16, 0xFF));
      DC_TRY(fill_add(c, fl, sd.tval.p, sd.cap * 4, 0xFF));
      DC_TRY(fill_flush(c, fl));
    }
    dc_launch(k_kv_insert, grid_for(c, sd.n, 256), 256, 0, c->stream, sd.rec, sd.W, sd.n, sd.bins, sd.tab.p, sd.tval.p, sd.cap - 1,
              sd.slot.p, tot.p + 2);
    DC_LAUNCHED(c);
    dc_launch(k_kv_heads, grid_for(c, sd.n, 256), 256, 0, c->stream, sd.slot.p, sd.tval.p, sd.n, sd.head.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, sd.head.p, sd.ridx.p, sd.n, tot.p + k));
  }
  uint32_t ht[3] = {0, 0, 0};
  DC_TRY(readback(c, tot.p, 12, ht));
  if (ht[2]) return fail(c, DC_ERR_STATE, "internal: merge hash table overflow");
  *n_out = ht[0];
  *b_out = ht[1];
  if (owned) {
    DC_TRY(alloc_pool(c, out_n, (uint64_t)ht[0] * f.W));
    DC_TRY(alloc_pool(c, out_b, (uint64_t)ht[1] * BIN_W));
  } else {
    DC_TRY(alloc(c, out_n, (uint64_t)ht[0] * f.W));
    DC_TRY(alloc(c, out_b, (uint64_t)ht[1] * BIN_W));
  }
  for (int k = 0; k < 2; ++k) {
    Side& sd = side[k];
    if (!sd.n) continue;
    uint64_t* out = k ? out_b.p : out_n.p;
    dc_launch(k_kv_init, grid_for(c, sd.n, 256), 256, 0, c->stream, sd.rec, sd.W, sd.n, sd.bins, f, sd.slot.p, sd.head.p, sd.ridx.p,
              sd.tidx.p, out);
    DC_LAUNCHED(c);
    dc_launch(k_kv_combine, grid_for(c, sd.n, 256), 256, 0, c->stream, sd.rec, sd.W, sd.n, sd.bins, f, sd.slot.p, sd.tval.p,
              sd.tidx.p, (unsigned long long*)out, d_collision);
    DC_LAUNCHED(c);
  }
  return DC_OK;
}

// ---------------------------------------------------------------- per-rank partition step
struct Slabs {
  Buf<uint64_t> nodes, bins;
  std::vector<uint64_t> ncnt, bcnt;  // per destination
};

static dc_status partition(Ctx* c, const dc_cct* t, const uint32_t* l2g, uint32_t P, const RecFmt& f, Slabs& s) {
  const uint64_t N = t->N;
  Buf<uint64_t> h;
  DC_TRY(alloc(c, h, 2 * N));
  if (N <= (1u << 16)) {
    dc_launch(k_hash_levels_one, 1, 1024, 0, c->stream, t->parent, t->frame, l2g, t->level_off, t->max_depth, h.p, c->merge_mask);
    DC_LAUNCHED(c);
  } else {
    dc_launch(k_hash_root, 1, 1, 0, c->stream, h.p);
    DC_LAUNCHED(c);
    std::vector<uint32_t> lo(t->max_depth + 2);
    DC_TRY(readback(c, t->level_off, lo.size() * 4, lo.data()));
    for (uint32_t d = 1; d <= t->max_depth; ++d) {
      const uint32_t a = lo[d], b = lo[d + 1];
      if (b > a) {
        dc_launch(k_hash_level, grid_for(c, b - a, 256), 256, 0, c->stream, t->parent, t->frame, l2g, a, b, h.p, c->merge_mask);
        DC_LAUNCHED(c);
      }
    }
  }
  Buf<unsigned long long> cnt, cur;
  DC_TRY(alloc_zero(c, cnt, 2 * P));
  DC_TRY(alloc(c, cur, 2 * P));
  dc_launch(k_part_count, grid_for(c, N, 256), 256, 0, c->stream, h.p, N, P, cnt.p);
  DC_LAUNCHED(c);
  if (t->Nbins)
    dc_launch(k_part_bins, grid_for(c, t->Nbins, 256), 256, 0, c->stream, h.p, t->bin_pcnode, t->bin_stall, t->bin_count, t->pc_ctx,
                                                                   t->pc_off, N, t->Nbins, P, 1, cnt.p + P, nullptr);
  DC_LAUNCHED(c);
  std::vector<uint64_t> hc(2 * P);
  DC_TRY(readback(c, cnt.p, 16 * P, hc.data()));
  s.ncnt.assign(hc.begin(), hc.begin() + P);
  s.bcnt.assign(hc.begin() + P, hc.end());
  std::vector<uint64_t> ex(2 * P);
  uint64_t an = 0, ab = 0;
  for (uint32_t q = 0; q < P; ++q) {
    ex[q] = an;
    an += s.ncnt[q];
    ex[P + q] = ab;
    ab += s.bcnt[q];
  }
  DC_CUDA(c, cudaMemcpyAsync(cur.p, ex.data(), 16 * P, cudaMemcpyHostToDevice, c->stream));
  DC_TRY(alloc(c, s.nodes, an * f.W));
  DC_TRY(alloc(c, s.bins, ab * BIN_W));
  const uint64_t* mc = t->mcols;
  dc_launch(k_part_nodes, grid_for(c, N, 256), 256, 0, c->stream, h.p, t->parent, t->frame, t->depth, l2g, t->xcnt, t->icnt, mc,
                                                           t->xsamples, t->isamples, t->xstall, t->istall, N, f, P, cur.p,
                                                           s.nodes.p);
  DC_LAUNCHED(c);
  if (t->Nbins) {
    dc_launch(k_part_bins, grid_for(c, t->Nbins, 256), 256, 0, c->stream, h.p, t->bin_pcnode, t->bin_stall, t->bin_count, t->pc_ctx,
                                                                   t->pc_off, N, t->Nbins, P, 0, cur.p + P, s.bins.p);
    DC_LAUNCHED(c);
  }
  DC_CUDA(c, cudaStreamSynchronize(c->stream));  // ex[] (host) must outlive the async copy
  return DC_OK;
}

// a merged partition: unique node records + unique bin records (kept in record form)
static dc_cct* make_partition(Ctx* c, const RecFmt& f, uint64_t n_nodes, Buf<uint64_t>& nodes, uint64_t n_bins,
                              Buf<uint64_t>& bins, uint32_t n_frames) {
  dc_cct* t = new dc_cct();
  t->device = c->device;
  t->owner_uid = adopt_handle(c);
  t->M = f.M;
  t->S = f.has_pc ? f.S : 0;
  t->N = n_nodes;
  t->n_frames = n_frames;
  t->state = 2;
  t->partition = true;
  t->part_nodes = nodes.release_ownership();
  t->part_bins = bins.release_ownership();
  t->part_nbins = n_bins;
  t->part_W = f.W;
  t->part_has_pc = f.has_pc;
  return t;
}

// ---------------------------------------------------------------- canonicalisation (gather)
// all unique node records (any order) -> canonical CCT
__global__ void k_canon_depthkey(const uint64_t* __restrict__ rec, uint32_t W, uint64_t n, uint64_t* __restrict__ key,
                                 uint32_t* __restrict__ val) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    key[i] = rec[i * W + 4] >> 32;  // depth
    val[i] = (uint32_t)i;
  }
}

// hash table h(128) -> canonical id
__device__ __forceinline__ uint64_t htab_slot(uint64_t lo, uint64_t hi, uint64_t mask) { return mix64(lo ^ (hi * 3)) & mask; }
__global__ void k_htab_insert(const uint64_t* __restrict__ rec, uint32_t W, const uint32_t* __restrict__ order, uint32_t a, uint32_t b,
                              const uint32_t* __restrict__ canon_of_pos, ulonglong2* tab, uint32_t* tid, uint64_t mask) { DC_PDL_ENTER();
  for (uint32_t i = a + blockIdx.x * blockDim.x + threadIdx.x; i < b; i += gridDim.x * blockDim.x) {
    const uint64_t* r = rec + (uint64_t)order[i] * W;
    const uint64_t lo = r[0], hi = r[1];
    uint64_t s = htab_slot(lo, hi, mask);
    while (true) {
      unsigned __int128 expect = ~(unsigned __int128)0;
      unsigned __int128 want = ((unsigned __int128)hi << 64) | lo;
      unsigned __int128 old = atomicCAS(reinterpret_cast<unsigned __int128*>(tab + s), expect, want);
      if (old == expect || old == want) break;
      s = (s + 1) & mask;
    }
    tid[s] = canon_of_pos[i];
  }
}
__device__ __forceinline__ uint32_t htab_find(const ulonglong2* tab, const uint32_t* tid, uint64_t mask, uint64_t lo, uint64_t hi) {
  uint64_t s = htab_slot(lo, hi, mask);
  while (true) {
    ulonglong2 v = tab[s];
    if (v.x == lo && v.y == hi) return tid[s];
    if (v.x == ~0ull && v.y == ~0ull) return DC_NO_NODE;
    s = (s + 1) & mask;
  }
}

// level d: key = (parent canonical id - level_start(d-1)) << fbits | gframe for records order[a..b)
__global__ void k_canon_keys(const uint64_t* __restrict__ rec, uint32_t W, const uint32_t* __restrict__ order, uint32_t a, uint32_t b,
                             const ulonglong2* __restrict__ tab, const uint32_t* __restrict__ tid, uint64_t mask, uint32_t prev_start,
                             int fbits, uint64_t* __restrict__ key, uint32_t* __restrict__ val, uint32_t* d_err) { DC_PDL_ENTER();
  for (uint32_t i = a + blockIdx.x * blockDim.x + threadIdx.x; i < b; i += gridDim.x * blockDim.x) {
    const uint64_t* r = rec + (uint64_t)order[i] * W;
    const uint32_t p = htab_find(tab, tid, mask, r[2], r[3]);
    if (p == DC_NO_NODE) atomicOr(d_err, 1u);
    key[i - a] = ((uint64_t)(p - prev_start) << fbits) | (uint32_t)r[4];
    val[i - a] = order[i];
  }
}

__global__ void k_canon_emit(const uint64_t* __restrict__ rec, RecFmt f, const uint32_t* __restrict__ src, uint64_t n_level,
                             const uint64_t* __restrict__ key, int fbits, uint32_t prev_start, uint32_t start, uint64_t N,
                             uint32_t* __restrict__ parent, uint32_t* __restrict__ frame, uint16_t* __restrict__ depth,
                             uint64_t* __restrict__ xcnt, uint64_t* __restrict__ icnt, uint64_t* __restrict__ mcols,
                             uint64_t* __restrict__ xs, uint64_t* __restrict__ is, uint64_t* __restrict__ xst,
                             uint64_t* __restrict__ ist, uint32_t* __restrict__ canon_of_pos, uint32_t dpt) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_level; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = start + (uint32_t)i;
    const uint64_t* r = rec + (uint64_t)src[i] * f.W;
    parent[id] = dpt == 0 ? DC_NO_NODE : prev_start + (uint32_t)(key[i] >> fbits);
    frame[id] = dpt == 0 ? DC_NO_NODE : (uint32_t)r[4];
    depth[id] = (uint16_t)dpt;
    xcnt[id] = r[5];
    icnt[id] = r[6];
    for (uint32_t m = 0; m < f.M; ++m)
      for (uint32_t w = 0; w < 8; ++w) mcols[((uint64_t)w * f.M + m) * N + id] = r[7 + 8 * m + w];
    if (f.has_pc) {
      const uint64_t* q = r + 7 + 8 * f.M;
      xs[id] = q[0];
      is[id] = q[1];
      for (uint32_t s = 0; s < f.S; ++s) {
        xst[(uint64_t)s * N + id] = q[2 + 2 * s];
        ist[(uint64_t)s * N + id] = q[3 + 2 * s];
      }
    }
    canon_of_pos[i] = id;
  }
}

// bins -> (ctx canonical, pc, stall) sort keys
__global__ void k_canon_binkeys(const uint64_t* __restrict__ bins, uint64_t nb, const ulonglong2* __restrict__ tab,
                                const uint32_t* __restrict__ tid, uint64_t mask, int pcb, uint64_t* __restrict__ key,
                                uint32_t* __restrict__ val, uint32_t* d_err) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t* r = bins + i * BIN_W;
    const uint32_t ctx = htab_find(tab, tid, mask, r[0], r[1]);
    if (ctx == DC_NO_NODE) atomicOr(d_err, 1u);
    const uint32_t pc = (uint32_t)r[2], stall = (uint32_t)(r[2] >> 32);
    key[i] = ((((uint64_t)ctx << pcb) | pc) << 5) | stall;
    val[i] = (uint32_t)i;
  }
}
__global__ void k_canon_binmax(const uint64_t* __restrict__ bins, uint64_t nb, unsigned int* mx) { DC_PDL_ENTER();
  uint32_t m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, (uint32_t)bins[i * BIN_W + 2]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(mx, m);
}
__global__ void k_canon_binheads(const uint64_t* __restrict__ key, uint64_t nb, uint32_t* __restrict__ head) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (key[i - 1] >> 5) != (key[i] >> 5)) ? 1u : 0u;
}
__global__ void k_canon_binemit(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val, const uint64_t* __restrict__ bins,
                                uint64_t nb, int pcb, const uint32_t* __restrict__ head, const uint32_t* __restrict__ run, uint64_t N,
                                uint32_t* __restrict__ pc_ctx, uint32_t* __restrict__ pc_off, uint32_t* __restrict__ bin_pcnode,
                                uint16_t* __restrict__ bin_stall, uint64_t* __restrict__ bin_count) { DC_PDL_ENTER();
  const uint64_t pm = (1ull << pcb) - 1ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    const uint32_t p = run[i] + head[i] - 1u;
    if (head[i]) {
      pc_ctx[p] = (uint32_t)((k >> 5) >> pcb);
      pc_off[p] = (uint32_t)((k >> 5) & pm);
    }
    bin_pcnode[i] = (uint32_t)(N + p);
    bin_stall[i] = (uint16_t)(k & 31u);
    bin_count[i] = bins[(uint64_t)val[i] * BIN_W + 3];
  }
}

static dc_status canonicalize(Ctx* c, const uint64_t* rec, uint64_t n, const uint64_t* bins, uint64_t nb, const RecFmt& f,
                              uint32_t n_frames, dc_cct** out) {
  *out = nullptr;
  if (n == 0) return fail(c, DC_ERR_STATE, "merge: no node records (the root is missing)");
  // order by depth (stable)
  Buf<uint64_t> k0, k1;
  Buf<uint32_t> v0, v1;
  DC_TRY(alloc(c, k0, n));
  DC_TRY(alloc(c, k1, n));
  DC_TRY(alloc(c, v0, n));
  DC_TRY(alloc(c, v1, n));
  dc_launch(k_canon_depthkey, grid_for(c, n, 256), 256, 0, c->stream, rec, f.W, n, k0.p, v0.p);
  DC_LAUNCHED(c);
  bool in1 = false;
  DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, n, 0, 16, &in1));
  Buf<uint32_t> byd;  // record indices ordered by depth
  DC_TRY(alloc(c, byd, n));
  DC_CUDA(c, cudaMemcpyAsync(byd.p, in1 ? v1.p : v0.p, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  std::vector<uint64_t> dk(n);
  DC_TRY(readback(c, in1 ? k1.p : k0.p, n * 8, dk.data()));
  // level boundaries
  std::vector<uint32_t> lvl;
  for (uint64_t i = 0; i < n; ++i)
    if (i == 0 || dk[i] != dk[i - 1]) {
      if (dk[i] != lvl.size()) return fail(c, DC_ERR_COLLISION, "merge: depth levels are not contiguous");
      lvl.push_back((uint32_t)i);
    }
  lvl.push_back((uint32_t)n);
  const uint32_t L = (uint32_t)lvl.size() - 1;
  if (lvl[1] != 1) return fail(c, DC_ERR_COLLISION, "merge: %u root records", lvl[1]);
  dc_cct* t = new dc_cct();
  t->device = c->device;
  t->owner_uid = adopt_handle(c);
  t->N = n;
  t->n_frames = n_frames;
  t->max_depth = L - 1;
  t->S = f.has_pc ? f.S : 0;
  DC_TRY(palloc(c, t->parent, n));
  DC_TRY(palloc(c, t->frame, n));
  DC_TRY(palloc(c, t->depth, n));
  DC_TRY(palloc(c, t->level_off, L + 1));
  DC_CUDA(c, cudaMemcpyAsync(t->level_off, lvl.data(), (L + 1) * 4, cudaMemcpyHostToDevice, c->stream));
  DC_TRY(palloc(c, t->xcnt, n));
  DC_TRY(palloc(c, t->icnt, n));
  if (f.M) {
    t->M = 0;
    DC_TRY(ensure_metric_cols(c, t, f.M));
  }
  if (f.has_pc) {
    DC_TRY(palloc(c, t->xsamples, n));
    DC_TRY(palloc(c, t->isamples, n));
    DC_TRY(palloc(c, t->xstall, (uint64_t)f.S * n));
    DC_TRY(palloc(c, t->istall, (uint64_t)f.S * n));
  }
  uint64_t cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  Buf<ulonglong2> tab;
  Buf<uint32_t> tid, canon, err;
  DC_TRY(alloc(c, tab, cap));
  DC_TRY(alloc(c, tid, cap));
  DC_TRY(alloc(c, canon, n));
  DC_TRY(alloc_zero(c, err, 1));
  DC_CUDA(c, cudaMemsetAsync(tab.p, 0xFF, cap * 16, c->stream));
  const int fbits = bits_for(n_frames > 1 ? n_frames - 1 : 1);
  uint32_t prev_start = 0;
  for (uint32_t d = 0; d < L; ++d) {
    const uint32_t a = lvl[d], b = lvl[d + 1], m = b - a;
    const uint32_t* src;
    uint64_t* keys = k0.p;
    if (d == 0) {
      src = byd.p;
      DC_CUDA(c, cudaMemsetAsync(k0.p, 0, 8, c->stream));
    } else {
      const int pbits = bits_for(lvl[d] - lvl[d - 1] > 1 ? lvl[d] - lvl[d - 1] - 1 : 1);
      dc_launch(k_canon_keys, grid_for(c, m, 256), 256, 0, c->stream, rec, f.W, byd.p, a, b, tab.p, tid.p, cap - 1, prev_start, fbits,
                                                               k0.p, v0.p, err.p);
      DC_LAUNCHED(c);
      bool r1 = false;
      DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, m, 0, pbits + fbits, &r1));
      keys = r1 ? k1.p : k0.p;
      src = r1 ? v1.p : v0.p;
    }
    dc_launch(k_canon_emit, grid_for(c, m, 256), 256, 0, c->stream, rec, f, src, m, keys, fbits, prev_start, a, n, t->parent, t->frame,
                                                             t->depth, t->xcnt, t->icnt, t->mcols, t->xsamples, t->isamples,
                                                             t->xstall, t->istall, canon.p, d);
    DC_LAUNCHED(c);
    // register this level's hashes: position i (in emit order) -> canonical id a + i
    // (emit order == src order; insert needs the record index per position)
    dc_launch(k_htab_insert, grid_for(c, m, 256), 256, 0, c->stream, rec, f.W, src, 0, m, canon.p, tab.p, tid.p, cap - 1);
    DC_LAUNCHED(c);
    prev_start = a;
  }
  uint32_t herr = 0;
  DC_TRY(readback(c, err.p, 4, &herr));
  if (herr) return fail(c, DC_ERR_COLLISION, "merge: a node's parent hash was not found at the previous level");
  // bins
  if (f.has_pc && nb) {
    Buf<uint64_t> bk0, bk1;
    Buf<uint32_t> bv0, bv1, head, run, tot;
    Buf<unsigned int> mx;
    DC_TRY(alloc(c, bk0, nb));
    DC_TRY(alloc(c, bk1, nb));
    DC_TRY(alloc(c, bv0, nb));
    DC_TRY(alloc(c, bv1, nb));
    DC_TRY(alloc_zero(c, mx, 1));
    dc_launch(k_canon_binmax, grid_for(c, nb, 256), 256, 0, c->stream, bins, nb, mx.p);
    DC_LAUNCHED(c);
    uint32_t hm = 0;
    DC_TRY(readback(c, mx.p, 4, &hm));
    const int pcb = bits_for(hm) ? bits_for(hm) : 1;
    dc_launch(k_canon_binkeys, grid_for(c, nb, 256), 256, 0, c->stream, bins, nb, tab.p, tid.p, cap - 1, pcb, bk0.p, bv0.p, err.p);
    DC_LAUNCHED(c);
    bool r1 = false;
    DC_TRY(radix_sort_pairs(c, bk0.p, bv0.p, bk1.p, bv1.p, nb, 0, bits_for(n) + pcb + 5, &r1));
    uint64_t* sk = r1 ? bk1.p : bk0.p;
    uint32_t* sv = r1 ? bv1.p : bv0.p;
    DC_TRY(alloc(c, head, nb));
    DC_TRY(alloc(c, run, nb));
    DC_TRY(alloc(c, tot, 1));
    dc_launch(k_canon_binheads, grid_for(c, nb, 256), 256, 0, c->stream, sk, nb, head.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, head.p, run.p, nb, tot.p));
    uint32_t npc = 0;
    DC_TRY(readback(c, tot.p, 4, &npc));
    t->Npc = npc;
    t->Nbins = nb;
    DC_TRY(palloc(c, t->pc_ctx, npc));
    DC_TRY(palloc(c, t->pc_off, npc));
    DC_TRY(palloc(c, t->bin_pcnode, nb));
    DC_TRY(palloc(c, t->bin_stall, nb));
    DC_TRY(palloc(c, t->bin_count, nb));
    dc_launch(k_canon_binemit, grid_for(c, nb, 256), 256, 0, c->stream, sk, sv, bins, nb, pcb, head.p, run.p, n, t->pc_ctx, t->pc_off,
                                                                 t->bin_pcnode, t->bin_stall, t->bin_count);
    DC_LAUNCHED(c);
  }
  t->pc_done = f.has_pc;
  t->state = 2;
  *out = t;
  return DC_OK;
}

// ---------------------------------------------------------------- dictionary unify
__global__ void k_l2g(const uint32_t* __restrict__ ids, uint64_t base, uint64_t D, uint32_t* __restrict__ l2g) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < D; i += (uint64_t)gridDim.x * blockDim.x)
    l2g[i] = ids[base + i];
}

// keys of P dictionaries concatenated (key_off[p] .. key_off[p+1]) -> global dict + per-p l2g maps
static dc_status unify_dicts(Ctx* c, const dc_frame_key* all_keys, const std::vector<uint64_t>& key_off, dc_dict** gdict,
                             std::vector<Buf<uint32_t>>& l2g) {
  const uint64_t total = key_off.back();
  Buf<uint32_t> ids;
  DC_TRY(alloc(c, ids, total));
  uint64_t dmax = 0;  // the union has at least the largest rank's distinct keys, at most all of them
  for (size_t p = 0; p + 1 < key_off.size(); ++p) dmax = std::max<uint64_t>(dmax, key_off[p + 1] - key_off[p]);
  DC_TRY(intern_frames(c, all_keys, total, ids.p, gdict, std::min<uint64_t>(total, 2 * dmax)));
  l2g.resize(key_off.size() - 1);
  for (size_t p = 0; p + 1 < key_off.size(); ++p) {
    const uint64_t D = key_off[p + 1] - key_off[p];
    DC_TRY(alloc(c, l2g[p], D));
    if (D) {
      dc_launch(k_l2g, grid_for(c, D, 256), 256, 0, c->stream, ids.p, key_off[p], D, l2g[p].p);
      DC_LAUNCHED(c);
    }
  }
  DC_CUDA(c, cudaStreamSynchronize(c->stream));
  return DC_OK;
}

static RecFmt fmt_of(const dc_cct* t) { return rec_fmt(t->M, t->S, t->xsamples != nullptr); }

}  // namespace dc

using namespace dc;

// ---------------------------------------------------------------- NCCL communicator
struct dc_comm {
  int nranks = 1, rank = 0, device = 0;
#if DC_HAVE_NCCL
  ncclComm_t comm = nullptr;
#endif
};

#if DC_HAVE_NCCL
#define NCCL_TRY(c, expr)                                                                       \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess) return fail((c), DC_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(_r)); \
  } while (0)
#endif

extern "C" {

dc_status dc_merge_plan(uint32_t P, const uint64_t* send_counts, const uint64_t* recv_counts, uint64_t* send_off,
                        uint64_t* recv_off, uint64_t* recv_total) {
  if (!P || !send_counts || !recv_counts || !send_off || !recv_off || !recv_total) return DC_ERR_ARG;
  uint64_t so[2] = {0, 0}, ro[2] = {0, 0};
  for (uint32_t q = 0; q < P; ++q)
    for (int k = 0; k < 2; ++k) {
      send_off[2 * q + k] = so[k];
      recv_off[2 * q + k] = ro[k];
      so[k] += send_counts[2 * q + k];
      ro[k] += recv_counts[2 * q + k];
    }
  recv_total[0] = ro[0];
  recv_total[1] = ro[1];
  return DC_OK;
}

dc_status dc_nccl_unique_id(uint8_t out_h[128]) {
#if DC_HAVE_NCCL
  if (!out_h) return DC_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DC_ERR_NCCL;
  memcpy(out_h, id.internal, 128);
  return DC_OK;
#else
  return DC_ERR_NCCL;
#endif
}

dc_status dc_comm_create(dc_ctx* ctx, const uint8_t uid[128], int nranks, int rank, dc_comm** out) {
  if (!ctx || !uid || !out || nranks < 1 || rank < 0 || rank >= nranks || (uint32_t)nranks > PART_MAXP) return DC_ERR_ARG;
#if DC_HAVE_NCCL
  cudaSetDevice(ctx->device);
  dc_comm* cm = new dc_comm();
  cm->nranks = nranks;
  cm->rank = rank;
  cm->device = ctx->device;
  ncclUniqueId id;
  memcpy(id.internal, uid, 128);
  ncclResult_t r = ncclCommInitRank(&cm->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete cm;
    return fail(ctx, DC_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = cm;
  return DC_OK;
#else
  return fail(ctx, DC_ERR_NCCL, "built without NCCL");
#endif
}

void dc_comm_destroy(dc_comm* cm) {
  if (!cm) return;
#if DC_HAVE_NCCL
  if (cm->comm) ncclCommDestroy(cm->comm);
#endif
  delete cm;
}

dc_status dc_cct_merge_ranks(dc_ctx* ctx, dc_comm* cm, const dc_cct* local, const dc_dict* local_dict, dc_cct** out_partition,
                             dc_dict** out_global_dict) {
  if (!ctx || !cm || !local || !local_dict || !out_partition || !out_global_dict) return DC_ERR_ARG;
  if (local->state != 2 || local->partition) return fail(ctx, DC_ERR_STATE, "dc_cct_merge_ranks needs a rolled-up local tree");
  if (local_dict->D != local->n_frames) return fail(ctx, DC_ERR_ARG, "dictionary size != tree n_frames");
#if DC_HAVE_NCCL
  Ctx* c = ctx;
  DC_CUDA(c, cudaSetDevice(c->device));
  c->arena_reset();
  Region rg(c, "merge");
  const int P = cm->nranks;
  // 1. dictionaries: all-gather sizes together with each rank's record format (M, S, has_pc);
  // every rank sees the same table, so a disagreement fails on every rank before any transfer
  Buf<uint64_t> dsz;
  DC_TRY(alloc(c, dsz, 4 * (uint64_t)P));
  const RecFmt f = fmt_of(local);
  const uint64_t mine[4] = {local_dict->D, local->M, f.has_pc ? local->S : 0, f.has_pc ? 1u : 0u};
  DC_CUDA(c, cudaMemcpyAsync(dsz.p + 4 * cm->rank, mine, 32, cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, ncclAllGather(dsz.p + 4 * cm->rank, dsz.p, 4, ncclUint64, cm->comm, c->stream));
  std::vector<uint64_t> tab(4 * (size_t)P), Ds(P);
  DC_TRY(readback(c, dsz.p, 32 * (size_t)P, tab.data()));
  for (int p = 0; p < P; ++p) {
    Ds[p] = tab[4 * p];
    if (tab[4 * p + 1] != tab[1] || tab[4 * p + 2] != tab[2] || tab[4 * p + 3] != tab[3])
      return fail(c, DC_ERR_ARG, "merge: rank %d has (M=%llu, S=%llu, pc=%llu) but rank 0 has (M=%llu, S=%llu, pc=%llu)", p,
                  (unsigned long long)tab[4 * p + 1], (unsigned long long)tab[4 * p + 2], (unsigned long long)tab[4 * p + 3],
                  (unsigned long long)tab[1], (unsigned long long)tab[2], (unsigned long long)tab[3]);
  }
  uint64_t Dmax = 1;
  for (auto d : Ds) Dmax = d > Dmax ? d : Dmax;
  Buf<dc_frame_key> pad, all, packed;
  DC_TRY(alloc(c, pad, Dmax));
  DC_TRY(alloc(c, all, Dmax * P));
  const uint64_t myD = local_dict->D;
  if (myD) DC_CUDA(c, cudaMemcpyAsync(pad.p, local_dict->keys, myD * 16, cudaMemcpyDeviceToDevice, c->stream));
  NCCL_TRY(c, ncclAllGather(pad.p, all.p, Dmax * 2, ncclUint64, cm->comm, c->stream));
  std::vector<uint64_t> koff(P + 1, 0);
  for (int p = 0; p < P; ++p) koff[p + 1] = koff[p] + Ds[p];
  DC_TRY(alloc(c, packed, koff[P]));
  for (int p = 0; p < P; ++p)
    if (Ds[p]) DC_CUDA(c, cudaMemcpyAsync(packed.p + koff[p], all.p + (uint64_t)p * Dmax, Ds[p] * 16, cudaMemcpyDeviceToDevice, c->stream));
  dc_dict* gd = nullptr;
  std::vector<Buf<uint32_t>> l2g;
  DC_TRY(unify_dicts(c, packed.p, koff, &gd, l2g));
  // 2-3. hash + partition
  Slabs s;
  DC_TRY(partition(c, local, l2g[cm->rank].p, P, f, s));
  // 4. exchange counts, then slabs
  Buf<uint64_t> sc, rc;
  DC_TRY(alloc(c, sc, 2 * P));
  DC_TRY(alloc(c, rc, 2 * P));
  std::vector<uint64_t> hsc(2 * P);
  for (int q = 0; q < P; ++q) {
    hsc[2 * q] = s.ncnt[q];
    hsc[2 * q + 1] = s.bcnt[q];
  }
  DC_CUDA(c, cudaMemcpyAsync(sc.p, hsc.data(), 16 * P, cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, ncclAlltoAll(sc.p, rc.p, 2, ncclUint64, cm->comm, c->stream));
  std::vector<uint64_t> hrc(2 * P), soff(2 * P), roff(2 * P);
  DC_TRY(readback(c, rc.p, 16 * P, hrc.data()));
  uint64_t rtot[2];
  DC_TRY(dc_merge_plan((uint32_t)P, hsc.data(), hrc.data(), soff.data(), roff.data(), rtot));  // host-only exchange plan
  const uint64_t rn = rtot[0], rb = rtot[1];
  Buf<uint64_t> rnodes, rbins;
  DC_TRY(alloc(c, rnodes, rn * f.W));
  DC_TRY(alloc(c, rbins, rb * BIN_W));
  {
    NCCL_TRY(c, ncclGroupStart());
    for (int q = 0; q < P; ++q) {
      if (hsc[2 * q]) NCCL_TRY(c, ncclSend(s.nodes.p + soff[2 * q] * f.W, hsc[2 * q] * f.W, ncclUint64, q, cm->comm, c->stream));
      if (hrc[2 * q]) NCCL_TRY(c, ncclRecv(rnodes.p + roff[2 * q] * f.W, hrc[2 * q] * f.W, ncclUint64, q, cm->comm, c->stream));
      if (hsc[2 * q + 1])
        NCCL_TRY(c, ncclSend(s.bins.p + soff[2 * q + 1] * BIN_W, hsc[2 * q + 1] * BIN_W, ncclUint64, q, cm->comm, c->stream));
      if (hrc[2 * q + 1])
        NCCL_TRY(c, ncclRecv(rbins.p + roff[2 * q + 1] * BIN_W, hrc[2 * q + 1] * BIN_W, ncclUint64, q, cm->comm, c->stream));
    }
    NCCL_TRY(c, ncclGroupEnd());
  }
  // 5. reduce + verify
  Buf<uint32_t> coll;
  DC_TRY(alloc_zero(c, coll, 1));
  Buf<uint64_t> un, ub;
  uint64_t nun = 0, nub = 0;
  DC_TRY(reduce_received(c, rnodes.p, rn, rbins.p, rb, f, un, &nun, ub, &nub, coll.p, true));
  uint32_t hcoll = 0;
  DC_TRY(readback(c, coll.p, 4, &hcoll));
  if (hcoll) {
    c->host_collisions += 1;
    dc_dict_free(gd);
    return fail(c, DC_ERR_COLLISION, "merge: 128-bit path hash collision detected");
  }
  c->bytes_host += (rn * f.W + rb * BIN_W) * 8 * 2;
  *out_partition = make_partition(c, f, nun, un, nub, ub, (uint32_t)gd->D);
  *out_global_dict = gd;
  return DC_OK;
#else
  return fail(ctx, DC_ERR_NCCL, "built without NCCL");
#endif
}

dc_status dc_cct_gather(dc_ctx* ctx, dc_comm* cm, const dc_cct* part, int root, dc_cct** out_canonical) {
  if (!ctx || !cm || !part || !out_canonical || root < 0 || root >= cm->nranks) return DC_ERR_ARG;
  if (!part->partition) return fail(ctx, DC_ERR_STATE, "dc_cct_gather takes a partition from dc_cct_merge_ranks");
  *out_canonical = nullptr;
#if DC_HAVE_NCCL
  Ctx* c = ctx;
  DC_CUDA(c, cudaSetDevice(c->device));
  c->arena_reset();
  const int P = cm->nranks;
  const RecFmt f = rec_fmt(part->M, part->S, part->part_has_pc);
  Buf<uint64_t> cnt;
  DC_TRY(alloc(c, cnt, 2 * P));
  uint64_t mine[2] = {part->N, part->part_nbins};
  DC_CUDA(c, cudaMemcpyAsync(cnt.p + 2 * cm->rank, mine, 16, cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, ncclAllGather(cnt.p + 2 * cm->rank, cnt.p, 2, ncclUint64, cm->comm, c->stream));
  std::vector<uint64_t> hc(2 * P);
  DC_TRY(readback(c, cnt.p, 16 * P, hc.data()));
  uint64_t tn = 0, tb = 0;
  for (int q = 0; q < P; ++q) {
    tn += hc[2 * q];
    tb += hc[2 * q + 1];
  }
  Buf<uint64_t> allv, allb;
  if (cm->rank == root) {
    DC_TRY(alloc(c, allv, tn * f.W));
    DC_TRY(alloc(c, allb, tb * BIN_W));
  }
  NCCL_TRY(c, ncclGroupStart());
  if (part->N) NCCL_TRY(c, ncclSend(part->part_nodes, part->N * f.W, ncclUint64, root, cm->comm, c->stream));
  if (part->part_nbins) NCCL_TRY(c, ncclSend(part->part_bins, part->part_nbins * BIN_W, ncclUint64, root, cm->comm, c->stream));
  if (cm->rank == root) {
    uint64_t o = 0, ob = 0;
    for (int q = 0; q < P; ++q) {
      if (hc[2 * q]) NCCL_TRY(c, ncclRecv(allv.p + o * f.W, hc[2 * q] * f.W, ncclUint64, q, cm->comm, c->stream));
      if (hc[2 * q + 1]) NCCL_TRY(c, ncclRecv(allb.p + ob * BIN_W, hc[2 * q + 1] * BIN_W, ncclUint64, q, cm->comm, c->stream));
      o += hc[2 * q];
      ob += hc[2 * q + 1];
    }
  }
  NCCL_TRY(c, ncclGroupEnd());
  if (cm->rank != root) {
    DC_CUDA(c, cudaStreamSynchronize(c->stream));
    return DC_OK;
  }
  return canonicalize(c, allv.p, tn, allb.p, tb, f, part->n_frames, out_canonical);
#else
  return fail(ctx, DC_ERR_NCCL, "built without NCCL");
#endif
}

dc_status dc_cct_merge_local(dc_ctx* ctx, uint32_t P, dc_cct* const* locals, dc_dict* const* dicts, dc_cct** out_canonical,
                             dc_dict** out_global_dict) {
  if (!ctx || !P || P > PART_MAXP || !locals || !dicts || !out_canonical || !out_global_dict) return DC_ERR_ARG;
  Ctx* c = ctx;
  DC_CUDA(c, cudaSetDevice(c->device));
  c->arena_reset();
  for (uint32_t p = 0; p < P; ++p) {
    if (!locals[p] || !dicts[p] || locals[p]->state != 2) return fail(c, DC_ERR_STATE, "local tree %u is not rolled up", p);
    if (dicts[p]->D != locals[p]->n_frames) return fail(c, DC_ERR_ARG, "dictionary %u size != n_frames", p);
    if (locals[p]->M != locals[0]->M || locals[p]->S != locals[0]->S ||
        (locals[p]->xsamples != nullptr) != (locals[0]->xsamples != nullptr))
      return fail(c, DC_ERR_ARG, "local trees disagree on metric / stall columns");
  }
  Region r_all(c, "merge");
  // 1. dictionaries (loopback all-gather = concatenation)
  std::unique_ptr<Region> r1(new Region(c, "merge:dict"));
  std::vector<uint64_t> koff(P + 1, 0);
  for (uint32_t p = 0; p < P; ++p) koff[p + 1] = koff[p] + dicts[p]->D;
  Buf<dc_frame_key> packed;
  DC_TRY(alloc(c, packed, koff[P]));
  for (uint32_t p = 0; p < P; ++p)
    if (dicts[p]->D)
      DC_CUDA(c, cudaMemcpyAsync(packed.p + koff[p], dicts[p]->keys, dicts[p]->D * 16, cudaMemcpyDeviceToDevice, c->stream));
  dc_dict* gd = nullptr;
  std::vector<Buf<uint32_t>> l2g;
  DC_TRY(unify_dicts(c, packed.p, koff, &gd, l2g));
  const RecFmt f = fmt_of(locals[0]);
  r1.reset();
  // 2-3. every logical rank partitions
  std::vector<Slabs> slabs(P);
  {
    Region rp(c, "merge:partition");
    for (uint32_t p = 0; p < P; ++p) DC_TRY(partition(c, locals[p], l2g[p].p, P, f, slabs[p]));
  }
  std::unique_ptr<Region> r3(new Region(c, "merge:exchange+reduce"));
  // 4. loopback exchange + 5. reduce per destination; 6. gather = concatenation of partitions
  std::vector<Buf<uint64_t>> parts_n(P), parts_b(P);
  std::vector<uint64_t> pn(P), pb(P);
  Buf<uint32_t> coll;
  DC_TRY(alloc_zero(c, coll, 1));
  // the exchange plan of every logical rank (the same host-only dc_merge_plan as the NCCL path)
  std::vector<std::vector<uint64_t>> sc(P, std::vector<uint64_t>(2 * P)), soff(P, std::vector<uint64_t>(2 * P));
  for (uint32_t p = 0; p < P; ++p) {
    for (uint32_t q = 0; q < P; ++q) {
      sc[p][2 * q] = slabs[p].ncnt[q];
      sc[p][2 * q + 1] = slabs[p].bcnt[q];
    }
    std::vector<uint64_t> none(2 * P, 0), unused(2 * P);
    uint64_t rt[2];
    DC_TRY(dc_merge_plan(P, sc[p].data(), none.data(), soff[p].data(), unused.data(), rt));
  }
  for (uint32_t q = 0; q < P; ++q) {
    std::vector<uint64_t> rc(2 * P), roff(2 * P), unused(2 * P);
    for (uint32_t p = 0; p < P; ++p) {
      rc[2 * p] = sc[p][2 * q];
      rc[2 * p + 1] = sc[p][2 * q + 1];
    }
    uint64_t rtot[2];
    DC_TRY(dc_merge_plan(P, sc[q].data(), rc.data(), unused.data(), roff.data(), rtot));
    const uint64_t rn = rtot[0], rb = rtot[1];
    Buf<uint64_t> rnodes, rbins;
    DC_TRY(alloc(c, rnodes, rn * f.W));
    DC_TRY(alloc(c, rbins, rb * BIN_W));
    for (uint32_t p = 0; p < P; ++p) {  // loopback "send": p's slab for q lands at q's receive offset for p
      if (sc[p][2 * q])
        DC_CUDA(c, cudaMemcpyAsync(rnodes.p + roff[2 * p] * f.W, slabs[p].nodes.p + soff[p][2 * q] * f.W, sc[p][2 * q] * f.W * 8,
                                   cudaMemcpyDeviceToDevice, c->stream));
      if (sc[p][2 * q + 1])
        DC_CUDA(c, cudaMemcpyAsync(rbins.p + roff[2 * p + 1] * BIN_W, slabs[p].bins.p + soff[p][2 * q + 1] * BIN_W,
                                   sc[p][2 * q + 1] * BIN_W * 8, cudaMemcpyDeviceToDevice, c->stream));
    }
    DC_TRY(reduce_received(c, rnodes.p, rn, rbins.p, rb, f, parts_n[q], &pn[q], parts_b[q], &pb[q], coll.p, false));
  }
  uint32_t hcoll = 0;
  DC_TRY(readback(c, coll.p, 4, &hcoll));
  if (hcoll) {
    dc_dict_free(gd);
    c->host_collisions += 1;
    return fail(c, DC_ERR_COLLISION, "merge: 128-bit path hash collision detected");
  }
  uint64_t tn = 0, tb = 0;
  for (uint32_t q = 0; q < P; ++q) {
    tn += pn[q];
    tb += pb[q];
  }
  Buf<uint64_t> allv, allb;
  DC_TRY(alloc(c, allv, tn * f.W));
  DC_TRY(alloc(c, allb, tb * BIN_W));
  uint64_t o = 0, ob = 0;
  for (uint32_t q = 0; q < P; ++q) {
    if (pn[q]) DC_CUDA(c, cudaMemcpyAsync(allv.p + o * f.W, parts_n[q].p, pn[q] * f.W * 8, cudaMemcpyDeviceToDevice, c->stream));
    if (pb[q]) DC_CUDA(c, cudaMemcpyAsync(allb.p + ob * BIN_W, parts_b[q].p, pb[q] * BIN_W * 8, cudaMemcpyDeviceToDevice, c->stream));
    o += pn[q];
    ob += pb[q];
  }
  r3.reset();
  dc_cct* canon = nullptr;
  {
    Region rc(c, "merge:canonicalize");
    DC_TRY(canonicalize(c, allv.p, tn, allb.p, tb, f, (uint32_t)gd->D, &canon));
  }
  if (gd->D) {  // kinds for views
    DC_TRY(palloc(c, canon->frame_kind, gd->D));
    DC_CUDA(c, cudaMemcpyAsync(canon->frame_kind, gd->kinds, gd->D, cudaMemcpyDeviceToDevice, c->stream));
  }
  *out_canonical = canon;
  *out_global_dict = gd;
  return DC_OK;
}

}  // extern "C"
