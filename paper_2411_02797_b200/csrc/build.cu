// build.cu — a2/a3: CCT construction ("constructed by inserting call paths
// ... and collapsing frames that refer to the same locations").
//
// a2 path streaming + exact dedup: one warp per record streams its frames (coalesced),
//    validates them and forms a 64-bit path hash; records are grouped by hash in an L2 hash
//    table whose representative is the smallest record index (atomicMin, deterministic);
//    every record is then compared frame-by-frame with its representative, and a mismatch
//    (hash collision) makes the record a representative of its own — so the dedup is exact.
// a3 level-wise construction over the P distinct representative paths: at depth d each
//    active item has key (parent-local-index << fbits | frame_d); a stable radix sort of the
//    keys and a run-length encoding assign node ids base_{d+1} + run, which is exactly the
//    canonical (depth, lexicographic) order (reading R2). P <= SMALL_P runs entirely inside
//    one CTA (shared memory, no host round trips); larger P runs one kernel sequence per level.
#include "prim.cuh"

namespace dc {

constexpr uint32_t SMALL_P = 4096;
constexpr int SB_THREADS = 1024;

__device__ __forceinline__ int bits_for_dev(uint32_t v) { return v ? 32 - __clz(v) : 0; }

// ------------------------------------------------------------------ a2: hash + dedup
__device__ __forceinline__ uint64_t frame_hash(uint32_t f, uint32_t j) {
  return mix64(((uint64_t)j << 32 | f) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull);
}

__global__ void k_path_hash(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames, uint64_t R,
                            uint32_t n_frames, uint64_t* __restrict__ hash, uint32_t* __restrict__ len, uint32_t* d_flags,
                            unsigned long long* d_diag, uint64_t hash_mask) {
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t maxd = 0, empties = 0, flags = 0;
  for (uint64_t r = warp; r < R; r += nw) {
    uint64_t o0 = off[r], o1 = off[r + 1];
    uint64_t L = o1 >= o0 ? o1 - o0 : 0;
    if (o1 < o0) flags |= FLAG_BAD_OFFSETS;
    if (L > DC_MAX_DEPTH) {
      flags |= FLAG_TOO_DEEP;
      L = DC_MAX_DEPTH;
    }
    uint64_t h = 0;
    for (uint32_t j = lane; j < L; j += 32) {
      uint32_t f = frames[o0 + j];
      if (f >= n_frames) flags |= FLAG_BAD_FRAME;
      h += frame_hash(f, j);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0) {
      h = mix64(h ^ (L * 0xC2B2AE3D27D4EB4Full)) & hash_mask;
      if (h == ~0ull) h = ~1ull;
      hash[r] = h;
      len[r] = (uint32_t)L;
    }
    maxd = max(maxd, (uint32_t)L);
    empties += (L == 0);
  }
  flags = __reduce_or_sync(0xffffffffu, flags);  // a bad frame may be seen by any lane
  if (lane == 0) {
    if (maxd) atomicMax(&d_diag[DG_MAXDEPTH], (unsigned long long)maxd);
    if (empties) atomicAdd(&d_diag[DG_EMPTY], (unsigned long long)empties);
    if (flags) atomicOr(d_flags, flags);
  }
}

__global__ void k_path_insert(const uint64_t* __restrict__ hash, uint64_t R, unsigned long long* htab, uint32_t* rtab,
                              uint64_t mask, uint32_t* __restrict__ slot_of_rec, unsigned int* d_count) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = hash[r];
    uint64_t s = (h * 0x9E3779B97F4A7C15ull >> 17) & mask;
    bool found = false;
    for (uint64_t probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
      unsigned long long cur = ld_relaxed_u64(htab + s);
      if (cur == h) { found = true; break; }
      if (cur == ~0ull) {
        unsigned long long old = atomicCAS(htab + s, ~0ull, (unsigned long long)h);
        if (old == ~0ull) {
          atomicAdd(d_count, 1u);
          found = true;
          break;
        }
        if (old == h) { found = true; break; }
      }
    }
    if (!found) {  // table full: the host retries with a larger table
      atomicOr(d_count + 3, 1u);
      slot_of_rec[r] = 0;
      continue;
    }
    atomicMin(rtab + s, (uint32_t)r);
    slot_of_rec[r] = (uint32_t)s;
  }
}

// exact verification: warp per record against its representative
__global__ void k_path_verify(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                              const uint32_t* __restrict__ len, uint64_t R, const uint32_t* __restrict__ rtab,
                              uint32_t* __restrict__ slot_of_rec, uint32_t* __restrict__ extra_rec, unsigned int* d_extra,
                              uint64_t cap) {
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r = warp; r < R; r += nw) {
    uint32_t s = slot_of_rec[r];
    uint32_t rep = rtab[s];
    if (rep == (uint32_t)r) continue;
    uint32_t L = len[r];
    bool diff = len[rep] != L;
    if (!diff) {
      const uint32_t* a = frames + off[r];
      const uint32_t* b = frames + off[rep];
      for (uint32_t j = lane; j < L; j += 32)
        if (a[j] != b[j]) diff = true;
      diff = __any_sync(0xffffffffu, diff);
    }
    if (diff && lane == 0) {  // collision: r becomes a representative of its own
      unsigned e = atomicAdd(d_extra, 1u);
      extra_rec[e] = (uint32_t)r;
      slot_of_rec[r] = (uint32_t)(cap + e);
    }
  }
}

__global__ void k_path_compact(const unsigned long long* __restrict__ htab, const uint32_t* __restrict__ rtab, uint64_t cap,
                               uint32_t* __restrict__ pid_of_slot, uint32_t* __restrict__ item_rec, unsigned int* d_pos) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    if (htab[s] == ~0ull) continue;
    unsigned p = atomicAdd(d_pos, 1u);
    pid_of_slot[s] = p;
    item_rec[p] = rtab[s];
  }
}

__global__ void k_items_finish(uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ extra_rec, uint32_t P0,
                               uint32_t n_extra, const uint32_t* __restrict__ len, uint32_t* __restrict__ item_len,
                               unsigned long long* d_sumlen) {
  uint32_t P = P0 + n_extra;
  unsigned long long acc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    if (i >= P0) item_rec[i] = extra_rec[i - P0];
    uint32_t L = len[item_rec[i]];
    item_len[i] = L;
    acc += L;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane_id() == 0 && acc) atomicAdd(d_sumlen, acc);
}

__global__ void k_rec_leaf(const uint32_t* __restrict__ slot_of_rec, const uint32_t* __restrict__ pid_of_slot, uint64_t cap,
                           uint32_t P0, const uint32_t* __restrict__ leaf_of_item, uint64_t R, uint32_t* __restrict__ leaf) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = slot_of_rec[r];
    uint32_t item = s < cap ? pid_of_slot[s] : P0 + (uint32_t)(s - cap);
    leaf[r] = leaf_of_item[item];
  }
}

// ------------------------------------------------------------------ a3: small P, one CTA
struct SmallSmem {
  uint64_t key[2][SMALL_P];
  uint32_t val[2][SMALL_P];
  uint32_t node_of_item[SMALL_P];
  uint64_t off_of_item[SMALL_P];
  uint16_t len_of_item[SMALL_P];
  uint32_t wcnt[32][256];
};

// stable block radix sort of n <= SMALL_P pairs held in sm.key[cur]/val[cur]; returns buffer index
__device__ int block_sort(SmallSmem& sm, uint32_t n, int bits, int cur) {
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint32_t per_warp = (n + 31) / 32;  // contiguous chunk per warp
  for (int shift = 0; shift < bits; shift += 8) {
    const int nb = bits - shift < 8 ? bits - shift : 8;
    const uint32_t mask = (1u << nb) - 1u;
    for (int i = threadIdx.x; i < 32 * 256; i += SB_THREADS) (&sm.wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t b0 = w * per_warp, b1 = min(n, b0 + per_warp);
    for (uint32_t base = b0; base < b1; base += 32) {
      uint32_t j = base + lane;
      bool ok = j < b1;
      uint32_t d = ok ? (uint32_t)(sm.key[cur][j] >> shift) & mask : 0xFFFFFFFFu;
      uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (ok && (peers & lanemask_lt()) == 0) sm.wcnt[w][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // digit totals and exclusive prefix (digit-major, then warp)
    uint32_t tot = 0;
    if (threadIdx.x < 256) {
      for (int ww = 0; ww < 32; ++ww) tot += sm.wcnt[ww][threadIdx.x];
    }
    uint32_t ex = block_excl_scan<uint32_t, SB_THREADS>(threadIdx.x < 256 ? tot : 0u, nullptr);
    if (threadIdx.x < 256) {
      uint32_t run = ex;
      for (int ww = 0; ww < 32; ++ww) {
        uint32_t c = sm.wcnt[ww][threadIdx.x];
        sm.wcnt[ww][threadIdx.x] = run;
        run += c;
      }
    }
    __syncthreads();
    for (uint32_t base = b0; base < b1; base += 32) {
      uint32_t j = base + lane;
      bool ok = j < b1;
      uint64_t k = ok ? sm.key[cur][j] : 0;
      uint32_t v = ok ? sm.val[cur][j] : 0;
      uint32_t d = ok ? (uint32_t)(k >> shift) & mask : 0xFFFFFFFFu;
      uint32_t peers = __match_any_sync(0xffffffffu, d);
      uint32_t pos = ok ? sm.wcnt[w][d] + __popc(peers & lanemask_lt()) : 0;
      __syncwarp();
      if (ok && (peers & lanemask_lt()) == 0) sm.wcnt[w][d] += __popc(peers);
      __syncwarp();
      if (ok) {
        sm.key[cur ^ 1][pos] = k;
        sm.val[cur ^ 1][pos] = v;
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

// The whole level loop for P <= SMALL_P distinct paths in one CTA. Per level: keys
// (parent-local << fbits | frame), a sort only when the keys are not already in order (after
// the first branching level most levels are), then one fused pass that run-length encodes
// (node ids, node table), retires finished items and compacts the active list.
__global__ void __launch_bounds__(SB_THREADS, 1) k_build_small(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                                                               const uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ item_len,
                                                               uint32_t P, int fbits, uint32_t* __restrict__ parent,
                                                               uint32_t* __restrict__ frame_out, uint16_t* __restrict__ depth,
                                                               uint32_t* __restrict__ level_off, uint32_t* __restrict__ leaf_of_item,
                                                               uint32_t* d_N) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmallSmem& sm = *reinterpret_cast<SmallSmem*>(smem_raw);
  const uint64_t fmask = (1ull << fbits) - 1ull;
  if (threadIdx.x == 0) {
    parent[0] = DC_NO_NODE;
    frame_out[0] = DC_NO_NODE;
    depth[0] = 0;
    level_off[0] = 0;
    level_off[1] = 1;
  }
  // active items: those with len > 0 (in item order); empty paths -> root
  uint32_t n_active = 0;
  int act = 0;  // buffer holding the active list
  for (uint32_t base = 0; base < P; base += SB_THREADS) {
    uint32_t i = base + threadIdx.x;
    uint32_t L = i < P ? item_len[i] : 0;
    uint32_t keep = (i < P && L > 0) ? 1u : 0u;
    if (i < P) {
      if (!keep) leaf_of_item[i] = 0;
      sm.off_of_item[i] = off[item_rec[i]];
      sm.len_of_item[i] = (uint16_t)L;
      sm.node_of_item[i] = 0;
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan<uint32_t, SB_THREADS>(keep, &tot);
    if (keep) sm.val[0][n_active + ex] = i;
    n_active += tot;
  }
  __syncthreads();
  uint32_t lvl_start = 0, width = 1, next = 1;
  for (uint32_t d = 0; n_active > 0; ++d) {
    const int pbits = bits_for_dev(width - 1);
    for (uint32_t i = threadIdx.x; i < n_active; i += SB_THREADS) {
      const uint32_t it = sm.val[act][i];
      const uint32_t f = frames[sm.off_of_item[it] + d];
      sm.key[act][i] = ((uint64_t)(sm.node_of_item[it] - lvl_start) << fbits) | f;
    }
    __syncthreads();
    bool in_order = true;
    for (uint32_t i = 1 + threadIdx.x; i < n_active; i += SB_THREADS) in_order &= sm.key[act][i - 1] <= sm.key[act][i];
    const int cur = __syncthreads_and(in_order) ? act : block_sort(sm, n_active, pbits + fbits, act);
    // fused: run heads -> node ids; retire items of length d+1; compact the rest into the other buffer
    uint32_t n_keep = 0, n_runs = 0;
    for (uint32_t base = 0; base < n_active; base += SB_THREADS) {
      const uint32_t i = base + threadIdx.x;
      const bool ok = i < n_active;
      const uint64_t k = ok ? sm.key[cur][i] : 0;
      const uint32_t it = ok ? sm.val[cur][i] : 0;
      const uint32_t head = ok && (i == 0 || sm.key[cur][i - 1] != k) ? 1u : 0u;
      const uint32_t keep = ok && sm.len_of_item[it] > d + 1 ? 1u : 0u;
      // one scan for both flags: (head count << 16 | keep count); n_active <= 4096 < 2^16
      uint32_t tot;
      const uint32_t ex = block_excl_scan<uint32_t, SB_THREADS>((head << 16) | keep, &tot);
      if (ok) {
        const uint32_t node = next + n_runs + (ex >> 16) + head - 1;  // inclusive run index - 1
        if (head) {
          parent[node] = lvl_start + (uint32_t)(k >> fbits);
          frame_out[node] = (uint32_t)(k & fmask);
          depth[node] = (uint16_t)(d + 1);
        }
        sm.node_of_item[it] = node;
        if (!keep) leaf_of_item[it] = node;
        else sm.val[cur ^ 1][n_keep + (ex & 0xFFFFu)] = it;
      }
      n_runs += tot >> 16;
      n_keep += tot & 0xFFFFu;
      __syncthreads();
    }
    act = cur ^ 1;
    lvl_start = next;
    width = n_runs;
    next += n_runs;
    if (threadIdx.x == 0) level_off[d + 2] = next;
    n_active = n_keep;
  }
  if (threadIdx.x == 0) *d_N = next;
}

// ------------------------------------------------------------------ a3: large P, per level
__global__ void k_lvl_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                           const uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ active, uint32_t n_active,
                           const uint32_t* __restrict__ node_of_item, uint32_t lvl_start, uint32_t d, int fbits,
                           uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_active; i += gridDim.x * blockDim.x) {
    uint32_t it = active[i];
    uint32_t f = frames[off[item_rec[it]] + d];
    key[i] = ((uint64_t)(node_of_item[it] - lvl_start) << fbits) | f;
    val[i] = it;
  }
}

__global__ void k_lvl_heads(const uint64_t* __restrict__ key, uint32_t n, uint32_t* __restrict__ head) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i - 1] != key[i]) ? 1u : 0u;
}

__global__ void k_lvl_assign(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val, uint32_t n,
                             const uint32_t* __restrict__ run_excl, uint32_t lvl_start, uint32_t next, uint32_t d, int fbits,
                             const uint32_t* __restrict__ item_len, uint32_t* __restrict__ parent, uint32_t* __restrict__ frame_out,
                             uint16_t* __restrict__ depth, uint32_t* __restrict__ node_of_item, uint32_t* __restrict__ leaf_of_item,
                             uint32_t* __restrict__ keep) {
  const uint64_t fmask = (1ull << fbits) - 1ull;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint64_t k = key[i];
    bool head = (i == 0 || key[i - 1] != k);
    // run_excl is the exclusive scan of heads: run index = run_excl[i] + head - 1
    uint32_t node = next + run_excl[i] + (head ? 1u : 0u) - 1u;
    uint32_t it = val[i];
    if (head) {
      parent[node] = lvl_start + (uint32_t)(k >> fbits);
      frame_out[node] = (uint32_t)(k & fmask);
      depth[node] = (uint16_t)(d + 1);
    }
    node_of_item[it] = node;
    uint32_t L = item_len[it];
    if (L == d + 1) leaf_of_item[it] = node;
    keep[i] = L > d + 1 ? 1u : 0u;
  }
}

__global__ void k_lvl_compact(const uint32_t* __restrict__ val, const uint32_t* __restrict__ keep,
                              const uint32_t* __restrict__ keep_excl, uint32_t n, uint32_t* __restrict__ active) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (keep[i]) active[keep_excl[i]] = val[i];
}

__global__ void k_lvl_init(const uint32_t* __restrict__ item_len, uint32_t P, uint32_t* __restrict__ keep,
                           uint32_t* __restrict__ node_of_item, uint32_t* __restrict__ leaf_of_item, uint32_t* __restrict__ idx) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    keep[i] = item_len[i] > 0;
    node_of_item[i] = 0;
    idx[i] = i;
    if (item_len[i] == 0) leaf_of_item[i] = 0;
  }
}

__global__ void k_root(uint32_t* parent, uint32_t* frame_out, uint16_t* depth, uint32_t* level_off) {
  parent[0] = DC_NO_NODE;
  frame_out[0] = DC_NO_NODE;
  depth[0] = 0;
  level_off[0] = 0;
  level_off[1] = 1;
}

static dc_status build_large(Ctx* c, const dc_paths* p, const uint32_t* item_rec, const uint32_t* item_len, uint32_t P,
                             uint32_t Lmax, int fbits, dc_cct* t, uint32_t* leaf_of_item, uint32_t* h_levels,
                             uint64_t* h_N) {
  Buf<uint32_t> keep, keep_ex, active, node_of_item, idx, v0, v1, runs;
  Buf<uint64_t> k0, k1;
  DC_TRY(alloc(c, keep, P));
  DC_TRY(alloc(c, keep_ex, P));
  DC_TRY(alloc(c, active, P));
  DC_TRY(alloc(c, node_of_item, P));
  DC_TRY(alloc(c, idx, P));
  DC_TRY(alloc(c, v0, P));
  DC_TRY(alloc(c, v1, P));
  DC_TRY(alloc(c, runs, P));
  DC_TRY(alloc(c, k0, P));
  DC_TRY(alloc(c, k1, P));
  Buf<uint32_t> tot;
  DC_TRY(alloc(c, tot, 2));
  k_root<<<1, 1, 0, c->stream>>>(t->parent, t->frame, t->depth, t->level_off);
  DC_LAUNCHED(c);
  k_lvl_init<<<grid_for(c, P, 256), 256, 0, c->stream>>>(item_len, P, keep.p, node_of_item.p, leaf_of_item, idx.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint32_t>(c, keep.p, keep_ex.p, P, tot.p));
  k_lvl_compact<<<grid_for(c, P, 256), 256, 0, c->stream>>>(idx.p, keep.p, keep_ex.p, P, active.p);
  DC_LAUNCHED(c);
  uint32_t hn[2];
  DC_TRY(readback(c, tot.p, 4, hn));
  uint32_t n_active = hn[0];
  uint32_t lvl_start = 0, width = 1, next = 1;
  std::vector<uint32_t> lo = {0, 1};
  uint32_t d = 0;
  for (; n_active > 0; ++d) {
    int pbits = bits_for(width - 1);
    k_lvl_keys<<<grid_for(c, n_active, 256), 256, 0, c->stream>>>(p->offsets, p->frames, item_rec, active.p, n_active,
                                                                  node_of_item.p, lvl_start, d, fbits, k0.p, v0.p);
    DC_LAUNCHED(c);
    bool in1 = false;
    DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, n_active, 0, pbits + fbits, &in1));
    uint64_t* ks = in1 ? k1.p : k0.p;
    uint32_t* vs = in1 ? v1.p : v0.p;
    k_lvl_heads<<<grid_for(c, n_active, 256), 256, 0, c->stream>>>(ks, n_active, keep.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, keep.p, runs.p, n_active, tot.p));
    k_lvl_assign<<<grid_for(c, n_active, 256), 256, 0, c->stream>>>(ks, vs, n_active, runs.p, lvl_start, next, d, fbits,
                                                                    item_len, t->parent, t->frame, t->depth,
                                                                    node_of_item.p, leaf_of_item, keep.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, keep.p, keep_ex.p, n_active, tot.p + 1));
    k_lvl_compact<<<grid_for(c, n_active, 256), 256, 0, c->stream>>>(vs, keep.p, keep_ex.p, n_active, active.p);
    DC_LAUNCHED(c);
    DC_TRY(readback(c, tot.p, 8, hn));
    uint32_t n_runs = hn[0];
    lvl_start = next;
    width = n_runs;
    next += n_runs;
    lo.push_back(next);
    n_active = hn[1];
  }
  DC_CUDA(c, cudaMemcpyAsync(t->level_off, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice, c->stream));
  DC_CUDA(c, cudaStreamSynchronize(c->stream));
  *h_levels = d;
  *h_N = next;
  return DC_OK;
}

dc_status cct_build(Ctx* c, const dc_paths* p, const dc_dict* dict, uint32_t n_frames, uint32_t* out_leaf, dc_cct** out) {
  *out = nullptr;
  const uint64_t R = p->n_records;
  if (R >= (1ull << 32)) return fail(c, DC_ERR_CAPACITY, "dc_cct_build: n_records >= 2^32");
  dc_cct* t = new dc_cct();
  t->device = c->device;
  t->R = R;
  t->n_frames = n_frames;
  const int fbits = bits_for(n_frames > 0 ? n_frames - 1 : 0) > 0 ? bits_for(n_frames - 1) : 1;
  if (dict) {
    DC_TRY(palloc(c, t->frame_kind, n_frames));
    DC_CUDA(c, cudaMemcpyAsync(t->frame_kind, dict->kinds, n_frames, cudaMemcpyDeviceToDevice, c->stream));
  }
  // ---- a2: hash, group, verify
  Buf<uint64_t> hash;
  Buf<uint32_t> len, slot_of_rec, rtab, extra_rec, pid_of_slot, item_rec, item_len, leaf_of_item, leafbuf;
  Buf<unsigned long long> htab, sumlen;
  Buf<unsigned int> cnt;
  DC_TRY(alloc(c, hash, R));
  DC_TRY(alloc(c, len, R));
  DC_TRY(alloc(c, slot_of_rec, R));
  k_path_hash<<<grid_for(c, R * 32, 256), 256, 0, c->stream>>>(p->offsets, p->frames, R, n_frames, hash.p, len.p,
                                                                c->d_flags, (unsigned long long*)c->d_diag, c->hash_mask);
  DC_LAUNCHED(c);
  // path table sized for the distinct paths, not the records (retry once if it fills up)
  uint64_t cap = 1024;
  while (cap < 2 * (R < (1ull << 20) ? R : (1ull << 20))) cap <<= 1;
  for (int attempt = 0;; ++attempt) {
    DC_TRY(alloc(c, htab, cap));
    DC_TRY(alloc(c, rtab, cap));
    DC_CUDA(c, cudaMemsetAsync(htab.p, 0xFF, cap * 8, c->stream));
    DC_CUDA(c, cudaMemsetAsync(rtab.p, 0xFF, cap * 4, c->stream));
    DC_TRY(alloc_zero(c, cnt, 4));  // [0] distinct, [1] extra, [2] compact pos, [3] overflow
    k_path_insert<<<grid_for(c, R, 256), 256, 0, c->stream>>>(hash.p, R, htab.p, rtab.p, cap - 1, slot_of_rec.p, cnt.p);
    DC_LAUNCHED(c);
    uint32_t hcnt[4];
    DC_TRY(readback(c, cnt.p, 16, hcnt));
    if (!hcnt[3] && (uint64_t)hcnt[0] * 2 <= cap) break;
    if (attempt || cap >= (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "dc_cct_build: path table overflow");
    cap = 1024;
    while (cap < 2 * R) cap <<= 1;
    if (cap > (1ull << 31)) cap = 1ull << 31;
  }
  DC_TRY(alloc(c, extra_rec, R));
  k_path_verify<<<grid_for(c, R * 32, 256), 256, 0, c->stream>>>(p->offsets, p->frames, len.p, R, rtab.p, slot_of_rec.p,
                                                                  extra_rec.p, cnt.p + 1, cap);
  DC_LAUNCHED(c);
  DC_TRY(alloc(c, pid_of_slot, cap));
  uint32_t hc[4];
  DC_TRY(readback(c, cnt.p, 8, hc));
  const uint32_t P0 = hc[0], n_extra = hc[1], P = P0 + n_extra;
  DC_TRY(alloc(c, item_rec, P));
  DC_TRY(alloc(c, item_len, P));
  DC_TRY(alloc(c, leaf_of_item, P));
  DC_TRY(alloc_zero(c, sumlen, 1));
  k_path_compact<<<grid_for(c, cap, 256), 256, 0, c->stream>>>(htab.p, rtab.p, cap, pid_of_slot.p, item_rec.p, cnt.p + 2);
  DC_LAUNCHED(c);
  k_items_finish<<<grid_for(c, P, 256), 256, 0, c->stream>>>(item_rec.p, extra_rec.p, P0, n_extra, len.p, item_len.p,
                                                             sumlen.p);
  DC_LAUNCHED(c);
  uint64_t hsum = 0, hmaxd = 0;
  DC_TRY(readback(c, sumlen.p, 8, &hsum));
  DC_TRY(readback(c, c->d_diag + DG_MAXDEPTH, 8, &hmaxd));
  DC_TRY(check_flags(c));
  const uint64_t Nbound = 1 + hsum;
  if (Nbound >= (1ull << 32)) return fail(c, DC_ERR_CAPACITY, "dc_cct_build: more than 2^32 nodes");
  // hmaxd is the deepest path seen on this context so far (>= this trace's): sizes level_off
  const uint32_t Lmax = (uint32_t)hmaxd;
  DC_TRY(palloc(c, t->parent, Nbound));
  DC_TRY(palloc(c, t->frame, Nbound));
  DC_TRY(palloc(c, t->depth, Nbound));
  DC_TRY(palloc(c, t->level_off, (uint64_t)Lmax + 2));
  uint64_t N = 0;
  uint32_t levels = 0;
  if (P <= SMALL_P) {
    Buf<uint32_t> dN;
    DC_TRY(alloc(c, dN, 1));
    size_t smem = sizeof(SmallSmem);
    DC_CUDA(c, cudaFuncSetAttribute(k_build_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_build_small<<<1, SB_THREADS, smem, c->stream>>>(p->offsets, p->frames, item_rec.p, item_len.p, P, fbits, t->parent,
                                                      t->frame, t->depth, t->level_off, leaf_of_item.p, dN.p);
    DC_LAUNCHED(c);
    uint32_t hN = 0;
    DC_TRY(readback(c, dN.p, 4, &hN));
    N = hN;
  } else {
    DC_TRY(build_large(c, p, item_rec.p, item_len.p, P, Lmax, fbits, t, leaf_of_item.p, &levels, &N));
  }
  // max depth of this tree
  t->N = N;
  uint32_t* leaf = out_leaf;
  if (!leaf) {
    DC_TRY(alloc(c, leafbuf, R));
    leaf = leafbuf.p;
  }
  k_rec_leaf<<<grid_for(c, R, 256), 256, 0, c->stream>>>(slot_of_rec.p, pid_of_slot.p, cap, P0, leaf_of_item.p, R, leaf);
  DC_LAUNCHED(c);
  // depth of the tree = largest d with a node
  {
    uint16_t md = 0;
    if (N > 1) DC_TRY(readback(c, t->depth + (N - 1), 2, &md));
    t->max_depth = md;
  }
  // node columns (exclusive/inclusive counts), metric columns come with attribute
  DC_TRY(palloc(c, t->xcnt, N));
  DC_TRY(palloc(c, t->icnt, N));
  DC_CUDA(c, cudaMemsetAsync(t->xcnt, 0, N * 8, c->stream));
  DC_CUDA(c, cudaMemsetAsync(t->icnt, 0, N * 8, c->stream));
  // algorithmic bytes: offsets + frames of every record once, leaf, node table
  uint64_t F = 0;
  DC_TRY(readback(c, p->offsets + R, 8, &F));
  c->bytes_host += 8 * (R + 1) + 4 * F + 4 * R + 10 * N;
  c->host_levels += t->max_depth;
  c->host_collisions += n_extra;
  (void)levels;
  t->state = 0;
  *out = t;
  return DC_OK;
}

}  // namespace dc
