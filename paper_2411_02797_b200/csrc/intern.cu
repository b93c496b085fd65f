// intern.cu — a1: frame interning (§4.2 frame identity/unification).
//
// K1 insert: one raw 16-B key per thread (vector load); a per-CTA shared-memory cache of
//    (key -> slot) answers repeated keys (the common case: a few hundred to a few thousand
//    distinct frames among millions of entries); a cache miss probes the open-addressing table
//    of 16-B slots in L2 (read-first, 128-bit atomicCAS only to claim an empty slot). Emits the
//    slot of each key into out_ids (reused as scratch).
// K2 canon: compact the D occupied slots, stable LSD radix sort by (addr) then
//    (kind<<32|str_id) -> lexicographic rank; slot -> rank table.
// K3 remap: out_ids[j] = rank[slot[j]].
#include "prim.cuh"

namespace dc {

static constexpr uint64_t EMPTY = ~0ull;

__device__ __forceinline__ uint64_t key_lo(const dc_frame_key& k) { return (uint64_t)k.kind | ((uint64_t)k.str_id << 32); }

// Per-CTA shared-memory cache of (key -> table slot): traces repeat a few thousand distinct
// frames across millions of entries, so after warm-up almost every key is resolved in shared
// memory and the L2 table is probed only on a cache miss. Entries are claimed with a CAS on
// their slot word (EMPTY -> BUSY), written, then published; they are never evicted.
constexpr int IC_SLOTS = 2048;        // cache entries per CTA (40 KB)
constexpr int IC_PROBE = 8;           // linear probe window
constexpr uint32_t IC_EMPTY = 0xFFFFFFFFu, IC_BUSY = 0xFFFFFFFEu;

__global__ void __launch_bounds__(256) k_intern_insert(const dc_frame_key* __restrict__ keys, uint64_t n, ulonglong2* table,
                                                       uint64_t mask, uint32_t* __restrict__ out_slot,
                                                       unsigned long long* d_count, uint32_t* d_overflow, uint32_t* d_flags,
                                                       unsigned long long* d_max) { DC_PDL_WAIT();
  __shared__ unsigned long long c_lo[IC_SLOTS], c_hi[IC_SLOTS];
  __shared__ uint32_t c_slot[IC_SLOTS];
  for (int i = threadIdx.x; i < IC_SLOTS; i += blockDim.x) c_slot[i] = IC_EMPTY;
  __syncthreads();
  uint64_t mx_addr = 0, mx_ks = 0;  // radix widths of the canonical sort (max addr, max kind<<32|str)
  auto process = [&](uint64_t j, ulonglong2 kv) {
    const uint64_t lo = kv.x, hi = kv.y;                                    // lo = kind | str<<32, hi = addr
    if ((uint32_t)lo == 0xFFFFFFFFu) {
      atomicOr(d_flags, FLAG_BAD_KEY);
      out_slot[j] = 0;
      return;
    }
    mx_addr = max(mx_addr, hi);
    mx_ks = max(mx_ks, (lo << 32) | (lo >> 32));
    const uint64_t h = mix64(lo ^ mix64(hi + 0x9E3779B97F4A7C15ull));
    // ---- shared cache
    const uint32_t c0 = (uint32_t)(h >> 40) & (IC_SLOTS - 1);
    uint32_t found = 0xFFFFFFFFu, claim = IC_EMPTY;
    for (int k = 0; k < IC_PROBE; ++k) {
      const uint32_t e = (c0 + k) & (IC_SLOTS - 1);
      uint32_t v;  // acquire: a published slot word orders the entry's key before it
      asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&c_slot[e])) : "memory");
      if (v == IC_EMPTY) {  // the key is not cached: claim this entry for it (best effort)
        if (atomicCAS(&c_slot[e], IC_EMPTY, IC_BUSY) == IC_EMPTY) claim = e;
        break;
      }
      if (v == IC_BUSY) continue;
      if (c_lo[e] == lo && c_hi[e] == hi) {
        found = v;
        break;
      }
    }
    if (found == 0xFFFFFFFFu) {  // ---- L2 table
      uint64_t s = h & mask;
      for (uint64_t probe = 0; probe <= (mask < 4096 ? mask : 4096); ++probe, s = (s + 1) & mask) {  // bounded: overflow, retried larger
        // past half load the host retries with a larger table anyway: stop walking long runs
        if (probe == 32 && ld_relaxed_u64(d_count) * 2 > mask + 1) break;
        ulonglong2 cur = ld_relaxed_v2(table + s);
        if (cur.x == lo && cur.y == hi && hi != EMPTY) { found = (uint32_t)s; break; }
        bool maybe_partial = ((uint32_t)cur.x == 0xFFFFFFFFu) || cur.y == EMPTY;  // empty, or a torn read of a claim
        if (!maybe_partial) continue;                                          // a different, fully written key
        unsigned __int128 expect = ((unsigned __int128)EMPTY << 64) | EMPTY;
        unsigned __int128 want = ((unsigned __int128)hi << 64) | lo;
        unsigned __int128 old = atomicCAS(reinterpret_cast<unsigned __int128*>(table + s), expect, want);
        if (old == expect) {
          atomicAdd(d_count, 1ull);
          found = (uint32_t)s;
          break;
        }
        if ((uint64_t)old == lo && (uint64_t)(old >> 64) == hi) { found = (uint32_t)s; break; }
      }
      if (found == 0xFFFFFFFFu) {
        atomicOr(d_overflow, 1u);
        found = 0;
      }
    }
    if (claim != IC_EMPTY) {  // publish the cache entry (key first, slot word last)
      c_lo[claim] = lo;
      c_hi[claim] = hi;
      __threadfence_block();
      atomicExch(&c_slot[claim], found);
    }
    out_slot[j] = found;
  };
  // four keys per thread in flight: their 16-B loads are issued before any of them is resolved
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j0 < n; j0 += 4 * stride) {
    ulonglong2 kv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      kv[u] = j0 + u * stride < n ? __ldg(reinterpret_cast<const ulonglong2*>(keys) + j0 + u * stride) : make_ulonglong2(0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u * stride < n) process(j0 + u * stride, kv[u]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx_addr = max(mx_addr, (uint64_t)__shfl_xor_sync(0xffffffffu, mx_addr, o));
    mx_ks = max(mx_ks, (uint64_t)__shfl_xor_sync(0xffffffffu, mx_ks, o));
  }
  if (lane_id() == 0) {
    if (mx_addr) atomicMax(&d_max[0], (unsigned long long)mx_addr);
    if (mx_ks) atomicMax(&d_max[1], (unsigned long long)mx_ks);
  }
}

__global__ void k_intern_compact(const ulonglong2* __restrict__ table, uint64_t cap, uint64_t* __restrict__ addr_key,
                                 uint64_t* __restrict__ ks_key, uint32_t* __restrict__ slot_of, unsigned int* d_pos) { DC_PDL_ENTER();
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    ulonglong2 cur = table[s];
    if ((uint32_t)cur.x == 0xFFFFFFFFu) continue;
    unsigned p = atomicAdd(d_pos, 1u);
    addr_key[p] = cur.y;
    uint32_t kind = (uint32_t)cur.x, str = (uint32_t)(cur.x >> 32);
    ks_key[p] = ((uint64_t)kind << 32) | str;
    slot_of[p] = (uint32_t)s;
  }
}

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t* __restrict__ dst,
                             uint64_t n) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// rank r -> dictionary key; slot -> rank
__global__ void k_intern_rank(const uint32_t* __restrict__ order, const uint32_t* __restrict__ slot_of,
                              const ulonglong2* __restrict__ table, uint32_t* __restrict__ rank_of_slot,
                              dc_frame_key* __restrict__ dict, uint8_t* __restrict__ kinds, uint64_t D) { DC_PDL_ENTER();
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < D; r += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = slot_of[order[r]];
    rank_of_slot[s] = (uint32_t)r;
    ulonglong2 cur = table[s];
    dc_frame_key k;
    k.kind = (uint32_t)cur.x;
    k.str_id = (uint32_t)(cur.x >> 32);
    k.addr = cur.y;
    dict[r] = k;
    kinds[r] = (uint8_t)(k.kind < 255 ? k.kind : 255);
  }
}

// Small dictionaries (D <= IR_MAX_D, every config with raw keys): the rank of each distinct key
// is the number of smaller keys, counted directly — one launch instead of two radix sorts, a
// gather and the rank kernel. CTA: 32 keys (one per lane), its warps split the comparison
// range (broadcast loads), partial counts summed in shared memory. Keys are distinct.
constexpr uint32_t IR_MAX_D = 8192;
constexpr int IR_WARPS = 8;
__global__ void __launch_bounds__(32 * IR_WARPS) k_intern_rank_small(const uint64_t* __restrict__ ka, const uint64_t* __restrict__ kb,
                                                                     const uint32_t* __restrict__ slot_of, const ulonglong2* __restrict__ table,
                                                                     uint32_t* __restrict__ rank_of_slot, dc_frame_key* __restrict__ dict,
                                                                     uint8_t* __restrict__ kinds, uint32_t D,
                                                                     const unsigned long long* d_cnt, const uint32_t* d_ovf,
                                                                     uint64_t cap) { DC_PDL_ENTER();
  __shared__ uint32_t part[IR_WARPS][32];
  if (d_cnt) {  // speculative launch (before the host has read D): D from the device, no-op unless
                // the insert fit (no overflow, at most half load) and D is small enough for this path
    const uint64_t dd = *d_cnt;
    if (*d_ovf || dd * 2 > cap || dd > IR_MAX_D) return;
    D = (uint32_t)dd;
  }
  if (blockIdx.x * 32 >= D) return;  // CTA-uniform
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t i = blockIdx.x * 32 + lane;
  const bool ok = i < D;
  const uint64_t a = ok ? ka[i] : 0, b = ok ? kb[i] : 0;  // (kind << 32 | str_id, addr) order
  const uint32_t per = (D + IR_WARPS - 1) / IR_WARPS, j0 = w * per, j1 = min(D, j0 + per);
  uint32_t r = 0;
#pragma unroll 4
  for (uint32_t j = j0; j < j1; ++j) {
    const uint64_t bj = kb[j], aj = ka[j];
    r += (bj < b) | ((bj == b) & (aj < a));
  }
  part[w][lane] = r;
  __syncthreads();
  if (w == 0 && ok) {
    uint32_t rank = 0;
#pragma unroll
    for (int ww = 0; ww < IR_WARPS; ++ww) rank += part[ww][lane];
    const uint32_t s = slot_of[i];
    rank_of_slot[s] = rank;
    const ulonglong2 cur = table[s];
    dc_frame_key k;
    k.kind = (uint32_t)cur.x;
    k.str_id = (uint32_t)(cur.x >> 32);
    k.addr = cur.y;
    dict[rank] = k;
    kinds[rank] = (uint8_t)(k.kind < 255 ? k.kind : 255);
  }
}

__global__ void k_intern_remap(uint32_t* ids, uint64_t n, const uint32_t* __restrict__ rank_of_slot, const unsigned long long* d_cnt,
                               const uint32_t* d_ovf, uint64_t cap) { DC_PDL_ENTER();
  if (d_cnt) {  // speculative launch: the same guard as k_intern_rank_small
    const uint64_t dd = *d_cnt;
    if (*d_ovf || dd * 2 > cap || dd > IR_MAX_D) return;
  }
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    ids[j] = rank_of_slot[ids[j]];
}

__global__ void k_iota(uint32_t* a, uint64_t n) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void k_kinds_of(const dc_frame_key* __restrict__ dict, uint8_t* kinds, uint64_t D) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < D; i += (uint64_t)gridDim.x * blockDim.x)
    kinds[i] = (uint8_t)(dict[i].kind < 255 ? dict[i].kind : 255);
}

static uint64_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

// d_hint: expected distinct keys (0: unknown; the first table then has 64K slots)
dc_status intern_frames(Ctx* c, const dc_frame_key* keys, uint64_t n, uint32_t* out_ids, dc_dict** out, uint64_t d_hint) {
  dc_dict* d = new dc_dict();
  HandleGuard<dc_dict, dc_dict_free> guard{d};  // frees the dictionary on any error return
  d->device = c->device;
  d->owner_uid = adopt_handle(c);
  *out = nullptr;
  if (n == 0) {
    d->D = 0;
    DC_TRY(palloc(c, d->keys, 1));
    DC_TRY(palloc(c, d->kinds, 1));
    guard.h = nullptr;
    *out = d;
    return DC_OK;
  }
  if (n >= (1ull << 32)) return fail(c, DC_ERR_CAPACITY, "dc_intern_frames: n >= 2^32 keys");
  Buf<ulonglong2> table;
  Buf<unsigned long long> cnt;
  uint64_t mxh[2] = {0, 0};
  // distinct keys are few in practice (hundreds to tens of thousands): start with a 64K-slot table
  // (1 MB to clear and compact) and retry once with a table sized by the keys if it overflows
  uint64_t cap = next_pow2(2 * (n < (1ull << 15) ? n : (1ull << 15)));
  if (d_hint) cap = std::max<uint64_t>(cap, next_pow2(2 * (d_hint < n ? d_hint : n)));
  if (cap < 1024) cap = 1024;
  uint64_t D = 0;
  Buf<uint64_t> ka, kb, ka2;
  Buf<uint32_t> slot_of, ord0, ord1, rank_of_slot;
  bool spec = false;  // compact + small rank + remap enqueued behind the first readback
  for (int attempt = 0; attempt < 2; ++attempt) {
    FillList fl;
    DC_TRY(alloc_fill(c, fl, table, cap, 0xFF));
    DC_TRY(alloc_fill(c, fl, cnt, 5));  // [0] distinct, [1] overflow flag (u32), [2..3] maxima, [4] compact position
    DC_TRY(fill_flush(c, fl));
    unsigned long long* mxp = cnt.p + 2;
    uint32_t* ovp = reinterpret_cast<uint32_t*>(cnt.p + 1);
    {
      Region rk(c, "k:intern_insert");
      // CTAs walk at least ~4k keys each (the shared key cache warms up once per CTA), 2 to 8
      // waves: config 3's 840k keys 30 -> 23 us with 2 waves; large inputs keep 8 waves for
      // latency hiding (config 2's 32M keys: 0.22 ms with 8, 0.35 with 2)
      const uint64_t kw = n / (4096ull * (uint64_t)c->num_sms);
      const int iwaves = kw < 2 ? 2 : kw > 8 ? 8 : (int)kw;
      dc_launch(k_intern_insert, grid_for(c, (n + 3) / 4, 256, iwaves), 256, 0, c->stream, keys, n, table.p, cap - 1, out_ids, cnt.p, ovp,
                                                                   c->d_flags, mxp);
      DC_LAUNCHED(c);
    }
    uint64_t h[2] = {0, 0};
    spec = attempt == 0 && !getenv("DC_TEST_INTERN_RADIX");
    if (spec) {
      // Speculative small path: the host reads (D, overflow, maxima) behind an event while the
      // device goes on with the compaction, the small rank and the remap, which read D on the
      // device and do nothing unless the table held the keys at most half full and D <= IR_MAX_D
      // (then the host takes the retry / radix path below; the dictionary is sized IR_MAX_D).
      DC_TRY(readback_begin(c, {{cnt.p, 8, &h[0]}, {ovp, 4, &h[1]}, {mxp, 16, mxh}}));
      DC_TRY(alloc(c, ka, cap));
      DC_TRY(alloc(c, kb, cap));
      DC_TRY(alloc(c, slot_of, cap));
      DC_TRY(alloc(c, rank_of_slot, cap));
      dc_launch(k_intern_compact, grid_for(c, cap, 256), 256, 0, c->stream, table.p, cap, ka.p, kb.p, slot_of.p,
                reinterpret_cast<unsigned int*>(cnt.p + 4));
      DC_LAUNCHED(c);
      DC_TRY(palloc(c, d->keys, IR_MAX_D));
      DC_TRY(palloc(c, d->kinds, IR_MAX_D));
      dc_launch(k_intern_rank_small, (uint32_t)(IR_MAX_D / 32), 32 * IR_WARPS, 0, c->stream, ka.p, kb.p, slot_of.p, table.p,
                rank_of_slot.p, d->keys, d->kinds, (uint32_t)0, (const unsigned long long*)cnt.p, (const uint32_t*)ovp, cap);
      DC_LAUNCHED(c);
      dc_launch(k_intern_remap, grid_for(c, n, 256), 256, 0, c->stream, out_ids, n, rank_of_slot.p, (const unsigned long long*)cnt.p,
                (const uint32_t*)ovp, cap);
      DC_LAUNCHED(c);
      DC_TRY(readback_end(c));
    } else {
      DC_TRY(readback_multi(c, {{cnt.p, 8, &h[0]}, {ovp, 4, &h[1]}, {mxp, 16, mxh}}));
    }
    D = h[0];
    bool overflow = (uint32_t)h[1] != 0;
    if (!overflow && D * 2 <= cap) break;
    if (attempt == 1) return fail(c, DC_ERR_CAPACITY, "dc_intern_frames: hash table overflow");
    if (spec) {  // the speculative kernels did nothing: drop their dictionary arrays
      cudaFreeAsync(d->keys, c->stream);
      cudaFreeAsync(d->kinds, c->stream);
      d->keys = nullptr;
      d->kinds = nullptr;
      spec = false;
    }
    cap = next_pow2(2 * n);
    if (cap < 1024) cap = 1024;
  }
  d->D = D;
  if (spec && D <= IR_MAX_D) {  // the speculative small path was right: everything is enqueued
    c->bytes_host += 20 * n + 16 * D;
    guard.h = nullptr;
    *out = d;
    return DC_OK;
  }
  if (spec) {  // D > IR_MAX_D: keys / slots are compacted already; the dictionary is resized below
    cudaFreeAsync(d->keys, c->stream);
    cudaFreeAsync(d->kinds, c->stream);
    d->keys = nullptr;
    d->kinds = nullptr;
  } else {
    DC_TRY(alloc(c, ka, D));
    DC_TRY(alloc(c, kb, D));
    DC_TRY(alloc(c, slot_of, D));
    DC_TRY(alloc(c, rank_of_slot, cap));
    dc_launch(k_intern_compact, grid_for(c, cap, 256), 256, 0, c->stream, table.p, cap, ka.p, kb.p, slot_of.p,
              reinterpret_cast<unsigned int*>(cnt.p + 4));
    DC_LAUNCHED(c);
  }
  DC_TRY(alloc(c, ka2, D));
  DC_TRY(alloc(c, ord0, D));
  DC_TRY(alloc(c, ord1, D));
  if (D <= IR_MAX_D && !spec && !getenv("DC_TEST_INTERN_RADIX")) {  // small D after a retry
    DC_TRY(palloc(c, d->keys, D));
    DC_TRY(palloc(c, d->kinds, D));
    dc_launch(k_intern_rank_small, (uint32_t)((D + 31) / 32), 32 * IR_WARPS, 0, c->stream, ka.p, kb.p, slot_of.p, table.p,
              rank_of_slot.p, d->keys, d->kinds, (uint32_t)D, (const unsigned long long*)nullptr, (const uint32_t*)nullptr,
              (uint64_t)0);
    DC_LAUNCHED(c);
    dc_launch(k_intern_remap, grid_for(c, n, 256), 256, 0, c->stream, out_ids, n, rank_of_slot.p,
              (const unsigned long long*)nullptr, (const uint32_t*)nullptr, (uint64_t)0);
    DC_LAUNCHED(c);
    c->bytes_host += 20 * n + 16 * D;
    guard.h = nullptr;
    *out = d;
    return DC_OK;
  }
  dc_launch(k_iota, grid_for(c, D, 256), 256, 0, c->stream, ord0.p, D);
  DC_LAUNCHED(c);
  // LSD: by addr, then (stable) by kind<<32|str  ==> lexicographic (kind, str_id, addr)
  bool in1 = false;
  DC_TRY(radix_sort_pairs(c, ka.p, ord0.p, ka2.p, ord1.p, D, 0, bits_for(mxh[0]), &in1));
  uint32_t* ord = in1 ? ord1.p : ord0.p;
  uint32_t* ord_alt = in1 ? ord0.p : ord1.p;
  dc_launch(k_gather_u64, grid_for(c, D, 256), 256, 0, c->stream, kb.p, ord, ka.p, D);  // ka <- kb[ord]
  DC_LAUNCHED(c);
  bool in1b = false;
  DC_TRY(radix_sort_pairs(c, ka.p, ord, ka2.p, ord_alt, D, 0, bits_for(mxh[1]), &in1b));
  uint32_t* final_ord = in1b ? ord_alt : ord;
  DC_TRY(palloc(c, d->keys, D));
  DC_TRY(palloc(c, d->kinds, D));
  dc_launch(k_intern_rank, grid_for(c, D, 256), 256, 0, c->stream, final_ord, slot_of.p, table.p, rank_of_slot.p, d->keys,
                                                            d->kinds, D);
  DC_LAUNCHED(c);
  dc_launch(k_intern_remap, grid_for(c, n, 256), 256, 0, c->stream, out_ids, n, rank_of_slot.p,
            (const unsigned long long*)nullptr, (const uint32_t*)nullptr, (uint64_t)0);
  DC_LAUNCHED(c);
  c->bytes_host += 20 * n + 16 * D;
  guard.h = nullptr;
  *out = d;
  return DC_OK;
}

dc_status dict_from_sorted(Ctx* c, const dc_frame_key* keys, uint64_t D, dc_dict** out) {
  dc_dict* d = new dc_dict();
  HandleGuard<dc_dict, dc_dict_free> guard{d};
  d->device = c->device;
  d->owner_uid = adopt_handle(c);
  d->D = D;
  DC_TRY(palloc(c, d->keys, D));
  DC_TRY(palloc(c, d->kinds, D));
  if (D) {
    DC_TRY(dcopy(c, d->keys, keys, D * sizeof(dc_frame_key)));
    dc_launch(k_kinds_of, grid_for(c, D, 256), 256, 0, c->stream, d->keys, d->kinds, D);
    DC_LAUNCHED(c);
  }
  guard.h = nullptr;
  *out = d;
  return DC_OK;
}

}  // namespace dc
