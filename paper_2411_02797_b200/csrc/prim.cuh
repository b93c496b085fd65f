// prim.cuh — device-wide primitives of libdc (own implementations, no CUB on the hot path):
// exclusive scan (single pass, decoupled look-back) and a stable LSD radix sort of
// (u64 key, u32 value) pairs over the significant bit range only.
#pragma once
#include "common.cuh"

namespace dc {

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (uint32_t)o) v += u;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns exclusive prefix, *total = block sum
template <class T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_sums[NT / 32];
  T inc = warp_incl_scan(v);
  const int w = threadIdx.x >> 5;
  if (lane_id() == 31) warp_sums[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane_id() < (uint32_t)(NT / 32) ? warp_sums[lane_id()] : T(0);
    T si = warp_incl_scan(s);
    if (lane_id() < (uint32_t)(NT / 32)) warp_sums[lane_id()] = si - s;
  }
  __syncthreads();
  T excl = warp_sums[w] + inc - v;
  if (total) {
    __shared__ T tot;
    if (threadIdx.x == NT - 1) tot = excl + v;
    __syncthreads();
    *total = tot;
  }
  __syncthreads();
  return excl;
}

// ------------------------------------------------------------------ single-pass chained scan
// One launch for any length: tile ids come from a ticket counter (so every earlier tile is
// already running), each tile publishes its aggregate, then one warp looks back over the
// predecessors' (aggregate | inclusive prefix) flags 32 at a time (decoupled look-back). The
// flags carry the call's sequence number, so the context's persistent tile state needs no
// reset between calls. Up to two arrays are scanned by the same tiles (pair scans).
constexpr int CS_THREADS = 256;

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class A, class B, int ITEMS>
__global__ void __launch_bounds__(CS_THREADS) k_scan_chained(const A* ia, A* oa, A* ta, const B* ib, B* ob, B* tb, uint64_t n,
                                                             unsigned long long* ctr, uint64_t ticket_base, uint64_t* flag,
                                                             uint64_t* val, uint64_t seq) { DC_PDL_ENTER();
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_pre[2];
  if (threadIdx.x == 0) s_tile = (uint32_t)(atomicAdd(ctr, 1ull) - ticket_base);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * (CS_THREADS * ITEMS) + (uint64_t)threadIdx.x * ITEMS;
  const bool two = ib != nullptr;
  A va[ITEMS];
  B vb[ITEMS];
  A sa = 0;
  B sb = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t j = base + i;
    va[i] = j < n ? ia[j] : A(0);
    vb[i] = (two && j < n) ? ib[j] : B(0);
    sa += va[i];
    sb += vb[i];
  }
  A tota;
  B totb;
  A exa = block_excl_scan<A, CS_THREADS>(sa, &tota);
  B exb = two ? block_excl_scan<B, CS_THREADS>(sb, &totb) : B(0);
  if (!two) totb = 0;
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint64_t pa = 0, pb = 0;
    if (tile == 0) {
      if (lane == 0) {
        val[2] = (uint64_t)tota;
        val[3] = (uint64_t)totb;
        st_release_u64(flag, (seq << 2) | 2u);
      }
    } else {
      if (lane == 0) {
        val[4ull * tile] = (uint64_t)tota;
        val[4ull * tile + 1] = (uint64_t)totb;
        st_release_u64(flag + tile, (seq << 2) | 1u);
      }
      int64_t j = (int64_t)tile - 1 - (int64_t)lane;
      for (uint64_t spins = 0;;) {
        uint32_t st = 2;  // lanes past tile 0 never matter (tile 0 is inclusive)
        if (j >= 0) {
          const uint64_t f = ld_acquire_u64(flag + j);
          st = (f >> 2) == seq ? (uint32_t)(f & 3u) : 0u;
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, st == 2);
        const int first = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive predecessor
        const uint32_t need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
        if (__ballot_sync(0xffffffffu, st == 0) & need) {  // a needed predecessor has not published
          if (++spins > DC_SPIN_LIMIT) __trap();
          continue;
        }
        uint64_t a = 0, b = 0;
        if ((int)lane <= first && j >= 0) {
          a = __ldcg(val + 4ull * j + (st == 2 ? 2 : 0));
          b = __ldcg(val + 4ull * j + (st == 2 ? 3 : 1));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        pa += a;
        pb += b;
        if (incl) break;
        j -= 32;
      }
      if (lane == 0) {
        val[4ull * tile + 2] = pa + (uint64_t)tota;
        val[4ull * tile + 3] = pb + (uint64_t)totb;
        st_release_u64(flag + tile, (seq << 2) | 2u);
      }
    }
    if (lane == 0) {
      s_pre[0] = pa;
      s_pre[1] = pb;
    }
  }
  __syncthreads();
  A ra = (A)s_pre[0] + exa;
  B rb = (B)s_pre[1] + exb;
  const uint64_t n_tiles = (n + CS_THREADS * ITEMS - 1) / (CS_THREADS * ITEMS);
  if (tile == n_tiles - 1 && threadIdx.x == CS_THREADS - 1) {
    if (ta) *ta = (A)s_pre[0] + exa + sa;
    if (tb) *tb = (B)s_pre[1] + exb + sb;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t j = base + i;
    if (j < n) {
      oa[j] = ra;
      if (two) ob[j] = rb;
    }
    ra += va[i];
    rb += vb[i];
  }
}

// the context's persistent chained-scan tile state (allocated on first use)
dc_status scan_state(Ctx* c, uint64_t n_tiles, uint64_t** flag, uint64_t** val, uint64_t* seq, Buf<uint64_t>& tmp);

template <class A, class B>
dc_status scan_chained(Ctx* c, const A* ia, A* oa, A* ta, const B* ib, B* ob, B* tb, uint64_t n) {
  if (n == 0) {
    if (ta) DC_CUDA(c, cudaMemsetAsync(ta, 0, sizeof(A), c->stream));
    if (tb) DC_CUDA(c, cudaMemsetAsync(tb, 0, sizeof(B), c->stream));
    return DC_OK;
  }
  constexpr int ITEMS = (sizeof(A) == 8 || sizeof(B) == 8) ? 8 : 16;
  const uint64_t nt = (n + CS_THREADS * ITEMS - 1) / (CS_THREADS * ITEMS);
  if (nt >= (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "scan of %llu elements", (unsigned long long)n);
  uint64_t *flag, *val, seq;
  Buf<uint64_t> tmp;
  DC_TRY(scan_state(c, nt, &flag, &val, &seq, tmp));
  const uint64_t base = c->scan_tickets;
  c->scan_tickets += nt;
  dc_launch(k_scan_chained<A, B, ITEMS>, (unsigned)nt, CS_THREADS, 0, c->stream, ia, oa, ta, ib, ob, tb, n, c->scan_ctr, base, flag,
            val, seq);
  DC_LAUNCHED(c);
  return DC_OK;
}

// out[i] = sum(in[0..i)); total (device) optional. in may equal out. One launch.
template <class T>
dc_status excl_scan(Ctx* c, const T* in, T* out, uint64_t n, T* total_dev) {
  return scan_chained<T, T>(c, in, out, total_dev, (const T*)nullptr, (T*)nullptr, (T*)nullptr, n);
}
// two exclusive scans of length n in one launch
template <class A, class B>
dc_status excl_scan_pair(Ctx* c, const A* ia, A* oa, A* ta, const B* ib, B* ob, B* tb, uint64_t n) {
  return scan_chained<A, B>(c, ia, oa, ta, ib, ob, tb, n);
}

// ------------------------------------------------------------------ radix sort (pairs)
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 8;                      // keys per lane
constexpr int RS_WARP_KEYS = 32 * RS_ROUNDS;      // contiguous keys owned by one warp
constexpr int RS_TILE = RS_WARPS * RS_WARP_KEYS;  // 2048

__device__ __forceinline__ uint32_t rs_digit(uint64_t k, int shift, uint32_t mask) {
  return (uint32_t)(k >> shift) & mask;
}

// per-tile digit histogram, digit-major: hist[d * n_tiles + tile]
static __global__ void __launch_bounds__(RS_THREADS) k_rs_count(const uint64_t* __restrict__ keys, uint32_t n, int shift,
                                                         uint32_t mask, uint32_t* __restrict__ hist, uint32_t n_tiles) { DC_PDL_ENTER();
  __shared__ uint32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint32_t base = blockIdx.x * RS_TILE + w * RS_WARP_KEYS;
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    uint32_t j = base + r * 32 + lane;
    bool ok = j < n;
    uint32_t d = ok ? rs_digit(keys[j], shift, mask) : 0xFFFFFFFFu;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (ok && (peers & lanemask_lt()) == 0) atomicAdd(&cnt[d], __popc(peers));
  }
  __syncthreads();
  hist[threadIdx.x * n_tiles + blockIdx.x] = cnt[threadIdx.x];
}

static __global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                           uint64_t* __restrict__ okeys, uint32_t* __restrict__ ovals, uint32_t n,
                                                           int shift, uint32_t mask, const uint32_t* __restrict__ offs,
                                                           uint32_t n_tiles) { DC_PDL_ENTER();
  __shared__ uint32_t wcnt[RS_WARPS][256];
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint32_t base = blockIdx.x * RS_TILE + w * RS_WARP_KEYS;
  uint64_t k[RS_ROUNDS];
  uint32_t v[RS_ROUNDS];
  uint32_t d[RS_ROUNDS];
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    uint32_t j = base + r * 32 + lane;
    bool ok = j < n;
    k[r] = ok ? keys[j] : 0;
    v[r] = ok ? vals[j] : 0;
    d[r] = ok ? rs_digit(k[r], shift, mask) : 0xFFFFFFFFu;
    uint32_t peers = __match_any_sync(0xffffffffu, d[r]);
    if (ok && (peers & lanemask_lt()) == 0) wcnt[w][d[r]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {  // per digit: exclusive prefix over warps + global tile offset
    uint32_t dg = threadIdx.x;
    uint32_t run = offs[dg * n_tiles + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
      uint32_t c = wcnt[ww][dg];
      wcnt[ww][dg] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    uint32_t peers = __match_any_sync(0xffffffffu, d[r]);
    bool ok = d[r] != 0xFFFFFFFFu;
    uint32_t pos = 0;
    if (ok) pos = wcnt[w][d[r]] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (ok && (peers & lanemask_lt()) == 0) wcnt[w][d[r]] += __popc(peers);
    __syncwarp();
    if (ok) {
      okeys[pos] = k[r];
      ovals[pos] = v[r];
    }
  }
}

// Small sorts (n <= SS_MAX): every pass in one 1024-thread CTA in shared memory, one launch.
constexpr int SS_THREADS = 1024;
constexpr uint32_t SS_MAX = 4096;
struct SmallSortSmem {
  uint64_t k[2][SS_MAX];
  uint32_t v[2][SS_MAX];
  uint32_t wcnt[32][256];
};

static __global__ void __launch_bounds__(SS_THREADS, 1) k_sort_small(const uint64_t* __restrict__ ik, const uint32_t* __restrict__ iv,
                                                                  uint64_t* __restrict__ ok, uint32_t* __restrict__ ov, uint32_t n,
                                                                  int begin_bit, int end_bit) { DC_PDL_ENTER();
  extern __shared__ __align__(128) unsigned char ss_raw[];
  SmallSortSmem& sm = *reinterpret_cast<SmallSortSmem*>(ss_raw);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (uint32_t i = tid; i < n; i += SS_THREADS) {
    sm.k[0][i] = ik[i];
    sm.v[0][i] = iv[i];
  }
  __syncthreads();
  int cur = 0;
  const uint32_t per_warp = (n + 31) / 32;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const int nb = end_bit - shift < 8 ? end_bit - shift : 8;
    const uint32_t mask = (1u << nb) - 1u;
    for (int i = tid; i < 32 * 256; i += SS_THREADS) (&sm.wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t b0 = w * per_warp, b1 = min(n, b0 + per_warp);
    for (uint32_t bs = b0; bs < b1; bs += 32) {
      const uint32_t j = bs + lane;
      const bool okk = j < b1;
      const uint32_t d = okk ? (uint32_t)(sm.k[cur][j] >> shift) & mask : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (okk && (peers & lanemask_lt()) == 0) sm.wcnt[w][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    uint32_t tot = 0;
    if (tid < 256)
      for (int ww = 0; ww < 32; ++ww) tot += sm.wcnt[ww][tid];
    const uint32_t ex = block_excl_scan<uint32_t, SS_THREADS>(tid < 256 ? tot : 0u, nullptr);
    if (tid < 256) {
      uint32_t run = ex;
      for (int ww = 0; ww < 32; ++ww) {
        const uint32_t cc = sm.wcnt[ww][tid];
        sm.wcnt[ww][tid] = run;
        run += cc;
      }
    }
    __syncthreads();
    for (uint32_t bs = b0; bs < b1; bs += 32) {
      const uint32_t j = bs + lane;
      const bool okk = j < b1;
      const uint64_t kk = okk ? sm.k[cur][j] : 0;
      const uint32_t vv = okk ? sm.v[cur][j] : 0;
      const uint32_t d = okk ? (uint32_t)(kk >> shift) & mask : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t pos = okk ? sm.wcnt[w][d] + __popc(peers & lanemask_lt()) : 0;
      __syncwarp();
      if (okk && (peers & lanemask_lt()) == 0) sm.wcnt[w][d] += __popc(peers);
      __syncwarp();
      if (okk) {
        sm.k[cur ^ 1][pos] = kk;
        sm.v[cur ^ 1][pos] = vv;
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  for (uint32_t i = tid; i < n; i += SS_THREADS) {
    ok[i] = sm.k[cur][i];
    ov[i] = sm.v[cur][i];
  }
}

// Stable sort of n pairs by bits [begin_bit, end_bit) of the key. Ping-pongs between
// (k0,v0) and (k1,v1); *result_in_1 tells where the sorted data ended up.
static inline dc_status radix_sort_pairs(Ctx* c, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint64_t n,
                                  int begin_bit, int end_bit, bool* result_in_1) {
  *result_in_1 = false;
  if (n <= 1 || end_bit <= begin_bit) return DC_OK;
  if (n <= SS_MAX) {
    DC_SMEM_OPTIN(c, k_sort_small);
    dc_launch(k_sort_small, 1, SS_THREADS, sizeof(SmallSortSmem), c->stream, k0, v0, k1, v1, (uint32_t)n, begin_bit, end_bit);
    DC_LAUNCHED(c);
    *result_in_1 = true;
    return DC_OK;
  }
  if (n >= (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "radix sort of %llu > 2^31 keys", (unsigned long long)n);
  uint32_t nt = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
  Buf<uint32_t> hist;
  DC_TRY(alloc(c, hist, (size_t)256 * nt));
  bool in1 = false;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    int nb = end_bit - shift < 8 ? end_bit - shift : 8;
    uint32_t mask = (1u << nb) - 1u;
    const uint64_t* ik = in1 ? k1 : k0;
    const uint32_t* iv = in1 ? v1 : v0;
    uint64_t* ok = in1 ? k0 : k1;
    uint32_t* ov = in1 ? v0 : v1;
    dc_launch(k_rs_count, nt, RS_THREADS, 0, c->stream, ik, (uint32_t)n, shift, mask, hist.p, nt);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, hist.p, hist.p, (uint64_t)256 * nt, nullptr));
    dc_launch(k_rs_scatter, nt, RS_THREADS, 0, c->stream, ik, iv, ok, ov, (uint32_t)n, shift, mask, hist.p, nt);
    DC_LAUNCHED(c);
    in1 = !in1;
  }
  *result_in_1 = in1;
  return DC_OK;
}

}  // namespace dc
