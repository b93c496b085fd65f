// prim.cuh — device-wide primitives of libdc (own implementations, no CUB on the hot path):
// exclusive scan (reduce-then-scan, 3 phases) and a stable LSD radix sort of
// (u64 key, u32 value) pairs over the significant bit range only.
#pragma once
#include "common.cuh"

namespace dc {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

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

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const T* __restrict__ in, uint64_t n, T* __restrict__ sums) { DC_PDL_ENTER();
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    uint64_t j = base + (uint64_t)i * SCAN_THREADS + threadIdx.x;
    if (j < n) s += in[j];
  }
  T tot;
  block_excl_scan<T, SCAN_THREADS>(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// single-block scan of a medium array (out may equal in): warp w owns the contiguous chunk
// [w*C, (w+1)*C); pass 1 sums the chunks, one warp scans the 32 chunk sums, pass 2 re-reads each
// chunk (L1/L2-resident) and scans it 32 elements at a time with a running carry.
constexpr int SCAN1_THREADS = 1024;
constexpr uint64_t SCAN1_MAX = 1ull << 16;
template <class T>
__global__ void __launch_bounds__(SCAN1_THREADS) k_scan_one(const T* in, T* out, uint64_t n, T* total) { DC_PDL_ENTER();
  __shared__ T wsum[32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t C = (n + 31) / 32;
  const uint64_t lo = w * C, hi = lo + C < n ? lo + C : n;
  T s = 0;
  for (uint64_t j = lo + lane; j < hi; j += 32) s += in[j];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) wsum[w] = s;
  __syncthreads();
  if (w == 0) {
    const T v = wsum[lane];
    const T inc = warp_incl_scan(v);
    wsum[lane] = inc - v;
    if (lane == 31 && total) *total = inc;
  }
  __syncthreads();
  T carry = wsum[w];
  for (uint64_t b = lo; b < hi; b += 32) {
    const uint64_t j = b + lane;
    const T v = j < hi ? in[j] : T(0);
    const T inc = warp_incl_scan(v);
    if (j < hi) out[j] = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// two independent exclusive scans of the same length in one launch (each pass of k_scan_one,
// done for both arrays: their load latencies overlap)
template <class A, class B>
__global__ void __launch_bounds__(SCAN1_THREADS) k_scan_one_pair(const A* ia, A* oa, A* ta, const B* ib, B* ob, B* tb, uint64_t n) { DC_PDL_ENTER();
  __shared__ A wa[32];
  __shared__ B wb[32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t C = (n + 31) / 32;
  const uint64_t lo = w * C, hi = lo + C < n ? lo + C : n;
  A sa = 0;
  B sb = 0;
  for (uint64_t j = lo + lane; j < hi; j += 32) {
    sa += ia[j];
    sb += ib[j];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if (lane == 0) {
    wa[w] = sa;
    wb[w] = sb;
  }
  __syncthreads();
  if (w == 0) {
    const A va = wa[lane];
    const A inca = warp_incl_scan(va);
    wa[lane] = inca - va;
    const B vb = wb[lane];
    const B incb = warp_incl_scan(vb);
    wb[lane] = incb - vb;
    if (lane == 31) {
      if (ta) *ta = inca;
      if (tb) *tb = incb;
    }
  }
  __syncthreads();
  A ca = wa[w];
  B cb = wb[w];
  for (uint64_t b = lo; b < hi; b += 32) {
    const uint64_t j = b + lane;
    const A va = j < hi ? ia[j] : A(0);
    const B vb = j < hi ? ib[j] : B(0);
    const A inca = warp_incl_scan(va);
    const B incb = warp_incl_scan(vb);
    if (j < hi) {
      oa[j] = ca + inca - va;
      ob[j] = cb + incb - vb;
    }
    ca += __shfl_sync(0xffffffffu, inca, 31);
    cb += __shfl_sync(0xffffffffu, incb, 31);
  }
}

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(const T* __restrict__ in, T* out, uint64_t n,
                                                            const T* __restrict__ offs) { DC_PDL_ENTER();
  // each thread owns SCAN_ITEMS consecutive elements of the tile
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  T v[SCAN_ITEMS];
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    uint64_t j = base + i;
    v[i] = j < n ? in[j] : T(0);
    s += v[i];
  }
  T ex = block_excl_scan<T, SCAN_THREADS>(s, nullptr) + offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    uint64_t j = base + i;
    if (j < n) out[j] = ex;
    ex += v[i];
  }
}

template <class T>
dc_status excl_scan(Ctx* c, const T* in, T* out, uint64_t n, T* total_dev);
// two exclusive scans of length n (one launch when n <= SCAN1_MAX)
template <class A, class B>
dc_status excl_scan_pair(Ctx* c, const A* ia, A* oa, A* ta, const B* ib, B* ob, B* tb, uint64_t n) {
  if (n == 0 || n > SCAN1_MAX) {
    DC_TRY(excl_scan<A>(c, ia, oa, n, ta));
    return excl_scan<B>(c, ib, ob, n, tb);
  }
  dc_launch(k_scan_one_pair<A, B>, 1, SCAN1_THREADS, 0, c->stream, ia, oa, ta, ib, ob, tb, n);
  DC_LAUNCHED(c);
  return DC_OK;
}

// out[i] = sum(in[0..i)); total (device) optional. in may equal out.
template <class T>
dc_status excl_scan(Ctx* c, const T* in, T* out, uint64_t n, T* total_dev) {
  if (n == 0) {
    if (total_dev) DC_CUDA(c, cudaMemsetAsync(total_dev, 0, sizeof(T), c->stream));
    return DC_OK;
  }
  uint64_t nt = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (n <= SCAN1_MAX) {  // one launch
    dc_launch(k_scan_one<T>, 1, SCAN1_THREADS, 0, c->stream, in, out, n, total_dev);
    DC_LAUNCHED(c);
    return DC_OK;
  }
  Buf<T> sums;
  DC_TRY(alloc(c, sums, nt));
  dc_launch(k_scan_reduce<T>, (unsigned)nt, SCAN_THREADS, 0, c->stream, in, n, sums.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<T>(c, sums.p, sums.p, nt, total_dev));
  dc_launch(k_scan_down<T>, (unsigned)nt, SCAN_THREADS, 0, c->stream, in, out, n, sums.p);
  DC_LAUNCHED(c);
  return DC_OK;
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
    static bool attr = false;
    if (!attr) {
      DC_CUDA(c, cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmallSortSmem)));
      attr = true;
    }
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
