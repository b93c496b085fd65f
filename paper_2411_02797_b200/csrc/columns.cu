// columns.cu — a4 exclusive attribution, a5 inclusive rollup, a8 derived floats.
//
// a4: record r's metrics go to node leaf[r]: count, sum, min and the
//    128-bit sum of squares, with integer atomics (order-independent, so deterministic).
// a5: incl = excl (+) excl of all descendants. Implemented as the paper
//    states it, in bulk: every node holding exclusive content pushes it to each ancestor on
//    its path to the root (one thread per (node, column group); integer atomics), which
//    needs no per-level barrier — depth-256 trees cost one launch.
// a8: mean/std from the exact integers with single roundings (reading R18).
#include <stdlib.h>

#include <algorithm>

#include "prim.cuh"

namespace dc {

// K > 1 (small trees with many records per node): CTA b updates copy b % K of the columns
// (strides cs / ms), so K times fewer updates meet on one address; k_attr_fold adds the copies
// into the node columns. K = 1 updates the node columns directly.
#ifndef DC_ATTR_U
#define DC_ATTR_U 4
#endif
// U records per thread per round (U = DC_ATTR_U for the direct columns; the K-copy path keeps
// U = 1: config 2 0.110 ms vs 0.123 with 4, its updates meet in a few MB of L2-hot copies), U grid strides apart (every slice stays a coalesced warp
// access): their loads, the min reads and the returned square atomics are issued U at a time, so
// a thread pays each of those latencies once per U records instead of once per record (the
// kernel is bound by them: ncu long-scoreboard stalls 26 per issue on config 4 with U = 1).
// Warp-level pre-aggregation of equal leaves cannot help here: 32 consecutive records of config
// 4 have 32 distinct leaves (config 2: 20.5 on average, and its heavily shared nodes take the K
// column copies instead).
template <int U>
__global__ void k_attribute(const uint32_t* __restrict__ leaf, uint64_t R, const uint64_t* __restrict__ X, uint32_t M,
                            uint64_t ld, uint64_t N, unsigned long long* __restrict__ xcnt0, unsigned long long* __restrict__ mcols0,
                            uint32_t* d_flags, uint32_t K, uint64_t cs, uint64_t ms) { DC_PDL_WAIT();
  unsigned long long* xcnt = xcnt0 + (uint64_t)(blockIdx.x % K) * cs;
  unsigned long long* mcols = mcols0 + (uint64_t)(blockIdx.x % K) * ms;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r0 < R; r0 += U * T) {
    uint32_t n[U];
    bool v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = r0 + u * T < R;
      n[u] = v[u] ? leaf[r0 + u * T] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v[u] && n[u] >= N) {
        atomicOr(d_flags, FLAG_BAD_LEAF);
        v[u] = false;
      }
      if (v[u]) atomicAdd(xcnt + n[u], 1ull);
    }
    for (uint32_t m = 0; m < M; ++m) {
      uint64_t x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = v[u] ? X[m * ld + r0 + u * T] : 0ull;
      unsigned long long* sum = mcols + ((uint64_t)C_XSUM * M + m) * N;
      unsigned long long* mn = mcols + ((uint64_t)C_XMIN * M + m) * N;
      unsigned long long* sql = mcols + ((uint64_t)C_XSQLO * M + m) * N;
      unsigned long long* sqh = mcols + ((uint64_t)C_XSQHI * M + m) * N;
      // min only when x can lower it: after the first few records of a node the plain read
      // (an L2 hit) settles almost every record without an atomic
      uint64_t cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = v[u] ? ld_relaxed_u64(mn + n[u]) : 0ull;
      unsigned long long old[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v[u]) atomicAdd(sum + n[u], (unsigned long long)x[u]);
        old[u] = v[u] ? atomicAdd(sql + n[u], (unsigned long long)(x[u] * x[u])) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v[u] && x[u] < cur[u]) atomicMin(mn + n[u], (unsigned long long)x[u]);
        // 128-bit square: the returned low word tells the carry into the high word
        const uint64_t lo = x[u] * x[u], hi = __umul64hi(x[u], x[u]) + ((old[u] + lo) < old[u] ? 1u : 0u);
        if (v[u] && hi) atomicAdd(sqh + n[u], (unsigned long long)hi);
      }
    }
  }
}

// the K copies: count, then per metric (sum, min, sq_lo, sq_hi); min starts at UINT64_MAX
__global__ void k_attr_init_copies(uint64_t* __restrict__ cnt, uint64_t* __restrict__ cols, uint32_t K, uint32_t M, uint64_t N) { DC_PDL_ENTER();
  const uint64_t MN = (uint64_t)M * N, tot_c = (uint64_t)K * N, tot_m = (uint64_t)K * 4 * MN;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < tot_c + tot_m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < tot_c) {
      cnt[i] = 0;
    } else {
      const uint64_t j = i - tot_c;
      cols[j] = ((j / MN) % 4 == C_XMIN) ? ~0ull : 0ull;
    }
  }
}
// node columns += the K copies (exact: u64 count / sum, min, 128-bit sum of squares)
__global__ void k_attr_fold(const uint64_t* __restrict__ cnt, const uint64_t* __restrict__ cols, uint32_t K, uint32_t M, uint64_t N,
                            uint64_t* __restrict__ xcnt, uint64_t* __restrict__ mcols) { DC_PDL_ENTER();
  const uint64_t MN = (uint64_t)M * N;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N * (1 + M); i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = i / N, n = i - g * N;
    if (g == 0) {
      uint64_t c = 0;
      for (uint32_t k = 0; k < K; ++k) c += cnt[(uint64_t)k * N + n];
      xcnt[n] += c;
      continue;
    }
    const uint64_t m = g - 1;
    uint64_t sum = 0, mn = ~0ull, lo = 0, hi = 0;
    for (uint32_t k = 0; k < K; ++k) {
      const uint64_t* b = cols + (uint64_t)k * 4 * MN;
      sum += b[(uint64_t)C_XSUM * MN + m * N + n];
      mn = min(mn, b[(uint64_t)C_XMIN * MN + m * N + n]);
      const uint64_t l = b[(uint64_t)C_XSQLO * MN + m * N + n];
      const uint64_t t = lo + l;
      hi += b[(uint64_t)C_XSQHI * MN + m * N + n] + (t < lo);
      lo = t;
    }
    mcols[(uint64_t)C_XSUM * MN + m * N + n] += sum;
    uint64_t& xm = mcols[(uint64_t)C_XMIN * MN + m * N + n];
    xm = min(xm, mn);
    uint64_t& ql = mcols[(uint64_t)C_XSQLO * MN + m * N + n];
    uint64_t& qh = mcols[(uint64_t)C_XSQHI * MN + m * N + n];
    const uint64_t nl = ql + lo;
    qh = qh + hi + (nl < lo);
    ql = nl;
  }
}

// all metric columns in one pass: min columns start at UINT64_MAX (reading R11), the rest at 0
__global__ void k_init_cols(uint64_t* __restrict__ mcols, uint32_t M, uint64_t N) { DC_PDL_ENTER();
  const uint64_t total = 8ull * M * N;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t which = i / ((uint64_t)M * N);
    mcols[i] = (which == C_XMIN || which == C_IMIN) ? ~0ull : 0ull;
  }
}

dc_status ensure_metric_cols(Ctx* c, dc_cct* t, uint32_t M) {
  if (t->mcols) {
    if (t->M != M) return fail(c, DC_ERR_ARG, "metric count %u differs from the first call's %u", M, t->M);
    return DC_OK;
  }
  t->M = M;
  const uint64_t N = t->N;
  DC_TRY(palloc(c, t->mcols, (uint64_t)8 * M * N));
  if (M) {
    dc_launch(k_init_cols, grid_for(c, 8ull * M * N, 256), 256, 0, c->stream, t->mcols, M, N);
    DC_LAUNCHED(c);
  }
  return DC_OK;
}

dc_status attribute_metrics(Ctx* c, dc_cct* t, const uint32_t* leaf, uint64_t R, const uint64_t* X, uint32_t M, uint64_t ld) {
  DC_TRY(ensure_metric_cols(c, t, M));
  const uint64_t N = t->N;
  // contention: with many records per node, same-address atomics serialise; spread them over K
  // copies of the columns (a few MB at most) and fold the copies afterwards
  const uint32_t K = (N <= (1u << 16) && R >= 64 * N && !getenv("DC_TEST_ATTR_DIRECT")) ? 16u : 1u;
  if (R && K == 1) {
    dc_launch(k_attribute<DC_ATTR_U>, grid_for(c, R, 256), 256, 0, c->stream, leaf, R, X, M, ld, N, (unsigned long long*)t->xcnt,
                                                            (unsigned long long*)t->mcols, c->d_flags, 1, 0, 0);
    DC_LAUNCHED(c);
  } else if (R) {
    Buf<uint64_t> ccnt, ccols;
    DC_TRY(alloc(c, ccnt, (uint64_t)K * N));
    DC_TRY(alloc(c, ccols, (uint64_t)K * 4 * M * N + 1));
    dc_launch(k_attr_init_copies, grid_for(c, (uint64_t)K * N * (1 + 4 * M), 256), 256, 0, c->stream, ccnt.p, ccols.p, K, M, N);
    DC_LAUNCHED(c);
    dc_launch(k_attribute<1>, grid_for(c, R, 256), 256, 0, c->stream, leaf, R, X, M, ld, N, (unsigned long long*)ccnt.p,
                                                            (unsigned long long*)ccols.p, c->d_flags, K, N, 4ull * M * N);
    DC_LAUNCHED(c);
    dc_launch(k_attr_fold, grid_for(c, N * (1 + M), 256), 256, 0, c->stream, ccnt.p, ccols.p, K, M, N, t->xcnt, t->mcols);
    DC_LAUNCHED(c);
  }
  t->state = 1;
  c->bytes_host += 8ull * M * R + 4 * R + (8 + 32ull * M) * t->N;
  return DC_OK;
}

// --------------------------------------------------------------------------- a5 rollup
// column groups: 0 = count; 1..M = metric m-1 (sum, min, sq); M+1 = samples; M+2+s = stall s
__global__ void k_push(const uint32_t* __restrict__ parent, uint64_t N, uint32_t M, uint32_t S, uint32_t G,
                       const uint64_t* __restrict__ xcnt, unsigned long long* __restrict__ icnt,
                       unsigned long long* __restrict__ mcols, const uint64_t* __restrict__ xsamples,
                       unsigned long long* __restrict__ isamples, const uint64_t* __restrict__ xstall,
                       unsigned long long* __restrict__ istall) { DC_PDL_ENTER();
  const uint64_t total = (N - 1) * (uint64_t)G;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t n = 1 + t / G;
    const uint32_t g = (uint32_t)(t % G);
    if (g == 0) {
      uint64_t v = xcnt[n];
      if (!v) continue;
      // ids strictly decrease towards the root (parent[n] < n), which also bounds the walk
      for (uint32_t a = parent[n], prev = (uint32_t)n; a < prev; prev = a, a = parent[a]) {
        atomicAdd(icnt + a, (unsigned long long)v);
        if (a == 0) break;
      }
    } else if (g <= M) {
      if (!xcnt[n]) continue;
      const uint32_t m = g - 1;
      uint64_t s = mcols[((uint64_t)C_XSUM * M + m) * N + n];
      uint64_t mn = mcols[((uint64_t)C_XMIN * M + m) * N + n];
      uint64_t qlo = mcols[((uint64_t)C_XSQLO * M + m) * N + n];
      uint64_t qhi = mcols[((uint64_t)C_XSQHI * M + m) * N + n];
      // ids strictly decrease towards the root (parent[n] < n), which also bounds the walk
      for (uint32_t a = parent[n], prev = (uint32_t)n; a < prev; prev = a, a = parent[a]) {
        if (s) atomicAdd(mcols + ((uint64_t)C_ISUM * M + m) * N + a, (unsigned long long)s);
        unsigned long long* pm = mcols + ((uint64_t)C_IMIN * M + m) * N + a;
        if (mn < ld_relaxed_u64(pm)) atomicMin(pm, (unsigned long long)mn);
        if (qlo | qhi)
          atomic_add_u128(mcols + ((uint64_t)C_ISQLO * M + m) * N + a, mcols + ((uint64_t)C_ISQHI * M + m) * N + a, qlo, qhi);
        if (a == 0) break;
      }
    } else if (g == M + 1) {
      uint64_t v = xsamples[n];
      if (!v) continue;
      // ids strictly decrease towards the root (parent[n] < n), which also bounds the walk
      for (uint32_t a = parent[n], prev = (uint32_t)n; a < prev; prev = a, a = parent[a]) {
        atomicAdd(isamples + a, (unsigned long long)v);
        if (a == 0) break;
      }
    } else {
      const uint32_t s = g - M - 2;
      uint64_t v = xstall[(uint64_t)s * N + n];
      if (!v) continue;
      // ids strictly decrease towards the root (parent[n] < n), which also bounds the walk
      for (uint32_t a = parent[n], prev = (uint32_t)n; a < prev; prev = a, a = parent[a]) {
        atomicAdd(istall + (uint64_t)s * N + a, (unsigned long long)v);
        if (a == 0) break;
      }
    }
  }
}

// Push without any returned atomic (the variant used for trees that fit the shared-memory
// parent array, N <= PL_MAX_N): the parent array is staged in shared memory, so the ancestor
// walk costs a shared load per step; count / sum / samples / stall are fire-and-forget adds,
// min a fire-and-forget atomicMin, and the u128 square sum is pushed as four 32-bit limbs into
// limb accumulators L[m][k][a] (each < 2^64: at most N < 2^32 contributions of < 2^32), folded
// exactly into the inclusive (sq_lo, sq_hi) by k_push_fold. Every walk step issues and moves on.
constexpr uint32_t PL_MAX_N = 48u << 10;
__global__ void __launch_bounds__(1024) k_push_limbs(const uint32_t* __restrict__ parent, uint64_t N, uint32_t M, uint32_t G,
                                                     const uint64_t* __restrict__ xcnt, unsigned long long* __restrict__ icnt,
                                                     unsigned long long* __restrict__ mcols, unsigned long long* __restrict__ limbs,
                                                     const uint64_t* __restrict__ xsamples, unsigned long long* __restrict__ isamples,
                                                     const uint64_t* __restrict__ xstall, unsigned long long* __restrict__ istall) { DC_PDL_ENTER();
  extern __shared__ uint32_t spar[];
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) spar[i] = parent[i];
  __syncthreads();
  const uint64_t total = (N - 1) * (uint64_t)G;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n = (uint32_t)(1 + t / G);
    const uint32_t g = (uint32_t)(t % G);
    if (g >= 1 && g <= M) {
      if (!xcnt[n]) continue;
      const uint32_t m = g - 1;
      const uint64_t sm = mcols[((uint64_t)C_XSUM * M + m) * N + n];
      const uint64_t mn = mcols[((uint64_t)C_XMIN * M + m) * N + n];
      const uint64_t qlo = mcols[((uint64_t)C_XSQLO * M + m) * N + n];
      const uint64_t qhi = mcols[((uint64_t)C_XSQHI * M + m) * N + n];
      const uint64_t q0 = qlo & 0xFFFFFFFFull, q1 = qlo >> 32, q2 = qhi & 0xFFFFFFFFull, q3 = qhi >> 32;
      unsigned long long* isum = mcols + ((uint64_t)C_ISUM * M + m) * N;
      unsigned long long* imin = mcols + ((uint64_t)C_IMIN * M + m) * N;
      unsigned long long* L = limbs + (uint64_t)m * 4 * N;
      // ids strictly decrease towards the root (parent[n] < n), which also bounds the walk
      for (uint32_t a = spar[n], prev = n; a < prev; prev = a, a = spar[a]) {
        if (sm) atomicAdd(isum + a, (unsigned long long)sm);
        atomicMin(imin + a, (unsigned long long)mn);
        if (q0) atomicAdd(L + a, (unsigned long long)q0);
        if (q1) atomicAdd(L + N + a, (unsigned long long)q1);
        if (q2) atomicAdd(L + 2 * N + a, (unsigned long long)q2);
        if (q3) atomicAdd(L + 3 * N + a, (unsigned long long)q3);
        if (a == 0) break;
      }
      continue;
    }
    unsigned long long* col;
    uint64_t v;
    if (g == 0) {
      col = icnt;
      v = xcnt[n];
    } else if (g == M + 1) {
      col = isamples;
      v = xsamples[n];
    } else {
      const uint32_t st = g - M - 2;
      col = istall + (uint64_t)st * N;
      v = xstall[(uint64_t)st * N + n];
    }
    if (!v) continue;
    for (uint32_t a = spar[n], prev = n; a < prev; prev = a, a = spar[a]) {
      atomicAdd(col + a, (unsigned long long)v);
      if (a == 0) break;
    }
  }
}

// incl sq (u128) += L0 + L1 * 2^32 + L2 * 2^64 + L3 * 2^96, exactly (u192 intermediate)
__global__ void k_push_fold(uint64_t N, uint32_t M, const unsigned long long* __restrict__ limbs,
                            unsigned long long* __restrict__ mcols) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)M * N; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m = i / N, n = i % N;
    const unsigned long long* L = limbs + m * 4 * N;
    const uint64_t l0 = L[n], l1 = L[N + n], l2 = L[2 * N + n], l3 = L[3 * N + n];
    if ((l0 | l1 | l2 | l3) == 0) continue;
    uint64_t* plo = (uint64_t*)mcols + ((uint64_t)C_ISQLO * M + m) * N + n;
    uint64_t* phi = (uint64_t*)mcols + ((uint64_t)C_ISQHI * M + m) * N + n;
    // lo word: existing lo + l0 + (l1 << 32); hi word: existing hi + (l1 >> 32) + l2 + (l3 << 32) + carries
    uint64_t lo = *plo, hi = *phi;
    uint64_t t = lo + l0;
    hi += t < lo ? 1u : 0u;
    lo = t;
    t = lo + (l1 << 32);
    hi += t < lo ? 1u : 0u;
    lo = t;
    hi += (l1 >> 32) + l2 + (l3 << 32);  // the u128 total fits by definition (exact square sums)
    *plo = lo;
    *phi = hi;
  }
}

// Level-synchronous rollup for deep / large trees: one persistent cooperative kernel walks the
// levels bottom-up; every node of level d adds its (final) inclusive values into its parent,
// with a software grid barrier between levels. Siblings are contiguous (canonical order), so a
// warp whose 32 nodes share one parent reduces in registers and issues one update.
struct RollArgs {
  const uint32_t* parent;
  const uint32_t* level_off;
  uint32_t maxd;
  uint64_t N;
  uint32_t M, S, G;
  unsigned long long *icnt, *mcols, *isamples, *istall;
  unsigned int* bar;  // [0] arrivals, [1] generation
};

__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      for (uint64_t spin = 0; *gen == g; ++spin)
        if (spin > DC_SPIN_LIMIT) __trap();
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, (uint64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ void warp_sum_u128(uint64_t& lo, uint64_t& hi) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    const uint64_t t = lo + l2;
    hi += h2 + (t < lo);
    lo = t;
  }
}

// column loads: CG = the one-CTA run of narrow levels (below), where the values were last
// changed by this CTA's own global atomics and only a __syncthreads separates the levels, so
// the loads must not be served from a stale L1 line (relaxed gpu-scope loads go to L2)
template <bool CG>
__device__ __forceinline__ uint64_t rl_ld(const unsigned long long* p) {
  return CG ? ld_relaxed_u64(p) : *p;
}

// one level d of the rollup: items (node of the level, column group) t = tid0, tid0 + nthreads, ...
template <bool CG>
__device__ __forceinline__ void roll_level(const RollArgs& a, uint32_t d, uint64_t tid0, uint64_t nthreads) {
  const uint64_t N = a.N;
  const uint32_t M = a.M, lane = lane_id();
  const uint64_t lo = a.level_off[d], width = a.level_off[d + 1] - lo;
  const uint64_t items = width * a.G;
  const uint64_t rounds = (items + nthreads - 1) / nthreads;
  for (uint64_t k = 0; k < rounds; ++k) {  // warp-uniform trip count (shuffles below)
    const uint64_t t = k * nthreads + tid0;
    const bool act = t < items;
    const uint32_t g = act ? (uint32_t)(t / width) : 0xFFFFFFFFu;
    const uint64_t m = act ? lo + t % width : 0;
    const uint32_t p = act ? a.parent[m] : 0xFFFFFFFFu;
    // every lane takes part in these shuffles (none inside a short-circuit)
    const uint32_t p0 = __shfl_sync(0xffffffffu, p, 0), g0 = __shfl_sync(0xffffffffu, g, 0);
    const bool uni = __all_sync(0xffffffffu, act && p == p0 && g == g0);
    if (g == 0 || (uni && g0 == 0)) {
      uint64_t v = act ? rl_ld<CG>(a.icnt + m) : 0;
      if (uni) v = warp_sum_u64(v);
      if (v && (!uni || lane == 0)) atomicAdd(a.icnt + p, (unsigned long long)v);
    } else if (g <= M) {
      const uint32_t mm = g - 1;
      const uint64_t cnt = rl_ld<CG>(a.icnt + m);
      uint64_t sum = rl_ld<CG>(a.mcols + ((uint64_t)C_ISUM * M + mm) * N + m);
      uint64_t mn = rl_ld<CG>(a.mcols + ((uint64_t)C_IMIN * M + mm) * N + m);
      uint64_t qlo = rl_ld<CG>(a.mcols + ((uint64_t)C_ISQLO * M + mm) * N + m);
      uint64_t qhi = rl_ld<CG>(a.mcols + ((uint64_t)C_ISQHI * M + mm) * N + m);
      if (uni) {
        sum = warp_sum_u64(sum);
        mn = warp_min_u64(mn);
        warp_sum_u128(qlo, qhi);
      }
      const bool any = uni ? __any_sync(0xffffffffu, cnt != 0) : cnt != 0;
      if (any && (!uni || lane == 0)) {
        if (sum) atomicAdd(a.mcols + ((uint64_t)C_ISUM * M + mm) * N + p, (unsigned long long)sum);
        atomicMin(a.mcols + ((uint64_t)C_IMIN * M + mm) * N + p, (unsigned long long)mn);
        if (qlo | qhi)
          atomic_add_u128(a.mcols + ((uint64_t)C_ISQLO * M + mm) * N + p, a.mcols + ((uint64_t)C_ISQHI * M + mm) * N + p, qlo, qhi);
      }
    } else if (act || uni) {
      unsigned long long* col = g == M + 1 ? a.isamples : a.istall + (uint64_t)(g - M - 2) * N;
      uint64_t v = act ? rl_ld<CG>(col + m) : 0;
      if (uni) v = warp_sum_u64(v);
      if (v && (!uni || lane == 0)) atomicAdd(col + p, (unsigned long long)v);
    }
  }
}

// Level-synchronous rollup for deep / large trees: one grid barrier per level. A run of
// consecutive narrow levels (at most RL_NARROW items each: the deep recursion chains of config
// 4) is walked by CTA 0 alone with a block barrier per level and one grid barrier for the run.
#ifndef DC_RL_NARROW
#define DC_RL_NARROW 1024
#endif
constexpr uint64_t RL_NARROW = DC_RL_NARROW;
__global__ void __launch_bounds__(256) k_rollup_levels(RollArgs a) { DC_PDL_ENTER();
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  auto items_of = [&](uint32_t d) -> uint64_t { return (uint64_t)(a.level_off[d + 1] - a.level_off[d]) * a.G; };
  for (uint32_t d = a.maxd; d >= 1;) {
    if (RL_NARROW && items_of(d) <= RL_NARROW) {
      uint32_t e = d;  // the run [e, d] of narrow levels (every CTA computes the same run)
      while (e > 1 && items_of(e - 1) <= RL_NARROW) --e;
      if (blockIdx.x == 0) {
        for (uint32_t dd = d; dd >= e; --dd) {
          roll_level<true>(a, dd, threadIdx.x, blockDim.x);
          __syncthreads();
        }
      }
      grid_barrier(a.bar);
      d = e - 1;
    } else {
      roll_level<false>(a, d, blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nthreads);
      grid_barrier(a.bar);
      --d;
    }
  }
}

// Small trees (N <= RC_MAX_N, configs 1-3, 5): one CTA per inclusive column holds the whole
// column in shared memory and walks the levels bottom-up (children contiguous, level_off gives
// each level's range): every node of level d adds (or min-s) its final value into its parent's
// slot with a shared-memory atomic, one barrier per level. The u128 square sums go as four
// 32-bit limb columns (each sum < 2^32 * N < 2^64, exact), folded by k_roll_fold. Every
// inclusive column is written whole (no copy of the exclusive block first): 2 launches.
// Column c: 0 count; 1 + 6m + {0 sum, 1 min, 2..5 square limb 0..3}; 1 + 6M samples; 2 + 6M + s stall s.
constexpr uint32_t RC_MAX_N = 26u << 10;
#ifndef DC_RC_THREADS
#define DC_RC_THREADS 1024
#endif
constexpr int RC_THREADS = DC_RC_THREADS;  // (A/B builds: 256 / 512)
__global__ void __launch_bounds__(RC_THREADS, 1) k_roll_cols(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ level_off,
                                                            uint32_t maxd, uint32_t N, uint32_t M, const uint64_t* __restrict__ xcnt,
                                                            uint64_t* __restrict__ icnt, uint64_t* __restrict__ mcols,
                                                            uint64_t* __restrict__ limbs, const uint64_t* __restrict__ xsamples,
                                                            uint64_t* __restrict__ isamples, const uint64_t* __restrict__ xstall,
                                                            uint64_t* __restrict__ istall, int use_spar) { DC_PDL_ENTER();
  extern __shared__ unsigned long long racc[];
  // after the column: the level offsets, and the parents as u16 when they fit (use_spar): the
  // level loop then touches no global memory (one barrier per level is its only latency)
  uint32_t* slev = reinterpret_cast<uint32_t*>(racc + N);
  uint16_t* spar = reinterpret_cast<uint16_t*>(slev + ((maxd + 2 + 3) & ~3u));
  const uint32_t col = blockIdx.x, tid = threadIdx.x;
  for (uint32_t i = tid; i < maxd + 2; i += RC_THREADS) slev[i] = level_off[i];
  if (use_spar)
    for (uint32_t i = tid; i < N; i += RC_THREADS) spar[i] = (uint16_t)parent[i];
  const uint64_t* src;
  uint64_t* dst;
  bool is_min = false;
  int limb = -1;
  if (col == 0) {
    src = xcnt;
    dst = icnt;
  } else if (col <= 6 * M) {
    const uint32_t m = (col - 1) / 6, r = (col - 1) % 6;
    if (r == 0) {
      src = mcols + ((uint64_t)C_XSUM * M + m) * N;
      dst = mcols + ((uint64_t)C_ISUM * M + m) * N;
    } else if (r == 1) {
      src = mcols + ((uint64_t)C_XMIN * M + m) * N;
      dst = mcols + ((uint64_t)C_IMIN * M + m) * N;
      is_min = true;
    } else {
      limb = (int)r - 2;
      src = mcols + ((uint64_t)(limb < 2 ? C_XSQLO : C_XSQHI) * M + m) * N;
      dst = limbs + ((uint64_t)m * 4 + limb) * N;
    }
  } else if (col == 6 * M + 1) {
    src = xsamples;
    dst = isamples;
  } else {
    const uint64_t st = col - 6 * M - 2;
    src = xstall + st * N;
    dst = istall + st * N;
  }
  for (uint32_t i = tid; i < N; i += RC_THREADS) {
    uint64_t v = src[i];
    if (limb >= 0) v = (limb & 1) ? v >> 32 : v & 0xFFFFFFFFull;
    racc[i] = v;
  }
  __syncthreads();
  const uint32_t lane = tid & 31;
  for (uint32_t d = maxd; d >= 1; --d) {
    const uint32_t lo = slev[d], hi = slev[d + 1];
    for (uint32_t b0 = lo; b0 < hi; b0 += RC_THREADS) {  // block-uniform trip count (warp shuffles below)
      if (b0 + (tid & ~31u) >= hi) continue;             // warp-uniform: this warp has no node of the level
      const uint32_t n = b0 + tid;
      const bool act = n < hi;
      unsigned long long v = act ? racc[n] : (is_min ? ~0ull : 0ull);
      const uint32_t p = act ? (use_spar ? (uint32_t)spar[n] : __ldg(parent + n)) : 0xFFFFFFFFu;
      // siblings are contiguous: segmented reduction over the lanes with the same parent, then
      // one shared-memory atomic per segment (its last lane)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
        const uint32_t pu = __shfl_up_sync(0xffffffffu, p, o);
        if (lane >= (uint32_t)o && pu == p) v = is_min ? (u < v ? u : v) : v + u;
      }
      const uint32_t pn = __shfl_down_sync(0xffffffffu, p, 1);
      if (act && (lane == 31 || pn != p)) {
        if (is_min) {
          if (v != ~0ull) atomicMin(&racc[p], v);
        } else if (v) {
          atomicAdd(&racc[p], v);
        }
      }
    }
    __syncthreads();
  }
  for (uint32_t i = tid; i < N; i += RC_THREADS) dst[i] = racc[i];
}

// inclusive (sq_lo, sq_hi) = L0 + L1 * 2^32 + L2 * 2^64 + L3 * 2^96 (the u128 total fits)
__global__ void k_roll_fold(uint64_t N, uint32_t M, const uint64_t* __restrict__ limbs, uint64_t* __restrict__ mcols) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)M * N; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m = i / N, n = i % N;
    const uint64_t* L = limbs + m * 4 * N;
    const uint64_t l0 = L[n], l1 = L[N + n], l2 = L[2 * N + n], l3 = L[3 * N + n];
    const uint64_t lo = l0 + (l1 << 32);
    const uint64_t hi = (l1 >> 32) + l2 + (l3 << 32) + (lo < l0 ? 1u : 0u);
    mcols[((uint64_t)C_ISQLO * M + m) * N + n] = lo;
    mcols[((uint64_t)C_ISQHI * M + m) * N + n] = hi;
  }
}

dc_status rollup(Ctx* c, dc_cct* t) {
  const uint64_t N = t->N;
  const uint32_t M = t->M, S = t->S;
  cudaStream_t s = c->stream;
  if (N > 1 && N <= RC_MAX_N && N * 8 + 4ull * (t->max_depth + 6) <= c->smem_optin && !getenv("DC_TEST_ROLLUP_PUSH") && !getenv("DC_TEST_ROLLUP_LEVELS") &&
      !getenv("DC_TEST_ROLLUP_PUSH_RETURNED")) {
    Buf<uint64_t> limbs;
    if (M) DC_TRY(alloc(c, limbs, 4ull * M * N));
    const uint32_t cols = 1 + 6 * M + (t->xsamples ? 1 + S : 0);
    const size_t base = N * 8 + 4ull * ((t->max_depth + 2 + 3) & ~3u);
    const int use_spar = N <= 65535 && base + 2 * N <= c->smem_optin;
    const size_t smem = base + (use_spar ? 2 * N : 0);
    DC_SMEM_OPTIN(c, k_roll_cols);
    dc_launch(k_roll_cols, cols, RC_THREADS, smem, s, t->parent, t->level_off, t->max_depth, (uint32_t)N, M, t->xcnt, t->icnt,
              t->mcols, limbs.p, t->xsamples, t->isamples, t->xstall, t->istall, use_spar);
    DC_LAUNCHED(c);
    if (M) {
      dc_launch(k_roll_fold, grid_for(c, (uint64_t)M * N, 256), 256, 0, s, N, M, limbs.p, t->mcols);
      DC_LAUNCHED(c);
    }
    t->state = 2;
    c->bytes_host += (2 * (8 + 32ull * M) + 4) * N;
    return DC_OK;
  }
  DC_CUDA(c, cudaMemcpyAsync(t->icnt, t->xcnt, N * 8, cudaMemcpyDeviceToDevice, s));
  // the exclusive block [xsum, xmin, xsq_lo, xsq_hi][M][N] is contiguous, and so is the inclusive one
  if (M) DC_CUDA(c, cudaMemcpyAsync(t->col(C_ISUM, 0), t->col(C_XSUM, 0), 4ull * M * N * 8, cudaMemcpyDeviceToDevice, s));
  if (t->xsamples) {
    DC_CUDA(c, cudaMemcpyAsync(t->isamples, t->xsamples, N * 8, cudaMemcpyDeviceToDevice, s));
    DC_CUDA(c, cudaMemcpyAsync(t->istall, t->xstall, (uint64_t)S * N * 8, cudaMemcpyDeviceToDevice, s));
  }
  const uint32_t G = 1 + M + (t->xsamples ? 1 + S : 0);
  // walk cost of the per-node ancestor push ~ N * depth; deep / large trees go level by level
  const bool levels = ((uint64_t)N * t->max_depth > (16ull << 20) || getenv("DC_TEST_ROLLUP_LEVELS")) && !getenv("DC_TEST_ROLLUP_PUSH");
  if (N > 1 && levels) {
    int per_sm = 0;
    DC_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rollup_levels, 256, 0));
    Buf<unsigned int> bar;
    DC_TRY(alloc_zero(c, bar, 2));
    RollArgs ra{t->parent, t->level_off, t->max_depth, N, M, S, G, (unsigned long long*)t->icnt, (unsigned long long*)t->mcols,
                (unsigned long long*)t->isamples, (unsigned long long*)t->istall, bar.p};
    void* args[] = {&ra};
    const int grid = c->num_sms * std::max(1, std::min(per_sm, 4));
    DC_CUDA(c, cudaLaunchCooperativeKernel((void*)k_rollup_levels, grid, 256, args, 0, s));
    DC_LAUNCHED(c);
  } else if (N > 1 && N <= PL_MAX_N && !getenv("DC_TEST_ROLLUP_PUSH_RETURNED")) {
    Buf<unsigned long long> limbs;
    if (M) DC_TRY(alloc_zero(c, limbs, 4ull * M * N));
    const size_t smem = N * 4;
    DC_SMEM_OPTIN(c, k_push_limbs);
    const uint64_t work = (N - 1) * G;
    uint64_t grid = (work + 1023) / 1024;
    if (grid > (uint64_t)c->num_sms) grid = c->num_sms;
    dc_launch(k_push_limbs, (uint32_t)grid, 1024, smem, s, t->parent, N, M, G, t->xcnt, (unsigned long long*)t->icnt,
              (unsigned long long*)t->mcols, limbs.p, t->xsamples, (unsigned long long*)t->isamples, t->xstall,
              (unsigned long long*)t->istall);
    DC_LAUNCHED(c);
    if (M) {
      dc_launch(k_push_fold, grid_for(c, (uint64_t)M * N, 256), 256, 0, s, N, M, limbs.p, (unsigned long long*)t->mcols);
      DC_LAUNCHED(c);
    }
  } else if (N > 1) {
    dc_launch(k_push, grid_for(c, (N - 1) * G, 256, 16), 256, 0, s, t->parent, N, M, S, G, t->xcnt, (unsigned long long*)t->icnt,
                                                             (unsigned long long*)t->mcols, t->xsamples,
                                                             (unsigned long long*)t->isamples, t->xstall,
                                                             (unsigned long long*)t->istall);
    DC_LAUNCHED(c);
  }
  t->state = 2;
  c->bytes_host += (2 * (8 + 32ull * M) + 4) * N;
  return DC_OK;
}

// --------------------------------------------------------------------------- a8 derived
// u192 -> double, round to nearest even: normalise the top 64 bits, fold the rest into a
// sticky bit at bit 0 (below the rounding position), convert with __ull2double_rn, scale.
__device__ double u192_to_double_rn(uint64_t w2, uint64_t w1, uint64_t w0) {
  if (w2) {
    int lz = __clzll(w2);
    uint64_t top = lz ? (w2 << lz) | (w1 >> (64 - lz)) : w2;
    uint64_t rest1 = lz ? (w1 << lz) : w1;
    uint64_t sticky = (rest1 | w0) ? 1u : 0u;
    return scalbn(__ull2double_rn(top | sticky), 128 - lz);
  }
  if (w1) {
    int lz = __clzll(w1);
    uint64_t top = lz ? (w1 << lz) | (w0 >> (64 - lz)) : w1;
    uint64_t sticky = (lz ? (w0 << lz) : w0) ? 1u : 0u;
    return scalbn(__ull2double_rn(top | sticky), 64 - lz);
  }
  return __ull2double_rn(w0);
}

__global__ void k_derived(const uint64_t* __restrict__ cnt, const uint64_t* __restrict__ sum, const uint64_t* __restrict__ sq_lo,
                          const uint64_t* __restrict__ sq_hi, uint64_t N, double* __restrict__ mean, double* __restrict__ stdv) { DC_PDL_ENTER();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t n = cnt[i];
    if (!n) {
      mean[i] = 0.0;
      stdv[i] = 0.0;
      continue;
    }
    uint64_t s = sum[i], ql = sq_lo[i], qh = sq_hi[i];
    double dn = __ull2double_rn(n);
    mean[i] = __ddiv_rn(__ull2double_rn(s), dn);
    // n * (qh:ql) -> 192 bits
    uint64_t p0l = n * ql, p0h = __umul64hi(n, ql);
    uint64_t p1l = n * qh, p1h = __umul64hi(n, qh);
    uint64_t w0 = p0l;
    uint64_t w1 = p0h + p1l;
    uint64_t w2 = p1h + (w1 < p0h ? 1u : 0u);
    // minus s^2 (128 bits)
    uint64_t s2l = s * s, s2h = __umul64hi(s, s);
    uint64_t b0 = w0 < s2l ? 1u : 0u;
    w0 -= s2l;
    uint64_t sub1 = s2h + b0;
    uint64_t b1 = (w1 < sub1 || (b0 && sub1 == 0)) ? 1u : 0u;
    w1 -= sub1;
    w2 -= b1;
    double D = u192_to_double_rn(w2, w1, w0);
    stdv[i] = __ddiv_rn(__dsqrt_rn(D), dn);
  }
}

dc_status derived(Ctx* c, const dc_cct* t, uint32_t metric, int incl, double* mean, double* stdv) {
  if (metric >= t->M) return fail(c, DC_ERR_ARG, "metric %u >= M = %u", metric, t->M);
  if (incl && t->state != 2) return fail(c, DC_ERR_STATE, "inclusive derived values need dc_cct_rollup first");
  const uint64_t* cnt = incl ? t->icnt : t->xcnt;
  dc_launch(k_derived, grid_for(c, t->N, 256), 256, 0, c->stream, cnt, t->col(incl ? C_ISUM : C_XSUM, metric),
                                                           t->col(incl ? C_ISQLO : C_XSQLO, metric),
                                                           t->col(incl ? C_ISQHI : C_XSQHI, metric), t->N, mean, stdv);
  DC_LAUNCHED(c);
  return DC_OK;
}

}  // namespace dc
