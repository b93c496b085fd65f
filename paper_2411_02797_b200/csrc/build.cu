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
#include <stdlib.h>

#include <algorithm>

#include "prim.cuh"

namespace dc {

constexpr uint32_t SMALL_P = 4096;
constexpr int SB_THREADS = 512;            // 512 measured best for the level loop (1024: 110 us, 256: 117 us on config 3)
constexpr int SB_WARPS = SB_THREADS / 32;

__device__ __forceinline__ int bits_for_dev(uint32_t v) { return v ? 32 - __clz(v) : 0; }

// ------------------------------------------------------------------ a2: path streaming + exact dedup
// Two passes over the records:
//  1. k_path_hash streams the frames once: tiles of PT_T consecutive records, whose frames are
//     one contiguous range, are staged in shared memory with TMA bulk copies (cp.async.bulk +
//     mbarrier, double-buffered: the copy of the next tile is in flight while this one is
//     hashed) together with the tile's offsets. Each record is cut into chunks of PT_CH frames
//     (odd, so the chunks a warp works on start in different shared-memory banks); a thread per
//     chunk accumulates the position-keyed sum f*A[j] (one 32x32+64-bit multiply-add per frame)
//     and adds its two 32-bit halves to its record with native shared atomics. Output: one
//     64-bit hash per record (its length mixed in); frame ids and offsets are validated.
//  2. k_path_group: lane i of a warp inserts / finds record r0+i's hash in an L2-resident table
//     whose slot names a representative record (the first inserter) with its frame offset and
//     length; then the warp compares each record with its representative, 32 frames at a time
//     (coalesced on both sides). A mismatch (a hash collision) makes the record a
//     representative of its own, so the dedup is exact whatever the hash.
constexpr int PT_T = 128;           // records per tile (96 with a 24 KB window: 13.4 ms vs 11.0 on config 4)
#ifndef DC_PT_THREADS
#define DC_PT_THREADS 256
#endif
constexpr int PT_THREADS = DC_PT_THREADS;
constexpr int PT_WARPS = PT_THREADS / 32;
constexpr int PT_RPW = PT_T / PT_WARPS;  // records per warp (16)
#ifndef DC_PT_ST
#define DC_PT_ST 2
#endif
#ifndef DC_PT_FW
#define DC_PT_FW 8192
#endif
constexpr int PT_ST = DC_PT_ST;     // k_path_hash stages (tiles in flight per CTA)
constexpr uint32_t PT_FW = DC_PT_FW;  // staged frame window per stage (32 KB)
// chunk length (odd: bank spread). The same for staged and global tiles: the high half of the
// hash sums each chunk's high word, so the hash of a path is a function of its frames and of
// the chunk boundaries — different chunkings would give one path two hashes (two items).
#ifndef DC_PT_CH
#define DC_PT_CH 17
#endif
constexpr uint32_t PT_CH = DC_PT_CH;
constexpr uint32_t PT_NONE = 0xFFFFFFFFu;
constexpr int PG_U = 4;             // k_path_group: records verified per round (per-record verify)
#ifndef DC_PG_W
#define DC_PG_W 8
#endif
#ifndef DC_PG_MINB
#define DC_PG_MINB 4
#endif
constexpr int PG_W = DC_PG_W;       // k_path_group: 32-frame windows per round (sweep verify)

struct __align__(32) PathSlot {
  unsigned long long key;  // record hash, ~0 = empty
  unsigned long long off;  // representative: first frame, length, record index (rep written last)
  uint32_t len, rep;
  // (first frame << 11) | length, one 64-bit word (~0 until published): readers spin on it with
  // relaxed gpu-scope loads and need no acquire (an acquire load invalidates the SM's L1, where
  // the representatives' frames are cached for the verify)
  unsigned long long offlen;
};

struct PathWarp {  // per warp: its 16 records of the tile
  unsigned long long o[PT_RPW];
  uint32_t L[PT_RPW];
  uint32_t cs[PT_RPW + 1];  // chunk starts (exclusive scan), cs[16] = chunks
  uint32_t h1[PT_RPW], h2[PT_RPW];
};

struct PathSmem {
  uint32_t fr[PT_ST][PT_FW];
  unsigned long long offs[PT_ST][PT_T + 2];
  uint32_t pos[DC_MAX_DEPTH];
  unsigned long long full[PT_ST];
  unsigned long long meta_f0[PT_ST], meta_f1[PT_ST];
  uint32_t meta_mode[PT_ST];
  PathWarp wp[PT_WARPS];
};

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {  // read-once data: no L1 allocation
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// one warp's chunks: lane takes chunks lane, lane+32, ...; its record by a 4-step search of the
// warp's chunk starts
template <bool STAGED>
__device__ __forceinline__ void pt_hash_chunks(PathWarp& W, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ src,
                                               uint64_t base, uint32_t n_chunks, uint32_t n_frames, uint32_t& bad) {
  constexpr uint32_t CH = PT_CH;
  for (uint32_t ci = lane_id(); ci < n_chunks; ci += 32) {
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1)  // largest record whose chunk start <= ci (PT_RPW <= 32)
      if (k + step < PT_RPW && W.cs[k + step] <= ci) k += step;
    const uint32_t j0 = (ci - W.cs[k]) * CH;
    const uint32_t j1 = min(j0 + CH, W.L[k]);
    const uint32_t* q = src + (W.o[k] - base);
    unsigned long long acc = 0;  // sum of f * A[j]: one 32x32+64 multiply-add per frame
    uint32_t mx = 0;
#pragma unroll 4
    for (uint32_t j = j0; j < j1; ++j) {
      const uint32_t f = STAGED ? q[j] : ld_stream_u32(q + j);
      acc += (unsigned long long)f * pos[j];
      mx = max(mx, f);
    }
    if (j1 > j0 && mx >= n_frames) bad = 1;
    atomicAdd(&W.h1[k], (uint32_t)acc);  // two native 32-bit adds (a deterministic function of
    atomicAdd(&W.h2[k], (uint32_t)(acc >> 32));  // the path: chunking depends only on positions)
  }
}

__global__ void __launch_bounds__(PT_THREADS) k_path_hash(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                                                          uint64_t R, uint32_t n_frames, uint64_t* __restrict__ hash,
                                                          unsigned int* __restrict__ d_cnt, uint32_t* d_flags,
                                                          unsigned long long* d_diag, uint64_t hash_mask, int tma_ok) { DC_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PathSmem& sm = *reinterpret_cast<PathSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  PathWarp& W = sm.wp[w];
  const uint64_t n_tiles = (R + PT_T - 1) / PT_T, G = gridDim.x;
  for (uint32_t j = tid; j < DC_MAX_DEPTH; j += PT_THREADS) {
    const uint64_t m = mix64(0x9E3779B97F4A7C15ull * (j + 1));
    sm.pos[j] = (uint32_t)(m >> 32) | 0x80000001u;
  }
  if (tid == 0) {
    for (int j = 0; j < PT_ST; ++j) mbar_init(&sm.full[j], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t flags = 0, maxd = 0, empties = 0;
  const uint64_t Ftot = off[R];
  // ---- producer (thread 0): stage tile t into buffer s; F0/F1 = first/end frame of the tile
  auto issue = [&](uint64_t t, int s, uint64_t F0, uint64_t F1) {
    const uint64_t r0 = t * PT_T;
    uint32_t mode = 0, bytes = 0;
    const uint64_t a = F0 & ~3ull, b = (F1 + 3) & ~3ull;
    if (tma_ok && F1 >= F0 && b - a <= PT_FW && b <= Ftot) {
      mode |= 1;
      bytes += (uint32_t)(b - a) * 4u;
    }
    if (tma_ok && r0 + PT_T + 2 <= R + 1) {
      mode |= 2;
      bytes += (PT_T + 2) * 8u;
    }
    sm.meta_f0[s] = F0;
    sm.meta_f1[s] = F1;
    sm.meta_mode[s] = mode;
    if (bytes) {
      mbar_expect_tx(&sm.full[s], bytes);
      if ((mode & 1) && b > a) tma_bulk_g2s(sm.fr[s], frames + a, (uint32_t)(b - a) * 4u, &sm.full[s]);
      if (mode & 2) tma_bulk_g2s(sm.offs[s], off + r0, (PT_T + 2) * 8u, &sm.full[s]);
    } else {
      mbar_arrive(&sm.full[s]);
    }
  };
  // tiles t, t + G, ... of this CTA go round PT_ST stages: tile k + PT_ST - 1 is issued at the
  // top of iteration k into the stage that iteration k - 1 released (its closing barrier)
  uint64_t t = blockIdx.x, nf0 = 0, nf1 = 0;
  if (tid == 0) {
    for (int j = 0; j < PT_ST - 1; ++j) {
      const uint64_t tj = t + (uint64_t)j * G;
      if (tj < n_tiles) issue(tj, j, off[tj * PT_T], off[min(R, tj * PT_T + PT_T)]);
    }
    const uint64_t tn = t + (uint64_t)(PT_ST - 1) * G;
    if (tn < n_tiles) {
      nf0 = off[tn * PT_T];
      nf1 = off[min(R, tn * PT_T + PT_T)];
    }
  }
  for (uint32_t k = 0; t < n_tiles; ++k, t += G) {
    const int s = (int)(k % PT_ST);
    if (tid == 0) {
      const uint64_t ti = t + (uint64_t)(PT_ST - 1) * G;
      if (ti < n_tiles) issue(ti, (int)((k + PT_ST - 1) % PT_ST), nf0, nf1);  // offsets loaded one tile ago
      const uint64_t t2 = t + (uint64_t)PT_ST * G;
      if (t2 < n_tiles) {
        nf0 = off[t2 * PT_T];
        nf1 = off[min(R, t2 * PT_T + PT_T)];
      }
    }
    mbar_wait(&sm.full[s], (k / PT_ST) & 1u);
    const uint64_t r0 = t * PT_T;
    const uint32_t n = (uint32_t)min((uint64_t)PT_T, R - r0);
    const uint32_t mode = sm.meta_mode[s];
    const bool staged = mode & 1;
    const uint64_t F0 = sm.meta_f0[s], F1 = sm.meta_f1[s];
    const uint32_t ch = PT_CH;
    // ---- this warp's records: bounds, length, chunk starts (warp scan); no block barrier
    const uint32_t i = w * PT_RPW + lane;  // tile-local record of lanes 0..15
    const bool mine = lane < PT_RPW && i < n;
    uint32_t c = 0, L = 0;
    uint64_t o = 0;
    if (mine) {
      uint64_t o0, o1;
      if (mode & 2) {
        o0 = sm.offs[s][i];
        o1 = sm.offs[s][i + 1];
      } else {
        o0 = off[r0 + i];
        o1 = off[r0 + i + 1];
      }
      uint64_t LL = o1 >= o0 ? o1 - o0 : 0;
      if (o1 < o0) flags |= FLAG_BAD_OFFSETS;
      if (LL > DC_MAX_DEPTH) {
        flags |= FLAG_TOO_DEEP;
        LL = DC_MAX_DEPTH;
      }
      // frames outside the staged window / the array: malformed offsets (never read)
      if (LL && (staged ? (o0 < F0 || o0 + LL > F1) : (o0 + LL > Ftot))) {
        flags |= FLAG_BAD_OFFSETS;
        LL = 0;
      }
      o = o0;
      L = (uint32_t)LL;
      c = (L + ch - 1) / ch;
      maxd = max(maxd, L);
      empties += L == 0;
    }
    const uint32_t incl = warp_incl_scan<uint32_t>(c);
    const uint32_t n_chunks = __shfl_sync(0xffffffffu, incl, 31);
    if (lane < PT_RPW) {
      W.o[lane] = o;
      W.L[lane] = L;
      W.cs[lane] = incl - c;
      W.h1[lane] = 0;
      W.h2[lane] = 0;
      if (lane == PT_RPW - 1) W.cs[PT_RPW] = incl;
    }
    __syncwarp();
    uint32_t bad = 0;
    if (staged) pt_hash_chunks<true>(W, sm.pos, sm.fr[s], F0 & ~3ull, n_chunks, n_frames, bad);
    else pt_hash_chunks<false>(W, sm.pos, frames, 0, n_chunks, n_frames, bad);
    if (bad) flags |= FLAG_BAD_FRAME;
    __syncwarp();
    if (mine) {
      uint64_t H = mix64(((uint64_t)W.h1[lane] << 32 | W.h2[lane]) ^ ((uint64_t)L * 0xC2B2AE3D27D4EB4Full)) & hash_mask;
      if (H == ~0ull) H = ~1ull;
      hash[r0 + i] = H;
    }
    __syncthreads();  // stage s is free for the copy issued next iteration
  }
  // ---- diag / flags, one atomic per warp
  flags = __reduce_or_sync(0xffffffffu, flags);
  maxd = __reduce_max_sync(0xffffffffu, maxd);
  empties = __reduce_add_sync(0xffffffffu, empties);
  if (lane == 0) {
    if (maxd) atomicMax(&d_diag[DG_MAXDEPTH], (unsigned long long)maxd);
    if (empties) atomicAdd(d_cnt + 4, empties);  // added to the diag once (k_items_finish)
    if (flags) atomicOr(d_flags, flags);
  }
}

// lane i: record r0 + i into the table; then the warp verifies each record against its
// representative frame by frame
constexpr uint64_t PG_SKIP = 0x8000000000000000ull;  // k_path_group sweep: rank not verified
#ifndef DC_PG_BM
#define DC_PG_BM 1
#endif
template <bool SWEEP>
__global__ void __launch_bounds__(256, DC_PG_MINB) k_path_group(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                                                    const uint64_t* __restrict__ hash, uint64_t R, PathSlot* __restrict__ tab,
                                                    uint64_t mask, uint32_t* __restrict__ slot_of_rec,
                                                    uint32_t* __restrict__ extra_rec, unsigned int* __restrict__ d_cnt) { DC_PDL_WAIT();
  __shared__ unsigned long long s_delta[8][32];  // per warp (256 threads): rep start - own start by nonempty rank
  const uint32_t lane = lane_id();
  unsigned long long* const sdelta = s_delta[(threadIdx.x >> 5) & 7];
#if DC_PG_BM
  // per warp: bitmap of the 32 records' start positions over their frame span (<= 32 * 1024
  // frames), so a window's start mask is one shared load instead of a warp OR-reduction
  __shared__ uint32_t s_bm[SWEEP ? 8 : 1][SWEEP ? DC_MAX_DEPTH : 1];
  uint32_t* const sbm = s_bm[SWEEP ? (threadIdx.x >> 5) & 7 : 0];
  if (SWEEP) {
    for (uint32_t i = lane; i < DC_MAX_DEPTH; i += 32) sbm[i] = 0;
    __syncwarp();
  }
#endif
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t r0 = warp * 32; r0 < R; r0 += nw * 32) {
    const uint64_t r = r0 + lane;
    const bool act = r < R;
    uint64_t o = 0, ro = 0, o1 = 0;
    uint32_t L = 0, sl = PT_NONE, need = 0;
    bool mine = false;
    if (act) {
      o = off[r];
      o1 = off[r + 1];
      L = (uint32_t)(o1 >= o ? min(o1 - o, (uint64_t)DC_MAX_DEPTH) : 0);  // validated by k_path_hash
      const uint64_t H = hash[r];
      uint64_t q = (H * 0x9E3779B97F4A7C15ull >> 17) & mask;
      for (uint64_t probe = 0; probe <= (mask < 4096 ? mask : 4096); ++probe, q = (q + 1) & mask) {  // bounded: a long run = overflow, retried larger
        const unsigned long long cur = ld_relaxed_u64(&tab[q].key);
        if (cur == H) {
          sl = (uint32_t)q;
          break;
        }
        if (cur == ~0ull) {
          const unsigned long long old = atomicCAS(&tab[q].key, ~0ull, (unsigned long long)H);
          if (old == ~0ull) {
            sl = (uint32_t)q;
            mine = true;
            break;
          }
          if (old == H) {
            sl = (uint32_t)q;
            break;
          }
        }
      }
      if (mine) {
        tab[sl].off = o;
        tab[sl].len = L;
        st_release_u32(&tab[sl].rep, (uint32_t)r);
        *(volatile unsigned long long*)&tab[sl].offlen = (o << 11) | L;  // o < 2^40, L <= 1024
        const unsigned ins = atomicAdd(d_cnt, 1u);
        if ((uint64_t)ins * 2 >= mask) atomicOr(d_cnt + 3, 1u);  // past half load: retry larger
      }
      if (sl == PT_NONE) atomicOr(d_cnt + 3, 1u);  // table full
    }
    __syncwarp();  // this warp's representatives are published
    if (act && sl != PT_NONE && !mine) {
      unsigned long long w;
      for (uint64_t spin = 0; (w = ld_relaxed_u64(&tab[sl].offlen)) == ~0ull; ++spin)
        if (spin > DC_SPIN_LIMIT) __trap();
      ro = w >> 11;
      const uint32_t rl = (uint32_t)(w & 0x7FFu);
      need = rl != L ? 2u : (L ? 1u : 0u);
    }
    uint32_t todo = __ballot_sync(0xffffffffu, need == 1u);
    // Sweep verify: the 32 records' frames are one contiguous range [Fb, Fe) (checked: every
    // record ends where the next begins, no clamped length). The warp walks it in aligned
    // 32-frame windows, one frame per lane (own frames: one 128-B line per load); a lane finds
    // its frame's record by the rank of the nonempty record starts up to its position (warp OR of
    // the starts falling in the window, popc), reads that record's rep - own delta from shared
    // memory and compares the frame with the representative's frame at the same position.
    if (SWEEP && todo && __all_sync(0xffffffffu, !act || o1 == o + L)) {
      const bool nz = act && L > 0;
      const uint32_t NZ = __ballot_sync(0xffffffffu, nz);
      const uint32_t rk = __popc(NZ & lanemask_lt());
      if (nz) sdelta[rk] = need == 1u ? ro - o : PG_SKIP;
      __syncwarp();
      const uint64_t Fb = __shfl_sync(0xffffffffu, o, 0);
      const uint32_t last = 31 - __clz(__ballot_sync(0xffffffffu, act));
      const uint32_t span = (uint32_t)(__shfl_sync(0xffffffffu, o + L, last) - Fb);  // <= 32 * DC_MAX_DEPTH
      const uint32_t orel = (uint32_t)(o - Fb);
      const uint32_t* const own = frames + Fb;
      const uint32_t le = lanemask_lt() | (1u << lane);
      uint32_t before = 0, badm = 0;
#if DC_PG_BM
      if (nz) atomicOr(&sbm[orel >> 5], 1u << (orel & 31u));
      __syncwarp();
#endif
      // PG_W windows per round: every window's rank and delta first, then all loads, then the
      // compares (the own frames' DRAM latency is paid once per round, not once per window)
      for (uint32_t wb0 = 0; wb0 < span; wb0 += 32 * PG_W) {
        uint32_t cr[PG_W], a[PG_W], b[PG_W];
        uint64_t dd[PG_W];
#pragma unroll
        for (int u = 0; u < PG_W; ++u) {
          const uint32_t wb = wb0 + 32 * u;
#if DC_PG_BM
          const uint32_t M = wb < span ? sbm[wb >> 5] : 0u;
#else
          const uint32_t sr = orel - wb;  // record start relative to the window (wraps if before)
          const uint32_t M = __reduce_or_sync(0xffffffffu, nz && sr < 32u ? 1u << sr : 0u);
#endif
          cr[u] = before + __popc(M & le) - 1;  // rank of my frame's record (nonempty starts at or before it, - 1)
          before += __popc(M);
          dd[u] = wb + lane < span ? sdelta[cr[u] & 31] : PG_SKIP;
        }
#pragma unroll
        for (int u = 0; u < PG_W; ++u) {
          const uint32_t pr = wb0 + 32 * u + lane;
          const bool v = dd[u] != PG_SKIP;
          a[u] = v ? ld_stream_u32(own + pr) : 0u;
          b[u] = v ? __ldg(own + pr + dd[u]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < PG_W; ++u)
          if (a[u] != b[u]) badm |= 1u << (cr[u] & 31);
      }
#if DC_PG_BM
      __syncwarp();
      if (nz) sbm[orel >> 5] = 0u;  // the next group starts from a clear bitmap
#endif
      badm = __reduce_or_sync(0xffffffffu, badm);
      if (nz && need == 1u && ((badm >> rk) & 1u)) need = 2u;
      __syncwarp();  // sdelta reused by the next group
      todo = 0;
    }
    // verify, PG_U records at a time: their first 64 frames on both sides are loaded before any
    // compare, so the DRAM latency of the own frames is paid once per group
    while (todo) {
      int idx[PG_U];
      uint64_t oo[PG_U], rr[PG_U];
      uint32_t ll[PG_U];
#pragma unroll
      for (int u = 0; u < PG_U; ++u) {
        idx[u] = todo ? __ffs(todo) - 1 : -1;
        if (todo) todo &= todo - 1;
        const int i = idx[u] < 0 ? 0 : idx[u];
        oo[u] = __shfl_sync(0xffffffffu, o, i);
        rr[u] = __shfl_sync(0xffffffffu, ro, i);
        const uint32_t li = __shfl_sync(0xffffffffu, L, i);
        ll[u] = idx[u] < 0 ? 0u : li;
      }
      uint32_t a0[PG_U], b0[PG_U], a1[PG_U], b1[PG_U];
#pragma unroll
      for (int u = 0; u < PG_U; ++u) {
        const bool p0 = lane < ll[u], p1 = lane + 32 < ll[u];
        a0[u] = p0 ? ld_stream_u32(frames + oo[u] + lane) : 0u;
        b0[u] = p0 ? __ldg(frames + rr[u] + lane) : 0u;
        a1[u] = p1 ? ld_stream_u32(frames + oo[u] + lane + 32) : 0u;
        b1[u] = p1 ? __ldg(frames + rr[u] + lane + 32) : 0u;
      }
#pragma unroll
      for (int u = 0; u < PG_U; ++u) {
        bool diff = (a0[u] != b0[u]) | (a1[u] != b1[u]);
        for (uint32_t j = lane + 64; j < ll[u]; j += 32) diff |= ld_stream_u32(frames + oo[u] + j) != __ldg(frames + rr[u] + j);
        if (__any_sync(0xffffffffu, diff) && lane == (uint32_t)idx[u]) need = 2u;
      }
    }
    if (act) {
      uint32_t out = sl;
      if (need == 2u) {  // collision: a representative of its own
        const unsigned e = atomicAdd(d_cnt + 1, 1u);
        extra_rec[e] = (uint32_t)r;
        const uint64_t v = mask + 1 + (uint64_t)e;
        if (v >= PT_NONE) atomicOr(d_cnt + 3, 2u);
        out = (uint32_t)v;
      }
      if (out == PT_NONE) out = 0;  // overflow: the host retries
      slot_of_rec[r] = out;
    }
  }
}

// representatives in table-slot order: item ids, their record and path length
__global__ void k_path_compact(const PathSlot* __restrict__ tab, uint64_t cap, uint32_t* __restrict__ pid_of_slot,
                               uint32_t* __restrict__ item_rec, uint32_t* __restrict__ item_len, unsigned int* d_pos) { DC_PDL_ENTER();
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    if (tab[s].key == ~0ull) continue;
    unsigned p = atomicAdd(d_pos, 1u);
    pid_of_slot[s] = p;
    item_rec[p] = tab[s].rep;
    item_len[p] = tab[s].len;
  }
}

// P0 (table items) and n_extra (collision extras) are the device counters of k_path_group, so
// this runs before the host has read them; after a table overflow (d_cnt[3]) the attempt is
// discarded by the host and nothing is added to the diagnostics
__global__ void k_items_finish(uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ extra_rec,
                               const uint64_t* __restrict__ off, uint32_t* __restrict__ item_len,
                               unsigned long long* d_sumlen, const unsigned int* d_cnt, unsigned long long* d_diag) { DC_PDL_ENTER();
  if (d_cnt[3]) return;
  const uint32_t P0 = d_cnt[0], n_extra = d_cnt[1];
  uint32_t P = P0 + n_extra;
  if (blockIdx.x == 0 && threadIdx.x == 0 && d_cnt[4]) atomicAdd(&d_diag[DG_EMPTY], (unsigned long long)d_cnt[4]);
  unsigned long long acc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    if (i >= P0) {  // collision extras: length from the offsets (validated by k_paths)
      const uint32_t r = extra_rec[i - P0];
      item_rec[i] = r;
      const uint64_t o0 = off[r], o1 = off[r + 1];
      item_len[i] = (uint32_t)(o1 >= o0 ? min(o1 - o0, (uint64_t)DC_MAX_DEPTH) : 0);
    }
    acc += item_len[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane_id() == 0 && acc) atomicAdd(d_sumlen, acc);
}

// slot -> leaf node (one L2-resident map), then one gather per record, 4 records per thread
__global__ void k_slot_leaf(const PathSlot* __restrict__ tab, uint64_t cap, const uint32_t* __restrict__ pid_of_slot,
                            const uint32_t* __restrict__ leaf_of_item, uint32_t* __restrict__ leaf_of_slot) { DC_PDL_ENTER();
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x)
    leaf_of_slot[s] = tab[s].key == ~0ull ? 0u : leaf_of_item[pid_of_slot[s]];
}

__global__ void k_rec_leaf(const uint32_t* __restrict__ slot_of_rec, const uint32_t* __restrict__ leaf_of_slot, uint64_t cap,
                           uint32_t P0, const uint32_t* __restrict__ leaf_of_item, uint64_t R, uint32_t* __restrict__ leaf) { DC_PDL_WAIT();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto map = [&](uint32_t sl) { return sl < cap ? leaf_of_slot[sl] : leaf_of_item[P0 + (uint32_t)(sl - cap)]; };
  if ((((uintptr_t)slot_of_rec | (uintptr_t)leaf) & 15u) == 0) {
    // 16-B aligned: 4 consecutive records per thread and 2 such groups per round (one 16-B load
    // and one 16-B store per group, 8 L2 gathers in flight), then the tail
    const uint64_t R4 = R / 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(slot_of_rec);
    uint4* l4 = reinterpret_cast<uint4*>(leaf);
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < R4; q += 2 * stride) {
      const bool two = q + stride < R4;
      const uint4 a = s4[q];
      const uint4 b = two ? s4[q + stride] : make_uint4(0, 0, 0, 0);
      const uint4 la = make_uint4(map(a.x), map(a.y), map(a.z), map(a.w));
      uint4 lb = make_uint4(0, 0, 0, 0);
      if (two) lb = make_uint4(map(b.x), map(b.y), map(b.z), map(b.w));
      l4[q] = la;
      if (two) l4[q + stride] = lb;
    }
    for (uint64_t r = 4 * R4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += stride) leaf[r] = map(slot_of_rec[r]);
    return;
  }
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R; r += 4 * stride) {
    uint32_t s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = r + u * stride < R ? slot_of_rec[r + u * stride] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r + u * stride < R) leaf[r + u * stride] = s[u] < cap ? leaf_of_slot[s[u]] : leaf_of_item[P0 + (uint32_t)(s[u] - cap)];
  }
}

// ------------------------------------------------------------------ a3: small P, one CTA
struct SmallSmem {
  uint64_t key[2][SMALL_P];
  uint32_t val[2][SMALL_P];
  uint32_t node_of_item[SMALL_P];
  uint64_t off_of_item[SMALL_P];
  uint16_t len_of_item[SMALL_P];
  uint32_t next_frame[SMALL_P];  // frame d of each active item, prefetched during level d-1
  uint32_t wcnt[SB_WARPS][256];
};

// stable block radix sort of n <= SMALL_P pairs held in sm.key[cur]/val[cur]; returns buffer index
__device__ int block_sort(SmallSmem& sm, uint32_t n, int bits, int cur) {
  const uint32_t w = threadIdx.x >> 5, lane = lane_id();
  const uint32_t per_warp = (n + SB_WARPS - 1) / SB_WARPS;  // contiguous chunk per warp
  for (int shift = 0; shift < bits; shift += 8) {
    const int nb = bits - shift < 8 ? bits - shift : 8;
    const uint32_t mask = (1u << nb) - 1u;
    for (int i = threadIdx.x; i < SB_WARPS * 256; i += SB_THREADS) (&sm.wcnt[0][0])[i] = 0;
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
      for (int ww = 0; ww < SB_WARPS; ++ww) tot += sm.wcnt[ww][threadIdx.x];
    }
    uint32_t ex = block_excl_scan<uint32_t, SB_THREADS>(threadIdx.x < 256 ? tot : 0u, nullptr);
    if (threadIdx.x < 256) {
      uint32_t run = ex;
      for (int ww = 0; ww < SB_WARPS; ++ww) {
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
                                                               uint32_t* d_N) { DC_PDL_ENTER();
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
  uint32_t lvl_start = 0, width = 1, next = 1, d = 0;
  for (uint32_t i = threadIdx.x; i < n_active; i += SB_THREADS) {
    const uint32_t it = sm.val[0][i];
    sm.next_frame[it] = frames[sm.off_of_item[it]];
  }
  __syncthreads();
  for (; n_active > 0; ++d) {
    const int pbits = bits_for_dev(width - 1);
    // this level's frames come from shared memory; the next level's are loaded now and land
    // while the level is sorted and numbered (the global-load latency leaves the level loop)
    constexpr int PF = SMALL_P / SB_THREADS;
    uint32_t pf_it[PF], pf_f[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const uint32_t i = threadIdx.x + u * SB_THREADS;
      pf_it[u] = DC_NO_NODE;
      if (i < n_active) {
        const uint32_t it = sm.val[act][i];
        const uint32_t f = sm.next_frame[it];
        sm.key[act][i] = ((uint64_t)(sm.node_of_item[it] - lvl_start) << fbits) | f;
        if (sm.len_of_item[it] > d + 1) {
          pf_it[u] = it;
          pf_f[u] = frames[sm.off_of_item[it] + d + 1];
        }
      }
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
#pragma unroll
    for (int u = 0; u < PF; ++u)
      if (pf_it[u] != DC_NO_NODE) sm.next_frame[pf_it[u]] = pf_f[u];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    d_N[0] = next;
    d_N[1] = d;  // levels built = depth of the tree
  }
}

// ------------------------------------------------------------------ a3: small P, no level loop
// The canonical order is the lexicographic order of the prefixes: node (depth d) ids follow
// (parent id, frame), so by induction the depth-d nodes are the distinct d-prefixes in lex
// order. Sorting the P distinct paths lexicographically therefore orders every level at once:
// with the paths sorted and LCP[k] = lcp(path[k-1], path[k]), sorted path k creates exactly the
// nodes of depths LCP[k]+1 .. len[k] (a shorter path cannot sit between two paths sharing a
// d-prefix, because the paths with a given prefix are contiguous in lex order), so
//   level_off[d] = 1 + sum_k max(0, min(len_k, d-1) - LCP_k),
//   id(k, d)     = level_off[d] + #{k' <= k : LCP_k' < d <= len_k'} - 1,
// and the parent of (k, d) is (k, d-1) by the same count at depth d-1. Two launches replace
// the one-CTA level loop (k_build_small): a rank kernel (all pairwise path comparisons, the
// paths staged in shared memory in 16-B chunks; LCP with the predecessor = the largest LCP over
// the smaller paths) and one CTA per depth that numbers and writes that level.
constexpr int SR_THREADS = 512;
constexpr uint32_t SR_WARPS = SR_THREADS / 32;
__device__ __forceinline__ void sr_block_sum_max(uint32_t& sum, uint32_t& mx) {
  __shared__ uint32_t s_sum[SR_THREADS / 32], s_max[SR_THREADS / 32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  sum = __reduce_add_sync(0xffffffffu, sum);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    s_sum[w] = sum;
    s_max[w] = mx;
  }
  __syncthreads();
  sum = 0;
  mx = 0;
  for (int i = 0; i < SR_THREADS / 32; ++i) {
    sum += s_sum[i];
    mx = max(mx, s_max[i]);
  }
  __syncthreads();
}

// Speculative small-P build (launched behind the record pass's readback, before the host knows
// P): the gate decides on the device exactly what the host decides after the readback (same
// integer conditions), and k_small_rank / k_small_emit do nothing when it says no.
struct SmallSpec {
  uint32_t ok, P, Lmax, pad;
};
constexpr uint64_t SPEC_NODES = 57857;  // node arrays of a speculative build: 1 + hsum fits the rank smem
__device__ __host__ inline bool small_spec_ok(uint32_t overflow, uint32_t flags, uint64_t P, uint64_t hsum, uint64_t Lmax,
                                              uint64_t smem_optin) {
  const uint64_t rank_smem = ((16ull * P + 15) & ~15ull) + 4ull * (hsum + 3ull * P);
  return !overflow && !flags && P <= SMALL_P && rank_smem + 1024 <= smem_optin && Lmax <= DC_MAX_DEPTH && 1 + hsum <= SPEC_NODES;
}
__global__ void k_small_gate(const unsigned int* __restrict__ cnt, const unsigned long long* __restrict__ sumlen,
                             const unsigned long long* __restrict__ maxd, const uint32_t* __restrict__ flags, uint64_t smem_optin,
                             SmallSpec* __restrict__ spec) { DC_PDL_ENTER();
  if (threadIdx.x == 0) {
    const uint32_t P = cnt[0] + cnt[1];
    const uint64_t Lmax = *maxd;
    spec->ok = small_spec_ok(cnt[3], *flags, P, *sumlen, Lmax, smem_optin) ? 1u : 0u;
    spec->P = P;
    spec->Lmax = (uint32_t)(Lmax < DC_MAX_DEPTH ? Lmax : DC_MAX_DEPTH);
  }
}

__global__ void __launch_bounds__(SR_THREADS, 1) k_small_rank(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                                                               const uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ item_len,
                                                               uint32_t P, uint32_t* __restrict__ sorted_item, uint32_t* __restrict__ lcp_s,
                                                               uint32_t* __restrict__ len_s, uint64_t* __restrict__ po_s,
                                                               uint32_t* __restrict__ leaf_of_item, const SmallSpec* spec) { DC_PDL_ENTER();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (spec) {  // speculative launch: P from the gate, nothing to do unless it said yes
    if (!spec->ok) return;
    P = spec->P;
  }
  if (blockIdx.x * SR_WARPS >= (P ? P : 1u)) return;  // CTA-uniform: no item for this CTA's warps
  uint64_t* spo = reinterpret_cast<uint64_t*>(smem_raw);     // [P] first frame of path i (global)
  uint32_t* sstart = reinterpret_cast<uint32_t*>(spo + P);   // [P] first 16-B chunk of path i
  uint32_t* slen = sstart + P;                               // [P]
  uint4* chunks = reinterpret_cast<uint4*>(smem_raw + ((16ull * P + 15) & ~15ull));
  uint32_t* fr = reinterpret_cast<uint32_t*>(chunks);
  // chunk starts: exclusive scan of ceil(len / 4); path offsets (loads of all items in flight)
  uint32_t run = 0;
  for (uint32_t base = 0; base < P; base += SR_THREADS) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t L = i < P ? item_len[i] : 0u;
    if (i < P) spo[i] = off[item_rec[i]];
    uint32_t tot;
    const uint32_t ex = block_excl_scan<uint32_t, SR_THREADS>((L + 3) / 4, &tot);
    if (i < P) {
      sstart[i] = run + ex;
      slen[i] = L;
    }
    run += tot;
  }
  __syncthreads();
  // stage the frames, one 16-B chunk per thread and step (the path found by binary search over
  // the chunk starts); 4 chunks per thread in flight. The pad of a last chunk is never compared.
  const uint32_t C = run;
  for (uint32_t q0 = threadIdx.x; q0 < C; q0 += 4 * SR_THREADS) {
    uint4 v[4];
    uint32_t qq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t q = q0 + u * SR_THREADS;
      qq[u] = q;
      v[u] = make_uint4(0, 0, 0, 0);
      if (q < C) {
        uint32_t lo = 0, hi = P;  // last i with sstart[i] <= q (an empty path shares its start)
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (sstart[mid] <= q) lo = mid;
          else hi = mid;
        }
        const uint32_t m = 4 * (q - sstart[lo]), L = slen[lo];
        const uint32_t* src = frames + spo[lo] + m;
        v[u].x = src[0];
        if (m + 1 < L) v[u].y = src[1];
        if (m + 2 < L) v[u].z = src[2];
        if (m + 3 < L) v[u].w = src[3];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (qq[u] < C) chunks[qq[u]] = v[u];
  }
  __syncthreads();
  // one warp per item: its lanes compare it with every path (no block barrier per item)
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i = blockIdx.x * SR_WARPS + (threadIdx.x >> 5); i < P; i += gridDim.x * SR_WARPS) {
    const uint32_t Li = slen[i];
    const uint4* A = chunks + sstart[i];
    const uint32_t* a = fr + 4ull * sstart[i];
    uint32_t rank = 0, mlcp = 0;
    for (uint32_t j = lane; j < P; j += 32) {
      const uint32_t Lj = slen[j];
      const uint4* B = chunks + sstart[j];
      const uint32_t* b = fr + 4ull * sstart[j];
      const uint32_t lim = min(Li, Lj);
      uint32_t c = 0;
      while (4 * c + 4 <= lim) {
        const uint4 x = A[c], y = B[c];
        if ((x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w)) break;
        ++c;
      }
      uint32_t m = 4 * c;
      while (m < lim && a[m] == b[m]) ++m;
      // path j < path i; equal paths (possible among collision extras) are ordered by index
      const bool less = m < lim ? b[m] < a[m] : (Lj < Li || (Lj == Li && j < i));
      if (less) {
        ++rank;
        mlcp = max(mlcp, m);
      }
    }
    rank = __reduce_add_sync(0xffffffffu, rank);
    mlcp = __reduce_max_sync(0xffffffffu, mlcp);
    if (lane == 0) {
      sorted_item[rank] = i;
      lcp_s[rank] = mlcp;  // the predecessor in lex order shares the longest prefix
      len_s[rank] = Li;
      po_s[rank] = spo[i];
      if (Li == 0) leaf_of_item[i] = 0;  // empty path -> root
    }
  }
}

// one CTA per depth d = blockIdx.x + 1 (d = Lmax + 1 only writes level_off[Lmax + 1] = N)
__global__ void __launch_bounds__(SR_THREADS) k_small_emit(const uint64_t* __restrict__ po_s, const uint32_t* __restrict__ frames,
                                                            uint32_t P,
                                                            const uint32_t* __restrict__ sorted_item, const uint32_t* __restrict__ lcp_s,
                                                            const uint32_t* __restrict__ len_s, uint32_t Lmax, uint32_t* __restrict__ parent,
                                                            uint32_t* __restrict__ frame_out, uint16_t* __restrict__ depth,
                                                            uint32_t* __restrict__ level_off, uint32_t* __restrict__ leaf_of_item,
                                                            uint32_t* d_N, const SmallSpec* spec) { DC_PDL_ENTER();
  if (spec) {  // speculative launch (grid DC_MAX_DEPTH + 1): P and Lmax from the gate
    if (!spec->ok || blockIdx.x > spec->Lmax) return;
    P = spec->P;
    Lmax = spec->Lmax;
  }
  const uint32_t d = blockIdx.x + 1;
  // nodes above depth d and above depth d - 1 (level_off[d] - 1, level_off[d-1] - 1)
  uint32_t above = 0, above_p = 0, maxlen = 0, dups = 0;
  for (uint32_t k = threadIdx.x; k < P; k += SR_THREADS) {
    const uint32_t L = len_s[k], g = lcp_s[k];
    dups += (L > 0 && g >= L) ? 1u : 0u;
    const uint32_t t1 = min(L, d - 1), t2 = d >= 2 ? min(L, d - 2) : 0u;
    above += t1 > g ? t1 - g : 0u;
    above_p += t2 > g ? t2 - g : 0u;
    maxlen = max(maxlen, L);
  }
  uint32_t dummy = 0;
  sr_block_sum_max(above, maxlen);
  sr_block_sum_max(above_p, dummy);
  sr_block_sum_max(dups, dummy);
  const uint32_t lo = 1 + above, lo_p = 1 + above_p;
  if (threadIdx.x == 0) {
    level_off[d] = lo;
    if (d == 1) {
      level_off[0] = 0;
      parent[0] = DC_NO_NODE;
      frame_out[0] = DC_NO_NODE;
      depth[0] = 0;
    }
    if (d == Lmax + 1) {
      d_N[0] = lo;       // N
      d_N[1] = maxlen;   // depth of the tree
      d_N[2] = dups;     // items repeating another item's path (0 unless the dedup split a path)
    }
  }
  if (d > Lmax) return;
  uint32_t run = 0;  // (count at d << 16 | count at d - 1) before this chunk; P <= 4096 < 2^16
  for (uint32_t base = 0; base < P; base += SR_THREADS) {
    const uint32_t k = base + threadIdx.x;
    uint32_t fd = 0, fp = 0;
    uint32_t L = 0;
    if (k < P) {
      L = len_s[k];
      const uint32_t g = lcp_s[k];
      fd = (g < d && d <= L) ? 1u : 0u;
      fp = (d >= 2 && g < d - 1 && d - 1 <= L) ? 1u : 0u;
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan<uint32_t, SR_THREADS>((fd << 16) | fp, &tot);
    const uint32_t inc = run + ex + (fd << 16) + fp;
    const uint32_t id = lo + (inc >> 16) - 1;  // the depth-d node on path k (created by k or before)
    if (fd) {
      parent[id] = d == 1 ? 0u : lo_p + (inc & 0xFFFFu) - 1;
      frame_out[id] = frames[po_s[k] + d - 1];
      depth[id] = (uint16_t)d;
    }
    // a path equal to its predecessor (an item the exact dedup split off after a hash collision
    // may repeat another item's path) creates no node; its leaf is the predecessor's
    if (k < P && L == d) leaf_of_item[sorted_item[k]] = id;
    run += tot;
  }
}

// ------------------------------------------------------------------ a3: large P, per level
__global__ void k_lvl_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                           const uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ active, uint32_t n_active,
                           const uint32_t* __restrict__ node_of_item, uint32_t lvl_start, uint32_t d, int fbits,
                           uint64_t* __restrict__ key, uint32_t* __restrict__ val) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_active; i += gridDim.x * blockDim.x) {
    uint32_t it = active[i];
    uint32_t f = frames[off[item_rec[it]] + d];
    key[i] = ((uint64_t)(node_of_item[it] - lvl_start) << fbits) | f;
    val[i] = it;
  }
}

__global__ void k_lvl_heads(const uint64_t* __restrict__ key, uint32_t n, uint32_t* __restrict__ head) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i - 1] != key[i]) ? 1u : 0u;
}

__global__ void k_lvl_assign(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val, uint32_t n,
                             const uint32_t* __restrict__ run_excl, uint32_t lvl_start, uint32_t next, uint32_t d, int fbits,
                             const uint32_t* __restrict__ item_len, uint32_t* __restrict__ parent, uint32_t* __restrict__ frame_out,
                             uint16_t* __restrict__ depth, uint32_t* __restrict__ node_of_item, uint32_t* __restrict__ leaf_of_item,
                             uint32_t* __restrict__ keep) { DC_PDL_ENTER();
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
                              const uint32_t* __restrict__ keep_excl, uint32_t n, uint32_t* __restrict__ active) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (keep[i]) active[keep_excl[i]] = val[i];
}

__global__ void k_lvl_init(const uint32_t* __restrict__ item_len, uint32_t P, uint32_t* __restrict__ keep,
                           uint32_t* __restrict__ node_of_item, uint32_t* __restrict__ leaf_of_item, uint32_t* __restrict__ idx) { DC_PDL_ENTER();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    keep[i] = item_len[i] > 0;
    node_of_item[i] = 0;
    idx[i] = i;
    if (item_len[i] == 0) leaf_of_item[i] = 0;
  }
}

__global__ void k_root(uint32_t* parent, uint32_t* frame_out, uint16_t* depth, uint32_t* level_off) { DC_PDL_ENTER();
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
  dc_launch(k_root, 1, 1, 0, c->stream, t->parent, t->frame, t->depth, t->level_off);
  DC_LAUNCHED(c);
  dc_launch(k_lvl_init, grid_for(c, P, 256), 256, 0, c->stream, item_len, P, keep.p, node_of_item.p, leaf_of_item, idx.p);
  DC_LAUNCHED(c);
  DC_TRY(excl_scan<uint32_t>(c, keep.p, keep_ex.p, P, tot.p));
  dc_launch(k_lvl_compact, grid_for(c, P, 256), 256, 0, c->stream, idx.p, keep.p, keep_ex.p, P, active.p);
  DC_LAUNCHED(c);
  uint32_t hn[2];
  DC_TRY(readback(c, tot.p, 4, hn));
  uint32_t n_active = hn[0];
  uint32_t lvl_start = 0, width = 1, next = 1;
  std::vector<uint32_t> lo = {0, 1};
  uint32_t d = 0;
  for (; n_active > 0; ++d) {
    int pbits = bits_for(width - 1);
    dc_launch(k_lvl_keys, grid_for(c, n_active, 256), 256, 0, c->stream, p->offsets, p->frames, item_rec, active.p, n_active,
                                                                  node_of_item.p, lvl_start, d, fbits, k0.p, v0.p);
    DC_LAUNCHED(c);
    bool in1 = false;
    DC_TRY(radix_sort_pairs(c, k0.p, v0.p, k1.p, v1.p, n_active, 0, pbits + fbits, &in1));
    uint64_t* ks = in1 ? k1.p : k0.p;
    uint32_t* vs = in1 ? v1.p : v0.p;
    dc_launch(k_lvl_heads, grid_for(c, n_active, 256), 256, 0, c->stream, ks, n_active, keep.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, keep.p, runs.p, n_active, tot.p));
    dc_launch(k_lvl_assign, grid_for(c, n_active, 256), 256, 0, c->stream, ks, vs, n_active, runs.p, lvl_start, next, d, fbits,
                                                                    item_len, t->parent, t->frame, t->depth,
                                                                    node_of_item.p, leaf_of_item, keep.p);
    DC_LAUNCHED(c);
    DC_TRY(excl_scan<uint32_t>(c, keep.p, keep_ex.p, n_active, tot.p + 1));
    dc_launch(k_lvl_compact, grid_for(c, n_active, 256), 256, 0, c->stream, vs, keep.p, keep_ex.p, n_active, active.p);
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

// ------------------------------------------------------------------ a3: large P, Euler tour
// Canonical numbering without a per-level loop (depth up to DC_MAX_DEPTH):
//  1. every prefix of every distinct path is inserted into a node hash table keyed by a
//     position-keyed prefix hash (warp per path, warp scan of the frame terms); a slot carries
//     (parent slot, frame). An existing key must carry the same (parent slot, frame): a
//     mismatch is a hash collision and is detected exactly (by induction from the root, equal
//     keys with equal (parent, frame) are equal prefixes) — the caller then falls back to the
//     level-wise build;
//  2. nodes are sorted by (parent, frame): siblings contiguous in frame order;
//  3. an Euler tour over first-child / next-sibling links is ranked by pointer jumping: the
//     number of "down" steps before a node is its DFS preorder with children in frame order,
//     i.e. its rank in the lexicographic order of paths;
//  4. sorting by (depth, preorder) gives the canonical (depth, lexicographic) ids (reading R2).
struct __align__(16) NodeSlot {
  unsigned long long key;  // prefix hash, ~0 = empty
  unsigned long long pay;  // parent slot << 32 | frame; ~0 until published
};
constexpr uint32_t NS_ROOT = 0xFFFFFFFEu;  // parent slot of depth-1 nodes

__device__ __forceinline__ unsigned long long node_pos(uint32_t j) { return mix64(0xD1B54A32D192ED03ull * (j + 1)) | 1ull; }

__global__ void k_prefix_nodes(const uint64_t* __restrict__ off, const uint32_t* __restrict__ frames,
                               const uint32_t* __restrict__ item_rec, const uint32_t* __restrict__ item_len, uint32_t P,
                               NodeSlot* __restrict__ tab, uint64_t mask, uint16_t* __restrict__ sdepth,
                               uint32_t* __restrict__ leaf_slot, unsigned int* d_cnt, uint64_t hmask) { DC_PDL_ENTER();
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t p = warp; p < P; p += nw) {
    const uint32_t L = item_len[p];
    if (L == 0) {
      if (lane == 0) leaf_slot[p] = PT_NONE;  // empty path: the root
      continue;
    }
    const uint64_t base = off[item_rec[p]];
    unsigned long long carry = 0;
    uint32_t parent = NS_ROOT, last = PT_NONE;
    for (uint32_t j0 = 0; j0 < L; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool act = j < L;
      const uint32_t f = act ? frames[base + j] : 0u;
      const unsigned long long g = act ? ((unsigned long long)f + 1ull) * node_pos(j) : 0ull;
      const unsigned long long incl = warp_incl_scan<unsigned long long>(g) + carry;
      uint64_t H = mix64(incl ^ ((uint64_t)(j + 1) * 0xC2B2AE3D27D4EB4Full)) & hmask;
      if (H == ~0ull) H = ~1ull;
      uint32_t sl = PT_NONE;
      bool mine = false;
      if (act) {
        uint64_t q = (H * 0x9E3779B97F4A7C15ull >> 17) & mask;
        for (uint64_t probe = 0; probe <= (mask < 4096 ? mask : 4096); ++probe, q = (q + 1) & mask) {  // bounded: a long run = overflow, retried larger
          const unsigned long long cur = ld_relaxed_u64(&tab[q].key);
          if (cur == H) {
            sl = (uint32_t)q;
            break;
          }
          if (cur == ~0ull) {
            const unsigned long long old = atomicCAS(&tab[q].key, ~0ull, (unsigned long long)H);
            if (old == ~0ull) {
              sl = (uint32_t)q;
              mine = true;
              break;
            }
            if (old == H) {
              sl = (uint32_t)q;
              break;
            }
          }
        }
      }
      uint32_t ps = __shfl_up_sync(0xffffffffu, sl, 1);
      if (lane == 0) ps = parent;
      const unsigned long long pay = (unsigned long long)ps << 32 | f;
      if (act && mine) {
        sdepth[sl] = (uint16_t)(j + 1);
        st_release_u64(&tab[sl].pay, pay);
        const unsigned ins = atomicAdd(d_cnt, 1u);
        if ((uint64_t)ins * 2 >= mask) atomicOr(d_cnt + 1, 1u);  // past half load: retry larger
      }
      if (act && sl == PT_NONE) atomicOr(d_cnt + 1, 1u);
      __syncwarp();
      if (act && !mine && sl != PT_NONE) {
        unsigned long long pp;
        // relaxed: the payload word is the data (no other field is read after it), and an acquire
        // load would invalidate the SM's L1 on every pass
        for (uint64_t spin = 0; (pp = ld_relaxed_u64(&tab[sl].pay)) == ~0ull; ++spin)
          if (spin > DC_SPIN_LIMIT) __trap();
        if (pp != pay) atomicOr(d_cnt + 2, 1u);  // same key, different (parent, frame): collision
      }
      carry = __shfl_sync(0xffffffffu, incl, 31);
      parent = __shfl_sync(0xffffffffu, sl, 31);
      last = __shfl_sync(0xffffffffu, sl, (L - 1 - j0) & 31u);
    }
    if (lane == 0) leaf_slot[p] = last;
  }
}

__global__ void k_node_compact(const NodeSlot* __restrict__ tab, uint64_t cap, uint32_t* __restrict__ nslot,
                               uint32_t* __restrict__ nidx, unsigned int* d_pos) { DC_PDL_ENTER();
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    if (tab[s].key == ~0ull) continue;
    const unsigned n = atomicAdd(d_pos, 1u);
    nslot[n] = (uint32_t)s;
    nidx[s] = n;
  }
}

// node fields (root = index Nn) and the sibling sort key (parent + 1, frame)
__global__ void k_node_fields(uint32_t Nn, const uint32_t* __restrict__ nslot, const uint32_t* __restrict__ nidx,
                              const NodeSlot* __restrict__ tab, const uint16_t* __restrict__ sdepth, int fbits,
                              uint32_t* __restrict__ par, uint32_t* __restrict__ frm, uint16_t* __restrict__ dep,
                              uint64_t* __restrict__ skey, uint32_t* __restrict__ sval) { DC_PDL_ENTER();
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < Nn; n += gridDim.x * blockDim.x) {
    const uint32_t s = nslot[n];
    const unsigned long long pay = tab[s].pay;
    const uint32_t ps = (uint32_t)(pay >> 32), f = (uint32_t)pay;
    const uint32_t pn = ps == NS_ROOT ? Nn : nidx[ps];
    par[n] = pn;
    frm[n] = f;
    dep[n] = sdepth[s];
    skey[n] = ((uint64_t)(ps == NS_ROOT ? 0u : pn + 1u) << fbits) | f;
    sval[n] = n;
  }
}

__global__ void k_euler_links(uint32_t Nn, const uint64_t* __restrict__ ks, const uint32_t* __restrict__ vs, int fbits,
                              uint32_t* __restrict__ first_child, uint32_t* __restrict__ next_sib) { DC_PDL_ENTER();
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < Nn; k += gridDim.x * blockDim.x) {
    const uint32_t n = vs[k];
    const uint64_t g = ks[k] >> fbits;
    if (k == 0 || (ks[k - 1] >> fbits) != g) first_child[g == 0 ? Nn : (uint32_t)(g - 1)] = n;
    next_sib[n] = (k + 1 < Nn && (ks[k + 1] >> fbits) == g) ? vs[k + 1] : PT_NONE;
  }
}

// tour elements: down(n) = n, up(n) = Nn + 1 + n (n <= Nn, root = Nn); packed (next << 32 | weight)
__global__ void k_euler_init(uint32_t Nn, const uint32_t* __restrict__ par, const uint32_t* __restrict__ first_child,
                             const uint32_t* __restrict__ next_sib, unsigned long long* __restrict__ tour) { DC_PDL_ENTER();
  const uint64_t M = 2ull * (Nn + 1);
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < M; x += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t nx, w;
    if (x <= Nn) {
      const uint32_t fc = first_child[x];
      nx = fc != PT_NONE ? fc : (uint32_t)(Nn + 1 + x);
      w = 1;
    } else {
      const uint32_t n = (uint32_t)(x - (Nn + 1));
      if (n == Nn) {
        nx = PT_NONE;
      } else {
        const uint32_t ns = next_sib[n];
        nx = ns != PT_NONE ? ns : Nn + 1 + par[n];
      }
      w = 0;
    }
    tour[x] = (unsigned long long)nx << 32 | w;
  }
}

// one pointer-jumping round: suffix weight sums along the tour
__global__ void k_wyllie(uint64_t M, const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out) { DC_PDL_ENTER();
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < M; x += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long e = in[x];
    const uint32_t nx = (uint32_t)(e >> 32);
    if (nx == PT_NONE) {
      out[x] = e;
    } else {
      const unsigned long long f = in[nx];
      out[x] = (f & 0xFFFFFFFF00000000ull) | (uint32_t)((uint32_t)e + (uint32_t)f);
    }
  }
}

__global__ void k_canon_keys(uint32_t Nn, const uint16_t* __restrict__ dep, const unsigned long long* __restrict__ tour,
                             int pbits, uint64_t* __restrict__ ck, uint32_t* __restrict__ cv) { DC_PDL_ENTER();
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < Nn; n += gridDim.x * blockDim.x) {
    const uint32_t pre = (Nn + 1) - (uint32_t)tour[n];  // down steps before down(n)
    ck[n] = ((uint64_t)dep[n] << pbits) | pre;
    cv[n] = n;
  }
}

__global__ void k_canon_ids(uint32_t Nn, const uint32_t* __restrict__ cv, uint32_t* __restrict__ canon) { DC_PDL_ENTER();
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < Nn; k += gridDim.x * blockDim.x) canon[cv[k]] = k + 1;
}

__global__ void k_canon_write(uint32_t Nn, const uint64_t* __restrict__ ck, const uint32_t* __restrict__ cv, int pbits,
                              const uint32_t* __restrict__ par, const uint32_t* __restrict__ frm,
                              const uint32_t* __restrict__ canon, uint32_t* __restrict__ parent, uint32_t* __restrict__ frame_out,
                              uint16_t* __restrict__ depth, uint32_t* __restrict__ level_off, uint32_t Lmax) { DC_PDL_ENTER();
  const uint64_t gid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (gid == 0) {
    parent[0] = DC_NO_NODE;
    frame_out[0] = DC_NO_NODE;
    depth[0] = 0;
    level_off[0] = 0;
    if (Nn == 0)
      for (uint32_t d = 1; d <= Lmax + 1; ++d) level_off[d] = 1;
  }
  for (uint32_t k = (uint32_t)gid; k < Nn; k += gridDim.x * blockDim.x) {
    const uint32_t n = cv[k], id = k + 1;
    const uint32_t pn = par[n];
    parent[id] = pn == Nn ? 0u : canon[pn];
    frame_out[id] = frm[n];
    const uint32_t d = (uint32_t)(ck[k] >> pbits);
    depth[id] = (uint16_t)d;
    if (k == 0 || (uint32_t)(ck[k - 1] >> pbits) != d) level_off[d] = id;
    if (k == Nn - 1)
      for (uint32_t dd = d + 1; dd <= Lmax + 1; ++dd) level_off[dd] = Nn + 1;
  }
}

__global__ void k_item_leaf(uint32_t P, const uint32_t* __restrict__ leaf_slot, const uint32_t* __restrict__ nidx,
                            const uint32_t* __restrict__ canon, uint32_t* __restrict__ leaf_of_item) { DC_PDL_ENTER();
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    const uint32_t ls = leaf_slot[p];
    leaf_of_item[p] = ls == PT_NONE ? 0u : canon[nidx[ls]];
  }
}

// returns *collided = true (and builds nothing) when a prefix-hash collision was detected
static dc_status build_euler(Ctx* c, const dc_paths* p, const uint32_t* item_rec, const uint32_t* item_len, uint32_t P,
                             uint64_t sumlen, uint32_t Lmax, int fbits, dc_cct* t, uint32_t* leaf_of_item, uint64_t* h_N,
                             bool* collided) {
  *collided = false;
  Buf<NodeSlot> tab;
  Buf<uint16_t> sdepth;
  Buf<uint32_t> leaf_slot;
  Buf<unsigned int> cnt;
  DC_TRY(alloc(c, leaf_slot, P));
  // nodes <= sumlen + 1; a tree with little sharing has far more than 8 per path: the last
  // call's node count (per context) keeps the first attempt from overflowing on repeated shapes
  const uint64_t want = std::min<uint64_t>(sumlen + 1, std::max<uint64_t>(8ull * P + 1024, c->euler_nodes_hint));
  uint64_t cap = 1024;
  while (cap < 2 * want) cap <<= 1;
  uint32_t hc[4];
  for (int attempt = 0;; ++attempt) {
    DC_TRY(alloc(c, tab, cap));
    DC_TRY(alloc(c, sdepth, cap));
    DC_CUDA(c, cudaMemsetAsync(tab.p, 0xFF, cap * sizeof(NodeSlot), c->stream));
    DC_TRY(alloc_zero(c, cnt, 4));  // [0] nodes, [1] overflow, [2] collision, [3] compact pos
    dc_launch(k_prefix_nodes, grid_for(c, (uint64_t)P * 32, 256), 256, 0, c->stream, p->offsets, p->frames, item_rec, item_len, P, tab.p,
                                                                              cap - 1, sdepth.p, leaf_slot.p, cnt.p,
                                                                              c->node_mask);
    DC_LAUNCHED(c);
    DC_TRY(readback(c, cnt.p, 16, hc));
    if (hc[2]) {
      *collided = true;
      return DC_OK;
    }
    if (!hc[1]) break;
    uint64_t big = 1024;
    while (big < 2 * (sumlen + 1)) big <<= 1;
    if (attempt || big <= cap || big > (1ull << 31)) return fail(c, DC_ERR_CAPACITY, "dc_cct_build: node table overflow");
    cap = big;
  }
  const uint32_t Nn = hc[0];  // nodes without the root
  c->euler_nodes_hint = (uint64_t)Nn + Nn / 4 + 1;
  Buf<uint32_t> nslot, nidx, par, frm, sv0, sv1, first_child, next_sib, canon;
  Buf<uint16_t> dep;
  Buf<uint64_t> sk0, sk1;
  Buf<unsigned long long> tour0, tour1;
  DC_TRY(alloc(c, nslot, Nn));
  DC_TRY(alloc(c, nidx, cap));
  DC_TRY(alloc(c, par, Nn));
  DC_TRY(alloc(c, frm, Nn));
  DC_TRY(alloc(c, dep, Nn));
  DC_TRY(alloc(c, sk0, Nn));
  DC_TRY(alloc(c, sk1, Nn));
  DC_TRY(alloc(c, sv0, Nn));
  DC_TRY(alloc(c, sv1, Nn));
  DC_TRY(alloc(c, first_child, (uint64_t)Nn + 1));
  DC_TRY(alloc(c, next_sib, Nn));
  DC_TRY(alloc(c, canon, Nn));
  const uint64_t M = 2ull * (Nn + 1);
  DC_TRY(alloc(c, tour0, M));
  DC_TRY(alloc(c, tour1, M));
  dc_launch(k_node_compact, grid_for(c, cap, 256), 256, 0, c->stream, tab.p, cap, nslot.p, nidx.p, cnt.p + 3);
  DC_LAUNCHED(c);
  dc_launch(k_node_fields, grid_for(c, Nn, 256), 256, 0, c->stream, Nn, nslot.p, nidx.p, tab.p, sdepth.p, fbits, par.p, frm.p, dep.p,
                                                            sk0.p, sv0.p);
  DC_LAUNCHED(c);
  bool in1 = false;
  DC_TRY(radix_sort_pairs(c, sk0.p, sv0.p, sk1.p, sv1.p, Nn, 0, fbits + bits_for((uint64_t)Nn + 1), &in1));
  const uint64_t* ks = in1 ? sk1.p : sk0.p;
  const uint32_t* vs = in1 ? sv1.p : sv0.p;
  DC_CUDA(c, cudaMemsetAsync(first_child.p, 0xFF, ((uint64_t)Nn + 1) * 4, c->stream));
  dc_launch(k_euler_links, grid_for(c, Nn, 256), 256, 0, c->stream, Nn, ks, vs, fbits, first_child.p, next_sib.p);
  DC_LAUNCHED(c);
  dc_launch(k_euler_init, grid_for(c, M, 256), 256, 0, c->stream, Nn, par.p, first_child.p, next_sib.p, tour0.p);
  DC_LAUNCHED(c);
  unsigned long long *tin = tour0.p, *tout = tour1.p;
  for (uint64_t span = 1; span < M; span <<= 1) {
    dc_launch(k_wyllie, grid_for(c, M, 256), 256, 0, c->stream, M, tin, tout);
    DC_LAUNCHED(c);
    std::swap(tin, tout);
  }
  const int pbits = bits_for((uint64_t)Nn + 1);
  dc_launch(k_canon_keys, grid_for(c, Nn, 256), 256, 0, c->stream, Nn, dep.p, tin, pbits, sk0.p, sv0.p);
  DC_LAUNCHED(c);
  DC_TRY(radix_sort_pairs(c, sk0.p, sv0.p, sk1.p, sv1.p, Nn, 0, pbits + bits_for(Lmax), &in1));
  const uint64_t* cks = in1 ? sk1.p : sk0.p;
  const uint32_t* cvs = in1 ? sv1.p : sv0.p;
  dc_launch(k_canon_ids, grid_for(c, Nn, 256), 256, 0, c->stream, Nn, cvs, canon.p);
  DC_LAUNCHED(c);
  dc_launch(k_canon_write, grid_for(c, Nn ? Nn : 1, 256), 256, 0, c->stream, Nn, cks, cvs, pbits, par.p, frm.p, canon.p, t->parent,
                                                                    t->frame, t->depth, t->level_off, Lmax);
  DC_LAUNCHED(c);
  dc_launch(k_item_leaf, grid_for(c, P, 256), 256, 0, c->stream, P, leaf_slot.p, nidx.p, canon.p, leaf_of_item);
  DC_LAUNCHED(c);
  *h_N = (uint64_t)Nn + 1;
  return DC_OK;
}

dc_status cct_build(Ctx* c, const dc_paths* p, const dc_dict* dict, uint32_t n_frames, uint32_t* out_leaf, dc_cct** out) {
  *out = nullptr;
  const uint64_t R = p->n_records;
  if (R >= (1ull << 32)) return fail(c, DC_ERR_CAPACITY, "dc_cct_build: n_records >= 2^32");
  dc_cct* t = new dc_cct();
  HandleGuard<dc_cct, dc_cct_free> guard{t};  // frees the handle and its arrays on any error return
  t->device = c->device;
  t->owner_uid = adopt_handle(c);
  t->R = R;
  t->n_frames = n_frames;
  const int fbits = bits_for(n_frames > 0 ? n_frames - 1 : 0) > 0 ? bits_for(n_frames - 1) : 1;
  if (dict) {
    DC_TRY(palloc(c, t->frame_kind, n_frames));
    DC_TRY(dcopy(c, t->frame_kind, dict->kinds, n_frames));
  }
  // ---- a2: hash pass (frames streamed once), then group + exact verification
  Buf<uint32_t> slot_of_rec, extra_rec, pid_of_slot, item_rec, item_len, leaf_of_item, leafbuf;
  Buf<uint64_t> hash;
  Buf<PathSlot> tab;
  Buf<unsigned long long> sumlen;
  Buf<unsigned int> cnt;
  DC_TRY(alloc(c, hash, R));
  DC_TRY(alloc(c, slot_of_rec, R));
  DC_TRY(alloc(c, extra_rec, R));
  // path table sized for the distinct paths, not the records (retry if it passes half load)
  uint64_t cap = 1024;
  while (cap < 2 * (R < (1ull << 19) ? R : (1ull << 19))) cap <<= 1;
  if (getenv("DC_TEST_PATH_CAP")) cap = 1024;  // test only: force the table-overflow retry
  {  // every fill of the record pass in one launch
    FillList fl;
    DC_TRY(alloc_fill(c, fl, cnt, 8));  // [0] distinct, [1] extra, [2] compact pos, [3] overflow, [4] empty paths
    DC_TRY(alloc_fill(c, fl, tab, cap, 0xFF));
    DC_TRY(alloc_fill(c, fl, sumlen, 1));
    DC_TRY(fill_flush(c, fl));
  }
  const int tma_ok = ((uintptr_t)p->offsets % 16 == 0) && ((uintptr_t)p->frames % 16 == 0) && !getenv("DC_TEST_NO_TMA");
  DC_SMEM_OPTIN(c, k_path_hash);  // once per context
  if (R) {
    if (!c->path_hash_per_sm)
      DC_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->path_hash_per_sm, k_path_hash, PT_THREADS, sizeof(PathSmem)));
    const int per_sm = c->path_hash_per_sm;
    const uint64_t n_tiles = (R + PT_T - 1) / PT_T;
    const int hgrid = (int)std::min<uint64_t>(n_tiles, (uint64_t)c->num_sms * std::max(per_sm, 1));
    Region rk(c, "k:path_hash");
    dc_launch(k_path_hash, hgrid, PT_THREADS, sizeof(PathSmem), c->stream, p->offsets, p->frames, R, n_frames, hash.p, cnt.p,
                                                                     c->d_flags, (unsigned long long*)c->d_diag,
                                                                     c->hash_mask, tma_ok);
    DC_LAUNCHED(c);
  }
  // One round trip for the whole record pass: the item arrays are sized by the records (every
  // item has its own representative record), compaction and item lengths run on the device
  // counters, and the counters, length sum, deepest path, flags and frame count come back
  // together. A table past half load (rare) repeats the attempt with a larger table.
  uint32_t hc[8];
  uint64_t hsum = 0, hmaxd = 0, F = 0;
  uint32_t hflags = 0;
  const uint64_t ibound = R ? R : 1;
  DC_TRY(alloc(c, item_rec, ibound));
  DC_TRY(alloc(c, item_len, ibound));
  DC_TRY(alloc(c, leaf_of_item, ibound));
  // speculative small-P build (see below)
  bool spec = false, spec_ok = false;
  Buf<SmallSpec> sspec;
  Buf<uint32_t> sdN, ssrt, slcp, slen;
  Buf<uint64_t> spos;
  for (int attempt = 0;; ++attempt) {
    if (attempt) {  // a larger table: fresh table, counters [0..3] ([4] empty paths kept), length sum
      FillList fl;
      DC_TRY(alloc_fill(c, fl, tab, cap, 0xFF));
      DC_TRY(fill_add(c, fl, cnt.p, 16));
      DC_TRY(fill_add(c, fl, sumlen.p, 8));
      DC_TRY(fill_flush(c, fl));
    }
    if (R) {
      Region rk(c, "k:path_group");
      const bool pg_rows = getenv("DC_PG_ROWS") != nullptr;  // tests / A/B: the per-record verify
      dc_launch(pg_rows ? k_path_group<false> : k_path_group<true>, grid_for(c, (R + 31) / 32 * 32, 256), 256, 0, c->stream, p->offsets, p->frames, hash.p, R, tab.p,
                                                                                cap - 1, slot_of_rec.p, extra_rec.p, cnt.p);
      DC_LAUNCHED(c);
    }
    DC_TRY(alloc(c, pid_of_slot, cap));
    dc_launch(k_path_compact, grid_for(c, cap, 256), 256, 0, c->stream, tab.p, cap, pid_of_slot.p, item_rec.p, item_len.p, cnt.p + 2);
    DC_LAUNCHED(c);
    dc_launch(k_items_finish, grid_for(c, ibound, 256), 256, 0, c->stream, item_rec.p, extra_rec.p, p->offsets, item_len.p, sumlen.p,
              cnt.p, (unsigned long long*)c->d_diag);
    DC_LAUNCHED(c);
    spec = attempt == 0 && !getenv("DC_TEST_BUILD_LEVELS") && !getenv("DC_TEST_BUILD_NOSPEC");
    if (spec) {
      // Speculative small-P build behind the readback: the device keeps ranking and emitting the
      // tree while the host reads (P, sum of lengths, depth, flags); k_small_gate applies on the
      // device the same test the host applies below, so both agree on whether it ran.
      DC_TRY(readback_begin(c, {{cnt.p, 32, hc}, {sumlen.p, 8, &hsum}, {c->d_diag + DG_MAXDEPTH, 8, &hmaxd},
                                {c->d_flags, 4, &hflags}, {p->offsets + R, 8, &F}}));
      DC_TRY(alloc(c, sspec, 1));
      DC_TRY(alloc(c, sdN, 3));
      DC_TRY(alloc(c, spos, SMALL_P));
      DC_TRY(alloc(c, ssrt, SMALL_P));
      DC_TRY(alloc(c, slcp, SMALL_P));
      DC_TRY(alloc(c, slen, SMALL_P));
      DC_TRY(palloc(c, t->parent, SPEC_NODES));
      DC_TRY(palloc(c, t->frame, SPEC_NODES));
      DC_TRY(palloc(c, t->depth, SPEC_NODES));
      DC_TRY(palloc(c, t->level_off, (uint64_t)DC_MAX_DEPTH + 2));
      dc_launch(k_small_gate, 1, 32, 0, c->stream, (const unsigned int*)cnt.p, (const unsigned long long*)sumlen.p,
                (const unsigned long long*)(c->d_diag + DG_MAXDEPTH), (const uint32_t*)c->d_flags, (uint64_t)c->smem_optin, sspec.p);
      DC_LAUNCHED(c);
      DC_SMEM_OPTIN(c, k_small_rank);
      if (!c->small_rank_smem) {
        cudaFuncAttributes fa;
        DC_CUDA(c, cudaFuncGetAttributes(&fa, k_small_rank));
        c->small_rank_smem = c->smem_optin - fa.sharedSizeBytes;
      }
      dc_launch(k_small_rank, (uint32_t)c->num_sms, SR_THREADS, c->small_rank_smem, c->stream, p->offsets, p->frames, item_rec.p,
                item_len.p, 0u, ssrt.p, slcp.p, slen.p, spos.p, leaf_of_item.p, (const SmallSpec*)sspec.p);
      DC_LAUNCHED(c);
      dc_launch(k_small_emit, (uint32_t)DC_MAX_DEPTH + 1, SR_THREADS, 0, c->stream, spos.p, p->frames, 0u, ssrt.p, slcp.p, slen.p, 0u,
                t->parent, t->frame, t->depth, t->level_off, leaf_of_item.p, sdN.p, (const SmallSpec*)sspec.p);
      DC_LAUNCHED(c);
      DC_TRY(readback_end(c));
    } else {
      DC_TRY(readback_multi(c, {{cnt.p, 32, hc}, {sumlen.p, 8, &hsum}, {c->d_diag + DG_MAXDEPTH, 8, &hmaxd}, {c->d_flags, 4, &hflags},
                                {p->offsets + R, 8, &F}}));
    }
    spec_ok = spec && small_spec_ok(hc[3], hflags, (uint64_t)hc[0] + hc[1], hsum, hmaxd, c->smem_optin);
    if (spec && !spec_ok) {  // the speculative kernels did nothing: the node arrays are sized below
      void* q[] = {t->parent, t->frame, t->depth, t->level_off};
      for (void* x : q) cudaFreeAsync(x, c->stream);
      t->parent = t->frame = t->level_off = nullptr;
      t->depth = nullptr;
    }
    if (!hc[3]) break;
    if ((hc[3] & 2) || attempt > 2 || cap >= (1ull << 31))
      return fail(c, DC_ERR_CAPACITY, "dc_cct_build: path table overflow");
    cap = cap * 8 < (1ull << 31) ? cap * 8 : (1ull << 31);
  }
  const uint32_t P0 = hc[0], n_extra = hc[1], P = P0 + n_extra;
  DC_TRY(flags_status(c, hflags));
  const uint64_t Nbound = 1 + hsum;
  if (Nbound >= (1ull << 32)) return fail(c, DC_ERR_CAPACITY, "dc_cct_build: more than 2^32 nodes");
  // hmaxd is the deepest path seen on this context so far (>= this trace's): sizes level_off
  const uint32_t Lmax = (uint32_t)hmaxd;
  if (!spec_ok) {
    DC_TRY(palloc(c, t->parent, Nbound));
    DC_TRY(palloc(c, t->frame, Nbound));
    DC_TRY(palloc(c, t->depth, Nbound));
    DC_TRY(palloc(c, t->level_off, (uint64_t)Lmax + 2));
  }
  uint64_t N = 0;
  uint32_t levels = 0;
  const uint64_t rank_smem = ((16ull * P + 15) & ~15ull) + 4ull * (hsum + 3ull * P);
  uint32_t hN3[3] = {0, 0, 0};
  if (spec_ok) {  // ranked and emitted already (speculative kernels): the node count is read behind
                  // the leaf kernels and the count-column fill below (split-phase readback)
    DC_TRY(readback_begin(c, {{sdN.p, 12, hN3}}));
  } else if (P <= SMALL_P && rank_smem + 1024 <= c->smem_optin && !getenv("DC_TEST_BUILD_LEVELS")) {
    // lexicographic rank of the distinct paths + one CTA per depth (no level loop)
    Buf<uint32_t> dN, srt, lcp, len;
    Buf<uint64_t> pos;
    DC_TRY(alloc(c, dN, 3));
    DC_TRY(alloc(c, pos, P));
    DC_TRY(alloc(c, srt, P));
    DC_TRY(alloc(c, lcp, P));
    DC_TRY(alloc(c, len, P));
    DC_SMEM_OPTIN(c, k_small_rank);
    const uint32_t Gi = (P + SR_WARPS - 1) / SR_WARPS;  // one warp per item
    const uint32_t G = Gi == 0 ? 1u : Gi < (uint32_t)c->num_sms ? Gi : (uint32_t)c->num_sms;
    dc_launch(k_small_rank, G, SR_THREADS, rank_smem, c->stream, p->offsets, p->frames, item_rec.p, item_len.p, P, srt.p, lcp.p,
              len.p, pos.p, leaf_of_item.p, (const SmallSpec*)nullptr);
    DC_LAUNCHED(c);
    dc_launch(k_small_emit, Lmax + 1, SR_THREADS, 0, c->stream, pos.p, p->frames, P, srt.p, lcp.p, len.p, Lmax,
              t->parent, t->frame, t->depth, t->level_off, leaf_of_item.p, dN.p, (const SmallSpec*)nullptr);
    DC_LAUNCHED(c);
    uint32_t hN[3] = {0, 0, 0};
    DC_TRY(readback(c, dN.p, 12, hN));
    N = hN[0];
    t->max_depth = hN[1];
    // distinct table slots must hold distinct paths (the tree is right either way: equal paths
    // share their nodes); DC_STRICT=1 (the test suite) turns a lost dedup into an error;
    // collision extras may repeat each other's path, table items never do
    if (hN[2] > n_extra && getenv("DC_STRICT"))
      return fail(c, DC_ERR_STATE, "internal: %u of %u path items repeat a path (%u collision extras)", hN[2], P, n_extra);
  } else if (P <= SMALL_P) {
    Buf<uint32_t> dN;
    DC_TRY(alloc(c, dN, 2));
    size_t smem = sizeof(SmallSmem);
    DC_SMEM_OPTIN(c, k_build_small);
    dc_launch(k_build_small, 1, SB_THREADS, smem, c->stream, p->offsets, p->frames, item_rec.p, item_len.p, P, fbits, t->parent,
                                                      t->frame, t->depth, t->level_off, leaf_of_item.p, dN.p);
    DC_LAUNCHED(c);
    uint32_t hN[2] = {0, 0};
    DC_TRY(readback(c, dN.p, 8, hN));
    N = hN[0];
    t->max_depth = hN[1];
  } else {
    bool collided = true;
    if (!getenv("DC_TEST_LEVELWISE"))
      DC_TRY(build_euler(c, p, item_rec.p, item_len.p, P, hsum, Lmax, fbits, t, leaf_of_item.p, &N, &collided));
    if (collided) {  // prefix-hash collision (or forced): exact level-wise construction
      if (!getenv("DC_TEST_LEVELWISE")) c->host_collisions += 1;
      DC_TRY(build_large(c, p, item_rec.p, item_len.p, P, Lmax, fbits, t, leaf_of_item.p, &levels, &N));
    }
  }
  // max depth of this tree
  uint32_t* leaf = out_leaf;
  if (!leaf) {
    DC_TRY(alloc(c, leafbuf, R));
    leaf = leafbuf.p;
  }
  {
    Buf<uint32_t> leaf_of_slot;
    DC_TRY(alloc(c, leaf_of_slot, cap));
    dc_launch(k_slot_leaf, grid_for(c, cap, 256), 256, 0, c->stream, tab.p, cap, pid_of_slot.p, leaf_of_item.p, leaf_of_slot.p);
    DC_LAUNCHED(c);
    dc_launch(k_rec_leaf, grid_for(c, (R + 3) / 4, 256), 256, 0, c->stream, slot_of_rec.p, leaf_of_slot.p, cap, P0, leaf_of_item.p, R,
                                                                     leaf);
    DC_LAUNCHED(c);
  }
  // node columns (exclusive/inclusive counts), metric columns come with attribute; a speculative
  // build sizes them by its node bound (the node count is still in flight)
  const uint64_t Ncols = spec_ok ? SPEC_NODES : N;
  DC_TRY(palloc(c, t->xcnt, Ncols));
  DC_TRY(palloc(c, t->icnt, Ncols));
  // icnt is written whole by dc_cct_rollup (every schedule) and unreadable before it
  {
    FillList fx;
    DC_TRY(fill_add(c, fx, t->xcnt, Ncols * 8));
    DC_TRY(fill_flush(c, fx));
  }
  if (spec_ok) {
    DC_TRY(readback_end(c));
    N = hN3[0];
    t->max_depth = hN3[1];
    if (hN3[2] > n_extra && getenv("DC_STRICT"))
      return fail(c, DC_ERR_STATE, "internal: %u of %u path items repeat a path (%u collision extras)", hN3[2], P, n_extra);
  }
  t->N = N;
  // depth of the tree = largest d with a node
  if (P > SMALL_P) {
    uint16_t md = 0;
    if (N > 1) DC_TRY(readback(c, t->depth + (N - 1), 2, &md));
    t->max_depth = md;
  }
  // algorithmic bytes: offsets + frames of every record once, leaf, node table
  c->bytes_host += 8 * (R + 1) + 4 * F + 4 * R + 10 * N;
  c->host_levels += t->max_depth;
  c->host_collisions += n_extra;
  (void)levels;
  t->state = 0;
  guard.h = nullptr;
  *out = t;
  return DC_OK;
}

}  // namespace dc
