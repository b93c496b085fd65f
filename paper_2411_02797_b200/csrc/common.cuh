// common.cuh — context, handles, error plumbing and small device helpers of libdc.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <chrono>
#include <initializer_list>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dc.h"

namespace dc {

// device-side data-error flag bits (reported as DC_ERR_TRACE)
enum : uint32_t {
  FLAG_BAD_FRAME = 1u,      // frame id >= n_frames
  FLAG_BAD_KEY = 2u,        // raw key with reserved kind
  FLAG_TOO_DEEP = 4u,       // path longer than DC_MAX_DEPTH
  FLAG_BAD_LEAF = 8u,       // launch_leaf / leaf entry not a node
  FLAG_BAD_OFFSETS = 16u,   // offsets not monotone
  FLAG_INTERNAL = 0x80000000u,
};

// device diag slots
enum { DG_EMPTY = 0, DG_BAD_LAUNCH, DG_BAD_STALL, DG_ZERO, DG_COLL, DG_LEVELS, DG_MAXDEPTH, DG_BYTES, DG_N };

struct RBPending;
struct Ctx {
  int device = 0;
  uint64_t uid = 0;  // unique per context (handle frees look it up)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // the context's own stream-ordered memory pool: every library allocation comes from it, its
  // release threshold (kept at "never release" so steady-state steps reuse memory) affects
  // nothing else in the process, and dc_ctx_trim / dc_ctx_destroy hand the memory back
  cudaMemPool_t pool = nullptr;
  // chained-scan tile state (prim.cuh): flags [scan_cap], values [4 * scan_cap], ticket counter
  uint64_t* scan_flag = nullptr;
  uint64_t* scan_val = nullptr;
  unsigned long long* scan_ctr = nullptr;
  uint64_t scan_cap = 0, scan_seq = 0, scan_tickets = 0;
  // Scratch arena: every Buf of a public call is carved from these pool chunks by a bump pointer
  // that rewinds at the next public call (all work is ordered on the one context stream, so the
  // previous call's kernels are done with the memory before the next call's use it). One
  // allocation per chunk instead of a cudaMallocAsync / cudaFreeAsync pair per scratch buffer
  // (~150 host API calls per config-3 step). Chunks are kept until dc_ctx_trim / destroy.
  std::vector<std::pair<char*, size_t>> arena;
  size_t arena_ci = 0, arena_off = 0;
  void arena_reset() {
    arena_ci = 0;
    arena_off = 0;
  }
  uint64_t pc_bins_hint = 0;   // bins of the last PC-histogram call (+1/8): capacity guess of the next
  uint64_t pc_words_hint = 0;  // bitmap words of the last context reduce (+1/8): its scratch guess
  uint64_t pc_big_hint = 0;    // bins of big contexts (counted in scratch) of the last call (+1/8)
  uint64_t pc_generic_hint = 0;  // distinct bins of the last generic-schedule call
  uint64_t euler_nodes_hint = 0;  // nodes of the last Euler-tour build (+1/4): its table size guess
  std::string err;
  uint32_t* d_flags = nullptr;   // [1]
  uint64_t* d_diag = nullptr;    // [DG_N]
  uint64_t* h_pinned = nullptr;  // small pinned readback buffer
  cudaEvent_t rb_event = nullptr;  // split-phase readback (readback_begin / readback_end)
  RBPending* rb_pending = nullptr;
  int num_sms = 148;
  size_t smem_optin = 0;
  std::vector<const void*> smem_set;  // kernels whose dynamic shared-memory cap is raised to smem_optin
  int path_hash_per_sm = 0;           // cached occupancy of k_path_hash
  size_t small_rank_smem = 0;         // k_small_rank's largest dynamic shared memory
  uint64_t launches = 0;
  uint64_t bytes_host = 0;       // host-accumulated algorithmic bytes
  uint64_t host_levels = 0;      // tree levels built
  uint64_t host_collisions = 0;  // path-hash collisions resolved exactly
  uint64_t hash_mask = ~0ull;    // fault injection: DC_TEST_WEAK_HASH=bits shortens path hashes
  uint64_t merge_mask = ~0ull;
  uint64_t node_mask = ~0ull;    // fault injection: DC_TEST_WEAK_NODE_HASH=bits shortens prefix-node hashes   // fault injection: DC_TEST_WEAK_MERGE_HASH=bits shortens merge hashes
  // optional CUDA-event timers (dc_ctx_set_timing): (name, start, stop) per timed region
  bool timing = false;
  struct Timed { const char* name; cudaEvent_t a, b; };
  std::vector<Timed> timed;
  struct HTimed { const char* name; double ms; };
  std::vector<HTimed> htimed;  // host-side durations ("h:<name>" in the report)
  std::vector<cudaEvent_t> ev_pool;  // timing events, reused after each report
  size_t ev_next = 0;
  cudaEvent_t event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
};

// RAII host wall-clock timer (no-op unless timing is on): finds host stalls between kernels
struct HostRegion {
  Ctx* c;
  const char* name;
  std::chrono::steady_clock::time_point t0;
  HostRegion(Ctx* ctx, const char* n) : c(ctx), name(n) {
    if (c->timing) t0 = std::chrono::steady_clock::now();
  }
  ~HostRegion() {
    if (c->timing)
      c->htimed.push_back({name, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count()});
  }
};

// RAII CUDA-event timer of a region on the context stream (no-op unless timing is on)
struct Region {
  Ctx* c;
  const char* name;
  cudaEvent_t a = nullptr;
  Region(Ctx* ctx, const char* n) : c(ctx), name(n) {
    if (c->timing) {
      a = c->event();
      cudaEventRecord(a, c->stream);
    }
  }
  ~Region() {
    if (c->timing && a) {
      cudaEvent_t b = c->event();
      cudaEventRecord(b, c->stream);
      c->timed.push_back({name, a, b});
    }
  }
};

}  // namespace dc

struct dc_ctx : dc::Ctx {};

// Handles remember the context that made them: while that context is alive they are freed
// stream-ordered on its stream (cudaFreeAsync, no device synchronisation); otherwise with a
// device synchronisation and cudaFree.
namespace dc {
void register_ctx(Ctx* c, bool live);
void free_handle_ptrs(uint64_t owner_uid, void* const* ps, size_t n);
void flush_pending_frees(Ctx* c);  // issue the deferred stream-ordered frees of freed handles
uint64_t adopt_handle(Ctx* c);  // a new handle of context c: returns its owner uid (c->uid)
}  // namespace dc

struct dc_dict {
  int device = 0;
  uint64_t owner_uid = 0;  // context that allocated the arrays (0: none)
  uint64_t D = 0;
  dc_frame_key* keys = nullptr;  // dev [D]
  uint8_t* kinds = nullptr;      // dev [D]
};

struct dc_cct {
  int device = 0;
  uint64_t owner_uid = 0;  // context that allocated the arrays (0: none)
  uint64_t N = 0, Npc = 0, Nbins = 0, R = 0;
  uint32_t M = 0, S = 0, max_depth = 0, n_frames = 0;
  int state = 0;  // 0 BUILT, 1 DIRTY, 2 ROLLED
  bool pc_done = false;
  // structure
  uint32_t *parent = nullptr, *frame = nullptr, *level_off = nullptr;
  uint16_t* depth = nullptr;
  uint8_t* frame_kind = nullptr;  // dev [n_frames] or null
  // columns (one allocation each group)
  uint64_t *xcnt = nullptr, *icnt = nullptr;
  uint64_t* mcols = nullptr;  // [8][M][N]: xsum,xmin,xsq_lo,xsq_hi,isum,imin,isq_lo,isq_hi
  uint64_t *xsamples = nullptr, *isamples = nullptr, *xstall = nullptr, *istall = nullptr;
  uint32_t *pc_ctx = nullptr, *pc_off = nullptr, *bin_pcnode = nullptr;
  uint16_t* bin_stall = nullptr;
  uint64_t* bin_count = nullptr;
  // merge partition (dc_cct_merge_ranks output): unique node / bin records, see merge.cu
  bool partition = false;
  uint64_t* part_nodes = nullptr;
  uint64_t* part_bins = nullptr;
  uint64_t part_nbins = 0;
  uint32_t part_W = 0;
  bool part_has_pc = false;
  uint64_t* col(int which, uint32_t m) const { return mcols + ((uint64_t)which * M + m) * N; }
};
enum { C_XSUM = 0, C_XMIN, C_XSQLO, C_XSQHI, C_ISUM, C_IMIN, C_ISQLO, C_ISQHI };

namespace dc {

// Scope guard of a library handle under construction: frees it (and every array it holds)
// when an error returns early; set h = nullptr to hand it out.
template <class H, void (*FreeFn)(H*)>
struct HandleGuard {
  H* h;
  ~HandleGuard() {
    if (h) FreeFn(h);
  }
};

#define DC_TRY(expr)                      \
  do {                                    \
    dc_status _s = (expr);                \
    if (_s != DC_OK) return _s;           \
  } while (0)

dc_status cuda_fail(Ctx* c, cudaError_t e, const char* what);
dc_status fail(Ctx* c, dc_status s, const char* fmt, ...);

#define DC_CUDA(ctx, expr)                                           \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) return ::dc::cuda_fail((ctx), _e, #expr); \
  } while (0)

// after a kernel launch: count it and check the launch error
#define DC_STR2(x) #x
#define DC_STR(x) DC_STR2(x)
// Raise a kernel's dynamic shared-memory cap to the device's opt-in maximum (less its static
// shared memory), once per context
// (the cap only permits larger launches; every context sets the same value, so contexts on one
// device never lower each other's setting)
#define DC_SMEM_OPTIN(ctx, kern)                                                                          \
  do {                                                                                                   \
    const void* k_ = (const void*)(kern);                                                                \
    bool set_ = false;                                                                                   \
    for (const void* q_ : (ctx)->smem_set) set_ |= q_ == k_;                                             \
    if (!set_) {                                                                                         \
      cudaFuncAttributes fa_;                                                                            \
      DC_CUDA(ctx, cudaFuncGetAttributes(&fa_, k_));                                                     \
      DC_CUDA(ctx, cudaFuncSetAttribute(k_, cudaFuncAttributeMaxDynamicSharedMemorySize,                 \
                                        (int)((ctx)->smem_optin - fa_.sharedSizeBytes)));                \
      (ctx)->smem_set.push_back(k_);                                                                     \
    }                                                                                                    \
  } while (0)
#define DC_LAUNCHED(ctx)                                                                              \
  do {                                                                                                \
    (ctx)->launches++;                                                                                \
    cudaError_t _e = cudaGetLastError();                                                              \
    if (_e != cudaSuccess) return ::dc::cuda_fail((ctx), _e, "kernel launch at " __FILE__ ":" DC_STR(__LINE__)); \
  } while (0)

// Programmatic dependent launch. Every kernel of the library starts with DC_PDL_ENTER():
// griddepcontrol.wait blocks until the preceding grid on the stream has completed and its
// memory is visible (so the stream-order semantics are unchanged), then launch_dependents lets
// the NEXT grid's CTAs be scheduled while this one runs — they park at their own wait. This
// hides the launch latency of the ~45 short kernels of one step. When the
// previous stream operation is not a kernel (memset, memcpy, event) the attribute has no effect.
// Long, machine-filling kernels (the record and key passes, the PC histogram) use
// DC_PDL_WAIT() instead: they wait for their predecessor but do not let the next grid's CTAs
// be scheduled early — parked CTAs of a dependent grid on every SM during a 10-ms pass cost
// measurably (config 4 build: 37.5 ms with the early trigger vs 27.9 ms without); the next
// grid then launches when their CTAs exit, as without PDL.
#define DC_PDL_WAIT()                                  \
  do {                                                 \
    asm volatile("griddepcontrol.wait;" ::: "memory"); \
  } while (0)

#define DC_PDL_ENTER()                                 \
  do {                                                 \
    asm volatile("griddepcontrol.wait;" ::: "memory"); \
    asm volatile("griddepcontrol.launch_dependents;"); \
  } while (0)

bool pdl_enabled();  // env DC_NO_PDL=1 launches without the attribute (A/B measurement)

template <typename... KArgs, typename... Args>
inline void dc_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  // errors surface through cudaGetLastError in DC_LAUNCHED
  (void)cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// stream-ordered device allocation (memory pool); RAII buffer
template <class T>
struct Buf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool arena = false;  // carved from the context's scratch arena: nothing to free
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p(o.p), n(o.n), s(o.s), arena(o.arena) { o.p = nullptr; o.n = 0; }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; arena = o.arena; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~Buf() { release(); }
  void release() {
    if (p && !arena) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* release_ownership() {  // only for pool buffers (alloc_pool): arena memory is recycled
    T* q = arena ? nullptr : p;
    p = nullptr;
    n = 0;
    return q;
  }
};

void* arena_take(Ctx* c, size_t bytes);  // nullptr on OOM

// scratch buffer (arena; lives until the next public call)
template <class T>
dc_status alloc(Ctx* c, Buf<T>& b, size_t n) {
  b.release();
  b.s = c->stream;
  b.n = n;
  b.arena = true;
  b.p = (T*)arena_take(c, (n ? n : 1) * sizeof(T));
  if (!b.p) return fail(c, DC_ERR_OOM, "device allocation of %zu bytes failed", (n ? n : 1) * sizeof(T));
  return DC_OK;
}
// buffer from the pool (may be handed to a handle with release_ownership)
template <class T>
dc_status alloc_pool(Ctx* c, Buf<T>& b, size_t n) {
  HostRegion hr(c, "alloc");
  b.release();
  b.s = c->stream;
  b.n = n;
  b.arena = false;
  if (n == 0) n = 1;
  cudaError_t e = cudaMallocFromPoolAsync((void**)&b.p, n * sizeof(T), c->pool, c->stream);
  if (e != cudaSuccess) {
    b.p = nullptr;
    cudaGetLastError();
    return fail(c, DC_ERR_OOM, "device allocation of %zu bytes failed: %s", n * sizeof(T), cudaGetErrorString(e));
  }
  return DC_OK;
}
template <class T>
dc_status alloc_zero(Ctx* c, Buf<T>& b, size_t n) {
  DC_TRY(alloc(c, b, n));
  DC_CUDA(c, cudaMemsetAsync(b.p, 0, (n ? n : 1) * sizeof(T), c->stream));
  return DC_OK;
}
// persistent (handle-owned) allocation
template <class T>
dc_status palloc(Ctx* c, T*& p, size_t n) {
  HostRegion hr(c, "palloc");
  cudaError_t e = cudaMallocFromPoolAsync((void**)&p, (n ? n : 1) * sizeof(T), c->pool, c->stream);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return fail(c, DC_ERR_OOM, "device allocation of %zu bytes failed", n * sizeof(T));
  }
  return DC_OK;
}

// Several memsets as ONE kernel launch: a memset between two kernels breaks the programmatic
// dependent launch chain (the next kernel waits for a full launch latency), so the fills a
// stage needs are collected and issued together (fill_flush) before the stage's first kernel.
constexpr int FILL_MAX = 16;
struct FillList {
  void* p[FILL_MAX];
  uint64_t bytes[FILL_MAX];
  uint32_t byte[FILL_MAX];
  int n = 0;
};
__global__ void k_fill_multi(FillList f);
dc_status fill_flush(Ctx* c, FillList& f);
// device-to-device copy by a kernel (keeps the PDL chain)
dc_status dcopy(Ctx* c, void* dst, const void* src, uint64_t bytes);
// queue a fill of `bytes` bytes at p with the byte value v (flushes when the list is full)
dc_status fill_add(Ctx* c, FillList& f, void* p, uint64_t bytes, uint32_t v = 0);
template <class T>
dc_status alloc_fill(Ctx* c, FillList& f, Buf<T>& b, size_t n, uint32_t v = 0) {
  DC_TRY(alloc(c, b, n));
  return fill_add(c, f, b.p, (n ? n : 1) * sizeof(T), v);
}

// synchronous small readback through the pinned buffer
dc_status readback(Ctx* c, const void* dev, size_t bytes, void* host);
dc_status check_flags(Ctx* c);  // synchronizes; DC_ERR_TRACE if a flag is set
// several small readbacks behind one stream synchronisation (<= 4 KB in total)
struct RB {
  const void* dev;
  size_t bytes;
  void* host;
};
dc_status readback_multi(Ctx* c, std::initializer_list<RB> items);
// split-phase readback: _begin enqueues the copy kernel and records an event; work enqueued after
// it keeps the device busy while the host waits in _end for the event only (speculative launches
// whose kernels check the read values on the device themselves)
dc_status readback_begin(Ctx* c, std::initializer_list<RB> items);
dc_status readback_end(Ctx* c);
dc_status flags_status(Ctx* c, uint32_t flags);  // DC_ERR_TRACE if any flag bit is set
dc_status add_diag(Ctx* c, const unsigned long long* src_dev);  // d_diag[i] += src[i], i < DG_N

inline int grid_for(Ctx* c, uint64_t work, int per_block, int waves = 8) {
  uint64_t g = (work + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)c->num_sms * waves;
  if (g > cap) g = cap;
  return g ? (int)g : 1;
}

inline int bits_for(uint64_t v) {  // bits needed to represent values < v+1 (0 -> 0)
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 31;
  z *= 0x7FB5D329728EA185ull;
  z ^= z >> 27;
  z *= 0x81DADEF4BC2DD44Dull;
  z ^= z >> 33;
  return z;
}
// 16-B relaxed load at GPU scope (sees other CTAs' atomics; not guaranteed single-copy atomic,
// callers treat a half-empty result as "possibly torn" and resolve it with atomicCAS)
__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// 128-bit add into (lo, hi) device words with exact carry
__device__ __forceinline__ void atomic_add_u128(unsigned long long* lo, unsigned long long* hi, uint64_t add_lo,
                                                uint64_t add_hi) {
  unsigned long long old = atomicAdd(lo, (unsigned long long)add_lo);
  uint64_t carry = (old + add_lo) < old ? 1u : 0u;
  if (add_hi + carry) atomicAdd(hi, (unsigned long long)(add_hi + carry));
}

// ---------------------------------------------------------------- mbarrier / TMA bulk-copy helpers (sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Every device-side wait is bounded: a wait that outlives DC_SPIN_LIMIT polls is a bug (a lost
// arrival), and the kernel traps (a launch error the host reports) instead of hanging the GPU.
constexpr uint64_t DC_SPIN_LIMIT = 1ull << 28;
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  for (uint64_t i = 0; !mbar_try_wait(b, parity); ++i)
    if (i > DC_SPIN_LIMIT) __trap();
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
}  // namespace dc
