// capi.cu — the exported C ABI of libdc (include/dc.h): argument checks, handle state
// machine, context plumbing. Every compute step runs in the kernels of the other files.
#include <mutex>
#include <unordered_map>
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include "prim.cuh"

namespace dc {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DC_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

dc_status intern_frames(Ctx* c, const dc_frame_key* keys, uint64_t n, uint32_t* out_ids, dc_dict** out, uint64_t d_hint = 0);
dc_status dict_from_sorted(Ctx* c, const dc_frame_key* keys, uint64_t D, dc_dict** out);
dc_status cct_build(Ctx* c, const dc_paths* p, const dc_dict* dict, uint32_t n_frames, uint32_t* out_leaf, dc_cct** out);
dc_status attribute_metrics(Ctx* c, dc_cct* t, const uint32_t* leaf, uint64_t R, const uint64_t* X, uint32_t M, uint64_t ld);
dc_status rollup(Ctx* c, dc_cct* t);
dc_status pc_attribute(Ctx* c, dc_cct* t, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf, uint64_t n_launch,
                       const uint64_t* launch_off, uint32_t S);
dc_status analyze_flags(Ctx* c, const dc_cct* t, dc_rule rule, const dc_rule_params* p, uint32_t* out_h, uint32_t cap,
                        uint32_t* n_out_h);
dc_status analyze_stalls(Ctx* c, const dc_cct* t, uint32_t metric, uint32_t kind_mask, double hot_threshold,
                         double stall_threshold, uint32_t k, dc_stall_issue* out_h, uint32_t cap, uint32_t* n_out_h);
dc_status export_folded(Ctx* c, const dc_cct* t, uint32_t metric, uint32_t* node_h, uint64_t* value_h, uint64_t* off_h,
                        uint32_t* frames_h, uint64_t cap_lines, uint64_t cap_frames, uint64_t* n_lines_h, uint64_t* n_frames_h);
dc_status cpu_intervals(Ctx* c, const uint32_t* thread, const uint8_t* kind, const uint64_t* ts, uint64_t n,
                        uint64_t* out_interval, uint8_t* out_valid);
dc_status seq_associate(Ctx* c, const int64_t* fseq, const uint64_t* foff, const uint32_t* ffr, uint64_t nf, const int64_t* bseq,
                        const uint64_t* boff, const uint32_t* bfr, uint64_t nb, uint64_t* out_off, uint32_t* out_frames,
                        uint64_t cap_frames, uint64_t* n_frames_h, uint64_t* n_unmatched_h);
dc_status hotspots_topk(Ctx* c, const dc_cct* t, dc_view view, uint32_t metric, uint32_t kind_mask, double threshold,
                        uint32_t k, uint32_t stall_node, dc_topk_entry* out_h, uint32_t* n_out_h);
dc_status derived(Ctx* c, const dc_cct* t, uint32_t metric, int incl, double* mean, double* stdv);
dc_status cct_invert(Ctx* c, const dc_cct* t, uint32_t metric, dc_cct** out);

dc_status fail(Ctx* c, dc_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

dc_status cuda_fail(Ctx* c, cudaError_t e, const char* what) {
  return fail(c, DC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Small readbacks: one kernel copies up to RB_MAX items straight into the context's pinned
// buffer (device-accessible under unified addressing) instead of one DMA copy per item. The
// kernel is part of the PDL chain (launched while its predecessor runs, waiting for it with
// griddepcontrol.wait), so the readback costs no extra launch latency before the stream drains.
constexpr int RB_MAX = 8;
struct RbItems {
  const unsigned char* src[RB_MAX];
  uint32_t bytes[RB_MAX], off[RB_MAX];
  uint32_t n;
  unsigned char* dst;
};
__global__ void k_readback(RbItems it) { DC_PDL_ENTER();
  for (uint32_t i = 0; i < it.n; ++i)
    for (uint32_t b = threadIdx.x; b < it.bytes[i]; b += blockDim.x) it.dst[it.off[i] + b] = it.src[i][b];
}

dc_status readback(Ctx* c, const void* dev, size_t bytes, void* host) {
  if (bytes == 0) return DC_OK;
  HostRegion hr(c, "readback");
  if (bytes <= 4096) {
    RbItems it{};
    it.src[0] = (const unsigned char*)dev;
    it.bytes[0] = (uint32_t)bytes;
    it.n = 1;
    it.dst = (unsigned char*)c->h_pinned;
    dc_launch(k_readback, 1, 256, 0, c->stream, it);
    DC_LAUNCHED(c);
    flush_pending_frees(c);
    DC_CUDA(c, cudaStreamSynchronize(c->stream));
    memcpy(host, c->h_pinned, bytes);
  } else {
    DC_CUDA(c, cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    DC_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  return DC_OK;
}

dc_status readback_multi(Ctx* c, std::initializer_list<RB> items) {
  HostRegion hr(c, "readback");
  size_t o = 0;
  RbItems rb{};
  rb.dst = (unsigned char*)c->h_pinned;
  for (const RB& it : items) {
    if (o + it.bytes > 4096 || rb.n == RB_MAX) return fail(c, DC_ERR_ARG, "readback_multi: more than 4 KB or %d items", RB_MAX);
    if (it.bytes) {
      rb.src[rb.n] = (const unsigned char*)it.dev;
      rb.bytes[rb.n] = (uint32_t)it.bytes;
      rb.off[rb.n] = (uint32_t)o;
      ++rb.n;
    }
    o += (it.bytes + 7) & ~(size_t)7;
  }
  if (rb.n) {
    dc_launch(k_readback, 1, 256, 0, c->stream, rb);
    DC_LAUNCHED(c);
  }
  flush_pending_frees(c);
  DC_CUDA(c, cudaStreamSynchronize(c->stream));
  o = 0;
  for (const RB& it : items) {
    memcpy(it.host, (char*)c->h_pinned + o, it.bytes);
    o += (it.bytes + 7) & ~(size_t)7;
  }
  return DC_OK;
}

struct RBPending {
  void* host[RB_MAX];
  uint32_t bytes[RB_MAX], off[RB_MAX];
  uint32_t n = 0;
  bool active = false;
};
dc_status readback_begin(Ctx* c, std::initializer_list<RB> items) {
  if (!c->rb_pending) c->rb_pending = new RBPending();
  if (!c->rb_event) DC_CUDA(c, cudaEventCreateWithFlags(&c->rb_event, cudaEventDisableTiming));
  RBPending& pd = *c->rb_pending;
  pd.n = 0;
  RbItems rb{};
  rb.dst = (unsigned char*)c->h_pinned;
  size_t o = 0;
  for (const RB& it : items) {
    if (o + it.bytes > 4096 || rb.n == RB_MAX) return fail(c, DC_ERR_ARG, "readback_begin: more than 4 KB or %d items", RB_MAX);
    if (it.bytes) {
      rb.src[rb.n] = (const unsigned char*)it.dev;
      rb.bytes[rb.n] = (uint32_t)it.bytes;
      rb.off[rb.n] = (uint32_t)o;
      pd.host[rb.n] = it.host;
      pd.bytes[rb.n] = (uint32_t)it.bytes;
      pd.off[rb.n] = (uint32_t)o;
      ++rb.n;
    }
    o += (it.bytes + 7) & ~(size_t)7;
  }
  pd.n = rb.n;
  if (rb.n) {
    dc_launch(k_readback, 1, 256, 0, c->stream, rb);
    DC_LAUNCHED(c);
  }
  DC_CUDA(c, cudaEventRecord(c->rb_event, c->stream));
  pd.active = true;
  return DC_OK;
}
dc_status readback_end(Ctx* c) {
  HostRegion hr(c, "readback");
  RBPending& pd = *c->rb_pending;
  if (!pd.active) return fail(c, DC_ERR_STATE, "internal: readback_end without readback_begin");
  pd.active = false;
  flush_pending_frees(c);
  DC_CUDA(c, cudaEventSynchronize(c->rb_event));
  for (uint32_t i = 0; i < pd.n; ++i) memcpy(pd.host[i], (char*)c->h_pinned + pd.off[i], pd.bytes[i]);
  return DC_OK;
}

dc_status flags_status(Ctx* c, uint32_t f) {
  if (f) {
    const char* why = (f & FLAG_BAD_FRAME)    ? "frame id >= n_frames"
                      : (f & FLAG_BAD_KEY)    ? "raw frame key with reserved kind 0xFFFFFFFF"
                      : (f & FLAG_TOO_DEEP)   ? "call path deeper than DC_MAX_DEPTH"
                      : (f & FLAG_BAD_LEAF)   ? "leaf / launch_leaf entry is not a node of the tree"
                      : (f & FLAG_BAD_OFFSETS)? "record offsets are not non-decreasing"
                                              : "internal error";
    return fail(c, DC_ERR_TRACE, "malformed trace (flags 0x%x): %s", f, why);
  }
  return DC_OK;
}

// Contexts and the handles they made. A handle's arrays come from its context's private pool;
// the pool lives until the context is destroyed AND the last of its handles is freed.
struct CtxEntry {
  cudaStream_t stream;
  cudaMemPool_t pool;
  int device;
  bool live;
  uint64_t handles;
  // arrays of handles freed while the context is live: their stream-ordered frees are issued at
  // the context's next blocking point (readback, sync, trim, destroy), where the host waits for
  // the device anyway, instead of on the host's critical path between launches
  std::vector<void*> pending;
};
static std::mutex g_ctx_mu;
static std::unordered_map<uint64_t, CtxEntry> g_ctx;  // context uid -> entry
static uint64_t g_next_uid = 1;
static void drop_entry_locked(std::unordered_map<uint64_t, CtxEntry>::iterator it) {
  cudaSetDevice(it->second.device);
  cudaMemPoolDestroy(it->second.pool);
  g_ctx.erase(it);
}
void register_ctx(Ctx* c, bool live) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if (live) {
    c->uid = g_next_uid++;
    g_ctx[c->uid] = CtxEntry{c->stream, c->pool, c->device, true, 0, {}};
    return;
  }
  auto it = g_ctx.find(c->uid);
  if (it == g_ctx.end()) return;
  it->second.live = false;
  if (it->second.handles == 0) drop_entry_locked(it);
}
uint64_t adopt_handle(Ctx* c) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  auto it = g_ctx.find(c->uid);
  if (it != g_ctx.end()) it->second.handles++;
  return c->uid;
}
void free_handle_ptrs(uint64_t owner_uid, void* const* ps, size_t n) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  auto it = g_ctx.find(owner_uid);
  if (it == g_ctx.end()) return;  // not made by a context (nothing allocated)
  CtxEntry& e = it->second;
  if (e.live) {  // stream-ordered (after every queued use on the context stream), deferred
    for (size_t i = 0; i < n; ++i)
      if (ps[i]) e.pending.push_back(ps[i]);
  } else {  // the context is gone: free in order after all device work
    cudaSetDevice(e.device);
    cudaDeviceSynchronize();
    for (size_t i = 0; i < n; ++i)
      if (ps[i]) cudaFreeAsync(ps[i], 0);
    cudaStreamSynchronize(0);
  }
  if (e.handles) e.handles--;
  if (!e.live && e.handles == 0) drop_entry_locked(it);
}

void flush_pending_frees(Ctx* c) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  auto it = g_ctx.find(c->uid);
  if (it == g_ctx.end()) return;
  for (void* p : it->second.pending) cudaFreeAsync(p, it->second.stream);
  it->second.pending.clear();
}

dc_status check_flags(Ctx* c) {
  uint32_t f = 0;
  DC_TRY(readback(c, c->d_flags, 4, &f));
  if (f) {
    const char* why = (f & FLAG_BAD_FRAME)    ? "frame id >= n_frames"
                      : (f & FLAG_BAD_KEY)    ? "raw frame key with reserved kind 0xFFFFFFFF"
                      : (f & FLAG_TOO_DEEP)   ? "call path deeper than DC_MAX_DEPTH"
                      : (f & FLAG_BAD_LEAF)   ? "leaf / launch_leaf entry is not a node of the tree"
                      : (f & FLAG_BAD_OFFSETS)? "record offsets are not non-decreasing"
                                              : "internal error";
    return fail(c, DC_ERR_TRACE, "malformed trace (flags 0x%x): %s", f, why);
  }
  return DC_OK;
}

void* arena_take(Ctx* c, size_t bytes) {
  HostRegion hr(c, "alloc");
  bytes = (bytes + 255) & ~(size_t)255;
  while (c->arena_ci < c->arena.size()) {
    auto& ch = c->arena[c->arena_ci];
    if (c->arena_off + bytes <= ch.second) {
      void* p = ch.first + c->arena_off;
      c->arena_off += bytes;
      return p;
    }
    ++c->arena_ci;
    c->arena_off = 0;
  }
  size_t sz = (size_t)64 << 20;
  if (!c->arena.empty() && 2 * c->arena.back().second > sz) sz = 2 * c->arena.back().second;
  if (bytes > sz) sz = bytes;
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, sz, c->pool, c->stream) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  c->arena.push_back({(char*)p, sz});
  c->arena_ci = c->arena.size() - 1;
  c->arena_off = bytes;
  return p;
}

static void arena_free(Ctx* c) {  // after a stream synchronisation
  for (auto& ch : c->arena) cudaFreeAsync(ch.first, c->stream);
  c->arena.clear();
  c->arena_reset();
}

__global__ void k_fill_multi(FillList f) { DC_PDL_ENTER();
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < f.n; ++r) {
    const uint32_t v = f.byte[r] & 0xFFu;
    const uint64_t pat = v * 0x0101010101010101ull;
    const uint64_t words = f.bytes[r] / 8;
    uint64_t* p8 = (uint64_t*)f.p[r];  // arena / pool memory: 256-byte aligned
    if (((uintptr_t)p8 & 7) == 0) {
      for (uint64_t i = tid; i < words; i += nt) p8[i] = pat;
      for (uint64_t i = words * 8 + tid; i < f.bytes[r]; i += nt) ((uint8_t*)f.p[r])[i] = (uint8_t)v;
    } else {
      for (uint64_t i = tid; i < f.bytes[r]; i += nt) ((uint8_t*)f.p[r])[i] = (uint8_t)v;
    }
  }
}

dc_status fill_flush(Ctx* c, FillList& f) {
  if (!f.n) return DC_OK;
  uint64_t tot = 0;
  for (int i = 0; i < f.n; ++i) tot += f.bytes[i];
  dc_launch(k_fill_multi, grid_for(c, tot / 8 + 1, 256), 256, 0, c->stream, f);
  DC_LAUNCHED(c);
  f.n = 0;
  return DC_OK;
}

// device-to-device copy as a kernel (stays in the PDL chain; a DMA copy between two PDL-chained
// kernels makes the next one pay a full launch latency)
__global__ void k_copy_bytes(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src, uint64_t bytes) { DC_PDL_ENTER();
  const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const uint64_t n16 = bytes / 16;
    for (uint64_t i = i0; i < n16; i += st) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (uint64_t i = 16 * n16 + i0; i < bytes; i += st) dst[i] = src[i];
  } else {
    for (uint64_t i = i0; i < bytes; i += st) dst[i] = src[i];
  }
}
dc_status dcopy(Ctx* c, void* dst, const void* src, uint64_t bytes) {
  if (!bytes) return DC_OK;
  dc_launch(k_copy_bytes, grid_for(c, bytes / 16 + 1, 256), 256, 0, c->stream, (unsigned char*)dst, (const unsigned char*)src, bytes);
  DC_LAUNCHED(c);
  return DC_OK;
}

dc_status fill_add(Ctx* c, FillList& f, void* p, uint64_t bytes, uint32_t v) {
  if (f.n == FILL_MAX) DC_TRY(fill_flush(c, f));
  f.p[f.n] = p;
  f.bytes[f.n] = bytes;
  f.byte[f.n] = v;
  ++f.n;
  return DC_OK;
}

dc_status scan_state(Ctx* c, uint64_t n_tiles, uint64_t** flag, uint64_t** val, uint64_t* seq, Buf<uint64_t>& tmp) {
  constexpr uint64_t CAP = 1ull << 16;
  if (!c->scan_ctr) {  // first use: persistent, zeroed once (flags carry a call sequence number)
    if (cudaMalloc(&c->scan_flag, CAP * 8) != cudaSuccess || cudaMalloc(&c->scan_val, 4 * CAP * 8) != cudaSuccess ||
        cudaMalloc(&c->scan_ctr, 8) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, DC_ERR_OOM, "scan state allocation failed");
    }
    DC_CUDA(c, cudaMemsetAsync(c->scan_flag, 0, CAP * 8, c->stream));
    DC_CUDA(c, cudaMemsetAsync(c->scan_ctr, 0, 8, c->stream));
    c->scan_cap = CAP;
  }
  if (n_tiles <= c->scan_cap) {
    *flag = c->scan_flag;
    *val = c->scan_val;
    *seq = ++c->scan_seq;
    return DC_OK;
  }
  // more tiles than the persistent state holds: fresh zeroed state for this call
  DC_TRY(alloc_zero(c, tmp, 5 * n_tiles));
  *flag = tmp.p;
  *val = tmp.p + n_tiles;
  *seq = 1;
  return DC_OK;
}

__global__ void k_add_diag(unsigned long long* dst, const unsigned long long* src) { DC_PDL_ENTER();
  if (threadIdx.x < DG_N) dst[threadIdx.x] += src[threadIdx.x];
}

dc_status add_diag(Ctx* c, const unsigned long long* src_dev) {
  dc_launch(k_add_diag, 1, 32, 0, c->stream, (unsigned long long*)c->d_diag, src_dev);
  DC_LAUNCHED(c);
  return DC_OK;
}

}  // namespace dc

using namespace dc;

#define CHECK_CTX(ctx) \
  if (!(ctx)) return DC_ERR_ARG
#define ARG(cond, ...)                                     \
  do {                                                     \
    if (!(cond)) return fail(ctx, DC_ERR_ARG, __VA_ARGS__); \
  } while (0)
// every public call starts on the context's device with the scratch arena rewound
#define ON_DEVICE(ctx)                                 \
  do {                                                 \
    DC_CUDA(ctx, cudaSetDevice((ctx)->device));        \
    (ctx)->arena_reset();                              \
  } while (0)

extern "C" {

dc_status dc_ctx_create(int device, void* cuda_stream, dc_ctx** out) {
  if (!out) return DC_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return DC_ERR_CUDA;
  }
  dc_ctx* ctx = new dc_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return DC_ERR_CUDA;
  }
  // the caller's stream, used as given (NULL = the legacy default stream), so the library is
  // ordered with the caller's producers/consumers of the device buffers on that stream
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->own_stream = false;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  ctx->num_sms = prop.multiProcessorCount;
  if (const char* w = getenv("DC_TEST_WEAK_HASH")) {  // test-only fault injection (collision paths)
    int b = atoi(w);
    if (b > 0 && b < 64) ctx->hash_mask = (1ull << b) - 1ull;
  }
  if (const char* w = getenv("DC_TEST_WEAK_NODE_HASH")) {
    int b = atoi(w);
    if (b > 0 && b < 64) ctx->node_mask = (1ull << b) - 1ull;
  }
  if (const char* w = getenv("DC_TEST_WEAK_MERGE_HASH")) {
    int b = atoi(w);
    if (b > 0 && b < 64) ctx->merge_mask = (1ull << b) - 1ull;
  }
  ctx->smem_optin = prop.sharedMemPerBlockOptin;
  // the context's private pool; freed memory stays cached in it (stream-ordered allocations are
  // reused across calls) without touching the device's default pool
  {
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    if (cudaMemPoolCreate(&ctx->pool, &pp) != cudaSuccess) {
      cudaGetLastError();
      delete ctx;
      return DC_ERR_CUDA;
    }
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (cudaMalloc(&ctx->d_flags, 4) != cudaSuccess || cudaMalloc(&ctx->d_diag, DG_N * 8) != cudaSuccess ||
      cudaMallocHost(&ctx->h_pinned, 4096) != cudaSuccess) {
    cudaGetLastError();
    cudaMemPoolDestroy(ctx->pool);
    delete ctx;
    return DC_ERR_OOM;
  }
  cudaMemsetAsync(ctx->d_flags, 0, 4, ctx->stream);
  cudaMemsetAsync(ctx->d_diag, 0, DG_N * 8, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  dc::register_ctx(ctx, true);
  *out = ctx;
  return DC_OK;
}

dc_status dc_ctx_sync(dc_ctx* ctx) {
  CHECK_CTX(ctx);
  ON_DEVICE(ctx);
  flush_pending_frees(ctx);
  DC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return check_flags(ctx);
}

dc_status dc_ctx_diag(dc_ctx* ctx, dc_diag* out_h) {
  CHECK_CTX(ctx);
  ARG(out_h, "out_h is NULL");
  ON_DEVICE(ctx);
  uint64_t d[DG_N];
  DC_TRY(readback(ctx, ctx->d_diag, sizeof d, d));
  out_h->empty_paths = d[DG_EMPTY];
  out_h->samples_bad_launch = d[DG_BAD_LAUNCH];
  out_h->samples_bad_stall = d[DG_BAD_STALL];
  out_h->samples_zero_count = d[DG_ZERO];
  out_h->collisions_detected = d[DG_COLL] + ctx->host_collisions;
  out_h->levels_built = ctx->host_levels;
  out_h->max_depth_seen = d[DG_MAXDEPTH];
  out_h->bytes_moved_est = ctx->bytes_host;
  return DC_OK;
}

void dc_ctx_destroy(dc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  dc::flush_pending_frees(ctx);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  arena_free(ctx);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_diag);
  cudaFree(ctx->scan_flag);
  cudaFree(ctx->scan_val);
  cudaFree(ctx->scan_ctr);
  cudaFreeHost(ctx->h_pinned);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->rb_event) cudaEventDestroy(ctx->rb_event);
  delete ctx->rb_pending;
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  // outstanding handles keep their arrays: the pool is destroyed once the last one is freed
  // (handles outliving the context free synchronously from now on)
  dc::register_ctx(ctx, false);
  delete ctx;
}

const char* dc_last_error(const dc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
uint64_t dc_ctx_launch_count(const dc_ctx* ctx) { return ctx ? ctx->launches : 0; }

dc_status dc_ctx_set_timing(dc_ctx* ctx, int on) {
  CHECK_CTX(ctx);
  ctx->timing = on != 0;
  return DC_OK;
}

dc_status dc_ctx_reserve(dc_ctx* ctx, uint64_t bytes) {
  CHECK_CTX(ctx);
  ON_DEVICE(ctx);
  if (!bytes) return DC_OK;
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, DC_ERR_OOM, "dc_ctx_reserve: cannot reserve %llu bytes", (unsigned long long)bytes);
  }
  DC_CUDA(ctx, cudaFreeAsync(p, ctx->stream));
  DC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return DC_OK;
}

dc_status dc_ctx_trim(dc_ctx* ctx, uint64_t keep_bytes) {
  CHECK_CTX(ctx);
  ON_DEVICE(ctx);
  flush_pending_frees(ctx);
  DC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  arena_free(ctx);
  DC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  DC_CUDA(ctx, cudaMemPoolTrimTo(ctx->pool, keep_bytes));
  return DC_OK;
}

dc_status dc_ctx_timer_report(dc_ctx* ctx, char* buf, size_t len) {
  CHECK_CTX(ctx);
  ARG(buf && len, "buf is NULL");
  ON_DEVICE(ctx);
  DC_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<std::string> names;
  std::vector<double> tot;
  std::vector<uint64_t> cnt;
  for (auto& t : ctx->timed) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    size_t i = 0;
    while (i < names.size() && names[i] != t.name) ++i;
    if (i == names.size()) {
      names.push_back(t.name);
      tot.push_back(0);
      cnt.push_back(0);
    }
    tot[i] += ms;
    cnt[i] += 1;
  }
  ctx->timed.clear();
  ctx->ev_next = 0;  // the events are reused by the next timed regions
  for (auto& h : ctx->htimed) {
    std::string nm = std::string("h:") + h.name;
    size_t i = 0;
    while (i < names.size() && names[i] != nm) ++i;
    if (i == names.size()) {
      names.push_back(nm);
      tot.push_back(0);
      cnt.push_back(0);
    }
    tot[i] += h.ms;
    cnt[i] += 1;
  }
  ctx->htimed.clear();
  std::string s;
  char line[256];
  for (size_t i = 0; i < names.size(); ++i) {
    snprintf(line, sizeof line, "%s %llu %.6f\n", names[i].c_str(), (unsigned long long)cnt[i], tot[i]);
    s += line;
  }
  snprintf(buf, len, "%s", s.c_str());
  return DC_OK;
}

dc_status dc_intern_frames(dc_ctx* ctx, const dc_frame_key* keys, uint64_t n, uint32_t* out_ids, dc_dict** out_dict) {
  CHECK_CTX(ctx);
  ARG(out_dict, "out_dict is NULL");
  ARG(n == 0 || (keys && out_ids), "keys/out_ids must be device pointers when n > 0");
  ARG(((uintptr_t)keys & 15) == 0, "keys must be 16-byte aligned");
  ON_DEVICE(ctx);
  Region rg(ctx, "intern");
  return intern_frames(ctx, keys, n, out_ids, out_dict);
}

dc_status dc_dict_from_sorted(dc_ctx* ctx, const dc_frame_key* keys, uint64_t D, dc_dict** out_dict) {
  CHECK_CTX(ctx);
  ARG(out_dict && (D == 0 || keys), "bad arguments");
  ON_DEVICE(ctx);
  return dict_from_sorted(ctx, keys, D, out_dict);
}

uint64_t dc_dict_size(const dc_dict* d) { return d ? d->D : 0; }

dc_status dc_dict_arrays(const dc_dict* d, const dc_frame_key** keys_dev, const uint8_t** kinds_dev) {
  if (!d) return DC_ERR_ARG;
  if (keys_dev) *keys_dev = d->keys;
  if (kinds_dev) *kinds_dev = d->kinds;
  return DC_OK;
}

void dc_dict_free(dc_dict* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  void* ps[] = {d->keys, d->kinds};
  dc::free_handle_ptrs(d->owner_uid, ps, 2);
  delete d;
}

dc_status dc_cct_build(dc_ctx* ctx, const dc_paths* paths, const dc_dict* dict, uint32_t n_frames, uint32_t* out_leaf,
                       dc_cct** out) {
  CHECK_CTX(ctx);
  ARG(paths && out, "paths/out is NULL");
  ARG(paths->offsets, "paths->offsets is NULL");
  ARG(!dict || dict->D == n_frames, "dictionary size %llu != n_frames %u", (unsigned long long)(dict ? dict->D : 0), n_frames);
  ARG(n_frames < 0xFFFFFFFFu, "n_frames must be < 2^32-1");
  ON_DEVICE(ctx);
  if (!paths->frames && paths->n_records) {  // allowed only when every path is empty
    uint64_t F = 0;
    DC_TRY(readback(ctx, paths->offsets + paths->n_records, 8, &F));
    ARG(F == 0, "paths->frames is NULL but offsets[n_records] = %llu", (unsigned long long)F);
  }
  Region rg(ctx, "build");
  return cct_build(ctx, paths, dict, n_frames, out_leaf, out);
}

dc_status dc_cct_attribute_metrics(dc_ctx* ctx, dc_cct* cct, const uint32_t* leaf, uint64_t n_records, const uint64_t* metrics,
                                   uint32_t M, uint64_t ld) {
  CHECK_CTX(ctx);
  ARG(cct, "cct is NULL");
  ARG(M > 0 && M <= 64, "M must be in [1, 64]");
  ARG(n_records == 0 || (leaf && metrics), "leaf/metrics must be device pointers");
  ARG(ld >= n_records, "ld < n_records");
  ON_DEVICE(ctx);
  Region rg(ctx, "attribute");
  return attribute_metrics(ctx, cct, leaf, n_records, metrics, M, ld);
}

dc_status dc_cct_rollup(dc_ctx* ctx, dc_cct* cct) {
  CHECK_CTX(ctx);
  ARG(cct, "cct is NULL");
  ON_DEVICE(ctx);
  Region rg(ctx, "rollup");
  return rollup(ctx, cct);
}

dc_status dc_pc_sample_attribute(dc_ctx* ctx, dc_cct* cct, const dc_pc_sample* s, uint64_t n, const uint32_t* launch_leaf,
                                 uint64_t n_launch, const uint64_t* launch_sample_off, uint32_t n_stall) {
  CHECK_CTX(ctx);
  ARG(cct, "cct is NULL");
  ARG(n_stall >= 1 && n_stall <= DC_MAX_STALL, "n_stall must be in [1, %u]", DC_MAX_STALL);
  ARG(n == 0 || s, "samples pointer is NULL");
  ARG(n_launch == 0 || launch_leaf, "launch_leaf is NULL");
  ARG(((uintptr_t)s & 15) == 0, "samples must be 16-byte aligned");
  if (cct->partition) return fail(ctx, DC_ERR_STATE, "a merged partition is read-only");
  // repeated calls accumulate (e.g. one call per chunk of samples); S is fixed by the first
  if (cct->pc_done && n_stall != cct->S)
    return fail(ctx, DC_ERR_ARG, "n_stall %u differs from the first call's %u", n_stall, cct->S);
  ON_DEVICE(ctx);
  Region rg(ctx, "pc");
  return pc_attribute(ctx, cct, s, n, launch_leaf, n_launch, launch_sample_off, n_stall);
}

dc_status dc_hotspots_topk(dc_ctx* ctx, const dc_cct* cct, dc_view view, uint32_t metric, uint32_t kind_mask, double threshold,
                           uint32_t k, uint32_t stall_node, dc_topk_entry* out_h, uint32_t* n_out_h) {
  CHECK_CTX(ctx);
  ARG(cct && n_out_h && (k == 0 || out_h), "bad arguments");
  ON_DEVICE(ctx);
  Region rg(ctx, "topk");
  return hotspots_topk(ctx, cct, view, metric, kind_mask, threshold, k, stall_node, out_h, n_out_h);
}

dc_status dc_analyze_flags(dc_ctx* ctx, const dc_cct* cct, dc_rule rule, const dc_rule_params* params, uint32_t* out_ids_h,
                           uint32_t cap, uint32_t* n_out_h) {
  CHECK_CTX(ctx);
  ARG(cct && params && n_out_h && (cap == 0 || out_ids_h), "bad arguments");
  ON_DEVICE(ctx);
  Region rg(ctx, "rules");
  return analyze_flags(ctx, cct, rule, params, out_ids_h, cap, n_out_h);
}

dc_status dc_analyze_stalls(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, uint32_t kind_mask, double hot_threshold,
                            double stall_threshold, uint32_t k, dc_stall_issue* out_h, uint32_t cap, uint32_t* n_out_h) {
  CHECK_CTX(ctx);
  ARG(cct && n_out_h && (cap == 0 || out_h), "bad arguments");
  ON_DEVICE(ctx);
  Region rg(ctx, "rules");
  return analyze_stalls(ctx, cct, metric, kind_mask, hot_threshold, stall_threshold, k, out_h, cap, n_out_h);
}

dc_status dc_export_folded(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, uint32_t* node_h, uint64_t* value_h,
                           uint64_t* off_h, uint32_t* frames_h, uint64_t cap_lines, uint64_t cap_frames, uint64_t* n_lines_h,
                           uint64_t* n_frames_h) {
  CHECK_CTX(ctx);
  ARG(cct && n_lines_h && n_frames_h, "bad arguments");
  ARG((cap_lines == 0 || (node_h && value_h && off_h)) && (cap_frames == 0 || frames_h), "bad arguments");
  ON_DEVICE(ctx);
  Region rg(ctx, "export");
  return export_folded(ctx, cct, metric, node_h, value_h, off_h, frames_h, cap_lines, cap_frames, n_lines_h, n_frames_h);
}

dc_status dc_cct_invert(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, dc_cct** out) {
  CHECK_CTX(ctx);
  ARG(cct && out, "bad arguments");
  ON_DEVICE(ctx);
  Region rg(ctx, "invert");
  return cct_invert(ctx, cct, metric, out);
}

dc_status dc_cpu_intervals(dc_ctx* ctx, const uint32_t* thread, const uint8_t* kind, const uint64_t* ts, uint64_t n,
                           uint64_t* out_interval, uint8_t* out_valid) {
  CHECK_CTX(ctx);
  ARG(n == 0 || (thread && kind && ts && out_interval && out_valid), "bad arguments");
  ON_DEVICE(ctx);
  Region rg(ctx, "intervals");
  return cpu_intervals(ctx, thread, kind, ts, n, out_interval, out_valid);
}

dc_status dc_seq_associate(dc_ctx* ctx, const int64_t* fwd_seq, const uint64_t* fwd_off, const uint32_t* fwd_frames,
                           uint64_t nf, const int64_t* bwd_seq, const uint64_t* bwd_off, const uint32_t* bwd_frames,
                           uint64_t nb, uint64_t* out_off, uint32_t* out_frames, uint64_t cap_frames, uint64_t* n_frames_h,
                           uint64_t* n_unmatched_h) {
  CHECK_CTX(ctx);
  ARG(n_frames_h && n_unmatched_h && out_off, "bad arguments");
  ARG(nf == 0 || (fwd_seq && fwd_off), "bad forward registry");
  ARG(nb == 0 || (bwd_seq && bwd_off), "bad backward records");
  ON_DEVICE(ctx);
  Region rg(ctx, "associate");
  return seq_associate(ctx, fwd_seq, fwd_off, fwd_frames, nf, bwd_seq, bwd_off, bwd_frames, nb, out_off, out_frames, cap_frames,
                       n_frames_h, n_unmatched_h);
}

dc_status dc_cct_derived(dc_ctx* ctx, const dc_cct* cct, uint32_t metric, int incl, double* out_mean, double* out_std) {
  CHECK_CTX(ctx);
  ARG(cct && out_mean && out_std, "bad arguments");
  ON_DEVICE(ctx);
  return derived(ctx, cct, metric, incl, out_mean, out_std);
}

dc_status dc_cct_view_get(const dc_cct* t, dc_cct_view* v) {
  if (!t || !v) return DC_ERR_ARG;
  memset(v, 0, sizeof *v);
  v->n_nodes = t->N;
  v->n_pc_nodes = t->Npc;
  v->n_bins = t->Nbins;
  v->n_records = t->R;
  v->n_metrics = t->M;
  v->n_stall = t->S;
  v->max_depth = t->max_depth;
  v->n_frames = t->n_frames;
  v->parent = t->parent;
  v->frame = t->frame;
  v->depth = t->depth;
  v->level_off = t->level_off;
  v->xcnt = t->xcnt;
  v->icnt = t->icnt;
  if (t->mcols) {
    v->xsum = t->col(C_XSUM, 0);
    v->xmin = t->col(C_XMIN, 0);
    v->xsq_lo = t->col(C_XSQLO, 0);
    v->xsq_hi = t->col(C_XSQHI, 0);
    v->isum = t->col(C_ISUM, 0);
    v->imin = t->col(C_IMIN, 0);
    v->isq_lo = t->col(C_ISQLO, 0);
    v->isq_hi = t->col(C_ISQHI, 0);
  }
  v->xsamples = t->xsamples;
  v->isamples = t->isamples;
  v->xstall = t->xstall;
  v->istall = t->istall;
  v->pc_ctx = t->pc_ctx;
  v->pc_off = t->pc_off;
  v->bin_pcnode = t->bin_pcnode;
  v->bin_stall = t->bin_stall;
  v->bin_count = t->bin_count;
  v->state = t->state;
  if (t->state != 2) {  // inclusive columns are defined only after dc_cct_rollup
    v->icnt = v->isum = v->imin = v->isq_lo = v->isq_hi = v->isamples = v->istall = nullptr;
    return DC_ERR_STATE;
  }
  return DC_OK;
}

void dc_cct_free(dc_cct* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  void* ps[] = {t->parent, t->frame, t->level_off, t->depth, t->frame_kind, t->xcnt, t->icnt, t->mcols, t->xsamples,
                t->isamples, t->xstall, t->istall, t->pc_ctx, t->pc_off, t->bin_pcnode, t->bin_stall, t->bin_count,
                t->part_nodes, t->part_bins};
  dc::free_handle_ptrs(t->owner_uid, ps, sizeof ps / sizeof ps[0]);
  delete t;
}

}  // extern "C"
