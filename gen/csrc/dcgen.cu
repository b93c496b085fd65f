// dcgen.cu — host loops and device kernels of the synthetic trace generator (TEST/BENCH
// INPUT ONLY; see gen_core.h). Host and device paths call the same gen_core.h draw
// functions, so for equal program tables they emit byte-identical arrays.
#include <cuda_runtime.h>
#include <string.h>
#include "gen_core.h"

extern "C" {

/* ---------------- host ---------------- */
void dcgen_lengths_host(const gen_prog* p, uint64_t r0, uint64_t n, uint32_t* out_len) {
  for (uint64_t i = 0; i < n; ++i) out_len[i] = gen_record_shape(p, r0 + i).len;
}

/* frames: off[n+1] relative offsets (off[0] may be nonzero: base of the output arrays).
   out_ids (u32) and/or out_keys (16 B) may be NULL. */
void dcgen_frames_host(const gen_prog* p, uint64_t r0, uint64_t n, const uint64_t* off,
                       const gen_key* pool, uint32_t* out_ids, gen_key* out_keys) {
  for (uint64_t i = 0; i < n; ++i) {
    gen_shape s = gen_record_shape(p, r0 + i);
    uint64_t o = off[i] - off[0];
    for (uint32_t j = 0; j < s.len; ++j) {
      uint32_t f = gen_record_frame(p, &s, j);
      if (out_ids) out_ids[o + j] = f;
      if (out_keys) out_keys[o + j] = pool[f];
    }
  }
}

/* metrics column-major [M][ld] */
void dcgen_metrics_host(const gen_prog* p, uint64_t r0, uint64_t n, uint64_t* out, uint64_t ld) {
  for (uint64_t i = 0; i < n; ++i) {
    gen_shape s = gen_record_shape(p, r0 + i);
    for (uint32_t m = 0; m < p->n_metrics; ++m) out[m * ld + i] = gen_record_metric(p, &s, r0 + i, m);
  }
}

/* samples of launches [l0, l1): written at out[launch_off[l] - launch_off[l0] ...] */
void dcgen_pc_host(const gen_pc_prog* q, uint32_t l0, uint32_t l1, gen_pc_sample* out) {
  uint64_t base = q->launch_off[l0];
  for (uint32_t l = l0; l < l1; ++l)
    for (uint64_t i = q->launch_off[l]; i < q->launch_off[l + 1]; ++i) out[i - base] = gen_pc_draw(q, l, i);
}

/* ---------------- device ---------------- */
__global__ void k_lengths(gen_prog p, uint64_t r0, uint64_t n, uint32_t* out_len) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out_len[i] = gen_record_shape(&p, r0 + i).len;
}

/* one warp per record: lanes write consecutive frames (coalesced) */
__global__ void k_frames(gen_prog p, uint64_t r0, uint64_t n, const uint64_t* off, const gen_key* pool,
                         uint32_t* out_ids, gen_key* out_keys) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t off0 = off[0];
  for (uint64_t i = warp; i < n; i += nwarps) {
    gen_shape s = gen_record_shape(&p, r0 + i);
    uint64_t o = off[i] - off0;
    for (uint32_t j = lane; j < s.len; j += 32) {
      uint32_t f = gen_record_frame(&p, &s, j);
      if (out_ids) out_ids[o + j] = f;
      if (out_keys) out_keys[o + j] = pool[f];
    }
  }
}

__global__ void k_metrics(gen_prog p, uint64_t r0, uint64_t n, uint64_t* out, uint64_t ld) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    gen_shape s = gen_record_shape(&p, r0 + i);
    for (uint32_t m = 0; m < p.n_metrics; ++m) out[m * ld + i] = gen_record_metric(&p, &s, r0 + i, m);
  }
}

/* one block per launch (grid-stride over launches) */
__global__ void k_pc(gen_pc_prog q, uint32_t l0, uint32_t l1, gen_pc_sample* out) {
  uint64_t base = q.launch_off[l0];
  for (uint32_t l = l0 + blockIdx.x; l < l1; l += gridDim.x)
    for (uint64_t i = q.launch_off[l] + threadIdx.x; i < q.launch_off[l + 1]; i += blockDim.x)
      out[i - base] = gen_pc_draw(&q, l, i);
}

static int grid_for(uint64_t n, int per) {
  uint64_t g = (n + per - 1) / per;
  if (g > 148 * 64) g = 148 * 64;
  return g ? (int)g : 1;
}

int dcgen_lengths_dev(const gen_prog* p, uint64_t r0, uint64_t n, uint32_t* out_len, void* stream) {
  k_lengths<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*p, r0, n, out_len);
  return (int)cudaGetLastError();
}
int dcgen_frames_dev(const gen_prog* p, uint64_t r0, uint64_t n, const uint64_t* off, const gen_key* pool,
                     uint32_t* out_ids, gen_key* out_keys, void* stream) {
  k_frames<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(*p, r0, n, off, pool, out_ids, out_keys);
  return (int)cudaGetLastError();
}
int dcgen_metrics_dev(const gen_prog* p, uint64_t r0, uint64_t n, uint64_t* out, uint64_t ld, void* stream) {
  k_metrics<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*p, r0, n, out, ld);
  return (int)cudaGetLastError();
}
int dcgen_pc_dev(const gen_pc_prog* q, uint32_t l0, uint32_t l1, gen_pc_sample* out, void* stream) {
  uint32_t nl = l1 - l0;
  k_pc<<<nl < 148 * 16 ? (nl ? nl : 1) : 148 * 16, 256, 0, (cudaStream_t)stream>>>(*q, l0, l1, out);
  return (int)cudaGetLastError();
}

}  // extern "C"
