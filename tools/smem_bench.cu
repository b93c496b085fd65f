// smem_bench.cu — microbenchmark of shared-memory update primitives on this GPU (measurement
// only): per-SM throughput of 32-bit shared atomics / reductions / 16-B loads on random slots
// of a 96 KB table, 1 CTA x 1024 threads per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int T = 12224;  // u32 slots (~48 KB static limit)
constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, uint32_t hot_mask) {
  __shared__ __align__(16) uint32_t tab[T];
  for (int i = threadIdx.x; i < T; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t acc = 0, x = threadIdx.x * 0x9E3779B1u + blockIdx.x;
  for (int it = 0; it < ITERS; ++it) {
    x = hsh(x + it);
    uint32_t s = x % T;
    if ((x >> 24) < hot_mask) s = (x >> 8) & 7;  // a fraction of updates hits 8 hot slots
    if (MODE == 0) acc += atomicAdd(&tab[s], 1u);
    else if (MODE == 1) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&tab[s])), "r"(1u));
    else if (MODE == 2) {
      uint4 v = *reinterpret_cast<const uint4*>(&tab[s & ~3u]);
      acc += v.x ^ v.y ^ v.z ^ v.w;
    } else if (MODE == 3) {  // load + plain store (non-atomic RMW)
      uint32_t v = tab[s];
      tab[s] = v + 1;
    } else if (MODE == 4) {  // 16-B load + atomic (the histogram's per-sample pattern)
      uint4 v = *reinterpret_cast<const uint4*>(&tab[s & ~3u]);
      acc += v.x;
      atomicAdd(&tab[(s & ~3u) + (v.y & 3)], 1u);
    }
  }
  __syncthreads();
  if (acc == 0x12345u) out[0] = acc + tab[threadIdx.x];
}

template <int MODE>
float run(uint32_t* out, uint32_t hot) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<148, 1024>>>(out, hot);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<MODE><<<148, 1024>>>(out, hot);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 16);
  const char* names[] = {"atomicAdd(ret)", "red.shared.add", "lds.128", "lds+sts (non-atomic)", "lds.128+atomicAdd"};
  for (uint32_t hot : {0u, 26u}) {  // 0 % / ~10 % of updates on 8 hot slots
    float ms[5] = {run<0>(out, hot), run<1>(out, hot), run<2>(out, hot), run<3>(out, hot), run<4>(out, hot)};
    for (int m = 0; m < 5; ++m) {
      double ops_per_sm = 1024.0 * ITERS;
      double ns_per_op_sm = ms[m] * 1e6 / ops_per_sm;
      printf("{\"op\": \"%s\", \"hot_frac\": %.2f, \"ms\": %.4f, \"ns_per_lane_op_per_SM\": %.4f, \"cycles_at_1965MHz\": %.3f}\n",
             names[m], hot / 256.0, ms[m], ns_per_op_sm, ns_per_op_sm * 1.965);
    }
  }
  return 0;
}
