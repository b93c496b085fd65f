// tma_bench.cu — microbenchmark (measurement only): read bandwidth of a 1-CTA-per-SM TMA bulk
// (cp.async.bulk) streaming pipeline vs. stage count / stage size / copies per stage, and of a
// plain LDG.128 streaming kernel, over a 1.6 GB buffer (the owner histogram's input size).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// STAGES x SB bytes ring; each stage filled by NCP bulk copies; CW consumer warps read it (LDS.128)
template <int STAGES, int SB, int NCP, int CW>
__global__ void __launch_bounds__(32 * (CW + 1), 1) k_tma(const uint4* src, uint64_t n16, uint32_t* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint4* stage = reinterpret_cast<uint4*>(sm);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + STAGES * SB);
  unsigned long long* empty = full + STAGES;
  const uint64_t per = SB / 16;
  const uint64_t nst = n16 / per;  // whole stages only
  const uint64_t s0 = nst * blockIdx.x / gridDim.x, s1 = nst * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    if (lane == 0) {
      uint32_t st = 0, ph = 0;
      for (uint64_t s = s0; s < s1; ++s) {
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_expect_tx(&full[st], SB);
        for (int c = 0; c < NCP; ++c)
          tma_bulk_g2s(reinterpret_cast<unsigned char*>(stage) + st * SB + c * (SB / NCP),
                       reinterpret_cast<const unsigned char*>(src + s * per) + c * (SB / NCP), SB / NCP, &full[st]);
        if (++st == STAGES) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  uint32_t st = 0, ph = 0, acc = 0;
  const uint32_t cw = w - 1;
  for (uint64_t s = s0; s < s1; ++s) {
    mbar_wait(&full[st], ph);
    const uint4* p = stage + st * per;
    for (uint32_t i = cw * 32 + lane; i < per; i += CW * 32) acc ^= p[i].x + p[i].w;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == STAGES) { st = 0; ph ^= 1u; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_ldg(const uint4* __restrict__ src, uint64_t n16, uint32_t* out) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x + v[u].w;
  }
  for (; i < n16; i += stride) acc ^= src[i].x;
  if (acc == 0x12345678u) out[0] = acc;
}

template <int STAGES, int SB, int NCP, int CW>
void run_tma(const uint4* src, uint64_t n16, uint32_t* out) {
  const int smem = STAGES * SB + 2 * STAGES * 8;
  cudaFuncSetAttribute(k_tma<STAGES, SB, NCP, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_tma<STAGES, SB, NCP, CW><<<148, 32 * (CW + 1), smem>>>(src, n16, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_tma<STAGES, SB, NCP, CW><<<148, 32 * (CW + 1), smem>>>(src, n16, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  cudaError_t e = cudaGetLastError();
  printf("{\"kind\": \"tma\", \"stages\": %d, \"stage_kb\": %d, \"copies\": %d, \"cons_warps\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
         STAGES, SB / 1024, NCP, CW, ms, n16 * 16.0 / ms / 1e6, cudaGetErrorString(e));
}

int main() {
  const uint64_t bytes = 1600000000ull;
  const uint64_t n16 = bytes / 16;
  uint4* src;
  uint32_t* out;
  cudaMalloc(&src, bytes);
  cudaMalloc(&out, 16);
  cudaMemset(src, 1, bytes);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
      k_ldg<<<g, 256>>>(src, n16, out);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k_ldg<<<g, 256>>>(src, n16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("{\"kind\": \"ldg\", \"grid\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", g, ms, bytes / ms / 1e6);
    }
  }
  run_tma<4, 32768, 1, 16>(src, n16, out);
  run_tma<4, 32768, 4, 16>(src, n16, out);
  run_tma<4, 32768, 8, 16>(src, n16, out);
  run_tma<6, 32768, 1, 16>(src, n16, out);
  run_tma<8, 16384, 1, 16>(src, n16, out);
  run_tma<8, 16384, 4, 16>(src, n16, out);
  run_tma<16, 8192, 1, 16>(src, n16, out);
  run_tma<24, 8192, 1, 16>(src, n16, out);
  run_tma<12, 16384, 1, 16>(src, n16, out);
  run_tma<12, 16384, 1, 4>(src, n16, out);
  run_tma<4, 32768, 1, 4>(src, n16, out);
  return 0;
}
