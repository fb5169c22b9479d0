// tcgen05.mma.kind::i8 issue-rate probe: back-to-back MMAs (M = 128, N in {32..256}, K = 32) on zero smem
// operands from one thread per CTA, one CTA per SM; prints chip int8 TOPS per N.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
template <int N, bool RANDOM>
__global__ void __launch_bounds__(128, 1) k(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) ((int*)s)[i] = RANDOM ? (int)(i * 2654435761u + 12345u) : 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = sdesc(su32(s)), db = sdesc(su32(s + 128 * 128));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t acc = (it | q) ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                t + (uint32_t)((q & 1) * 256 % 512)),
            "l"(da + 2 * (q & 3)), "l"(db + 2 * (q & 3)), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(su32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}
template <int N, bool RANDOM>
void run() {
  int* out;
  cudaMalloc(&out, 4);
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(k<N, RANDOM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  k<N, RANDOM><<<148, 128, smem>>>(10, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<N, RANDOM><<<148, 128, smem>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 148 * iters * 8 * 128.0 * N * 32;
  printf("N=%3d random=%d: %.3f ms, %.0f TOPS, %.1f ns per MMA per SM (err %s)\n", N, (int)RANDOM, ms, ops / ms / 1e9, ms * 1e6 / (iters * 8.0),
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, false>();
  run<64, true>();
  run<128, false>();
  run<128, true>();
  run<256, true>();
  return 0;
}
