// tcgen05.mma.kind::i8 issue-rate probe for CTA pairs: cta_group::2 (M = 256, each CTA 128 rows of A and N/2
// rows of B) against cta_group::1 (M = 128), N in {64, 128, 256}, K = 32, random smem operands, one CTA per
// SM, back-to-back MMAs from one thread of the leader; prints chip int8 TOPS and ns per MMA.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
template <int N, int CG>
__global__ void __launch_bounds__(128, 1) k(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) ((int*)s)[i] = (int)(i * 2654435761u + 12345u + blockIdx.x);
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((128 * CG) >> 4) << 24);
    const uint64_t da = sdesc(su32(s)), db = sdesc(su32(s + 128 * 128));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t acc = (it | q) ? 1u : 0u;
        if (CG == 1)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                  t + (uint32_t)((q & 1) * 256 % 512)),
              "l"(da + 2 * (q & 3)), "l"(db + 2 * (q & 3)), "r"(idesc), "r"(acc));
        else
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                  t + (uint32_t)((q & 1) * 256 % 512)),
              "l"(da + 2 * (q & 3)), "l"(db + 2 * (q & 3)), "r"(idesc), "r"(acc));
      }
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)3));
  }
  if (threadIdx.x == 0)
    asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (threadIdx.x < 32) {
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}
template <int N, int CG>
void run() {
  int* out;
  cudaMalloc(&out, 4);
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(k<N, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k<N, CG>, 10, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k<N, CG>, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 148 * iters * 8 * 128.0 * N * 32;  // per SM: 128 rows of the M extent
  printf("cta_group::%d N=%3d: %.3f ms, %.0f TOPS, %.1f ns per MMA instruction (err %s)\n", CG, N, ms, ops / ms / 1e9,
         ms * 1e6 / (iters * 8.0), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, 1>();
  run<64, 2>();
  run<128, 1>();
  run<128, 2>();
  run<256, 1>();
  run<256, 2>();
  return 0;
}
