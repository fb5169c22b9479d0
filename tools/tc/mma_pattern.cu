// tcgen05.mma.kind::i8 cta_group::2 (M = 256, N = 128, K = 32) issue-rate probe with the operand patterns of
// oz_gemm_kernel: B cycling over 7 digit planes, D over 4 accumulator slots, signed/unsigned descriptors, a
// commit every few MMAs.  One CTA pair per TPC, back-to-back MMAs from the leader.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(bool as, bool bs) {
  return (2u << 4) | ((as ? 1u : 0u) << 7) | ((bs ? 1u : 0u) << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
// MODE bits: 1 = B over 7 planes, 2 = D over 4 slots, 4 = mixed signedness, 8 = commit every 4 MMAs
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t slot;
  // A: 16 KB at 0; B: 7 planes of 8 KB at 16 KB
  for (int i = threadIdx.x; i < (16 + 56) * 1024 / 4; i += blockDim.x) ((int*)s)[i] = (int)(i * 2654435761u + 12345u + blockIdx.x);
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar3)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  unsigned long long g0, c0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  c0 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t da = sdesc(su32(s)), db = sdesc(su32(s + 16384));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 28; ++q) {
        const uint32_t acc = (it | q) ? 1u : 0u;
        const int kk = q & 3, j = (MODE & 1) ? (q % 7) : 0;
        const uint32_t d = t + (uint32_t)(((MODE & 2) ? (q % 4) : (q & 1) * 2) * 128);
        const uint32_t id = (MODE & 4) ? idesc((q & 1) == 0, j == 0) : idesc(true, true);
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(da + 2 * kk), "l"(db + (uint64_t)(j * 512 + 2 * kk)), "r"(id), "r"(acc));
        if ((MODE & 8) && (q & 3) == 3)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar2)), "h"((uint16_t)3));
        if ((MODE & 16) && (q & 3) == 3) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if ((MODE & 32) && (q & 3) == 3)  // wait on an already-completed barrier (phase 1 of bar3 never completes: parity 1 returns at once)
          asm volatile("{\n .reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n @!p bra W2;\n}" ::"r"(su32(&bar3)) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)3));
  }
  if (threadIdx.x == 0)
    asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(su32(&bar)));
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long g1, c1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    c1 = clock64();
    out[1] = (int)((c1 - c0) / ((g1 - g0) / 1000.0 + 1e-9));  // MHz
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}
template <int MODE>
void run() {
  int* out;
  cudaMalloc(&out, 8);
  const int smem = 1024 + (16 + 56) * 1024;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k<MODE>, 10, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k<MODE>, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int hout[2];
  cudaMemcpy(hout, out, 8, cudaMemcpyDeviceToHost);
  printf("SM clock during the run: %d MHz; ", hout[1]);
  printf("mode %2d (B7=%d D4=%d mixed=%d commit=%d fence=%d wait=%d): %.1f ns per MMA (err %s)\n", MODE, MODE & 1, (MODE >> 1) & 1,
         (MODE >> 2) & 1, (MODE >> 3) & 1, (MODE >> 4) & 1, (MODE >> 5) & 1, ms * 1e6 / (iters * 28.0), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<15>();
  run<16>();
  run<32>();
  run<63>();
  return 0;
}
