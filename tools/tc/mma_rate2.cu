// tcgen05.mma.kind::i8 issue-rate probe (M = 128, N = 64, K = 32) varying the stream's properties one at a time:
//   bit 0: 8 accumulators (64-column slots) instead of 2
//   bit 1: B from 7 different shared-memory regions (8 KB apart) instead of one
//   bit 2: the instruction descriptor alternates s8/u8 operand types
//   bit 3: tcgen05.commit to an mbarrier after every 20 MMAs
//   bit 4: tcgen05.fence::after_thread_sync before every 20 MMAs
//   bit 6: A from a 6-stage ring of 16 KB tiles (a fresh A tile every 20 MMAs, as the GEMM's data ring)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (6 * 16384 + 7 * 8192) / 4; i += blockDim.x) ((int*)s)[i] = (int)(i * 2654435761u);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
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
    const uint64_t da0 = sdesc(su32(s)), db0 = sdesc(su32(s + 6 * 16384));
    int cnt = 0;
    for (int it = 0; it < iters; ++it) {
      if (MODE & 16) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = da0 + ((MODE & 64) ? (uint64_t)((it % 6) * 1024) : 0);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const uint32_t acc_col = (MODE & 1) ? (uint32_t)(((j + it) & 7) * 64) : (uint32_t)((j & 1) * 256);
          const uint64_t db = db0 + ((MODE & 2) ? (uint64_t)(j * 512) : 0) + 2 * kk;
          const uint32_t idesc = (2u << 4) | (((MODE & 4) ? (j == 0) : 1u) << 7) | (((MODE & 4) ? (kk & 1) : 1u) << 10) |
                                 ((64u >> 3) << 17) | ((128u >> 4) << 24);
          const uint32_t acc = (it | kk | j) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                  t + acc_col),
              "l"(da + 2 * kk), "l"(db), "r"(idesc), "r"(acc));
          ++cnt;
        }
      if (MODE & 8)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(su32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}
template <int MODE>
void run() {
  int* out;
  cudaMalloc(&out, 4);
  const int smem = 1024 + 6 * 16384 + 7 * 8192;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<MODE><<<148, 128, smem>>>(10, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, 128, smem>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("mode %2d: %.1f ns per MMA per SM (%s)\n", MODE, ms * 1e6 / (iters * 20.0), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>();
  run<31>();
  run<64>();
  run<95>();
  return 0;
}
