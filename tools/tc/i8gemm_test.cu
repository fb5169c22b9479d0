// Stage-1 probe for the Ozaki-split FD path: a tcgen05 (kind::i8) GEMM, C[M x N] (s32) = A[M x K] * B[N x K]^T,
// A and B int8 K-major, TMA (SWIZZLE_128B) -> smem ring -> tcgen05.mma (single issuing thread) -> TMEM ->
// tcgen05.ld epilogue.  Checks against a host integer GEMM and times a 65536 x 256 x 256 problem.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
// smem matrix descriptor: K-major, SWIZZLE_128B (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t sdesc_sw128(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // version (sm100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4)            // D = s32
         | (1u << 7)          // A = s8
         | (1u << 10)         // B = s8
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int BN, int S, bool AT>
__global__ void __launch_bounds__(128, 1) i8gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                                 int32_t* C, int M, int N, int K) {
  constexpr int BM = 128, BK = 128;
  constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK;
  constexpr uint32_t TCOLS = 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * A_BYTES;
  uint64_t* full = (uint64_t*)(sB + S * B_BYTES);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tslot = (uint32_t*)(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KC = K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = *tslot;

  if (warp == 0 && lane == 0) {
    for (int kc = 0; kc < KC; ++kc) {
      const int s = kc % S;
      if (kc >= S) mbar_wait(&empty[s], ((kc / S) - 1) & 1);
      mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
      tma2d(sA + s * A_BYTES, &ma, kc * BK, m0, &full[s]);
      tma2d(sB + s * B_BYTES, &mb, kc * BK, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_i8<BM, BN>();
    for (int kc = 0; kc < KC; ++kc) {
      const int s = kc % S;
      mbar_wait(&full[s], (kc / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint64_t da = sdesc_sw128(sA + s * A_BYTES), db = sdesc_sw128(sB + s * B_BYTES);
#pragma unroll
      for (int k = 0; k < BK / 32; ++k) {
        const uint32_t acc = (kc > 0 || k > 0) ? 1u : 0u;
        if (AT) {
          const uint32_t ta = tbase + 256 + (uint32_t)((s & 1) * 32 + k * 8);
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta), "l"(da + (uint64_t)(k * 2)));
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                  tbase),
              "r"(ta), "l"(db + (uint64_t)(k * 2)), "r"(idesc), "r"(acc));
        } else {
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                  tbase),
              "l"(da + (uint64_t)(k * 2)), "l"(db + (uint64_t)(k * 2)), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(done))
                 : "memory");
  }
  __syncwarp();
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = m0 + warp * 32 + lane;
#pragma unroll
  for (int c = 0; c < BN; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tbase + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < M)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (n0 + c + j < N) C[(int64_t)row * N + n0 + c + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(TCOLS));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (EncodeFn)fn;
}
static CUtensorMap make_map(EncodeFn enc, const void* base, int rows, int K, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

template <int BN, int S, bool AT = false>
void run(int M, int N, int K, bool check) {
  std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
  uint32_t st = 12345;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (int8_t)((st >> 24) % 255 - 127); };
  for (auto& v : hA) v = rnd();
  for (auto& v : hB) v = rnd();
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, hA.size()));
  CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, (size_t)M * N * 4));
  EncodeFn enc = get_encode();
  CUtensorMap ma = make_map(enc, dA, M, K, 128), mb = make_map(enc, dB, N, K, BN);
  const size_t smem = 1024 + S * (128 * 128 + BN * 128) + (2 * S + 1) * 8 + 16;
  auto kern = i8gemm<BN, S, AT>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((M + 127) / 128, (N + BN - 1) / BN);
  kern<<<grid, 128, smem>>>(ma, mb, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  if (check) {
    std::vector<int32_t> hC((size_t)M * N);
    CK(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int m = 0; m < M; m += (M > 4096 ? 37 : 1))
      for (int n = 0; n < N; ++n) {
        int32_t s = 0;
        for (int k = 0; k < K; ++k) s += (int32_t)hA[(size_t)m * K + k] * (int32_t)hB[(size_t)n * K + k];
        if (s != hC[(size_t)m * N + n]) {
          if (bad < 5) printf("  mismatch m=%d n=%d got %d want %d\n", m, n, hC[(size_t)m * N + n], s);
          ++bad;
        }
      }
    printf("BN=%d S=%d AT=%d M=%d N=%d K=%d: %s (%ld bad)\n", BN, S, (int)AT, M, N, K, bad ? "FAIL" : "ok", bad);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) kern<<<grid, 128, smem>>>(ma, mb, dC, M, N, K);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) kern<<<grid, 128, smem>>>(ma, mb, dC, M, N, K);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("BN=%d S=%d AT=%d M=%d N=%d K=%d: %.2f us, %.1f TOPS\n", BN, S, (int)AT, M, N, K, ms * 1e3, 2.0 * M * N * K / ms / 1e9);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
}

int main() {
  run<64, 4, false>(1024, 256, 512, true);
  run<64, 4, true>(1024, 256, 512, true);
  run<128, 4, true>(1024, 256, 512, true);
  run<64, 4, true>(65536, 256, 256, true);
  run<64, 4, false>(8192, 64, 8192, false);
  run<64, 4, true>(8192, 64, 8192, false);
  run<256, 3, false>(8192, 256, 4096, false);
  run<256, 3, true>(8192, 256, 4096, false);
  return 0;
}
