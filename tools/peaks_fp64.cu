// FP64 roofline denominators for sm_100a: DMMA (mma.sync m8n8k4 f64) and DFMA
// register-resident loops, plus a device-property dump. Writes one JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_fp64 peaks_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0 - 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
static float timeit(K kern, dim3 g, dim3 b, double* out, int iters, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<g, b>>>(out, iters, 0.5);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<g, b>>>(out, iters, 0.5);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0, memclk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  printf("{\"name\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"smem_per_block_optin\": %zu, "
         "\"smem_per_sm\": %zu, \"l2_bytes\": %d, \"regs_per_sm\": %d, \"clock_khz\": %d, \"mem_clock_khz\": %d, "
         "\"global_mem\": %zu}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.l2CacheSize, p.regsPerMultiprocessor, clk, memclk, p.totalGlobalMem);
  double* out; CK(cudaMalloc(&out, 8));
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      dim3 g(sms * bps), b(32 * warps);
      float ms = timeit(dmma_loop<8>, g, b, out, iters, 5);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)g.x * warps;
      printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             warps, bps, ms, flops / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    for (int bps : {1, 2}) {
      dim3 g(sms * bps), b(32 * warps);
      float ms = timeit(dfma_loop<8>, g, b, out, iters * 4, 5);
      double flops = 2.0 * 8 * 4.0 * iters * (double)g.x * warps * 32;
      printf("{\"kind\": \"dfma\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             warps, bps, ms, flops / ms / 1e9);
    }
  }
  // sustained: dmma back-to-back for ~3 s
  {
    dim3 g(sms * 2), b(32 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    int launches = 0; float ms = 0;
    while (ms < 3000.f) {
      for (int i = 0; i < 10; ++i) dmma_loop<8><<<g, b>>>(out, iters, 0.5);
      launches += 10;
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)g.x * 8 * launches;
    printf("{\"kind\": \"dmma_sustained\", \"ms\": %.1f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
