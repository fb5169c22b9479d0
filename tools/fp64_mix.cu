// Does DMMA (mma.sync m8n8k4 f64) share the FP64 units with DFMA on sm_100a?  Interleave both in one loop
// and compare the combined FLOP rate with the pure loops.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF>
__global__ void mix(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3, bf = 1.0 - 1e-9;
  double c[NM > 0 ? NM : 1][2], f[NF > 0 ? NF : 1];
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) c[i][0] = c[i][1] = 0.0;
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], bf, a);
  }
  double s = 0;
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  if (s == 1234.5) out[0] = s;
}

template <int NM, int NF>
void run(const char* name, int sms, double* out) {
  const int iters = 20000, warps = 8, bps = 2;
  dim3 g(sms * bps), bl(32 * warps);
  mix<NM, NF><<<g, bl>>>(out, iters, 0.5);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mix<NM, NF><<<g, bl>>>(out, iters, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double nthreads = (double)g.x * warps * 32, nwarps = (double)g.x * warps;
  const double fm = 2.0 * 8 * 8 * 4 * NM * (double)iters * nwarps, ff = 2.0 * NF * (double)iters * nthreads;
  printf("%-28s %8.3f ms  dmma %6.2f TF  dfma %6.2f TF  total %6.2f TF\n", name, best, fm / best / 1e9,
         ff / best / 1e9, (fm + ff) / best / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<8, 0>("dmma only (8 acc)", sms, out);
  run<0, 16>("dfma only (16 acc)", sms, out);
  run<8, 8>("dmma 8 + dfma 8", sms, out);
  run<8, 16>("dmma 8 + dfma 16", sms, out);
  run<4, 16>("dmma 4 + dfma 16", sms, out);
  run<8, 32>("dmma 8 + dfma 32", sms, out);
  return 0;
}
