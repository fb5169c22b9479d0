// Deterministic block reductions shared by the Krylov kernels (krylov.cu, bicgstab.cu).
#pragma once
#include "common.cuh"

namespace fdiga {

constexpr int RT = 256;  // threads per block of the vector kernels

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-reduce CNT accumulators (slots < cnt are live) into part[blockIdx.x][*]; the last block to
// finish then sums the partials in block order into out[*] and returns true (in all its threads).
template <int CNT>
__device__ __forceinline__ bool reduce_last(double (&acc)[CNT], int cnt, double* part, unsigned int* counter,
                                            double* out) {
  __shared__ double red[RT / 32][CNT];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < CNT; ++i) {
    if (i < cnt) {
      const double v = warp_sum(acc[i]);
      if (lane == 0) red[warp][i] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    double s = 0;
    for (int w = 0; w < RT / 32; ++w) s += red[w][i];
    part[(int64_t)blockIdx.x * CNT + i] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  // one warp per output value, fixed order over blocks (lane-strided, then a fixed shuffle tree)
  for (int i = warp; i < cnt; i += RT / 32) {
    double s = 0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(part + (int64_t)b * CNT + i);
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}


}  // namespace fdiga
