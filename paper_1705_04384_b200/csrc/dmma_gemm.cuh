// FP64 tensor-core GEMM for the FD mode-k products (sm_100a).
//
// On sm_100a the only FP64 tensor instruction is the warp-level DMMA.8x8x4 (PTX
// mma.sync.aligned.m8n8k4.row.col.f64); tcgen05.mma has no f64 kind, so there is no TMEM/UMMA
// path for FP64 and accumulators live in registers.
// Measured on the pool's B200: 37.1 TFLOP/s for a register-resident DMMA loop (profiles/r01_peaks_fp64.jsonl).
//
//   C[M x N] = A[M x K] * B[K x N]   (+ optional epilogue C /= lam_m[m] + lam_n[n % inner])
//   A: row-major, k contiguous (lda)
//   B: BLayout::KN (modes 2..d: left-multiply a strided axis by the factor A = F_l):
//        column n of B and C lives at colOff(n) = (n / inner) * bstride + n % inner, i.e. the batch of
//        slices X[i_{l+1}..][0..n_l)[0..inner) is flattened into one long N = inner * batch, so a tile
//        never straddles padding and ragged n_l only costs the M (= n_l) edge.
//        B[k][n] = B[colOff(n) + k ldb],  C[m][n] = C[colOff(n) + m ldc]
//      BLayout::NK (mode 1: right-multiply the contiguous axis by F_1^T):
//        B[k][n] = B[n ldb + k] (the factor, k contiguous),  C[m][n] = C[m ldc + n]
//
// One CTA per output tile, 1-D grid ordered so that the tiles sharing the big operand are adjacent
// (the few tiles along the factor dimension run together and hit the same L2 lines).  Tiles are
// staged global->shared with cp.async (16 B when rows are 16 B aligned, else 8 B), zero-filled outside
// [M,N,K], into a STAGES-deep ring; shared rows are padded (stride == 4 mod 16 doubles) so the m8n8k4
// fragment loads (8 rows x 4 k, or 4 k x 8 cols) are bank-conflict free.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

namespace fdiga {

enum class BLayout { KN, NK };

struct GemmParams {
  int M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int64_t inner;        // KN: columns per batch slice (== N when there is a single slice)
  int64_t bstride;      // KN: elements between consecutive slices of B and C
  const double* lam_m;  // epilogue divide (nullptr: none): C[m][n] = acc / (lam_m[m] + lam_n[n % inner])
  const double* lam_n;
  const int* skip;      // device flag: nonzero -> the launch does nothing (GMRES graph early exit)
  int tiles_m, tiles_n;
};

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int KV_ = 0, int NP_ = 0, int MINB_ = 1>
struct TileCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  // MINB: resident CTAs per SM the register allocation must allow (__launch_bounds__ min blocks); 4 x 64x64
  // CTAs per SM (config 16) measured no faster than 3 at n = 256: the loss is not wave quantisation
  static constexpr int MINB = MINB_;
  // NP = 1 (KN layout, with KV, warp tiles 64 wide): n-permuted fragments.  Within a warp tile the
  // logical column (MMA j, lane row r) is the physical column r NJ + j, so a thread's NJ B fragments of
  // one k are NJ consecutive doubles (16-byte loads) and its accumulators map to two runs of NJ
  // consecutive output columns.  The shared B tile is unpadded with its 16-byte chunks XOR-swizzled by
  // (k / 4) mod 4, which makes those 16-byte loads bank-conflict free.
  static constexpr int NP = NP_;
  // KV = 1 (BK = 16): k-permuted fragments.  MMA step kk of a k-tile contracts the k indices
  // {kk, kk + 4, kk + 8, kk + 12}, thread lc taking k = 4 lc + kk, so a thread's four A (and NK-B)
  // fragments of the tile are 4 consecutive doubles: two 16-byte shared loads instead of four 8-byte
  // ones.  The same permutation on both operands leaves the product unchanged (summation order only).
  static constexpr int KV = KV_;
  static_assert(KV == 0 || BK == 16, "k-permuted fragments need BK = 16");
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MI = WTM / 8, NJ = WTN / 8;
  // A row stride (doubles): == 4 (mod 16) -> conflict-free 8-byte fragment loads; KV: == 2 (mod 16) ->
  // conflict-free 16-byte loads (a quarter-warp covers two rows x four 4-word groups)
  static constexpr int SA = BK + (KV ? 2 : 4);
  static constexpr int SBkn = NP ? BN : BN + 4;  // B [k][n] row stride (padded: == 4 mod 16 for BN % 16 == 0)
  static constexpr int SBnk = BK + (KV ? 2 : 4);  // B [n][k] row stride
  static_assert(WTM % 8 == 0 && WTN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert(NP == 0 || (KV == 1 && WTN == 64), "n-permuted fragments need KV and 64-wide warp tiles");
  static constexpr int A_ELEMS = BM * SA;
  static constexpr int B_ELEMS_KN = BK * SBkn;
  static constexpr int B_ELEMS_NK = BN * SBnk;
  template <BLayout L>
  __host__ __device__ static constexpr int b_elems() { return L == BLayout::KN ? B_ELEMS_KN : B_ELEMS_NK; }
  template <BLayout L>
  __host__ __device__ static constexpr size_t smem_bytes() {
    return size_t(STAGES) * (A_ELEMS + b_elems<L>()) * sizeof(double);
  }
};

// VA / VB: doubles per cp.async chunk for A / B (2 needs 16-byte aligned rows, else 1).
// RAG: K is not a multiple of BK (the last k-tile runs only the k-steps that reach below K)
template <class T, BLayout BL, int VA, int VB, bool RAG>
__global__ void __launch_bounds__(T::THREADS, T::MINB) dmma_gemm_kernel(GemmParams p) {
  // programmatic dependent launch: this grid may start while the previous kernel of the stream drains;
  // nothing it produced (the B/A operand, the skip flag) is read before its completion is awaited here
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (p.skip && *p.skip) return;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + T::STAGES * T::A_ELEMS;
  constexpr int BE = T::template b_elems<BL>();

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int warp_m = warp / T::WN, warp_n = warp % T::WN;
  // tile order: the factor dimension (M for KN, N for NK) runs fastest
  int mt, nt;
  if (BL == BLayout::KN) {
    mt = blockIdx.x % p.tiles_m;
    nt = blockIdx.x / p.tiles_m;
  } else {
    nt = blockIdx.x % p.tiles_n;
    mt = blockIdx.x / p.tiles_n;
  }
  const int m0 = mt * T::BM, n0 = nt * T::BN;
  const double* __restrict__ A = p.A;
  const double* __restrict__ B = p.B;
  double* __restrict__ C = p.C;
  const int M = p.M, N = p.N, K = p.K;
  const int KT = (K + T::BK - 1) / T::BK;

  // KN: per-thread B column offsets are the same for every k-stage (THREADS % (BN / VB) == 0)
  constexpr int CPR_B_KN = T::BN / VB;
  static_assert(BL != BLayout::KN || T::THREADS % CPR_B_KN == 0, "B loader mapping");
  int64_t b_col_off = 0;
  int b_col_bytes = 0;
  if (BL == BLayout::KN) {
    const int gn = n0 + (tid % CPR_B_KN) * VB;
    if (gn < N) {
      b_col_off = (int64_t)(gn / p.inner) * p.bstride + gn % p.inner;
      b_col_bytes = (VB == 2 && gn + 1 >= N) ? 8 : VB * 8;
    }
  }

  auto load_tile = [&](int stage, int kt) {
    const int k0 = kt * T::BK;
    {  // A tile: BM x BK, rows m, cols k
      constexpr int CPR = T::BK / VA;
      constexpr int CH = T::BM * CPR;
      double* dst = sA + stage * T::A_ELEMS;
#pragma unroll
      for (int c = tid; c < CH; c += T::THREADS) {
        const int r = c / CPR, cc = c % CPR;
        const int gm = m0 + r, gk = k0 + cc * VA;
        const uint32_t d = smem_u32(dst + r * T::SA + cc * VA);
        int bytes = 0;
        const double* src = A;
        if (gm < M && gk < K) {
          bytes = (VA == 2 && gk + 1 >= K) ? 8 : VA * 8;
          src = A + (int64_t)gm * p.lda + gk;
        }
        if (VA == 2) cp_async16(d, src, bytes); else cp_async8(d, src, bytes);
      }
    }
    double* dstB = sB + stage * BE;
    if (BL == BLayout::KN) {
      constexpr int CH = T::BK * CPR_B_KN;
      const int cc = tid % CPR_B_KN;
#pragma unroll
      for (int c = tid; c < CH; c += T::THREADS) {
        const int r = c / CPR_B_KN;
        const int gk = k0 + r;
        int pc = cc * VB;  // physical column of the chunk (NP: 16-byte chunks XOR-swizzled by (k / 4) mod 4)
        if (T::NP) pc = ((((cc * VB) >> 1) ^ ((r >> 2) & 3)) << 1) | ((cc * VB) & 1);
        const uint32_t d = smem_u32(dstB + r * T::SBkn + pc);
        int bytes = 0;
        const double* src = B;
        if (gk < K && b_col_bytes) {
          bytes = b_col_bytes;
          src = B + b_col_off + (int64_t)gk * p.ldb;
        }
        if (VB == 2) cp_async16(d, src, bytes); else cp_async8(d, src, bytes);
      }
    } else {
      constexpr int CPR = T::BK / VB;
      constexpr int CH = T::BN * CPR;
#pragma unroll
      for (int c = tid; c < CH; c += T::THREADS) {
        const int r = c / CPR, cc = c % CPR;
        const int gn = n0 + r, gk = k0 + cc * VB;
        const uint32_t d = smem_u32(dstB + r * T::SBnk + cc * VB);
        int bytes = 0;
        const double* src = B;
        if (gn < N && gk < K) {
          bytes = (VB == 2 && gk + 1 >= K) ? 8 : VB * 8;
          src = B + (int64_t)gn * p.ldb + gk;
        }
        if (VB == 2) cp_async16(d, src, bytes); else cp_async8(d, src, bytes);
      }
    }
  };

  double acc[T::MI][T::NJ][2];
#pragma unroll
  for (int i = 0; i < T::MI; ++i)
#pragma unroll
    for (int j = 0; j < T::NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < T::STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }

  const int lr = lane >> 2, lc = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<T::STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + T::STAGES - 1;
      if (nk < KT) load_tile(nk % T::STAGES, nk);
      cp_async_commit();
    }
    const int st = kt % T::STAGES;
    const double* a_s = sA + st * T::A_ELEMS + (warp_m * T::WTM + lr) * T::SA + lc;
    const double* b_s = sB + st * BE;
    if (T::KV) {
      // k-permuted fragments: thread lc holds k = 4 lc + kk for the four steps kk of the tile
      const double* a_v = a_s - lc + 4 * lc;
      double af[T::MI][4], bf[T::NJ][4];
#pragma unroll
      for (int i = 0; i < T::MI; ++i) {
        const double2 x0 = *reinterpret_cast<const double2*>(a_v + i * 8 * T::SA);
        const double2 x1 = *reinterpret_cast<const double2*>(a_v + i * 8 * T::SA + 2);
        af[i][0] = x0.x;
        af[i][1] = x0.y;
        af[i][2] = x1.x;
        af[i][3] = x1.y;
      }
#pragma unroll
      for (int j = 0; j < T::NJ; ++j) {
        if (BL == BLayout::KN && T::NP) {
          if (j % 2 == 0) {  // physical columns warp_n WTN + lr NJ + j, j + 1: one 16-byte chunk
            const int c16 = ((warp_n * T::WTN + lr * T::NJ + j) >> 1) ^ lc;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const double2 y = *reinterpret_cast<const double2*>(b_s + (4 * lc + kk) * T::SBkn + 2 * c16);
              bf[j][kk] = y.x;
              bf[j + 1][kk] = y.y;
            }
          }
        } else if (BL == BLayout::KN) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) bf[j][kk] = b_s[(4 * lc + kk) * T::SBkn + warp_n * T::WTN + j * 8 + lr];
        } else {
          const double* bp = b_s + (warp_n * T::WTN + j * 8 + lr) * T::SBnk + 4 * lc;
          const double2 y0 = *reinterpret_cast<const double2*>(bp);
          const double2 y1 = *reinterpret_cast<const double2*>(bp + 2);
          bf[j][0] = y0.x;
          bf[j][1] = y0.y;
          bf[j][2] = y1.x;
          bf[j][3] = y1.y;
        }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
          for (int j = 0; j < T::NJ; ++j) dmma_8x8x4(acc[i][j], af[i][kk], bf[j][kk]);
    } else {
      auto kstep = [&](int kk) {
        double af[T::MI], bf[T::NJ];
#pragma unroll
        for (int i = 0; i < T::MI; ++i) af[i] = a_s[i * 8 * T::SA + kk * 4];
#pragma unroll
        for (int j = 0; j < T::NJ; ++j) {
          if (BL == BLayout::KN)
            bf[j] = b_s[(kk * 4 + lc) * T::SBkn + warp_n * T::WTN + j * 8 + lr];
          else
            bf[j] = b_s[(warp_n * T::WTN + j * 8 + lr) * T::SBnk + kk * 4 + lc];
        }
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
          for (int j = 0; j < T::NJ; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
      };
      // the last k-tile runs only the k-steps of 4 that reach below K (K = 131: 1 of 4); a separate,
      // non-unrolled loop, so the hot unrolled loop stays free of predicates
      const int ksteps = (RAG && kt == KT - 1) ? (K - kt * T::BK + 3) >> 2 : T::BK / 4;
      if (!RAG || ksteps >= T::BK / 4) {
#pragma unroll
        for (int kk = 0; kk < T::BK / 4; ++kk) kstep(kk);
      } else {
#pragma unroll 1
        for (int kk = 0; kk < ksteps; ++kk) kstep(kk);
      }
    }
  }
  cp_async_wait<0>();
  // the next mode product may begin launching its CTAs (they wait for this grid's completion)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  // ---- epilogue: optional eigenvalue-sum divide (eq:FD3D diagonal term), store
  const bool c_vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((p.ldc & 1) == 0) &&
                     (BL == BLayout::NK || ((p.inner & 1) == 0 && (p.bstride & 1) == 0));
  if constexpr (T::NP != 0) {
    // accumulator (i, j, h) is physical column warp_n WTN + (2 lc + h) NJ + j: pairs (j, j + 1) adjacent
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < T::NJ; j += 2) {
        const int col = n0 + warp_n * T::WTN + (2 * lc + h) * T::NJ + j;
        if (col >= N) continue;
        const bool two = col + 1 < N;
        const int64_t sl = col / p.inner, lidx = col - sl * p.inner;
        const int64_t coff = sl * p.bstride + lidx;
        int64_t coff1 = coff + 1, lidx1 = lidx + 1;
        if (two && lidx1 >= p.inner) {
          lidx1 = 0;
          coff1 = (sl + 1) * p.bstride;
        }
        const double ln0 = p.lam_m ? p.lam_n[lidx] : 0.0;
        const double ln1 = (p.lam_m && two) ? p.lam_n[lidx1] : 0.0;
#pragma unroll
        for (int i = 0; i < T::MI; ++i) {
          const int row = m0 + warp_m * T::WTM + i * 8 + lr;
          if (row >= M) continue;
          double v0 = acc[i][j][h], v1 = acc[i][j + 1][h];
          if (p.lam_m) {
            const double lm = p.lam_m[row];
            v0 = v0 / (lm + ln0);
            v1 = v1 / (lm + ln1);
          }
          double* dst = C + (int64_t)row * p.ldc;
          if (c_vec && two && coff1 == coff + 1) {
            *reinterpret_cast<double2*>(dst + coff) = make_double2(v0, v1);
          } else {
            dst[coff] = v0;
            if (two) dst[coff1] = v1;
          }
        }
      }
  } else {
#pragma unroll
  for (int j = 0; j < T::NJ; ++j) {
    const int col = n0 + warp_n * T::WTN + j * 8 + 2 * lc;
    if (col >= N) continue;
    int64_t coff;
    int64_t lidx = col;
    if (BL == BLayout::KN) {
      const int64_t sl = col / p.inner;
      lidx = col - sl * p.inner;
      coff = sl * p.bstride + lidx;
    } else {
      coff = col;
    }
    const bool two = col + 1 < N;
    // the pair (col, col+1) stays in one slice when inner is even; otherwise recompute for col+1
    int64_t coff1 = coff + 1, lidx1 = lidx + 1;
    if (BL == BLayout::KN && two && (p.inner & 1)) {
      const int64_t sl = (col + 1) / p.inner;
      lidx1 = (col + 1) - sl * p.inner;
      coff1 = sl * p.bstride + lidx1;
    }
    const double ln0 = p.lam_m ? p.lam_n[lidx] : 0.0;
    const double ln1 = (p.lam_m && two) ? p.lam_n[lidx1] : 0.0;
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
      const int row = m0 + warp_m * T::WTM + i * 8 + lr;
      if (row >= M) continue;
      double v0 = acc[i][j][0], v1 = acc[i][j][1];
      if (p.lam_m) {
        const double lm = p.lam_m[row];
        v0 = v0 / (lm + ln0);
        v1 = v1 / (lm + ln1);
      }
      double* dst = C + (int64_t)row * p.ldc;
      if (c_vec && two) {
        *reinterpret_cast<double2*>(dst + coff) = make_double2(v0, v1);
      } else {
        dst[coff] = v0;
        if (two) dst[coff1] = v1;
      }
    }
  }
  }  // NP == 0
}

}  // namespace fdiga
