// FD mode products on tcgen05 int8 tensor cores with exact digit splitting (see oz.cuh).
//
//   oz_split_*_kernel : FP64 operand -> S = 7 int8 digit planes + per-row exponents (HBM-bound pass; the
//                       strided modes are transposed so every GEMM operand is K-major)
//   oz_gemm_kernel    : persistent, warp-specialised tcgen05 GEMM.  Warp 8 streams the data digit planes
//                       through a TMA (SWIZZLE_128B) ring; warp 9 (converged, one elected lane per stage)
//                       issues tcgen05.mma.kind::i8 into NW = 8 int32 accumulators in TMEM (one per
//                       digit-pair weight t = i + j); warps 0-7 read them back with tcgen05.ld, combine in
//                       FP64, scale by the row exponents and store.  The factor's digit planes for the CTA's
//                       column tile stay resident in shared memory (K <= 256) or stream one k chunk at a time
//                       (K <= 512).
//                       Outputs of "wide" rows (oz.cuh: guard) are then recomputed by the CTA that owns them
//                       as IEEE FP64 dot products of the FP64 operands (oz_cta_fixup).
#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <vector>

#include "oz.cuh"
#include "ptx.cuh"

namespace fdiga {

void OzOperand::release() {
  if (digits) cudaFree(digits);
  if (exps) cudaFree(exps);
  if (wide) cudaFree(wide);
  if (ft) cudaFree(ft);
  ft = nullptr;
  digits = nullptr;
  exps = nullptr;
  wide = nullptr;
  rows = rows_p = kp = 0;
}

namespace {

// ---------------------------------------------------------------------------------------------
// digit split
// ---------------------------------------------------------------------------------------------
// 2^k for |k| <= 2044 as a product of two normal powers (each built from its bits)
__device__ __forceinline__ double pow2(int k) {
  k = max(-2044, min(2044, k));
  const int k1 = k / 2, k2 = k - k1;
  return __longlong_as_double((long long)(k1 + 1023) << 52) * __longlong_as_double((long long)(k2 + 1023) << 52);
}

__device__ __forceinline__ int row_exponent(double mx) {
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): every |x| <= mx < 2^e
  return e;
}

// running guard state of a row: max |x|, min nonzero |x|, any non-finite value
struct RowStat {
  double mx = 0.0, mn = INFINITY;
  bool nf = false;
  __device__ __forceinline__ void add(double v) {
    const double a = fabs(v);
    mx = fmax(mx, a);
    mn = fmin(mn, a == 0.0 ? INFINITY : a);
    nf |= !(a <= 1.7976931348623157e308);  // NaN or Inf
  }
};

// stored exponent of a row: e, or e + OZ_WIDE when the row goes to the FP64 fallback (oz.cuh)
__device__ __forceinline__ int row_code(const RowStat& r, int e) {
  const bool wide = r.nf || (r.mx > 0.0 && (e < OZ_EMIN || r.mn < pow2(e - OZ_SPREAD)));
  return wide ? e + OZ_WIDE : e;
}
__device__ __forceinline__ bool code_wide(int c) { return c >= OZ_WIDE / 2; }
__device__ __forceinline__ int code_exp(int c) { return code_wide(c) ? c - OZ_WIDE : c; }

// 1 / d for a normal d on the FP64 pipe (MUFU.RCP and the F2F conversions a float seed needs run on the XU
// pipe, which bounds the dividing split): the bit-pattern seed 0x7FDE623822FC16E6 - bits(|d|) is within
// 12.5 % of 1 / |d|; Newton r <- r + r (1 - |d| r) squares the relative error, so five steps reach rounding
// level (0.125 -> 1.6e-2 -> 2.4e-4 -> 6e-8 -> 3.6e-15 -> 1e-29).
__device__ __forceinline__ double rcp_fp64(double d) {
  const double a = fabs(d);
  double r = __longlong_as_double(0x7FDE623822FC16E6LL - __double_as_longlong(a));
#pragma unroll
  for (int i = 0; i < 5; ++i) r = fma(r, fma(-a, r, 1.0), r);
  return copysign(r, d);
}

// q = floor(v) for |v| < 2^62 as two 32-bit words, on the FP64 pipe (the F2I.S64.F64 conversion runs on
// the XU pipe).  h = floor(v 2^-32): adding 1.5 2^52 with round-down leaves it in the low mantissa word
// (two's complement, |h| <= 2^30); l = floor(v - h 2^32) in [0, 2^32) the same way with 2^52.  Every
// operation rounds down, and floor(rd(t)) = floor(t) for any t (the integer floor(t) is representable and
// rounding is monotone): the scaling may underflow for tiny v, and v - h 2^32 for a tiny negative v
// (2^32 - |v|) is not representable -- rounded to nearest it would give 2^32 and l = 0 instead of 2^32 - 1.
__device__ __forceinline__ void q_words(double v, uint32_t& h, uint32_t& l) {
  constexpr double M = 6755399441055744.0;  // 1.5 * 2^52
  const double a = __dadd_rd(__dmul_rd(v, 0x1p-32), M);
  h = (uint32_t)__double2loint(a);
  const double lo = __fma_rd(-(a - M), 4294967296.0, v);
  l = (uint32_t)__double2loint(__dadd_rd(lo, 4503599627370496.0));
}

// 8 consecutive values -> S packed 8-byte digit words.  q = floor(x 2^(62 - e)) in [-2^62, 2^62) (bits
// below 2^-62 of the row scale are beyond digit S anyway; the scaling rounds down so that an underflowing
// negative x still floors to -1); digit 0 = q >> 55 (signed), digits 1..6 = the bytes of q at bits 47..7.
__device__ __forceinline__ void split8(const double (&v)[8], int e, uint64_t (&w)[OZ_S]) {
  static_assert(OZ_S == 7, "digit extraction written for a signed 8-bit leading digit and 6 unsigned bytes");
  // q = floor(x 2^(62 - e)) in [-2^62, 2^62): digit 0 = q >> 55 (signed, [-128, 127]), digits 1..6 = the
  // unsigned bytes of q at bits 47, 39, .., 7 (two's complement makes the lower digits non-negative).  Taken
  // as q' = floor(x 2^(55 - e)) = q >> 7, every digit is a whole byte of q' (digit s = byte 6 - s), and four
  // values' digits pack into a word with three byte permutes
  const double sc = pow2(55 - e);
  uint32_t h[8], l[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) q_words(__dmul_rd(v[j], sc), h[j], l[j]);
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) {
    const unsigned b = (unsigned)(6 - s) & 3u;  // byte within the word: s = 0..2 from h, 3..6 from l
    const unsigned sel = b | ((b + 4u) << 4);
    uint32_t half[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const uint32_t* src = s < 3 ? h : l;
      const uint32_t t01 = __byte_perm(src[4 * g], src[4 * g + 1], sel);
      const uint32_t t23 = __byte_perm(src[4 * g + 2], src[4 * g + 3], sel);
      half[g] = __byte_perm(t01, t23, 0x5410);
    }
    w[s] = ((uint64_t)half[1] << 32) | half[0];
  }
}

// inner == 1: rows of K contiguous values.  One warp per row, 8 values per lane per 256-wide chunk.
template <int NCH>
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const double* __restrict__ x, int64_t rows, int K, int64_t ldx,
                                                            int8_t* __restrict__ digits, int32_t* __restrict__ exps,
                                                            int32_t* __restrict__ wide, int64_t rows_p, int kp,
                                                            const int* skip) {
  if (skip && *skip) return;
  const int lane = threadIdx.x & 31;
  const int64_t m = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (m >= rows) return;
  const double* xr = x + m * ldx;
  double v[NCH][8];
  RowStat st;
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = c * 256 + lane * 8 + j;
      v[c][j] = k < K ? xr[k] : 0.0;
      st.add(v[c][j]);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st.mx = fmax(st.mx, __shfl_xor_sync(0xffffffffu, st.mx, o));
    st.mn = fmin(st.mn, __shfl_xor_sync(0xffffffffu, st.mn, o));
  }
  st.nf = __any_sync(0xffffffffu, st.nf);
  const int e = row_exponent(st.mx);
  if (lane == 0) {
    const int code = row_code(st, e);
    exps[m] = code;
    if (code_wide(code)) wide[2 + atomicAdd(wide, 1)] = (int32_t)m;
  }
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int k0 = c * 256 + lane * 8;
    if (k0 >= kp) break;
    uint64_t w[OZ_S];
    split8(v[c], e, w);
#pragma unroll
    for (int s = 0; s < OZ_S; ++s)
      *reinterpret_cast<uint64_t*>(digits + ((int64_t)s * rows_p + m) * kp + k0) = w[s];
  }
}

// inner > 1: the contracted index k is strided; rows m = b inner + i.  A block stages a K x 32 tile
// (coalesced over i), takes the column maxima, and writes the digit rows k-contiguous (transposed).
// CW = 16 columns i per block (a K x 16 tile: 32 KB at K = 256, six blocks per SM; the launch site records
// the measured alternatives).  Lane l of a warp covers column l % CW of rows k = l / CW (mod 32 / CW).
template <int CW>
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const double* __restrict__ x, int64_t batch, int K,
                                                            int64_t inner, int8_t* __restrict__ digits,
                                                            int32_t* __restrict__ exps, int32_t* __restrict__ wide,
                                                            int64_t rows_p, int kp,
                                                            const double* __restrict__ lam_row,
                                                            const double* __restrict__ lam_k, const int* skip) {
  if (skip && *skip) return;
  constexpr int RPW = 32 / CW;  // rows per warp instruction
  // [K][CW] tile, column i of row k stored at i ^ ((k / 8) mod CW): conflict-free both for the row-wise
  // staging (lanes = i) and for the digit pass (lanes = 8-row chunks c of one column i)
  extern __shared__ double tile[];
  __shared__ double pmax[8 * RPW][CW], pmin[8 * RPW][CW];
  __shared__ int pnf[CW];
  __shared__ int es[CW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = lane % CW, rsub = lane / CW;
  const int64_t tiles_i = (inner + CW - 1) / CW;
  const int64_t b = blockIdx.x / tiles_i;
  const int64_t i0 = (blockIdx.x % tiles_i) * CW;
  const double* xb = x + b * K * inner;
  RowStat st;
  const bool iv = i0 + col < inner;
  if (threadIdx.x < CW) pnf[threadIdx.x] = 0;
  // the whole K x CW tile in flight at once: 8-byte cp.async (zero-filled outside [0, inner)), no registers
  for (int k = warp * RPW + rsub; k < K; k += 8 * RPW)
    cp_async8(smem_u32(&tile[k * CW + (col ^ ((k >> 3) & (CW - 1)))]),
              iv ? xb + (int64_t)k * inner + i0 + col : xb, iv ? 8 : 0);
  cp_async_commit();
  cp_async_wait<0>();
  // each thread revisits only the elements it copied itself: no barrier needed before this pass
  // the eigenvalue-sum divide of the FD (eq:FD3D) when the split feeds the backward mode-d product
  const double lr = (lam_row && iv) ? lam_row[b * inner + i0 + col] : 0.0;
  for (int k = warp * RPW + rsub; k < K; k += 8 * RPW) {
    double* tp = &tile[k * CW + (col ^ ((k >> 3) & (CW - 1)))];
    double val = *tp;
    if (lam_row) {  // val / (lr + lam_k[k]) (< 1 ulp off), all on the FP64 pipe
      val *= rcp_fp64(lr + lam_k[k]);
      *tp = val;
    }
    st.add(val);
  }
  pmax[warp * RPW + rsub][col] = st.mx;
  pmin[warp * RPW + rsub][col] = st.mn;
  __syncthreads();  // (also orders the pnf reset above before the flags below)
  if (st.nf) atomicOr(&pnf[col], 1);
  __syncthreads();
  if (threadIdx.x < CW) {
    RowStat r;
    r.nf = pnf[threadIdx.x] != 0;
#pragma unroll
    for (int w = 0; w < 8 * RPW; ++w) {
      r.mx = fmax(r.mx, pmax[w][threadIdx.x]);
      r.mn = fmin(r.mn, pmin[w][threadIdx.x]);
    }
    const int e = row_exponent(r.mx);
    es[threadIdx.x] = e;
    if (i0 + threadIdx.x < inner) {
      const int code = row_code(r, e);
      exps[b * inner + i0 + threadIdx.x] = code;
      if (code_wide(code)) wide[2 + atomicAdd(wide, 1)] = (int32_t)(b * inner + i0 + threadIdx.x);
    }
  }
  __syncthreads();
  const int cpr = kp / 8;  // 8-byte chunks per digit row
  for (int item = threadIdx.x; item < CW * cpr; item += 256) {
    const int i = item / cpr, c = item % cpr;
    if (i0 + i >= inner) continue;
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = c * 8 + j;
      v[j] = k < K ? tile[k * CW + (i ^ ((k >> 3) & (CW - 1)))] : 0.0;
    }
    uint64_t w[OZ_S];
    split8(v, es[i], w);
    const int64_t m = b * inner + i0 + i;
#pragma unroll
    for (int s = 0; s < OZ_S; ++s)
      *reinterpret_cast<uint64_t*>(digits + ((int64_t)s * rows_p + m) * kp + c * 8) = w[s];
  }
}

// ---------------------------------------------------------------------------------------------
// tcgen05 GEMM
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
// K-major operand tile of 128-byte rows written by TMA with SWIZZLE_128B: 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Issued by a whole, converged warp with warp-uniform operands: one elected lane executes the MMA.  (Issuing
// from a single-lane branch made the compiler wrap every MMA in an ELECT / R2UR.BROADCAST loop to build its
// uniform-register operands: ~13 instructions and 43 ns per N = 64 MMA instead of ~26 ns.)
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  // the two descriptors share their high words (SBO, version, swizzle); only the low words (start address,
  // LBO) differ, and offsets added to them never carry (shared addresses < 2^18): 32-bit operands
  const uint32_t alo = (uint32_t)da, blo = (uint32_t)db, hi = (uint32_t)(da >> 32);
  asm volatile(
      "{\n .reg .pred p, e;\n .reg .b64 a, b;\n elect.sync _|e, 0xffffffff;\n mov.b64 a, {%1, %3};\n"
      " mov.b64 b, {%2, %3};\n setp.ne.b32 p, %5, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], a, b, %4, p;\n}\n" ::"r"(tmem_d),
      "r"(alo), "r"(blo), "r"(hi), "r"(idesc), "r"(acc));
}
// single-thread variant, for use inside a warp-converged `if (elect_one())` around a whole stage
__device__ __forceinline__ void mma_i8_1(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t e = 0;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(e));
  return e != 0;
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// instruction descriptor: D s32, A / B s8 (signed digit 0) or u8, K-major, N = 64, M = 128
__host__ __device__ constexpr uint32_t oz_idesc(bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
         ((uint32_t)(OZ_BM >> 4) << 24);
}
template <int I, int NKS>
__device__ __forceinline__ void oz_stage_mmas(uint32_t tbase, uint32_t tile, uint64_t da, uint64_t db_kc,
                                              bool first_kc);
template <int I>
__device__ __noinline__ void oz_stage_mmas_rt(uint32_t tbase, uint32_t tile, uint64_t da, uint64_t db_kc,
                                              bool first_kc, int nks);
constexpr int OZ_STAGES = 6;
constexpr int OZ_EW = 8;                    // epilogue warps: 4 lane quarters x 2 column halves
constexpr int OZ_EC = OZ_BN / (OZ_EW / 4);  // columns per epilogue thread
constexpr int OZ_THREADS = (OZ_EW + 2) * 32;  // + TMA producer warp + MMA warp
constexpr int OZ_XBYTES = OZ_BM * OZ_BK;  // one data digit plane chunk: 128 rows x 128 B
constexpr int OZ_FBYTES = OZ_BN * OZ_BK;  // one factor digit plane chunk: 64 rows x 128 B

struct OzKernelArgs {
  int64_t M, Nf;     // data rows, factor rows
  int64_t x_rows_p, f_rows_p;
  int KC;            // 128-wide k chunks
  int ks_last;       // K-steps of 32 in the last chunk that reach below the contraction length (1..4)
  int mt, nt;        // tiles along M and Nf
  int K;             // contraction length
  const int32_t* ex;
  const int32_t* ef;
  double* y;
  int64_t inner, bstride, mstride, fstride;
  bool yvec;         // y 16-byte aligned (double2 stores of column pairs when fstride == 1)
  // FP64 operands for the wide-row fallback (oz.cuh: OzGemmArgs)
  const double* xs;
  int64_t xs_b, xs_i, xs_k;
  const double* lam_row;
  const double* lam_k;
  const double* fs;
  int64_t ldf;
  const double* ft;  // F^T [k][f]
  int32_t* xw;       // wide lists (oz.cuh: OzOperand::wide) of the data and the factor
  const int32_t* fw;
  const int* skip;
};

__device__ __forceinline__ int64_t oz_out_off(const OzKernelArgs& a, int64_t m) {
  return (m / a.inner) * a.bstride + (m % a.inner) * a.mstride;
}
// X[m][k] of the FP64 data operand (divided by the eigenvalue sum when the split did so)
__device__ __forceinline__ double oz_x(const OzKernelArgs& a, const double* xr, double lr, int k) {
  const double xv = xr[k * a.xs_k];
  return a.lam_row ? xv / (lr + a.lam_k[k]) : xv;
}
// The guard's fallback (oz.cuh), run by the epilogue warps of every GEMM CTA after its last tile: the outputs
// of the CTA's tiles (its row tiles x its column tile) that belong to a wide data row (X's list) or a wide
// factor row (F's list) are recomputed as IEEE FP64 dot products of the FP64 operands and stored over the
// int8 results (each output has one owner CTA, so no grid-wide ordering is needed).  Items of 32 outputs:
// the item's shared operand row (K values) is staged in shared memory; thread (c, s) of the 8 epilogue warps
// sums k = s, s + 8, .. for output c (loads of F^T / of the data coalesced over c, 16 in flight), and the 8
// partial sums per output are added in a fixed order.  The last CTA to finish resets X's list for the next
// split.  No wide row: two loads and one atomic per CTA.
__device__ __forceinline__ void oz_bar_epi() { asm volatile("bar.sync 1, %0;\n" ::"n"(256) : "memory"); }
__device__ __forceinline__ void oz_fix_item(const OzKernelArgs& a, int64_t m, int64_t f, bool wide_row, double* sv,
                                            double* part, int c, int sl) {
  // sv holds the item's shared row; this thread's output is (m, f)
  double acc = 0.0;
  if (wide_row) {
    const int64_t fc = min(f, a.Nf - 1);
#pragma unroll 16
    for (int k = sl; k < a.K; k += 8) acc = fma(a.ft[k * a.Nf + fc], sv[k], acc);
  } else {
    const int64_t mc = min(m, a.M - 1);
    const double* xr = a.xs + (mc / a.inner) * a.xs_b + (mc % a.inner) * a.xs_i;
    const double lr = a.lam_row ? a.lam_row[mc] : 0.0;
#pragma unroll 16
    for (int k = sl; k < a.K; k += 8) acc = fma(sv[k], oz_x(a, xr, lr, k), acc);
  }
  part[sl * 32 + c] = acc;
  oz_bar_epi();
  if (sl == 0 && m < a.M && f < a.Nf) {
    double t = part[c];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += part[q * 32 + c];
    a.y[oz_out_off(a, m) + f * a.fstride] = t;
  }
  oz_bar_epi();
}
// mt_first / per_nt: the CTA's row tiles; [n0, n0 + BN) its factor rows.  Called by the 256 epilogue threads.
__device__ void oz_cta_fixup(const OzKernelArgs& a, int32_t* xw, const int32_t* fw, int mt_first, int per_nt,
                             int n0, double* sv, double* part) {
  const int c = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int nx = *(volatile int32_t*)xw, nf = *(volatile const int32_t*)fw;
  for (int i = 0; i < nx; ++i) {
    const int64_t m = xw[2 + i];
    const int mt = (int)(m / OZ_BM);
    if (mt < mt_first || (mt - mt_first) % per_nt) continue;
    const double* xr = a.xs + (m / a.inner) * a.xs_b + (m % a.inner) * a.xs_i;
    const double lr = a.lam_row ? a.lam_row[m] : 0.0;
    for (int k = threadIdx.x; k < a.K; k += 256) sv[k] = oz_x(a, xr, lr, k);
    oz_bar_epi();
    for (int h = 0; h < OZ_BN; h += 32) oz_fix_item(a, m, n0 + h + c, true, sv, part, c, sl);
  }
  for (int i = 0; i < nf; ++i) {
    const int64_t f = fw[2 + i];
    if (f < n0 || f >= n0 + OZ_BN) continue;
    for (int k = threadIdx.x; k < a.K; k += 256) sv[k] = a.fs[f * a.ldf + k];
    oz_bar_epi();
    for (int mt = mt_first; mt < a.mt; mt += per_nt)
      for (int r = 0; r < OZ_BM; r += 32) oz_fix_item(a, (int64_t)mt * OZ_BM + r + c, f, false, sv, part, c, sl);
  }
  // reset X's list once every CTA has read its count
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&xw[1], 1) == (int)gridDim.x - 1) {
      xw[0] = 0;
      xw[1] = 0;
    }
  }
}


// Accumulator hand-off between tiles.  Weight t (digit pairs i + j = t) of tile T lives in TMEM slot
// p(t, T) = t (T even) or NW - 1 - t (T odd).  The first k chunk of a tile takes the data digits in
// descending order (digit i first touches weight i), later chunks ascending, so in the last chunk weight t
// completes right after digit t.  The epilogue drains weights in ascending order, i.e. slots in the order
// 0, 1, .., NW - 1 for either parity, which is exactly the order in which the next tile first writes them:
// the epilogue of tile T runs under the MMAs of tile T + 1.
__device__ __forceinline__ int oz_slot(int t, uint32_t tile) { return (tile & 1) ? OZ_NW - 1 - t : t; }

// the MMAs of data digit I: pairs (I, j), j = 0..min(S - 1, NW - 1 - I), into weight I + j; 4 K-steps of 32.
// db_kc: descriptor of factor digit 0 of this k chunk (digit j is j chunks further).  Digit 0 is signed, the
// others unsigned: the instruction descriptor is chosen per pair.  In the first k chunk (descending digits)
// pair (I, 0) is the first write of weight I, and for the first digit (S - 1) also pair (I, 1) of weight
// I + 1 = NW - 1: those MMAs overwrite their slot.
template <int I, int NKS>
__device__ __forceinline__ void oz_stage_mmas(uint32_t tbase, uint32_t tile, uint64_t da, uint64_t db_kc,
                                              bool first_kc) {
  const uint32_t odd = tile & 1;
  // k step outer, digit pair inner: consecutive MMAs share the A (data) operand.  NKS K-steps of 32: fewer
  // than 4 in a last chunk that holds only padding zeros past the contraction length.  One elected lane
  // issues the whole stage (operands computed by the converged warp before the branch).
  if (elect_one()) {
#pragma unroll
    for (int kk = 0; kk < NKS; ++kk)
#pragma unroll
      for (int j = 0; j < OZ_S && I + j < OZ_NW; ++j) {
        const uint32_t td = tbase + (uint32_t)((odd ? OZ_NW - 1 - (I + j) : (I + j)) * OZ_BN);
        const bool first_touch = first_kc && (j == 0 || I == OZ_S - 1);
        mma_i8_1(td, da + 2 * kk, db_kc + (uint64_t)(j * (OZ_BN * OZ_BK >> 4) + 2 * kk), oz_idesc(I == 0, j == 0),
                 (kk != 0 || !first_touch) ? 1u : 0u);
      }
  }
  __syncwarp();
}

template <int I>
__device__ __noinline__ void oz_stage_mmas_rt(uint32_t tbase, uint32_t tile, uint64_t da, uint64_t db_kc,
                                              bool first_kc, int nks) {
  const uint32_t odd = tile & 1;
#pragma unroll 1
  for (int kk = 0; kk < nks; ++kk)
#pragma unroll
    for (int j = 0; j < OZ_S && I + j < OZ_NW; ++j) {
      const uint32_t td = tbase + (uint32_t)((odd ? OZ_NW - 1 - (I + j) : (I + j)) * OZ_BN);
      const bool first_touch = first_kc && (j == 0 || I == OZ_S - 1);
      mma_i8(td, da + 2 * kk, db_kc + (uint64_t)(j * (OZ_BN * OZ_BK >> 4) + 2 * kk), oz_idesc(I == 0, j == 0),
             (kk != 0 || !first_touch) ? 1u : 0u);
    }
}

// STREAM = false: the CTA's factor digits for all k chunks stay resident (K <= 256).  STREAM = true (K up to
// 512): one k chunk of the factor digits (7 x 8 KB) at a time, double-buffered, reloaded for every tile.
template <bool STREAM>
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_gemm_kernel(const __grid_constant__ CUtensorMap xmap,
                                                         const __grid_constant__ CUtensorMap fmap,
                                                         const __grid_constant__ OzKernelArgs a) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(1024) uint8_t oz_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~uintptr_t(1023));
  const int KC = a.KC;
  uint8_t* sF = smem;  // [KC][S] factor chunks (resident) or [2][S] (streamed)
  uint8_t* sX = smem + OZ_S * (STREAM ? 2 : KC) * OZ_FBYTES;  // data ring
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + OZ_STAGES * OZ_XBYTES);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* fbar = empty + OZ_STAGES;  // resident: [1] factor landed; streamed: [2] full + [2] empty
  uint64_t* sfull = fbar + 4;      // [NW] accumulator slot complete (MMA -> epilogue)
  uint64_t* sempty = sfull + OZ_NW;  // [NW] accumulator slot drained (epilogue -> MMA)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + OZ_NW);
  double* sSF = reinterpret_cast<double*>(sempty + OZ_NW + 2);  // 2^(e_f - WSHIFT) of the CTA's factor rows
  double* sFix = sSF + OZ_BN;                                   // fixup: [OZ_MAXKP] row + [8][32] partial sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int f = 0; f < 4; ++f) mbar_init(&fbar[f], 1);
    for (int t = 0; t < OZ_NW; ++t) {
      mbar_init(&sfull[t], 1);
      mbar_init(&sempty[t], OZ_EW);
    }
    fence_barrier_init();
  }
  if (warp == OZ_EW + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  // tile sequence of this CTA: column tile nt0 fixed, row tiles strided
  const int per_nt = gridDim.x / a.nt;
  const int nt0 = blockIdx.x % a.nt;
  const int mt_first = blockIdx.x / a.nt;
  const int n0 = nt0 * OZ_BN;

  if (warp == OZ_EW) {
    if (lane == 0) {
      if (!STREAM) {  // resident factor digit planes of this column tile, [kc][digit] chunks
        mbar_arrive_expect_tx(fbar, (uint32_t)(OZ_S * KC * OZ_FBYTES));
        for (int s = 0; s < OZ_S; ++s)
          for (int kc = 0; kc < KC; ++kc)
            tma_load_2d(sF + (kc * OZ_S + s) * OZ_FBYTES, &fmap, kc * OZ_BK, (int)(s * a.f_rows_p + n0), fbar);
      }
      uint32_t st = 0, ph = 0, fc = 0;
      bool wrapped = false;
      for (int mt = mt_first; mt < a.mt; mt += per_nt) {
        const int m0 = mt * OZ_BM;
        for (int kc = 0; kc < KC; ++kc) {
          if (STREAM) {  // this k chunk's factor digits into factor slot fc % 2
            const uint32_t fs = fc & 1;
            if (fc >= 2) mbar_wait(&fbar[2 + fs], ((fc >> 1) - 1) & 1);
            mbar_arrive_expect_tx(&fbar[fs], (uint32_t)(OZ_S * OZ_FBYTES));
            for (int s = 0; s < OZ_S; ++s)
              tma_load_2d(sF + (fs * OZ_S + s) * OZ_FBYTES, &fmap, kc * OZ_BK, (int)(s * a.f_rows_p + n0), &fbar[fs]);
            ++fc;
          }
          for (int pos = 0; pos < OZ_S; ++pos) {
            const int i = kc == 0 ? OZ_S - 1 - pos : pos;  // the MMA warp's digit order
            if (wrapped) mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], OZ_XBYTES);
            tma_load_2d(sX + st * OZ_XBYTES, &xmap, kc * OZ_BK, (int)(i * a.x_rows_p + m0), &full[st]);
            if (++st == OZ_STAGES) {
              st = 0;
              ph ^= 1;
              wrapped = true;
            }
          }
        }
      }
    }
  } else if (warp == OZ_EW + 1) {
    {  // the whole warp runs the issue loop (uniform operands); one elected lane issues
      if (!STREAM) mbar_wait(fbar, 0);
      tc_fence_after();
      const uint64_t da0 = sdesc_sw128(smem_u32(sX)), db0 = sdesc_sw128(smem_u32(sF));
      uint32_t st = 0, ph = 0, tl = 0, fc = 0;
      for (int mt = mt_first; mt < a.mt; mt += per_nt, ++tl) {
        for (int kc = 0; kc < KC; ++kc) {
          uint64_t dbk = db0 + (uint64_t)(kc * OZ_S * (OZ_FBYTES >> 4));
          if (STREAM) {
            const uint32_t fs = fc & 1;
            mbar_wait(&fbar[fs], (fc >> 1) & 1);
            tc_fence_after();
            dbk = db0 + (uint64_t)(fs * OZ_S * (OZ_FBYTES >> 4));
          }
          const bool first = kc == 0, last = kc == KC - 1;
          const int nks = last ? a.ks_last : OZ_BK / 32;  // K-steps of 32 carrying real contraction indices
          // one ring stage per data digit, its digit pairs fully unrolled (descriptor offsets are immediates)
#define OZ_STAGE(I)                                                                                  \
  {                                                                                                  \
    mbar_wait(&full[st], ph);                                                                        \
    tc_fence_after();                                                                                \
    if (first && tl > 0) { /* weights first written by this stage: their slots must be drained */  \
      if (I == OZ_S - 1) mbar_wait(&sempty[oz_slot(OZ_NW - 1, tl)], (tl - 1) & 1);                  \
      mbar_wait(&sempty[oz_slot(I, tl)], (tl - 1) & 1);                                              \
      tc_fence_after();                                                                              \
    }                                                                                                \
    {                                                                                                \
      const uint64_t da_ = da0 + (uint64_t)(st * (OZ_XBYTES >> 4));                                  \
      if (nks == OZ_BK / 32)                                                                         \
        oz_stage_mmas<I, OZ_BK / 32>(tbase, tl, da_, dbk, first);                                    \
      else /* short last chunk: a runtime K-step loop keeps the issue code small */                 \
        oz_stage_mmas_rt<I>(tbase, tl, da_, dbk, first, nks);                                        \
    }                                                                                                \
    tc_commit_elect(&empty[st]); /* frees the ring slot when these MMAs have read it */                    \
    if (last && !first) { /* ascending: weight I complete (and the last weight after the last digit) */ \
      tc_commit_elect(&sfull[oz_slot(I, tl)]);                                                             \
      if (I == OZ_S - 1) tc_commit_elect(&sfull[oz_slot(OZ_NW - 1, tl)]);                                  \
    }                                                                                                \
    if (++st == OZ_STAGES) {                                                                         \
      st = 0;                                                                                        \
      ph ^= 1;                                                                                       \
    }                                                                                                \
  }
          if (first) {
            static_assert(OZ_S == 7 && OZ_NW == 8, "stage sequences written for 7 digits, 8 weights");
            OZ_STAGE(6) OZ_STAGE(5) OZ_STAGE(4) OZ_STAGE(3) OZ_STAGE(2) OZ_STAGE(1) OZ_STAGE(0)
          } else {
            OZ_STAGE(0) OZ_STAGE(1) OZ_STAGE(2) OZ_STAGE(3) OZ_STAGE(4) OZ_STAGE(5) OZ_STAGE(6)
          }
#undef OZ_STAGE
          if (STREAM) {
            tc_commit_elect(&fbar[2 + (fc & 1)]);  // the factor slot is free when this chunk's MMAs have read it
            ++fc;
          }
          if (first && last)  // single k chunk (descending): every weight completes at its end
            for (int t = 0; t < OZ_NW; ++t) tc_commit_elect(&sfull[oz_slot(t, tl)]);
        }
      }
    }
  } else {
    // epilogue: warp w owns TMEM lanes 32w..32w+31 = data rows m0 + 32w + lane
    if (threadIdx.x < OZ_BN) {
      const int64_t f = n0 + threadIdx.x;
      sSF[threadIdx.x] = pow2(code_exp(f < a.Nf ? a.ef[f] : 0) - OZ_WSHIFT);
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(OZ_EW * 32) : "memory");  // epilogue warps only
    uint32_t tl = 0;
    // warp w: TMEM lanes 32 (w % 4).. (data rows), columns [32 (w / 4), +32) of every weight slot
    const int quarter = warp & 3, c0 = (warp >> 2) * OZ_EC;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int mt = mt_first; mt < a.mt; mt += per_nt, ++tl) {
      const int64_t m = (int64_t)mt * OZ_BM + quarter * 32 + lane;
      const bool mv = m < a.M;
      const int64_t mm = mv ? m : 0;
      const int64_t row_off = oz_out_off(a, mm);
      const double sx = pow2(code_exp(mv ? a.ex[mm] : 0));  // (outputs of wide rows: replaced by oz_fixup)
      // sum_t 2^{8 (NW - 1 - t)} C_t over the weights as they complete (largest weight first)
      double acc[OZ_EC];
#pragma unroll
      for (int c = 0; c < OZ_EC; ++c) acc[c] = 0.0;
#pragma unroll 1
      for (int t = 0; t < OZ_NW; ++t) {
        const int p = oz_slot(t, tl);
        mbar_wait(&sfull[p], tl & 1);
        tc_fence_after();
        const double w = (double)(1ll << (8 * (OZ_NW - 1 - t)));
#pragma unroll
        for (int c = 0; c < OZ_EC; c += 16) {
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tbase + lane_off + (uint32_t)(p * OZ_BN + c0 + c)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          // int32 -> double without I2F: the bits 0x43300000:(v ^ 2^31) are 2^52 + 2^31 + v exactly, and
          // subtracting 2^52 + 2^31 is exact
          for (int q = 0; q < 16; ++q)
            acc[c + q] = fma(__hiloint2double(0x43300000, (int)(v[q] ^ 0x80000000u)) - 4503601774854144.0, w,
                             acc[c + q]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[p]);
      }
      if (mv) {  // (outputs of wide rows: replaced by oz_cta_fixup after the last tile)
        const bool vec = a.yvec && a.fstride == 1 && ((row_off + n0 + c0) & 1) == 0;
#pragma unroll
        for (int c = 0; c < OZ_EC; c += 2) {
          const int64_t f = n0 + c0 + c;
          // two exact power-of-two scalings: the factor row's (with the digit weight) and the data row's
          const double y0 = (acc[c] * sSF[c0 + c]) * sx;
          const double y1 = (acc[c + 1] * sSF[c0 + c + 1]) * sx;
          if (vec && f + 1 < a.Nf) {  // contiguous factor index (mode 1): one 16-byte store per pair
            *reinterpret_cast<double2*>(a.y + row_off + f) = make_double2(y0, y1);
          } else {
            if (f < a.Nf) a.y[row_off + f * a.fstride] = y0;
            if (f + 1 < a.Nf) a.y[row_off + (f + 1) * a.fstride] = y1;
          }
        }
      }
    }
    oz_cta_fixup(a, a.xw, a.fw, mt_first, per_nt, n0, sFix, sFix + OZ_MAXKP);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == OZ_EW + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// ---------------------------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int get_encode(EncodeTiledFn* fn) {
  static EncodeTiledFn f = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess) f = reinterpret_cast<EncodeTiledFn>(p);
  });
  FDIGA_CHECK(f, FDIGA_ERR_CUDA, "cuTensorMapEncodeTiled not available (%s)", cudaGetErrorString(err));
  *fn = f;
  return FDIGA_OK;
}

constexpr size_t oz_smem_bytes(int KC) {
  return 1024 + (size_t)OZ_S * (KC > 2 ? 2 : KC) * OZ_FBYTES + (size_t)OZ_STAGES * OZ_XBYTES +
         (2 * OZ_STAGES + 4 + 2 * OZ_NW + 2) * 8 +
         (OZ_BN + OZ_MAXKP + 8 * 32) * sizeof(double);
}

// cudaFuncSetAttribute is per device: one flag bit per device ordinal
bool attr_once(std::atomic<uint64_t>& done, int device) {
  const uint64_t bit = 1ull << (device & 63);
  return !(done.fetch_or(bit) & bit);
}

}  // namespace

int oz_operand_alloc(OzOperand& op, int64_t rows, int64_t k, int box_rows) {
  const int64_t kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
  const int64_t rows_p = (rows + box_rows - 1) / box_rows * box_rows;
  FDIGA_CHECK(kp <= OZ_MAXKP, FDIGA_ERR_NOT_SUPPORTED, "int8-split FD: contraction length %lld > %d",
              (long long)k, OZ_MAXKP);
  if (rows == 0) {  // a rank without planes / chunk: nothing to split or multiply
    op.release();
    op.box_rows = box_rows;
    op.kp = kp;
    return FDIGA_OK;
  }
  if (op.digits && op.rows_p == rows_p && op.kp == kp && op.box_rows == box_rows) {
    op.rows = rows;
    FDIGA_CUDA(cudaMemset(op.wide, 0, 2 * sizeof(int32_t)));
    return FDIGA_OK;
  }
  op.release();
  FDIGA_CUDA(cudaMalloc(&op.digits, (size_t)OZ_S * rows_p * kp));
  FDIGA_CUDA(cudaMemset(op.digits, 0, (size_t)OZ_S * rows_p * kp));
  FDIGA_CUDA(cudaMalloc(&op.exps, (size_t)rows_p * sizeof(int32_t)));
  FDIGA_CUDA(cudaMemset(op.exps, 0, (size_t)rows_p * sizeof(int32_t)));
  FDIGA_CUDA(cudaMalloc(&op.wide, (size_t)(rows_p + 2) * sizeof(int32_t)));
  FDIGA_CUDA(cudaMemset(op.wide, 0, 2 * sizeof(int32_t)));
  op.rows = rows;
  op.rows_p = rows_p;
  op.kp = kp;
  op.box_rows = box_rows;
  EncodeTiledFn enc;
  FDIGA_TRY(get_encode(&enc));
  cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)(OZ_S * rows_p)};
  cuuint64_t strides[1] = {(cuuint64_t)kp};
  cuuint32_t box[2] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  static_assert(sizeof(CUtensorMap) <= sizeof(op.tmap), "tensor map size");
  const CUresult r = enc(reinterpret_cast<CUtensorMap*>(op.tmap), CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, op.digits, dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  FDIGA_CHECK(r == CUDA_SUCCESS, FDIGA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FDIGA_OK;
}

int oz_operand_set_ft(OzOperand& op, const double* F_host, int64_t n) {
  std::vector<double> t((size_t)(n * n));
  for (int64_t f = 0; f < n; ++f)
    for (int64_t k = 0; k < n; ++k) t[(size_t)(k * n + f)] = F_host[f * n + k];
  if (op.ft) cudaFree(op.ft);
  op.ft = nullptr;
  FDIGA_CUDA(cudaMalloc(&op.ft, t.size() * sizeof(double)));
  FDIGA_CUDA(cudaMemcpy(op.ft, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice));
  return FDIGA_OK;
}

int oz_split(fdiga_ctx* ctx, cudaStream_t stream, const double* x, int64_t batch, int64_t K, int64_t inner,
             int64_t ldx, OzOperand& op, const int* skip, const double* lam_row, const double* lam_k) {

  const int64_t rows = batch * inner;
  FDIGA_CHECK(rows == op.rows && K <= op.kp, FDIGA_ERR_INVALID_ARG, "oz_split: operand shape mismatch");
  if (rows == 0) return FDIGA_OK;
  if (inner == 1 && !lam_row) {  // (the divide is done by the strided kernel, which handles inner == 1 too)
    const unsigned grid = (unsigned)((rows + 7) / 8);
    if (op.kp <= 256)
      oz_split_rows_kernel<1><<<grid, 256, 0, stream>>>(x, rows, (int)K, ldx, op.digits, op.exps, op.wide, op.rows_p,
                                                        (int)op.kp, skip);
    else
      oz_split_rows_kernel<2><<<grid, 256, 0, stream>>>(x, rows, (int)K, ldx, op.digits, op.exps, op.wide, op.rows_p,
                                                        (int)op.kp, skip);
  } else {
    static std::atomic<uint64_t> attr{0};
    if (attr_once(attr, ctx->device))
      FDIGA_CUDA(cudaFuncSetAttribute(oz_split_cols_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    // 16 columns per block for every K (<= 512): 32 KB tiles at K = 256, six blocks per SM; at n = 256 this
    // beats 32 columns (three blocks per SM: 1.351 vs 1.336 ms per apply) and 8 (64-byte row segments: 1.368)
    const int64_t tiles = batch * ((inner + 15) / 16);
    oz_split_cols_kernel<16><<<(unsigned)tiles, 256, (size_t)K * 16 * sizeof(double), stream>>>(
        x, batch, (int)K, inner, op.digits, op.exps, op.wide, op.rows_p, (int)op.kp, lam_row, lam_k, skip);
  }
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

int oz_gemm(fdiga_ctx* ctx, cudaStream_t stream, const OzGemmArgs& g) {
  const OzOperand& X = *g.X;
  const OzOperand& F = *g.F;
  FDIGA_CHECK(g.K >= 1 && g.K <= X.kp, FDIGA_ERR_INVALID_ARG, "oz_gemm: contraction length %lld outside (0, %lld]",
              (long long)g.K, (long long)X.kp);
  FDIGA_CHECK(X.kp == F.kp && X.box_rows == OZ_BM && F.box_rows == OZ_BN, FDIGA_ERR_INVALID_ARG,
              "oz_gemm: operand mismatch");
  if (X.rows == 0 || F.rows == 0) return FDIGA_OK;
  OzKernelArgs a{};
  a.M = X.rows;
  a.Nf = F.rows;
  a.x_rows_p = X.rows_p;
  a.f_rows_p = F.rows_p;
  a.KC = (int)(X.kp / OZ_BK);
  a.ks_last = (int)((g.K - (a.KC - 1) * OZ_BK + 31) / 32);  // g.K: the true contraction length
  a.mt = (int)(X.rows_p / OZ_BM);
  a.nt = (int)(F.rows_p / OZ_BN);
  a.K = (int)g.K;
  a.ex = X.exps;
  a.ef = F.exps;
  a.y = g.y;
  a.inner = g.inner;
  a.bstride = g.bstride;
  a.mstride = g.mstride;
  a.fstride = g.fstride;
  a.yvec = (reinterpret_cast<uintptr_t>(g.y) & 15) == 0;
  a.xs = g.xs;
  a.xs_b = g.xs_b;
  a.xs_i = g.xs_i;
  a.xs_k = g.xs_k;
  a.lam_row = g.lam_row;
  a.lam_k = g.lam_k;
  a.fs = g.fs;
  a.ldf = g.ldf;
  a.ft = F.ft;
  a.xw = X.wide;
  a.fw = F.wide;
  a.skip = g.skip;
  FDIGA_CHECK(g.xs && g.fs && F.ft, FDIGA_ERR_INVALID_ARG, "oz_gemm: FP64 operands for the wide-row fallback missing");
  FDIGA_CHECK(a.nt <= ctx->sm_count, FDIGA_ERR_NOT_SUPPORTED, "oz_gemm: too many column tiles");
  const size_t smem = oz_smem_bytes(a.KC);
  static std::atomic<uint64_t> attr{0};
  if (attr_once(attr, ctx->device)) {
    FDIGA_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz_smem_bytes(2)));
    FDIGA_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz_smem_bytes(4)));
  }
  // persistent grid: a multiple of the column-tile count, at most one CTA per SM (TMEM: 512 columns)
  int64_t grid = (int64_t)(ctx->sm_count / a.nt) * a.nt;
  grid = std::min<int64_t>(grid, (int64_t)a.mt * a.nt);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 0;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  const bool stream_f = a.KC > 2;
  auto kern = stream_f ? oz_gemm_kernel<true> : oz_gemm_kernel<false>;
  FDIGA_CUDA(cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(X.tmap),
                                *reinterpret_cast<const CUtensorMap*>(F.tmap), a));
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

}  // namespace fdiga
