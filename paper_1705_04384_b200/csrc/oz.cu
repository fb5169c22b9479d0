// FD mode products on tcgen05 int8 tensor cores with exact digit splitting (see oz.cuh).
//
//   oz_split_*_kernel : FP64 operand -> S = 7 int8 digit planes + per-row exponents (HBM-bound pass; the
//                       strided modes are transposed so every GEMM operand is K-major)
//   oz_gemm_kernel    : persistent, warp-specialised tcgen05 GEMM on CTA pairs (cta_group::2, M = 256, N = 128).
//                       Warp 16 streams the data digit planes through a TMA (SWIZZLE_64B) ring, one full /
//                       empty barrier pair per 64-wide k chunk; warps 17 and 18 of the leader CTA (converged,
//                       one elected lane) issue tcgen05.mma.kind::i8 into int32 accumulators in TMEM (one per
//                       digit-pair weight t = i + j, two passes of four weights over the contraction); warps
//                       0-15 read them back with tcgen05.ld, combine in FP64,
//                       scale by the row exponents and store.  The factor's digit planes for the CTA's half of
//                       the column tile stay resident in shared memory for contractions <= 256; longer ones
//                       (<= 512) stream them through the ring beside the data planes (oz_gemm_kernel<true>).
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
// Programmatic dependent launch: every kernel of the int8 path is launched with the programmatic-stream-
// serialization attribute, lets its successor be scheduled at once (pdl_trigger) and waits for its predecessor's
// completion and memory (pdl_wait) before it touches anything that kernel wrote or still reads.  The
// successor's launch latency and prologue (barrier set-up, TMEM allocation) then overlap this kernel's tail.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

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
  pdl_trigger();
  pdl_wait();
  if (skip && *skip) return;
  const int lane = threadIdx.x & 31;
  // blocks run over the rows from the last to the first: the GEMM before this split wrote y in increasing row
  // order and the GEMM after it reads the digits in increasing row order, so the split reads what was written
  // last (still in L2) first and leaves the digits the next GEMM needs first for last
  const int64_t m = (int64_t)(gridDim.x - 1 - blockIdx.x) * 8 + (threadIdx.x >> 5);
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

// inner > 1: the contracted index k is strided; rows m = b inner + i.  A block stages a K x 16 tile
// (16 columns i, coalesced 128-byte rows), takes the column statistics, and writes the digit rows
// k-contiguous (transposed).  Column i of row k is stored at i ^ ((k / 8) mod 16): conflict-free both for the
// row-wise staging (lanes = i) and for the digit pass (lanes = 8-row chunks c of one column).  The loops
// step pointers and swizzle terms incrementally and the digit pass maps thread t to column t / 16 and the
// chunks c = t mod 16 (+ 16, ..): no integer division or 64-bit multiply per element (an earlier version
// was issue-bound on address arithmetic: 3.5 warp instructions per element).
constexpr int OZ_CW = 16;
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const double* __restrict__ x, int64_t batch, int K,
                                                            int64_t inner, int8_t* __restrict__ digits,
                                                            int32_t* __restrict__ exps, int32_t* __restrict__ wide,
                                                            int64_t rows_p, int kp,
                                                            const double* __restrict__ lam_row,
                                                            const double* __restrict__ lam_k, const int* skip) {
  pdl_trigger();
  pdl_wait();
  if (skip && *skip) return;
  constexpr int CW = OZ_CW, RG = 256 / CW;  // 16 columns, 16 row groups
  extern __shared__ double tile[];
  __shared__ double pmax[RG][CW], pmin[RG][CW];
  __shared__ int pnf[RG][CW];
  __shared__ int es[CW];
  const int col = threadIdx.x % CW, rg = threadIdx.x / CW;
  const int64_t tiles_i = (inner + CW - 1) / CW;
  const int64_t blk = (int64_t)gridDim.x - 1 - blockIdx.x;  // last tiles first (see oz_split_rows_kernel)
  const int64_t b = blk / tiles_i;
  const int64_t i0 = (blk - b * tiles_i) * CW;
  const bool iv = i0 + col < inner;
  // ---- stage the K x 16 tile: thread (col, rg) copies rows k = rg, rg + 16, .. of its column
  {
    const double* src = x + b * K * inner + (int64_t)rg * inner + i0 + col;
    const int64_t step = RG * inner;
    uint32_t dst = smem_u32(tile) + 8u * (uint32_t)(rg * CW);
    for (int k = rg; k < K; k += RG, src += step, dst += 8u * RG * CW)
      cp_async8(dst + 8u * (uint32_t)(col ^ ((k >> 3) & (CW - 1))), iv ? src : x, iv ? 8 : 0);
    cp_async_commit();
    cp_async_wait<0>();
  }
  // ---- column statistics over the elements this thread copied (no barrier needed); the eigenvalue-sum
  // divide of the FD (eq:FD3D) when the split feeds the backward mode-d product
  RowStat st;
  {
    const double lr = (lam_row && iv) ? lam_row[b * inner + i0 + col] : 0.0;
    double* tp = tile + rg * CW;
    for (int k = rg; k < K; k += RG, tp += RG * CW) {
      double* e = tp + (col ^ ((k >> 3) & (CW - 1)));
      double val = *e;
      if (lam_row) {  // val / (lr + lam_k[k]) (< 1 ulp off), all on the FP64 pipe
        val *= rcp_fp64(lr + lam_k[k]);
        *e = val;
      }
      st.add(val);
    }
  }
  pmax[rg][col] = st.mx;
  pmin[rg][col] = st.mn;
  pnf[rg][col] = st.nf ? 1 : 0;
  __syncthreads();
  if (threadIdx.x < CW) {
    RowStat r;
#pragma unroll
    for (int w = 0; w < RG; ++w) {
      r.mx = fmax(r.mx, pmax[w][threadIdx.x]);
      r.mn = fmin(r.mn, pmin[w][threadIdx.x]);
      r.nf |= pnf[w][threadIdx.x] != 0;
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
  // ---- digits: thread (i = t / 16, chunks c = t mod 16, + 16, ..) of 8 k values each
  const int i = threadIdx.x / 16, cq = threadIdx.x % 16;
  if (i0 + i >= inner) return;
  const int e = es[i];
  const int64_t plane = rows_p * (int64_t)kp;
  int8_t* drow = digits + (b * inner + i0 + i) * (int64_t)kp;
  const int cpr = kp / 8;
  for (int c = cq; c < cpr; c += 16) {
    const double* tc = tile + (8 * c) * CW + (i ^ (c & (CW - 1)));
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (8 * c + j < K) ? tc[j * CW] : 0.0;
    uint64_t w[OZ_S];
    split8(v, e, w);
    int8_t* dp = drow + 8 * c;
#pragma unroll
    for (int s2 = 0; s2 < OZ_S; ++s2, dp += plane) *reinterpret_cast<uint64_t*>(dp) = w[s2];
  }
}

// ---------------------------------------------------------------------------------------------
// tcgen05 GEMM (CTA pairs, cta_group::2)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cluster address of `p`'s counterpart in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// remote arrive (CTA-scope release: the arriving warp's tcgen05.ld are complete, and it orders no global
// stores for the peer -- a cluster-scope release would wait for the warp's outstanding y stores)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}
// pair TMA: the bytes land in this CTA's shared memory, completion is signalled on the leader's mbarrier
__device__ __forceinline__ void tma_load_2sm(void* dst, const void* map, int x, int y, uint32_t bar_leader) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_leader)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
// single-thread MMA of the pair (issued by the leader CTA inside a warp-converged `if (elect_one())` around a
// whole stage): D (128 lanes x N columns in each CTA's TMEM) += A (128 rows from each CTA) B^T (N / 2 rows
// from each CTA), both operands at the same shared-memory offsets in the two CTAs
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t e = 0;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(e));
  return e != 0;
}
// arrive on the mbarrier at `bar`'s offset in both CTAs of the pair once the MMAs issued so far complete
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// instruction descriptor: D s32, A / B s8 (signed digit 0) or u8, K-major, N = 128, M = 256 (the pair)
__host__ __device__ constexpr uint32_t oz_idesc(bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
         ((uint32_t)(OZ_PM >> 4) << 24);
}
// K-major operand tile of 64-byte rows written by TMA with SWIZZLE_64B: 8-row atoms 512 B apart
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
constexpr int OZ_NSLOT = 4;                 // TMEM accumulator slots of OZ_BN columns (4 x 128 = 512)
constexpr int OZ_EW = 16;                   // epilogue warps: 4 lane quarters x 4 column groups of 32
constexpr int OZ_EC = 32;                   // columns per epilogue thread
constexpr int OZ_THREADS = (OZ_EW + 3) * 32;  // + TMA producer warp + two MMA warps
constexpr int OZ_KCH = 64;                  // k per chunk (bytes of a SWIZZLE_64B row)
constexpr int OZ_KCMAX = 4;                 // chunks per launch: contraction <= 256 per launch
constexpr int OZ_XPL = OZ_BM * OZ_KCH;      // one data digit plane chunk per CTA: 128 rows x 64 B = 8 KB
constexpr int OZ_FPL = OZ_BNH * OZ_KCH;     // one factor digit plane chunk per CTA: 64 rows x 64 B = 4 KB
constexpr int OZ_NXS = 14;                  // data plane slots in the ring (two 7-plane chunks)
// Streamed-factor variant (contractions 256 < K <= 512 in one launch): no resident factor; every ring slot holds
// a data digit plane chunk (8 KB) and, behind it, the same digit's factor plane chunk (4 KB)
constexpr int OZ_NXS_SF = 18;
constexpr int OZ_SLOT_SF = OZ_BM * 64 + OZ_BNH * 64;  // = OZ_XPL + OZ_FPL (defined below): 12 KB
constexpr int OZ_NCB = 8;                   // chunk barriers (full / empty pairs): more than the chunks in flight
static_assert(OZ_EC * (OZ_EW / 4) == OZ_BN, "epilogue column groups cover the tile");

struct OzKernelArgs {
  int64_t M, Nf;     // data rows, factor rows
  int64_t x_rows_p, f_rows_p;
  int KC;            // 64-wide k chunks of this launch
  int kbase;         // first k of this launch (contractions > 256 take two launches)
  int ks_last;       // K-steps of 32 in the last chunk that reach below the contraction length (1..2)
  int mt, nt;        // pair tiles along M (256 rows) and Nf (128 rows)
  int K;             // contraction length (all launches)
  bool accum;        // y += (the second launch of a split contraction); else y =
  bool fixup;        // the launch that recomputes the outputs of wide rows (the last one)
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
// of the CTA's 128-row halves of its pair tiles (x the pair's factor rows) that belong to a wide data row
// (X's list) or a wide factor row (F's list) are recomputed as IEEE FP64 dot products of the FP64 operands and
// stored over the int8 results (each output has one owner CTA, so no grid-wide ordering is needed).  Items of
// 32 outputs: the item's shared operand row (K values) is staged in shared memory; thread (c, s) of the
// OZ_EW epilogue warps sums k = s, s + OZ_EW, .. for output c (loads of F^T / of the data coalesced over c),
// and the partial sums per output are added in a fixed order.  The last CTA to finish resets X's list for the
// next split.  No wide row: two loads and one atomic per CTA.
__device__ __forceinline__ void oz_bar_epi() { asm volatile("bar.sync 1, %0;\n" ::"n"(OZ_EW * 32) : "memory"); }
__device__ __forceinline__ void oz_fix_item(const OzKernelArgs& a, int64_t m, int64_t f, bool wide_row, double* sv,
                                            double* part, int c, int sl) {
  // sv holds the item's shared row; this thread's output is (m, f)
  double acc = 0.0;
  if (wide_row) {
    const int64_t fc = min(f, a.Nf - 1);
#pragma unroll 8
    for (int k = sl; k < a.K; k += OZ_EW) acc = fma(a.ft[k * a.Nf + fc], sv[k], acc);
  } else {
    const int64_t mc = min(m, a.M - 1);
    const double* xr = a.xs + (mc / a.inner) * a.xs_b + (mc % a.inner) * a.xs_i;
    const double lr = a.lam_row ? a.lam_row[mc] : 0.0;
#pragma unroll 8
    for (int k = sl; k < a.K; k += OZ_EW) acc = fma(sv[k], oz_x(a, xr, lr, k), acc);
  }
  part[sl * 32 + c] = acc;
  oz_bar_epi();
  if (sl == 0 && m < a.M && f < a.Nf) {
    double t = part[c];
#pragma unroll
    for (int q = 1; q < OZ_EW; ++q) t += part[q * 32 + c];
    a.y[oz_out_off(a, m) + f * a.fstride] = t;
  }
  oz_bar_epi();
}
// The CTA's rows: [mt OZ_PM + rank OZ_BM, + OZ_BM) for mt = mt_first, mt_first + per_nt, ..; its factor rows
// [n0, n0 + OZ_BN).  Called by the OZ_EW epilogue warps.
__device__ void oz_cta_fixup(const OzKernelArgs& a, int mt_first, int per_nt, uint32_t rank, int n0, double* sv,
                             double* part) {
  const int c = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int nx = *(volatile int32_t*)a.xw, nf = *(volatile const int32_t*)a.fw;
  // the wide-row list is scanned from shared memory, a batch of OZ_EW * 32 entries per coalesced load (scanned
  // from global memory it cost every CTA one dependent L2 round trip per entry: ~12 k cycles of tail per GEMM
  // for two dozen wide rows)
  int32_t* lst = reinterpret_cast<int32_t*>(part + OZ_EW * OZ_BN);
  for (int i = 0; i < nx; ++i) {
    if (i % (OZ_EW * 32) == 0) {
      oz_bar_epi();
      if (i + (int)threadIdx.x < nx) lst[threadIdx.x] = a.xw[2 + i + threadIdx.x];
      oz_bar_epi();
    }
    const int64_t m = lst[i % (OZ_EW * 32)];
    const int mt = (int)(m / OZ_PM);
    if (mt < mt_first || (mt - mt_first) % per_nt || (uint32_t)((m % OZ_PM) / OZ_BM) != rank) continue;
    const double* xr = a.xs + (m / a.inner) * a.xs_b + (m % a.inner) * a.xs_i;
    const double lr = a.lam_row ? a.lam_row[m] : 0.0;
    for (int k = threadIdx.x; k < a.K; k += OZ_EW * 32) sv[k] = oz_x(a, xr, lr, k);
    oz_bar_epi();
    // all OZ_BN outputs of the row at once: thread (c, sl) sums k = sl, sl + OZ_EW, .. for the columns
    // c, c + 32, .. (independent loads in flight), then the OZ_EW partial sums per output in a fixed order
    constexpr int NQ = OZ_BN / 32;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    const double* ftc = a.ft + n0 + c;
#pragma unroll 4
    for (int k = sl; k < a.K; k += OZ_EW) {
      const double xv = sv[k];
      const double* fk = ftc + (int64_t)k * a.Nf;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (n0 + c + 32 * q < a.Nf) acc[q] = fma(fk[32 * q], xv, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) part[sl * OZ_BN + 32 * q + c] = acc[q];
    oz_bar_epi();
    if (threadIdx.x < OZ_BN) {
      const int64_t f = n0 + threadIdx.x;
      if (f < a.Nf) {
        double t = part[threadIdx.x];
#pragma unroll
        for (int q = 1; q < OZ_EW; ++q) t += part[q * OZ_BN + threadIdx.x];
        a.y[oz_out_off(a, m) + f * a.fstride] = t;
      }
    }
    oz_bar_epi();
  }
  for (int i = 0; i < nf; ++i) {
    if (i % (OZ_EW * 32) == 0) {
      oz_bar_epi();
      if (i + (int)threadIdx.x < nf) lst[threadIdx.x] = a.fw[2 + i + threadIdx.x];
      oz_bar_epi();
    }
    const int64_t f = lst[i % (OZ_EW * 32)];
    if (f < n0 || f >= n0 + OZ_BN) continue;
    for (int k = threadIdx.x; k < a.K; k += OZ_EW * 32) sv[k] = a.fs[f * a.ldf + k];
    oz_bar_epi();
    for (int mt = mt_first; mt < a.mt; mt += per_nt)
      for (int r = 0; r < OZ_BM; r += 32)
        oz_fix_item(a, (int64_t)mt * OZ_PM + rank * OZ_BM + r + c, f, false, sv, part, c, sl);
  }
  // reset X's list once every CTA has read its count
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.xw[1], 1) == (int)gridDim.x - 1) {
      a.xw[0] = 0;
      a.xw[1] = 0;
    }
  }
}

// Passes per tile over the contraction (FDIGA_OZ_NPASS):
//   2 (default): two passes of four weights, pass 0 the weights 0..3 (data digits 0..3), pass 1 the weights 6, 5,
//      7, 4 (digits 0..6): all four 128-column TMEM slots per pass, 11 data plane chunks per 64 k.
//   4: four passes of two weights each.  The slots form two groups {0, 1} and {2, 3} used by alternating passes,
//      so the epilogue drains a pass's two accumulators while the MMAs of the next pass fill the other group.
//      Price: a pass streams the data digit planes its weights need again, 19 plane chunks per 64 k instead of 11.
//      Pass order (0,1) (2,3) (4,5) (6,7) (FDIGA_OZ_ORDER 1: 2, 4, 6, 7 planes); order 0 = (4,5) (6,7) (0,3) (1,2)
//      and order 2 = (0,7) (1,6) (2,5) (3,4) (balanced MMA counts, 25 planes) measured 1 % and 8 % slower.
// Measured (in-kernel clock64 timeline, tools/oz_trace.py; tools/oz_ab.py, tools/oz_sustained.py): both schedules
// run at ~32 k cycles per tile at n = 256 against 17.4 k cycles of MMAs (272 at the probe rate).  What bounds a
// tile is the interference between the tensor pipe and the epilogue inside the SM, not the schedule: under a
// saturated MMA stream a slot drain takes 4-7 k cycles instead of ~1 k alone (tcgen05.ld gets what the MMAs'
// accumulator traffic leaves), and the tile's 128 KB of y stores take 6 k instead of 3 k cycles while they in
// turn slow the MMAs (138 instead of ~80 cycles each: the stores and the MMAs' operand reads share the L1 /
// shared-memory path).  From idle (burst) the two schedules are within 1 % at n = 256 (four passes 2.5 % ahead
// at n = 384, two passes 2 % ahead at n = 512); under sustained load the path is limited by the board's 1000 W
// power cap, and the schedule that moves less data wins: two passes 1.230 vs 1.253 ms per n = 256 apply (SM
// clock 1732 vs 1702 MHz), 20.2 vs 20.6 ms at n = 512, equal at n = 384.  Hence the default.
// Phase q = NPASS tile + pass; its k-th weight lives in slot (pass WPP + k) mod 4, used for the (q / NGRP)-th
// time.  Within every 64-wide k chunk the MMAs go weight by weight, so a pass's slots complete one after
// another in the last chunk and the epilogue drains slot k while the remaining weights' MMAs run.
#ifndef FDIGA_OZ_PDL_DEFAULT
#define FDIGA_OZ_PDL_DEFAULT 2
#endif
#ifndef FDIGA_OZ_NPASS
#define FDIGA_OZ_NPASS 2
#endif
#ifndef FDIGA_OZ_ORDER
#define FDIGA_OZ_ORDER 1
#endif
#ifdef FDIGA_OZ_TRACE  // in-kernel clock64 timeline of CTA pair 0 (variant builds; tools/oz_trace.py)
__device__ long long oz_trace_buf[4096];
#define OZ_TR(cond, idx, val)                                 \
  do {                                                        \
    if ((cond) && blockIdx.x == 0 && (threadIdx.x & 31) == 0) oz_trace_buf[(idx)] = (val); \
  } while (0)
#else
#define OZ_TR(cond, idx, val) do { } while (0)
#endif
constexpr int OZ_NPASS = FDIGA_OZ_NPASS;
constexpr int OZ_WPP = OZ_NW / OZ_NPASS;      // weights per pass
constexpr int OZ_NGRP = OZ_NSLOT / OZ_WPP;    // slot groups (passes in flight: one filling, the others draining)
static_assert(OZ_NPASS == 2 || OZ_NPASS == 4, "two passes of four weights or four passes of two");
__host__ __device__ constexpr int oz_weight(int P, int k) {
  if (OZ_NPASS == 2) return P == 0 ? k : (k == 0 ? 6 : k == 1 ? 5 : k == 2 ? 7 : 4);
  if (FDIGA_OZ_ORDER == 1) return 2 * P + k;                                  // (0,1) (2,3) (4,5) (6,7)
  if (FDIGA_OZ_ORDER == 2) return k == 0 ? P : 7 - P;                         // (0,7) (1,6) (2,5) (3,4)
  return P == 0 ? 4 + k : P == 1 ? 6 + k : P == 2 ? (k == 0 ? 0 : 3) : 1 + k;  // (4,5) (6,7) (0,3) (1,2)
}
// data digit planes 0 .. nd - 1 a pass needs: weight t pairs data digit i <= min(t, S - 1) with factor digit t - i
__host__ __device__ constexpr int oz_nd(int P) {
  int nd = 0;
  for (int k = 0; k < OZ_WPP; ++k) {
    const int t = oz_weight(P, k), hi = t < OZ_S - 1 ? t : OZ_S - 1;
    nd = hi + 1 > nd ? hi + 1 : nd;
  }
  return nd;
}
__host__ __device__ constexpr int oz_slot(int P, int k) { return (P * OZ_WPP + k) % OZ_NSLOT; }
// the schedule covers every weight exactly once, and a pass loads every data digit its weights pair with
constexpr bool oz_schedule_ok() {
  int seen = 0;
  for (int P = 0; P < OZ_NPASS; ++P)
    for (int k = 0; k < OZ_WPP; ++k) {
      const int t = oz_weight(P, k);
      if (t < 0 || t >= OZ_NW || (seen >> t & 1)) return false;
      seen |= 1 << t;
      if ((t < OZ_S - 1 ? t : OZ_S - 1) + 1 > oz_nd(P) || oz_nd(P) > OZ_S) return false;
    }
  return seen == (1 << OZ_NW) - 1;
}
static_assert(oz_schedule_ok(), "pass schedule");

// the MMAs of weight T (slot sk) in one chunk: pairs (i, T - i), NKS K-steps of 32 each.  xd[i]: descriptor of
// data digit i's plane chunk, fdv[j]: descriptor of factor digit j's plane chunk.
// first: the weight's first MMA overwrites its slot.  One elected lane issues (operands computed by the
// converged warp).
template <int T>
__device__ __forceinline__ void oz_weight_mmas(uint32_t td, const uint64_t (&xd)[OZ_S], const uint64_t (&fdv)[OZ_S],
                                               bool first, int nks) {
  constexpr int ilo = T > OZ_S - 1 ? T - (OZ_S - 1) : 0, ihi = T < OZ_S - 1 ? T : OZ_S - 1;
  if (elect_one()) {
    if (nks == 2) {
#pragma unroll
      for (int i = ilo; i <= ihi; ++i)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          mma_i8_pair(td, xd[i] + 2 * kk, fdv[T - i] + 2 * kk,
                      oz_idesc(i == 0, T - i == 0), (first && i == ilo && kk == 0) ? 0u : 1u);
    } else {
#pragma unroll
      for (int i = ilo; i <= ihi; ++i)
        mma_i8_pair(td, xd[i], fdv[T - i], oz_idesc(i == 0, T - i == 0),
                    (first && i == ilo) ? 0u : 1u);
    }
  }
  __syncwarp();
}

// One CTA pair (cluster of 2, the SMs of a TPC) per pair tile: 256 data rows (128 per CTA = the TMEM lanes of
// each CTA) x 128 factor rows (64 per CTA), four accumulator slots of 128 columns in each CTA's TMEM.  The
// leader (rank 0) issues every MMA (M = 256, N = 128, K = 32); both CTAs keep their half of the factor digits
// resident (<= 256 k) and stream their own data rows through a ring of 14 plane slots (64 k each) by TMA,
// completion counted on the leader's barriers, and drain their own accumulators.
// SF (streamed factor, contractions 256 < K <= 512 in one launch): no resident factor; ring slot i of a chunk
// holds data digit i's plane chunk and, behind it, factor digit i's (the passes need the same digits of both).
// One launch then runs one epilogue per tile over the whole contraction instead of two launches of half the
// contraction each, the second re-reading and accumulating into y.
template <bool SF>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(96)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap fmap,
                   const __grid_constant__ OzKernelArgs a) {
  constexpr int NXS = SF ? OZ_NXS_SF : OZ_NXS;              // ring slots
  constexpr int SLOT = SF ? OZ_XPL + OZ_FPL : OZ_XPL;       // bytes per ring slot
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t oz_smem_raw[];
  // (offset arithmetic on the shared array, not an integer round trip: derived pointers stay in the shared
  // address space for the compiler -- LDS / STS instead of generic accesses)
  uint8_t* smem = oz_smem_raw + ((1024u - (smem_u32(oz_smem_raw) & 1023u)) & 1023u);
  const int KC = a.KC;
  uint8_t* sF = smem;                                    // [KC][S] resident factor planes, this CTA's 64 rows
  uint8_t* sX = smem + (SF ? 0 : OZ_KCMAX * OZ_S * OZ_FPL);  // ring [NXS] of plane slots
  // One full / empty barrier pair per k chunk in flight (chunk number mod NCB): a chunk's nd planes occupy
  // consecutive ring slots, land on one transaction barrier and are released by one commit per MMA warp (a
  // barrier pair per plane cost each MMA warp nd commits per chunk, ~90 cycles each, as long as the MMAs of a
  // short chunk)
  uint64_t* full = reinterpret_cast<uint64_t*>(sX + NXS * SLOT);       // [NCB] (leader: both CTAs' bytes)
  uint64_t* empty = full + OZ_NCB;                                     // [NCB] (each CTA, multicast commit)
  uint64_t* fbar = empty + OZ_NCB;    // [KCMAX] factor chunk landed (leader)
  uint64_t* sfull = fbar + OZ_KCMAX;  // [4] accumulator slot complete (MMA -> epilogues of both CTAs)
  uint64_t* sempty = sfull + OZ_NSLOT;  // [4] accumulator slot drained by both CTAs (leader)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + OZ_NSLOT);
  double* sSF = reinterpret_cast<double*>(sempty + OZ_NSLOT + 2);  // 2^(e_f - WSHIFT) of the pair's factor rows
  double* sFix = reinterpret_cast<double*>(sX);  // fixup scratch after the last tile: [OZ_MAXKP] + [OZ_EW][OZ_BN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  OZ_TR(warp == 0, 0, clock64());
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_NCB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // both MMA warps commit
    }
    for (int s = 0; s < OZ_KCMAX; ++s) mbar_init(&fbar[s], 1);
    for (int t = 0; t < OZ_NSLOT; ++t) {
      mbar_init(&sfull[t], 1);
      mbar_init(&sempty[t], 2 * OZ_EW);
    }
    fence_barrier_init();
  }
  if (warp == OZ_EW + 1) {  // the same warp in both CTAs allocates the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // set-up done (barriers, TMEM): now wait for the preceding kernel (the split that wrote the data digits;
  // transitively everything before it) before reading anything it wrote
  pdl_wait();
  const bool skip = a.skip && *a.skip;  // (both CTAs of a pair read the same flag)
  OZ_TR(warp == 0, 1, clock64());

  // tile sequence of this pair: column tile nt0 fixed, row tiles strided
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int per_nt = npairs / a.nt;
  const int nt0 = pair % a.nt;
  const int mt_first = pair / a.nt;
  const int n0 = nt0 * OZ_BN;

  if (skip) {
    // (solver graphs: the step is switched off; fall through to the TMEM release)
  } else if (warp == OZ_EW) {
    if (lane == 0) {
      // resident factor digit planes: this CTA's 64 of the pair's 128 rows, [kc][digit] chunks, each chunk on
      // its own barrier and issued just before the first data chunk that needs it (the first MMAs start after
      // one chunk, not after the whole factor)
      const uint32_t fbar_l = mapa(fbar, 0);
      uint32_t n = 0, pos = 0;           // chunk number, ring slot of its first plane
      uint32_t tn = 0, occ = 0;          // oldest chunk whose slots are still held; slots held by tn .. n - 1
      int tpass = 0, tkc = 0;
      for (int mt = mt_first; mt < a.mt; mt += per_nt) {
        const int m0 = mt * OZ_PM + (int)rank * OZ_BM;
        for (int pass = 0; pass < OZ_NPASS; ++pass) {
          const uint32_t nd = oz_nd(pass);  // data digit planes of this pass
          for (int kc = 0; kc < KC; ++kc, ++n) {
            if (!SF && n < (uint32_t)KC) {
              if (leader) mbar_arrive_expect_tx(&fbar[kc], (uint32_t)(2 * OZ_S * OZ_FPL));
              for (int s = 0; s < OZ_S; ++s)
                tma_load_2sm(sF + (kc * OZ_S + s) * OZ_FPL, &fmap, a.kbase + kc * OZ_KCH,
                             (int)(s * a.f_rows_p + n0 + rank * OZ_BNH), fbar_l + 8u * (uint32_t)kc);
            }
            while (occ + nd > NXS) {  // the chunks whose slots this one overwrites must be complete
              mbar_wait(&empty[tn % OZ_NCB], (tn / OZ_NCB) & 1);
              occ -= oz_nd(tpass);
              if (++tkc == KC) {
                tkc = 0;
                if (++tpass == OZ_NPASS) tpass = 0;
              }
              ++tn;
            }
            const uint32_t fb = mapa(&full[n % OZ_NCB], 0);
            if (leader) mbar_arrive_expect_tx(&full[n % OZ_NCB], 2 * nd * SLOT);
            for (uint32_t i = 0; i < nd; ++i) {
              tma_load_2sm(sX + pos * SLOT, &xmap, a.kbase + kc * OZ_KCH, (int)(i * a.x_rows_p + m0), fb);
              if (SF)
                tma_load_2sm(sX + pos * SLOT + OZ_XPL, &fmap, a.kbase + kc * OZ_KCH,
                             (int)(i * a.f_rows_p + n0 + rank * OZ_BNH), fb);
              if (++pos == NXS) pos = 0;
            }
            occ += nd;
          }
        }
      }
    }
  } else if (warp >= OZ_EW + 1) {
    // two MMA warps (leader CTA), each issuing half of a pass's weights (four passes: warp k the pass's k-th
    // weight; two passes: slots 0, 3 and 1, 2), so one warp's barrier waits and commits overlap the other's
    // MMAs (a single issuing thread left the tensor pipe idle between short weight groups)
    const int mw = warp - (OZ_EW + 1);
    if (leader) {  // each warp runs its issue loop converged (uniform operands); one elected lane issues
      const uint32_t sx0 = smem_u32(sX);
      const uint64_t fd0 = sdesc_sw64(smem_u32(sF));
      uint32_t n = 0, pos = 0, q = 0;  // chunk number, ring slot of its first plane, phase
      for (int mt = mt_first; mt < a.mt; mt += per_nt) {
        for (int pass = 0; pass < OZ_NPASS; ++pass, ++q) {
          const int nd = oz_nd(pass);
          const uint32_t use = q / OZ_NGRP;  // how often this pass's slots were used before
          OZ_TR(true, 16 + mw * 512 + q * 8 + 0, clock64());
          for (int kc = 0; kc < KC; ++kc, ++n) {
            OZ_TR(kc <= 1, 16 + mw * 512 + q * 8 + 1 + 2 * kc, clock64());
            const bool first = kc == 0, last = kc == KC - 1;
            const int nks = last ? a.ks_last : OZ_KCH / 32;  // K-steps of 32 carrying real contraction indices
            if (!SF && n < (uint32_t)KC) mbar_wait(&fbar[kc], 0);  // (first pass of the first tile: the factor chunk)
            mbar_wait(&full[n % OZ_NCB], (n / OZ_NCB) & 1);
            // this chunk's data planes: slots pos, pos + 1, .. (mod NXS)
            uint64_t xd[OZ_S], fdv[OZ_S];
#pragma unroll
            for (int i = 0; i < OZ_S; ++i) {
              if (i < nd) {
                xd[i] = sdesc_sw64(sx0 + pos * SLOT);
                fdv[i] = SF ? sdesc_sw64(sx0 + pos * SLOT + OZ_XPL)
                            : fd0 + (uint64_t)((kc * OZ_S + i) * (OZ_FPL >> 4));
                if (++pos == NXS) pos = 0;
              } else {
                xd[i] = 0;
                fdv[i] = 0;
              }
            }
            tc_fence_after();
            OZ_TR(kc <= 1, 16 + mw * 512 + q * 8 + 2 + 2 * kc, clock64());
#define OZ_WEIGHT(P, K)                                                                                \
  if (mw == (OZ_NPASS == 4 ? K : ((K == 0 || K == 3) ? 0 : 1))) {                                      \
    if (first && use > 0) { /* the slot's previous accumulator must be drained */                    \
      mbar_wait(&sempty[oz_slot(P, K)], (use - 1) & 1);                                                \
      tc_fence_after();                                                                                \
    }                                                                                                  \
    oz_weight_mmas<oz_weight(P, K)>(tbase + (uint32_t)(oz_slot(P, K) * OZ_BN), xd, fdv, first, nks);   \
    if (last) tc_commit_pair(&sfull[oz_slot(P, K)]); /* weight complete */                             \
  }
            static_assert(OZ_S == 7 && OZ_NW == 8, "weight sequences written for 7 digits, 8 weights");
#if FDIGA_OZ_NPASS == 4
            switch (pass) {
              case 0: OZ_WEIGHT(0, 0) OZ_WEIGHT(0, 1) break;
              case 1: OZ_WEIGHT(1, 0) OZ_WEIGHT(1, 1) break;
              case 2: OZ_WEIGHT(2, 0) OZ_WEIGHT(2, 1) break;
              default: OZ_WEIGHT(3, 0) OZ_WEIGHT(3, 1) break;
            }
#else
            if (pass == 0) {
              OZ_WEIGHT(0, 0) OZ_WEIGHT(0, 1) OZ_WEIGHT(0, 3) OZ_WEIGHT(0, 2)
            } else {
              OZ_WEIGHT(1, 0) OZ_WEIGHT(1, 1) OZ_WEIGHT(1, 3) OZ_WEIGHT(1, 2)
            }
#endif
#undef OZ_WEIGHT
            OZ_TR(kc == 0, 16 + mw * 512 + q * 8 + 5, clock64());
            OZ_TR(last, 16 + mw * 512 + q * 8 + 6, clock64());
            // free the chunk's plane slots in both CTAs when its MMAs are done
            tc_commit_pair(&empty[n % OZ_NCB]);
          }
        }
      }
    }
  } else {
    // epilogue (both CTAs): warp w owns TMEM lanes 32 (w % 4).. = this CTA's data rows, columns
    // [32 (w / 4), +32) of every slot
    if (threadIdx.x < OZ_BN) {
      const int64_t f = n0 + threadIdx.x;
      sSF[threadIdx.x] = pow2(code_exp(f < a.Nf ? a.ef[f] : 0) - OZ_WSHIFT);
    }
    oz_bar_epi();
    uint32_t q = 0;
    const int quarter = warp & 3, c0 = (warp >> 2) * OZ_EC;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int mt = mt_first; mt < a.mt; mt += per_nt) {
      const int64_t m = (int64_t)mt * OZ_PM + rank * OZ_BM + quarter * 32 + lane;
      const bool mv = m < a.M;
      const int64_t mm = mv ? m : 0;
      const int64_t row_off = oz_out_off(a, mm);
      const double sx = pow2(code_exp(mv ? a.ex[mm] : 0));  // (outputs of wide rows: replaced by oz_cta_fixup)
      OZ_TR(warp == 0 && sx != 0.0, 3072 + (q / OZ_NPASS) * 4 + 2, clock64());
      // sum_t 2^{8 (NW - 1 - t)} C_t over the weights as they complete
      double acc[OZ_EC];
#pragma unroll
      for (int c = 0; c < OZ_EC; ++c) acc[c] = 0.0;
#pragma unroll 1
      for (int pass = 0; pass < OZ_NPASS; ++pass, ++q) {
#pragma unroll 1
        for (int k = 0; k < OZ_WPP; ++k) {
          const int t = oz_weight(pass, k), slot = oz_slot(pass, k);
          OZ_TR(warp == 0, 2048 + (q * OZ_WPP + k) * 4 + 0, clock64());
          mbar_wait(&sfull[slot], (q / OZ_NGRP) & 1);
          tc_fence_after();
          OZ_TR(warp == 0, 2048 + (q * OZ_WPP + k) * 4 + 1, clock64());
          const double wt = (double)(1ll << (8 * (OZ_NW - 1 - t)));
#pragma unroll
          for (int c = 0; c < OZ_EC; c += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15])
                : "r"(tbase + lane_off + (uint32_t)(slot * OZ_BN + c0 + c)));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            // int32 -> double without I2F: the bits 0x43300000:(v ^ 2^31) are 2^52 + 2^31 + v exactly, and
            // subtracting 2^52 + 2^31 is exact
#pragma unroll
            for (int r = 0; r < 16; ++r)
              acc[c + r] = fma(__hiloint2double(0x43300000, (int)(v[r] ^ 0x80000000u)) - 4503601774854144.0, wt,
                               acc[c + r]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa(&sempty[slot], 0));
          OZ_TR(warp == 0, 2048 + (q * OZ_WPP + k) * 4 + 2, clock64());
        }
      }
      OZ_TR(warp == 0, 3072 + (q / OZ_NPASS - 1) * 4, clock64());
      if (mv && !a.accum && n0 + OZ_BN <= a.Nf) {
        // full column tile (the common case): straight-line stores, one f stride per column; for every
        // column a warp stores 32 consecutive rows' values (mstride == 1 in every FD product: 256 contiguous
        // bytes).  Two exact power-of-two scalings: the factor row's (with the digit weight) and the data row's
        double* yp = a.y + row_off + (n0 + c0) * a.fstride;
        const double2* sf = reinterpret_cast<const double2*>(sSF + c0);
#pragma unroll
        for (int c = 0; c < OZ_EC; c += 2) {
          const double2 f2 = sf[c >> 1];
          yp[0] = (acc[c] * f2.x) * sx;
          yp[a.fstride] = (acc[c + 1] * f2.y) * sx;
          yp += 2 * a.fstride;
        }
      } else if (mv) {
        const bool vec = a.yvec && a.fstride == 1 && ((row_off + n0 + c0) & 1) == 0;
#pragma unroll
        for (int c = 0; c < OZ_EC; c += 2) {
          const int64_t f = n0 + c0 + c;
          // two exact power-of-two scalings: the factor row's (with the digit weight) and the data row's
          double y0 = (acc[c] * sSF[c0 + c]) * sx;
          double y1 = (acc[c + 1] * sSF[c0 + c + 1]) * sx;
          if (vec && f + 1 < a.Nf) {  // contiguous factor index (mode 1): one 16-byte store per pair
            double2* p = reinterpret_cast<double2*>(a.y + row_off + f);
            if (a.accum) {
              const double2 o = *p;
              y0 += o.x;
              y1 += o.y;
            }
            *p = make_double2(y0, y1);
          } else {
            if (f < a.Nf) {
              double* p = a.y + row_off + f * a.fstride;
              *p = a.accum ? *p + y0 : y0;
            }
            if (f + 1 < a.Nf) {
              double* p = a.y + row_off + (f + 1) * a.fstride;
              *p = a.accum ? *p + y1 : y1;
            }
          }
        }
      }
      OZ_TR(warp == 0, 3072 + (q / OZ_NPASS - 1) * 4 + 1, clock64());
    }
    OZ_TR(warp == 0, 2, clock64());
    if (a.fixup) {
      oz_bar_epi();  // (every epilogue warp past its last drain: the data ring is free for the fixup)
      oz_cta_fixup(a, mt_first, per_nt, rank, n0, sFix, sFix + OZ_MAXKP);
    }
  }
  OZ_TR(warp == 0, 3, clock64());
  tc_fence_before();
  cluster_sync();  // every MMA done and every remote arrive delivered before the pair's TMEM is released
  tc_fence_after();
  if (warp == OZ_EW + 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  OZ_TR(warp == 0, 4, clock64());
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

constexpr size_t oz_smem_bytes(bool sf) {
  return 1024 + (sf ? (size_t)OZ_NXS_SF * (OZ_XPL + OZ_FPL) : (size_t)OZ_KCMAX * OZ_S * OZ_FPL + (size_t)OZ_NXS * OZ_XPL) +
         (2 * OZ_NCB + OZ_KCMAX + 2 * OZ_NSLOT + 2) * 8 + OZ_BN * sizeof(double);
}
static_assert(oz_smem_bytes(false) <= 227 * 1024 && oz_smem_bytes(true) <= 227 * 1024, "shared memory per CTA");
static_assert(OZ_SLOT_SF == OZ_XPL + OZ_FPL, "streamed-factor ring slot");
static_assert((OZ_MAXKP + OZ_EW * OZ_BN) * sizeof(double) + OZ_EW * 32 * sizeof(int32_t) <= (size_t)OZ_NXS * OZ_XPL,
              "fixup scratch in the data ring");

// cudaFuncSetAttribute is per device: one flag bit per device ordinal
bool attr_once(std::atomic<uint64_t>& done, int device) {
  const uint64_t bit = 1ull << (device & 63);
  return !(done.fetch_or(bit) & bit);
}

}  // namespace

int oz_operand_alloc(OzOperand& op, int64_t rows, int64_t k, int box_rows) {
  const int64_t kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
  // rows padded to the pair tile (data: 256 = two 128-row boxes; factor: 64 = two 32-row halves)
  const int64_t pad = 2 * box_rows;
  const int64_t rows_p = (rows + pad - 1) / pad * pad;
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
  cuuint32_t box[2] = {(cuuint32_t)OZ_KCH, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  static_assert(sizeof(CUtensorMap) <= sizeof(op.tmap), "tensor map size");
  const CUresult r = enc(reinterpret_cast<CUtensorMap*>(op.tmap), CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, op.digits, dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
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

// FDIGA_OZ_PDL: bit 0 = the splits carry the attribute (a split may start under the preceding GEMM's tail), bit 1
// = the GEMMs carry it (a GEMM sets up -- barriers, TMEM, cluster sync -- under the preceding split's tail);
// without the attribute a kernel's griddepcontrol instructions are no-ops.  Measured at n = 256 (apply, ms):
// 0: 1.118, 1: 1.149, 2: 1.098, 3: 1.127 -- early split blocks take SMs from the GEMM's last tiles, the GEMM's
// early set-up is free.  Default 2.
int pdl_mode() {
  static const int mode = [] {
    const char* e = std::getenv("FDIGA_OZ_PDL");
    return e ? std::atoi(e) : FDIGA_OZ_PDL_DEFAULT;
  }();
  return mode;
}
// launch with the programmatic-stream-serialization attribute (see pdl_trigger / pdl_wait)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl_mode() & 1) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int oz_split(fdiga_ctx* ctx, cudaStream_t stream, const double* x, int64_t batch, int64_t K, int64_t inner,
             int64_t ldx, OzOperand& op, const int* skip, const double* lam_row, const double* lam_k) {

  const int64_t rows = batch * inner;
  FDIGA_CHECK(rows == op.rows && K <= op.kp, FDIGA_ERR_INVALID_ARG, "oz_split: operand shape mismatch");
  if (rows == 0) return FDIGA_OK;
  if (inner == 1 && !lam_row) {  // (the divide is done by the strided kernel, which handles inner == 1 too)
    const unsigned grid = (unsigned)((rows + 7) / 8);
    FDIGA_CUDA(launch_pdl(op.kp <= 256 ? oz_split_rows_kernel<1> : oz_split_rows_kernel<2>, dim3(grid), dim3(256), 0,
                          stream, x, rows, (int)K, ldx, op.digits, op.exps, op.wide, op.rows_p, (int)op.kp, skip));
  } else {
    static std::atomic<uint64_t> attr{0};
    if (attr_once(attr, ctx->device))
      FDIGA_CUDA(cudaFuncSetAttribute(oz_split_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    // 16 columns per block for every K (<= 512): 32 KB tiles at K = 256, six blocks per SM; at n = 256 this
    // beats 32 columns (three blocks per SM: 1.351 vs 1.336 ms per apply) and 8 (64-byte row segments: 1.368)
    const int64_t tiles = batch * ((inner + OZ_CW - 1) / OZ_CW);
    FDIGA_CUDA(launch_pdl(oz_split_cols_kernel, dim3((unsigned)tiles), dim3(256), (size_t)K * OZ_CW * sizeof(double),
                          stream, x, batch, (int)K, inner, op.digits, op.exps, op.wide, op.rows_p, (int)op.kp, lam_row,
                          lam_k, skip));
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
  FDIGA_CHECK(X.kp == F.kp && X.box_rows == OZ_BM && F.box_rows == OZ_BNH, FDIGA_ERR_INVALID_ARG,
              "oz_gemm: operand mismatch");
  if (X.rows == 0 || F.rows == 0) return FDIGA_OK;
  OzKernelArgs a{};
  a.M = X.rows;
  a.Nf = F.rows;
  a.x_rows_p = X.rows_p;
  a.f_rows_p = F.rows_p;
  a.mt = (int)(X.rows_p / OZ_PM);
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
  const int npairs_max = ctx->sm_count / 2;
  FDIGA_CHECK(a.nt <= npairs_max, FDIGA_ERR_NOT_SUPPORTED, "oz_gemm: too many column tiles");
  // contractions up to 256: the factor digits resident in shared memory; longer ones (<= 512): one launch of
  // the streamed-factor kernel (FDIGA_OZ_SF=0: two resident-factor launches, the second accumulating into y)
  static const int sf_mode = [] {
    const char* e = std::getenv("FDIGA_OZ_SF");
    return e ? std::atoi(e) : 1;
  }();
  const bool sf = sf_mode == 2 || (sf_mode == 1 && g.K > OZ_KCMAX * OZ_KCH);  // (2: every contraction, for A/B runs)
  static std::atomic<uint64_t> attr{0};
  if (attr_once(attr, ctx->device)) {
    FDIGA_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz_smem_bytes(false)));
    FDIGA_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz_smem_bytes(true)));
  }
  // persistent grid of CTA pairs (clusters of 2): a multiple of the column-tile count, one CTA per SM
  int64_t npairs = (int64_t)(npairs_max / a.nt) * a.nt;
  npairs = std::min<int64_t>(npairs, (int64_t)a.mt * a.nt);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * npairs));
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = oz_smem_bytes(sf);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl_mode() & 2) ? 1 : 0;
  auto kern = sf ? oz_gemm_kernel<true> : oz_gemm_kernel<false>;
  const int kmax = sf ? (int)g.K : OZ_KCMAX * OZ_KCH;  // contraction per launch
  for (int kbase = 0; kbase < g.K; kbase += kmax) {
    const int klen = (int)std::min<int64_t>(g.K - kbase, kmax);
    a.kbase = kbase;
    a.KC = (klen + OZ_KCH - 1) / OZ_KCH;
    a.ks_last = (klen - (a.KC - 1) * OZ_KCH + 31) / 32;  // K-steps of the last chunk below the contraction length
    a.accum = kbase > 0;
    a.fixup = kbase + klen >= g.K;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(X.tmap),
                                             *reinterpret_cast<const CUtensorMap*>(F.tmap), a);
    if (e != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      FDIGA_CHECK(false, FDIGA_ERR_CUDA, "oz_gemm launch: %s (grid %u, block %u, smem %zu; kernel: %d regs, max %d threads, "
                  "static smem %zu, max dyn smem %d)", cudaGetErrorString(e), cfg.gridDim.x, cfg.blockDim.x,
                  cfg.dynamicSmemBytes, fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
                  fa.maxDynamicSharedSizeBytes);
    }
    if (kbase > 0) count_launch(ctx);
  }
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

}  // namespace fdiga

#ifdef FDIGA_OZ_TRACE
extern "C" int fdiga_oz_trace_read(long long* dst, int n) {
  return (int)cudaMemcpyFromSymbol(dst, fdiga::oz_trace_buf, sizeof(long long) * (size_t)n);
}
#endif
