// FD mode products on the 5th-generation tensor cores: FP64 contractions by exact int8 splitting
// ("Ozaki scheme") on tcgen05.mma.kind::i8 with TMEM accumulators (oz.cu).
//
// Every operand row (a row of the factor W_l / U_l, or a fibre of the data tensor along the contracted
// axis) gets an exponent e with max |x| < 2^e and is written through q = floor(x 2^(62 - e)) in [-2^62, 2^62)
// as x ~ 2^(e - 62) (a_0 2^55 + sum_{i=1..6} a_i 2^(55 - 8i)), a_0 = q >> 55 a signed byte, a_1..a_6 the
// unsigned bytes of q below it (exact to 2^(-55) of the row scale).  A contraction sum_k f_k x_k is then
//   2^(e_f + e_x - 124) sum_t 2^(110 - 8t) C_t,   C_t = sum_{i+j=t} sum_k f_{k,j} x_{k,i}   (int32, exact)
// for the 8 weights t = 0..7 (34 digit pairs; i + j > 7 dropped), and only the final FP64 combination of the
// integer accumulators rounds.  The dropped pairs are below 2^(-53) of the row scales per dot product of
// length 256: FP64-level accuracy.
#pragma once
#include "common.cuh"

namespace fdiga {

constexpr int OZ_S = 7;      // digit planes per operand (digit 0 signed, 1..6 unsigned)
constexpr int OZ_NW = 8;     // digit-pair weights t = i + j = 0..7 (= int32 accumulators in TMEM)
constexpr int OZ_WSHIFT = 14 + 8 * (OZ_NW - 1);  // 2^(e_x + e_f - WSHIFT) scales sum_t 2^(8 (NW - 1 - t)) C_t
constexpr int OZ_BM = 128;   // data rows per CTA (TMEM lanes); a CTA pair (cta_group::2) covers OZ_PM
constexpr int OZ_PM = 256;   // data rows per pair tile (MMA M)
constexpr int OZ_BN = 128;   // factor rows per pair tile (MMA N = TMEM columns per accumulator)
constexpr int OZ_BNH = 64;   // factor rows per CTA (each CTA of the pair holds half of B)
constexpr int OZ_BK = 128;   // the contraction length of an operand is padded to a multiple of this (zero digits);
                             // the TMA boxes are 64 k wide (SWIZZLE_64B rows, oz.cu: OZ_KCH)
constexpr int OZ_MAXKP = 512;  // contraction lengths up to 512 (factor digits resident up to 256, streamed beside the
                               // data digits above: one launch either way)
// Guard ("accuracy contract"): a row (data fibre or factor row) is "wide" when it holds a
// non-finite value, a nonzero |x| < 2^(e - OZ_SPREAD) (its digits would keep fewer than 55 - OZ_SPREAD = 31
// significant bits of that value), or its exponent is below OZ_EMIN (the digit scaling 2^(55 - e) would leave
// the double range).  The split marks it by adding OZ_WIDE to the stored exponent and appends the row to the
// operand's wide list; after its last tile, every GEMM CTA recomputes its outputs of wide data rows and wide
// factor rows as IEEE FP64 dot products of the FP64 operands (over the int8 results).
#ifndef FDIGA_OZ_SPREAD
#define FDIGA_OZ_SPREAD 24
#endif
constexpr int OZ_SPREAD = FDIGA_OZ_SPREAD;
constexpr int OZ_EMIN = -900;
constexpr int OZ_WIDE = 1 << 20;

// digit pairs (i, j), i, j < S, i + j < NW: the MMAs per k step of a tile
constexpr int oz_pairs() {
  int n = 0;
  for (int i = 0; i < OZ_S; ++i)
    for (int j = 0; j < OZ_S; ++j) n += (i + j < OZ_NW) ? 1 : 0;
  return n;
}

// Split operand: S digit planes [S][rows_p][kp] (int8, k contiguous, zero padded) and the row
// exponents e[rows_p] (+ OZ_WIDE for a wide row); the tensor map views the planes as a 2D [S rows_p] x [kp]
// int8 matrix.  wide: [0] count, [1] ticket (the GEMM's last-CTA reset), [2 ..] the wide rows (at most
// rows_p), appended by the split in no particular order.
struct OzOperand {
  int8_t* digits = nullptr;
  int32_t* exps = nullptr;
  int32_t* wide = nullptr;
  double* ft = nullptr;  // factor operands: the FP64 factor transposed, [k][row] (oz_fixup's coalesced reads)
  int64_t rows = 0, rows_p = 0, kp = 0;
  int box_rows = 0;
  alignas(64) unsigned char tmap[128];  // CUtensorMap
  void release();
};

// Allocate (or grow) an operand for `rows` rows of k values; box_rows = OZ_BM (data) or OZ_BNH (factor); rows
// are padded to 2 box_rows (the pair tile).
int oz_operand_alloc(OzOperand& op, int64_t rows, int64_t k, int box_rows);
// Factor operands: keep F^T ([k][row], n x n) for the fixup; F row-major n x n on the host.
int oz_operand_set_ft(OzOperand& op, const double* F_host, int64_t n);
// Split x (element (b, k, i) at x[b K inner + k inner + i]; for inner == 1 row b at x[b ldx]) into op,
// row m = b inner + i, on `stream`.
// lam_row / lam_k (may be NULL): divide element (b, k, i) by lam_row[b inner + i] + lam_k[k]
// first (the FD eigenvalue-sum scaling, applied as the data enters the backward mode-d product).
int oz_split(fdiga_ctx* ctx, cudaStream_t stream, const double* x, int64_t batch, int64_t K, int64_t inner,
             int64_t ldx, OzOperand& op, const int* skip, const double* lam_row = nullptr,
             const double* lam_k = nullptr);

// y[off(m, f)] = sum_k F[f][k] X[m][k] for data rows m < M and factor rows f < Nf,
// off(m, f) = (m / inner) bstride + (m % inner) mstride + f fstride.
// The FP64 operands the digits were split from (for the wide-row fallback): X[m][k] =
// xs[(m / inner) xs_b + (m % inner) xs_i + k xs_k] (divided by lam_row[m] + lam_k[k] when lam_row is set, as the
// split did), F[f][k] = fs[f ldf + k].
struct OzGemmArgs {
  const OzOperand* X;  // data (M rows)
  const OzOperand* F;  // factor (Nf rows)
  int64_t K;           // contraction length (<= kp; the digits past it are zero)
  double* y;
  int64_t inner, bstride, mstride, fstride;
  const double* xs;
  int64_t xs_b, xs_i, xs_k;
  const double* lam_row;
  const double* lam_k;
  const double* fs;
  int64_t ldf;
  const int* skip;
};
// oz_gemm: the int8 GEMM, including the outputs of wide data rows (X's list, reset afterwards for the next
// split) and of wide factor rows (F's list, kept: the factor is split once at setup).
int oz_gemm(fdiga_ctx* ctx, cudaStream_t stream, const OzGemmArgs& a);

}  // namespace fdiga
