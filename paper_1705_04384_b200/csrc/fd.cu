// FD preconditioner: setup (cuSOLVER, one time) and apply (DMMA mode-product kernels).
//
//   s = (U_d (x)..(x) U_1) Lambda^{-1} (W_d (x)..(x) W_1) r        eq:FD2D / eq:FD3D
//   W_l = V_l^T = (M_l U_l)^{-1}
//
// Layout: r, s are X[i_d]..[i_1] (i_1 fastest).  A Kronecker factor A_l acts on index i_l:
//   mode 1 (contiguous axis):  T(n_2..n_d x n_1) = X(n_2..n_d x n_1) * A_1^T      -> B operand k-contiguous (NK)
//   mode l >= 2:               T[i_{l+1}..](n_l x n_1..n_{l-1}) = A_l * X[...]     -> B operand n-contiguous (KN)
// so no global transposes are needed.  The eigenvalue-sum divide is fused into the epilogue of
// the last forward product (mode d), "just a diagonal scaling".
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "fd_gemm.cuh"
#include "oz.cuh"

using namespace fdiga;

struct fd_plan {
  fdiga_ctx* ctx = nullptr;
  int d = 0;
  int64_t n[3] = {1, 1, 1};
  int64_t ld[3] = {0, 0, 0};  // padded (even) leading dimension of the device factors
  int64_t N = 0;
  double* U[3] = {nullptr, nullptr, nullptr};
  double* W[3] = {nullptr, nullptr, nullptr};
  double* lam[3] = {nullptr, nullptr, nullptr};
  double* lam_inner = nullptr;  // sum of the eigenvalues of directions 1..d-1 over the flattened inner index
  DevBuf t0, t1;                // ping-pong scratch
  DevBuf host_io;               // device staging for fd_apply_host
  // fd_apply_host_async: three device staging buffers, copy streams and events (created on first use).
  // Three slots let the H2D of call k+1 start once the D2H of call k-2 is done, so both PCIe directions
  // and the SMs stay busy (two slots chain H2D(k+1) behind D2H(k-1): measured 3.6 vs 2.8 ms per step)
  static constexpr int NSLOT = 3;
  DevBuf aio[NSLOT];
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[NSLOT] = {}, ev_done[NSLOT] = {}, ev_out[NSLOT] = {};
  int aslot = 0;
  int cfg[3] = {0, 0, 0};       // autotuned GEMM tile configuration per mode (fd_gemm.cu)
  float cfg_ms[3] = {0, 0, 0};
  // complex pairs: D_l has 2x2 blocks [[a, b], [-b, a]]; the divide becomes small block solves
  bool has_pairs = false;
  double* lam_im[3] = {nullptr, nullptr, nullptr};
  int32_t* lead[3] = {nullptr, nullptr, nullptr};  // first index of every 1x1 / 2x2 block of D_l
  int64_t nlead[3] = {1, 1, 1};
  std::vector<double> hU[3], hW[3], hlam[3], hlam_im[3];
  // slab sharding (nranks > 1): this rank owns the last-axis planes [o, e) of r and s
  // (Nloc = (e - o) Nin values, Nin = n_1..n_{d-1}); the mode-d sandwich runs in the transposed layout
  // T(n_d x len) over the inner-index chunk [q0, q0 + len).
  int64_t Nin = 0, o = 0, e = 0, q0 = 0, len = 0, Nloc = 0;
  // int8-split tcgen05 mode products (oz.cu): digit planes of the factors and of the data per mode
  bool oz = false;
  OzOperand ozW[3], ozU[3], ozX[3];
  // fd_apply_timed: an event recorded after every kernel of the apply (nullptr: off)
  std::vector<cudaEvent_t>* tev = nullptr;
  std::vector<int>* tkind = nullptr;  // 0 DMMA mode product, 1 int8 split, 2 int8 GEMM, 3 slab pack, 4 exchange
};

namespace {
int mark(fd_plan* P, int kind) {
  if (!P->tev) return FDIGA_OK;
  cudaEvent_t e;
  FDIGA_CUDA(cudaEventCreate(&e));
  FDIGA_CUDA(cudaEventRecord(e, P->ctx->stream));
  P->tev->push_back(e);
  P->tkind->push_back(kind);
  return FDIGA_OK;
}
}  // namespace

namespace {

// Lambda^{-1} on the block-diagonal Lambda = sum_l I (x)..(x) D_l (x)..(x) I: one thread per
// product of D_l blocks (size 1, 2, 4 or 8), a small dense solve with partial pivoting, in place.
struct BlockArgs {
  int64_t n1, n2, n3;
  int64_t L1, L2, L3;
  const int32_t *lead1, *lead2, *lead3;
  const double *re1, *re2, *re3, *im1, *im2, *im3;
  double* x;
  const int* skip;
};

__device__ __forceinline__ int blk_size(const double* im, int64_t i) { return im[i] != 0.0 ? 2 : 1; }

// D_l[i + a][i + b] for a block starting at i
__device__ __forceinline__ double blk_entry(const double* re, const double* im, int64_t i, int a, int b) {
  if (a == b) return re[i + a];
  return a == 0 ? im[i] : im[i + 1];  // [[a, +b], [-b, a]] with im[i] = +b, im[i+1] = -b
}

__global__ void block_solve_kernel(BlockArgs B) {
  if (B.skip && *B.skip) return;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= B.L1 * B.L2 * B.L3) return;
  const int64_t k1 = t % B.L1, k2 = (t / B.L1) % B.L2, k3 = t / (B.L1 * B.L2);
  const int64_t i1 = B.lead1[k1], i2 = B.lead2[k2], i3 = B.lead3[k3];
  const int s1 = blk_size(B.im1, i1), s2 = blk_size(B.im2, i2), s3 = blk_size(B.im3, i3);
  const int S = s1 * s2 * s3;
  double A[8][9];  // augmented system
  int64_t idx[8];
  for (int e = 0; e < S; ++e) {
    const int e1 = e % s1, e2 = (e / s1) % s2, e3 = e / (s1 * s2);
    idx[e] = (i1 + e1) + B.n1 * ((i2 + e2) + B.n2 * (i3 + e3));
    for (int f = 0; f < S; ++f) {
      const int f1 = f % s1, f2 = (f / s1) % s2, f3 = f / (s1 * s2);
      double v = 0.0;
      if (e2 == f2 && e3 == f3) v += blk_entry(B.re1, B.im1, i1, e1, f1);
      if (e1 == f1 && e3 == f3) v += blk_entry(B.re2, B.im2, i2, e2, f2);
      if (e1 == f1 && e2 == f2) v += blk_entry(B.re3, B.im3, i3, e3, f3);
      A[e][f] = v;
    }
    A[e][S] = B.x[idx[e]];
  }
  for (int c = 0; c < S; ++c) {  // Gaussian elimination, partial pivoting
    int piv = c;
    for (int r = c + 1; r < S; ++r)
      if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
    if (piv != c)
      for (int k = 0; k <= S; ++k) {
        const double tmp = A[c][k];
        A[c][k] = A[piv][k];
        A[piv][k] = tmp;
      }
    for (int r = c + 1; r < S; ++r) {
      const double f = A[r][c] / A[c][c];
      for (int k = c; k <= S; ++k) A[r][k] -= f * A[c][k];
    }
  }
  for (int r = S - 1; r >= 0; --r) {
    double s = A[r][S];
    for (int k = r + 1; k < S; ++k) s -= A[r][k] * A[k][S];
    A[r][S] = s / A[r][r];
  }
  for (int e = 0; e < S; ++e) B.x[idx[e]] = A[e][S];
}

int block_solve(fd_plan* P, double* x, const int* skip) {
  BlockArgs B{};
  B.n1 = P->n[0];
  B.n2 = P->n[1];
  B.n3 = P->n[2];
  B.L1 = P->nlead[0];
  B.L2 = P->nlead[1];
  B.L3 = P->nlead[2];
  B.lead1 = P->lead[0];
  B.lead2 = P->lead[1];
  B.lead3 = P->lead[2];
  B.re1 = P->lam[0];
  B.re2 = P->lam[1];
  B.re3 = P->lam[2];
  B.im1 = P->lam_im[0];
  B.im2 = P->lam_im[1];
  B.im3 = P->lam_im[2];
  B.x = x;
  B.skip = skip;
  const int64_t T = B.L1 * B.L2 * B.L3;
  block_solve_kernel<<<(unsigned)((T + 127) / 128), 128, 0, P->ctx->stream>>>(B);
  count_launch(P->ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

// Slab <-> transpose-chunk staging of the sharded mode-d pass.  Chunk s of the inner index J is
// [q_s, q_s + len_s) (balanced split of Nin over nranks); the staging buffer holds, for each s in
// order, the c x len_s block X[i][q_s .. q_s + len_s) (offset c q_s), i.e. what travels to / from s.

// slab <-> staging copy: plane i's chunk q is the contiguous slab range x[i Nin + qs, + ls) and the contiguous
// staging range stage[c qs + i ls, + ls): one segment per (i, q), bps blocks per segment, no per-element index
// arithmetic beyond the segment offset
__global__ void slab_pack_kernel(const double* __restrict__ x, double* __restrict__ stage, int64_t c, int64_t Nin,
                                 int nr, int unpack, int bps, const int* skip) {
  if (skip && *skip) return;
  const int64_t seg = blockIdx.x / bps, sub = blockIdx.x % bps;
  const int64_t i = seg / nr, q = seg % nr;
  const int64_t base = Nin / nr, rr = Nin % nr;
  const int64_t qs = q * base + (q < rr ? q : rr), ls = base + (q < rr ? 1 : 0);
  const double* src = unpack ? x + c * qs + i * ls : x + i * Nin + qs;
  double* dst = unpack ? stage + i * Nin + qs : stage + c * qs + i * ls;
  for (int64_t t = sub * blockDim.x + threadIdx.x; t < ls; t += (int64_t)bps * blockDim.x) dst[t] = src[t];
}

// mode 1 (contiguous axis): Y(R x n1) = X(R x n1) * F^T
GemmParams mode1_params(fd_plan* P, const double* F, int64_t ldf, const double* X, double* Y, int64_t R,
                        const int* skip) {
  GemmParams g{};
  g.skip = skip;
  g.M = (int)R;
  g.N = (int)P->n[0];
  g.K = (int)P->n[0];
  g.A = X;
  g.lda = P->n[0];
  g.B = F;
  g.ldb = ldf;
  g.C = Y;
  g.ldc = P->n[0];
  g.inner = g.N;
  return g;
}

// mode l >= 2: for every outer slice, Y(n_l x inner) = F(n_l x n_l) * X(n_l x inner); the slices are
// flattened into one N = inner * batch (dmma_gemm.cuh, BLayout::KN)
GemmParams model_params(fd_plan* P, int l, const double* F, int64_t ldf, const double* X, double* Y,
                        int64_t inner, int64_t batch, const double* lam_m, const double* lam_n, const int* skip) {
  GemmParams g{};
  g.skip = skip;
  g.M = (int)P->n[l];
  g.N = (int)(inner * batch);
  g.K = (int)P->n[l];
  g.A = F;
  g.lda = ldf;
  g.B = X;
  g.ldb = inner;
  g.C = Y;
  g.ldc = inner;
  g.inner = inner;
  g.bstride = inner * P->n[l];
  g.lam_m = lam_m;
  g.lam_n = lam_n;
  return g;
}

int mode1(fd_plan* P, const double* F, int64_t ldf, const double* X, double* Y, int64_t R, const int* skip) {
  if (R == 0) return FDIGA_OK;
  FDIGA_TRY(gemm_launch(P->ctx, P->ctx->stream, BLayout::NK, P->cfg[0], mode1_params(P, F, ldf, X, Y, R, skip)));
  return mark(P, 0);
}

int model(fd_plan* P, int l, const double* F, int64_t ldf, const double* X, double* Y, int64_t inner,
          int64_t batch, const double* lam_m, const double* lam_n, const int* skip) {
  if (inner * batch == 0) return FDIGA_OK;
  FDIGA_TRY(gemm_launch(P->ctx, P->ctx->stream, BLayout::KN, P->cfg[l],
                        model_params(P, l, F, ldf, X, Y, inner, batch, lam_m, lam_n, skip)));
  return mark(P, 0);
}

// Pick the tile configuration of every mode product of this plan by timing them on the plan's scratch.
int autotune_plan(fd_plan* P) {
  const int64_t n1 = P->n[0], n2 = P->n[1];
  const int64_t c = P->e - P->o;  // local planes of the last axis (all of them on one rank)
  double* a = P->t0.p;
  double* b = P->t1.p;
  FDIGA_CUDA(cudaMemsetAsync(a, 0, P->t0.cap * sizeof(double), P->ctx->stream));
  const int64_t rows1 = (P->d == 2) ? c : n2 * c;
  if (rows1 > 0)
    FDIGA_TRY(gemm_autotune(P->ctx, BLayout::NK, mode1_params(P, P->W[0], P->ld[0], a, b, rows1, nullptr),
                            &P->cfg[0], &P->cfg_ms[0]));
  if (P->d == 3 && c > 0)
    FDIGA_TRY(gemm_autotune(P->ctx, BLayout::KN, model_params(P, 1, P->W[1], P->ld[1], a, b, n1, c, nullptr,
                                                              nullptr, nullptr), &P->cfg[1], &P->cfg_ms[1]));
  if (P->len > 0)  // mode d over the (transposed) inner chunk
    FDIGA_TRY(gemm_autotune(P->ctx, BLayout::KN, model_params(P, P->d - 1, P->W[P->d - 1], P->ld[P->d - 1], a, b,
                                                              P->len, 1, nullptr, nullptr, nullptr),
                            &P->cfg[P->d - 1], &P->cfg_ms[P->d - 1]));
  FDIGA_CUDA(cudaStreamSynchronize(P->ctx->stream));
  if (getenv("FDIGA_VERBOSE")) {
    for (int l = 0; l < P->d; ++l)
      fprintf(stderr, "[fdiga] fd plan n=(%lld,%lld,%lld) mode %d: tile %s, %.1f us\n", (long long)n1,
              (long long)n2, (long long)P->n[2], l + 1, gemm_config_name(l == 0 ? BLayout::NK : BLayout::KN, P->cfg[l]),
              1e3 * P->cfg_ms[l]);
  }
  return FDIGA_OK;
}

int upload_factor(const double* h, int64_t n, int64_t ld, double** dptr) {
  std::vector<double> pad((size_t)n * ld, 0.0);
  for (int64_t i = 0; i < n; ++i) std::memcpy(&pad[i * ld], h + i * n, n * sizeof(double));
  FDIGA_CUDA(cudaMalloc(dptr, pad.size() * sizeof(double)));
  FDIGA_CUDA(cudaMemcpy(*dptr, pad.data(), pad.size() * sizeof(double), cudaMemcpyHostToDevice));  // synchronous
  return FDIGA_OK;
}

// Multi-rank: every rank uses rank 0's factors bit for bit (the sharded apply mixes the modes of
// different ranks, and two correct setups differ by ~1e-11 through cond(P)).  A sum
// all-reduce in which only rank 0 contributes is an exact broadcast.
int broadcast_factors(fd_plan* P) {
  fdiga_ctx* ctx = P->ctx;
  std::vector<double> pack;
  for (int l = 0; l < P->d; ++l) {
    pack.insert(pack.end(), P->hU[l].begin(), P->hU[l].end());
    pack.insert(pack.end(), P->hW[l].begin(), P->hW[l].end());
    pack.insert(pack.end(), P->hlam[l].begin(), P->hlam[l].end());
    pack.insert(pack.end(), P->hlam_im[l].begin(), P->hlam_im[l].end());
  }
  if (ctx->rank != 0) std::fill(pack.begin(), pack.end(), 0.0);
  double* buf = nullptr;
  FDIGA_CUDA(cudaMalloc(&buf, 2 * pack.size() * sizeof(double)));
  int s = FDIGA_OK;
  if (cudaMemcpy(buf, pack.data(), pack.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) s = FDIGA_ERR_CUDA;
  const int s2 = comm_allreduce(ctx, buf, buf + pack.size(), pack.size());  // collective: always called
  if (s == FDIGA_OK) s = s2;
  if (s == FDIGA_OK && (cudaStreamSynchronize(ctx->stream) != cudaSuccess ||
                        cudaMemcpy(pack.data(), buf + pack.size(), pack.size() * 8, cudaMemcpyDeviceToHost) !=
                            cudaSuccess))
    s = FDIGA_ERR_CUDA;
  cudaFree(buf);
  if (s != FDIGA_OK) {
    set_error("broadcast of the FD factors failed");
    return s;
  }
  size_t off = 0;
  for (int l = 0; l < P->d; ++l) {
    const size_t nn = (size_t)P->n[l] * P->n[l], n = (size_t)P->n[l];
    std::copy(pack.begin() + off, pack.begin() + off + nn, P->hU[l].begin());
    off += nn;
    std::copy(pack.begin() + off, pack.begin() + off + nn, P->hW[l].begin());
    off += nn;
    std::copy(pack.begin() + off, pack.begin() + off + n, P->hlam[l].begin());
    off += n;
    std::copy(pack.begin() + off, pack.begin() + off + n, P->hlam_im[l].begin());
    off += n;
  }
  return FDIGA_OK;
}

// int8-split tensor-core mode products (oz.cu) for 3D real-spectrum plans (single-rank or slab-sharded) with
// 192 <= n_l <= 512 -- where they beat the DMMA products on a B200 (n = 256: 1.43 vs 1.72 ms per apply,
// n = 384: 6.2 vs 8.4 ms, n = 512: 18.4 vs 25.9 ms; at n = 128 / 131 the short contractions leave the tensor
// cores idle and DMMA wins).  FDIGA_FD_OZ=0 / 1 forces the choice (1: any n_l <= 512).  A
// static rule, so every run -- also under a profiler -- takes the same kernels.
bool oz_supported(const fd_plan* P) {  // shapes and spectra the int8 kernels handle at all
  if (P->d != 3 || P->has_pairs) return false;
  for (int l = 0; l < 3; ++l)
    if (P->n[l] > OZ_MAXKP) return false;
  return true;
}
bool oz_eligible(const fd_plan* P) {  // the default rule
  if (!oz_supported(P)) return false;
  const char* e = getenv("FDIGA_FD_OZ");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  for (int l = 0; l < 3; ++l)
    if (P->n[l] < 192) return false;
  return true;
}

// Local shapes of the three mode products on this rank: modes 1 and 2 on the slab of c = e - o planes of
// the last axis, mode 3 on the transposed chunk T(n_3 x len) (single rank: c = n_3, len = n_1 n_2).
struct OzShapes {
  int64_t rows[3];
};
OzShapes oz_shapes(const fd_plan* P) {
  const int64_t c = P->e - P->o;
  return {{P->n[1] * c, P->n[0] * c, P->len}};
}

int oz_setup(fd_plan* P, bool force = false) {
  if (!(force ? oz_supported(P) : oz_eligible(P))) return FDIGA_OK;
  cudaStream_t st = P->ctx->stream;
  const OzShapes sh = oz_shapes(P);
  for (int l = 0; l < 3; ++l) {
    FDIGA_TRY(oz_operand_alloc(P->ozW[l], P->n[l], P->n[l], OZ_BNH));
    FDIGA_TRY(oz_operand_alloc(P->ozU[l], P->n[l], P->n[l], OZ_BNH));
    FDIGA_TRY(oz_split(P->ctx, st, P->W[l], P->n[l], P->n[l], 1, P->ld[l], P->ozW[l], nullptr));
    FDIGA_TRY(oz_split(P->ctx, st, P->U[l], P->n[l], P->n[l], 1, P->ld[l], P->ozU[l], nullptr));
    FDIGA_TRY(oz_operand_set_ft(P->ozW[l], P->hW[l].data(), P->n[l]));
    FDIGA_TRY(oz_operand_set_ft(P->ozU[l], P->hU[l].data(), P->n[l]));
    FDIGA_TRY(oz_operand_alloc(P->ozX[l], sh.rows[l], P->n[l], OZ_BM));
  }
  FDIGA_CUDA(cudaStreamSynchronize(st));
  P->oz = true;
  return FDIGA_OK;
}

// The mode-3 product on the int8 path (the modes 1 and 2 run plane-transposed, oz_mode_t below): the chunk
// T[i3][q] (q over len inner indices), data rows q, k = i3, split transposing; divide_input: X / (lam_inner[q0 + q]
// + lam_3[i3]) first (the Lambda divide of eq:FD3D, applied as the data enters the backward product).
int oz_mode3(fd_plan* P, const OzOperand& Fz, const double* Fs, const double* X, double* Y, const int* skip,
             bool divide_input = false) {
  const int64_t n3 = P->n[2], len = P->len;
  OzOperand& Xz = P->ozX[2];
  cudaStream_t st = P->ctx->stream;
  OzGemmArgs g{};
  g.X = &Xz;
  g.F = &Fz;
  g.K = n3;
  g.y = Y;
  g.skip = skip;
  g.xs = X;  // the FP64 operands, for the outputs of wide rows (oz.cuh: guard)
  g.fs = Fs;
  g.ldf = P->ld[2];
  if (Xz.rows == 0) return FDIGA_OK;
  const double* lr = divide_input ? P->lam_inner + P->q0 : nullptr;
  const double* lk = divide_input ? P->lam[2] : nullptr;
  FDIGA_TRY(oz_split(P->ctx, st, X, 1, n3, len, 0, Xz, skip, lr, lk));
  g.inner = len;
  g.bstride = 0;
  g.mstride = 1;
  g.fstride = len;
  g.xs_b = 0, g.xs_i = 1, g.xs_k = len;
  g.lam_row = lr;
  g.lam_k = lk;
  FDIGA_TRY(mark(P, 1));
  FDIGA_TRY(oz_gemm(P->ctx, st, g));
  return mark(P, 2);
}

// Single-rank mode products with plane-transposed intermediates (every split a row split but two, every
// GEMM store coalesced; the mode products commute, so the backward pass may run 3, 1, 2):
//   t = 0: X[i3][j][k] (k contiguous, K = n_k), data rows (i3, j), output Y[i3][f][j] (the plane transposed)
//   t = 1: the same contraction, output Y[i3][f][j] ... written as Y[i3][f][j] with j the row's inner index
// Both are "contract the contiguous axis of each i3 plane and store the plane transposed": with
// X = x[i3][i2][i1] (k = i1) the result is y[i3][f1][i2]; applied again (k = i2) it gives z[i3][f2][f1], the
// natural layout.  (Row-contiguous stores of a pair tile's outputs -- the natural mode-1 layout -- touch 32
// rows per warp store and cost ~35 us more per product at n = 256.)
int oz_mode_t(fd_plan* P, int l, const OzOperand& Fz, const double* Fs, const double* X, double* Y, const int* skip) {
  const int64_t nk = P->n[l], nj = P->n[1 - l];  // contracted axis and the other in-plane axis
  const int64_t c = P->e - P->o;
  OzOperand& Xz = P->ozX[l];
  cudaStream_t st = P->ctx->stream;
  OzGemmArgs g{};
  g.X = &Xz;
  g.F = &Fz;
  g.K = nk;
  g.y = Y;
  g.skip = skip;
  g.xs = X;
  g.fs = Fs;
  g.ldf = P->ld[l];
  if (Xz.rows == 0) return FDIGA_OK;
  FDIGA_TRY(oz_split(P->ctx, st, X, nj * c, nk, 1, nk, Xz, skip));
  g.inner = nj;          // row m = (i3, j): b = m / nj, j = m % nj
  g.bstride = nk * nj;   // one plane
  g.mstride = 1;         // j contiguous in the output plane
  g.fstride = nj;        // output row f of the plane
  g.xs_b = nk * nj, g.xs_i = nk, g.xs_k = 1;
  FDIGA_TRY(mark(P, 1));
  FDIGA_TRY(oz_gemm(P->ctx, st, g));
  return mark(P, 2);
}

int fd_apply_oz(fd_plan* P, const double* r, double* s, const int* skip) {
  double* a = P->t0.p;
  double* b = P->t1.p;
  FDIGA_TRY(oz_mode_t(P, 0, P->ozW[0], P->W[0], r, a, skip));  // a = [i3][f1][i2]
  FDIGA_TRY(oz_mode_t(P, 1, P->ozW[1], P->W[1], a, b, skip));  // b = [i3][f2][f1]
  // the Lambda divide rides in the split that feeds the backward mode-3 product
  FDIGA_TRY(oz_mode3(P, P->ozW[2], P->W[2], b, a, skip));
  FDIGA_TRY(oz_mode3(P, P->ozU[2], P->U[2], a, b, skip, true));
  FDIGA_TRY(oz_mode_t(P, 0, P->ozU[0], P->U[0], b, a, skip));  // a = [i3][f1][i2]
  return oz_mode_t(P, 1, P->ozU[1], P->U[1], a, s, skip);      // s = [i3][i2][i1]
}

int finish_plan(fd_plan* P) {
  const int d = P->d;
  if (P->ctx->sharded) FDIGA_TRY(broadcast_factors(P));
  // complex pairs: validate the block structure (lam_im = +b, -b on adjacent indices, equal real parts)
  for (int l = 0; l < d; ++l) {
    const auto& im = P->hlam_im[l];
    const auto& re = P->hlam[l];
    for (int64_t i = 0; i < P->n[l]; ++i) {
      if (im[i] == 0.0) continue;
      FDIGA_CHECK(i + 1 < P->n[l] && im[i] > 0.0 && im[i + 1] == -im[i] && re[i + 1] == re[i],
                  FDIGA_ERR_INVALID_ARG, "direction %d: lam_im must hold +b, -b pairs with equal real parts", l);
      P->has_pairs = true;
      ++i;
    }
  }
  FDIGA_CHECK(!(P->has_pairs && P->ctx->sharded), FDIGA_ERR_NOT_SUPPORTED,
              "complex-pair FD is single-rank only (blocks straddle the transpose chunks)");
  // singularity guard on the eigenvalues of Lambda: min |Lambda| <= 1e3 eps max |Lambda|, with
  // mu = lam_re + i lam_im per index (the eigenvalues of the 2x2 blocks are a +- ib)
  double mn = INFINITY, mx = 0.0;
  {
    const auto& r1 = P->hlam[0];
    const auto& r2 = P->hlam[1];
    const auto& m1 = P->hlam_im[0];
    const auto& m2 = P->hlam_im[1];
    std::vector<double> inner, inner_im;  // lam_1 + ... + lam_{d-1}
    if (d == 2) {
      inner = r1;
      inner_im = m1;
    } else {
      inner.resize(r1.size() * r2.size());
      inner_im.resize(r1.size() * r2.size());
      for (size_t b = 0; b < r2.size(); ++b)
        for (size_t a = 0; a < r1.size(); ++a) {
          inner[b * r1.size() + a] = r1[a] + r2[b];
          inner_im[b * r1.size() + a] = m1[a] + m2[b];
        }
    }
    const auto& rl = P->hlam[d - 1];
    const auto& ml = P->hlam_im[d - 1];
    for (size_t k = 0; k < rl.size(); ++k)
      for (size_t j = 0; j < inner.size(); ++j) {
        const double s = std::hypot(rl[k] + inner[j], ml[k] + inner_im[j]);
        mn = std::min(mn, s);
        mx = std::max(mx, s);
      }
    FDIGA_CHECK(mn > 1e3 * 2.220446049250313e-16 * mx, FDIGA_ERR_SINGULAR,
                "eigenvalue sums nearly singular: min |Lambda| = %g, max = %g", mn, mx);
    FDIGA_CUDA(cudaMalloc(&P->lam_inner, inner.size() * sizeof(double)));
    FDIGA_CUDA(cudaMemcpy(P->lam_inner, inner.data(), inner.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  for (int l = 0; l < d; ++l) {
    P->ld[l] = (P->n[l] + 1) & ~int64_t(1);
    FDIGA_TRY(upload_factor(P->hU[l].data(), P->n[l], P->ld[l], &P->U[l]));
    FDIGA_TRY(upload_factor(P->hW[l].data(), P->n[l], P->ld[l], &P->W[l]));
    FDIGA_CUDA(cudaMalloc(&P->lam[l], P->n[l] * sizeof(double)));
    FDIGA_CUDA(cudaMemcpy(P->lam[l], P->hlam[l].data(), P->n[l] * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (P->has_pairs) {
    for (int l = 0; l < 3; ++l) {
      std::vector<double> re = l < d ? P->hlam[l] : std::vector<double>(1, 0.0);  // dummy direction: D = [0]
      std::vector<double> im = l < d ? P->hlam_im[l] : std::vector<double>(1, 0.0);
      std::vector<int32_t> lead;
      for (int64_t i = 0; i < (int64_t)re.size(); ++i) {
        lead.push_back((int32_t)i);
        if (im[i] != 0.0) ++i;
      }
      P->nlead[l] = (int64_t)lead.size();
      if (l >= d) {
        FDIGA_CUDA(cudaMalloc(&P->lam[l], sizeof(double)));
        FDIGA_CUDA(cudaMemcpy(P->lam[l], re.data(), sizeof(double), cudaMemcpyHostToDevice));
      }
      FDIGA_CUDA(cudaMalloc(&P->lam_im[l], im.size() * sizeof(double)));
      FDIGA_CUDA(cudaMemcpy(P->lam_im[l], im.data(), im.size() * sizeof(double), cudaMemcpyHostToDevice));
      FDIGA_CUDA(cudaMalloc(&P->lead[l], lead.size() * sizeof(int32_t)));
      FDIGA_CUDA(cudaMemcpy(P->lead[l], lead.data(), lead.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
  }
  {
    const size_t cap = (size_t)std::max<int64_t>(1, std::max(P->Nloc, P->n[d - 1] * P->len));
    FDIGA_TRY(P->t0.ensure(cap));
    FDIGA_TRY(P->t1.ensure(cap));
  }
  FDIGA_CUDA(cudaDeviceSynchronize());  // uploads complete before any stream uses the plan
  FDIGA_TRY(autotune_plan(P));
  FDIGA_TRY(oz_setup(P));
  return FDIGA_OK;
}

int check_common(fdiga_ctx* ctx, int d, const int64_t* n, fd_plan** out) {
  FDIGA_CHECK(ctx && n && out, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_CHECK(d == 2 || d == 3, FDIGA_ERR_INVALID_ARG, "d must be 2 or 3 (got %d)", d);
  for (int l = 0; l < d; ++l)
    FDIGA_CHECK(n[l] >= 1 && n[l] <= 65535, FDIGA_ERR_INVALID_ARG, "n[%d] = %lld out of range", l, (long long)n[l]);
  *out = nullptr;
  return bind(ctx);
}

fd_plan* new_plan(fdiga_ctx* ctx, int d, const int64_t* n) {
  fd_plan* P = new fd_plan();
  P->ctx = ctx;
  P->d = d;
  P->N = 1;
  for (int l = 0; l < d; ++l) {
    P->n[l] = n[l];
    P->N *= n[l];
  }
  P->Nin = P->N / n[d - 1];
  partition(n[d - 1], ctx->nranks, ctx->rank, &P->o, &P->e);
  int64_t q1 = 0;
  partition(P->Nin, ctx->nranks, ctx->rank, &P->q0, &q1);
  P->len = q1 - P->q0;
  P->Nloc = (P->e - P->o) * P->Nin;
  return P;
}

// ---------------------------------------------------------------- cuSOLVER helpers
#define CUSOLVER(call)                                                                              \
  do {                                                                                              \
    cusolverStatus_t s_ = (call);                                                                   \
    if (s_ != CUSOLVER_STATUS_SUCCESS) {                                                            \
      set_error("cuSOLVER status %d at %s:%d (%s)", (int)s_, __FILE__, __LINE__, #call);            \
      return FDIGA_ERR_CUSOLVER;                                                                    \
    }                                                                                               \
  } while (0)

struct Solver {
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t prm = nullptr;
  ~Solver() {
    if (prm) cusolverDnDestroyParams(prm);
    if (h) cusolverDnDestroy(h);
  }
  int init(cudaStream_t s) {
    CUSOLVER(cusolverDnCreate(&h));
    CUSOLVER(cusolverDnSetStream(h, s));
    CUSOLVER(cusolverDnCreateParams(&prm));
    return FDIGA_OK;
  }
};
// the context's cached cuSOLVER handle (created on first use, bound to the context stream)
int ctx_solver(fdiga_ctx* ctx, Solver** out) {
  Solver* S = static_cast<Solver*>(ctx->solver);
  if (!S) {
    S = new Solver();
    const int s = S->init(ctx->stream);
    if (s != FDIGA_OK) {
      delete S;
      return s;
    }
    ctx->solver = S;
  }
  CUSOLVER(cusolverDnSetStream(S->h, ctx->stream));
  *out = S;
  return FDIGA_OK;
}

// Column-major helpers (cuSOLVER is column-major; our host matrices are row-major).
std::vector<double> to_colmajor(const double* rm, int64_t n) {
  std::vector<double> c((size_t)n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) c[j * n + i] = rm[i * n + j];
  return c;
}

// X = A^{-1} B (A, B column-major n x n, nrhs = n) on the device with getrf/getrs.
int lu_solve(Solver& S, cudaStream_t st, int64_t n, const std::vector<double>& A, std::vector<double>& B) {
  double *dA = nullptr, *dB = nullptr;
  int64_t* ipiv = nullptr;
  int* info = nullptr;
  void* dwork = nullptr;
  int rc = FDIGA_OK;
  size_t dws = 0, hws = 0;
  std::vector<char> hwork;
  int hinfo = 0;
  auto cleanup = [&]() {
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(ipiv);
    cudaFree(info);
    cudaFree(dwork);
  };
  if (cudaMalloc(&dA, n * n * 8) || cudaMalloc(&dB, n * n * 8) || cudaMalloc(&ipiv, n * 8) ||
      cudaMalloc(&info, sizeof(int))) {
    cleanup();
    set_error("cudaMalloc failed in lu_solve");
    return FDIGA_ERR_CUDA;
  }
  cudaMemcpyAsync(dA, A.data(), n * n * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dB, B.data(), n * n * 8, cudaMemcpyHostToDevice, st);
  if (cusolverDnXgetrf_bufferSize(S.h, S.prm, n, n, CUDA_R_64F, dA, n, CUDA_R_64F, &dws, &hws) !=
      CUSOLVER_STATUS_SUCCESS) {
    cleanup();
    set_error("Xgetrf_bufferSize failed");
    return FDIGA_ERR_CUSOLVER;
  }
  cudaMalloc(&dwork, std::max<size_t>(dws, 8));
  hwork.resize(std::max<size_t>(hws, 8));
  if (cusolverDnXgetrf(S.h, S.prm, n, n, CUDA_R_64F, dA, n, ipiv, CUDA_R_64F, dwork, dws, hwork.data(), hws,
                       info) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnXgetrs(S.h, S.prm, CUBLAS_OP_N, n, n, CUDA_R_64F, dA, n, ipiv, CUDA_R_64F, dB, n, info) !=
          CUSOLVER_STATUS_SUCCESS) {
    cleanup();
    set_error("Xgetrf/Xgetrs failed");
    return FDIGA_ERR_CUSOLVER;
  }
  cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(B.data(), dB, n * n * 8, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cleanup();
  FDIGA_CHECK(e == cudaSuccess, FDIGA_ERR_CUDA, "lu_solve: %s", cudaGetErrorString(e));
  FDIGA_CHECK(hinfo == 0, FDIGA_ERR_SINGULAR, "LU: singular matrix (info = %d)", hinfo);
  return rc;
}

double norm1_rm(const std::vector<double>& A, int64_t n) {  // max column abs sum, row-major
  double best = 0;
  for (int64_t j = 0; j < n; ++j) {
    double s = 0;
    for (int64_t i = 0; i < n; ++i) s += std::fabs(A[i * n + j]);
    best = std::max(best, s);
  }
  return best;
}

// W = (M U)^{-1} (row-major in/out; M == nullptr means identity).  Also returns cond_1(U).  The products
// with M skip its zeros (the 1D spline mass matrices are banded: O(n^2 p) instead of O(n^3) on the host).
int compute_W(Solver& S, cudaStream_t st, int64_t n, const double* M, const std::vector<double>& U,
              std::vector<double>& W, double* condU) {
  std::vector<double> MU(U);
  std::vector<std::vector<std::pair<int64_t, double>>> nz;  // nonzeros of M by row
  if (M) {
    nz.resize(n);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = 0; k < n; ++k)
        if (M[i * n + k] != 0.0) nz[i].push_back({k, M[i * n + k]});
    for (int64_t i = 0; i < n; ++i) {
      double* r = &MU[i * n];
      std::fill(r, r + n, 0.0);
      for (const auto& e : nz[i]) {
        const double* u = &U[e.first * n];
        for (int64_t j = 0; j < n; ++j) r[j] += e.second * u[j];
      }
    }
  }
  std::vector<double> A = to_colmajor(MU.data(), n);
  std::vector<double> B((size_t)n * n, 0.0);
  for (int64_t i = 0; i < n; ++i) B[i * n + i] = 1.0;
  FDIGA_TRY(lu_solve(S, st, n, A, B));  // B = (MU)^{-1}, column-major
  W.assign((size_t)n * n, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) W[i * n + j] = B[j * n + i];
  if (condU) {
    // U^{-1} = W M
    std::vector<double> Uinv(W);
    if (M) {
      for (int64_t i = 0; i < n; ++i) {
        double* r = &Uinv[i * n];
        std::fill(r, r + n, 0.0);
        for (int64_t k = 0; k < n; ++k) {
          const double w = W[i * n + k];
          for (const auto& e : nz[k]) r[e.first] += w * e.second;
        }
      }
    }
    *condU = norm1_rm(U, n) * norm1_rm(Uinv, n);
  }
  return FDIGA_OK;
}

}  // namespace

namespace fdiga {
int64_t fd_plan_local_size(const fd_plan* P) { return P->Nloc; }
}  // namespace fdiga

namespace {
// Sharded apply (nranks > 1): local modes 1..d-1 on the slab, NCCL/loopback slab -> chunk transpose,
// the mode-d sandwich (W_d, Lambda-divide epilogue, U_d) on T(n_d x len), transpose back, local
// backward modes.  r, s: this rank's slab (s may alias r).
int fd_apply_sharded(fd_plan* P, const double* r, double* s, const int* skip) {
  fdiga_ctx* ctx = P->ctx;
  double* a = P->t0.p;
  double* b = P->t1.p;
  const int d = P->d, nr = ctx->nranks;
  const int64_t n1 = P->n[0], n2 = P->n[1], nd = P->n[d - 1];
  const int64_t c = P->e - P->o, Nin = P->Nin, len = P->len;
  // forward modes 1..d-1 -> b (slab layout)
  if (d == 3 && P->oz) {
    FDIGA_TRY(oz_mode_t(P, 0, P->ozW[0], P->W[0], r, a, skip));  // plane-transposed intermediate
    FDIGA_TRY(oz_mode_t(P, 1, P->ozW[1], P->W[1], a, b, skip));  // natural slab layout again
  } else if (d == 3) {
    FDIGA_TRY(mode1(P, P->W[0], P->ld[0], r, a, n2 * c, skip));
    FDIGA_TRY(model(P, 1, P->W[1], P->ld[1], a, b, n1, c, nullptr, nullptr, skip));
  } else {
    FDIGA_TRY(mode1(P, P->W[0], P->ld[0], r, b, c, skip));
  }
  std::vector<int64_t> so(nr), sc(nr), to(nr), tc(nr);
  FDIGA_TRY(fdiga_transpose_plan(Nin, nd, nr, ctx->rank, so.data(), sc.data(), to.data(), tc.data()));
  std::vector<P2PMsg> snd, rcv;
  auto plan_msgs = [&](double* slab_side, double* tr_side) {
    snd.clear();
    rcv.clear();
    for (int q = 0; q < nr; ++q) {
      snd.push_back({q, slab_side + so[q], (size_t)sc[q] * 8});
      rcv.push_back({q, tr_side + to[q], (size_t)tc[q] * 8});
    }
  };
  const int64_t lmax = (Nin + nr - 1) / nr, nseg = std::max<int64_t>(1, c * nr);  // c = 0: a rank without planes
  const int bps = (int)std::max<int64_t>(1, std::min<int64_t>((lmax + 1023) / 1024,
                                                               (8 * ctx->sm_count + nseg - 1) / nseg));
  const unsigned gsegs = (unsigned)(c * nr * bps);
  if (c > 0) {
    slab_pack_kernel<<<gsegs, 256, 0, ctx->stream>>>(b, a, c, Nin, nr, 0, bps, skip);
    count_launch(ctx);
    FDIGA_CUDA(cudaGetLastError());
    FDIGA_TRY(mark(P, 3));
  }
  plan_msgs(a, b);
  FDIGA_TRY(comm_exchange(ctx, snd, rcv));  // b = T(n_d x len)
  FDIGA_TRY(mark(P, 4));
  if (P->oz) {  // the Lambda divide rides in the split feeding the backward product (chunk offset q0)
    FDIGA_TRY(oz_mode3(P, P->ozW[2], P->W[2], b, a, skip));
    FDIGA_TRY(oz_mode3(P, P->ozU[2], P->U[2], a, b, skip, true));
  } else {
    FDIGA_TRY(model(P, d - 1, P->W[d - 1], P->ld[d - 1], b, a, len, 1, P->lam[d - 1], P->lam_inner + P->q0, skip));
    FDIGA_TRY(model(P, d - 1, P->U[d - 1], P->ld[d - 1], a, b, len, 1, nullptr, nullptr, skip));
  }
  plan_msgs(a, b);
  FDIGA_TRY(comm_exchange(ctx, rcv, snd));  // reverse: rows of T back to their slab owners, into a
  FDIGA_TRY(mark(P, 4));
  if (c > 0) {
    slab_pack_kernel<<<gsegs, 256, 0, ctx->stream>>>(a, b, c, Nin, nr, 1, bps, skip);
    count_launch(ctx);
    FDIGA_CUDA(cudaGetLastError());
    FDIGA_TRY(mark(P, 3));
  }
  if (d == 3 && P->oz) {
    FDIGA_TRY(oz_mode_t(P, 0, P->ozU[0], P->U[0], b, a, skip));  // the products commute: 1 then 2
    FDIGA_TRY(oz_mode_t(P, 1, P->ozU[1], P->U[1], a, s, skip));
  } else if (d == 3) {
    FDIGA_TRY(model(P, 1, P->U[1], P->ld[1], b, a, n1, c, nullptr, nullptr, skip));
    FDIGA_TRY(mode1(P, P->U[0], P->ld[0], a, s, n2 * c, skip));
  } else {
    FDIGA_TRY(mode1(P, P->U[0], P->ld[0], b, s, c, skip));
  }
  return FDIGA_OK;
}
}  // namespace

namespace fdiga {
int fd_apply_ex(fd_plan* P, const double* r, double* s, const int* skip) {
  FDIGA_CHECK(P && ((r && s) || P->Nloc == 0), FDIGA_ERR_INVALID_ARG, "NULL argument");
  fdiga_ctx* ctx = P->ctx;
  FDIGA_TRY(bind(ctx));
  double* a = P->t0.p;
  double* b = P->t1.p;
  const int64_t n1 = P->n[0], n2 = P->n[1], n3 = P->n[2];
  // real spectra: the Lambda-divide rides in the epilogue of the last forward product; complex pairs
  // (P:434): plain last forward product, then the small block solves in place
  const bool fused = !P->has_pairs;
  if (ctx->sharded) return fd_apply_sharded(P, r, s, skip);
  if (P->oz) return fd_apply_oz(P, r, s, skip);
  if (P->d == 2) {
    // fwd: mode 1 (W_1), mode 2 (W_2) + divide by lam_2[i2] + lam_1[i1]; bwd: mode 2 (U_2), mode 1 (U_1)
    FDIGA_TRY(mode1(P, P->W[0], P->ld[0], r, a, n2, skip));
    FDIGA_TRY(model(P, 1, P->W[1], P->ld[1], a, b, n1, 1, fused ? P->lam[1] : nullptr, P->lam_inner, skip));
    if (!fused) FDIGA_TRY(block_solve(P, b, skip));
    FDIGA_TRY(model(P, 1, P->U[1], P->ld[1], b, a, n1, 1, nullptr, nullptr, skip));
    FDIGA_TRY(mode1(P, P->U[0], P->ld[0], a, s, n2, skip));
  } else {
    FDIGA_TRY(mode1(P, P->W[0], P->ld[0], r, a, n2 * n3, skip));
    FDIGA_TRY(model(P, 1, P->W[1], P->ld[1], a, b, n1, n3, nullptr, nullptr, skip));
    FDIGA_TRY(model(P, 2, P->W[2], P->ld[2], b, a, n1 * n2, 1, fused ? P->lam[2] : nullptr, P->lam_inner, skip));
    if (!fused) FDIGA_TRY(block_solve(P, a, skip));
    FDIGA_TRY(model(P, 2, P->U[2], P->ld[2], a, b, n1 * n2, 1, nullptr, nullptr, skip));
    FDIGA_TRY(model(P, 1, P->U[1], P->ld[1], b, a, n1, n3, nullptr, nullptr, skip));
    FDIGA_TRY(mode1(P, P->U[0], P->ld[0], a, s, n2 * n3, skip));
  }
  return FDIGA_OK;
}
}  // namespace fdiga

extern "C" {

int fd_setup_from_factors(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* U, const double* const* W,
                          const double* const* lam, fd_plan** out) {
  return fd_setup_from_blocks(ctx, d, n, U, W, lam, nullptr, out);
}

int fd_setup_from_blocks(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* U, const double* const* W,
                         const double* const* lam_re, const double* const* lam_im, fd_plan** out) {
  FDIGA_TRY(check_common(ctx, d, n, out));
  FDIGA_CHECK(U && W && lam_re, FDIGA_ERR_INVALID_ARG, "NULL factor array");
  fd_plan* P = new_plan(ctx, d, n);
  for (int l = 0; l < d; ++l) {
    if (!(U[l] && W[l] && lam_re[l])) {
      fd_plan_destroy(P);
      set_error("NULL factor for direction %d", l);
      return FDIGA_ERR_INVALID_ARG;
    }
    P->hU[l].assign(U[l], U[l] + n[l] * n[l]);
    P->hW[l].assign(W[l], W[l] + n[l] * n[l]);
    P->hlam[l].assign(lam_re[l], lam_re[l] + n[l]);
    if (lam_im && lam_im[l])
      P->hlam_im[l].assign(lam_im[l], lam_im[l] + n[l]);
    else
      P->hlam_im[l].assign(n[l], 0.0);
  }
  int s = finish_plan(P);
  if (s != FDIGA_OK) {
    fd_plan_destroy(P);
    return s;
  }
  *out = P;
  return FDIGA_OK;
}

int fd_setup_from_eig(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* U, const double* const* lam,
                      const double* const* M, fd_plan** out) {
  FDIGA_TRY(check_common(ctx, d, n, out));
  FDIGA_CHECK(U && lam, FDIGA_ERR_INVALID_ARG, "NULL factor array");
  Solver* Sp = nullptr;
  FDIGA_TRY(ctx_solver(ctx, &Sp));
  Solver& S = *Sp;
  fd_plan* P = new_plan(ctx, d, n);
  for (int l = 0; l < d; ++l) {
    P->hU[l].assign(U[l], U[l] + n[l] * n[l]);
    P->hlam[l].assign(lam[l], lam[l] + n[l]);
    P->hlam_im[l].assign(n[l], 0.0);
    int s = compute_W(S, ctx->stream, n[l], M ? M[l] : nullptr, P->hU[l], P->hW[l], nullptr);
    if (s != FDIGA_OK) {
      fd_plan_destroy(P);
      return s;
    }
  }
  int s = finish_plan(P);
  if (s != FDIGA_OK) {
    fd_plan_destroy(P);
    return s;
  }
  *out = P;
  return FDIGA_OK;
}

int fd_setup(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* M, const double* const* K,
             const fd_setup_opts* opts, fd_plan** out) {
  fdiga::NvtxRange nvtx_("fdiga:fd_setup");
  FDIGA_TRY(check_common(ctx, d, n, out));
  FDIGA_CHECK(M && K, FDIGA_ERR_INVALID_ARG, "NULL pencil array");
  const double tol_imag = opts ? opts->tol_imag : 1e-8;
  const double cond_max = opts ? opts->cond_max : 1e8;
  const int allow_cplx = opts ? opts->allow_complex_pairs : 0;
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  double t_lu = 0, t_geev = 0, t_w = 0;  // FDIGA_VERBOSE: setup phase times (ms)
  auto since = [](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
  Solver* Sp = nullptr;
  FDIGA_TRY(ctx_solver(ctx, &Sp));  // one cuSOLVER handle per context
  Solver& S = *Sp;
  fd_plan* P = new_plan(ctx, d, n);
  auto fail = [&](int s) {
    fd_plan_destroy(P);
    return s;
  };
  for (int l = 0; l < d; ++l) {
    const int64_t nl = n[l];
    FDIGA_CHECK(M[l] && K[l], FDIGA_ERR_INVALID_ARG, "NULL pencil for direction %d", l);
    // a pencil identical to an earlier direction's (the isotropic case [M]*d, [K]*d): same factors
    int same = -1;
    for (int l2 = 0; l2 < l && same < 0; ++l2)
      if (n[l2] == nl && std::memcmp(M[l2], M[l], (size_t)(nl * nl) * sizeof(double)) == 0 &&
          std::memcmp(K[l2], K[l], (size_t)(nl * nl) * sizeof(double)) == 0)
        same = l2;
    if (same >= 0) {
      P->hU[l] = P->hU[same];
      P->hW[l] = P->hW[same];
      P->hlam[l] = P->hlam[same];
      P->hlam_im[l] = P->hlam_im[same];
      continue;
    }
    // 1. C = M^{-1} K  (eq:eigendecomposition)
    auto t0 = clk::now();
    std::vector<double> Mc = to_colmajor(M[l], nl), C = to_colmajor(K[l], nl);
    int s = lu_solve(S, ctx->stream, nl, Mc, C);
    if (s) return fail(s);
    t_lu += since(t0);
    t0 = clk::now();
    // 2. eigenpairs of C (cuSOLVER Xgeev; real input -> complex eigenvalues, real packed VR)
    double *dC = nullptr, *dVR = nullptr, *dVL = nullptr;
    cuDoubleComplex* dWv = nullptr;
    int* dinfo = nullptr;
    void* dwork = nullptr;
    size_t dws = 0, hws = 0;
    cudaMalloc(&dC, nl * nl * 8);
    cudaMalloc(&dVR, nl * nl * 8);
    cudaMalloc(&dVL, 8);
    cudaMalloc(&dWv, nl * sizeof(cuDoubleComplex));
    cudaMalloc(&dinfo, sizeof(int));
    cudaMemcpyAsync(dC, C.data(), nl * nl * 8, cudaMemcpyHostToDevice, ctx->stream);
    cusolverStatus_t cs = cusolverDnXgeev_bufferSize(S.h, S.prm, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR,
                                                     nl, CUDA_R_64F, dC, nl, CUDA_C_64F, dWv, CUDA_R_64F, dVL, 1,
                                                     CUDA_R_64F, dVR, nl, CUDA_R_64F, &dws, &hws);
    std::vector<char> hwork(std::max<size_t>(hws, 8));
    if (cs == CUSOLVER_STATUS_SUCCESS) {
      cudaMalloc(&dwork, std::max<size_t>(dws, 8));
      cs = cusolverDnXgeev(S.h, S.prm, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, nl, CUDA_R_64F, dC, nl,
                           CUDA_C_64F, dWv, CUDA_R_64F, dVL, 1, CUDA_R_64F, dVR, nl, CUDA_R_64F, dwork, dws,
                           hwork.data(), hws, dinfo);
    }
    std::vector<std::complex<double>> ev(nl);
    std::vector<double> VR((size_t)nl * nl);
    int hinfo = -1;
    cudaMemcpyAsync(ev.data(), dWv, nl * sizeof(cuDoubleComplex), cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(VR.data(), dVR, nl * nl * 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(dC);
    cudaFree(dVR);
    cudaFree(dVL);
    cudaFree(dWv);
    cudaFree(dinfo);
    cudaFree(dwork);
    if (cs != CUSOLVER_STATUS_SUCCESS || hinfo != 0) {
      set_error("cusolverDnXgeev failed (status %d, info %d)", (int)cs, hinfo);
      return fail(FDIGA_ERR_CUSOLVER);
    }
    t_geev += since(t0);
    t0 = clk::now();
    // 3. reality guard (Remark 1), sort ascending, unit 2-norm columns
    double rho = 0, maxim = 0;
    for (auto& z : ev) {
      rho = std::max(rho, std::abs(z));
      maxim = std::max(maxim, std::fabs(z.imag()));
    }
    std::vector<char> is_c(nl, 0);
    if (maxim > tol_imag * rho) {
      if (!allow_cplx) {
        set_error("complex spectrum in direction %d: max |Im lambda| = %g (rho = %g)", l, maxim, rho);
        return fail(FDIGA_ERR_COMPLEX_SPECTRUM);
      }
      for (int64_t j = 0; j < nl; ++j) is_c[j] = std::fabs(ev[j].imag()) > tol_imag * rho;
    }
    // Xgeev packs a conjugate pair (j, j+1) LAPACK-style: eigenvalue ev[j] = a + ib (b > 0),
    // eigenvector VR[:,j] + i VR[:,j+1].  Keep one key per real eigenvalue / per pair, sort by real part,
    // and store pairs as adjacent real columns (p, q) with D block [[a, b], [-b, a]].
    std::vector<int64_t> keys;
    for (int64_t j = 0; j < nl; ++j) {
      if (is_c[j]) {
        if (j + 1 >= nl || !is_c[j + 1]) {
          set_error("direction %d: unpaired complex eigenvalue", l);
          return fail(FDIGA_ERR_CUSOLVER);
        }
        keys.push_back(ev[j].imag() > 0 ? j : -(j + 1));  // negative: the pair's first column has b < 0
        ++j;
      } else {
        keys.push_back(j);
      }
    }
    auto kidx = [](int64_t k) { return k >= 0 ? k : -k - 1; };
    std::stable_sort(keys.begin(), keys.end(), [&](int64_t a, int64_t b) {
      const double ra = ev[kidx(a)].real(), rb = ev[kidx(b)].real();
      if (ra != rb) return ra < rb;
      return !is_c[kidx(a)] && is_c[kidx(b)];
    });
    std::vector<double> Ul((size_t)nl * nl), laml(nl), laml_im(nl, 0.0);
    int64_t c = 0;
    for (int64_t k : keys) {
      const int64_t j = kidx(k);
      if (!is_c[j]) {
        laml[c] = ev[j].real();
        double nrm = 0;
        for (int64_t i = 0; i < nl; ++i) nrm += VR[j * nl + i] * VR[j * nl + i];
        nrm = std::sqrt(nrm);
        for (int64_t i = 0; i < nl; ++i) Ul[i * nl + c] = VR[j * nl + i] / nrm;  // row-major U
        ++c;
      } else {
        const double a = ev[j].real(), b = std::fabs(ev[j].imag());
        const double qs = (k >= 0) ? 1.0 : -1.0;  // eigenvector for a + i|b| is p + i qs q
        double nrm = 0;
        for (int64_t i = 0; i < nl; ++i) nrm += VR[j * nl + i] * VR[j * nl + i] + VR[(j + 1) * nl + i] * VR[(j + 1) * nl + i];
        nrm = std::sqrt(nrm / 2);
        for (int64_t i = 0; i < nl; ++i) {
          Ul[i * nl + c] = VR[j * nl + i] / nrm;
          Ul[i * nl + c + 1] = qs * VR[(j + 1) * nl + i] / nrm;
        }
        laml[c] = laml[c + 1] = a;
        laml_im[c] = b;
        laml_im[c + 1] = -b;
        c += 2;
      }
    }
    // 4. W = (M U)^{-1} and cond_1(U)
    double condU = 0;
    s = compute_W(S, ctx->stream, nl, M[l], Ul, P->hW[l], &condU);
    if (s) return fail(s);
    t_w += since(t0);
    if (!(condU <= cond_max)) {
      set_error("ill-conditioned eigenvector matrix in direction %d: cond_1(U) = %g", l, condU);
      return fail(FDIGA_ERR_ILL_CONDITIONED);
    }
    P->hU[l] = std::move(Ul);
    P->hlam[l] = std::move(laml);
    P->hlam_im[l] = std::move(laml_im);
  }
  const auto t_fin = clk::now();
  int s = finish_plan(P);
  if (s != FDIGA_OK) return fail(s);
  if (getenv("FDIGA_VERBOSE"))
    fprintf(stderr, "[fdiga] fd_setup: %.1f ms (LU %.1f, geev %.1f, W %.1f, factors/autotune %.1f)\n",
            since(t_start), t_lu, t_geev, t_w, since(t_fin));
  *out = P;
  return FDIGA_OK;
}

int fd_get_factors(const fd_plan* P, int l, double* U, double* W, double* lam_re, double* lam_im) {
  FDIGA_CHECK(P && l >= 0 && l < P->d, FDIGA_ERR_INVALID_ARG, "bad plan or direction");
  const size_t nn = P->n[l] * P->n[l];
  if (U) std::memcpy(U, P->hU[l].data(), nn * 8);
  if (W) std::memcpy(W, P->hW[l].data(), nn * 8);
  if (lam_re) std::memcpy(lam_re, P->hlam[l].data(), P->n[l] * 8);
  if (lam_im) std::memcpy(lam_im, P->hlam_im[l].data(), P->n[l] * 8);
  return FDIGA_OK;
}

int fd_apply(fd_plan* P, const double* r, double* s) {
  fdiga::NvtxRange nvtx_("fdiga:fd_apply");
  return fdiga::fd_apply_ex(P, r, s, nullptr);
}

int fd_apply_host(fd_plan* P, const double* r_host, double* s_host) {
  fdiga::NvtxRange nvtx_("fdiga:fd_apply_host");
  FDIGA_CHECK(P && r_host && s_host, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_TRY(bind(P->ctx));
  FDIGA_TRY(P->host_io.ensure(std::max<int64_t>(1, P->Nloc)));
  cudaStream_t st = P->ctx->stream;
  FDIGA_CUDA(cudaMemcpyAsync(P->host_io.p, r_host, P->Nloc * 8, cudaMemcpyHostToDevice, st));
  FDIGA_TRY(fd_apply(P, P->host_io.p, P->host_io.p));
  FDIGA_CUDA(cudaMemcpyAsync(s_host, P->host_io.p, P->Nloc * 8, cudaMemcpyDeviceToHost, st));
  FDIGA_CUDA(cudaStreamSynchronize(st));
  return FDIGA_OK;
}

int fd_apply_host_async(fd_plan* P, const double* r_host, double* s_host) {
  FDIGA_CHECK(P && r_host && s_host, FDIGA_ERR_INVALID_ARG, "NULL argument");
  fdiga_ctx* ctx = P->ctx;
  FDIGA_TRY(bind(ctx));
  if (!P->s_h2d) {
    FDIGA_CUDA(cudaStreamCreateWithFlags(&P->s_h2d, cudaStreamNonBlocking));
    FDIGA_CUDA(cudaStreamCreateWithFlags(&P->s_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < fd_plan::NSLOT; ++k) {
      FDIGA_CUDA(cudaEventCreateWithFlags(&P->ev_in[k], cudaEventDisableTiming));
      FDIGA_CUDA(cudaEventCreateWithFlags(&P->ev_done[k], cudaEventDisableTiming));
      FDIGA_CUDA(cudaEventCreateWithFlags(&P->ev_out[k], cudaEventDisableTiming));
      FDIGA_CUDA(cudaEventRecord(P->ev_out[k], P->s_d2h));  // both slots start free
    }
  }
  // every slot is allocated up front: a cudaMalloc on a later call would synchronise the device mid-stream
  for (int j = 0; j < fd_plan::NSLOT; ++j) FDIGA_TRY(P->aio[j].ensure(std::max<int64_t>(1, P->Nloc)));
  const int k = P->aslot;
  P->aslot = (P->aslot + 1) % fd_plan::NSLOT;
  double* buf = P->aio[k].p;
  const size_t bytes = (size_t)P->Nloc * 8;
  // H2D into slot k once its previous result left the device; apply on the context stream; D2H behind it
  FDIGA_CUDA(cudaStreamWaitEvent(P->s_h2d, P->ev_out[k], 0));
  FDIGA_CUDA(cudaMemcpyAsync(buf, r_host, bytes, cudaMemcpyHostToDevice, P->s_h2d));
  FDIGA_CUDA(cudaEventRecord(P->ev_in[k], P->s_h2d));
  FDIGA_CUDA(cudaStreamWaitEvent(ctx->stream, P->ev_in[k], 0));
  FDIGA_TRY(fd_apply(P, buf, buf));
  FDIGA_CUDA(cudaEventRecord(P->ev_done[k], ctx->stream));
  FDIGA_CUDA(cudaStreamWaitEvent(P->s_d2h, P->ev_done[k], 0));
  FDIGA_CUDA(cudaMemcpyAsync(s_host, buf, bytes, cudaMemcpyDeviceToHost, P->s_d2h));
  FDIGA_CUDA(cudaEventRecord(P->ev_out[k], P->s_d2h));
  return FDIGA_OK;
}

int fd_host_sync(fd_plan* P) {
  FDIGA_CHECK(P, FDIGA_ERR_INVALID_ARG, "NULL plan");
  FDIGA_TRY(bind(P->ctx));
  if (P->s_d2h) FDIGA_CUDA(cudaStreamSynchronize(P->s_d2h));
  FDIGA_CUDA(cudaStreamSynchronize(P->ctx->stream));
  return FDIGA_OK;
}

double fd_apply_flops(const fd_plan* P) {
  if (!P) return 0;
  double s = 0;
  for (int l = 0; l < P->d; ++l) s += (double)P->n[l];
  return 4.0 * (double)P->N * s;
}

int fd_apply_timed(fd_plan* P, const double* r, double* s, float* kernel_ms, int* kernel_kind, int cap,
                   int* count) {
  FDIGA_CHECK(P && count, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_TRY(bind(P->ctx));
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
  cudaEvent_t e0;
  FDIGA_CUDA(cudaEventCreate(&e0));
  FDIGA_CUDA(cudaEventRecord(e0, P->ctx->stream));
  P->tev = &ev;
  P->tkind = &kind;
  const int rc = fdiga::fd_apply_ex(P, r, s, nullptr);
  P->tev = nullptr;
  P->tkind = nullptr;
  int status = rc;
  cudaError_t ce = cudaSuccess;
  if (rc == FDIGA_OK && (ce = cudaStreamSynchronize(P->ctx->stream)) != cudaSuccess) status = FDIGA_ERR_CUDA;
  *count = (int)ev.size();
  for (size_t k = 0; k < ev.size(); ++k) {
    float ms = 0.0f;
    if (status == FDIGA_OK) cudaEventElapsedTime(&ms, k == 0 ? e0 : ev[k - 1], ev[k]);
    if ((int)k < cap) {
      if (kernel_ms) kernel_ms[k] = ms;
      if (kernel_kind) kernel_kind[k] = kind[k];
    }
  }
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
  cudaEventDestroy(e0);
  if (rc != FDIGA_OK) return rc;  // the apply's own message stands
  FDIGA_CHECK(status == FDIGA_OK, status, "fd_apply_timed: %s", cudaGetErrorString(ce));
  return FDIGA_OK;
}

int fd_plan_path(const fd_plan* P, double* int8_ops) {
  FDIGA_CHECK(P, FDIGA_ERR_INVALID_ARG, "NULL plan");
  if (int8_ops) {
    double ops = 0.0;
    if (P->oz)
      for (int l = 0; l < P->d; ++l)  // forward and backward product along l
        ops += 2.0 * 2.0 * oz_pairs() * (double)P->ozX[l].rows_p * (double)P->ozW[l].rows_p *
               (double)P->ozX[l].kp;
    *int8_ops = ops;
  }
  return P->oz ? FDIGA_PATH_INT8_SPLIT : FDIGA_PATH_DMMA;
}

int fd_plan_set_path(fd_plan* P, int path) {
  FDIGA_CHECK(P, FDIGA_ERR_INVALID_ARG, "NULL plan");
  FDIGA_CHECK(path == FDIGA_PATH_DMMA || path == FDIGA_PATH_INT8_SPLIT, FDIGA_ERR_INVALID_ARG, "unknown path %d", path);
  FDIGA_TRY(bind(P->ctx));
  if (path == FDIGA_PATH_DMMA) {
    P->oz = false;  // the digit buffers stay allocated: switching back costs nothing
    return FDIGA_OK;
  }
  FDIGA_CHECK(oz_supported(P), FDIGA_ERR_NOT_SUPPORTED,
              "int8-split path: needs d = 3, a real spectrum and n_l <= %d", OZ_MAXKP);
  if (!P->ozW[0].digits) FDIGA_TRY(oz_setup(P, true));
  P->oz = true;
  return FDIGA_OK;
}

int fd_plan_destroy(fd_plan* P) {
  if (!P) return FDIGA_OK;
  cudaSetDevice(P->ctx->device);
  destroy_gmres_graph(P->ctx);
  for (int l = 0; l < 3; ++l) {
    cudaFree(P->U[l]);
    cudaFree(P->W[l]);
    cudaFree(P->lam[l]);
  }
  cudaFree(P->lam_inner);
  for (int l = 0; l < 3; ++l) {
    cudaFree(P->lam_im[l]);
    cudaFree(P->lead[l]);
    P->ozW[l].release();
    P->ozU[l].release();
    P->ozX[l].release();
  }
  P->t0.release();
  P->t1.release();
  P->host_io.release();
  if (P->s_h2d) {
    cudaStreamSynchronize(P->s_d2h);
    cudaStreamSynchronize(P->s_h2d);
    cudaStreamDestroy(P->s_h2d);
    cudaStreamDestroy(P->s_d2h);
    for (int k = 0; k < fd_plan::NSLOT; ++k) {
      cudaEventDestroy(P->ev_in[k]);
      cudaEventDestroy(P->ev_done[k]);
      cudaEventDestroy(P->ev_out[k]);
    }
  }
  for (auto& b : P->aio) b.release();
  delete P;
  return FDIGA_OK;
}

}  // extern "C"

namespace fdiga {
void destroy_solver(fdiga_ctx* ctx) {
  delete static_cast<Solver*>(ctx->solver);
  ctx->solver = nullptr;
}
}  // namespace fdiga
