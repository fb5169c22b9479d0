// Right-preconditioned restarted GMRES(m) (Saad & Schultz 1986), device resident.
//
// Every step of a restart cycle runs on the GPU with no host round trip:
//   z = P^{-1} v_j (fd_apply, DMMA), w = A z (stencil matvec),
//   classical Gram-Schmidt applied twice ("CGS2", twice is enough):
//     pass 1  h  = V_{0..j}^T w
//     pass 2  w' = w - V h,  h' = V^T w'        (update and re-orthogonalisation dots fused)
//     pass 3  w''= w' - V h', ||w''||^2          (the last block also applies the Givens rotations,
//                                                 updates g and tests |g_{j+1}| <= rtol ||b||)
//     v_{j+1} = w'' / h_{j+1,j}
// or (FDIGA_ORTH_DCGS2, the default) the same two projections with the second one delayed by a step and
// fused into the next step's first pass: two passes and one reduction per step (see dcgs_decide).
// Each pass reduces through per-block partials and a "last block" that sums them in fixed order
// (deterministic, no second launch).  The m steps of one cycle are captured once into a CUDA graph
// (cached on the context); after convergence is declared a device flag turns the remaining launches
// of the cycle into no-ops.  The host synchronises once per cycle, to read the true residual.
// Cycle close (y = R^{-1} g, x += P^{-1}(V y)) and the true residual also run on the device.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "reduce.cuh"
#include "ptx.cuh"

using namespace fdiga;

namespace {

constexpr int KMAX = 32;  // basis vectors per pass (m <= KMAX - 1)
constexpr int NCNT = 4;   // last-block counters

struct GmState {
  double H[(KMAX + 1) * KMAX];  // R of the rotated Hessenberg (row-major, stride KMAX)
  double cs[KMAX], sn[KMAX], g[KMAX + 1];
  double h1[KMAX + 1], h2[KMAX + 1], y[KMAX];
  // sharded (nranks > 1): per-rank partial sums, all-reduced into h1 / h2 / wn2 / rs
  double h1l[KMAX + 1], h2l[KMAX + 1], wn2l, wn2, rsl[2], rs[2];
  double beta, bnorm, target, invh, rel_implicit, rel_true;
  int stop;        // cycle stop flag: every remaining step launch of the cycle is a no-op
  int k;           // steps taken in the current cycle
  int iters;       // total Arnoldi steps
  int max_iters;
  int first;       // first residual of the solve (records ||b||)
  int breakdown;   // non-finite value met
  int reorth;      // CGS + DGKS: the current step needs the second pass
  int nreorth;     // second passes taken
  unsigned int counter[NCNT];
  // DCGS2 (delayed re-orthogonalisation): raw (unrotated) Hessenberg, the reduced [a; b; rho; c] of the
  // step, and the coefficients of its update pass
  double Hraw[(KMAX + 1) * KMAX];
  double dred[2 * KMAX + 2], dredl[2 * KMAX + 2];
  double pa[KMAX], pb[KMAX], gam, invb;
};

// ---- streaming Gram-Schmidt passes.  The k basis vectors and w are streamed through shared memory by
// the TMA engine (1D bulk copies, mbarrier completion) in chunks of SC elements, ST stages deep, so the
// bytes in flight do not depend on registers; every thread then owns one element of the chunk.  V rows
// and w are 512-byte aligned with a leading dimension ldv (multiple of 64) >= N, so every copy is a
// whole number of 16-byte units; elements >= N are masked.
constexpr int SC = RT;  // elements per chunk (one per thread)

enum { GS_DOT = 0, GS_UPD_DOT = 1, GS_UPD = 2, GS_UPD_SCALE = 3, GS_LINCOMB = 4 };

template <int K>
__host__ __device__ constexpr int gs_stages() {
  return (200 * 1024) / ((K + 1) * SC * 8) >= 4 ? 4 : ((200 * 1024) / ((K + 1) * SC * 8) >= 3 ? 3 : 2);
}

template <int K>
__host__ __device__ constexpr size_t gs_smem_bytes() {
  return (size_t)gs_stages<K>() * (K + 1) * SC * 8 + 64;
}

// acc[i] (i < K) = V_i . w or V_i . w' and acc[K] = w.w or w'.w' with w' = w - V hs (GS_UPD_DOT / GS_UPD,
// w' stored back to global); GS_UPD_SCALE stores scale * w' into `out` instead (no dots)
template <int K, int MODE>
__device__ __forceinline__ void gs_stream(const double* __restrict__ V, int64_t ldv, double* w, int64_t N,
                                          const double* hs, double (&acc)[K + 1], double* out = nullptr,
                                          double scale = 1.0) {
  constexpr int S = gs_stages<K>();
  extern __shared__ __align__(128) double gsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + (size_t)S * (K + 1) * SC);
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i <= K; ++i) acc[i] = 0.0;
  const int64_t nchunk = (N + SC - 1) / SC;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // warp 0 issues a stage: lane 0 posts the byte count, then lane i copies row i (V_i, or w for i = K)
  auto issue = [&](int64_t c, int s) {
    const int lane = tid & 31;
    const int64_t e0 = c * SC;
    const uint32_t bytes = (uint32_t)((ldv - e0 < SC ? ldv - e0 : SC) * 8);
    double* dst = gsm + (size_t)s * (K + 1) * SC;
    if (lane == 0) mbar_arrive_expect_tx(&full[s], (K + 1) * bytes);
    __syncwarp();
    if (lane <= K) bulk_g2s(dst + lane * SC, lane < K ? V + lane * ldv + e0 : w + e0, bytes, &full[s]);
  };
  if (tid < 32)
    for (int s = 0; s < S; ++s) {
      const int64_t c = blockIdx.x + (int64_t)s * gridDim.x;
      if (c < nchunk) issue(c, s);
    }
  int it = 0;
  for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x, ++it) {
    const int s = it % S;
    mbar_wait(&full[s], (uint32_t)((it / S) & 1));
    const double* buf = gsm + (size_t)s * (K + 1) * SC;
    const int64_t e = c * SC + tid;
    if (e < N && MODE == GS_LINCOMB) {  // out = sum_i hs[i] V_i
      double sacc = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) sacc = fma(hs[i], buf[i * SC + tid], sacc);
      out[e] = sacc;
    } else if (e < N) {
      double wv = buf[K * SC + tid];
      if (MODE != GS_DOT) {
#pragma unroll
        for (int i = 0; i < K; ++i) wv = fma(-hs[i], buf[i * SC + tid], wv);
        if (MODE == GS_UPD_SCALE)
          out[e] = scale * wv;
        else
          w[e] = wv;
      }
      if (MODE != GS_UPD && MODE != GS_UPD_SCALE) {
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = fma(buf[i * SC + tid], wv, acc[i]);
      }
      acc[K] = fma(wv, wv, acc[K]);
    }
    __syncthreads();  // every thread is done with stage s
    if (tid < 32) {
      const int64_t cn = c + (int64_t)S * gridDim.x;
      if (cn < nchunk) {
        fence_proxy_async();
        issue(cn, s);
      }
    }
  }
}

// DCGS2 streaming: the K rows of Q, then u and z (EXTRA = 2) or u only (EXTRA = 1, the cycle's last
// column); PASS 0 = dots, PASS 1 = the update writing q_K (into out) and u_{K+1} (into u, in place).
template <int K>
__host__ __device__ constexpr int dc_stages() {
  return (200 * 1024) / ((K + 2) * SC * 8) >= 4 ? 4 : ((200 * 1024) / ((K + 2) * SC * 8) >= 3 ? 3 : 2);
}
template <int K>
__host__ __device__ constexpr size_t dc_smem_bytes() {
  return (size_t)dc_stages<K>() * (K + 2) * SC * 8 + 64;
}

template <int K, int EXTRA, int PASS>
__device__ __forceinline__ void dc_stream(const double* __restrict__ V, int64_t ldv, const double* u,
                                          const double* z, int64_t N, const GmState* st, double (&acc)[2 * K + 2],
                                          double* out, double* uout) {
  constexpr int S = dc_stages<K>();
  constexpr int ROWS = K + EXTRA;
  extern __shared__ __align__(128) double dsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)S * (K + 2) * SC);
  __shared__ double pa[KMAX + 1], pb[KMAX + 1];
  const int tid = threadIdx.x;
  if (PASS == 1 && tid < K) {
    pa[tid] = st->pa[tid];
    pb[tid] = st->pb[tid];
  }
#pragma unroll
  for (int i = 0; i < 2 * K + 2; ++i) acc[i] = 0.0;
  const int64_t nchunk = (N + SC - 1) / SC;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // pass B walks the chunks from the last to the first: it follows pass A over the same (K + 2) vectors, whose
  // last chunks are what is still in L2 (up to ~126 MB of the (K + 2) 8 N bytes); it has no reduction, so the
  // order changes no result bit
  auto chunk_of = [&](int64_t c) { return PASS == 1 ? nchunk - 1 - c : c; };
  auto issue = [&](int64_t c, int s) {
    const int lane = tid & 31;
    const int64_t e0 = chunk_of(c) * SC;
    const uint32_t bytes = (uint32_t)((ldv - e0 < SC ? ldv - e0 : SC) * 8);
    double* dst = dsm + (size_t)s * (K + 2) * SC;
    if (lane == 0) mbar_arrive_expect_tx(&full[s], ROWS * bytes);
    __syncwarp();
    if (lane < ROWS)
      bulk_g2s(dst + lane * SC, lane < K ? V + lane * ldv + e0 : (lane == K ? u + e0 : z + e0), bytes, &full[s]);
  };
  if (tid < 32)
    for (int s = 0; s < S; ++s) {
      const int64_t c = blockIdx.x + (int64_t)s * gridDim.x;
      if (c < nchunk) issue(c, s);
    }
  const double gam = PASS == 1 ? st->gam : 0.0, ib = PASS == 1 ? st->invb : 0.0;
  int it = 0;
  for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x, ++it) {
    const int s = it % S;
    mbar_wait(&full[s], (uint32_t)((it / S) & 1));
    const double* buf = dsm + (size_t)s * (K + 2) * SC;
    const int64_t e = chunk_of(c) * SC + tid;
    if (e < N) {
      const double uv = buf[K * SC + tid];
      const double zv = EXTRA == 2 ? buf[(K + 1) * SC + tid] : 0.0;
      if (PASS == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const double q = buf[i * SC + tid];
          acc[i] = fma(q, uv, acc[i]);
          if (EXTRA == 2) acc[K + i] = fma(q, zv, acc[K + i]);
        }
        acc[2 * K] = fma(uv, uv, acc[2 * K]);
        if (EXTRA == 2) acc[2 * K + 1] = fma(uv, zv, acc[2 * K + 1]);
      } else {
        double qv = uv, nz = zv;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const double q = buf[i * SC + tid];
          qv = fma(-pa[i], q, qv);
          nz = fma(-pb[i], q, nz);
        }
        qv *= ib;
        out[e] = qv;
        uout[e] = (nz - gam * qv) * ib;
      }
    }
    __syncthreads();
    if (tid < 32) {
      const int64_t cn = c + (int64_t)S * gridDim.x;
      if (cn < nchunk) {
        fence_proxy_async();
        issue(cn, s);
      }
    }
  }
}

__device__ void dcgs_decide(GmState* st, int j, int m, const double* red, int withz, double* hist, int hist_cap);
__device__ void arnoldi_close_step(GmState* st, int j, int m, double wn2, double* hist, int hist_cap);

// DCGS2 pass A: [a; b; rho; c] (reduction); the last block decides (single rank) or leaves partials
template <int K, int EXTRA>
__global__ void __launch_bounds__(RT) dcgs_passA(const double* __restrict__ V, int64_t ldv, const double* u,
                                                 const double* z, int64_t N, double* part, GmState* st, int m,
                                                 double* hist, int hist_cap, int close) {
  if (st->stop) return;
  double acc[2 * K + 2];
  dc_stream<K, EXTRA, 0>(V, ldv, u, z, N, st, acc, nullptr, nullptr);
  // pack [a (K), b (K), rho, c] contiguously for the reduction
  double* out = close ? st->dred : st->dredl;
  if (reduce_last<2 * K + 2>(acc, 2 * K + 2, part, &st->counter[0], out) && close && threadIdx.x == 0)
    dcgs_decide(st, K, m, out, EXTRA == 2, hist, hist_cap);
}

// DCGS2 pass B: q_K and u_{K+1}
// (u and uout alias for K >= 1: every element is read from shared memory before its own thread writes it)
template <int K>
__global__ void __launch_bounds__(RT) dcgs_passB(const double* __restrict__ V, int64_t ldv, const double* u,
                                                 const double* z, int64_t N, GmState* st, double* qout,
                                                 double* uout) {
  if (st->stop) return;
  double acc[2 * K + 2];
  dc_stream<K, 2, 1>(V, ldv, u, z, N, st, acc, qout, uout);
}

// pass 1: h[i] = V_i . w (i < k), h[k] = w . w
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass1(const double* __restrict__ V, int64_t ldv, int /*k (= K)*/,
                                                    const double* __restrict__ w, int64_t N, double* part,
                                                    GmState* st, double* hout, int cond) {
  if (st->stop || (cond && !st->reorth)) return;
  double acc[K + 1];
  gs_stream<K, GS_DOT>(V, ldv, const_cast<double*>(w), N, nullptr, acc);
  reduce_last<K + 1>(acc, K + 1, part, &st->counter[0], hout);
}

// pass 2: w <- w - V h1 ; h2[i] = V_i . w (new w), h2[k] = ||w||^2 (V read once, from shared memory)
__device__ void arnoldi_close_step(GmState* st, int j, int m, double wn2, double* hist, int hist_cap);

// close == 1 (CGS2, single rank): the last block also closes step j with the Pythagorean norm
// ||w''||^2 = ||w'||^2 - ||h2||^2 of the second projection (h2 is O(eps kappa) small after the first one,
// so the subtraction loses nothing), which lets pass 3 write v_{j+1} directly without a reduction.
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass2(const double* __restrict__ V, int64_t ldv, int /*k (= K)*/,
                                                    double* __restrict__ w, int64_t N, double* part, GmState* st,
                                                    double* hout, int j, int m, double* hist, int hist_cap,
                                                    int close) {
  if (st->stop) return;
  __shared__ double hs[KMAX];
  if (threadIdx.x < K) hs[threadIdx.x] = st->h1[threadIdx.x];
  __syncthreads();
  double acc[K + 1];
  gs_stream<K, GS_UPD_DOT>(V, ldv, w, N, hs, acc);
  if (reduce_last<K + 1>(acc, K + 1, part, &st->counter[1], hout) && close && threadIdx.x == 0) {
    double wn2 = hout[K];
    for (int i = 0; i < K; ++i) wn2 -= hout[i] * hout[i];
    arnoldi_close_step(st, j, m, wn2, hist, hist_cap);
  }
}

// sharded CGS2: close step j from the all-reduced h2 (Pythagorean norm, as above)
__global__ void close_step_pyth_kernel(GmState* st, int j, int m, double* hist, int hist_cap) {
  if (st->stop) return;
  const int k = j + 1;
  double wn2 = st->h2[k];
  for (int i = 0; i < k; ++i) wn2 -= st->h2[i] * st->h2[i];
  arnoldi_close_step(st, j, m, wn2, hist, hist_cap);
}

// cycle close: out = sum_{i < K} y_i V_i, streamed like the Gram-Schmidt passes (w slot: row 0 again)
template <int K>
__global__ void __launch_bounds__(RT) lincomb_stream(const double* __restrict__ V, int64_t ldv,
                                                     double* __restrict__ out, int64_t N, const GmState* st) {
  __shared__ double hs[KMAX];
  if (threadIdx.x < K) hs[threadIdx.x] = st->y[threadIdx.x];
  __syncthreads();
  double acc[K + 1];
  gs_stream<K, GS_LINCOMB>(V, ldv, const_cast<double*>(V), N, hs, acc, out, 1.0);
}

// CGS2 pass 3: v_{j+1} = (w' - V h2) / h_{j+1,j} written straight into the basis (no reduction)
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass3n(const double* __restrict__ V, int64_t ldv,
                                                     double* __restrict__ w, int64_t N, GmState* st,
                                                     double* vnext) {
  if (st->stop) return;
  __shared__ double hs[KMAX];
  if (threadIdx.x < K) hs[threadIdx.x] = st->h2[threadIdx.x];
  __syncthreads();
  double acc[K + 1];
  gs_stream<K, GS_UPD_SCALE>(V, ldv, w, N, hs, acc, vnext, st->invh);
}

// Givens rotations / convergence test for step j (one thread), once h = h1 + h2 and ||w''||^2 are known.
__device__ void arnoldi_close_step(GmState* st, int j, int m, double wn2, double* hist, int hist_cap) {
  double* H = st->H;
  const int k = j + 1;
  double col[KMAX + 1];
  bool bad = !(wn2 >= 0.0) || !isfinite(wn2);
  for (int i = 0; i < k; ++i) {
    col[i] = st->h1[i] + st->h2[i];
    bad = bad || !isfinite(col[i]);
  }
  const double hn = sqrt(fmax(wn2, 0.0));
  col[k] = hn;
  for (int i = 0; i < j; ++i) {  // previous rotations
    const double t = st->cs[i] * col[i] + st->sn[i] * col[i + 1];
    col[i + 1] = -st->sn[i] * col[i] + st->cs[i] * col[i + 1];
    col[i] = t;
  }
  const double a = col[j], b = col[k];
  const double rr = hypot(a, b);
  const double c = rr == 0.0 ? 1.0 : a / rr, s = rr == 0.0 ? 0.0 : b / rr;
  st->cs[j] = c;
  st->sn[j] = s;
  col[j] = rr;
  col[k] = 0.0;
  for (int i = 0; i <= k; ++i) H[i * KMAX + j] = col[i];
  st->g[k] = -s * st->g[j];
  st->g[j] = c * st->g[j];
  st->iters += 1;
  st->k = k;
  st->reorth = 0;
  st->rel_implicit = fabs(st->g[k]) / st->bnorm;
  if (hist && st->iters - 1 < hist_cap) hist[st->iters - 1] = st->rel_implicit;
  st->invh = hn > 0.0 ? 1.0 / hn : 0.0;
  if (bad) st->breakdown = 1;
  if (bad || fabs(st->g[k]) <= st->target || hn == 0.0 || st->iters >= st->max_iters || k >= m) st->stop = 1;
}

// ---- DCGS2: classical Gram-Schmidt twice with the second pass delayed by one step (one reduction per
// step).  Step j holds Q_j = [q_0..q_{j-1}] (final) and u_j, the candidate for q_j projected once.  With
// z = B u_j (B = A P^{-1}):
//   pass A (one reduction):  a = Q_j^T u_j,  b = Q_j^T z,  rho = u_j.u_j,  c = u_j.z
//   decide:  beta^2 = rho - |a|^2 (Pythagoras: a is the O(eps kappa) second projection);  column j-1 of the
//            Hessenberg = h1_{j-1} + a, H[j][j-1] = beta  -> Givens / convergence;  gamma = (c - a.b) / beta;
//            the first-pass coefficients of column j: h1_j = ([b; gamma] - Hraw a) / beta  (because
//            B q_j = (z - Q_{j+1} Hraw a) / beta)
//   pass B:  q_j = (u_j - Q_j a) / beta  (final),  u_{j+1} = (z - Q_j b - gamma q_j) / beta
// Two streamed passes over Q_j per step instead of CGS2's three, and the same columns (iteration counts)
// as CGS2; the convergence of column j-1 is seen one operator application later (at step j).
__device__ void dcgs_decide(GmState* st, int j, int m, const double* red, int withz, double* hist, int hist_cap) {
  const double* a = red;
  const double* b = red + j;
  const double rho = red[2 * j], c = red[2 * j + 1];
  double aa = 0.0;
  for (int i = 0; i < j; ++i) aa += a[i] * a[i];
  const double b2 = rho - aa;
  double beta;
  if (j == 0) {
    beta = sqrt(fmax(b2, 0.0));
    st->g[0] *= beta;  // r = ||r|| u_0 = ||r|| beta q_0
    if (!(beta > 0.0) || !isfinite(beta)) {
      st->breakdown = !isfinite(beta);
      st->stop = 1;
      return;
    }
  } else {
    for (int i = 0; i < j; ++i) {
      st->h2[i] = a[i];
      st->Hraw[i * KMAX + (j - 1)] = st->h1[i] + a[i];
    }
    beta = sqrt(fmax(b2, 0.0));
    st->Hraw[j * KMAX + (j - 1)] = beta;
    arnoldi_close_step(st, j - 1, m, b2, hist, hist_cap);
    if (st->stop || !withz) return;
  }
  const double ib = 1.0 / beta;
  double ab = 0.0;
  for (int i = 0; i < j; ++i) ab += a[i] * b[i];
  const double gam = (c - ab) * ib;
  for (int i = 0; i <= j; ++i) {
    double ha = 0.0;  // (Hraw a)_i: column l of Hraw has rows 0..l+1
    for (int l = i > 0 ? i - 1 : 0; l < j; ++l) ha += st->Hraw[i * KMAX + l] * a[l];
    st->h1[i] = ((i < j ? b[i] : gam) - ha) * ib;
  }
  for (int i = 0; i < j; ++i) {
    st->pa[i] = a[i];
    st->pb[i] = b[i];
  }
  st->gam = gam;
  st->invb = ib;
}

__global__ void dcgs_decide_kernel(GmState* st, int j, int m, int withz, double* hist, int hist_cap) {
  if (st->stop) return;
  dcgs_decide(st, j, m, st->dred, withz, hist, hist_cap);
}

// CGS + DGKS decision after the first update (one thread): Daniel-Gragg-Kaufman-Stewart test
// ||w'|| < ||w|| / sqrt(2) (w.w before the update sits in h1[k]) -> a second pass; otherwise h2 = 0 and
// the step closes with the first pass.
__device__ void dgks_decide(GmState* st, int j, int m, double wn2, double* hist, int hist_cap) {
  const int k = j + 1;
  if (!(wn2 >= 0.5 * st->h1[k])) {  // also catches NaN
    st->reorth = 1;
    st->nreorth += 1;
    return;
  }
  for (int i = 0; i < k; ++i) st->h2[i] = 0.0;
  arnoldi_close_step(st, j, m, wn2, hist, hist_cap);
}

enum { P3_CLOSE = 0, P3_DGKS = 1, P3_CLOSE_IF_REORTH = 2 };

// pass 3: w <- w - V h ; ||w||^2 ; the last block closes the step.  mode P3_CLOSE (CGS2): h = h2, close;
// P3_DGKS (CGS first update): h = h1, DGKS decision; P3_CLOSE_IF_REORTH: only after a DGKS
// re-orthogonalisation, h = h2, close.
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass3(const double* __restrict__ V, int64_t ldv, int /*k (= K)*/,
                                                    double* __restrict__ w, int64_t N, double* part, GmState* st,
                                                    int j, int m, double* hist, int hist_cap, int close, int mode) {
  constexpr int k = K;
  if (st->stop || (mode == P3_CLOSE_IF_REORTH && !st->reorth)) return;
  __shared__ double hs[KMAX];
  if (threadIdx.x < k) hs[threadIdx.x] = mode == P3_DGKS ? st->h1[threadIdx.x] : st->h2[threadIdx.x];
  __syncthreads();
  double accs[K + 1];
  gs_stream<K, GS_UPD>(V, ldv, w, N, hs, accs);
  double acc[1] = {accs[K]};
  __shared__ double nrm[1];
  if (reduce_last<1>(acc, 1, part, &st->counter[2], nrm)) {
    if (threadIdx.x == 0) {
      if (!close)
        st->wn2l = nrm[0];  // sharded: all-reduced into wn2, then close_step_kernel
      else if (mode == P3_DGKS)
        dgks_decide(st, j, m, nrm[0], hist, hist_cap);
      else
        arnoldi_close_step(st, j, m, nrm[0], hist, hist_cap);
    }
  }
}

// sharded: close step j (or take the DGKS decision) once ||w||^2 is global
__global__ void close_step_kernel(GmState* st, int j, int m, double* hist, int hist_cap, int mode) {
  if (st->stop || (mode == P3_CLOSE_IF_REORTH && !st->reorth)) return;
  if (mode == P3_DGKS)
    dgks_decide(st, j, m, st->wn2, hist, hist_cap);
  else
    arnoldi_close_step(st, j, m, st->wn2, hist, hist_cap);
}

// v_{j+1} = w * invh (a no-op once the cycle stopped)
__global__ void next_basis_kernel(const double* __restrict__ w, double* __restrict__ out, int64_t N,
                                  const GmState* st) {
  if (st->stop) return;
  const double s = st->invh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = s * w[e];
}

// cycle start from ||r||^2 and ||b||^2 (one thread)
__device__ void begin_cycle(GmState* st, double rr, double bb, double rtol) {
  const double beta = sqrt(rr);
  if (st->first) {
    st->bnorm = sqrt(bb);
    st->target = rtol * st->bnorm;
    st->first = 0;
  }
  st->beta = beta;
  st->rel_true = st->bnorm > 0 ? beta / st->bnorm : 0.0;
  st->k = 0;
  for (int i = 0; i <= KMAX; ++i) st->g[i] = 0.0;
  st->g[0] = beta;
  st->invh = beta > 0.0 ? 1.0 / beta : 0.0;
  if (!isfinite(beta)) st->breakdown = 1;
  st->stop = (beta <= st->target || st->bnorm == 0.0 || st->iters >= st->max_iters || st->breakdown) ? 1 : 0;
}

// r = b - Ax -> V_0 ; ||r||, (first call) ||b|| ; the last block starts the cycle (single rank) or
// leaves the partial sums for the all-reduce (sharded)
__global__ void __launch_bounds__(RT) residual_start_kernel(const double* __restrict__ b,
                                                            const double* __restrict__ Ax, double* __restrict__ r,
                                                            int64_t N, double* part, GmState* st, double rtol,
                                                            int close) {
  double acc[2] = {0.0, 0.0};
  for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT) {
    const double bv = b[e];
    const double v = bv - Ax[e];
    r[e] = v;
    acc[0] = fma(v, v, acc[0]);
    acc[1] = fma(bv, bv, acc[1]);
  }
  __shared__ double out[2];
  if (reduce_last<2>(acc, 2, part, &st->counter[3], out) && threadIdx.x == 0) {
    if (close) {
      begin_cycle(st, out[0], out[1], rtol);
    } else {
      st->rsl[0] = out[0];
      st->rsl[1] = out[1];
    }
  }
}

__global__ void begin_cycle_kernel(GmState* st, double rtol) { begin_cycle(st, st->rs[0], st->rs[1], rtol); }

// V_0 = r / beta in place
__global__ void scale_start_kernel(double* __restrict__ v, int64_t N, const GmState* st) {
  if (st->stop) return;
  const double s = st->invh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    v[e] *= s;
}

// y = R_k^{-1} g_{0..k-1} (back substitution, one thread)
__global__ void solve_y_kernel(GmState* st) {
  const int k = st->k;
  for (int i = k - 1; i >= 0; --i) {
    double s = st->g[i];
    for (int c = i + 1; c < k; ++c) s -= st->H[i * KMAX + c] * st->y[c];
    st->y[i] = s / st->H[i * KMAX + i];
  }
}

// out = sum_{i<k} y_i V_i
__global__ void __launch_bounds__(RT) lincomb_kernel(const double* __restrict__ V, int64_t ldv,
                                                     double* __restrict__ out, int64_t N, const GmState* st) {
  __shared__ double ys[KMAX];
  const int k = st->k;
  if (threadIdx.x < k) ys[threadIdx.x] = st->y[threadIdx.x];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT) {
    double v = 0;
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) v = fma(ys[i], V[i * ldv + e], v);
    out[e] = v;
  }
}

__global__ void axpy_kernel(const double* __restrict__ z, double* __restrict__ x, int64_t N) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    x[e] += z[e];
}

struct Ws {
  int64_t N, ldv;
  int nblk;
  bool sh;  // nranks > 1: reductions are all-reduced between the passes
  int orth; // FDIGA_ORTH_*
  double *V, *z, *w, *u, *part, *hist;  // u: DCGS2's once-projected candidate u_j
  GmState* st;
};

// launch shape of the streaming passes for k = K: dynamic shared memory and a persistent grid of as
// many CTAs per SM as the stages allow (<= 8)
template <int K>
int gs_grid(fdiga_ctx* ctx, int64_t N, size_t* smem) {
  *smem = gs_smem_bytes<K>();
  static bool attr = false;
  if (!attr) {
    FDIGA_CUDA(cudaFuncSetAttribute(arnoldi_pass1<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    FDIGA_CUDA(cudaFuncSetAttribute(arnoldi_pass2<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    FDIGA_CUDA(cudaFuncSetAttribute(arnoldi_pass3<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    FDIGA_CUDA(cudaFuncSetAttribute(arnoldi_pass3n<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    FDIGA_CUDA(cudaFuncSetAttribute(lincomb_stream<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    attr = true;
  }
  const int per_sm = std::max(1, std::min(8, (int)((227 * 1024) / (*smem + 1024))));
  return (int)std::max<int64_t>(1, std::min<int64_t>((N + SC - 1) / SC, (int64_t)ctx->sm_count * per_sm));
}

template <int K>
int pass3_k(fdiga_ctx* ctx, const Ws& W, int j, int m, int hist_cap, int mode) {
  GmState* st = W.st;
  size_t smem = 0;
  const int grid = gs_grid<K>(ctx, W.N, &smem);
  arnoldi_pass3<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, j, m, W.hist, hist_cap,
                                                   W.sh ? 0 : 1, mode);
  count_launch(ctx);
  if (W.sh) {
    FDIGA_TRY(comm_allreduce(ctx, &st->wn2l, &st->wn2, 1));
    close_step_kernel<<<1, 1, 0, ctx->stream>>>(st, j, m, W.hist, hist_cap, mode);
    count_launch(ctx);
  }
  return FDIGA_OK;
}

template <int K>
int passes_k(fdiga_ctx* ctx, const Ws& W, int j, int m, int hist_cap) {
  GmState* st = W.st;
  size_t smem = 0;
  const int grid = gs_grid<K>(ctx, W.N, &smem);
  arnoldi_pass1<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, W.sh ? st->h1l : st->h1, 0);
  count_launch(ctx);
  if (W.sh) FDIGA_TRY(comm_allreduce(ctx, st->h1l, st->h1, K + 1));
  if (W.orth == FDIGA_ORTH_CGS2) {
    // classical Gram-Schmidt twice: pass 2 fuses the update with the second projection and (Pythagorean
    // norm) closes the step; pass 3 writes the normalised v_{j+1}.  Two reductions per step.
    arnoldi_pass2<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, W.sh ? st->h2l : st->h2,
                                                      j, m, W.hist, hist_cap, W.sh ? 0 : 1);
    count_launch(ctx);
    if (W.sh) {
      FDIGA_TRY(comm_allreduce(ctx, st->h2l, st->h2, K + 1));
      close_step_pyth_kernel<<<1, 1, 0, ctx->stream>>>(st, j, m, W.hist, hist_cap);
      count_launch(ctx);
    }
    arnoldi_pass3n<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, W.w, W.N, st, W.V + (int64_t)(j + 1) * W.ldv);
    count_launch(ctx);
    FDIGA_CUDA(cudaGetLastError());
    return FDIGA_OK;
  }
  // classical Gram-Schmidt with DGKS re-orthogonalisation: update, test, and only when the test fails a
  // second projection + update (device flag; the launches are no-ops otherwise)
  FDIGA_TRY(pass3_k<K>(ctx, W, j, m, hist_cap, P3_DGKS));
  arnoldi_pass1<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, W.sh ? st->h2l : st->h2, 1);
  count_launch(ctx);
  if (W.sh) FDIGA_TRY(comm_allreduce(ctx, st->h2l, st->h2, K + 1));
  return pass3_k<K>(ctx, W, j, m, hist_cap, P3_CLOSE_IF_REORTH);
}

// DCGS2 step j = K (EXTRA = 2: pass A, decide, pass B) or the cycle's closing pass A over K = m (EXTRA = 1)
template <int K, int EXTRA>
int dcgs_k(fdiga_ctx* ctx, const Ws& W, const double* u, int m, int hist_cap) {
  GmState* st = W.st;
  constexpr size_t smem = dc_smem_bytes<K>();
  static bool attr = false;
  if (!attr) {
    FDIGA_CUDA(cudaFuncSetAttribute(dcgs_passA<K, EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (EXTRA == 2)
      FDIGA_CUDA(cudaFuncSetAttribute(dcgs_passB<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int per_sm = std::max(1, std::min(8, (int)((227 * 1024) / (smem + 1024))));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((W.N + SC - 1) / SC, (int64_t)ctx->sm_count * per_sm));
  dcgs_passA<K, EXTRA><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, u, W.w, W.N, W.part, st, m, W.hist, hist_cap,
                                                        W.sh ? 0 : 1);
  count_launch(ctx);
  if (W.sh) {
    FDIGA_TRY(comm_allreduce(ctx, st->dredl, st->dred, 2 * K + 2));
    dcgs_decide_kernel<<<1, 1, 0, ctx->stream>>>(st, K, m, EXTRA == 2, W.hist, hist_cap);
    count_launch(ctx);
  }
  if (EXTRA == 2) {
    dcgs_passB<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, u, W.w, W.N, st, W.V + (int64_t)K * W.ldv, W.u);
    count_launch(ctx);
  }
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

int launch_dcgs(fdiga_ctx* ctx, const Ws& W, int j, const double* u, int m, int hist_cap, bool closing) {
  switch (j) {
#define FDIGA_K(K)                                                                                   \
  case K:                                                                                            \
    return closing ? dcgs_k<K, 1>(ctx, W, u, m, hist_cap) : dcgs_k<K, 2>(ctx, W, u, m, hist_cap);
    FDIGA_K(0) FDIGA_K(1) FDIGA_K(2) FDIGA_K(3) FDIGA_K(4) FDIGA_K(5) FDIGA_K(6) FDIGA_K(7) FDIGA_K(8)
    FDIGA_K(9) FDIGA_K(10) FDIGA_K(11) FDIGA_K(12) FDIGA_K(13) FDIGA_K(14) FDIGA_K(15) FDIGA_K(16)
    FDIGA_K(17) FDIGA_K(18) FDIGA_K(19) FDIGA_K(20) FDIGA_K(21) FDIGA_K(22) FDIGA_K(23) FDIGA_K(24)
    FDIGA_K(25) FDIGA_K(26) FDIGA_K(27) FDIGA_K(28) FDIGA_K(29) FDIGA_K(30) FDIGA_K(31)
#undef FDIGA_K
    default:
      break;
  }
  FDIGA_CHECK(false, FDIGA_ERR_INVALID_ARG, "basis size %d out of range", j);
}

template <int K>
int lincomb_k(fdiga_ctx* ctx, const Ws& W, double* out) {
  size_t smem = 0;
  const int grid = gs_grid<K>(ctx, W.N, &smem);
  lincomb_stream<K><<<grid, RT, smem, ctx->stream>>>(W.V, W.ldv, out, W.N, W.st);
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

int launch_lincomb(fdiga_ctx* ctx, const Ws& W, int k, double* out) {
  switch (k) {
#define FDIGA_K(K) \
  case K:          \
    return lincomb_k<K>(ctx, W, out);
    FDIGA_K(1) FDIGA_K(2) FDIGA_K(3) FDIGA_K(4) FDIGA_K(5) FDIGA_K(6) FDIGA_K(7) FDIGA_K(8)
    FDIGA_K(9) FDIGA_K(10) FDIGA_K(11) FDIGA_K(12) FDIGA_K(13) FDIGA_K(14) FDIGA_K(15) FDIGA_K(16)
    FDIGA_K(17) FDIGA_K(18) FDIGA_K(19) FDIGA_K(20) FDIGA_K(21) FDIGA_K(22) FDIGA_K(23) FDIGA_K(24)
    FDIGA_K(25) FDIGA_K(26) FDIGA_K(27) FDIGA_K(28) FDIGA_K(29) FDIGA_K(30) FDIGA_K(31)
#undef FDIGA_K
    default:
      break;
  }
  lincomb_kernel<<<W.nblk, RT, 0, ctx->stream>>>(W.V, W.ldv, out, W.N, W.st);  // k = 0 or out of range
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

// The three CGS2 passes of step j with k = j + 1 basis vectors (one instantiation per k: fully
// unrolled loops, accumulators in registers).
int launch_passes(fdiga_ctx* ctx, const Ws& W, int k, int j, int m, int hist_cap) {
  switch (k) {
#define FDIGA_K(K) \
  case K:          \
    FDIGA_TRY(passes_k<K>(ctx, W, j, m, hist_cap)); \
    break;
    FDIGA_K(1) FDIGA_K(2) FDIGA_K(3) FDIGA_K(4) FDIGA_K(5) FDIGA_K(6) FDIGA_K(7) FDIGA_K(8)
    FDIGA_K(9) FDIGA_K(10) FDIGA_K(11) FDIGA_K(12) FDIGA_K(13) FDIGA_K(14) FDIGA_K(15) FDIGA_K(16)
    FDIGA_K(17) FDIGA_K(18) FDIGA_K(19) FDIGA_K(20) FDIGA_K(21) FDIGA_K(22) FDIGA_K(23) FDIGA_K(24)
    FDIGA_K(25) FDIGA_K(26) FDIGA_K(27) FDIGA_K(28) FDIGA_K(29) FDIGA_K(30) FDIGA_K(31)
#undef FDIGA_K
    default:
      FDIGA_CHECK(false, FDIGA_ERR_INVALID_ARG, "basis size %d out of range", k);
  }
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

// Enqueue the m Arnoldi steps of one cycle on ctx->stream (captured by the caller).
int enqueue_cycle(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const Ws& W, int m, int hist_cap) {
  const int* stop = &W.st->stop;
  if (W.orth == FDIGA_ORTH_DCGS2) {
    // z = B u_j with u_0 = v_0 (the normalised residual) and u_j (j >= 1) in W.u; the first pass B reads
    // u_0 from V row 0 and writes q_0 over it and u_1 into W.u
    for (int j = 0; j < m; ++j) {
      const double* u = j == 0 ? W.V : W.u;
      if (P) {
        prof_mark(ctx, PROF_FD);
        FDIGA_TRY(fd_apply_ex(P, u, W.z, stop));
        prof_mark(ctx, PROF_MATVEC);
        FDIGA_TRY(stencil_matvec_ex(A, W.z, W.w, stop));
      } else {
        prof_mark(ctx, PROF_MATVEC);
        FDIGA_TRY(stencil_matvec_ex(A, u, W.w, stop));
      }
      prof_mark(ctx, PROF_ORTH);
      FDIGA_TRY(launch_dcgs(ctx, W, j, u, m, hist_cap, false));
    }
    return launch_dcgs(ctx, W, m, m == 0 ? W.V : W.u, m, hist_cap, true);
  }
  for (int j = 0; j < m; ++j) {
    double* vj = W.V + (int64_t)j * W.ldv;
    if (P) {
      prof_mark(ctx, PROF_FD);
      FDIGA_TRY(fd_apply_ex(P, vj, W.z, stop));
      prof_mark(ctx, PROF_MATVEC);
      FDIGA_TRY(stencil_matvec_ex(A, W.z, W.w, stop));
    } else {
      prof_mark(ctx, PROF_MATVEC);
      FDIGA_TRY(stencil_matvec_ex(A, vj, W.w, stop));
    }
    prof_mark(ctx, PROF_ORTH);
    const int k = j + 1;
    FDIGA_TRY(launch_passes(ctx, W, k, j, m, hist_cap));
    if (W.orth != FDIGA_ORTH_CGS2) {  // CGS2's pass 3 already wrote v_{j+1}
      next_basis_kernel<<<W.nblk, RT, 0, ctx->stream>>>(W.w, W.V + (int64_t)(j + 1) * W.ldv, W.N, W.st);
      count_launch(ctx);
    }
    FDIGA_CUDA(cudaGetLastError());
  }
  return FDIGA_OK;
}

}  // namespace

// Cached captured cycle (per context), valid for one (A, P, m, N, workspace) combination.
struct GmresGraph {
  fdiga_stencil* A = nullptr;
  fd_plan* P = nullptr;
  int m = 0, hist_cap = 0, orth = 0;
  int64_t N = 0;
  double* V = nullptr;
  double* hist = nullptr;
  double *z = nullptr, *part = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap_stream = nullptr;
};

namespace fdiga {
void destroy_gmres_graph(fdiga_ctx* ctx) {
  destroy_bicgstab_graph(ctx);
  GmresGraph* G = static_cast<GmresGraph*>(ctx->gmres_graph);
  if (!G) return;
  if (G->exec) cudaGraphExecDestroy(G->exec);
  if (G->cap_stream) cudaStreamDestroy(G->cap_stream);
  delete G;
  ctx->gmres_graph = nullptr;
}
}  // namespace fdiga

extern "C" int gmres_solve(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const double* b, double* x,
                           const gmres_opts* opts, gmres_report* rep) {
  FDIGA_CHECK(ctx && A && ((b && x) || stencil_local_rows(A) == 0), FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_TRY(bind(ctx));
  NvtxSolveScope nvtx_(ctx, "fdiga:gmres_solve");
  const int m = opts ? opts->m : 30;
  const double rtol = opts ? opts->rtol : 1e-8;
  const int max_iters = opts ? opts->max_iters : 1000;
  const int use_x0 = opts ? opts->use_x0 : 0;
  FDIGA_CHECK(m >= 1 && m <= KMAX - 1, FDIGA_ERR_INVALID_ARG, "restart length m = %d must be in [1, %d]", m, KMAX - 1);
  FDIGA_CHECK(max_iters >= 1, FDIGA_ERR_INVALID_ARG, "max_iters must be >= 1");
  int64_t nnz = 0, nd[3] = {1, 1, 1};
  FDIGA_TRY(stencil_info(A, &nnz, nd, nullptr, nullptr));
  Ws W;
  W.N = stencil_local_rows(A);
  W.sh = ctx->sharded;
  W.orth = opts ? opts->orth : FDIGA_ORTH_DCGS2;
  FDIGA_CHECK(W.orth == FDIGA_ORTH_CGS_DGKS || W.orth == FDIGA_ORTH_CGS2 || W.orth == FDIGA_ORTH_DCGS2,
              FDIGA_ERR_INVALID_ARG, "unknown orth %d", W.orth);
  const bool profile = opts && opts->profile;
  const bool use_graph = comm_capturable(ctx) && !profile;
  FDIGA_CHECK(!P || fd_plan_local_size(P) == W.N, FDIGA_ERR_INVALID_ARG,
              "preconditioner and operator sizes differ (%lld vs %lld local rows)",
              (long long)(P ? fd_plan_local_size(P) : 0), (long long)W.N);
  W.ldv = (W.N + 63) & ~int64_t(63);  // 512-byte aligned basis vectors
  W.nblk = (int)std::max<int64_t>(1, std::min<int64_t>((W.N + RT - 1) / RT, 4 * ctx->sm_count));
  const int hist_cap = std::max(max_iters, 1);
  const size_t st_doubles = (sizeof(GmState) + 7) / 8;
  FDIGA_TRY(ctx->ws[0].ensure((size_t)(m + 1) * W.ldv));
  FDIGA_TRY(ctx->ws[1].ensure((size_t)3 * W.ldv));
  FDIGA_TRY(ctx->ws[2].ensure((size_t)std::max(W.nblk, 8 * ctx->sm_count) * (2 * KMAX + 2)));
  FDIGA_TRY(ctx->ws[3].ensure(st_doubles + hist_cap));
  W.V = ctx->ws[0].p;
  W.z = ctx->ws[1].p;
  W.w = ctx->ws[1].p + W.ldv;
  W.u = ctx->ws[1].p + 2 * W.ldv;
  W.part = ctx->ws[2].p;
  W.st = reinterpret_cast<GmState*>(ctx->ws[3].p);
  W.hist = ctx->ws[3].p + st_doubles;
  cudaStream_t st = ctx->stream;
  FDIGA_TRY(ensure_pinned(ctx, st_doubles + 8));

  // ---- the captured cycle (once per (A, P, m, N, workspace))
  GmresGraph* G = static_cast<GmresGraph*>(ctx->gmres_graph);
  if (G && (G->A != A || G->P != P || G->m != m || G->N != W.N || G->V != W.V || G->hist != W.hist ||
            G->hist_cap != hist_cap || G->orth != W.orth || G->z != W.z || G->part != W.part)) {
    destroy_gmres_graph(ctx);
    G = nullptr;
  }
  if (!G && use_graph) {
    G = new GmresGraph();
    ctx->gmres_graph = G;
    G->A = A;
    G->P = P;
    G->m = m;
    G->N = W.N;
    G->V = W.V;
    G->hist = W.hist;
    G->hist_cap = hist_cap;
    G->orth = W.orth;
    G->z = W.z;
    G->part = W.part;
    FDIGA_CUDA(cudaStreamCreateWithFlags(&G->cap_stream, cudaStreamNonBlocking));
    FDIGA_CUDA(cudaStreamSynchronize(st));
    cudaStream_t saved = ctx->stream;
    ctx->stream = G->cap_stream;
    int s = FDIGA_OK;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(G->cap_stream, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      s = enqueue_cycle(ctx, A, P, W, m, hist_cap);
      cudaError_t e2 = cudaStreamEndCapture(G->cap_stream, &graph);
      if (e == cudaSuccess) e = e2;
    }
    ctx->stream = saved;
    if (e == cudaSuccess && s == FDIGA_OK) e = cudaGraphInstantiate(&G->exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (s != FDIGA_OK || e != cudaSuccess) {
      destroy_gmres_graph(ctx);
      if (s != FDIGA_OK) return s;
      set_error("gmres_solve: graph capture failed: %s", cudaGetErrorString(e));
      return FDIGA_ERR_CUDA;
    }
  }

  cudaEvent_t e0, e1;
  FDIGA_CUDA(cudaEventCreate(&e0));
  FDIGA_CUDA(cudaEventCreate(&e1));
  FDIGA_CUDA(cudaEventRecord(e0, st));
  std::vector<std::pair<int, cudaEvent_t>> prof_events;
  if (profile) {
    ctx->prof = &prof_events;
    prof_mark(ctx, PROF_OTHER);
  }
  struct ProfOff {  // the context stops recording on every exit path
    fdiga_ctx* c;
    ~ProfOff() {
      c->prof = nullptr;
      c->prof_stage = PROF_OTHER;
    }
  } prof_off{ctx};
  {
    GmState init;
    std::memset(&init, 0, sizeof(init));
    init.max_iters = max_iters;
    init.first = 1;
    std::memcpy(ctx->pinned, &init, sizeof(init));
    FDIGA_CUDA(cudaMemcpyAsync(W.st, ctx->pinned, sizeof(GmState), cudaMemcpyHostToDevice, st));
  }
  if (!use_x0) FDIGA_CUDA(cudaMemsetAsync(x, 0, W.N * sizeof(double), st));

  int status = FDIGA_OK, cycles = 0;
  GmState hs;
  std::memset(&hs, 0, sizeof(hs));
  while (true) {
    // true residual r = b - A x, cycle start (device decides whether to stop)
    prof_mark(ctx, PROF_MATVEC);
    FDIGA_TRY(stencil_matvec(A, x, W.w));
    prof_mark(ctx, PROF_OTHER);
    residual_start_kernel<<<W.nblk, RT, 0, st>>>(b, W.w, W.V, W.N, W.part, W.st, rtol, W.sh ? 0 : 1);
    if (W.sh) {
      FDIGA_TRY(comm_allreduce(ctx, W.st->rsl, W.st->rs, 2));
      begin_cycle_kernel<<<1, 1, 0, st>>>(W.st, rtol);
      count_launch(ctx);
    }
    scale_start_kernel<<<W.nblk, RT, 0, st>>>(W.V, W.N, W.st);
    count_launch(ctx, 2);
    FDIGA_CUDA(cudaGetLastError());
    FDIGA_CUDA(cudaMemcpyAsync(ctx->pinned, W.st, sizeof(GmState), cudaMemcpyDeviceToHost, st));
    FDIGA_CUDA(cudaStreamSynchronize(st));
    std::memcpy(&hs, ctx->pinned, sizeof(GmState));
    if (hs.breakdown) {
      status = FDIGA_ERR_BREAKDOWN;
      set_error("gmres_solve: non-finite value after %d iterations", hs.iters);
      break;
    }
    if (hs.beta <= hs.target || hs.bnorm == 0.0) break;  // converged on the true residual
    if (hs.iters >= max_iters) {
      status = FDIGA_ERR_NOT_CONVERGED;
      set_error("gmres_solve: %d iterations without convergence", hs.iters);
      break;
    }
    ++cycles;
    // one cycle: the captured Arnoldi steps, then x += P^{-1}(V y)
    if (G && !profile) {  // (a profiled solve enqueues its cycles eagerly, with stage events)
      FDIGA_CUDA(cudaGraphLaunch(G->exec, st));
      count_launch(ctx, 1);
    } else {
      FDIGA_TRY(enqueue_cycle(ctx, A, P, W, m, hist_cap));  // loopback transport: not capturable
    }
    prof_mark(ctx, PROF_ORTH);
    solve_y_kernel<<<1, 1, 0, st>>>(W.st);
    count_launch(ctx);
    // the cycle's basis size k is decided on the device: read it (one small copy per cycle) so the
    // combination x += P^{-1}(V y) streams exactly k rows with the TMA-fed kernel
    FDIGA_CUDA(cudaMemcpyAsync(ctx->pinned, &W.st->k, sizeof(int), cudaMemcpyDeviceToHost, st));
    FDIGA_CUDA(cudaStreamSynchronize(st));
    int kcyc = 0;
    std::memcpy(&kcyc, ctx->pinned, sizeof(int));
    FDIGA_TRY(launch_lincomb(ctx, W, kcyc, W.w));
    FDIGA_CUDA(cudaGetLastError());
    if (P) {
      prof_mark(ctx, PROF_FD);
      FDIGA_TRY(fd_apply(P, W.w, W.z));
      prof_mark(ctx, PROF_OTHER);
      axpy_kernel<<<W.nblk, RT, 0, st>>>(W.z, x, W.N);
    } else {
      prof_mark(ctx, PROF_OTHER);
      axpy_kernel<<<W.nblk, RT, 0, st>>>(W.w, x, W.N);
    }
    count_launch(ctx, 1);
    FDIGA_CUDA(cudaGetLastError());
  }
  FDIGA_CUDA(cudaEventRecord(e1, st));
  FDIGA_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // per-stage times: interval [e_i, e_{i+1}) (the last one up to e1) charged to stage i; the state upload
  // before the first mark is OTHER
  double stage_ms[PROF_NSTAGE] = {0, 0, 0, 0, 0};
  if (!prof_events.empty()) {
    float d = 0;
    if (cudaEventElapsedTime(&d, e0, prof_events[0].second) == cudaSuccess) stage_ms[PROF_OTHER] += d;
  }
  for (size_t i = 0; i < prof_events.size(); ++i) {
    float d = 0;
    if (cudaEventElapsedTime(&d, prof_events[i].second,
                             i + 1 < prof_events.size() ? prof_events[i + 1].second : e1) == cudaSuccess)
      stage_ms[prof_events[i].first] += d;
  }
  for (auto& pe : prof_events) cudaEventDestroy(pe.second);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->iters = hs.iters;
    rep->restarts = cycles;
    rep->converged = (status == FDIGA_OK) ? 1 : 0;
    rep->reorth = W.orth != FDIGA_ORTH_CGS_DGKS ? hs.iters : hs.nreorth;  // second Gram-Schmidt passes
    rep->rel_res_true = hs.rel_true;
    rep->rel_res_implicit = hs.rel_implicit;
    rep->t_total_ms = ms;
    rep->t_fd_ms = profile ? stage_ms[PROF_FD] : -1.0;
    rep->t_matvec_ms = profile ? stage_ms[PROF_MATVEC] : -1.0;
    rep->t_orth_ms = profile ? stage_ms[PROF_ORTH] : -1.0;
    rep->t_comm_ms = profile ? stage_ms[PROF_COMM] : -1.0;
    rep->t_other_ms = profile ? stage_ms[PROF_OTHER] : -1.0;
    if (rep->history && rep->history_cap > 0) {
      const int cnt = std::min(rep->history_cap, std::min(hs.iters, hist_cap));
      if (cnt > 0) FDIGA_CUDA(cudaMemcpy(rep->history, W.hist, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
  return status;
}
