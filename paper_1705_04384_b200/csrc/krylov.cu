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
  unsigned int counter[NCNT];
};

// Element loops of the three passes: each thread handles pairs of elements with 16-byte loads (V rows
// and w are 512-byte aligned, ldv even); a scalar tail covers odd N.
#define FDIGA_PAIRS(e2) for (int64_t e2 = blockIdx.x * (int64_t)RT + threadIdx.x; e2 < (N >> 1); e2 += (int64_t)gridDim.x * RT)
#define FDIGA_TAIL(e) for (int64_t e = (N & ~int64_t(1)) + blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT)

// pass 1: h1[i] = V_i . w (i < k), h1[k] = w . w
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass1(const double* __restrict__ V, int64_t ldv, int /*k (= K)*/,
                                                    const double* __restrict__ w, int64_t N, double* part,
                                                    GmState* st, double* hout) {
  constexpr int k = K;
  if (st->stop) return;
  double acc[KMAX + 1];
#pragma unroll
  for (int i = 0; i <= KMAX; ++i) acc[i] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  FDIGA_PAIRS(e2) {
    const double2 wv = w2[e2];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) {
        const double2 v = reinterpret_cast<const double2*>(V + i * ldv)[e2];
        acc[i] = fma(v.x, wv.x, fma(v.y, wv.y, acc[i]));
      }
    acc[KMAX] = fma(wv.x, wv.x, fma(wv.y, wv.y, acc[KMAX]));
  }
  FDIGA_TAIL(e) {
    const double wv = w[e];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) acc[i] = fma(V[i * ldv + e], wv, acc[i]);
    acc[KMAX] = fma(wv, wv, acc[KMAX]);
  }
#pragma unroll
  for (int i = 0; i < KMAX; ++i)
    if (i == k) acc[i] = acc[KMAX];  // w.w to slot k (static register indexing)
  reduce_last<KMAX + 1>(acc, k + 1, part, &st->counter[0], hout);
}

// pass 2: w <- w - V h1 ; h2[i] = V_i . w (new w), h2[k] = ||w||^2.  V_i is read twice per element
// pair; the second read hits L1 (the block's working set is <= 256 threads x 32 x 16 B).
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass2(const double* __restrict__ V, int64_t ldv, int /*k (= K)*/,
                                                    double* __restrict__ w, int64_t N, double* part, GmState* st,
                                                    double* hout) {
  constexpr int k = K;
  if (st->stop) return;
  __shared__ double hs[KMAX];
  if (threadIdx.x < k) hs[threadIdx.x] = st->h1[threadIdx.x];
  __syncthreads();
  double acc[KMAX + 1];
#pragma unroll
  for (int i = 0; i <= KMAX; ++i) acc[i] = 0.0;
  double2* w2 = reinterpret_cast<double2*>(w);
  FDIGA_PAIRS(e2) {
    double2 wv = w2[e2];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(V + i * ldv) + e2);
        wv.x = fma(-hs[i], v.x, wv.x);
        wv.y = fma(-hs[i], v.y, wv.y);
      }
    w2[e2] = wv;
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(V + i * ldv) + e2);
        acc[i] = fma(v.x, wv.x, fma(v.y, wv.y, acc[i]));
      }
    acc[KMAX] = fma(wv.x, wv.x, fma(wv.y, wv.y, acc[KMAX]));
  }
  FDIGA_TAIL(e) {
    double wv = w[e];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) wv = fma(-hs[i], V[i * ldv + e], wv);
    w[e] = wv;
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) acc[i] = fma(V[i * ldv + e], wv, acc[i]);
    acc[KMAX] = fma(wv, wv, acc[KMAX]);
  }
#pragma unroll
  for (int i = 0; i < KMAX; ++i)
    if (i == k) acc[i] = acc[KMAX];
  reduce_last<KMAX + 1>(acc, k + 1, part, &st->counter[1], hout);
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
  st->rel_implicit = fabs(st->g[k]) / st->bnorm;
  if (hist && st->iters - 1 < hist_cap) hist[st->iters - 1] = st->rel_implicit;
  st->invh = hn > 0.0 ? 1.0 / hn : 0.0;
  if (bad) st->breakdown = 1;
  if (bad || fabs(st->g[k]) <= st->target || hn == 0.0 || st->iters >= st->max_iters || k >= m) st->stop = 1;
}

// pass 3: w <- w - V h2 ; ||w||^2 ; the last block closes the step
template <int K>
__global__ void __launch_bounds__(RT) arnoldi_pass3(const double* __restrict__ V, int64_t ldv, int /*k (= K)*/,
                                                    double* __restrict__ w, int64_t N, double* part, GmState* st,
                                                    int j, int m, double* hist, int hist_cap, int close) {
  constexpr int k = K;
  if (st->stop) return;
  __shared__ double hs[KMAX];
  if (threadIdx.x < k) hs[threadIdx.x] = st->h2[threadIdx.x];
  __syncthreads();
  double acc[1] = {0.0};
  double2* w2 = reinterpret_cast<double2*>(w);
  FDIGA_PAIRS(e2) {
    double2 wv = w2[e2];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) {
        const double2 v = reinterpret_cast<const double2*>(V + i * ldv)[e2];
        wv.x = fma(-hs[i], v.x, wv.x);
        wv.y = fma(-hs[i], v.y, wv.y);
      }
    w2[e2] = wv;
    acc[0] = fma(wv.x, wv.x, fma(wv.y, wv.y, acc[0]));
  }
  FDIGA_TAIL(e) {
    double wv = w[e];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) wv = fma(-hs[i], V[i * ldv + e], wv);
    w[e] = wv;
    acc[0] = fma(wv, wv, acc[0]);
  }
  __shared__ double nrm[1];
  if (reduce_last<1>(acc, 1, part, &st->counter[2], nrm)) {
    if (threadIdx.x == 0) {
      if (close)
        arnoldi_close_step(st, j, m, nrm[0], hist, hist_cap);
      else
        st->wn2l = nrm[0];  // sharded: all-reduced into wn2, then close_step_kernel
    }
  }
}

// sharded: close step j once ||w''||^2 is global
__global__ void close_step_kernel(GmState* st, int j, int m, double* hist, int hist_cap) {
  if (st->stop) return;
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
  double *V, *z, *w, *part, *hist;
  GmState* st;
};

template <int K>
int passes_k(fdiga_ctx* ctx, const Ws& W, int j, int m, int hist_cap) {
  GmState* st = W.st;
  arnoldi_pass1<K><<<W.nblk, RT, 0, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, W.sh ? st->h1l : st->h1);
  if (W.sh) FDIGA_TRY(comm_allreduce(ctx, st->h1l, st->h1, K + 1));
  arnoldi_pass2<K><<<W.nblk, RT, 0, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, W.sh ? st->h2l : st->h2);
  if (W.sh) FDIGA_TRY(comm_allreduce(ctx, st->h2l, st->h2, K + 1));
  arnoldi_pass3<K><<<W.nblk, RT, 0, ctx->stream>>>(W.V, W.ldv, K, W.w, W.N, W.part, st, j, m, W.hist, hist_cap,
                                                   W.sh ? 0 : 1);
  if (W.sh) {
    FDIGA_TRY(comm_allreduce(ctx, &st->wn2l, &st->wn2, 1));
    close_step_kernel<<<1, 1, 0, ctx->stream>>>(st, j, m, W.hist, hist_cap);
    count_launch(ctx);
  }
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
  for (int j = 0; j < m; ++j) {
    double* vj = W.V + (int64_t)j * W.ldv;
    if (P) {
      FDIGA_TRY(fd_apply_ex(P, vj, W.z, stop));
      FDIGA_TRY(stencil_matvec_ex(A, W.z, W.w, stop));
    } else {
      FDIGA_TRY(stencil_matvec_ex(A, vj, W.w, stop));
    }
    const int k = j + 1;
    FDIGA_TRY(launch_passes(ctx, W, k, j, m, hist_cap));
    next_basis_kernel<<<W.nblk, RT, 0, ctx->stream>>>(W.w, W.V + (int64_t)(j + 1) * W.ldv, W.N, W.st);
    count_launch(ctx, 4);
    FDIGA_CUDA(cudaGetLastError());
  }
  return FDIGA_OK;
}

}  // namespace

// Cached captured cycle (per context), valid for one (A, P, m, N, workspace) combination.
struct GmresGraph {
  fdiga_stencil* A = nullptr;
  fd_plan* P = nullptr;
  int m = 0, hist_cap = 0;
  int64_t N = 0;
  double* V = nullptr;
  double* hist = nullptr;
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
  const bool use_graph = comm_capturable(ctx);
  FDIGA_CHECK(!P || fd_plan_local_size(P) == W.N, FDIGA_ERR_INVALID_ARG,
              "preconditioner and operator sizes differ (%lld vs %lld local rows)",
              (long long)(P ? fd_plan_local_size(P) : 0), (long long)W.N);
  W.ldv = (W.N + 63) & ~int64_t(63);  // 512-byte aligned basis vectors
  W.nblk = (int)std::max<int64_t>(1, std::min<int64_t>((W.N + RT - 1) / RT, 4 * ctx->sm_count));
  const int hist_cap = std::max(max_iters, 1);
  const size_t st_doubles = (sizeof(GmState) + 7) / 8;
  FDIGA_TRY(ctx->ws[0].ensure((size_t)(m + 1) * W.ldv));
  FDIGA_TRY(ctx->ws[1].ensure((size_t)2 * W.ldv));
  FDIGA_TRY(ctx->ws[2].ensure((size_t)W.nblk * (KMAX + 1)));
  FDIGA_TRY(ctx->ws[3].ensure(st_doubles + hist_cap));
  W.V = ctx->ws[0].p;
  W.z = ctx->ws[1].p;
  W.w = ctx->ws[1].p + W.ldv;
  W.part = ctx->ws[2].p;
  W.st = reinterpret_cast<GmState*>(ctx->ws[3].p);
  W.hist = ctx->ws[3].p + st_doubles;
  cudaStream_t st = ctx->stream;
  FDIGA_TRY(ensure_pinned(ctx, st_doubles + 8));

  // ---- the captured cycle (once per (A, P, m, N, workspace))
  GmresGraph* G = static_cast<GmresGraph*>(ctx->gmres_graph);
  if (G && (G->A != A || G->P != P || G->m != m || G->N != W.N || G->V != W.V || G->hist != W.hist ||
            G->hist_cap != hist_cap)) {
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
    FDIGA_TRY(stencil_matvec(A, x, W.w));
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
    if (G) {
      FDIGA_CUDA(cudaGraphLaunch(G->exec, st));
      count_launch(ctx, 1);
    } else {
      FDIGA_TRY(enqueue_cycle(ctx, A, P, W, m, hist_cap));  // loopback transport: not capturable
    }
    solve_y_kernel<<<1, 1, 0, st>>>(W.st);
    lincomb_kernel<<<W.nblk, RT, 0, st>>>(W.V, W.ldv, W.w, W.N, W.st);
    count_launch(ctx, 2);
    FDIGA_CUDA(cudaGetLastError());
    if (P) {
      FDIGA_TRY(fd_apply(P, W.w, W.z));
      axpy_kernel<<<W.nblk, RT, 0, st>>>(W.z, x, W.N);
    } else {
      axpy_kernel<<<W.nblk, RT, 0, st>>>(W.w, x, W.N);
    }
    count_launch(ctx, 1);
    FDIGA_CUDA(cudaGetLastError());
  }
  FDIGA_CUDA(cudaEventRecord(e1, st));
  FDIGA_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->iters = hs.iters;
    rep->restarts = cycles;
    rep->converged = (status == FDIGA_OK) ? 1 : 0;
    rep->reorth = hs.iters;  // CGS2: every step re-orthogonalises
    rep->rel_res_true = hs.rel_true;
    rep->rel_res_implicit = hs.rel_implicit;
    rep->t_total_ms = ms;
    if (rep->history && rep->history_cap > 0) {
      const int cnt = std::min(rep->history_cap, std::min(hs.iters, hist_cap));
      if (cnt > 0) FDIGA_CUDA(cudaMemcpy(rep->history, W.hist, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
  return status;
}
