// Right-preconditioned BiCGStab (van der Vorst 1992), the paper's Krylov solver, with the
// paper's half-iteration accounting (reading 15), device resident.
//
// Iteration k (1-based), r^ = r_0 the shadow residual:
//   p   = r + beta (p - omega v)        beta = (rho / rho_prev)(alpha / omega); p = r when k = 1
//   p^  = P^{-1} p   (fd_apply)         v = A p^ (stencil matvec)
//   alpha = rho / (r^ . v)                                           [reduction 1]
//   s   = r - alpha v (in place of r);  x += alpha p^;  ||s||         [reduction 2, BiCG half step test]
//   s^  = P^{-1} s;  t = A s^
//   omega = (t . s) / (t . t)                                         [reduction 3]
//   x  += omega s^;  r = s - omega t;  ||r||, r^ . r (next rho)      [reduction 4, full step test]
// Every reduction ends in a deterministic "last block" (reduce.cuh) that takes the scalar decision on
// the device (single rank), or, when sharded, leaves its partial sums for an all-reduce followed by a
// one-thread decision kernel.  A decided stop turns every later launch into a no-op (device flag), so
// chunks of iterations are captured once in a CUDA graph and the host syncs once per chunk.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "reduce.cuh"

using namespace fdiga;

namespace {

constexpr int CHUNK = 8;  // iterations per captured graph

struct BcState {
  double rho, rho_prev, alpha, omega;
  double bnorm, target, rel_rec, rel_true, iters;
  double loc[4], glob[4];  // reduction results (local partials; all-reduced when sharded)
  int stop, converged, breakdown, half, k, max_iters, hist_cap, pad;
  unsigned int counter[5];
  double* hist;  // recursive relative residual after every half step (device, hist_cap entries)
};

struct BcVecs {
  int64_t N;
  int nblk;
  bool sh;
  double *r, *rhat, *p, *v, *phat, *shat, *t, *x, *part, *hist;
  const double* b;
  BcState* st;
};

// ---- one-thread decisions (called by the last block, or by decide_kernel after the all-reduce)
__device__ void decide_start(BcState* st, const double* g, double rtol) {
  const double rr = g[0], bb = g[1];
  st->bnorm = sqrt(bb);
  st->target = rtol * st->bnorm;
  st->rho = rr;  // r^ = r_0
  st->rho_prev = st->alpha = st->omega = 1.0;
  st->k = 1;
  st->iters = 0.0;
  st->rel_rec = st->bnorm > 0 ? sqrt(rr) / st->bnorm : 0.0;
  if (!isfinite(rr)) st->breakdown = 1;
  if (sqrt(rr) <= st->target || st->bnorm == 0.0) st->converged = 1;
  if (st->converged || st->breakdown || st->max_iters < 1) st->stop = 1;
}

__device__ void decide_alpha(BcState* st, const double* g) {
  const double sigma = g[0];
  if (sigma == 0.0 || !isfinite(sigma)) {
    st->breakdown = 1;
    st->stop = 1;
    return;
  }
  st->alpha = st->rho / sigma;
}

__device__ void decide_half(BcState* st, const double* g) {
  const double sn = sqrt(g[0]);
  st->rel_rec = sn / st->bnorm;
  const int h = 2 * (st->k - 1);
  if (st->hist_cap > h) st->hist[h] = st->rel_rec;
  if (!isfinite(sn)) {
    st->breakdown = 1;
    st->stop = 1;
  } else if (sn <= st->target) {  // converged after the BiCG half step: k - 0.5
    st->iters = st->k - 0.5;
    st->half = 1;
    st->converged = 1;
    st->stop = 1;
  }
}

__device__ void decide_omega(BcState* st, const double* g) {
  const double ts = g[0], tt = g[1];
  if (tt == 0.0 || !isfinite(tt)) {
    st->breakdown = 1;
    st->stop = 1;
    return;
  }
  st->omega = ts / tt;
}

__device__ void decide_full(BcState* st, const double* g) {
  const double rn = sqrt(g[0]), rho_new = g[1];
  st->rel_rec = rn / st->bnorm;
  st->iters = st->k;
  const int h = 2 * (st->k - 1) + 1;
  if (st->hist_cap > h) st->hist[h] = st->rel_rec;
  if (!isfinite(rn)) {
    st->breakdown = 1;
    st->stop = 1;
  } else if (rn <= st->target) {
    st->converged = 1;
    st->stop = 1;
  } else if (st->omega == 0.0 || rho_new == 0.0) {
    st->breakdown = 1;
    st->stop = 1;
  } else {
    st->rho_prev = st->rho;
    st->rho = rho_new;
    st->k += 1;
    if (st->k > st->max_iters) st->stop = 1;
  }
}

enum Stage { START = 0, ALPHA = 1, HALF = 2, OMEGA = 3, FULL = 4 };

__device__ void decide(BcState* st, int stage, const double* g, double rtol) {
  switch (stage) {
    case START: decide_start(st, g, rtol); break;
    case ALPHA: decide_alpha(st, g); break;
    case HALF: decide_half(st, g); break;
    case OMEGA: decide_omega(st, g); break;
    default: decide_full(st, g); break;
  }
}

// finish a reduction: the last block decides (single rank) or stores the partial sums (sharded)
template <int CNT>
__device__ __forceinline__ void finish(double (&acc)[CNT], double* part, BcState* st, int stage, int close,
                                       double rtol) {
  __shared__ double out[CNT];
  if (reduce_last<CNT>(acc, CNT, part, &st->counter[stage], out) && threadIdx.x == 0) {
    if (close)
      decide(st, stage, out, rtol);
    else
      for (int i = 0; i < CNT; ++i) st->loc[i] = out[i];
  }
}

__global__ void decide_kernel(BcState* st, int stage, double rtol, int check_stop) {
  if (check_stop && st->stop) return;
  decide(st, stage, st->glob, rtol);
}

#define BC_LOOP(e) for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT)

// r = b - A x (Ax in r on entry), r^ = r; ||r||^2, ||b||^2
__global__ void __launch_bounds__(RT) bc_start_kernel(const double* __restrict__ b, double* __restrict__ r,
                                                      double* __restrict__ rhat, int64_t N, double* part, BcState* st,
                                                      int close, double rtol) {
  double acc[2] = {0.0, 0.0};
  BC_LOOP(e) {
    const double bv = b[e], v = bv - r[e];
    r[e] = v;
    rhat[e] = v;
    acc[0] = fma(v, v, acc[0]);
    acc[1] = fma(bv, bv, acc[1]);
  }
  finish<2>(acc, part, st, START, close, rtol);
}

// p = r (k = 1) or r + beta (p - omega v)
__global__ void __launch_bounds__(RT) bc_p_kernel(const double* __restrict__ r, double* __restrict__ p,
                                                  const double* __restrict__ v, int64_t N, const BcState* st) {
  if (st->stop) return;
  if (st->k == 1) {
    BC_LOOP(e) p[e] = r[e];
    return;
  }
  const double beta = (st->rho / st->rho_prev) * (st->alpha / st->omega), om = st->omega;
  BC_LOOP(e) p[e] = fma(beta, fma(-om, v[e], p[e]), r[e]);
}

// sigma = r^ . v
__global__ void __launch_bounds__(RT) bc_sigma_kernel(const double* __restrict__ rhat, const double* __restrict__ v,
                                                      int64_t N, double* part, BcState* st, int close) {
  if (st->stop) return;
  double acc[1] = {0.0};
  BC_LOOP(e) acc[0] = fma(rhat[e], v[e], acc[0]);
  finish<1>(acc, part, st, ALPHA, close, 0.0);
}

// s = r - alpha v (in r); x += alpha p^; ||s||^2
__global__ void __launch_bounds__(RT) bc_s_kernel(double* __restrict__ r, const double* __restrict__ v,
                                                  double* __restrict__ x, const double* __restrict__ phat, int64_t N,
                                                  double* part, BcState* st, int close) {
  if (st->stop) return;
  const double al = st->alpha;
  double acc[1] = {0.0};
  BC_LOOP(e) {
    const double s = fma(-al, v[e], r[e]);
    r[e] = s;
    x[e] = fma(al, phat[e], x[e]);
    acc[0] = fma(s, s, acc[0]);
  }
  finish<1>(acc, part, st, HALF, close, 0.0);
}

// t . s, t . t
__global__ void __launch_bounds__(RT) bc_ts_kernel(const double* __restrict__ t, const double* __restrict__ s,
                                                   int64_t N, double* part, BcState* st, int close) {
  if (st->stop) return;
  double acc[2] = {0.0, 0.0};
  BC_LOOP(e) {
    const double tv = t[e];
    acc[0] = fma(tv, s[e], acc[0]);
    acc[1] = fma(tv, tv, acc[1]);
  }
  finish<2>(acc, part, st, OMEGA, close, 0.0);
}

// x += omega s^; r = s - omega t (in r); ||r||^2, r^ . r
__global__ void __launch_bounds__(RT) bc_xr_kernel(double* __restrict__ x, const double* __restrict__ shat,
                                                   double* __restrict__ r, const double* __restrict__ t,
                                                   const double* __restrict__ rhat, int64_t N, double* part,
                                                   BcState* st, int close) {
  if (st->stop) return;
  const double om = st->omega;
  double acc[2] = {0.0, 0.0};
  BC_LOOP(e) {
    x[e] = fma(om, shat[e], x[e]);
    const double rv = fma(-om, t[e], r[e]);
    r[e] = rv;
    acc[0] = fma(rv, rv, acc[0]);
    acc[1] = fma(rhat[e], rv, acc[1]);
  }
  finish<2>(acc, part, st, FULL, close, 0.0);
}

// ||b - A x||^2 (Ax in t) -> loc[0] / rel_true
__global__ void __launch_bounds__(RT) bc_true_kernel(const double* __restrict__ b, const double* __restrict__ ax,
                                                     int64_t N, double* part, BcState* st) {
  double acc[1] = {0.0};
  BC_LOOP(e) {
    const double d = b[e] - ax[e];
    acc[0] = fma(d, d, acc[0]);
  }
  __shared__ double out[1];
  if (reduce_last<1>(acc, 1, part, &st->counter[0], out) && threadIdx.x == 0) st->loc[0] = out[0];
}

__global__ void bc_true_finish_kernel(BcState* st, int sharded) {
  const double v = sharded ? st->glob[0] : st->loc[0];
  st->rel_true = st->bnorm > 0 ? sqrt(v) / st->bnorm : 0.0;
}

// all-reduce the partials and decide (sharded only)
int reduce_decide(fdiga_ctx* ctx, const BcVecs& W, int stage, int cnt, double rtol, int check_stop) {
  if (!W.sh) return FDIGA_OK;
  FDIGA_TRY(comm_allreduce(ctx, W.st->loc, W.st->glob, cnt));
  decide_kernel<<<1, 1, 0, ctx->stream>>>(W.st, stage, rtol, check_stop);
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

// enqueue `iters` BiCGStab iterations on ctx->stream
int enqueue_iters(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const BcVecs& W, int iters) {
  const int* stop = &W.st->stop;
  const int close = W.sh ? 0 : 1;
  cudaStream_t s = ctx->stream;
  for (int it = 0; it < iters; ++it) {
    bc_p_kernel<<<W.nblk, RT, 0, s>>>(W.r, W.p, W.v, W.N, W.st);
    count_launch(ctx);
    const double* pin = W.p;
    if (P) {
      FDIGA_TRY(fd_apply_ex(P, W.p, W.phat, stop));
      pin = W.phat;
    }
    FDIGA_TRY(stencil_matvec_ex(A, pin, W.v, stop));
    bc_sigma_kernel<<<W.nblk, RT, 0, s>>>(W.rhat, W.v, W.N, W.part, W.st, close);
    count_launch(ctx);
    FDIGA_TRY(reduce_decide(ctx, W, ALPHA, 1, 0.0, 1));
    bc_s_kernel<<<W.nblk, RT, 0, s>>>(W.r, W.v, W.x, pin, W.N, W.part, W.st, close);
    count_launch(ctx);
    FDIGA_TRY(reduce_decide(ctx, W, HALF, 1, 0.0, 1));
    const double* sin_ = W.r;
    if (P) {
      FDIGA_TRY(fd_apply_ex(P, W.r, W.shat, stop));
      sin_ = W.shat;
    }
    FDIGA_TRY(stencil_matvec_ex(A, sin_, W.t, stop));
    bc_ts_kernel<<<W.nblk, RT, 0, s>>>(W.t, W.r, W.N, W.part, W.st, close);
    count_launch(ctx);
    FDIGA_TRY(reduce_decide(ctx, W, OMEGA, 2, 0.0, 1));
    bc_xr_kernel<<<W.nblk, RT, 0, s>>>(W.x, sin_, W.r, W.t, W.rhat, W.N, W.part, W.st, close);
    count_launch(ctx);
    FDIGA_TRY(reduce_decide(ctx, W, FULL, 2, 0.0, 1));
    FDIGA_CUDA(cudaGetLastError());
  }
  return FDIGA_OK;
}

}  // namespace

struct BicgGraph {
  fdiga_stencil* A = nullptr;
  fd_plan* P = nullptr;
  int64_t N = 0;
  double* base = nullptr;
  double* x = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap_stream = nullptr;
};

namespace fdiga {
void destroy_bicgstab_graph(fdiga_ctx* ctx) {
  BicgGraph* G = static_cast<BicgGraph*>(ctx->bicg_graph);
  if (!G) return;
  if (G->exec) cudaGraphExecDestroy(G->exec);
  if (G->cap_stream) cudaStreamDestroy(G->cap_stream);
  delete G;
  ctx->bicg_graph = nullptr;
}
}  // namespace fdiga

extern "C" int bicgstab_solve(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const double* b, double* x,
                              const bicgstab_opts* opts, bicgstab_report* rep) {
  FDIGA_CHECK(ctx && A && ((b && x) || stencil_local_rows(A) == 0), FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_TRY(bind(ctx));
  NvtxSolveScope nvtx_(ctx, "fdiga:bicgstab_solve");
  const double rtol = opts ? opts->rtol : 1e-8;
  const int max_iters = opts ? opts->max_iters : 1000;
  const int use_x0 = opts ? opts->use_x0 : 0;
  FDIGA_CHECK(max_iters >= 1 && rtol > 0, FDIGA_ERR_INVALID_ARG, "bad bicgstab options");
  BcVecs W;
  W.N = stencil_local_rows(A);
  W.sh = ctx->sharded;
  FDIGA_CHECK(!P || fd_plan_local_size(P) == W.N, FDIGA_ERR_INVALID_ARG,
              "preconditioner and operator sizes differ");
  const int64_t ld = (W.N + 63) & ~int64_t(63);
  W.nblk = (int)std::max<int64_t>(1, std::min<int64_t>((W.N + RT - 1) / RT, 4 * ctx->sm_count));
  const int hist_cap = 2 * max_iters;
  const size_t st_doubles = (sizeof(BcState) + 7) / 8;
  FDIGA_TRY(ctx->ws[0].ensure((size_t)7 * ld + 1));
  FDIGA_TRY(ctx->ws[2].ensure((size_t)W.nblk * 4));
  FDIGA_TRY(ctx->ws[3].ensure(st_doubles + hist_cap));
  double* base = ctx->ws[0].p;
  W.r = base;
  W.rhat = base + ld;
  W.p = base + 2 * ld;
  W.v = base + 3 * ld;
  W.phat = base + 4 * ld;
  W.shat = base + 5 * ld;
  W.t = base + 6 * ld;
  W.x = x;
  W.b = b;
  W.part = ctx->ws[2].p;
  W.st = reinterpret_cast<BcState*>(ctx->ws[3].p);
  W.hist = ctx->ws[3].p + st_doubles;
  cudaStream_t st = ctx->stream;
  FDIGA_TRY(ensure_pinned(ctx, st_doubles + 8));
  const bool use_graph = comm_capturable(ctx);

  BicgGraph* G = static_cast<BicgGraph*>(ctx->bicg_graph);
  if (G && (G->A != A || G->P != P || G->N != W.N || G->base != base || G->x != x)) {
    destroy_bicgstab_graph(ctx);
    G = nullptr;
  }
  if (!G && use_graph) {
    G = new BicgGraph();
    ctx->bicg_graph = G;
    G->A = A;
    G->P = P;
    G->N = W.N;
    G->base = base;
    G->x = x;
    FDIGA_CUDA(cudaStreamCreateWithFlags(&G->cap_stream, cudaStreamNonBlocking));
    FDIGA_CUDA(cudaStreamSynchronize(st));
    cudaStream_t saved = ctx->stream;
    ctx->stream = G->cap_stream;
    int s = FDIGA_OK;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(G->cap_stream, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      s = enqueue_iters(ctx, A, P, W, CHUNK);
      cudaError_t e2 = cudaStreamEndCapture(G->cap_stream, &graph);
      if (e == cudaSuccess) e = e2;
    }
    ctx->stream = saved;
    if (e == cudaSuccess && s == FDIGA_OK) e = cudaGraphInstantiate(&G->exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (s != FDIGA_OK || e != cudaSuccess) {
      destroy_bicgstab_graph(ctx);
      if (s != FDIGA_OK) return s;
      set_error("bicgstab_solve: graph capture failed: %s", cudaGetErrorString(e));
      return FDIGA_ERR_CUDA;
    }
  }

  cudaEvent_t e0, e1;
  FDIGA_CUDA(cudaEventCreate(&e0));
  FDIGA_CUDA(cudaEventCreate(&e1));
  FDIGA_CUDA(cudaEventRecord(e0, st));
  {
    BcState init;
    std::memset(&init, 0, sizeof(init));
    init.max_iters = max_iters;
    init.hist_cap = hist_cap;
    init.hist = W.hist;
    std::memcpy(ctx->pinned, &init, sizeof(init));
    FDIGA_CUDA(cudaMemcpyAsync(W.st, ctx->pinned, sizeof(BcState), cudaMemcpyHostToDevice, st));
  }
  if (!use_x0 && W.N) FDIGA_CUDA(cudaMemsetAsync(x, 0, W.N * sizeof(double), st));
  // r = b - A x, r^ = r, rho = ||r||^2
  FDIGA_TRY(stencil_matvec(A, x, W.r));
  bc_start_kernel<<<W.nblk, RT, 0, st>>>(b, W.r, W.rhat, W.N, W.part, W.st, W.sh ? 0 : 1, rtol);
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  FDIGA_TRY(reduce_decide(ctx, W, START, 2, rtol, 0));
  // p starts at r; v at 0 (beta is not used at k = 1, but keep v finite)
  if (W.N) FDIGA_CUDA(cudaMemsetAsync(W.v, 0, W.N * sizeof(double), st));
  BcState hs;
  std::memset(&hs, 0, sizeof(hs));
  int done_iters = 0;
  while (true) {
    FDIGA_CUDA(cudaMemcpyAsync(ctx->pinned, W.st, sizeof(BcState), cudaMemcpyDeviceToHost, st));
    FDIGA_CUDA(cudaStreamSynchronize(st));
    std::memcpy(&hs, ctx->pinned, sizeof(BcState));
    if (hs.stop) break;
    if (G) {
      FDIGA_CUDA(cudaGraphLaunch(G->exec, st));
      count_launch(ctx);
    } else {
      FDIGA_TRY(enqueue_iters(ctx, A, P, W, CHUNK));
    }
    done_iters += CHUNK;
    if (done_iters > max_iters + CHUNK) break;  // safety net (the device flag stops earlier)
  }
  // true residual ||b - A x|| / ||b||
  FDIGA_TRY(stencil_matvec(A, x, W.t));
  bc_true_kernel<<<W.nblk, RT, 0, st>>>(b, W.t, W.N, W.part, W.st);
  count_launch(ctx);
  if (W.sh) FDIGA_TRY(comm_allreduce(ctx, W.st->loc, W.st->glob, 1));
  bc_true_finish_kernel<<<1, 1, 0, st>>>(W.st, W.sh ? 1 : 0);
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  FDIGA_CUDA(cudaEventRecord(e1, st));
  FDIGA_CUDA(cudaMemcpyAsync(ctx->pinned, W.st, sizeof(BcState), cudaMemcpyDeviceToHost, st));
  FDIGA_CUDA(cudaEventSynchronize(e1));
  FDIGA_CUDA(cudaStreamSynchronize(st));
  std::memcpy(&hs, ctx->pinned, sizeof(BcState));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  int status = FDIGA_OK;
  if (hs.breakdown) {
    status = FDIGA_ERR_BREAKDOWN;
    set_error("bicgstab_solve: breakdown (rho, r^.v or t.t vanished, or a non-finite value) after %.1f iterations",
              hs.iters);
  } else if (!hs.converged) {
    status = FDIGA_ERR_NOT_CONVERGED;
    set_error("bicgstab_solve: %d iterations without convergence", max_iters);
  }
  if (rep) {
    rep->iters = hs.iters;
    rep->converged = hs.converged;
    rep->breakdown = hs.breakdown;
    rep->half = hs.half;
    rep->rel_res_true = hs.rel_true;
    rep->rel_res_recursive = hs.rel_rec;
    rep->t_total_ms = ms;
    if (rep->history && rep->history_cap > 0) {
      const int cnt = std::min(rep->history_cap, std::min(hist_cap, (int)std::lround(2 * hs.iters)));
      if (cnt > 0) FDIGA_CUDA(cudaMemcpy(rep->history, W.hist, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
  return status;
}
