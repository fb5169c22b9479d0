// Right-preconditioned restarted GMRES(m) (Saad & Schultz 1986) driven from the host,
// with every vector operation in device kernels:
//   Arnoldi step j:  z = P^{-1} v_j (fd_apply),  w = A z (stencil_matvec),
//                    [h_0..h_j, w.w] = V_{0..j}^T w, w.w  (one fused multi-dot pass, warp-shuffle trees)
//                    w <- w - V h  fused with ||w||^2     (one pass)
//                    DGKS: repeat both when ||w'|| < ||w|| / sqrt(2)
//                    Givens rotations and the convergence test on the host (O(j) scalars),
//                    v_{j+1} = w / h_{j+1,j}
//   cycle close:     y = R^{-1} g (host), x += P^{-1}(V y), true residual b - A x.
// Reductions are two-level (per-block partials, then one block in fixed order): deterministic.
// The host reads back j+3 scalars per step through pinned memory (one stream sync per step).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

using namespace fdiga;

namespace {

constexpr int KMAX = 32;  // basis vectors per reduction pass (m <= KMAX - 1)
constexpr int RT = 256;   // threads per reduction block

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-reduce `cnt` per-thread values acc[0..cnt) and write them to part[blockIdx.x * stride + i].
template <int CNT>
__device__ __forceinline__ void block_store(double (&acc)[CNT], int cnt, double* part, int stride) {
  __shared__ double red[RT / 32][CNT];
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
    part[(int64_t)blockIdx.x * stride + i] = s;
  }
}

// part[b][i] for i < k: V_i . w ;  part[b][k]: w . w
__global__ void __launch_bounds__(RT) multidot_kernel(const double* __restrict__ V, int64_t ldv, int k,
                                                      const double* __restrict__ w, int64_t N, double* part) {
  double acc[KMAX + 1];
#pragma unroll
  for (int i = 0; i <= KMAX; ++i) acc[i] = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT) {
    const double wv = w[e];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) acc[i] = fma(V[i * ldv + e], wv, acc[i]);
    acc[KMAX] = fma(wv, wv, acc[KMAX]);
  }
  // block reduction: slot i < k gets V_i . w, slot k gets w . w (static register indexing only)
  __shared__ double red[RT / 32][KMAX + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i <= KMAX; ++i) {
    if (i < k || i == KMAX) {
      const double v = warp_sum(acc[i]);
      if (lane == 0) red[warp][i == KMAX ? k : i] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += blockDim.x) {
    double s = 0;
    for (int ww = 0; ww < RT / 32; ++ww) s += red[ww][i];
    part[(int64_t)blockIdx.x * (KMAX + 1) + i] = s;
  }
}

// w <- w - sum_i h[i] V_i ; part[b][0] = ||w||^2 (new w)
__global__ void __launch_bounds__(RT) update_kernel(const double* __restrict__ V, int64_t ldv, int k,
                                                    const double* __restrict__ h, double* __restrict__ w, int64_t N,
                                                    double* part) {
  __shared__ double hs[KMAX];
  if (threadIdx.x < k) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double acc[1] = {0.0};
  for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT) {
    double v = w[e];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) v = fma(-hs[i], V[i * ldv + e], v);
    w[e] = v;
    acc[0] = fma(v, v, acc[0]);
  }
  block_store<1>(acc, 1, part, KMAX + 1);
}

// out[i] = sum_b part[b][i], i < cnt, in fixed block order (one warp per output value)
__global__ void reduce_partials_kernel(const double* part, int nblocks, int cnt, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < cnt; i += nw) {
    double s = 0;
    for (int b = lane; b < nblocks; b += 32) s += part[(int64_t)b * (KMAX + 1) + i];
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
}

// out = alpha * in
__global__ void scale_kernel(const double* __restrict__ in, double alpha, double* __restrict__ out, int64_t N) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = alpha * in[e];
}

// out = sum_i c[i] V_i  (c in device memory, k <= KMAX)
__global__ void __launch_bounds__(RT) lincomb_kernel(const double* __restrict__ V, int64_t ldv, int k,
                                                     const double* __restrict__ c, double* __restrict__ out,
                                                     int64_t N) {
  __shared__ double cs[KMAX];
  if (threadIdx.x < k) cs[threadIdx.x] = c[threadIdx.x];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT) {
    double v = 0;
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) v = fma(cs[i], V[i * ldv + e], v);
    out[e] = v;
  }
}

// x += z
__global__ void axpy_kernel(const double* __restrict__ z, double* __restrict__ x, int64_t N) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    x[e] += z[e];
}

// r = b - Ax ; part[b][0] = ||r||^2, part[b][1] = ||b||^2
__global__ void __launch_bounds__(RT) residual_kernel(const double* __restrict__ b, const double* __restrict__ Ax,
                                                      double* __restrict__ r, int64_t N, double* part) {
  double acc[2] = {0.0, 0.0};
  for (int64_t e = blockIdx.x * (int64_t)RT + threadIdx.x; e < N; e += (int64_t)gridDim.x * RT) {
    const double bv = b[e];
    const double v = bv - Ax[e];
    r[e] = v;
    acc[0] = fma(v, v, acc[0]);
    acc[1] = fma(bv, bv, acc[1]);
  }
  block_store<2>(acc, 2, part, KMAX + 1);
}

struct Gm {
  fdiga_ctx* ctx;
  fdiga_stencil* A;
  fd_plan* P;
  int64_t N, ldv;
  double *V, *z, *w, *part, *small;
  int nblk;
  cudaStream_t st;


  int reduce(int cnt, double* out) {
    reduce_partials_kernel<<<1, 1024, 0, st>>>(part, nblk, cnt, out);
    count_launch(ctx);
    FDIGA_CUDA(cudaGetLastError());
    return FDIGA_OK;
  }
  // host copy of `cnt` doubles from device `src` (pinned staging), synchronising the stream
  int fetch(const double* src, int cnt, double* dst) {
    FDIGA_TRY(ensure_pinned(ctx, 64));
    FDIGA_CUDA(cudaMemcpyAsync(ctx->pinned, src, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
    FDIGA_CUDA(cudaStreamSynchronize(st));
    std::copy(ctx->pinned, ctx->pinned + cnt, dst);
    return FDIGA_OK;
  }
  int precond(const double* in, double* out) {
    if (P) return fd_apply(P, in, out);
    FDIGA_CUDA(cudaMemcpyAsync(out, in, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return FDIGA_OK;
  }
  int launch_check() {
    count_launch(ctx);
    FDIGA_CUDA(cudaGetLastError());
    return FDIGA_OK;
  }
};

}  // namespace

extern "C" int gmres_solve(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const double* b, double* x,
                           const gmres_opts* opts, gmres_report* rep) {
  FDIGA_CHECK(ctx && A && b && x, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_TRY(bind(ctx));
  const int m = opts ? opts->m : 30;
  const double rtol = opts ? opts->rtol : 1e-8;
  const int max_iters = opts ? opts->max_iters : 1000;
  const int orth = opts ? opts->orth : FDIGA_ORTH_CGS_DGKS;
  const int use_x0 = opts ? opts->use_x0 : 0;
  FDIGA_CHECK(m >= 1 && m <= KMAX - 1, FDIGA_ERR_INVALID_ARG, "restart length m = %d must be in [1, %d]", m, KMAX - 1);
  int64_t nnz = 0, nd[3] = {1, 1, 1};
  FDIGA_TRY(stencil_info(A, &nnz, nd, nullptr, nullptr));
  Gm g;
  g.ctx = ctx;
  g.A = A;
  g.P = P;
  g.N = nd[0] * nd[1] * nd[2];
  g.ldv = (g.N + 63) & ~int64_t(63);  // 512-byte aligned basis vectors
  g.st = ctx->stream;
  g.nblk = std::min<int64_t>((g.N + RT - 1) / RT, 2 * ctx->sm_count);
  FDIGA_TRY(ctx->ws[0].ensure((size_t)(m + 1) * g.ldv));
  FDIGA_TRY(ctx->ws[1].ensure((size_t)2 * g.ldv));
  FDIGA_TRY(ctx->ws[2].ensure((size_t)g.nblk * (KMAX + 1)));
  FDIGA_TRY(ctx->ws[3].ensure(4 * (KMAX + 1)));
  g.V = ctx->ws[0].p;
  g.z = ctx->ws[1].p;
  g.w = ctx->ws[1].p + g.ldv;
  g.part = ctx->ws[2].p;
  g.small = ctx->ws[3].p;
  double* hdev = g.small;                 // h (and w.w) of the current pass
  double* h2dev = g.small + (KMAX + 1);   // second DGKS pass
  double* nrm = g.small + 2 * (KMAX + 1); // norms
  double* ydev = g.small + 3 * (KMAX + 1);
  const int grid = g.nblk;

  cudaEvent_t e0, e1;
  FDIGA_CUDA(cudaEventCreate(&e0));
  FDIGA_CUDA(cudaEventCreate(&e1));
  FDIGA_CUDA(cudaEventRecord(e0, g.st));

  if (!use_x0) FDIGA_CUDA(cudaMemsetAsync(x, 0, g.N * sizeof(double), g.st));

  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), hcol(KMAX + 2), h2(KMAX + 2);
  int iters = 0, restarts = 0, reorth = 0, converged = 0, status = FDIGA_OK;
  double bnorm = 0, rel_implicit = NAN, beta = 0;
  auto Hc = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };

  while (true) {
    // r = b - A x  -> V_0 ; beta = ||r||, ||b||
    FDIGA_TRY(stencil_matvec(A, x, g.w));
    residual_kernel<<<grid, RT, 0, g.st>>>(b, g.w, g.V, g.N, g.part);
    FDIGA_TRY(g.launch_check());
    FDIGA_TRY(g.reduce(2, nrm));
    double nb[2];
    FDIGA_TRY(g.fetch(nrm, 2, nb));
    beta = std::sqrt(nb[0]);
    bnorm = std::sqrt(nb[1]);
    if (!std::isfinite(beta)) {
      status = FDIGA_ERR_BREAKDOWN;
      set_error("gmres_solve: non-finite residual");
      break;
    }
    if (beta <= rtol * bnorm || bnorm == 0.0) {
      converged = 1;
      break;
    }
    if (iters >= max_iters) {
      status = FDIGA_ERR_NOT_CONVERGED;
      set_error("gmres_solve: %d iterations without convergence", iters);
      break;
    }
    ++restarts;
    scale_kernel<<<grid, RT, 0, g.st>>>(g.V, 1.0 / beta, g.V, g.N);
    FDIGA_TRY(g.launch_check());
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      double* vj = g.V + (int64_t)j * g.ldv;
      FDIGA_TRY(g.precond(vj, g.z));
      FDIGA_TRY(stencil_matvec(A, g.z, g.w));
      ++iters;
      const int nk = j + 1;
      // pass 1: h = V^T w, w.w ; w -= V h ; ||w||^2
      multidot_kernel<<<grid, RT, 0, g.st>>>(g.V, g.ldv, nk, g.w, g.N, g.part);
      FDIGA_TRY(g.launch_check());
      FDIGA_TRY(g.reduce(nk + 1, hdev));
      update_kernel<<<grid, RT, 0, g.st>>>(g.V, g.ldv, nk, hdev, g.w, g.N, g.part);
      FDIGA_TRY(g.launch_check());
      FDIGA_TRY(g.reduce(1, hdev + nk + 1));
      FDIGA_TRY(g.fetch(hdev, nk + 2, hcol.data()));
      double ww = hcol[nk], wn2 = hcol[nk + 1];
      if (orth == FDIGA_ORTH_CGS2 || wn2 < 0.5 * ww) {  // DGKS criterion ||w'|| < ||w||/sqrt(2)
        ++reorth;
        multidot_kernel<<<grid, RT, 0, g.st>>>(g.V, g.ldv, nk, g.w, g.N, g.part);
        FDIGA_TRY(g.launch_check());
        FDIGA_TRY(g.reduce(nk + 1, h2dev));
        update_kernel<<<grid, RT, 0, g.st>>>(g.V, g.ldv, nk, h2dev, g.w, g.N, g.part);
        FDIGA_TRY(g.launch_check());
        FDIGA_TRY(g.reduce(1, h2dev + nk + 1));
        FDIGA_TRY(g.fetch(h2dev, nk + 2, h2.data()));
        for (int i = 0; i < nk; ++i) hcol[i] += h2[i];
        wn2 = h2[nk + 1];
      }
      for (int i = 0; i < nk; ++i) Hc(i, j) = hcol[i];
      const double hn = std::sqrt(std::max(wn2, 0.0));
      Hc(j + 1, j) = hn;
      bool bad = !std::isfinite(hn);
      for (int i = 0; i < nk; ++i) bad = bad || !std::isfinite(hcol[i]);
      if (bad) {
        status = FDIGA_ERR_BREAKDOWN;
        set_error("gmres_solve: non-finite Hessenberg entry at step %d", iters);
        break;
      }
      // apply previous rotations, form the new one
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * Hc(i, j) + sn[i] * Hc(i + 1, j);
        Hc(i + 1, j) = -sn[i] * Hc(i, j) + cs[i] * Hc(i + 1, j);
        Hc(i, j) = t;
      }
      const double a = Hc(j, j), bb = Hc(j + 1, j);
      const double rr = std::hypot(a, bb);
      if (rr == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = a / rr;
        sn[j] = bb / rr;
      }
      Hc(j, j) = rr;
      Hc(j + 1, j) = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      rel_implicit = std::fabs(gv[j + 1]) / bnorm;
      if (rep && rep->history && iters - 1 < rep->history_cap) rep->history[iters - 1] = rel_implicit;
      k = j + 1;
      if (std::fabs(gv[j + 1]) <= rtol * bnorm || bb == 0.0 || iters >= max_iters) break;
      scale_kernel<<<grid, RT, 0, g.st>>>(g.w, 1.0 / hn, g.V + (int64_t)(j + 1) * g.ldv, g.N);
      FDIGA_TRY(g.launch_check());
    }
    if (status != FDIGA_OK) break;
    // y = R_k^{-1} g, x += P^{-1} (V_k y)
    std::vector<double> y(k, 0.0);
    for (int i = k - 1; i >= 0; --i) {
      double s = gv[i];
      for (int c = i + 1; c < k; ++c) s -= Hc(i, c) * y[c];
      y[i] = s / Hc(i, i);
    }
    FDIGA_CUDA(cudaMemcpyAsync(ydev, y.data(), k * sizeof(double), cudaMemcpyHostToDevice, g.st));
    lincomb_kernel<<<grid, RT, 0, g.st>>>(g.V, g.ldv, k, ydev, g.w, g.N);
    FDIGA_TRY(g.launch_check());
    FDIGA_TRY(g.precond(g.w, g.z));
    axpy_kernel<<<grid, RT, 0, g.st>>>(g.z, x, g.N);
    FDIGA_TRY(g.launch_check());
    FDIGA_CUDA(cudaStreamSynchronize(g.st));  // y lives on the host stack
  }
  FDIGA_CUDA(cudaEventRecord(e1, g.st));
  FDIGA_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->iters = iters;
    rep->restarts = restarts;
    rep->converged = converged;
    rep->reorth = reorth;
    rep->rel_res_true = bnorm > 0 ? beta / bnorm : 0.0;
    rep->rel_res_implicit = rel_implicit;
    rep->t_total_ms = ms;
  }
  return status;
}
