// Matrix-free collocation matvec (NEXT-1; the paper's future-work direction "if the matrix-vector
// products could be computed faster"; the matvec dominates in 3D).
//
// Row i = tau_i of eq:collocation with the chain rule of DESIGN.md:
//   (A x)_i = sum_t c_t(tau_i) [ (D_3^{t_3} (x) D_2^{t_2} (x) D_1^{t_1}) x ]_i,
//   D_l^{(r)}[i, j] = B_j^{(r)}(tau_{l,i}),  t in {e_a + e_b} (c_t = -G_ab, x2 off the diagonal) and {e_a}
//   (c_t = beta_a),  G = (J^T J)^{-1},  beta_a = sum_c (J^{-1})_{ac} tr(G H_c).
// One CTA computes an 8 x 8 x 8 tile of rows by sum factorisation over the banded 1D windows:
//   stage 0  x box [lo_3, hi_3) x [lo_2, hi_2) x [lo_1, hi_1) -> shared memory (halo planes when sharded)
//   stage 1  X1_r[i1][j3][j2]       = sum_c D_1^{(r)}[i1, c] x[j3][j2][s_1(i1) + c],      r = 0, 1, 2
//   stage 2  X12_{r1 r2}[i1 i2][j3] = sum_c D_2^{(r2)}[i2, c] X1_{r1}[i1][j3][s_2(i2) + c], r1 + r2 <= 2
//   stage 3  Z_t[i1 i2 i3]          = sum_c D_3^{(r3)}[i3, c] X12_{r1 r2}[i1 i2][s_3(i3) + c], 1 <= |t| <= 2
//   y = sum_t c_t Z_t with c_t from the analytic map at tau_i (geometry.cuh).
// Bytes per row: 8 (x, read through L2 once per tile box) + 8 (y); no stored values.  Arithmetic is
// FP64 FMA on shared-memory operands.
#include <algorithm>

#include "matfree.cuh"
#include "ptx.cuh"

namespace fdiga {

namespace {

constexpr int T = MF_T;
constexpr int NT = 256;  // threads per CTA

__device__ __forceinline__ const double* mf_plane(const MfArgs& A, int64_t g, int64_t n12) {
  if (!A.sharded) return A.x + g * n12;
  if (g < A.o) return A.halo_lo + (g - A.lo) * n12;
  if (g >= A.e) return A.halo_hi + (g - A.e) * n12;
  return A.x + (g - A.o) * n12;
}

// Issue the x box of tile `tile` into xs with cp.async (8-byte LDGSTS): warp w takes the planes
// j3 = w, w + 8, ...; its two half-warps take the rows j2 = 0, 1 (+2, ...), lanes the contiguous j1.
// tile coordinates along the three directions; the persistent CTA walks them by a fixed stride (gridDim.x)
// with carry propagation instead of per-tile integer divisions
struct MfTileQ {
  int q1, q2, q3;
};
__device__ __forceinline__ MfTileQ mf_tile_q(int tl, int t1, int t2) { return {tl % t1, (tl / t1) % t2, tl / (t1 * t2)}; }
__device__ __forceinline__ MfTileQ mf_advance(MfTileQ q, MfTileQ d, int t1, int t2) {
  q.q1 += d.q1;
  if (q.q1 >= t1) {
    q.q1 -= t1;
    ++q.q2;
  }
  q.q2 += d.q2;
  if (q.q2 >= t2) {
    q.q2 -= t2;
    ++q.q3;
  }
  q.q3 += d.q3;
  return q;
}

__device__ __forceinline__ void mf_issue_box(const MfArgs& A, MfTileQ q, double* xs, int* lo, int* bx) {
  const int q1 = q.q1, q2 = q.q2, q3 = q.q3;
  const int l1 = __ldg(A.box1 + 2 * q1), b1 = __ldg(A.box1 + 2 * q1 + 1);
  const int l2 = __ldg(A.box2 + 2 * q2), b2 = __ldg(A.box2 + 2 * q2 + 1);
  const int l3 = __ldg(A.box3 + 2 * q3), b3 = __ldg(A.box3 + 2 * q3 + 1);
  if (threadIdx.x == 0) {
    lo[0] = l1;
    lo[1] = l2;
    lo[2] = l3;
    bx[0] = b1;
    bx[1] = b2;
    bx[2] = b3;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n1 = A.n1, n12 = A.n1 * A.n2;
  const uint32_t xs0 = smem_u32(xs);
  for (int j3 = warp; j3 < b3; j3 += NT / 32) {
    const double* pl = mf_plane(A, l3 + j3, n12) + (int64_t)l2 * n1 + l1;
    for (int j2 = lane >> 4; j2 < b2; j2 += 2) {
      const double* src = pl + (int64_t)j2 * n1;
      const int row = j3 * b2 + j2;
      for (int j1 = lane & 15; j1 < b1; j1 += 16) cp_async8(xs0 + 8u * (uint32_t)(row * b1 + j1), src + j1, 8);
    }
  }
  cp_async_commit();
}

template <int WM>
__global__ void __launch_bounds__(NT, 2) matfree_kernel(MfArgs A) {
  if (A.skip && *A.skip) return;
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const int64_t ntiles = A.t1 * A.t2 * A.t3;
  // shared-memory regions: xs = x box (B1 B2 B3), X1 = 3 x T x (B3 B2 | 1), X12 = 6 x T T x (B3 | 1).
  // The next tile's box is prefetched into xs (cp.async) while stages 2 and 3 of this tile run.
  // padded (odd) strides keep the 8-byte shared accesses of a warp on distinct banks
  const int ps1 = (A.B3 * A.B2) | 1;  // X1: per (r, i1) plane of B3 x B2
  const int pb3 = A.B3 | 1;           // X12: per (combo, pixel) line of B3
  double* xs = sm;
  double* x1 = sm + A.B1 * A.B2 * A.B3;
  double* x12 = x1 + 3 * T * ps1;
  __shared__ int lo_s[2][3], bx_s[2][3];
  int buf = 0;
  const int t1 = (int)A.t1, t2 = (int)A.t2;
  const MfTileQ dq = mf_tile_q((int)gridDim.x, t1, t2);
  MfTileQ cq = mf_tile_q((int)blockIdx.x, t1, t2);
  if (blockIdx.x < ntiles) mf_issue_box(A, cq, xs, lo_s[0], bx_s[0]);
  const int64_t n12 = A.n1 * A.n2;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
  const int q1 = cq.q1, q2 = cq.q2, q3 = cq.q3;
  const MfTileQ nq = mf_advance(cq, dq, t1, t2);
  const int a1 = q1 * T, a2 = q2 * T, a3 = (int)A.o + q3 * T;  // first row of the tile (global; 32-bit)
  const int n1i = (int)A.n1, n2i = (int)A.n2, n3i = (int)A.n3, Wt = A.W;
  const int m1 = (int)(A.n1 - a1 < T ? A.n1 - a1 : T), m2 = (int)(A.n2 - a2 < T ? A.n2 - a2 : T),
            m3 = (int)(A.e - a3 < T ? A.e - a3 : T);
  cp_async_wait<0>();
  __syncthreads();  // the box has landed; the previous tile's stage 3 is done with X12
  const int* lo = lo_s[buf];
  const int b1 = bx_s[buf][0], b2 = bx_s[buf][1], b3 = bx_s[buf][2];
  // ---- stage 1: direction 1 (thread: fixed i1, loop over (j3, j2))
  {
    const int i1 = tid & (T - 1);
    if (i1 < m1) {
      const int g1 = a1 + i1;
      const int w = __ldg(A.w1 + g1), o = __ldg(A.st1 + g1) - lo[0];
      double d0[WM], d1[WM], d2[WM];
#pragma unroll
      for (int c = 0; c < WM; ++c) {
        const bool on = c < w;
        d0[c] = on ? __ldg(A.tab1 + (0 * n1i + g1) * Wt + c) : 0.0;
        d1[c] = on ? __ldg(A.tab1 + (1 * n1i + g1) * Wt + c) : 0.0;
        d2[c] = on ? __ldg(A.tab1 + (2 * n1i + g1) * Wt + c) : 0.0;
      }
      const int npair = b3 * b2;
      double* o0 = x1 + (0 * T + i1) * ps1;
      double* o1 = x1 + (1 * T + i1) * ps1;
      double* o2 = x1 + (2 * T + i1) * ps1;
      // box row pq = j3 b2 + j2 of xs maps to entry pq of X1 (compact [j3][j2], stride b2); two rows per
      // iteration for independent FMA chains
      constexpr int STEP = NT / T;
      for (int pq = tid / T; pq < npair; pq += 2 * STEP) {
        const bool two = pq + STEP < npair;
        const double* xa = xs + pq * b1 + o;
        const double* xb = xa + (two ? STEP * b1 : 0);
        double s0 = 0, s1 = 0, s2 = 0, u0 = 0, u1 = 0, u2 = 0;
#pragma unroll
        for (int c = 0; c < WM; ++c)
          if (c < w) {
            const double v = xa[c], vb = xb[c];
            s0 = fma(d0[c], v, s0);
            s1 = fma(d1[c], v, s1);
            s2 = fma(d2[c], v, s2);
            u0 = fma(d0[c], vb, u0);
            u1 = fma(d1[c], vb, u1);
            u2 = fma(d2[c], vb, u2);
          }
        o0[pq] = s0;
        o1[pq] = s1;
        o2[pq] = s2;
        if (two) {
          o0[pq + STEP] = u0;
          o1[pq + STEP] = u1;
          o2[pq + STEP] = u2;
        }
      }
    }
  }
  __syncthreads();  // xs is free: prefetch the next tile's box
  if (tile + gridDim.x < ntiles) mf_issue_box(A, nq, xs, lo_s[buf ^ 1], bx_s[buf ^ 1]);
  // ---- stage 2: direction 2 (thread: fixed (i1, i2), loop over j3)
  {
    const int i1 = tid & (T - 1), i2 = (tid / T) & (T - 1), jg = tid / (T * T);
    if (i1 < m1 && i2 < m2) {
      const int g2 = a2 + i2;
      const int w = __ldg(A.w2 + g2), o = __ldg(A.st2 + g2) - lo[1];
      double d0[WM], d1[WM], d2[WM];
#pragma unroll
      for (int c = 0; c < WM; ++c) {
        const bool on = c < w;
        d0[c] = on ? __ldg(A.tab2 + (0 * n2i + g2) * Wt + c) : 0.0;
        d1[c] = on ? __ldg(A.tab2 + (1 * n2i + g2) * Wt + c) : 0.0;
        d2[c] = on ? __ldg(A.tab2 + (2 * n2i + g2) * Wt + c) : 0.0;
      }
      const double* in0 = x1 + (0 * T + i1) * ps1;
      const double* in1 = x1 + (1 * T + i1) * ps1;
      const double* in2 = x1 + (2 * T + i1) * ps1;
      const int pix = i2 * T + i1;
      for (int j3 = jg; j3 < b3; j3 += NT / (T * T)) {
        double s00 = 0, s01 = 0, s02 = 0, s10 = 0, s11 = 0, s20 = 0;
        const int base = j3 * b2 + o;
#pragma unroll
        for (int c = 0; c < WM; ++c)
          if (c < w) {
            const double v0 = in0[base + c], v1 = in1[base + c], v2 = in2[base + c];
            s00 = fma(d0[c], v0, s00);
            s01 = fma(d1[c], v0, s01);
            s02 = fma(d2[c], v0, s02);
            s10 = fma(d0[c], v1, s10);
            s11 = fma(d1[c], v1, s11);
            s20 = fma(d0[c], v2, s20);
          }
        // X12 combos: 0 = (0,0), 1 = (0,1), 2 = (0,2), 3 = (1,0), 4 = (1,1), 5 = (2,0)   [(r1, r2)]
        const int st = T * T * pb3;
        x12[0 * st + pix * pb3 + j3] = s00;
        x12[1 * st + pix * pb3 + j3] = s01;
        x12[2 * st + pix * pb3 + j3] = s02;
        x12[3 * st + pix * pb3 + j3] = s10;
        x12[4 * st + pix * pb3 + j3] = s11;
        x12[5 * st + pix * pb3 + j3] = s20;
      }
    }
  }
  __syncthreads();
  // ---- stage 3: direction 3 and the geometry coefficients (thread: (i1, i2), two rows i3)
  {
    const int pix = tid & (T * T - 1), i1 = pix % T, i2 = pix / T;  // i1 fastest: coalesced y stores
    if (i1 < m1 && i2 < m2) {
      const int st = T * T * pb3;
      const int g1 = a1 + i1, g2 = a2 + i2;
      const double xi1 = __ldg(A.tau1 + g1);
      double sn[3], cs[3];
      sn[0] = __ldg(A.trig1 + 2 * g1);
      cs[0] = __ldg(A.trig1 + 2 * g1 + 1);
      sn[1] = __ldg(A.trig2 + 2 * g2);
      cs[1] = __ldg(A.trig2 + 2 * g2 + 1);
      // the ring maps do not depend on xi_3: one coefficient set per (i1, i2)
      const bool dep3 = A.geo.id == FDIGA_GEOM_DEFORMED_CUBE;
      double G[3][3], beta[3];
      double Fp[3], wv[3];
      if (!dep3) {  // the ring maps and the winds used with them do not depend on xi_3
        sn[2] = 0.0;
        cs[2] = 1.0;
        geometry_F(A.geo, xi1, __ldg(A.tau2 + g2), 0.0, sn, cs, Fp);
        wind_at(A.geo, Fp, wv);
        colloc_coeffs<3>(geometry_jh(A.geo, xi1, sn, cs), G, beta, A.geo.wind ? wv : nullptr);
      }
      for (int i3 = tid / (T * T); i3 < m3; i3 += NT / (T * T)) {
        const int g3 = a3 + i3;
        const int w = __ldg(A.w3 + g3), o = __ldg(A.st3 + g3) - lo[2];
        double z[9], f0[WM], f1[WM], f2[WM];
#pragma unroll
        for (int k = 0; k < 9; ++k) z[k] = 0.0;
#pragma unroll
        for (int c = 0; c < WM; ++c) {
          const bool on = c < w;
          f0[c] = on ? __ldg(A.tab3 + (0 * n3i + g3) * Wt + c) : 0.0;
          f1[c] = on ? __ldg(A.tab3 + (1 * n3i + g3) * Wt + c) : 0.0;
          f2[c] = on ? __ldg(A.tab3 + (2 * n3i + g3) * Wt + c) : 0.0;
        }
        const double* in = x12 + pix * pb3 + o;
#pragma unroll
        for (int c = 0; c < WM; ++c)
          if (c < w) {
            const double e0 = f0[c], e1 = f1[c], e2 = f2[c];
            const double v00 = in[0 * st + c], v01 = in[1 * st + c], v02 = in[2 * st + c];
            const double v10 = in[3 * st + c], v11 = in[4 * st + c], v20 = in[5 * st + c];
            z[0] = fma(e1, v00, z[0]);  // (0,0,1)
            z[1] = fma(e2, v00, z[1]);  // (0,0,2)
            z[2] = fma(e0, v01, z[2]);  // (0,1,0)
            z[3] = fma(e1, v01, z[3]);  // (0,1,1)
            z[4] = fma(e0, v02, z[4]);  // (0,2,0)
            z[5] = fma(e0, v10, z[5]);  // (1,0,0)
            z[6] = fma(e1, v10, z[6]);  // (1,0,1)
            z[7] = fma(e0, v11, z[7]);  // (1,1,0)
            z[8] = fma(e0, v20, z[8]);  // (2,0,0)
          }
        if (dep3) {
          sn[2] = __ldg(A.trig3 + 2 * g3);
          cs[2] = __ldg(A.trig3 + 2 * g3 + 1);
          geometry_F(A.geo, xi1, __ldg(A.tau2 + g2), __ldg(A.tau3 + g3), sn, cs, Fp);
          wind_at(A.geo, Fp, wv);
          colloc_coeffs<3>(geometry_jh(A.geo, xi1, sn, cs), G, beta, A.geo.wind ? wv : nullptr);
        }
        double yv = beta[2] * z[0] - G[2][2] * z[1] + beta[1] * z[2] - 2.0 * G[1][2] * z[3] - G[1][1] * z[4] +
                    beta[0] * z[5] - 2.0 * G[0][2] * z[6] - 2.0 * G[0][1] * z[7] - G[0][0] * z[8];
        A.y[(int64_t)(g3 - (int)A.o) * n12 + g2 * n1i + g1] = yv;
      }
    }
  }
  cq = nq;
  }  // tile loop
}

}  // namespace

size_t matfree_smem_bytes(int B1, int B2, int B3) {
  const size_t r0 = (size_t)B1 * B2 * B3;
  const size_t r1 = (size_t)3 * T * ((B3 * B2) | 1);
  const size_t r2 = (size_t)6 * T * T * (B3 | 1);
  return (r0 + r1 + r2) * sizeof(double);
}

int matfree_launch(const MfArgs& a, cudaStream_t stream) {
  const int64_t tiles = a.t1 * a.t2 * a.t3;
  if (tiles == 0) return FDIGA_OK;
  const size_t smem = matfree_smem_bytes(a.B1, a.B2, a.B3);
  // persistent CTAs: two per SM (register and shared-memory limits), striding over the tiles
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, 2 * (int64_t)nsm);
  switch (a.W) {
#define FDIGA_MF(WMV)                                                                                     \
  case WMV: {                                                                                            \
    static bool attr = false;                                                                            \
    if (!attr) {                                                                                         \
      FDIGA_CUDA(cudaFuncSetAttribute(matfree_kernel<WMV>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                      200 * 1024));                                                      \
      attr = true;                                                                                       \
    }                                                                                                    \
    matfree_kernel<WMV><<<grid, NT, smem, stream>>>(a);                                                  \
    break;                                                                                               \
  }
    FDIGA_MF(2)
    FDIGA_MF(3)
    FDIGA_MF(4)
    FDIGA_MF(5)
    FDIGA_MF(6)
    FDIGA_MF(7)
    FDIGA_MF(8)
    FDIGA_MF(9)
#undef FDIGA_MF
    default:
      FDIGA_CHECK(false, FDIGA_ERR_NOT_SUPPORTED, "matrix-free operator: degree p = %d out of range", a.W - 1);
  }
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

}  // namespace fdiga
