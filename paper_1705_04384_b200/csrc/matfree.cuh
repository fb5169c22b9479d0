// Matrix-free collocation operator: y = A_C x by sum factorisation
// with the geometry coefficients evaluated on the fly from the analytic map.
#pragma once
#include "common.cuh"
#include "geometry.cuh"

namespace fdiga {

constexpr int MF_T = 8;  // output tile edge (8 x 8 x 8 rows per CTA)

struct MfArgs {
  int64_t n1, n2, n3;        // global sizes
  int64_t o, e, lo;          // local planes [o, e) of direction 3; halo planes start at lo
  int64_t t1, t2, t3;        // tiles per direction (t3 over the local planes)
  const double* x;           // local planes [o, e)
  const double *halo_lo, *halo_hi;
  double* y;                 // local rows
  const int32_t *st1, *st2, *st3, *w1, *w2, *w3;
  const double *tab1, *tab2, *tab3;  // tab_l[(r n_l + i) W + c] = B^{(r)}_{start_l(i) + c}(tau_{l,i})
  const double *tau1, *tau2, *tau3;
  const double *trig1, *trig2, *trig3;  // (sin, cos)(geo_theta * tau_{l,i}) pairs
  int W;                     // table row stride (p + 1)
  int B1, B2, B3;            // max x-box extent per direction over all tiles (shared-memory layout)
  const int32_t *box1, *box2, *box3;  // per tile index along direction l: (first column, extent) of its x box
  Geo geo;
  const int* skip;
  int sharded;
};

// shared memory (bytes) of one CTA for the given box bounds
size_t matfree_smem_bytes(int B1, int B2, int B3);
int matfree_launch(const MfArgs& a, cudaStream_t stream);

}  // namespace fdiga
