/*
 * fdiga.h — C ABI of libfdiga.so: the B200 (sm_100a) hot path of the nonsymmetric
 * Fast-Diagonalization (FD) preconditioner inside restarted GMRES for isogeometric
 * collocation of the Poisson problem (M. Tani, arXiv:1705.04384).
 *
 * Citations "P:<line>" refer to the paper's text, "S:<line>" to SPEC.md.
 *
 * Conventions shared by every entry point
 *   - Return value: 0 (FDIGA_OK) or a negative fdiga_status.  No exception crosses the ABI.
 *     A human-readable message for the last failure on the calling thread is returned by
 *     fdiga_last_error().
 *   - Vectors of the discrete problem are FP64, contiguous, in the flattened order of P:159:
 *     i = i_1 + n_1 (i_2 + n_2 i_3) (0-based), i.e. an array X[i_d]...[i_1] with i_1 fastest.
 *     On nranks > 1 a vector argument holds only this rank's slab of the last index
 *     i_d in [begin, end) (fdiga_slab).
 *   - Matrices passed from the host are row-major FP64, copied before the call returns
 *     (the caller keeps ownership).  Handles own all device memory they allocate; plans and operators
 *     must be destroyed before the context they were created on.
 *   - Device vector arguments are caller-owned device pointers (e.g. torch data_ptr()).
 *   - Stream semantics: fd_apply and stencil_matvec are asynchronous on the context's stream;
 *     fd_setup*, colloc_assemble, stencil_create and gmres_solve synchronise before returning.
 *   - Multi-rank: every call is collective; all ranks call it in the same order with the
 *     same global arguments.
 *   - Environment (read once per process; none changes results beyond rounding):
 *       FDIGA_FD_OZ=0/1     force the FP64 DMMA / the int8-split tensor-core FD path for every plan that supports
 *                           it (default rule: int8 for 3D real-spectrum plans with 192 <= n_l <= 512; fd_plan_set_path
 *                           switches one plan)
 *       FDIGA_OZ_PDL=k      programmatic dependent launch on the int8 path: bit 0 the digit splits, bit 1 the GEMMs
 *                           (default 2)
 *       FDIGA_OZ_SF=0/1/2   int8 GEMM with streamed factor digits: never (two launches for 256 < n_l <= 512) / for
 *                           n_l > 256 (default) / always
 *       FDIGA_NVTX=1        NVTX ranges per API call and per solve stage (fdiga:fd, fdiga:matvec, fdiga:orth, ...)
 *       FDIGA_VERBOSE=1/2   set-up phase timings / autotuner results on stderr
 *       FDIGA_GEMM_TABLE, FDIGA_GEMM_TABLE_OUT, FDIGA_GEMM_TUNE_ALWAYS   the DMMA tile table (fd_gemm.cu)
 */
#ifndef FDIGA_H
#define FDIGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FDIGA_OK = 0,
  FDIGA_ERR_INVALID_ARG = -1,
  FDIGA_ERR_CUDA = -2,
  FDIGA_ERR_CUSOLVER = -3,
  FDIGA_ERR_NCCL = -4,
  FDIGA_ERR_COMPLEX_SPECTRUM = -5, /* complex eigenvalues and opts->allow_complex_pairs == 0 */
  FDIGA_ERR_ILL_CONDITIONED = -6,  /* cond_1(U_l) > opts->cond_max (Remark 1) */
  FDIGA_ERR_SINGULAR = -7,         /* min |Lambda| <= 1e3 eps max |Lambda| */
  FDIGA_ERR_NOT_CONVERGED = -8,    /* gmres_solve hit max_iters; report filled, x = last iterate */
  FDIGA_ERR_BREAKDOWN = -9,        /* NaN/Inf met inside gmres_solve */
  FDIGA_ERR_NOT_SUPPORTED = -10,
  FDIGA_ERR_OOM = -11
} fdiga_status;

/* Geometry ids for colloc_assemble (analytic maps of BASELINE.json's configs). */
enum {
  FDIGA_GEOM_IDENTITY = 0,      /* F = id on [0,1]^d */
  FDIGA_GEOM_ANNULUS = 1,       /* 2D quarter annulus, geo_params = {r0, r1} */
  FDIGA_GEOM_DEFORMED_CUBE = 2, /* 3D x_k = xi_k + a prod_l sin(pi xi_l), geo_params = {a} */
  FDIGA_GEOM_THICK_RING = 3     /* 3D quarter annulus x [0,h], geo_params = {r0, r1, h} */
};

/* Wind ids for colloc_assemble_cd (convection-diffusion, NEXT-4; eq:convection P:345). */
enum {
  FDIGA_WIND_NONE = 0,
  FDIGA_WIND_CONSTANT = 1, /* w = (wind_params[0], wind_params[1], wind_params[2]) */
  FDIGA_WIND_ROTATING = 2  /* w = omega (-x_2, x_1, 0), omega = wind_params[0] */
};

typedef struct fdiga_ctx fdiga_ctx;
typedef struct fd_plan fd_plan;
typedef struct fdiga_stencil fdiga_stencil;
typedef struct fdiga_loopback fdiga_loopback;

/* ---------------------------------------------------------------- context ---- */

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t to run on (caller-owned,
 * must outlive the context), or NULL for the legacy default stream.  nranks/rank/nccl_unique_id: the process group
 * (nccl_unique_id = 128-byte ncclUniqueId from fdiga_nccl_unique_id; required when nranks > 1).  A unique id
 * selects the NCCL transport and the slab-sharded code path: vectors hold the rank's
 * slab of the last axis, the FD mode-d pass runs after an all-to-all slab transpose, the matvec
 * exchanges halo planes and GMRES all-reduces its dot products.  With nranks == 1 and a unique id the
 * same path runs over a one-rank NCCL communicator (self messages); NULL runs the single-GPU path.
 * Sharded operators are 3D only (2D problems run as replicas); complex-pair FD is single-GPU only. */
int fdiga_ctx_create(int device, void* cuda_stream, int nranks, int rank, const void* nccl_unique_id,
                     fdiga_ctx** out);
int fdiga_ctx_destroy(fdiga_ctx* ctx); /* NULL -> no-op; collective when nranks > 1 */
/* This rank's slab [begin, end) of the last tensor index for a last-axis length n_last
 * (balanced: the first n_last % nranks ranks own one extra plane). */
int fdiga_slab(const fdiga_ctx* ctx, int64_t n_last, int64_t* begin, int64_t* end);
/* Fill a 128-byte buffer with a fresh ncclUniqueId (call on rank 0, broadcast it).  libnccl.so.2 is
 * resolved at run time (the copy torch loaded); FDIGA_ERR_NCCL if it cannot be found. */
int fdiga_nccl_unique_id(void* out128);
/* Loopback transport: `nranks` contexts in ONE process on ONE device, each used from its own host
 * thread with its own stream; collectives exchange device pointers and CUDA events through the hub
 * (no kernel waits on another rank).  Runs the sharded path of every rank on a single GPU.
 * Destroy the hub after all of its contexts. */
int fdiga_loopback_create(int nranks, fdiga_loopback** out);
int fdiga_loopback_destroy(fdiga_loopback* hub);
int fdiga_ctx_create_loopback(int device, void* cuda_stream, fdiga_loopback* hub, int rank, fdiga_ctx** out);
/* Balanced split of [0, n) into nparts contiguous ranges; part's range is [begin, end) (host only).
 * Slabs of the last axis (fdiga_slab) and the mode-d transpose chunks use it. */
int fdiga_partition(int64_t n, int nparts, int part, int64_t* begin, int64_t* end);
/* Exchange schedule of the sharded FD mode-d pass (host only; what fd_apply uses).  n_inner =
 * n_1..n_{d-1}, n_last = n_d.  Rank r owns slab planes [o_r, e_r) and, after the transpose, the inner
 * chunk [q_r, q_r + len_r) of all n_last planes as T(n_last x len_r).  For every peer q (arrays of
 * length nranks, in doubles): slab_off/slab_cnt = my (e_r - o_r) x len_q block of chunk q in the
 * staging buffer; tr_off/tr_cnt = rows [o_q, e_q) of my T.  Forward pass: send the slab blocks,
 * receive the T rows; backward pass: the reverse. */
int fdiga_transpose_plan(int64_t n_inner, int64_t n_last, int nranks, int rank, int64_t* slab_off, int64_t* slab_cnt,
                         int64_t* tr_off, int64_t* tr_cnt);
/* Halo schedule of the sharded matvec (host only; what stencil_matvec uses).  start/width: the
 * last-axis column windows (length n_last).  Out: the planes [lo, hi) this rank's rows read, and for
 * every peer q the planes [send_b[q], send_e[q]) it sends to q and [recv_b[q], recv_e[q]) it
 * receives from q (global plane indices; empty when b == e).  At most one message per pair. */
int fdiga_halo_plan(int64_t n_last, const int32_t* start, const int32_t* width, int nranks, int rank, int64_t* lo,
                    int64_t* hi, int64_t* send_b, int64_t* send_e, int64_t* recv_b, int64_t* recv_e);
const char* fdiga_status_string(int status);
const char* fdiga_last_error(void);

/* ------------------------------------------------------ FD preconditioner ---- */

typedef struct {
  double tol_imag;         /* |Im lambda| <= tol_imag * rho(M^{-1}K) counts as real (default 1e-8) */
  double cond_max;         /* reject cond_1(U_l) above this (default 1e8) */
  int allow_complex_pairs; /* 1: keep complex pairs as real 2x2 blocks of D_l; 0: fail */
} fd_setup_opts;

/* Setup from the 1D pencils (eq:eigendecomposition):
 *   M_l^{-1} K_l U_l = U_l D_l,  W_l := V_l^T = (M_l U_l)^{-1},  l = 1..d,
 * with U_l columns of unit 2-norm and eigenvalues ascending.  d in {2,3};
 * n[l] = size of direction l+1; M[l], K[l]: host row-major n[l] x n[l].  opts may be NULL.
 * Computed with cuSOLVER (getrf/getrs, Xgeev) — one time, not on the hot path. */
int fd_setup(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* M, const double* const* K,
             const fd_setup_opts* opts, fd_plan** out);
/* Setup from explicit real factors (host, row-major): U[l], W[l] = (M_l U_l)^{-1}, lam[l]. */
int fd_setup_from_factors(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* U,
                          const double* const* W, const double* const* lam, fd_plan** out);
/* Same with complex pairs in real 2x2-block form: a pair a +- ib with eigenvector p + iq is
 * stored in adjacent columns (p, q) of U[l] with lam_re = (a, a), lam_im = (+b, -b) (b > 0), i.e. the
 * block [[a, b], [-b, a]] of D_l.  lam_im (or lam_im[l]) NULL means a real spectrum.  The divide step
 * then solves the (<= 2^d x 2^d) diagonal blocks of Lambda.  INVALID_ARG on a malformed pair. */
int fd_setup_from_blocks(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* U,
                         const double* const* W, const double* const* lam_re, const double* const* lam_im,
                         fd_plan** out);
/* Setup from an eigenbasis: W_l = (M_l U_l)^{-1} computed on the device (M = NULL means M_l = I,
 * i.e. W_l = U_l^{-1}: BASELINE.json configs[3] "U_k^{-1} computed exactly in setup"). */
int fd_setup_from_eig(fdiga_ctx* ctx, int d, const int64_t* n, const double* const* U,
                      const double* const* lam, const double* const* M, fd_plan** out);
/* Copy factors of direction l (0-based) to host buffers (any may be NULL).  lam_im holds the
 * imaginary parts (+b/-b on the two members of a complex pair, else 0). */
int fd_get_factors(const fd_plan* plan, int l, double* U, double* W, double* lam_re, double* lam_im);
/* s = P^{-1} r by eq:FD2D / eq:FD3D:
 *   s = (U_d (x)..(x) U_1) Lambda^{-1} (W_d (x)..(x) W_1) r,  Lambda = sum_l I(x)..D_l..(x)I.
 * r, s: device, local slab, length N_local; s may alias r.  Asynchronous on the ctx stream. */
int fd_apply(fd_plan* plan, const double* r, double* s);
/* Same, with HOST buffers r, s (copied in and out inside the call; synchronises). */
int fd_apply_host(fd_plan* plan, const double* r_host, double* s_host);
/* Streaming variant: enqueue H2D of r_host, the apply and D2H into s_host and return at once.  Consecutive
 * calls rotate over three device staging buffers on dedicated copy streams, so the H2D of one call,
 * the apply of the previous one and the D2H of the one before overlap (both PCIe directions and the
 * SMs busy at once).  r_host / s_host must stay valid (and pinned, for real overlap) until fd_host_sync;
 * a later call may reuse them only after the earlier results were consumed. */
int fd_apply_host_async(fd_plan* plan, const double* r_host, double* s_host);
/* Wait for every fd_apply_host_async of this plan. */
int fd_host_sync(fd_plan* plan);
/* Algorithmic flops of one apply: 4 N sum_l n_l (= 12 n^4 in 3D P:481, 8 n^3 in 2D P:464). */
double fd_apply_flops(const fd_plan* plan);
/* Kernel family of the mode products: FDIGA_PATH_DMMA (FP64 mma.sync DMMA tiles) or FDIGA_PATH_INT8_SPLIT
 * (exact int8 digit splitting on tcgen05.mma.kind::i8 with TMEM accumulators; 3D real-spectrum plans with
 * 192 <= n_l <= 512 by default, single-rank or sharded).  int8_ops (may be NULL) receives the int8 tensor-core
 * operations one apply issues on that path (2 M N K per digit-pair MMA, padded shapes), else 0. */
enum { FDIGA_PATH_DMMA = 0, FDIGA_PATH_INT8_SPLIT = 1 };
int fd_plan_path(const fd_plan* plan, double* int8_ops);
/* Select the kernel family of this plan's mode products (default: the rule above).  FDIGA_PATH_DMMA is IEEE
 * FP64 (every output of a mode product is an FP64 dot product; always allowed).  FDIGA_PATH_INT8_SPLIT
 * needs d = 3, a real spectrum and n_l <= 512 (else NOT_SUPPORTED, plan unchanged); its accuracy contract
 * (DESIGN.md §5.1): per mode product y = F x, |y^ - y| <= 8u|y| + 2^-51.9 K max_k|x_k| max_k|F_ik| for every
 * output (u = 2^-53, K the contraction length) -- FP64-level relative to the fibre and factor-row maxima,
 * not componentwise -- and fibres / factor rows holding NaN/Inf, a nonzero |x| below 2^-24 of the row's
 * scale, or exponents below -900 are computed as IEEE FP64 dot products instead.  Synchronous. */
int fd_plan_set_path(fd_plan* plan, int path);
/* One fd_apply with a CUDA event recorded on the ctx stream after every kernel (and, sharded, after every
 * exchange) it issues; synchronises; collective like fd_apply.  kernel_ms[k] = duration of step k (event to
 * event), kernel_kind[k] = 0 (DMMA mode product), 1 (int8 digit split), 2 (int8 tensor-core GEMM), 3 (slab
 * pack) or 4 (NCCL / loopback exchange), for k < cap; *count = steps.  Diagnostics for per-kernel rooflines
 * (bench.py); the events serialise nothing that fd_apply overlaps. */
int fd_apply_timed(fd_plan* plan, const double* r, double* s, float* kernel_ms, int* kernel_kind, int cap,
                   int* count);
int fd_plan_destroy(fd_plan* plan);

/* ----------------------------------------------------- collocation operator ---- */

/* Stored collocation matrix A_C (eq:collocationsystem) in "tensor-window" form.
 * Row i = (i_1..i_d) couples to the box of columns j_l in [start_l[i_l], start_l[i_l] + width_l[i_l]).
 * values: for each row in flattened order, the w_d*..*w_1 values of its box, j_1 fastest;
 * row offsets are implied by the prefix sums of the widths (no index arrays).
 * start[l], width[l]: host int32 arrays of length n[l].  values: host or device
 * (values_on_device = 1), copied either way.  The library may re-layout values internally. */
int stencil_create(fdiga_ctx* ctx, int d, const int64_t* n, const int32_t* const* start,
                   const int32_t* const* width, const double* values, int values_on_device,
                   fdiga_stencil** out);
/* Assemble A_C on the device for degree p, ne[l] uniform elements per direction, open knots
 * (P:144-148), Greville collocation points, K = I, on geometry `geometry_id`
 * with parameters geo_params (see FDIGA_GEOM_*).  Row i holds (L (B_j o F^{-1}))(F(tau_i)). */
int colloc_assemble(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                    fdiga_stencil** out);
/* The same operator applied MATRIX-FREE (the paper's future work):
 * no values are stored; stencil_matvec evaluates sum_t c_t(tau_i) (D_3^{t_3} (x) D_2^{t_2} (x) D_1^{t_1}) x
 * by sum factorisation over the 1D windows with the geometry coefficients c_t computed on the fly from
 * the analytic map (8 + 8 bytes of HBM traffic per row instead of 8 nnz/row + 16).  3D only; usable
 * wherever a stencil is (matvec, gmres_solve, bicgstab_solve, sharded).  stencil_get_values reports
 * NOT_SUPPORTED; stencil_info's nnz is the structural count of the equivalent stored operator. */
int colloc_matrix_free(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                       fdiga_stencil** out);
/* Convection-diffusion operator L_w = -Lap + w . grad (eq:convection; NEXT-4), collocated like
 * colloc_assemble: row i holds (L_w (B_j o F^{-1}))(F(tau_i)), i.e. the first-order coefficient becomes
 * beta_a + (J^{-1} w(F(tau_i)))_a.  wind_id: FDIGA_WIND_*, wind_params: d constants or {omega}.
 * matrix_free = 1 builds the on-the-fly operator (3D only), else stored values. */
int colloc_assemble_cd(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                       int wind_id, const double* wind_params, int matrix_free, fdiga_stencil** out);
/* Weighted-quadrature Galerkin operator A_wq (eq:WQapprox P:195-199, eq:Q P:192) on
 * the same analytic maps, stored in the tensor-window layout (windows |i_l - j_l| <= p): degree p <= 5,
 * ne elements per direction (same in every direction).  The 1D rule (reading 18) is built on
 * the host, Q = det(J) J^{-1} J^{-T} on the device point grid, the rows by sum factorisation on the
 * device.  Sharded contexts assemble their slab's rows (3D).  Setup only; synchronises. */
int wq_assemble(fdiga_ctx* ctx, int d, int p, int64_t ne, int geometry_id, const double* geo_params,
                fdiga_stencil** out);
/* Univariate Galerkin factors (eq:univariateWQ P:209; host out, row-major n x n):
 * M[i][j] = int B_i B_j, K[i][j] = int B'_i B'_j -- the symmetric pencils of the WQ preconditioner. */
int galerkin_1d_factors(int p, int64_t ne, double* M, double* K);
/* y = A x.  x, y: device, length N (no aliasing).  Asynchronous on the ctx stream. */
int stencil_matvec(fdiga_stencil* A, const double* x, double* y);
/* Number of stored values and the 1D window tables (host copies; any pointer may be NULL). */
int stencil_info(const fdiga_stencil* A, int64_t* nnz, int64_t* n_out, int32_t* start_l0, int32_t* width_l0);
/* Copy the canonical (tensor-window, row-major box) values to a host buffer of length nnz. */
int stencil_get_values(const fdiga_stencil* A, double* values_host);
int stencil_destroy(fdiga_stencil* A);
/* Univariate collocation factors of the same discretisation (host out, row-major n x n):
 * M[i][j] = B_j(tau_i), K[i][j] = -B''_j(tau_i) (eq:univariatecolloc). */
int colloc_1d_factors(int p, int64_t ne, double* M, double* K);
/* The 1D column windows of the stored operator (host only): row i of direction l couples to columns
 * [start[i], start[i] + width[i]) (length n = ne + p - 2). */
int colloc_1d_windows(int p, int64_t ne, int32_t* start, int32_t* width);
/* The 1D convection factor of the collocation analogue of eq:convec_prec_2 (reading 17),
 * host only: H[i][j] = wt[i] B'_j(tau_i), wt = the univariate wind w~_l at the n Greville points (host). */
int colloc_1d_convection(int p, int64_t ne, const double* wt, double* H);

/* -------------------------------------------------------------------- GMRES ---- */

enum { FDIGA_ORTH_CGS_DGKS = 0, FDIGA_ORTH_CGS2 = 1, FDIGA_ORTH_DCGS2 = 2 };

typedef struct {
  int m;             /* restart length (default 30) */
  double rtol;       /* stop when ||b - A x|| <= rtol ||b|| (default 1e-8) */
  int max_iters;     /* Arnoldi steps over all cycles (default 1000) */
  int orth;          /* FDIGA_ORTH_DCGS2 is the default with opts == NULL.
                        FDIGA_ORTH_CGS2: classical Gram-Schmidt twice;
                        FDIGA_ORTH_CGS_DGKS: the second pass only when ||w'|| < ||w|| / sqrt(2) (with the FD
                        preconditioner A P^{-1} ~ I, so that test fails at every step and CGS2 is faster);
                        FDIGA_ORTH_DCGS2: CGS2 with the second projection delayed by one step and fused with
                        the next step's first (one reduction and two passes over the basis per step, the
                        Arnoldi relation unchanged up to rounding; one extra P^{-1} + A application per cycle) */
  int use_x0;        /* 1: x holds the initial guess; 0: x0 = 0 */
  int profile;       /* 1: per-stage breakdown in the report (gmres_report.t_*_ms): the cycles are launched
                        eagerly (not from the captured graph) with a CUDA event at every stage change, so the
                        total is slightly above a graph-launched solve's; 0: no breakdown (t_*_ms = -1) */
} gmres_opts;

typedef struct {
  int iters;              /* Arnoldi steps (one P^{-1} apply + one matvec each) */
  int restarts;           /* cycles started */
  int converged;
  int reorth;             /* DGKS second passes taken */
  double rel_res_true;    /* ||b - A x|| / ||b|| at return */
  double rel_res_implicit;/* |g_{j+1}| / ||b|| of the last step */
  double t_total_ms;
  double* history;        /* optional (caller-owned, length history_cap): implicit rel. residual per step */
  int history_cap;
  /* per-stage device time of a profiled solve (gmres_opts.profile = 1; else -1), summing to t_total_ms:
   * t_fd_ms     FD applies P^{-1} (eq:FD2D/eq:FD3D), Arnoldi steps and cycle closes
   * t_matvec_ms collocation matvecs A x (eq:collocationsystem), incl. the true residuals
   * t_orth_ms   Gram-Schmidt passes, Givens/least-squares decisions, basis combination
   * t_comm_ms   collectives of a sharded solve (halo exchange, slab transpose, all-reduce; 0 on one rank)
   * t_other_ms  the rest (residual scaling, x update, host round trips at cycle boundaries) */
  double t_fd_ms, t_matvec_ms, t_orth_ms, t_comm_ms, t_other_ms;
} gmres_report;

/* Right-preconditioned restarted GMRES(m) (Saad & Schultz 1986):
 * solve A x = b with A P^{-1} y = b, x = P^{-1} y.  P == NULL: unpreconditioned.
 * b, x: device, local slab.  opts/report may be NULL (defaults / no report).  Synchronises. */
int gmres_solve(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const double* b, double* x,
                const gmres_opts* opts, gmres_report* report);

/* ----------------------------------------------------------------- BiCGStab ---- */

typedef struct {
  double rtol;    /* stop when the recursive residual <= rtol ||b|| (default 1e-8) */
  int max_iters;  /* full iterations (default 1000) */
  int use_x0;     /* 1: x holds the initial guess; 0: x0 = 0 */
} bicgstab_opts;

typedef struct {
  double iters;            /* half-iteration count: k - 0.5 when the BiCG half of iteration k converged */
  int converged;
  int breakdown;           /* rho, r^.v or t.t vanished (or a non-finite value) before convergence */
  int half;                /* 1 when convergence happened at a BiCG half step */
  double rel_res_true;     /* ||b - A x|| / ||b|| at return */
  double rel_res_recursive;/* the recursive residual that met the test */
  double t_total_ms;
  double* history;         /* optional (caller-owned, length history_cap): recursive rel. residual per half step */
  int history_cap;
} bicgstab_report;

/* Right-preconditioned BiCGStab (van der Vorst 1992), the paper's solver: every iteration is
 * a BiCG step then one GMRES(1) step, each with one P^{-1} apply and one matvec; shadow residual r^ = r_0.
 * b, x: device, local slab.  Returns NOT_CONVERGED / BREAKDOWN with the report filled.  Synchronises. */
int bicgstab_solve(fdiga_ctx* ctx, fdiga_stencil* A, fd_plan* P, const double* b, double* x,
                   const bicgstab_opts* opts, bicgstab_report* report);

/* ------------------------------------------------------------ instrumentation ---- */
/* Number of kernels this library launched since the context was created (all entry points). */
int64_t fdiga_kernel_launches(const fdiga_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FDIGA_H */
