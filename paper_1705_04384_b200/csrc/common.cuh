// Internal helpers shared by the libfdiga translation units (never exported).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/fdiga.h"

namespace fdiga {

// Thread-local last-error text (fdiga_last_error).
void set_error(const char* fmt, ...);

#define FDIGA_CUDA(call)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::fdiga::set_error("CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), __FILE__,   \
                         __LINE__, #call);                                                  \
      return FDIGA_ERR_CUDA;                                                                \
    }                                                                                       \
  } while (0)

#define FDIGA_CHECK(cond, code, ...)   \
  do {                                 \
    if (!(cond)) {                     \
      ::fdiga::set_error(__VA_ARGS__); \
      return (code);                   \
    }                                  \
  } while (0)

#define FDIGA_TRY(call)           \
  do {                            \
    int s_ = (call);              \
    if (s_ != FDIGA_OK) return s_; \
  } while (0)

// Growable device scratch buffer (doubles).
struct DevBuf {
  double* p = nullptr;
  size_t cap = 0;
  int ensure(size_t n) {
    if (n <= cap) return FDIGA_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    FDIGA_CUDA(cudaMalloc(&p, n * sizeof(double)));
    cap = n;
    return FDIGA_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// One point-to-point message of an exchange (comm.cu): peer rank, device buffer, size in bytes.
struct P2PMsg {
  int peer;
  void* ptr;
  size_t bytes;
};

constexpr int FDIGA_MAX_RANKS = 64;

}  // namespace fdiga

struct fdiga_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nranks = 1, rank = 0;
  void* nccl_comm = nullptr;  // ncclComm_t when nranks > 1 (NCCL transport)
  fdiga_loopback* hub = nullptr;  // loopback transport (nranks contexts in one process), else NULL
  bool sharded = false;           // slab-sharded code path (a process group was given, even of 1 rank)
  int sm_count = 148;
  int64_t launches = 0;       // kernels launched by this context
  double* pinned = nullptr;   // small pinned host scratch (scalars coming back from reductions)
  size_t pinned_cap = 0;
  fdiga::DevBuf ws[4];        // GMRES workspace: basis V, z/w vectors, reduction partials, device state
  void* gmres_graph = nullptr; // cached captured GMRES cycle (krylov.cu)
  void* bicg_graph = nullptr;  // cached captured BiCGStab iterations (bicgstab.cu)
  void* solver = nullptr;      // cached cuSOLVER handle of fd_setup (fd.cu)
  // stage profiling of a solve (gmres_opts.profile): events recorded on the stream at every stage change;
  // interval [e_i, e_{i+1}) is charged to the stage of e_i (fdiga::prof_mark)
  std::vector<std::pair<int, cudaEvent_t>>* prof = nullptr;
  int prof_stage = 0;
  int nvtx_stage_open = -1;  // FDIGA_NVTX: -1 outside a solve, 0 inside without an open stage range, 1 with one
};

namespace fdiga {
// NVTX ranges (FDIGA_NVTX=1; header-only NVTX 3, no link dependency): one per API call (NvtxRange) and one per
// solve stage (prof_mark), so that profilers can filter by stage (ncu --nvtx --nvtx-include "fdiga:fd/").
inline bool nvtx_on() {
  static const bool on = [] {
    const char* e = std::getenv("FDIGA_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(nvtx_on()) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
inline void count_launch(fdiga_ctx* c, int k = 1) { c->launches += k; }
// solve stages for gmres_report's breakdown
enum { PROF_OTHER = 0, PROF_FD = 1, PROF_MATVEC = 2, PROF_ORTH = 3, PROF_COMM = 4, PROF_NSTAGE = 5 };
// start charging the stream's time to `stage` (no-op unless a profiled solve is running); returns the
// previous stage
inline int prof_mark(fdiga_ctx* c, int stage) {
  const int prev = c->prof_stage;
  if (nvtx_on() && c->nvtx_stage_open >= 0) {  // inside a solve: close the previous stage's range, open the next
    static const char* const names[PROF_NSTAGE] = {"fdiga:other", "fdiga:fd", "fdiga:matvec", "fdiga:orth", "fdiga:comm"};
    if (c->nvtx_stage_open) nvtxRangePop();
    nvtxRangePushA(names[stage]);
    c->nvtx_stage_open = 1;
    if (!c->prof) c->prof_stage = stage;
  }
  if (!c->prof) return prev;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) == cudaSuccess) {
    cudaEventRecord(e, c->stream);
    c->prof->push_back({stage, e});
  }
  c->prof_stage = stage;
  return prev;
}
// NVTX scope of a solve: the call's range plus the stage ranges prof_mark opens and closes inside it
struct NvtxSolveScope {
  fdiga_ctx* c;
  bool on;
  NvtxSolveScope(fdiga_ctx* ctx, const char* name) : c(ctx), on(nvtx_on()) {
    if (!on) return;
    nvtxRangePushA(name);
    c->nvtx_stage_open = 0;
  }
  ~NvtxSolveScope() {
    if (!on) return;
    if (c->nvtx_stage_open == 1) nvtxRangePop();
    c->nvtx_stage_open = -1;
    nvtxRangePop();
  }
  NvtxSolveScope(const NvtxSolveScope&) = delete;
  NvtxSolveScope& operator=(const NvtxSolveScope&) = delete;
};
void destroy_solver(fdiga_ctx* ctx);
// Set the device of the context for the calling thread.
inline int bind(const fdiga_ctx* c) {
  FDIGA_CUDA(cudaSetDevice(c->device));
  return FDIGA_OK;
}
int ensure_pinned(fdiga_ctx* c, size_t n_doubles);
// Internal variants with a device "skip" flag (nonzero: every launch is a no-op), used by the
// captured GMRES cycle graph for early exit.
int fd_apply_ex(fd_plan* P, const double* r, double* s, const int* skip);
int stencil_matvec_ex(fdiga_stencil* S, const double* x, double* y, const int* skip);
// Balanced split of [0, n) into nparts ranges; the first n % nparts get one extra element.
void partition(int64_t n, int nparts, int part, int64_t* begin, int64_t* end);
// Collectives on ctx->stream (comm.cu).  Every rank calls them in the same order.
int comm_exchange(fdiga_ctx* ctx, const std::vector<P2PMsg>& sends, const std::vector<P2PMsg>& recvs);
int comm_allreduce(fdiga_ctx* ctx, const double* send, double* recv, size_t count);  // sum, same bits on all ranks
bool comm_capturable(const fdiga_ctx* ctx);  // false for the loopback transport (host barriers)
int loopback_attach(fdiga_ctx* ctx, fdiga_loopback* hub);
// Rows of this rank's slab of a (possibly sharded) stencil.
int64_t stencil_local_rows(const fdiga_stencil* S);
int64_t fd_plan_local_size(const fd_plan* P);
// Drop the cached GMRES graph (it captures pointers of A, P and the workspace).
void destroy_gmres_graph(fdiga_ctx* ctx);  // also drops the BiCGStab graph
void destroy_bicgstab_graph(fdiga_ctx* ctx);
}  // namespace fdiga
