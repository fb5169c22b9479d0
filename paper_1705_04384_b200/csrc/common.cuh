// Internal helpers shared by the libfdiga translation units (never exported).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
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

}  // namespace fdiga

struct fdiga_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nranks = 1, rank = 0;
  void* nccl_comm = nullptr;  // ncclComm_t when nranks > 1
  int sm_count = 148;
  int64_t launches = 0;       // kernels launched by this context
  double* pinned = nullptr;   // small pinned host scratch (scalars coming back from reductions)
  size_t pinned_cap = 0;
  fdiga::DevBuf ws[4];        // GMRES workspace: basis V, z/w vectors, reduction partials, device state
  void* gmres_graph = nullptr; // cached captured GMRES cycle (krylov.cu)
};

namespace fdiga {
inline void count_launch(fdiga_ctx* c, int k = 1) { c->launches += k; }
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
// Drop the cached GMRES graph (it captures pointers of A, P and the workspace).
void destroy_gmres_graph(fdiga_ctx* ctx);
}  // namespace fdiga
