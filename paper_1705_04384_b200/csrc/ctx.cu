// Context, status strings, error plumbing.
#include <cstdarg>
#include <cstring>

#include "common.cuh"

namespace fdiga {
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int ensure_pinned(fdiga_ctx* c, size_t n) {
  if (n <= c->pinned_cap) return FDIGA_OK;
  if (c->pinned) cudaFreeHost(c->pinned);
  c->pinned = nullptr;
  c->pinned_cap = 0;
  FDIGA_CUDA(cudaMallocHost(&c->pinned, n * sizeof(double)));
  c->pinned_cap = n;
  return FDIGA_OK;
}
}  // namespace fdiga

using namespace fdiga;

extern "C" {

const char* fdiga_last_error(void) { return g_err; }

const char* fdiga_status_string(int s) {
  switch (s) {
    case FDIGA_OK: return "OK";
    case FDIGA_ERR_INVALID_ARG: return "INVALID_ARG";
    case FDIGA_ERR_CUDA: return "CUDA";
    case FDIGA_ERR_CUSOLVER: return "CUSOLVER";
    case FDIGA_ERR_NCCL: return "NCCL";
    case FDIGA_ERR_COMPLEX_SPECTRUM: return "COMPLEX_SPECTRUM";
    case FDIGA_ERR_ILL_CONDITIONED: return "ILL_CONDITIONED";
    case FDIGA_ERR_SINGULAR: return "SINGULAR";
    case FDIGA_ERR_NOT_CONVERGED: return "NOT_CONVERGED";
    case FDIGA_ERR_BREAKDOWN: return "BREAKDOWN";
    case FDIGA_ERR_NOT_SUPPORTED: return "NOT_SUPPORTED";
    case FDIGA_ERR_OOM: return "OOM";
    default: return "UNKNOWN";
  }
}

int fdiga_comm_init(fdiga_ctx* ctx, const void* uid);      // comm.cu
int fdiga_comm_destroy(fdiga_ctx* ctx);                     // comm.cu
int fdiga_loopback_nranks(const fdiga_loopback* hub, int* n); // comm.cu

namespace {
int ctx_new(int device, void* cuda_stream, int nranks, int rank, fdiga_ctx** out) {
  FDIGA_CHECK(out != nullptr, FDIGA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  FDIGA_CHECK(nranks >= 1 && nranks <= FDIGA_MAX_RANKS && rank >= 0 && rank < nranks, FDIGA_ERR_INVALID_ARG,
              "bad nranks/rank %d/%d", nranks, rank);
  int ndev = 0;
  FDIGA_CUDA(cudaGetDeviceCount(&ndev));
  FDIGA_CHECK(device >= 0 && device < ndev, FDIGA_ERR_INVALID_ARG, "device %d out of range (%d devices)", device,
              ndev);
  FDIGA_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  FDIGA_CUDA(cudaGetDeviceProperties(&prop, device));
  FDIGA_CHECK(prop.major == 10 && prop.minor == 0, FDIGA_ERR_NOT_SUPPORTED,
              "libfdiga is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major, prop.minor);
  fdiga_ctx* c = new fdiga_ctx();
  c->device = device;
  c->nranks = nranks;
  c->rank = rank;
  c->sm_count = prop.multiProcessorCount;
  // NULL selects the legacy default stream (ordered with every blocking stream, e.g. torch's default)
  c->stream = (cudaStream_t)cuda_stream;
  c->own_stream = false;
  *out = c;
  return FDIGA_OK;
}
}  // namespace

int fdiga_ctx_create(int device, void* cuda_stream, int nranks, int rank, const void* nccl_unique_id,
                     fdiga_ctx** out) {
  FDIGA_CHECK(nranks == 1 || nccl_unique_id != nullptr, FDIGA_ERR_INVALID_ARG,
              "nccl_unique_id required when nranks > 1");
  // a unique id (even with nranks == 1) selects the NCCL transport and the sharded code path
  fdiga_ctx* c = nullptr;
  FDIGA_TRY(ctx_new(device, cuda_stream, nranks, rank, &c));
  if (nccl_unique_id != nullptr) {
    c->sharded = true;
    int s = fdiga_comm_init(c, nccl_unique_id);
    if (s != FDIGA_OK) {
      delete c;
      return s;
    }
  }
  *out = c;
  return FDIGA_OK;
}

int fdiga_ctx_create_loopback(int device, void* cuda_stream, fdiga_loopback* hub, int rank, fdiga_ctx** out) {
  FDIGA_CHECK(hub != nullptr, FDIGA_ERR_INVALID_ARG, "hub is NULL");
  int nr = 0;
  FDIGA_TRY(fdiga_loopback_nranks(hub, &nr));
  fdiga_ctx* c = nullptr;
  FDIGA_TRY(ctx_new(device, cuda_stream, nr, rank, &c));
  int s = loopback_attach(c, hub);
  if (s != FDIGA_OK) {
    delete c;
    return s;
  }
  *out = c;
  return FDIGA_OK;
}

int fdiga_ctx_destroy(fdiga_ctx* c) {
  if (!c) return FDIGA_OK;
  cudaSetDevice(c->device);
  if (c->nccl_comm || c->hub) fdiga_comm_destroy(c);
  destroy_gmres_graph(c);
  destroy_solver(c);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto& b : c->ws) b.release();
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return FDIGA_OK;
}

int fdiga_slab(const fdiga_ctx* c, int64_t n_last, int64_t* begin, int64_t* end) {
  FDIGA_CHECK(c && begin && end && n_last >= 0, FDIGA_ERR_INVALID_ARG, "bad fdiga_slab arguments");
  partition(n_last, c->nranks, c->rank, begin, end);
  return FDIGA_OK;
}

int64_t fdiga_kernel_launches(const fdiga_ctx* c) { return c ? c->launches : -1; }

}  // extern "C"
