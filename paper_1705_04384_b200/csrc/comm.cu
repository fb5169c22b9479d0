// Multi-rank transport for the slab-sharded path.
//
// Two transports behind one internal interface (common.cuh):
//   * NCCL (one process per GPU, NVLink/NVSwitch): grouped ncclSend/ncclRecv for the FD mode-d
//     slab transpose and the matvec halo planes, ncclAllReduce for the GMRES dot products.  libnccl is
//     resolved at run time (dlopen of the copy torch already loaded, soname libnccl.so.2), so only one
//     NCCL is ever present in the process and the library loads on hosts without NCCL.
//   * loopback: nranks contexts inside ONE process on ONE device, each driven by its own host thread
//     (fdiga_loopback_create / fdiga_ctx_create_loopback).  A hub exchanges pointers and CUDA events
//     between the threads; receivers copy straight from the senders' buffers (device-to-device) after
//     waiting on the senders' events, so no kernel ever spins on another rank.  It runs the sharded
//     kernels and data movement of every rank on a single GPU (tests) and is the reference the NCCL
//     path must agree with.  Host barriers make it non-capturable (GMRES then runs uncaptured).
//
// Every exchange is described by (peer, pointer, bytes) lists; messages between one (src, dst) pair
// are matched in issue order, as in NCCL point-to-point semantics.
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include <nccl.h>

#include "common.cuh"

using namespace fdiga;

// ------------------------------------------------------------------------------------- NCCL (dlopen)
namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

int nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.loaded) return FDIGA_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  FDIGA_CHECK(h != nullptr, FDIGA_ERR_NCCL, "cannot load libnccl.so.2 (import torch first): %s", dlerror());
#define FDIGA_SYM(field, name)                                                              \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));                 \
  FDIGA_CHECK(g_nccl.field != nullptr, FDIGA_ERR_NCCL, "libnccl.so.2 lacks %s", name);
  FDIGA_SYM(GetUniqueId, "ncclGetUniqueId")
  FDIGA_SYM(CommInitRank, "ncclCommInitRank")
  FDIGA_SYM(CommDestroy, "ncclCommDestroy")
  FDIGA_SYM(AllReduce, "ncclAllReduce")
  FDIGA_SYM(Send, "ncclSend")
  FDIGA_SYM(Recv, "ncclRecv")
  FDIGA_SYM(GroupStart, "ncclGroupStart")
  FDIGA_SYM(GroupEnd, "ncclGroupEnd")
  FDIGA_SYM(GetErrorString, "ncclGetErrorString")
#undef FDIGA_SYM
  g_nccl.loaded = true;
  return FDIGA_OK;
}

#define FDIGA_NCCL(call)                                                                                  \
  do {                                                                                                    \
    ncclResult_t r_ = (call);                                                                             \
    if (r_ != ncclSuccess) {                                                                              \
      ::fdiga::set_error("NCCL error '%s' at %s:%d (%s)", g_nccl.GetErrorString(r_), __FILE__, __LINE__, \
                         #call);                                                                          \
      return FDIGA_ERR_NCCL;                                                                              \
    }                                                                                                     \
  } while (0)

}  // namespace

// ------------------------------------------------------------------------------------- loopback hub
struct fdiga_loopback {
  int nranks = 0;
  int device = -1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  int refs = 0;
  struct Slot {
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    std::vector<fdiga::P2PMsg> sends;
    const double* ar_send = nullptr;
    bool attached = false;
  };
  std::vector<Slot> slots;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {

// sum of nranks device buffers in rank order (identical bits on every rank)
struct SumArgs {
  const double* src[FDIGA_MAX_RANKS];
  int nsrc;
  double* dst;
  int64_t count;
};

__global__ void loopback_sum_kernel(SumArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = a.src[0][i];
    for (int r = 1; r < a.nsrc; ++r) s += a.src[r][i];
    a.dst[i] = s;
  }
}

int lb_finish(fdiga_ctx* ctx) {
  fdiga_loopback* H = ctx->hub;
  auto& me = H->slots[ctx->rank];
  FDIGA_CUDA(cudaEventRecord(me.done, ctx->stream));
  H->barrier();
  for (int s = 0; s < H->nranks; ++s)
    if (s != ctx->rank) FDIGA_CUDA(cudaStreamWaitEvent(ctx->stream, H->slots[s].done, 0));
  return FDIGA_OK;
}

int lb_exchange(fdiga_ctx* ctx, const std::vector<P2PMsg>& sends, const std::vector<P2PMsg>& recvs) {
  fdiga_loopback* H = ctx->hub;
  auto& me = H->slots[ctx->rank];
  me.sends = sends;
  FDIGA_CUDA(cudaEventRecord(me.ready, ctx->stream));
  H->barrier();
  std::vector<int> used(H->nranks, 0);  // messages from each source consumed so far
  std::vector<char> waited(H->nranks, 0);
  int status = FDIGA_OK;  // a mismatch still completes the protocol (no rank is left in a barrier)
  for (const P2PMsg& r : recvs) {
    const auto& src = H->slots[r.peer];
    int k = 0;
    const P2PMsg* match = nullptr;
    for (const P2PMsg& s : src.sends)
      if (s.peer == ctx->rank && k++ == used[r.peer]) {
        match = &s;
        break;
      }
    if (!match || match->bytes != r.bytes) {
      set_error("loopback: rank %d expects %zu bytes from %d, the sender posted %s", ctx->rank, r.bytes, r.peer,
                match ? "a different size" : "nothing");
      status = FDIGA_ERR_INVALID_ARG;
      continue;
    }
    ++used[r.peer];
    if (!waited[r.peer] && r.peer != ctx->rank) {
      if (cudaStreamWaitEvent(ctx->stream, src.ready, 0) != cudaSuccess) status = FDIGA_ERR_CUDA;
      waited[r.peer] = 1;
    }
    if (r.bytes && cudaMemcpyAsync(r.ptr, match->ptr, r.bytes, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
      status = FDIGA_ERR_CUDA;
  }
  const int s2 = lb_finish(ctx);
  return status != FDIGA_OK ? status : s2;
}

int lb_allreduce(fdiga_ctx* ctx, const double* send, double* recv, size_t count) {
  fdiga_loopback* H = ctx->hub;
  auto& me = H->slots[ctx->rank];
  me.ar_send = send;
  FDIGA_CUDA(cudaEventRecord(me.ready, ctx->stream));
  H->barrier();
  SumArgs a{};
  a.nsrc = H->nranks;
  for (int s = 0; s < H->nranks; ++s) {
    a.src[s] = H->slots[s].ar_send;
    if (s != ctx->rank) FDIGA_CUDA(cudaStreamWaitEvent(ctx->stream, H->slots[s].ready, 0));
  }
  a.dst = recv;
  a.count = (int64_t)count;
  if (count) {
    loopback_sum_kernel<<<(unsigned)std::min<int64_t>((count + 255) / 256, 1024), 256, 0, ctx->stream>>>(a);
    count_launch(ctx);
    FDIGA_CUDA(cudaGetLastError());
  }
  return lb_finish(ctx);
}

}  // namespace

namespace fdiga {

void partition(int64_t n, int nparts, int part, int64_t* begin, int64_t* end) {
  const int64_t q = n / nparts, r = n % nparts;
  *begin = part * q + (part < r ? part : r);
  *end = *begin + q + (part < r ? 1 : 0);
}

bool comm_capturable(const fdiga_ctx* ctx) { return ctx->hub == nullptr; }

int comm_exchange_impl(fdiga_ctx* ctx, const std::vector<P2PMsg>& sends, const std::vector<P2PMsg>& recvs);
int comm_allreduce_impl(fdiga_ctx* ctx, const double* send, double* recv, size_t count);
// the collectives are charged to the COMM stage of a profiled solve
int comm_exchange(fdiga_ctx* ctx, const std::vector<P2PMsg>& sends, const std::vector<P2PMsg>& recvs) {
  const int prev = prof_mark(ctx, PROF_COMM);
  const int s = comm_exchange_impl(ctx, sends, recvs);
  prof_mark(ctx, prev);
  return s;
}
int comm_allreduce(fdiga_ctx* ctx, const double* send, double* recv, size_t count) {
  const int prev = prof_mark(ctx, PROF_COMM);
  const int s = comm_allreduce_impl(ctx, send, recv, count);
  prof_mark(ctx, prev);
  return s;
}
int comm_exchange_impl(fdiga_ctx* ctx, const std::vector<P2PMsg>& sends, const std::vector<P2PMsg>& recvs) {
  if (ctx->hub) return lb_exchange(ctx, sends, recvs);
  if (!ctx->nccl_comm) {  // single rank without a process group: self messages only
    FDIGA_CHECK(sends.size() == recvs.size(), FDIGA_ERR_INVALID_ARG, "unmatched self messages");
    for (size_t i = 0; i < sends.size(); ++i)
      if (sends[i].bytes)
        FDIGA_CUDA(cudaMemcpyAsync(recvs[i].ptr, sends[i].ptr, sends[i].bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    return FDIGA_OK;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  FDIGA_NCCL(g_nccl.GroupStart());
  for (const P2PMsg& s : sends)
    if (s.bytes) FDIGA_NCCL(g_nccl.Send(s.ptr, s.bytes, ncclUint8, s.peer, comm, ctx->stream));
  for (const P2PMsg& r : recvs)
    if (r.bytes) FDIGA_NCCL(g_nccl.Recv(r.ptr, r.bytes, ncclUint8, r.peer, comm, ctx->stream));
  FDIGA_NCCL(g_nccl.GroupEnd());
  return FDIGA_OK;
}

int comm_allreduce_impl(fdiga_ctx* ctx, const double* send, double* recv, size_t count) {
  if (ctx->hub) return lb_allreduce(ctx, send, recv, count);
  if (!ctx->nccl_comm) {
    if (send != recv && count)
      FDIGA_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    return FDIGA_OK;
  }
  FDIGA_NCCL(g_nccl.AllReduce(send, recv, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(ctx->nccl_comm),
                              ctx->stream));
  return FDIGA_OK;
}

}  // namespace fdiga

extern "C" {

int fdiga_comm_init(fdiga_ctx* ctx, const void* uid) {
  FDIGA_TRY(nccl_load());
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  FDIGA_NCCL(g_nccl.CommInitRank(&comm, ctx->nranks, id, ctx->rank));
  ctx->nccl_comm = comm;
  return FDIGA_OK;
}

int fdiga_comm_destroy(fdiga_ctx* ctx) {
  if (ctx->nccl_comm && g_nccl.loaded) g_nccl.CommDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
  ctx->nccl_comm = nullptr;
  if (ctx->hub) {
    fdiga_loopback* H = ctx->hub;
    auto& me = H->slots[ctx->rank];
    // collective: peers may still be enqueueing waits on this rank's events from the last collective
    H->barrier();
    if (me.ready) cudaEventDestroy(me.ready);
    if (me.done) cudaEventDestroy(me.done);
    me.ready = me.done = nullptr;
    std::lock_guard<std::mutex> lk(H->mu);
    me.attached = false;
    --H->refs;
    ctx->hub = nullptr;
  }
  return FDIGA_OK;
}

int fdiga_nccl_unique_id(void* out128) {
  FDIGA_CHECK(out128 != nullptr, FDIGA_ERR_INVALID_ARG, "out is NULL");
  FDIGA_TRY(nccl_load());
  ncclUniqueId id;
  FDIGA_NCCL(g_nccl.GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return FDIGA_OK;
}

int fdiga_loopback_create(int nranks, fdiga_loopback** out) {
  FDIGA_CHECK(out && nranks >= 1 && nranks <= FDIGA_MAX_RANKS, FDIGA_ERR_INVALID_ARG,
              "loopback: nranks must be in [1, %d]", FDIGA_MAX_RANKS);
  fdiga_loopback* H = new fdiga_loopback();
  H->nranks = nranks;
  H->slots.resize(nranks);
  *out = H;
  return FDIGA_OK;
}

int fdiga_loopback_destroy(fdiga_loopback* H) {
  if (!H) return FDIGA_OK;
  {
    std::lock_guard<std::mutex> lk(H->mu);
    FDIGA_CHECK(H->refs == 0, FDIGA_ERR_INVALID_ARG, "loopback hub still has %d attached contexts", H->refs);
  }
  delete H;
  return FDIGA_OK;
}

int fdiga_loopback_nranks(const fdiga_loopback* H, int* n) {
  FDIGA_CHECK(H && n, FDIGA_ERR_INVALID_ARG, "NULL argument");
  *n = H->nranks;
  return FDIGA_OK;
}

int fdiga_transpose_plan(int64_t n_inner, int64_t n_last, int nranks, int rank, int64_t* slab_off, int64_t* slab_cnt,
                         int64_t* tr_off, int64_t* tr_cnt) {
  FDIGA_CHECK(slab_off && slab_cnt && tr_off && tr_cnt && n_inner >= 0 && n_last >= 0 && nranks >= 1 && rank >= 0 &&
                  rank < nranks,
              FDIGA_ERR_INVALID_ARG, "bad fdiga_transpose_plan arguments");
  int64_t o, e, q0, q1;
  partition(n_last, nranks, rank, &o, &e);
  partition(n_inner, nranks, rank, &q0, &q1);
  const int64_t c = e - o, len = q1 - q0;
  for (int q = 0; q < nranks; ++q) {
    int64_t qb, qe, ob, oe;
    partition(n_inner, nranks, q, &qb, &qe);
    partition(n_last, nranks, q, &ob, &oe);
    slab_off[q] = c * qb;  // my c x len_q block of inner chunk q
    slab_cnt[q] = c * (qe - qb);
    tr_off[q] = ob * len;  // rows [ob, oe) of my transposed chunk T(n_last x len)
    tr_cnt[q] = (oe - ob) * len;
  }
  return FDIGA_OK;
}

int fdiga_halo_plan(int64_t n_last, const int32_t* start, const int32_t* width, int nranks, int rank, int64_t* lo,
                    int64_t* hi, int64_t* send_b, int64_t* send_e, int64_t* recv_b, int64_t* recv_e) {
  FDIGA_CHECK(start && width && lo && hi && send_b && send_e && recv_b && recv_e && n_last >= 0 && nranks >= 1 &&
                  rank >= 0 && rank < nranks,
              FDIGA_ERR_INVALID_ARG, "bad fdiga_halo_plan arguments");
  // planes [lo, hi) read by the rows of slab [o, e): the union of their last-axis column windows
  auto need = [&](int64_t ob, int64_t oe, int64_t* l, int64_t* h) {
    *l = ob;
    *h = oe;
    for (int64_t i = ob; i < oe; ++i) {
      *l = std::min<int64_t>(*l, start[i]);
      *h = std::max<int64_t>(*h, (int64_t)start[i] + width[i]);
    }
  };
  int64_t o, e;
  partition(n_last, nranks, rank, &o, &e);
  need(o, e, lo, hi);
  for (int q = 0; q < nranks; ++q) {
    send_b[q] = send_e[q] = recv_b[q] = recv_e[q] = 0;
    if (q == rank) continue;
    int64_t qo, qe, qlo, qhi;
    partition(n_last, nranks, q, &qo, &qe);
    need(qo, qe, &qlo, &qhi);
    // my planes inside q's halo (below q's slab if q is above me, above it otherwise)
    const int64_t sb = std::max(o, q > rank ? qlo : qe), se = std::min(e, q > rank ? qo : qhi);
    if (se > sb) {
      send_b[q] = sb;
      send_e[q] = se;
    }
    // q's planes inside my halo
    const int64_t rb = std::max(qo, q < rank ? *lo : e), re = std::min(qe, q < rank ? o : *hi);
    if (re > rb) {
      recv_b[q] = rb;
      recv_e[q] = re;
    }
  }
  return FDIGA_OK;
}

int fdiga_partition(int64_t n, int nparts, int part, int64_t* begin, int64_t* end) {
  FDIGA_CHECK(begin && end && n >= 0 && nparts >= 1 && part >= 0 && part < nparts, FDIGA_ERR_INVALID_ARG,
              "bad fdiga_partition arguments");
  partition(n, nparts, part, begin, end);
  return FDIGA_OK;
}

}  // extern "C"

namespace fdiga {
// attach a freshly created context to a hub (ctx.cu)
int loopback_attach(fdiga_ctx* ctx, fdiga_loopback* H) {
  {
    std::lock_guard<std::mutex> lk(H->mu);
    FDIGA_CHECK(!H->slots[ctx->rank].attached, FDIGA_ERR_INVALID_ARG, "loopback rank %d already attached",
                ctx->rank);
    FDIGA_CHECK(H->device < 0 || H->device == ctx->device, FDIGA_ERR_NOT_SUPPORTED,
                "loopback ranks must share one device");
    H->device = ctx->device;
    H->slots[ctx->rank].attached = true;
    ++H->refs;
  }
  auto& me = H->slots[ctx->rank];
  FDIGA_CUDA(cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming));
  FDIGA_CUDA(cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming));
  me.stream = ctx->stream;
  ctx->hub = H;
  ctx->sharded = true;
  return FDIGA_OK;
}
}  // namespace fdiga
