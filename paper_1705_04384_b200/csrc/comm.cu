// Multi-rank communicator (NCCL over NVLink).  This version is single-rank: ctx creation with
// nranks > 1 reports NOT_SUPPORTED.
#include "common.cuh"

using namespace fdiga;

extern "C" {
int fdiga_comm_init(fdiga_ctx* ctx, const void* uid) {
  (void)ctx;
  (void)uid;
  set_error("multi-rank contexts are not built in this version of libfdiga");
  return FDIGA_ERR_NOT_SUPPORTED;
}
int fdiga_comm_destroy(fdiga_ctx* ctx) {
  (void)ctx;
  return FDIGA_OK;
}
int fdiga_nccl_unique_id(void* out128) {
  (void)out128;
  set_error("NCCL is not linked in this version of libfdiga");
  return FDIGA_ERR_NOT_SUPPORTED;
}
}
