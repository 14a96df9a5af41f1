// rbd_comm.cu — multi-GPU plumbing (placeholder until the sharded path lands).
#include <string>

#include "rbd_cuda.h"

struct rbd_ctx_s;

void rbd_comm_release(rbd_ctx_t) {}

extern "C" {

int rbd_comm_unique_id(char out[RBD_UNIQUE_ID_BYTES]) {
  (void)out;
  return RBD_ERR_NCCL;
}

int rbd_ctx_init_comm(rbd_ctx_t, int, int, const char*) { return RBD_ERR_NCCL; }

int rbd_decompose_sharded(rbd_ctx_t, const double*, int64_t, int64_t, int64_t, int64_t, int64_t,
                          const rbd_config_t*, double*, double*, int64_t*, double*,
                          rbd_result_t*) {
  return RBD_ERR_NCCL;
}
}
