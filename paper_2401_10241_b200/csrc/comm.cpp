// NCCL transport (see comm.h).  Placeholder until the multi-process runner lands:
// attaching fails loudly instead of silently degrading.
#include "comm.h"

#include <stdexcept>

#include "abi_util.h"

namespace zb {

Comm::~Comm() {}
cudaEvent_t Comm::event() { return nullptr; }

void nccl_unique_id(void*) { throw Error(ZB_ENCCL, "NCCL transport not built in this version"); }
void attach_nccl(Ctx&, const void*, int, int) { throw Error(ZB_ENCCL, "NCCL transport not built in this version"); }
void run_iteration_nccl(Ctx&, const zb_pass_t*, int, const int32_t*, const int32_t*, int) {
  throw Error(ZB_ENCCL, "NCCL transport not built in this version");
}
void pv_recv_partial(Ctx&) { throw Error(ZB_ENCCL, "NCCL transport not built in this version"); }
void pv_send_partial(Ctx&) { throw Error(ZB_ENCCL, "NCCL transport not built in this version"); }
void pv_recv_full(Ctx&) { throw Error(ZB_ENCCL, "NCCL transport not built in this version"); }
void pv_send_full(Ctx&) { throw Error(ZB_ENCCL, "NCCL transport not built in this version"); }

}  // namespace zb
