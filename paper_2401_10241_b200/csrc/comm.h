// P2P transport between adjacent pipeline stages: NCCL (one process per GPU)
// or an in-process loopback group (p stages on one GPU, one host thread each).
//
// libnccl.so.2 is loaded lazily with dlopen (the single-GPU path never needs
// it).  Every adjacent pair (s, s+1) gets two 2-rank communicators: one for
// activations s -> s+1 and one for gradients s+1 -> s (separate
// directions never head-of-line block each other); each communicator is
// driven by its own stream on each side, and its message order is the
// microbatch order of the passes that produce / consume it, which is the same
// on both ends for every schedule (F and B lists are microbatch-monotone).
// The post-validation partial state rides the activation channel (after the
// iteration's last activation) and the full state rides the gradient channel
// (before the next iteration's first gradient).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "zb.h"

namespace zb {

struct Ctx;

// Point-to-point transport of one stage.  Channels (which):
//   0 activations to stage+1, 1 activations from stage-1,
//   2 gradients to stage-1,   3 gradients from stage+1.
// send / recv are enqueued on the channel's stream (stream[which]) and are
// asynchronous with respect to the host; messages on a channel are matched
// in order.
struct Transport {
  virtual ~Transport() = default;
  virtual void send(int which, const void* buf, size_t bytes, cudaStream_t st) = 0;
  virtual void recv(int which, void* buf, size_t bytes, cudaStream_t st) = 0;
};

// In-process loopback group: p contexts of one process (each driven by its
// own host thread) exchange messages through device staging buffers, so the
// multi-stage runner below executes unchanged on one GPU.  A send copies the
// payload into a staging buffer on the sender's channel stream and queues it
// (never blocks the host: eager semantics); a recv blocks the calling host
// thread until the matching message is queued (bounded wait, then ZB_EINTERNAL),
// then copies it out on the receiver's channel stream.
struct LoopbackGroup;
std::shared_ptr<LoopbackGroup> loopback_create(int world);
void attach_loopback(Ctx& c, const std::shared_ptr<LoopbackGroup>& g, int rank);

struct Comm {
  int rank = 0, world = 1;
  std::unique_ptr<Transport> tx;
  cudaStream_t stream[4] = {nullptr, nullptr, nullptr, nullptr};  // per channel (nullptr where absent)
  // send staging ring for activations (written by F, drained by the act-send stream)
  std::vector<void*> act_buf;
  std::vector<cudaEvent_t> act_buf_free;
  int act_next = 0;
  // send staging ring for f32 input gradients (written by B, drained by the grad-send stream)
  std::vector<float*> grad_buf;
  std::vector<cudaEvent_t> grad_buf_free;
  std::vector<cudaEvent_t> ev_pool;
  int ev_next = 0;
  void* scalars = nullptr;  // 2 x 16 B device buffer for PV messages
  ~Comm();
  cudaEvent_t event();
};

// Data parallelism: the D replicas of one stage share a
// D-rank communicator; gradient all-reduces (f32 sum, in place) run on its own stream, each
// ordered after the W unit that completes its gradient (plan.h dp_tail), so they overlap the
// remaining W work; the compute stream joins them at the end of the iteration (before the
// post-validation norm and the optimizer step).
struct DpComm {
  void* comm = nullptr;  // nullptr when world == 1
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> ev;
  int ev_next = 0;
  int64_t reduces = 0;  // all-reduce calls issued
  ~DpComm();
  cudaEvent_t event();
};
void attach_dp(Ctx& c, const void* id128, int dp_rank, int dp_world);
void dp_all_reduce(Ctx& c, int unit);  // after everything enqueued so far on the compute stream
void dp_join(Ctx& c);                  // the compute stream waits for every all-reduce issued
int64_t dp_reduce_count(const Ctx& c);

// ncclGetUniqueId through dlopen'ed libnccl (128 bytes).
void nccl_unique_id(void* id128);
// ids: 2*(world-1) unique ids, [k] for the activation comm of pair (k, k+1),
// [world-1+k] for the gradient comm of the same pair.
void attach_nccl(Ctx& c, const void* ids, int rank, int world);
// Chunk contexts (virtual stages v of nv) of worker `me` of a chunked schedule: links to
// chunks on other workers get 2-rank NCCL communicators (ids as attach_nccl with world =
// nv: [k] activations of link (k, k+1), [nv-1+k] its gradients), links between two chunks
// of this worker an in-process loopback channel.
void attach_nccl_chunks(const std::vector<Ctx*>& chunks, const void* ids, int nv, const std::vector<int>& worker_of,
                        int me);
// One iteration of this stage's passes with NCCL send / recv.
void run_iteration_nccl(Ctx& c, const zb_pass_t* passes, int n, const int32_t* tokens, const int32_t* labels,
                        int flags);
// One iteration of a WORKER holding several chunk contexts (virtual stages of a chunked
// schedule, zb_schedule_chunked): the chunks' plans merged in the worker's pass order
// (plan::worker_plan).  Every chunk context must be attached to a transport as virtual
// stage cfg.stage of cfg.p; post-validation must be finished before the next iteration.
void run_iteration_worker(const std::vector<Ctx*>& chunks, const zb_pass_t* passes, int n, const int32_t* tokens,
                          const int32_t* labels, int flags);
// Median round trip (ns) of one `bytes` message to stage+1 and back (0 on the last stage).
int64_t comm_probe(Ctx& c, size_t bytes, int iters);
// Post-validation chain messages over the attached communicators.
void pv_recv_partial(Ctx& c);
void pv_send_partial(Ctx& c);
void pv_recv_full(Ctx& c);
void pv_send_full(Ctx& c);

}  // namespace zb
