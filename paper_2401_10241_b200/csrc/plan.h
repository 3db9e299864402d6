// Per-stage operation plan of one iteration with P2P messages (host only).
//
// The NCCL runner (comm.cpp) executes exactly this sequence, and the gloo
// multi-process test (tests/test_comm_plan_gloo.py) executes it on CPU, so the
// message matching across ranks is tested without GPUs.
//
// Channels per adjacent pair: ACT (s -> s+1, activations after F, then the
// post-validation partial state) and GRAD (s+1 -> s, input gradients after B,
// then the full state).  Message order on each channel is the microbatch order.
//
// Post-validation speculation ("during the warm-up phase of the
// next iteration ... a rollback will be issued ... and then we redo"; DESIGN.md
// R-pv): stage s runs its first n'_s Fs of iteration i+1 on not-yet-validated
// weights, with n'_0 = leading Fs of stage 0 and n'_s = min(leading Fs of s,
// n'_{s-1}); then it VALIDATEs (receives the full state on GRAD, forwards it).
// If the full state amends the weights (clip needed or non-finite) every stage
// REPLAYs its n'_s speculative Fs.  On ACT, stage s-1 then emits its n'_{s-1}
// speculative messages, its n'_{s-1} replays, then F(j >= n'_{s-1}); stage s
// drains the stale messages [n'_s, n'_{s-1}) and maps F(j) -> message n'_{s-1}+j.
#pragma once
#include <cstdint>
#include <vector>

#include "zb.h"

namespace zb {
namespace plan {

enum OpType : int32_t {
  OP_F = 0, OP_B = 1, OP_W = 2,
  OP_RECV_ACT = 3, OP_SEND_ACT = 4, OP_RECV_GRAD = 5, OP_SEND_GRAD = 6,
  OP_VALIDATE = 7, OP_DISCARD_ACT = 8, OP_REPLAY_F = 9,
  OP_WP = 10,        // one W sub-computation: W unit `msg` of microbatch `mb` (data parallel tail)
  OP_ALLREDUCE = 11  // data-parallel gradient all-reduce of W unit `msg` (-1: the vector region)
};

struct Op {
  int32_t type, mb, msg, slot;
};

// n'_s of every stage (see header comment)
std::vector<int> speculative_counts(const zb_pass_t* passes, int n, int p);

// Plan of `stage` for one iteration.  pv_pending: a post-validation of the
// previous step is outstanding (validate at n'_stage); amend: the outcome of
// that validation changes weights (replays).  fused: 1F1B's monolithic
// backward (the gradient is sent after the W that follows its B).
std::vector<Op> stage_plan(const zb_pass_t* passes, int n, int p, int m, int stage, bool pv_pending, bool amend,
                           bool fused);

// ---- data parallelism (App. A) ---------------------------
// D replicas of the pipeline; the stage's gradients are summed over its D replicas by an
// all-reduce before the optimizer step.  A stage's W pass is n_units independent weight
// gradient computations ("W units", Ctx::weight_unit order: the LM head on the last stage,
// then per layer from the top fc2, fc1, proj, qkv, then the embedding on stage 0).  The W
// passes at the TAIL of the stage's list (the maximal run of W ops ending the plan) become
// OP_WP ops, one per (unit, microbatch), and each unit's OP_ALLREDUCE follows its last OP_WP:
//   reorder = false  microbatch-major (the original W passes): the all-reduces can only
//                    start inside the last tail W (App. A Fig. "poor overlapping")
//   reorder = true   unit-major: all tail sub-computations of one parameter are clustered, so
//                    its all-reduce overlaps the next parameter's sub-computations (App. A)
// A final OP_ALLREDUCE(-1) sums the vector region (LayerNorm gammas / betas, biases).
std::vector<Op> dp_tail(const std::vector<Op>& ops, int n_units, bool reorder);

// ---- workers holding several model chunks (zb_schedule_chunked: ZB-V, 1F1B-I) ----------
// Every chunk is a virtual stage v of an nv-stage chain (its own context and channels to
// v-1 / v+1); a worker executes the ops of its chunks in ITS pass order: the plan of each
// chunk (stage_plan over nv virtual stages, no post-validation speculation) is cut into one
// group per pass ([RECV] pass [SEND]) and the groups are merged in the order in which the
// worker's passes appear in `passes`.  worker_of[v] gives the worker of every virtual stage.
struct WOp {
  int32_t chunk;  // virtual stage the op belongs to
  Op op;
};
std::vector<WOp> worker_plan(const zb_pass_t* passes, int n, int nv, int m, int worker, const int* worker_of,
                             bool fused);

}  // namespace plan
}  // namespace zb
