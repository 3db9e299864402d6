// Stage context: one pipeline stage on one GPU (include/zb.h zb_ctx_t).
//
// Arena layout (all carved from one caller-owned device buffer, 256-B aligned):
//   params   f32 master theta, f32 grads, f32 AdamW m / v (flat; matrices and
//            embeddings first = the weight-decay region; linear matrices first
//            of all = the bf16 shadow region), bf16 shadow (bf16 mode)
//   slots    n_slots x stash slot: per layer X, LN1, QKV, O,
//            X1, LN2, U, G [T, *] + f32 stats; per slot DY [T,h], tokens,
//            labels; last stage XL, LNF [T,h]
//   scratch  spare QKV [T,3h] (pointer-swapped with a slot's QKV in B),
//            dO / dLN [T,h], attention delta, logits f32
//            [T,V] + dlogits [T,V] (last stage), loss rows, sort keys,
//            token / label staging [m,T], optimizer scratch.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "ops.h"
#include "zb.h"

namespace zb {

struct Comm;  // NCCL transport (comm.cpp)
struct DpComm;  // data-parallel all-reduce communicator (comm.cu)

struct LayerW {
  float *ln1_g, *ln1_b, *qkv_b, *proj_b, *ln2_g, *ln2_b, *fc1_b, *fc2_b;  // f32 master
  void *qkv_w, *proj_w, *fc1_w, *fc2_w;                                  // compute copies
  float *g_ln1_g, *g_ln1_b, *g_qkv_b, *g_proj_b, *g_ln2_g, *g_ln2_b, *g_fc1_b, *g_fc2_b;
  float *g_qkv_w, *g_proj_w, *g_fc1_w, *g_fc2_w;
};

struct LayerAct {
  void *x, *ln1, *qkv, *o, *x1, *ln2, *u, *g;
  float *mu1, *rs1, *mu2, *rs2, *lse;
};

struct Slot {
  std::vector<LayerAct> L;
  void* dlogits;  // last stage, head W in the W pass: bf16 / f32 [T, V] from B to W (else null)
  void* dy;       // gradient of the stage output, activation dtype (GEMM operand in B and W)
  float* dy32;    // the same gradient in f32 as received from stage+1 (residual chain, R-grad32)
  void* xl;
  void* lnf;
  float *muf, *rsf;
  int32_t* tok;
  int32_t* lab;
};

struct ParamRef {
  int64_t off, numel;
};

struct Ctx {
  zb_model_cfg_t cfg{};
  DType dt = DT_BF16;
  size_t esz = 2;
  cudaStream_t stream = nullptr;
  int T = 0, h = 0, a = 0, d = 0, Ls = 0, V = 0, s = 0, b = 0;
  bool first = false, last = false;
  bool head_w_eager = false;  // ZB_CFG_HEAD_W_EAGER: dW_head inside B (no dlogits stash)

  // parameters (flat)
  int64_t n_total = 0, n_wd = 0, n_shadow = 0;
  float *theta = nullptr, *grad = nullptr, *m = nullptr, *v = nullptr;
  bf16* shadow = nullptr;
  std::vector<ParamRef> params;  // canonical order
  std::vector<LayerW> lw;
  float *wte = nullptr, *wpe = nullptr, *lnf_g = nullptr, *lnf_b = nullptr;
  void* head_w = nullptr;
  float *g_wte = nullptr, *g_wpe = nullptr, *g_lnf_g = nullptr, *g_lnf_b = nullptr, *g_head_w = nullptr;

  // stash and scratch
  std::vector<Slot> slots;
  void *spare_qkv = nullptr, *d_o = nullptr, *dlogits = nullptr;
  float* d_ln = nullptr;  // LayerNorm-input gradient, f32 in both modes
  float *delta = nullptr, *logits = nullptr, *loss_rows = nullptr;
  float *g32_dx = nullptr, *g32_dx1 = nullptr;  // f32 residual-gradient stream of B (R-grad32)
  uint32_t* keys = nullptr;
  int32_t *tok_stage = nullptr, *lab_stage = nullptr;
  double* loss_acc = nullptr;
  double* norm_part = nullptr;
  int32_t* nf_part = nullptr;
  PvState* pv = nullptr;

  bool first_b_done = false, first_w_done = false;
  std::vector<uint8_t> unit_w_done;  // per W unit: its first contribution of the iteration landed (beta)

  // data parallelism (zb_ctx_attach_dp): the stage's D replicas sum their gradients
  std::unique_ptr<DpComm> dp;
  int dp_world = 1;  // the cross-entropy mean runs over T m dp_world tokens

  // post-validation with NCCL: a validation of the last step is outstanding
  bool pv_pending = false;
  float pv_clip = 1.f;
  float pv_opt[5] = {0, 0, 0, 0, 0};  // lr, beta1, beta2, eps, weight_decay of the pending step

  // timing (ZB_RUN_TIMING): events around every pass of the last timed run, the pass
  // kinds, and the per-kind durations collected by zb_ctx_profile (a1)
  std::vector<cudaEvent_t> ev_start, ev_end;
  std::vector<int> ev_kind, ev_group;  // kind of the timed entry; W passes it covers (W-grouping)
  int n_timed = 0;
  std::vector<int64_t> prof_ns[3];
  int64_t timed_runs = 0, prof_collected_run = 0;  // a timed run starts at pass index 0

  std::unique_ptr<Comm> comm;

  // ZB_RUN_GRAPH: the captured iteration and its key (pass list, flags, staged inputs)
  struct IterGraph {
    std::vector<zb_pass_t> passes;
    int flags = 0;
    const int32_t *tok = nullptr, *lab = nullptr;
    bool captured = false;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;  // kernel nodes of the graph (added to zb_dbg_launch_count per replay)
  };
  IterGraph graph;

  ~Ctx();

  // passes
  void forward(int mb, int slot, const void* in, void* out, const int32_t* labels);
  void backward_input(int mb, int slot, const void* dy, void* dx);
  void backward_weight(int mb, int slot);
  void backward_weight_group(const int* mbs, const int* slots, int k);  // W-grouping (k <= 4)
  // W units (plan.h dp_tail): unit u of the W pass — the LM head (last stage, deferred), then per
  // layer from the top fc2, fc1, proj, qkv (each with its bias), then the embedding (stage 0);
  // backward_weight_group runs all units in this order
  int n_w_units() const { return (last && !head_w_eager ? 1 : 0) + 4 * Ls + (first ? 1 : 0); }
  void weight_unit(int u, const int* slots, int k);
  // gradient range [offset, offset + count) of unit u in `grad` (the vector region: u = -1)
  void unit_grad_range(int u, int64_t* offset, int64_t* count) const;

  void timing_begin(int idx, int kind, int group = 1);
  void timing_end(int idx);
};

// arena sizing / carving (base == nullptr: size only)
size_t carve(Ctx& c, uint8_t* base);
size_t slot_bytes(const zb_model_cfg_t& cfg);
void validate_cfg(const zb_model_cfg_t& cfg);

}  // namespace zb
