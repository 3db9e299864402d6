// extern "C" context / pass / iteration / post-validation entry points (include/zb.h).
#include <algorithm>
#include <cstring>
#include <vector>

#include "abi_util.h"
#include "comm.h"
#include "gemm.h"
#include "ktimer.h"
#include "stage.h"

using namespace zb;

namespace {

Ctx* C_(zb_ctx_t* p) {
  if (p == nullptr) throw Error(ZB_EINVAL, "null context");
  return reinterpret_cast<Ctx*>(p);
}

void begin_iteration(Ctx& c) {
  c.first_b_done = false;
  c.first_w_done = false;
  c.unit_w_done.assign(c.n_w_units(), 0);
  ZB_CUDA(cudaMemsetAsync(c.loss_acc, 0, sizeof(double), c.stream));
}

// Post-validation helpers (§4; Algorithm 1).
void pv_local(Ctx& c) { grad_norm(c.grad, c.n_total, c.norm_part, c.nf_part, c.pv, c.stream); }
void pv_apply(Ctx& c, const zb_optim_cfg_t& o, bool validation) {
  adamw_apply(c.theta, c.m, c.v, c.grad, c.shadow, c.n_total, c.n_wd, c.shadow ? c.n_shadow : 0, o.lr, o.beta1,
              o.beta2, o.eps, o.weight_decay, c.pv, validation, c.stream);
  pv_finish_apply(c.pv, c.stream);
}
// copy src partial (sum, flag) -> dst partial_in / full, via a tiny device memcpy of the two fields
void copy_partial_to_in(Ctx& src, Ctx& dst) {
  ZB_CUDA(cudaMemcpyAsync(&dst.pv->partial_in_sumsq, &src.pv->partial_sumsq, sizeof(double),
                          cudaMemcpyDeviceToDevice, dst.stream));
  ZB_CUDA(cudaMemcpyAsync(&dst.pv->partial_in_nf, &src.pv->partial_nf, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                          dst.stream));
}
void copy_full(Ctx& src_with_partial, Ctx& dst, bool from_partial) {
  const double* sp = from_partial ? &src_with_partial.pv->partial_sumsq : &src_with_partial.pv->full_sumsq;
  const int32_t* sf = from_partial ? &src_with_partial.pv->partial_nf : &src_with_partial.pv->full_nf;
  ZB_CUDA(cudaMemcpyAsync(&dst.pv->full_sumsq, sp, sizeof(double), cudaMemcpyDeviceToDevice, dst.stream));
  ZB_CUDA(cudaMemcpyAsync(&dst.pv->full_nf, sf, sizeof(int32_t), cudaMemcpyDeviceToDevice, dst.stream));
}
// ABI-boundary validation of a stage's pass list (zb.h promises ZB_EINVAL for bad
// passes): every field in range, each (kind, microbatch) exactly once, F before B
// before W per microbatch (P:46 dependencies), B / W on the slot their F used, and no
// F reusing a slot whose previous microbatch has not run its W yet (the stash
// lifetime F -> W).
void check_stage_passes(const zb_pass_t* passes, int32_t n, int stage, int m, int n_slots) {
  std::vector<int> pos[3];
  for (auto& v : pos) v.assign(m, -1);
  std::vector<int> slot_of(m, -1), slot_user(n_slots, -1);
  int k = 0;
  for (int i = 0; i < n; ++i) {
    const zb_pass_t& q = passes[i];
    if (q.stage != stage) continue;
    if (q.kind < ZB_F || q.kind > ZB_W) throw Error(ZB_EINVAL, "pass kind out of range");
    if (q.microbatch < 0 || q.microbatch >= m) throw Error(ZB_EINVAL, "pass microbatch out of range");
    if (q.slot < 0 || q.slot >= n_slots) throw Error(ZB_EINVAL, "pass slot out of range");
    const int j = q.microbatch;
    if (pos[q.kind][j] >= 0) throw Error(ZB_EINVAL, "pass listed twice");
    if (q.kind == ZB_F) {
      if (slot_user[q.slot] >= 0) throw Error(ZB_EINVAL, "F reuses a stash slot before the W of its previous user");
      slot_user[q.slot] = j;
      slot_of[j] = q.slot;
    } else {
      if (pos[q.kind - 1][j] < 0) throw Error(ZB_EINVAL, "B before its F, or W before its B");
      if (q.slot != slot_of[j]) throw Error(ZB_EINVAL, "B / W slot differs from the slot of its F");
      if (q.kind == ZB_W) slot_user[q.slot] = -1;
    }
    pos[q.kind][j] = k++;
  }
  if (k != 3 * m) throw Error(ZB_EINVAL, "stage " + std::to_string(stage) + " needs 3m passes, got " + std::to_string(k));
}

void check_opt(const zb_optim_cfg_t* o) {
  if (o == nullptr) throw Error(ZB_EINVAL, "null optimizer config");
  if (o->lr * o->weight_decay == 1.0f) throw Error(ZB_ESTATE, "lr * weight_decay == 1: rollback undefined");
  if (!(o->beta1 > 0 && o->beta1 < 1 && o->beta2 > 0 && o->beta2 < 1)) throw Error(ZB_EINVAL, "betas in (0,1)");
  if (o->mode != ZB_OPT_SYNC && o->mode != ZB_OPT_PV) throw Error(ZB_EINVAL, "bad optimizer mode");
}

}  // namespace

extern "C" zb_status_t zb_ctx_arena_bytes(const zb_model_cfg_t* cfg, size_t* bytes) {
  ZB_TRY {
    if (!cfg || !bytes) return set_error(ZB_EINVAL, "null argument");
    validate_cfg(*cfg);
    Ctx c;
    c.cfg = *cfg;
    *bytes = carve(c, nullptr);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_slot_bytes(const zb_model_cfg_t* cfg, size_t* bytes) {
  ZB_TRY {
    if (!cfg || !bytes) return set_error(ZB_EINVAL, "null argument");
    validate_cfg(*cfg);
    *bytes = slot_bytes(*cfg);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_create(const zb_model_cfg_t* cfg, void* arena, size_t arena_bytes, void* stream,
                                     zb_ctx_t** out) {
  ZB_TRY {
    if (!cfg || !arena || !out) return set_error(ZB_EINVAL, "null argument");
    if (reinterpret_cast<uintptr_t>(arena) & 255) return set_error(ZB_EINVAL, "arena must be 256-byte aligned");
    validate_cfg(*cfg);
    auto c = std::make_unique<Ctx>();
    c->cfg = *cfg;
    const size_t need = carve(*c, nullptr);
    if (arena_bytes < need) return set_error(ZB_ECAP, "arena too small: need " + std::to_string(need) + " bytes");
    carve(*c, static_cast<uint8_t*>(arena));
    c->stream = static_cast<cudaStream_t>(stream);
    ZB_CUDA(cudaMemsetAsync(c->pv, 0, sizeof(PvState), c->stream));
    ZB_CUDA(cudaMemsetAsync(c->grad, 0, sizeof(float) * c->n_total, c->stream));
    begin_iteration(*c);
    *out = reinterpret_cast<zb_ctx_t*>(c.release());
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_destroy(zb_ctx_t* ctx) {
  ZB_TRY {
    if (ctx) {
      // queued work still writes into the caller's arena: drain it before the caller may
      // free / reuse the memory (a fault here is reported by the next CUDA call, not thrown)
      Ctx* c = reinterpret_cast<Ctx*>(ctx);
      (void)cudaStreamSynchronize(c->stream);
      delete c;
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_sync(zb_ctx_t* ctx) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_param_count(zb_ctx_t* ctx, int32_t* n) {
  ZB_TRY {
    *n = static_cast<int32_t>(C_(ctx)->params.size());
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_param_numel(zb_ctx_t* ctx, int64_t* numel) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    for (size_t i = 0; i < c->params.size(); ++i) numel[i] = c->params[i].numel;
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_set_params(zb_ctx_t* ctx, const float* const* host, int32_t n) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (n != static_cast<int32_t>(c->params.size())) return set_error(ZB_EINVAL, "wrong parameter count");
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    // every initialisation is ordered on the context's own (possibly non-blocking) stream
    ZB_CUDA(cudaMemsetAsync(c->theta, 0, sizeof(float) * c->n_total, c->stream));
    for (int i = 0; i < n; ++i)
      ZB_CUDA(cudaMemcpyAsync(c->theta + c->params[i].off, host[i], sizeof(float) * c->params[i].numel,
                              cudaMemcpyHostToDevice, c->stream));
    ZB_CUDA(cudaMemsetAsync(c->m, 0, sizeof(float) * c->n_total, c->stream));
    ZB_CUDA(cudaMemsetAsync(c->v, 0, sizeof(float) * c->n_total, c->stream));
    ZB_CUDA(cudaMemsetAsync(c->grad, 0, sizeof(float) * c->n_total, c->stream));
    ZB_CUDA(cudaMemsetAsync(c->pv, 0, sizeof(PvState), c->stream));
    if (c->shadow) convert_f32(DT_BF16, c->theta, c->shadow, c->n_shadow, c->stream);
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    return ZB_OK;
  }
  ZB_CATCH
}

static zb_status_t get_flat(zb_ctx_t* ctx, const float* src_base_sel, float* const* host, int32_t n) {
  Ctx* c = C_(ctx);
  if (n != static_cast<int32_t>(c->params.size())) return set_error(ZB_EINVAL, "wrong parameter count");
  ZB_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < n; ++i)
    if (host[i])  // a NULL entry skips that tensor
      ZB_CUDA(cudaMemcpy(host[i], src_base_sel + c->params[i].off, sizeof(float) * c->params[i].numel,
                         cudaMemcpyDeviceToHost));
  return ZB_OK;
}

extern "C" zb_status_t zb_ctx_get_params(zb_ctx_t* ctx, float* const* host, int32_t n) {
  ZB_TRY { return get_flat(ctx, C_(ctx)->theta, host, n); }
  ZB_CATCH
}
extern "C" zb_status_t zb_ctx_get_grads(zb_ctx_t* ctx, float* const* host, int32_t n) {
  ZB_TRY { return get_flat(ctx, C_(ctx)->grad, host, n); }
  ZB_CATCH
}
extern "C" zb_status_t zb_ctx_get_moments(zb_ctx_t* ctx, float* const* hm, float* const* hv, int32_t n) {
  ZB_TRY {
    zb_status_t r = get_flat(ctx, C_(ctx)->m, hm, n);
    if (r != ZB_OK) return r;
    return get_flat(ctx, C_(ctx)->v, hv, n);
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_begin_iteration(zb_ctx_t* ctx) {
  ZB_TRY {
    begin_iteration(*C_(ctx));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_read_loss(zb_ctx_t* ctx, double* loss) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!loss) return set_error(ZB_EINVAL, "null loss");
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    ZB_CUDA(cudaMemcpy(loss, c->loss_acc, sizeof(double), cudaMemcpyDeviceToHost));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_slot_ptr(zb_ctx_t* ctx, int32_t slot, int32_t which, void** ptr) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (slot < 0 || slot >= static_cast<int32_t>(c->slots.size()) || !ptr) return set_error(ZB_EINVAL, "bad slot");
    if (which == 0) *ptr = c->slots[slot].L[0].x;
    else if (which == 1) *ptr = c->slots[slot].dy32;
    else return set_error(ZB_EINVAL, "which must be 0 (input) or 1 (gradient)");
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_stage_forward(zb_ctx_t* ctx, int32_t mb, int32_t slot, const void* in, void* out,
                                        const int32_t* labels) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (slot < 0 || slot >= static_cast<int32_t>(c->slots.size())) return set_error(ZB_EINVAL, "bad slot");
    if (in == nullptr) return set_error(ZB_EINVAL, "null input");
    if (c->last && labels == nullptr) return set_error(ZB_EINVAL, "labels required on the last stage");
    c->forward(mb, slot, in, out, labels);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_stage_backward_input(zb_ctx_t* ctx, int32_t mb, int32_t slot, const void* dy, void* dx) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (slot < 0 || slot >= static_cast<int32_t>(c->slots.size())) return set_error(ZB_EINVAL, "bad slot");
    c->backward_input(mb, slot, dy, dx);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_stage_backward_weight(zb_ctx_t* ctx, int32_t mb, int32_t slot) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (slot < 0 || slot >= static_cast<int32_t>(c->slots.size())) return set_error(ZB_EINVAL, "bad slot");
    c->backward_weight(mb, slot);
    return ZB_OK;
  }
  ZB_CATCH
}

// ------------------------------------------------------------------ iterations
static void stage_inputs(Ctx& c, const int32_t*& tokens, const int32_t*& labels, int flags) {
  const size_t n = static_cast<size_t>(c.cfg.m) * c.T;
  if (flags & ZB_RUN_HOST_INPUTS) {
    if (c.first && tokens) {
      ZB_CUDA(cudaMemcpyAsync(c.tok_stage, tokens, n * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
      tokens = c.tok_stage;
    }
    if (c.last && labels) {
      ZB_CUDA(cudaMemcpyAsync(c.lab_stage, labels, n * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
      labels = c.lab_stage;
    }
  }
  if (c.first && !tokens) throw Error(ZB_EINVAL, "tokens required on stage 0");
  if (c.last && !labels) throw Error(ZB_EINVAL, "labels required on the last stage");
}

static void run_iteration_passes(Ctx* c, const zb_pass_t* passes, int32_t n, const int32_t* tokens,
                                 const int32_t* labels, int32_t flags);
static void run_iteration_graph(Ctx& c, const zb_pass_t* passes, int32_t n, const int32_t* tokens,
                                const int32_t* labels, int32_t flags);

extern "C" zb_status_t zb_run_iteration(zb_ctx_t* ctx, const zb_pass_t* passes, int32_t n, const int32_t* tokens,
                                        const int32_t* labels, int32_t flags) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!passes || n <= 0) return set_error(ZB_EINVAL, "no passes");
    check_stage_passes(passes, n, c->cfg.stage, c->cfg.m, static_cast<int>(c->slots.size()));
    if (c->comm) {
      run_iteration_nccl(*c, passes, n, tokens, labels, flags);
      return ZB_OK;
    }
    if (c->cfg.p != 1) return set_error(ZB_EINVAL, "p > 1 needs zb_ctx_attach_nccl or zb_run_iteration_local");
    stage_inputs(*c, tokens, labels, flags);
    // (the legacy default stream cannot be captured: contexts on it run eagerly)
    if ((flags & ZB_RUN_GRAPH) && !(flags & ZB_RUN_TIMING) && !ktimer::enabled() && c->stream != nullptr &&
        c->stream != cudaStreamLegacy && c->stream != cudaStreamPerThread) {
      run_iteration_graph(*c, passes, n, tokens, labels, flags);
      return ZB_OK;
    }
    run_iteration_passes(c, passes, n, tokens, labels, flags);
    return ZB_OK;
  }
  ZB_CATCH
}

// The launches of one single-stage iteration (zb_run_iteration, p = 1, no NCCL).
static void run_iteration_passes(Ctx* c, const zb_pass_t* passes, int32_t n, const int32_t* tokens,
                                 const int32_t* labels, int32_t flags) {
  {
    begin_iteration(*c);
    const int T = c->T;
    c->n_timed = 0;
    std::vector<const zb_pass_t*> mine;
    for (int i = 0; i < n; ++i)
      if (passes[i].stage == c->cfg.stage) mine.push_back(&passes[i]);
    for (size_t i = 0; i < mine.size(); ++i) {
      const zb_pass_t& q = *mine[i];
      if (q.kind == ZB_W) {
        int mbs[kMaxSeg], sls[kMaxSeg], k = 0;
        const int gmax = (flags & ZB_RUN_GROUP_W) ? kMaxSeg : 1;
        while (k < gmax && i + k < mine.size() && mine[i + k]->kind == ZB_W) {
          mbs[k] = mine[i + k]->microbatch;
          sls[k] = mine[i + k]->slot;
          ++k;
        }
        if (flags & ZB_RUN_TIMING) c->timing_begin(c->n_timed, ZB_W, k);
        c->backward_weight_group(mbs, sls, k);
        if (flags & ZB_RUN_TIMING) c->timing_end(c->n_timed++);
        i += k - 1;
        continue;
      }
      if (flags & ZB_RUN_TIMING) c->timing_begin(c->n_timed, q.kind);
      if (q.kind == ZB_F)
        c->forward(q.microbatch, q.slot, tokens + static_cast<int64_t>(q.microbatch) * T, nullptr,
                   labels + static_cast<int64_t>(q.microbatch) * T);
      else
        c->backward_input(q.microbatch, q.slot, nullptr, nullptr);
      if (flags & ZB_RUN_TIMING) c->timing_end(c->n_timed++);
    }
  }
}

// ZB_RUN_GRAPH: replay the captured iteration while its key (pass list, flags, input pointers)
// is unchanged.  A new key runs eagerly once (lazy per-stream buffers of the GEMM / column-sum
// paths are sized outside any capture), the next call with the same key captures (relaxed
// mode, the split-K counters restarted inside the graph) and launches the graph.
static void run_iteration_graph(Ctx& c, const zb_pass_t* passes, int32_t n, const int32_t* tokens,
                                const int32_t* labels, int32_t flags) {
  const size_t nt = static_cast<size_t>(c.cfg.m) * c.T;
  if (c.first && tokens != c.tok_stage) {  // per-step device inputs -> the fixed staging buffers
    ZB_CUDA(cudaMemcpyAsync(c.tok_stage, tokens, nt * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
    tokens = c.tok_stage;
  }
  if (c.last && labels != c.lab_stage) {
    ZB_CUDA(cudaMemcpyAsync(c.lab_stage, labels, nt * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
    labels = c.lab_stage;
  }
  Ctx::IterGraph& G = c.graph;
  const int key_flags = flags & ~ZB_RUN_HOST_INPUTS;
  const bool same = G.flags == key_flags && G.tok == tokens && G.lab == labels &&
                    G.passes.size() == static_cast<size_t>(n) &&
                    std::memcmp(G.passes.data(), passes, sizeof(zb_pass_t) * n) == 0;
  if (!same) {
    if (G.exec) ZB_CUDA(cudaGraphExecDestroy(G.exec));
    G.exec = nullptr;
    G.captured = false;
    G.passes.assign(passes, passes + n);
    G.flags = key_flags;
    G.tok = tokens;
    G.lab = labels;
    run_iteration_passes(&c, passes, n, tokens, labels, flags);
    return;
  }
  if (!G.captured) {
    ZB_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
    const int64_t l0 = launch_count(false);
    try {
      gemm_graph_begin(c.stream);
      run_iteration_passes(&c, passes, n, tokens, labels, flags);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(c.stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    ZB_CUDA(cudaStreamEndCapture(c.stream, &g));
    G.launches = launch_count(false) - l0;
    add_launches(-G.launches);  // captured, not executed: counted per replay below
    const cudaError_t e = cudaGraphInstantiate(&G.exec, g, 0);
    cudaGraphDestroy(g);
    ZB_CUDA(e);
    G.captured = true;
  }
  ZB_CUDA(cudaGraphLaunch(G.exec, c.stream));
  add_launches(G.launches);
}

extern "C" zb_status_t zb_ctx_attach_nccl_chunks(zb_ctx_t* const* chunks, int32_t k, const void* ids, int32_t nv,
                                                 const int32_t* worker_of, int32_t worker) {
  ZB_TRY {
    if (!chunks || k < 1 || !ids || nv < 2 || !worker_of) return set_error(ZB_EINVAL, "bad arguments");
    std::vector<Ctx*> cs(k);
    for (int i = 0; i < k; ++i) cs[i] = C_(chunks[i]);
    attach_nccl_chunks(cs, ids, nv, std::vector<int>(worker_of, worker_of + nv), worker);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_run_iteration_worker(zb_ctx_t* const* chunks, int32_t k, const zb_pass_t* passes,
                                               int32_t n, const int32_t* tokens, const int32_t* labels,
                                               int32_t flags) {
  ZB_TRY {
    if (!chunks || k < 1 || !passes || n <= 0) return set_error(ZB_EINVAL, "bad arguments");
    std::vector<Ctx*> cs(k);
    for (int i = 0; i < k; ++i) {
      cs[i] = C_(chunks[i]);
      check_stage_passes(passes, n, cs[i]->cfg.stage, cs[i]->cfg.m, static_cast<int>(cs[i]->slots.size()));
    }
    run_iteration_worker(cs, passes, n, tokens, labels, flags);
    return ZB_OK;
  }
  ZB_CATCH
}

// All p stages in one process on one device: a ready-driven global order in
// which F(s-1, j) writes straight into stage s's slot input once that slot's
// previous microbatch has finished its W, and B(s, j) writes dX straight into
// stage s-1's slot gradient buffer (no extra copies, no outboxes).
extern "C" zb_status_t zb_run_iteration_local(zb_ctx_t* const* ctxs, int32_t p, const zb_pass_t* passes, int32_t n,
                                              const int32_t* tokens, const int32_t* labels, int32_t flags) {
  ZB_TRY {
    if (!ctxs || p < 1 || !passes) return set_error(ZB_EINVAL, "bad arguments");
    std::vector<Ctx*> c(p);
    for (int s = 0; s < p; ++s) {
      c[s] = C_(ctxs[s]);
      if (c[s]->cfg.stage != s || c[s]->cfg.p != p) return set_error(ZB_EINVAL, "ctxs must be stages 0..p-1");
      if (c[s]->stream != c[0]->stream) return set_error(ZB_EINVAL, "local stages must share one stream");
    }
    const int m = c[0]->cfg.m, T = c[0]->T;
    for (int s = 0; s < p; ++s) {
      if (c[s]->cfg.m != m) return set_error(ZB_EINVAL, "stages disagree on m");
      check_stage_passes(passes, n, s, m, static_cast<int>(c[s]->slots.size()));
    }
    std::vector<std::vector<const zb_pass_t*>> L(p);
    for (int i = 0; i < n; ++i) {
      if (passes[i].stage < 0 || passes[i].stage >= p) return set_error(ZB_EINVAL, "pass stage out of range");
      L[passes[i].stage].push_back(&passes[i]);
    }
    // slot of (s, j) and the previous microbatch that used the same slot on s
    std::vector<std::vector<int>> slot(p, std::vector<int>(m, -1)), prev(p, std::vector<int>(m, -1));
    for (int s = 0; s < p; ++s) {
      std::vector<int> last_user(c[s]->slots.size(), -1);
      for (auto* q : L[s])
        if (q->kind == ZB_F) {
          if (q->slot < 0 || q->slot >= static_cast<int>(c[s]->slots.size()) || q->microbatch >= m)
            return set_error(ZB_EINVAL, "pass slot out of range");
          slot[s][q->microbatch] = q->slot;
          prev[s][q->microbatch] = last_user[q->slot];
          last_user[q->slot] = q->microbatch;
        }
    }
    stage_inputs(*c[0], tokens, labels, flags & ZB_RUN_HOST_INPUTS);
    if (c[p - 1] != c[0]) {
      const int32_t* t2 = nullptr;
      stage_inputs(*c[p - 1], t2, labels, flags & ZB_RUN_HOST_INPUTS);
    }
    for (int s = 0; s < p; ++s) {
      begin_iteration(*c[s]);
      c[s]->n_timed = 0;
    }
    std::vector<std::vector<char>> done[3];
    for (int k = 0; k < 3; ++k) done[k].assign(p, std::vector<char>(m, 0));
    std::vector<size_t> pos(p, 0);
    int remaining = n;
    while (remaining > 0) {
      bool progressed = false;
      for (int s = 0; s < p; ++s) {
        while (pos[s] < L[s].size()) {
          const zb_pass_t& q = *L[s][pos[s]];
          const int j = q.microbatch;
          bool ready;
          if (q.kind == ZB_F)
            ready = (s == 0 || done[ZB_F][s - 1][j]) &&
                    (s == p - 1 || prev[s + 1][j] < 0 || done[ZB_W][s + 1][prev[s + 1][j]]);
          else if (q.kind == ZB_B)
            ready = done[ZB_F][s][j] && (s == p - 1 || done[ZB_B][s + 1][j]);
          else
            ready = done[ZB_B][s][j];
          if (!ready) break;
          Ctx& cs = *c[s];
          if (flags & ZB_RUN_TIMING) cs.timing_begin(cs.n_timed, q.kind);
          if (q.kind == ZB_F) {
            const void* in = s == 0 ? static_cast<const void*>(tokens + static_cast<int64_t>(j) * T)
                                    : cs.slots[q.slot].L[0].x;
            void* out = s < p - 1 ? c[s + 1]->slots[slot[s + 1][j]].L[0].x : nullptr;
            cs.forward(j, q.slot, in, out, s == p - 1 ? labels + static_cast<int64_t>(j) * T : nullptr);
          } else if (q.kind == ZB_B) {
            void* dx = s > 0 ? c[s - 1]->slots[slot[s - 1][j]].dy32 : nullptr;
            cs.backward_input(j, q.slot, s < p - 1 ? cs.slots[q.slot].dy32 : nullptr, dx);
          } else {
            // W-grouping: the W passes adjacent to this one in the stage's list (their Bs precede
            // this W in list order, so they are done)
            int mbs[kMaxSeg], sls[kMaxSeg], k = 0;
            const int gmax = (flags & ZB_RUN_GROUP_W) ? kMaxSeg : 1;
            while (k < gmax && pos[s] + k < L[s].size() && L[s][pos[s] + k]->kind == ZB_W) {
              mbs[k] = L[s][pos[s] + k]->microbatch;
              sls[k] = L[s][pos[s] + k]->slot;
              ++k;
            }
            if (flags & ZB_RUN_TIMING) cs.ev_group[cs.n_timed] = k;
            cs.backward_weight_group(mbs, sls, k);
            for (int i = 1; i < k; ++i) {  // the group's other passes are done too
              done[ZB_W][s][mbs[i]] = 1;
              ++pos[s];
              --remaining;
            }
          }
          if (flags & ZB_RUN_TIMING) cs.timing_end(cs.n_timed++);
          done[q.kind][s][j] = 1;
          ++pos[s];
          --remaining;
          progressed = true;
        }
      }
      if (!progressed) return set_error(ZB_ESTATE, "pass lists deadlock");
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_read_stats(zb_ctx_t* ctx, zb_iter_stats_t* st) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!st) return set_error(ZB_EINVAL, "null stats");
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    const int n = std::min(c->n_timed, 3 * 1024);
    st->n_passes = n;
    for (int i = 0; i < n; ++i) {
      float a = 0.f, b = 0.f;
      ZB_CUDA(cudaEventElapsedTime(&a, c->ev_start[0], c->ev_start[i]));
      ZB_CUDA(cudaEventElapsedTime(&b, c->ev_start[0], c->ev_end[i]));
      st->pass_start_ms[i] = a;
      st->pass_end_ms[i] = b;
    }
    return ZB_OK;
  }
  ZB_CATCH
}

// a1 "Profile": per-kind pass durations of the ZB_RUN_TIMING runs since the last
// reset, medians in integer nanoseconds (the unit zb_schedule_per_stage takes).
extern "C" zb_status_t zb_ctx_profile(zb_ctx_t* ctx, int32_t reset, int64_t* T_ns, int32_t* n_samples) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (reset) {
      for (auto& v : c->prof_ns) v.clear();
      c->prof_collected_run = c->timed_runs;
      return ZB_OK;
    }
    if (!T_ns) return set_error(ZB_EINVAL, "null output");
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    if (c->timed_runs != c->prof_collected_run) {  // each timed run is collected once
      for (int i = 0; i < c->n_timed; ++i) {
        float ms = 0.f;
        ZB_CUDA(cudaEventElapsedTime(&ms, c->ev_start[i], c->ev_end[i]));
        const int g = c->ev_group[i];  // a grouped W entry covers g W passes
        for (int k = 0; k < g; ++k)
          c->prof_ns[c->ev_kind[i]].push_back(static_cast<int64_t>(static_cast<double>(ms) * 1e6 / g + 0.5));
      }
      c->prof_collected_run = c->timed_runs;
    }
    for (int k = 0; k < 3; ++k) {
      std::vector<int64_t> v = c->prof_ns[k];
      int64_t med = 0;
      if (!v.empty()) {
        std::sort(v.begin(), v.end());
        med = v.size() % 2 ? v[v.size() / 2] : (v[v.size() / 2 - 1] + v[v.size() / 2]) / 2;
      }
      T_ns[k] = med;
      if (n_samples) n_samples[k] = static_cast<int32_t>(v.size());
    }
    return ZB_OK;
  }
  ZB_CATCH
}

// ------------------------------------------------------------------ optimizer / post-validation
extern "C" zb_status_t zb_post_validate_step(zb_ctx_t* ctx, const zb_optim_cfg_t* o) {
  ZB_TRY {
    check_opt(o);
    Ctx* c = C_(ctx);
    pv_local(*c);
    if (c->comm) {
      pv_recv_partial(*c);  // partial state of stages < stage (zeros on stage 0)
    } else {
      if (c->cfg.p != 1) return set_error(ZB_EINVAL, "p > 1 needs NCCL or zb_post_validate_local");
      ZB_CUDA(cudaMemsetAsync(&c->pv->partial_in_sumsq, 0, sizeof(double), c->stream));
      ZB_CUDA(cudaMemsetAsync(&c->pv->partial_in_nf, 0, sizeof(int32_t), c->stream));
    }
    pv_combine(c->pv, c->stream);
    if (c->comm) pv_send_partial(*c);
    if (o->mode == ZB_OPT_SYNC) {
      if (c->comm && c->cfg.p > 1) {  // baseline: wait for the full state before stepping
        pv_recv_full(*c);
        pv_send_full(*c);
        ZB_CUDA(cudaMemcpyAsync(&c->pv->partial_sumsq, &c->pv->full_sumsq, sizeof(double), cudaMemcpyDeviceToDevice,
                                c->stream));
        ZB_CUDA(cudaMemcpyAsync(&c->pv->partial_nf, &c->pv->full_nf, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                c->stream));
      }
      pv_decide_first(c->pv, o->clip, 1, c->stream);
    } else {
      pv_decide_first(c->pv, o->clip, 0, c->stream);
    }
    pv_apply(*c, *o, false);
    if (c->comm && o->mode == ZB_OPT_PV) {  // validated inside the next iteration (or by _finish)
      c->pv_pending = true;
      c->pv_clip = o->clip;
      const float po[5] = {o->lr, o->beta1, o->beta2, o->eps, o->weight_decay};
      std::memcpy(c->pv_opt, po, sizeof(po));
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_post_validate_finish(zb_ctx_t* ctx, const zb_optim_cfg_t* o) {
  ZB_TRY {
    check_opt(o);
    Ctx* c = C_(ctx);
    if (o->mode == ZB_OPT_SYNC) return ZB_OK;  // nothing to validate
    if (c->comm) {
      if (!c->pv_pending) return ZB_OK;  // already validated inside an iteration
      pv_recv_full(*c);  // the last stage takes its own partial as the full state
      pv_send_full(*c);
      c->pv_pending = false;
    } else {
      if (c->cfg.p != 1) return set_error(ZB_EINVAL, "p > 1 needs NCCL or zb_post_validate_local");
      copy_full(*c, *c, true);
    }
    pv_decide_final(c->pv, o->clip, c->stream);
    pv_apply(*c, *o, true);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_post_validate_local(zb_ctx_t* const* ctxs, int32_t p, const zb_optim_cfg_t* o) {
  ZB_TRY {
    check_opt(o);
    if (!ctxs || p < 1) return set_error(ZB_EINVAL, "bad arguments");
    std::vector<Ctx*> c(p);
    for (int s = 0; s < p; ++s) {
      c[s] = C_(ctxs[s]);
      if (c[s]->cfg.stage != s || c[s]->cfg.p != p) return set_error(ZB_EINVAL, "ctxs must be stages 0..p-1");
      // the partial / full state moves between contexts with stream-ordered copies
      if (c[s]->stream != c[0]->stream) return set_error(ZB_EINVAL, "local stages must share one stream");
    }
    // partial chain 1 -> p (stage order summation)
    for (int s = 0; s < p; ++s) {
      pv_local(*c[s]);
      if (s == 0) {
        ZB_CUDA(cudaMemsetAsync(&c[s]->pv->partial_in_sumsq, 0, sizeof(double), c[s]->stream));
        ZB_CUDA(cudaMemsetAsync(&c[s]->pv->partial_in_nf, 0, sizeof(int32_t), c[s]->stream));
      } else {
        copy_partial_to_in(*c[s - 1], *c[s]);
      }
      pv_combine(c[s]->pv, c[s]->stream);
      if (o->mode == ZB_OPT_PV) {
        pv_decide_first(c[s]->pv, o->clip, 0, c[s]->stream);
        pv_apply(*c[s], *o, false);
      }
    }
    if (o->mode == ZB_OPT_SYNC) {  // all-reduced state first, then the conditioned step
      for (int s = 0; s < p; ++s) {
        if (s != p - 1) {
          ZB_CUDA(cudaMemcpyAsync(&c[s]->pv->partial_sumsq, &c[p - 1]->pv->partial_sumsq, sizeof(double),
                                  cudaMemcpyDeviceToDevice, c[s]->stream));
          ZB_CUDA(cudaMemcpyAsync(&c[s]->pv->partial_nf, &c[p - 1]->pv->partial_nf, sizeof(int32_t),
                                  cudaMemcpyDeviceToDevice, c[s]->stream));
        }
        pv_decide_first(c[s]->pv, o->clip, 1, c[s]->stream);
        pv_apply(*c[s], *o, false);
      }
      return ZB_OK;
    }
    // full state p -> 1, validation
    for (int s = p - 1; s >= 0; --s) {
      copy_full(*c[p - 1], *c[s], true);
      pv_decide_final(c[s]->pv, o->clip, c[s]->stream);
      pv_apply(*c[s], *o, true);
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_read_pv_report(zb_ctx_t* ctx, zb_pv_report_t* rep) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!rep) return set_error(ZB_EINVAL, "null report");
    PvState h;
    ZB_CUDA(cudaStreamSynchronize(c->stream));
    ZB_CUDA(cudaMemcpy(&h, c->pv, sizeof(PvState), cudaMemcpyDeviceToHost));
    rep->local_sumsq = h.local_sumsq;
    rep->partial_sumsq = h.partial_sumsq;
    rep->full_sumsq = h.full_sumsq;
    rep->local_nonfinite = h.local_nf;
    rep->partial_nonfinite = h.partial_nf;
    rep->full_nonfinite = h.full_nf;
    rep->first_action = h.first_action;
    rep->final_action = h.final_action;
    rep->t = h.t;
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_nccl_unique_id(void* id128) {
  ZB_TRY {
    if (!id128) return set_error(ZB_EINVAL, "null id");
    nccl_unique_id(id128);
    return ZB_OK;
  }
  ZB_CATCH
}

struct zb_loopback {
  std::shared_ptr<zb::LoopbackGroup> g;
};

extern "C" zb_status_t zb_loopback_create(int32_t world, zb_loopback_t** out) {
  ZB_TRY {
    if (!out || world < 1) return set_error(ZB_EINVAL, "bad loopback arguments");
    *out = new zb_loopback{loopback_create(world)};
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_loopback_destroy(zb_loopback_t* group) {
  delete group;
  return ZB_OK;
}

extern "C" zb_status_t zb_ctx_attach_loopback(zb_ctx_t* ctx, zb_loopback_t* group, int32_t rank) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!group) return set_error(ZB_EINVAL, "null loopback group");
    if (rank != c->cfg.stage) return set_error(ZB_EINVAL, "rank must be the context's stage");
    attach_loopback(*c, group->g, rank);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_comm_probe(zb_ctx_t* ctx, size_t bytes, int32_t iters, int64_t* roundtrip_ns) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!roundtrip_ns || iters < 1 || bytes == 0) return set_error(ZB_EINVAL, "bad probe arguments");
    if (!c->comm) return set_error(ZB_EINVAL, "zb_ctx_comm_probe needs zb_ctx_attach_nccl / _loopback");
    *roundtrip_ns = comm_probe(*c, bytes, iters);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_attach_nccl(zb_ctx_t* ctx, const void* ids, int32_t rank, int32_t world) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (!ids || world < 1 || rank < 0 || rank >= world) return set_error(ZB_EINVAL, "bad NCCL arguments");
    if (world != c->cfg.p || rank != c->cfg.stage) return set_error(ZB_EINVAL, "rank / world must be stage / p");
    attach_nccl(*c, ids, rank, world);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_ctx_attach_dp(zb_ctx_t* ctx, const void* id128, int32_t dp_rank, int32_t dp_world) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if ((!id128 && dp_world > 1) || dp_world < 1 || dp_rank < 0 || dp_rank >= dp_world)
      return set_error(ZB_EINVAL, "bad data-parallel arguments");
    if (c->dp) return set_error(ZB_ESTATE, "data parallelism already attached");
    attach_dp(*c, id128, dp_rank, dp_world);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_w_units(zb_ctx_t* ctx, int32_t* n_units, int64_t* dp_reduces) {
  ZB_TRY {
    Ctx* c = C_(ctx);
    if (n_units) *n_units = c->n_w_units();
    if (dp_reduces) *dp_reduces = dp_reduce_count(*c);
    return ZB_OK;
  }
  ZB_CATCH
}
