// Stage passes F / B / W over the stash slots (stage.h).
//
// F  (per layer)  LN1 -> QKV = LN1 Wqkv^T + b -> causal attention -> X1 = X + O Wproj^T + b
//                 -> LN2 -> U = LN2 Wfc1^T + b, G = GeLU(U) -> X' = X1 + G Wfc2^T + b
//                 stage 0 starts with the embedding; the last stage ends with LN_f.
// B  (reverse)    last stage: logits = LN_f Whead^T, cross-entropy -> dlogits (kept in the
//                 slot for W), d LN_f; per layer: dU = (dX' Wfc2) * GeLU'(U),
//                 dLN2 = dU Wfc1, dX1 = dX' + LN2_bwd, dO = dX1 Wproj, dQKV = attn_bwd,
//                 dLN1 = dQKV Wqkv, dX = dX1 + LN1_bwd; LayerNorm gamma/beta grads
//                 (deterministic chunk partials) are taken here (DESIGN.md R-ln).
// W  (per layer)  dW += dY^T X for fc2 (dX', G), fc1 (dU, LN2), proj (dX1, O),
//                 qkv (dQKV, LN1) with f32 accumulation into the persistent grads,
//                 bias grads = column sums of dY formed inside the same GEMMs;
//                 last stage: dWhead += dlogits^T LN_f (ZB_CFG_HEAD_W_EAGER: in B);
//                 stage 0: embedding scatter.
// In-place reuse keeps M_W = M_B: dU over U, dX1 over X1, dX over X, dQKV
// pointer-swapped with QKV.
#include <algorithm>
#include <cstring>

#include "attention.h"
#include "comm.h"
#include "gemm.h"
#include "stage.h"

namespace zb {

Ctx::~Ctx() {
  if (graph.exec) cudaGraphExecDestroy(graph.exec);
  for (auto e : ev_start) cudaEventDestroy(e);
  for (auto e : ev_end) cudaEventDestroy(e);
}

void validate_cfg(const zb_model_cfg_t& c) {
  auto bad = [](const char* m) { throw std::invalid_argument(m); };
  if (c.h <= 0 || c.a <= 0 || c.h % c.a) bad("h must be a positive multiple of a");
  const int d = c.h / c.a;
  if (d != 64 && d != 96 && d != 128) bad("head dim h/a must be 64, 96 or 128");
  if (c.h % 64) bad("h must be a multiple of 64");
  if (c.s <= 0 || c.b <= 0 || c.V <= 0 || c.V % 8) bad("s, b > 0 and V a positive multiple of 8");
  if (c.p < 1 || c.stage < 0 || c.stage >= c.p) bad("stage out of range");
  if (c.layer_first < 0 || c.layer_last <= c.layer_first || c.layer_last > c.L) bad("bad layer range");
  if (c.m < 1 || c.n_slots < 1) bad("m and n_slots must be >= 1");
  if (c.dtype != ZB_DTYPE_BF16 && c.dtype != ZB_DTYPE_F32) bad("bad dtype");
  if (static_cast<int64_t>(c.b) * c.s > 8192) bad("at most 8192 tokens per microbatch");
}

namespace {
struct Bump {
  uint8_t* base;
  size_t off = 0;
  explicit Bump(uint8_t* b) : base(b) {}
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  void* take_bytes(size_t n) { return take<uint8_t>(n); }
};
}  // namespace

// Parameter flat layout + stash + scratch.  Called twice: sizing (base null) and carving.
size_t carve(Ctx& c, uint8_t* base) {
  const zb_model_cfg_t& g = c.cfg;
  c.dt = g.dtype == ZB_DTYPE_BF16 ? DT_BF16 : DT_F32;
  c.esz = c.dt == DT_BF16 ? 2 : 4;
  c.h = g.h; c.a = g.a; c.d = g.h / g.a; c.Ls = g.layer_last - g.layer_first;
  c.V = g.V; c.s = g.s; c.b = g.b; c.T = g.b * g.s;
  c.first = g.stage == 0;
  c.last = g.stage == g.p - 1;
  c.head_w_eager = (g.flags & ZB_CFG_HEAD_W_EAGER) != 0;
  const int64_t h = c.h, T = c.T, V = c.V, Ls = c.Ls;

  // ---- flat parameter offsets (elements, 64-element aligned)
  int64_t off = 0;
  auto put = [&](int64_t n) { int64_t o = off; off += (n + 63) / 64 * 64; return o; };
  struct LOff { int64_t qkv_w, proj_w, fc1_w, fc2_w, ln1_g, ln1_b, qkv_b, proj_b, ln2_g, ln2_b, fc1_b, fc2_b; };
  std::vector<LOff> lo(Ls);
  for (int l = 0; l < Ls; ++l) {
    lo[l].qkv_w = put(3 * h * h);
    lo[l].proj_w = put(h * h);
    lo[l].fc1_w = put(4 * h * h);
    lo[l].fc2_w = put(4 * h * h);
  }
  int64_t head_o = c.last ? put(V * h) : -1;
  const int64_t n_shadow = off;
  int64_t wte_o = c.first ? put(V * h) : -1;
  int64_t wpe_o = c.first ? put(static_cast<int64_t>(c.s) * h) : -1;
  const int64_t n_wd = off;
  for (int l = 0; l < Ls; ++l) {
    lo[l].ln1_g = put(h); lo[l].ln1_b = put(h); lo[l].qkv_b = put(3 * h); lo[l].proj_b = put(h);
    lo[l].ln2_g = put(h); lo[l].ln2_b = put(h); lo[l].fc1_b = put(4 * h); lo[l].fc2_b = put(h);
  }
  int64_t lnfg_o = c.last ? put(h) : -1, lnfb_o = c.last ? put(h) : -1;
  c.n_total = off;
  c.n_wd = n_wd;
  c.n_shadow = n_shadow;
  // canonical order (zb_synth.param_specs)
  c.params.clear();
  if (c.first) {
    c.params.push_back({wte_o, V * h});
    c.params.push_back({wpe_o, static_cast<int64_t>(c.s) * h});
  }
  for (int l = 0; l < Ls; ++l) {
    const LOff& q = lo[l];
    c.params.push_back({q.ln1_g, h});     c.params.push_back({q.ln1_b, h});
    c.params.push_back({q.qkv_w, 3 * h * h}); c.params.push_back({q.qkv_b, 3 * h});
    c.params.push_back({q.proj_w, h * h}); c.params.push_back({q.proj_b, h});
    c.params.push_back({q.ln2_g, h});     c.params.push_back({q.ln2_b, h});
    c.params.push_back({q.fc1_w, 4 * h * h}); c.params.push_back({q.fc1_b, 4 * h});
    c.params.push_back({q.fc2_w, 4 * h * h}); c.params.push_back({q.fc2_b, h});
  }
  if (c.last) {
    c.params.push_back({lnfg_o, h});
    c.params.push_back({lnfb_o, h});
    c.params.push_back({head_o, V * h});
  }

  Bump bp(base);
  c.theta = bp.take<float>(c.n_total);
  c.grad = bp.take<float>(c.n_total);
  c.m = bp.take<float>(c.n_total);
  c.v = bp.take<float>(c.n_total);
  c.shadow = c.dt == DT_BF16 ? bp.take<bf16>(c.n_shadow) : nullptr;
  auto cw = [&](int64_t o) -> void* {  // compute copy of a linear matrix
    if (!base) return nullptr;
    return c.dt == DT_BF16 ? static_cast<void*>(c.shadow + o) : static_cast<void*>(c.theta + o);
  };
  auto th = [&](int64_t o) -> float* { return base ? c.theta + o : nullptr; };
  auto gr = [&](int64_t o) -> float* { return base ? c.grad + o : nullptr; };
  c.lw.assign(Ls, LayerW{});
  for (int l = 0; l < Ls; ++l) {
    const LOff& q = lo[l];
    LayerW& w = c.lw[l];
    w.ln1_g = th(q.ln1_g); w.ln1_b = th(q.ln1_b); w.qkv_b = th(q.qkv_b); w.proj_b = th(q.proj_b);
    w.ln2_g = th(q.ln2_g); w.ln2_b = th(q.ln2_b); w.fc1_b = th(q.fc1_b); w.fc2_b = th(q.fc2_b);
    w.qkv_w = cw(q.qkv_w); w.proj_w = cw(q.proj_w); w.fc1_w = cw(q.fc1_w); w.fc2_w = cw(q.fc2_w);
    w.g_ln1_g = gr(q.ln1_g); w.g_ln1_b = gr(q.ln1_b); w.g_qkv_b = gr(q.qkv_b); w.g_proj_b = gr(q.proj_b);
    w.g_ln2_g = gr(q.ln2_g); w.g_ln2_b = gr(q.ln2_b); w.g_fc1_b = gr(q.fc1_b); w.g_fc2_b = gr(q.fc2_b);
    w.g_qkv_w = gr(q.qkv_w); w.g_proj_w = gr(q.proj_w); w.g_fc1_w = gr(q.fc1_w); w.g_fc2_w = gr(q.fc2_w);
  }
  if (c.first) {
    c.wte = th(wte_o); c.wpe = th(wpe_o); c.g_wte = gr(wte_o); c.g_wpe = gr(wpe_o);
  }
  if (c.last) {
    c.lnf_g = th(lnfg_o); c.lnf_b = th(lnfb_o); c.head_w = cw(head_o);
    c.g_lnf_g = gr(lnfg_o); c.g_lnf_b = gr(lnfb_o); c.g_head_w = gr(head_o);
  }

  // ---- stash slots
  const size_t e = c.esz;
  c.slots.assign(g.n_slots, Slot{});
  for (int sidx = 0; sidx < g.n_slots; ++sidx) {
    Slot& sl = c.slots[sidx];
    sl.L.assign(Ls, LayerAct{});
    for (int l = 0; l < Ls; ++l) {
      LayerAct& A = sl.L[l];
      A.x = bp.take_bytes(T * h * e);
      A.ln1 = bp.take_bytes(T * h * e);
      A.qkv = bp.take_bytes(T * 3 * h * e);
      A.o = bp.take_bytes(T * h * e);
      A.x1 = bp.take_bytes(T * h * e);
      A.ln2 = bp.take_bytes(T * h * e);
      A.u = bp.take_bytes(T * 4 * h * e);
      A.g = bp.take_bytes(T * 4 * h * e);
      A.mu1 = bp.take<float>(T); A.rs1 = bp.take<float>(T);
      A.mu2 = bp.take<float>(T); A.rs2 = bp.take<float>(T);
      A.lse = bp.take<float>(static_cast<size_t>(c.a) * T);
    }
    sl.dy = bp.take_bytes(T * h * e);
    sl.dy32 = c.last ? nullptr : bp.take<float>(T * h);
    sl.tok = c.first ? bp.take<int32_t>(T) : nullptr;
    sl.lab = c.last ? bp.take<int32_t>(T) : nullptr;
    if (c.last) {
      sl.xl = bp.take_bytes(T * h * e);
      sl.lnf = bp.take_bytes(T * h * e);
      sl.muf = bp.take<float>(T);
      sl.rsf = bp.take<float>(T);
      sl.dlogits = c.head_w_eager ? nullptr : bp.take_bytes(T * V * e);
    } else {
      sl.xl = sl.lnf = nullptr;
      sl.muf = sl.rsf = nullptr;
      sl.dlogits = nullptr;
    }
  }
  // ---- scratch
  c.spare_qkv = bp.take_bytes(T * 3 * h * e);
  c.d_o = bp.take_bytes(T * h * e);
  c.d_ln = bp.take<float>(T * h);  // f32 in both modes (LayerNorm-input gradient)
  c.g32_dx = bp.take<float>(T * h);
  c.g32_dx1 = bp.take<float>(T * h);
  c.delta = bp.take<float>(static_cast<size_t>(c.a) * T);
  if (c.last) {
    c.logits = bp.take<float>(T * V);
    c.dlogits = c.head_w_eager ? bp.take_bytes(T * V * e) : nullptr;  // deferred: per slot
    c.loss_rows = bp.take<float>(T);
    c.lab_stage = bp.take<int32_t>(static_cast<size_t>(g.m) * T);
  }
  if (c.first) {
    c.keys = bp.take<uint32_t>(8192);
    c.tok_stage = bp.take<int32_t>(static_cast<size_t>(g.m) * T);
  }
  c.loss_acc = bp.take<double>(1);
  c.norm_part = bp.take<double>(kNormBlocks);
  c.nf_part = bp.take<int32_t>(kNormBlocks);
  c.pv = bp.take<PvState>(1);
  return bp.off + 256;
}

size_t slot_bytes(const zb_model_cfg_t& cfg) {
  Ctx a, b;
  zb_model_cfg_t one = cfg, two = cfg;
  one.n_slots = 1;
  two.n_slots = 2;
  a.cfg = one;
  b.cfg = two;
  return carve(b, nullptr) - carve(a, nullptr);
}

// ------------------------------------------------------------------ GEMM helpers
static void lin_fwd(Ctx& c, const void* X, const void* W, const float* bias, void* Y, int M, int N, int K, int epi,
                    void* aux) {
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = X; g.lda = K; g.a_mn = false;
  g.B = W; g.ldb = K; g.b_mn = false;
  g.epi = epi;
  g.ep = EpiArgs{Y, N, bias, aux, N, 0};
  gemm(g, c.dt, c.stream);
}
// dX [M, N] = dY [M, K] * W [K, N]   (W stored [n_out = K, n_in = N])
static void lin_dgrad(Ctx& c, const void* dY, const void* W, void* dX, int M, int N, int K, int epi, void* aux) {
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = dY; g.lda = K; g.a_mn = false;
  g.B = W; g.ldb = N; g.b_mn = true;
  g.epi = epi;
  g.ep = EpiArgs{dX, N, nullptr, aux, N, 0};
  gemm(g, c.dt, c.stream);
}
// dW [M = n_out, N = n_in] (+)= dY[T, M]^T X[T, N]; db [M] (+)= column sums of dY (W of the
// bias), formed inside the same GEMM from the dY tiles it streams (gemm.h bias_out)
static void lin_wgrad(Ctx& c, const void* dY, const void* X, float* dW, float* db, int M, int N, int K, int beta) {
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = dY; g.lda = M; g.a_mn = true;
  g.B = X; g.ldb = N; g.b_mn = true;
  g.epi = EPI_F32_ACC;
  g.ep = EpiArgs{dW, N, nullptr, nullptr, 0, beta};
  g.ep.bias_out = db;
  gemm(g, c.dt, c.stream);
}
static void ln_bwd(Ctx& c, const float* dy, const void* x, const float* mu, const float* rs, const float* g,
                   const float* resid, float* dx32, void* dx, float* gg, float* gb, int beta) {
  layernorm_bwd(c.dt, dy, x, mu, rs, g, resid, dx32, dx, gg, gb, beta, c.T, c.h,
                c.stream);
}

// ------------------------------------------------------------------ F
void Ctx::forward(int mb, int slot_idx, const void* in, void* out, const int32_t* labels) {
  (void)mb;
  Slot& sl = slots.at(slot_idx);
  const int H = h;
  if (first) {
    const int32_t* tok = static_cast<const int32_t*>(in);
    if (tok != sl.tok) ZB_CUDA(cudaMemcpyAsync(sl.tok, tok, sizeof(int32_t) * T, cudaMemcpyDeviceToDevice, stream));
    embed_fwd(dt, sl.tok, wte, wpe, sl.L[0].x, T, s, H, stream);
  } else if (in != sl.L[0].x) {
    ZB_CUDA(cudaMemcpyAsync(sl.L[0].x, in, esz * T * H, cudaMemcpyDeviceToDevice, stream));
  }
  if (last && labels != nullptr && labels != sl.lab)
    ZB_CUDA(cudaMemcpyAsync(sl.lab, labels, sizeof(int32_t) * T, cudaMemcpyDeviceToDevice, stream));
  AttnShape ash{b, s, a, d};
  for (int l = 0; l < Ls; ++l) {
    LayerAct& A = sl.L[l];
    const LayerW& w = lw[l];
    layernorm_fwd(dt, A.x, w.ln1_g, w.ln1_b, A.ln1, A.mu1, A.rs1, T, H, 1e-5f, stream);
    lin_fwd(*this, A.ln1, w.qkv_w, w.qkv_b, A.qkv, T, 3 * H, H, EPI_STORE, nullptr);
    attention_fwd(ash, dt, A.qkv, A.o, A.lse, stream);
    lin_fwd(*this, A.o, w.proj_w, w.proj_b, A.x1, T, H, H, EPI_RESID, A.x);
    layernorm_fwd(dt, A.x1, w.ln2_g, w.ln2_b, A.ln2, A.mu2, A.rs2, T, H, 1e-5f, stream);
    lin_fwd(*this, A.ln2, w.fc1_w, w.fc1_b, A.u, T, 4 * H, H, EPI_BIAS_GELU, A.g);
    void* next = l + 1 < Ls ? sl.L[l + 1].x : (last ? sl.xl : out);
    if (next == nullptr) throw std::invalid_argument("zb_stage_forward: out is required on stages < p-1");
    lin_fwd(*this, A.g, w.fc2_w, w.fc2_b, next, T, H, 4 * H, EPI_RESID, A.x1);
  }
  if (last) layernorm_fwd(dt, sl.xl, lnf_g, lnf_b, sl.lnf, sl.muf, sl.rsf, T, H, 1e-5f, stream);
}

// ------------------------------------------------------------------ B
void Ctx::backward_input(int mb, int slot_idx, const void* dy_in, void* dx_out) {
  (void)mb;
  Slot& sl = slots.at(slot_idx);
  const int H = h;
  const int beta = first_b_done ? 1 : 0;
  // The residual-gradient stream (dX', dX1, dX) is carried in f32 (g32_dx / g32_dx1,
  // DESIGN.md R-grad32); the activation-dtype copies written into the slot feed the
  // dgrad GEMMs now and the wgrad GEMMs in W.
  const float* dx2_32;
  if (last) {
    void* dl = head_w_eager ? dlogits : sl.dlogits;
    lin_fwd(*this, sl.lnf, head_w, nullptr, logits, T, V, H, EPI_F32_STORE, nullptr);
    cross_entropy(dt, logits, sl.lab, dl, loss_rows, loss_acc, T, V,
                  1.0f / (static_cast<float>(T) * static_cast<float>(cfg.m) * static_cast<float>(dp_world)), stream);
    if (head_w_eager) lin_wgrad(*this, dl, sl.lnf, g_head_w, nullptr, V, H, T, beta);  // C8 eager option
    lin_dgrad(*this, dl, head_w, d_ln, T, H, V, EPI_F32_STORE, nullptr);
    ln_bwd(*this, d_ln, sl.xl, sl.muf, sl.rsf, lnf_g, nullptr, g32_dx, sl.dy, g_lnf_g, g_lnf_b, beta);
    dx2_32 = g32_dx;
  } else {
    if (dy_in == nullptr) throw std::invalid_argument("zb_stage_backward_input: dy is required on stages < p-1");
    const float* dyf = static_cast<const float*>(dy_in);
    if (dyf != sl.dy32) ZB_CUDA(cudaMemcpyAsync(sl.dy32, dyf, sizeof(float) * T * H, cudaMemcpyDeviceToDevice, stream));
    convert_rows(dt, sl.dy32, sl.dy, static_cast<int64_t>(T) * H, stream);
    dx2_32 = sl.dy32;
  }
  AttnShape ash{b, s, a, d};
  for (int l = Ls - 1; l >= 0; --l) {
    LayerAct& A = sl.L[l];
    const LayerW& w = lw[l];
    void* dx2 = l == Ls - 1 ? sl.dy : sl.L[l + 1].x;
    lin_dgrad(*this, dx2, w.fc2_w, A.u, T, 4 * H, H, EPI_GELU_BWD, A.u);  // dU over U
    lin_dgrad(*this, A.u, w.fc1_w, d_ln, T, H, 4 * H, EPI_F32_STORE, nullptr);
    ln_bwd(*this, d_ln, A.x1, A.mu2, A.rs2, w.ln2_g, dx2_32, g32_dx1, A.x1, w.g_ln2_g, w.g_ln2_b, beta);  // dX1
    lin_dgrad(*this, A.x1, w.proj_w, d_o, T, H, H, EPI_STORE, nullptr);
    attention_bwd(ash, dt, A.qkv, A.o, d_o, A.lse, spare_qkv, delta, stream);
    std::swap(A.qkv, spare_qkv);                                                              // dQKV in the slot
    lin_dgrad(*this, A.qkv, w.qkv_w, d_ln, T, H, 3 * H, EPI_F32_STORE, nullptr);
    // the stage's input gradient (l == 0) goes straight to the caller's f32 buffer
    float* out32 = (l == 0 && !first && dx_out != nullptr) ? static_cast<float*>(dx_out) : g32_dx;
    ln_bwd(*this, d_ln, A.x, A.mu1, A.rs1, w.ln1_g, g32_dx1, out32, A.x, w.g_ln1_g, w.g_ln1_b, beta);     // dX
    dx2_32 = g32_dx;
  }
  first_b_done = true;
}

// ------------------------------------------------------------------ W
void Ctx::backward_weight(int mb, int slot_idx) { backward_weight_group(&mb, &slot_idx, 1); }

// W of k microbatches at once (W-grouping; P:59 lets a W run anywhere after
// its B): each linear's dW (+ its bias column sums) is ONE contraction over K = k T tokens
// whose segments are the k slots' (dY, X) operands, so at b = 1 (T = 1024) the f32
// gradient read-modify-write is amortised over k microbatches.  k = 1 is the plain W.
void Ctx::backward_weight_group(const int* mbs, const int* slot_idx, int k) {
  (void)mbs;
  const int nu = n_w_units();
  for (int u = 0; u < nu; ++u) weight_unit(u, slot_idx, k);
  first_w_done = true;
}

// One W unit over k microbatches (the "computations calculating gradients for different
// parameters" a W pass consists of, App. A).  beta = 0 on the unit's first contribution
// of the iteration, so the units of the tail may run in any order (data-parallel reordering).
void Ctx::weight_unit(int u, const int* slot_idx, int k) {
  if (k < 1 || k > kMaxSeg) throw std::invalid_argument("W group of 1..4 microbatches");
  const int nu = n_w_units();
  if (u < 0 || u >= nu) throw std::invalid_argument("W unit out of range");
  if (static_cast<int>(unit_w_done.size()) != nu) unit_w_done.assign(nu, 0);
  Slot* sl[kMaxSeg];
  for (int i = 0; i < k; ++i) sl[i] = &slots.at(slot_idx[i]);
  const int H = h;
  const int beta = unit_w_done[u] ? 1 : 0;
  unit_w_done[u] = 1;
  auto wgrad = [&](auto dy_of, auto x_of, float* dW, float* db, int M, int N) {
    GemmArgs g{};
    g.M = M; g.N = N; g.K = k * T;
    g.A = dy_of(*sl[0]); g.lda = M; g.a_mn = true;
    g.B = x_of(*sl[0]); g.ldb = N; g.b_mn = true;
    g.epi = EPI_F32_ACC;
    g.ep = EpiArgs{dW, N, nullptr, nullptr, 0, beta};
    g.ep.bias_out = db;
    if (k > 1) {
      g.nseg = k;
      for (int i = 0; i < k; ++i) {
        g.A_seg[i] = dy_of(*sl[i]);
        g.B_seg[i] = x_of(*sl[i]);
      }
    }
    gemm(g, dt, stream);
  };
  const bool head = last && !head_w_eager;
  if (head && u == 0) {  // the LM head's W: dW_head += dlogits^T LN_f
    wgrad([&](Slot& q) -> const void* { return q.dlogits; }, [&](Slot& q) -> const void* { return q.lnf; },
          g_head_w, nullptr, V, H);
    return;
  }
  const int v = u - (head ? 1 : 0);
  if (v == 4 * Ls) {  // stage 0: embedding scatter (wte, wpe)
    if (!beta) {
      ZB_CUDA(cudaMemsetAsync(g_wte, 0, sizeof(float) * static_cast<size_t>(V) * H, stream));
      ZB_CUDA(cudaMemsetAsync(g_wpe, 0, sizeof(float) * static_cast<size_t>(s) * H, stream));
    }
    for (int i = 0; i < k; ++i) embed_bwd(dt, sl[i]->tok, sl[i]->L[0].x, g_wte, g_wpe, keys, T, s, H, stream);
    return;
  }
  const int l = Ls - 1 - v / 4;
  const LayerW& w = lw[l];
  const bool top = l == Ls - 1;
  switch (v % 4) {
    case 0:
      wgrad([&](Slot& q) -> const void* { return top ? q.dy : q.L[l + 1].x; },
            [&](Slot& q) -> const void* { return q.L[l].g; }, w.g_fc2_w, w.g_fc2_b, H, 4 * H);
      break;
    case 1:
      wgrad([&](Slot& q) -> const void* { return q.L[l].u; }, [&](Slot& q) -> const void* { return q.L[l].ln2; },
            w.g_fc1_w, w.g_fc1_b, 4 * H, H);
      break;
    case 2:
      wgrad([&](Slot& q) -> const void* { return q.L[l].x1; }, [&](Slot& q) -> const void* { return q.L[l].o; },
            w.g_proj_w, w.g_proj_b, H, H);
      break;
    default:
      wgrad([&](Slot& q) -> const void* { return q.L[l].qkv; }, [&](Slot& q) -> const void* { return q.L[l].ln1; },
            w.g_qkv_w, w.g_qkv_b, 3 * H, H);
  }
}

void Ctx::unit_grad_range(int u, int64_t* offset, int64_t* count) const {
  if (u < 0) {  // LayerNorm gammas / betas and biases: [n_wd, n_total)
    *offset = n_wd;
    *count = n_total - n_wd;
    return;
  }
  const bool head = last && !head_w_eager;
  auto at = [&](const float* p, int64_t n) {
    *offset = p - grad;
    *count = n;
  };
  const int64_t H = h;
  if (head && u == 0) return at(g_head_w, static_cast<int64_t>(V) * H);
  const int v = u - (head ? 1 : 0);
  if (v == 4 * Ls) {  // wte and wpe are adjacent in the flat layout
    *offset = g_wte - grad;
    *count = (g_wpe - g_wte) + static_cast<int64_t>(s) * H;
    return;
  }
  const LayerW& w = lw[Ls - 1 - v / 4];
  switch (v % 4) {
    case 0: return at(w.g_fc2_w, 4 * H * H);
    case 1: return at(w.g_fc1_w, 4 * H * H);
    case 2: return at(w.g_proj_w, H * H);
    default: return at(w.g_qkv_w, 3 * H * H);
  }
}

void Ctx::timing_begin(int idx, int kind, int group) {
  while (static_cast<int>(ev_start.size()) <= idx) {
    cudaEvent_t a, b;
    ZB_CUDA(cudaEventCreate(&a));
    ZB_CUDA(cudaEventCreate(&b));
    ev_start.push_back(a);
    ev_end.push_back(b);
    ev_kind.push_back(0);
    ev_group.push_back(1);
  }
  ev_kind[idx] = kind;
  ev_group[idx] = group;
  if (idx == 0) ++timed_runs;
  ZB_CUDA(cudaEventRecord(ev_start[idx], stream));
}
void Ctx::timing_end(int idx) { ZB_CUDA(cudaEventRecord(ev_end[idx], stream)); }

}  // namespace zb
