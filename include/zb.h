/*
 * zb.h — C ABI of the B200-native Zero Bubble Pipeline Parallelism hot path
 * (arXiv 2401.10241; PAPER.md = /root/reference/PAPER.md, cited P:<line>).
 *
 * The hot path (BASELINE.json north_star) is one pipeline
 * stage of a GPT-style transformer whose backward is split into
 *   B: input gradient   dX  = dY W        ("B")
 *   W: weight gradient  dW += dY^T X      ("W")
 * with F/B/W passes ordered by 1F1B / ZB-H1 / ZB-H2 or the automatic
 * scheduler and an optimizer step with post-validation instead of
 * a synchronous grad-norm / NaN all-reduce (App. C).
 *
 * Conventions (all entry points):
 *  - Every call returns zb_status_t; 0 = ZB_OK, < 0 = error.  The message of
 *    the last error on the calling thread is returned by zb_last_error().
 *    No C++ exception crosses the ABI.
 *  - The caller owns every buffer it passes; the library never frees caller
 *    memory.  Device pointers ("dev") are CUDA device addresses on the
 *    context's device; host pointers ("host") are ordinary CPU memory.
 *  - Times are int64 nanoseconds (or any consistent integer unit), memory
 *    int64 bytes, so that schedules compare exactly.
 *  - Device work is asynchronous on the context's stream; launch errors are
 *    returned immediately, device faults surface at zb_ctx_sync().
 *  - Row-major layouts throughout; T = b*s tokens of one microbatch.
 */
#ifndef ZB_H
#define ZB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t zb_status_t;
enum {
  ZB_OK = 0,
  ZB_EINVAL = -1,  /* bad argument (sizes, pointers, family, call order)            */
  ZB_ELIMIT = -2,  /* M_limit < M_B, or a handcrafted family's peak exceeds M_limit  */
  ZB_ECAP = -3,    /* output capacity too small (out_cap < 3*p*m, arena too small)   */
  ZB_ECUDA = -4,   /* CUDA runtime / launch error                                    */
  ZB_ENCCL = -5,   /* NCCL error or libnccl unavailable                              */
  ZB_ESTATE = -6,  /* invalid state: rollback at t = 0, lr*wd == 1, missing passes   */
  ZB_ETIMEOUT = -7 /* a loopback-transport receive waited longer than 300 s          */
};

/* ------------------------------------------------------------------------ */
/* Schedules (§2, §3.1, App. F)         */
/* ------------------------------------------------------------------------ */

enum { ZB_F = 0, ZB_B = 1, ZB_W = 2 };                         /* pass kinds */
enum { ZB_1F1B = 0, ZB_H1 = 1, ZB_H2 = 2, ZB_AUTO = 3 };       /* families        */
#define ZB_MAX_STAGES 64

/* One pass (i, j, c) of App. F plus its stash slot and the
 * simulator's predicted start / end (same unit as the T_* inputs). */
typedef struct {
  int32_t stage, microbatch, kind, slot;
  int64_t start, end;
} zb_pass_t;

typedef struct {
  int64_t cost;                    /* max over stages of last end - first start */
  int64_t work;                    /* m (T_F + T_B + T_W)                               */
  double bubble_rate;              /* (cost - work) / cost                      */
  int64_t peak_bytes[ZB_MAX_STAGES];  /* order-based Delta-M prefix peak ((7))   */
  int32_t n_slots[ZB_MAX_STAGES];     /* stash slots per stage (lowest free at F, freed at W) */
  int32_t chosen;   /* AUTO: 2*fill_warmup + skip_lead (0..3), 4 = ZB-H1, 5 = ZB-H2; else -1/4/5 */
  int32_t n_passes; /* 3 p m                                                             */
} zb_sim_t;

/* zb_schedule: build the pass lists of `family` for p stages and m
 * microbatches.  T_F/T_B/T_W/T_comm: per-pass times (uniform across
 * stages); M_B / M_W: activation bytes one F / one B retains (Table 1,
 * P:95-107 as Delta-M); M_limit: per-stage activation budget
 * (AUTO: required, >= M_B; handcrafted families: <= 0 means unchecked).
 * out[0 .. 3pm) receives stage 0's list, then stage 1's, ... each in
 * execution order.  1F1B is simulated with its fused backward (upstream B
 * waits for the downstream W).  `sim` may be NULL.
 * Errors: ZB_EINVAL (p < 1, p > 64, m < 1, negative times, bad family),
 * ZB_ECAP (out_cap < 3pm), ZB_ELIMIT (see enum). */
zb_status_t zb_schedule(int32_t p, int32_t m, int64_t T_F, int64_t T_B, int64_t T_W, int64_t T_comm,
                        int64_t M_limit, int64_t M_B, int64_t M_W, int32_t family, zb_pass_t* out,
                        int32_t out_cap, zb_sim_t* sim);

/* zb_schedule_per_stage: zb_schedule with PER-STAGE pass times T_F[p],
 * T_B[p], T_W[p] (host int64 arrays) — "we first conducted a specific number
 * of iterations for profiling, collecting ... T_F, T_B, T_W, and T_comm ...
 * fed them into our automatic pipeline scheduling algorithm".  Stages
 * of one pipeline differ (stage 0 holds the embedding, the last stage the LM
 * head, P:169's partition).  The AUTO heuristic uses each stage's
 * own times (DESIGN.md R-auto-stage); the simulator / bubble rate use them for
 * every family.  Same errors as zb_schedule plus ZB_EINVAL for a NULL array. */
zb_status_t zb_schedule_per_stage(int32_t p, int32_t m, const int64_t* T_F, const int64_t* T_B, const int64_t* T_W,
                                  int64_t T_comm, int64_t M_limit, int64_t M_B, int64_t M_W, int32_t family,
                                  zb_pass_t* out, int32_t out_cap, zb_sim_t* sim);

/* zb_partition: layers per stage when L layers are cut into p stages —
 * P:169 "the first and last pipeline stage ... one fewer layer" when (L+2) is
 * divisible by p (and the middle stages hold >= 2 layers), else an even split
 * with the remainder on the middle stages first.  layers: host int32 [p].
 * ZB_EINVAL unless 1 <= p <= min(L, 64). */
zb_status_t zb_partition(int32_t L, int32_t p, int32_t* layers);

/* zb_simulate: ASAP timing (App. F constraints (4)-(6) as execution
 * semantics) of arbitrary per-stage lists in `passes` (grouped by stage, each
 * stage in execution order), with per-stage times T_F[p], T_B[p], T_W[p]
 * (host arrays) — used to predict bubbles from measured pass times (§5.3).
 * Writes start / end into passes[] and fills sim (peak_bytes from M_B/M_W).
 * fused != 0 models 1F1B's fused backward.  ZB_ESTATE if the lists deadlock. */
zb_status_t zb_simulate(int32_t p, int32_t m, zb_pass_t* passes, int32_t n, const int64_t* T_F,
                        const int64_t* T_B, const int64_t* T_W, int64_t T_comm, int64_t M_B, int64_t M_W,
                        int32_t fused, zb_sim_t* sim);

/* Schedules whose workers hold several model chunks ("virtual stages"
 * v in [0, chunks * p)), each chunk a contiguous block of layers:
 *   ZB_V      (chunks must be 2; §6): V placement — v < p
 *             on worker v, v >= p on worker 2p-1-v; the three-phase
 *             construction of P:322 and the W right-shift within M_limit
 *             (P:324), DESIGN.md R-zbv.  sim->chosen: 0 construction, 1 / 2
 *             W right-shift rule "gap" / "fill", whichever simulates fastest.
 *   ZB_1F1B_I (interleaved 1F1B, the Table 4 baseline): v on worker
 *             v mod p, Megatron-LM order (R-1f1bi), fused backward
 *             (simulated with the upstream B waiting for the downstream W);
 *             m must be a multiple of p.  sim->chosen = -1.
 * T_F/T_B/T_W and M_B/M_W are PER CHUNK PASS (a chunk holds 1/chunks of a
 * stage's layers).  M_limit: per-worker activation budget for the ZB-V
 * right-shift (<= 0: the construction's own peak, i.e. p stage-M_B).
 * out[0 .. 3*chunks*p*m) receives worker 0's list, then worker 1's, ...
 * each in execution order; in every pass `stage` is the VIRTUAL stage v
 * (the pipeline position of its chunk), `slot` the stash slot of chunk v.
 * sim: cost / work / bubble_rate per worker (work = busiest worker's busy
 * time), peak_bytes[w] per worker, n_slots[v] per virtual stage.
 * Errors: ZB_EINVAL (p < 1, m < 1, chunks * p > 64, chunks != 2 for ZB_V,
 * m % p != 0 for ZB_1F1B_I, bad family), ZB_ECAP (out_cap < 3*chunks*p*m),
 * ZB_ELIMIT (ZB_V with 0 < M_limit < the construction's per-worker peak). */
enum { ZB_V = 4, ZB_1F1B_I = 5 };
zb_status_t zb_schedule_chunked(int32_t p, int32_t m, int32_t chunks, int64_t T_F, int64_t T_B, int64_t T_W,
                                int64_t T_comm, int64_t M_limit, int64_t M_B, int64_t M_W, int32_t family,
                                zb_pass_t* out, int32_t out_cap, zb_sim_t* sim);

/* ------------------------------------------------------------------------ */
/* Stage context: one pipeline stage on one GPU                              */
/* ------------------------------------------------------------------------ */

enum { ZB_DTYPE_BF16 = 0, ZB_DTYPE_F32 = 1 };

typedef struct {
  int32_t h, a, L, s, b, V; /* hidden, heads, total layers, seq, microbatch, vocab */
  int32_t p, stage;         /* this context is stage `stage` of p                               */
  int32_t layer_first, layer_last; /* global layer range [first, last) held by the stage        */
  int32_t m;                /* microbatches per iteration (loss = (1/m) sum of token means)     */
  int32_t n_slots;          /* activation-stash slots (zb_sim_t.n_slots[stage])                 */
  int32_t dtype;            /* ZB_DTYPE_BF16: tcgen05 bf16 GEMMs, f32 accumulation;             */
                            /* ZB_DTYPE_F32: f32 everywhere (1e-5 parity mode)                   */
  int32_t flags;            /* ZB_CFG_* below (0 = defaults)                                    */
} zb_model_cfg_t;

/* zb_model_cfg_t.flags.  The last stage's LM-head weight gradient dW_head += dlogits^T LN_f
 * is a W computation and by default runs in the stage's W pass: the bf16 dlogits
 * [T, V] of a microbatch stay in its stash slot from B to W (M_B / M_W of the last stage grow
 * by 2 T V bytes; the B pass loses one T x V x h GEMM, which balances the head-carrying stage,
 * DESIGN.md R-head).  ZB_CFG_HEAD_W_EAGER runs it inside B instead (round-1 behaviour, no
 * dlogits stash).  Gradients are bitwise identical either way (same per-microbatch order). */
enum { ZB_CFG_HEAD_W_EAGER = 1 };

typedef struct zb_ctx zb_ctx_t;

/* Bytes of device memory the context carves out of the caller's arena:
 * parameters (f32 master + bf16 copy), gradients (f32), AdamW moments,
 * n_slots stash slots (M_B per slot, §8(a) a6) and per-stage scratch. */
zb_status_t zb_ctx_arena_bytes(const zb_model_cfg_t* cfg, size_t* bytes);

/* Activation bytes one F retains until its W (= M_B = M_W of this build). */
zb_status_t zb_ctx_slot_bytes(const zb_model_cfg_t* cfg, size_t* bytes);

/* Create a context.  arena: dev buffer of >= zb_ctx_arena_bytes (256-byte
 * aligned, owned by the caller, e.g. a torch uint8 tensor); stream: the
 * cudaStream_t all work is enqueued on (NULL = legacy default stream). */
zb_status_t zb_ctx_create(const zb_model_cfg_t* cfg, void* arena, size_t arena_bytes, void* stream,
                          zb_ctx_t** out);
zb_status_t zb_ctx_destroy(zb_ctx_t* ctx);
/* Wait for all device work of the context; returns ZB_ECUDA on a device fault. */
zb_status_t zb_ctx_sync(zb_ctx_t* ctx);

/* Number of parameter tensors of the stage and their element counts, in the
 * canonical order (zb_synth.param_specs: stage 0 wte, wpe; per layer ln1_g,
 * ln1_b, qkv_w [3h,h], qkv_b, proj_w [h,h], proj_b, ln2_g, ln2_b, fc1_w
 * [4h,h], fc1_b, fc2_w [h,4h], fc2_b; last stage lnf_g, lnf_b, head_w [V,h]). */
zb_status_t zb_ctx_param_count(zb_ctx_t* ctx, int32_t* n);
zb_status_t zb_ctx_param_numel(zb_ctx_t* ctx, int64_t* numel /* [n] */);
/* Upload host f32 parameters (canonical order); resets AdamW state and t. */
zb_status_t zb_ctx_set_params(zb_ctx_t* ctx, const float* const* host_params, int32_t n);
/* Download f32 master parameters / accumulated f32 gradients / AdamW moments (syncs).
 * A NULL entry of host_out skips that tensor (sampled reads of large models). */
zb_status_t zb_ctx_get_params(zb_ctx_t* ctx, float* const* host_out, int32_t n);
zb_status_t zb_ctx_get_grads(zb_ctx_t* ctx, float* const* host_out, int32_t n);
zb_status_t zb_ctx_get_moments(zb_ctx_t* ctx, float* const* host_m, float* const* host_v, int32_t n);
/* Start a new iteration: the first W (and first B for LayerNorm grads) of the
 * iteration overwrites instead of accumulating; the loss accumulator resets. */
zb_status_t zb_ctx_begin_iteration(zb_ctx_t* ctx);
/* Sum over microbatches of the stage's loss contributions (last stage), syncs. */
zb_status_t zb_ctx_read_loss(zb_ctx_t* ctx, double* loss);
/* Device pointer of a slot's [T,h] input buffer (stage > 0, context dtype)
 * or its [T,h] f32 received-gradient buffer (stage < p-1): which = 0 input,
 * 1 gradient. */
zb_status_t zb_ctx_slot_ptr(zb_ctx_t* ctx, int32_t slot, int32_t which, void** dev_ptr);

/* F of microbatch mb into stash `slot`.  in: stage 0: dev int32
 * tokens [T]; else dev activations [T,h] in the context dtype (copied into
 * the slot unless it is the slot's own input buffer).  out: dev [T,h] output
 * activations (stages < p-1; may be another context's slot input), ignored
 * on the last stage.  labels: dev int32 [T] on the last stage (else NULL).
 * Last stage: F ends at LN_f; the head and the loss run in its B. */
zb_status_t zb_stage_forward(zb_ctx_t* ctx, int32_t mb, int32_t slot, const void* in, void* out,
                             const int32_t* labels);
/* B of microbatch mb: all input gradients, attention backward,
 * LayerNorm parameter grads; keeps (X, dY) of the four linears in the slot
 * for W.  Gradients that cross stages are f32 in both modes (the residual-
 * gradient stream is carried in f32, DESIGN.md R-grad32).  dy: dev f32
 * [T,h] gradient of the stage output (stages < p-1; copied into the slot
 * unless it is the slot's own gradient buffer; NULL on the last stage).
 * dx: dev f32 [T,h] gradient of the stage input (stages > 0; else NULL).
 * Last stage: LM head + cross-entropy + head weight gradient (eager, C8). */
zb_status_t zb_stage_backward_input(zb_ctx_t* ctx, int32_t mb, int32_t slot, const void* dy, void* dx);
/* W of microbatch mb: dW += dY^T X for the four linears of every
 * layer (f32 accumulation into persistent f32 grads), bias grads, and on
 * stage 0 the embedding grads.  Frees nothing; the slot may be reused by
 * the next F after this call. */
zb_status_t zb_stage_backward_weight(zb_ctx_t* ctx, int32_t mb, int32_t slot);

/* ------------------------------------------------------------------------ */
/* Iterations                                                                 */
/* ------------------------------------------------------------------------ */

enum { ZB_RUN_HOST_INPUTS = 1, /* tokens / labels are host pointers: H2D inside the call */
       ZB_RUN_TIMING = 2,      /* record CUDA events at every pass boundary               */
       ZB_RUN_FUSED_BW = 4,    /* 1F1B: send the input gradient after the W that follows  */
                               /* its B (the monolithic backward of the baseline, C5)     */
       ZB_RUN_GROUP_W = 8,     /* W-grouping ("W ... anywhere after    */
                               /* the corresponding B"): up to 4 W passes that are ADJACENT */
                               /* in a stage's list run as one contraction per linear with */
                               /* K = k*T (one f32 gradient read-modify-write for k         */
                               /* microbatches).  The sums are grouped differently, so      */
                               /* results are bitwise equal between runs / runtimes with    */
                               /* the same adjacency, within tolerance otherwise.  Not for  */
                               /* zb_run_iteration_worker.  A timed group records one event */
                               /* pair; zb_ctx_profile counts it as k W passes of 1/k each. */
       ZB_RUN_DP_REORDER = 16, /* data parallelism (zb_ctx_attach_dp), App. A       */
                               /* the W passes at the tail of the stage's list   */
                               /* are reordered to cluster the computations of each         */
                               /* parameter, whose gradient all-reduce then starts while    */
                               /* the next parameter's computations run.  Without it the    */
                               /* tail keeps its W-major order (all-reduces start only      */
                               /* inside the last W).  Sub-computations of the tail are not */
                               /* timed (ZB_RUN_TIMING).                                    */
       ZB_RUN_GRAPH = 32       /* zb_run_iteration, p = 1 without NCCL: the iteration's     */
                               /* launches are captured once into a CUDA graph and the     */
                               /* graph is replayed while the pass list, the flags and the */
                               /* input pointers stay the same (the first call with a new  */
                               /* key runs eagerly and sizes lazy buffers, the second one  */
                               /* captures).  Device tokens / labels are copied into the   */
                               /* context's staging buffers first, so per-step input       */
                               /* buffers do not invalidate the graph.  Ignored (eager)    */
                               /* with ZB_RUN_TIMING, kernel timing on, or a context on    */
                               /* the default stream (not capturable).  Results are        */
                               /* bitwise those of the eager run.                          */ };

typedef struct {
  int32_t n_passes;
  float pass_start_ms[3 * 1024]; /* relative to the first pass start (ZB_RUN_TIMING)   */
  float pass_end_ms[3 * 1024];
  double loss;                   /* filled by zb_ctx_read_loss, not by the run calls    */
} zb_iter_stats_t;

/* Run this stage's passes (one iteration) in list order on one context.
 * Single-GPU, single-stage (p = 1) or with an attached NCCL communicator
 * (zb_ctx_attach_nccl) for p > 1.  tokens: int32 [m, b, s] (stage 0),
 * labels: int32 [m, b, s] (last stage); device unless ZB_RUN_HOST_INPUTS.
 * stats may be NULL; with ZB_RUN_TIMING it is filled at the next zb_ctx_sync
 * / zb_ctx_read_stats. */
zb_status_t zb_run_iteration(zb_ctx_t* ctx, const zb_pass_t* passes, int32_t n, const int32_t* tokens,
                             const int32_t* labels, int32_t flags);

/* Run all p stages of one iteration in one process on one GPU ("virtual
 * stages": SURVEY §4): ctxs[p] share the device; passes[] holds every
 * stage's list (zb_schedule output); execution follows the simulator's
 * predicted order, P2P replaced by device copies into the receiver's slot. */
zb_status_t zb_run_iteration_local(zb_ctx_t* const* ctxs, int32_t p, const zb_pass_t* passes, int32_t n,
                                   const int32_t* tokens, const int32_t* labels, int32_t flags);

/* One iteration of a WORKER that holds k model chunks of a chunked schedule
 * (zb_schedule_chunked: ZB-V, 1F1B-I; §6).  chunks[k]: the
 * worker's chunk contexts, each created as virtual stage v of nv = chunks*p
 * (cfg.stage = v, cfg.p = nv) and attached to a transport (zb_ctx_attach_loopback
 * with rank v); passes: the full zb_schedule_chunked output (grouped by worker).
 * The chunks' per-stage plans are merged in the worker's pass order, so the
 * worker runs ZB-V's three phases exactly as scheduled, one host thread per
 * worker.  Post-validation (zb_post_validate_step / _finish per chunk: steps in
 * ascending v, finishes in descending v on each worker) must be finished
 * before the next iteration (no speculative warm-up Fs): ZB_ESTATE otherwise. */
zb_status_t zb_run_iteration_worker(zb_ctx_t* const* chunks, int32_t k, const zb_pass_t* passes, int32_t n,
                                    const int32_t* tokens, const int32_t* labels, int32_t flags);

/* Per-pass event times of the last ZB_RUN_TIMING run (syncs). */
zb_status_t zb_ctx_read_stats(zb_ctx_t* ctx, zb_iter_stats_t* stats);

/* Profiling step of P:169 ("we first conducted a specific number of iterations
 * for profiling, collecting ... T_F, T_B, T_W"): collects the per-pass CUDA-event
 * durations of the last ZB_RUN_TIMING run (each pass once; replayed Fs count as
 * F) into the context's per-kind samples and returns the MEDIAN over all samples
 * since the last reset, in integer ns: T_ns[0] = T_F, [1] = T_B, [2] = T_W
 * (0 when a kind has no sample); n_samples[3] may be NULL.  The pass times
 * exclude waits for messages (events are recorded after the stream waits).
 * reset != 0 clears the samples (T_ns ignored).  Syncs the context's stream.
 * Each timed run is collected once however often this is called; it does not
 * disturb zb_ctx_read_stats. */
zb_status_t zb_ctx_profile(zb_ctx_t* ctx, int32_t reset, int64_t* T_ns, int32_t* n_samples);

/* ------------------------------------------------------------------------ */
/* Optimizer with post-validation (§4, App. C)   */
/* ------------------------------------------------------------------------ */

enum { ZB_OPT_SYNC = 0, ZB_OPT_PV = 1 };
enum { ZB_ACT_NONE = 0, ZB_ACT_STEP = 1, ZB_ACT_SKIP = 2, ZB_ACT_DEFER = 3, ZB_ACT_ROLLBACK = 4,
       ZB_ACT_ROLLBACK_REDO = 5, ZB_ACT_DEFERRED_STEP = 6, ZB_ACT_CLIPPED_STEP = 7 };

typedef struct {
  float lr, beta1, beta2, eps, weight_decay, clip;
  int32_t mode; /* ZB_OPT_SYNC or ZB_OPT_PV */
} zb_optim_cfg_t;

typedef struct {
  double local_sumsq, partial_sumsq, full_sumsq;
  int32_t local_nonfinite, partial_nonfinite, full_nonfinite;
  int32_t first_action, final_action; /* ZB_ACT_*                         */
  int32_t t;                          /* AdamW time stamp after the call  */
} zb_pv_report_t;

/* One optimizer step of the stage(s).  Single context (p = 1): local state
 * = partial = full; in ZB_OPT_PV mode the step is taken optimistically and
 * validated by zb_post_validate_finish.  With an attached NCCL communicator
 * the partial state (sum of squares, non-finite flag) is received from
 * stage-1, combined and sent to stage+1 before the predicated step (no host
 * synchronisation; the decision is made on the device).  All device side. */
zb_status_t zb_post_validate_step(zb_ctx_t* ctx, const zb_optim_cfg_t* cfg);
/* Validation with the fully reduced state (received from stage+1, forwarded
 * to stage-1): nothing, rollback (Algorithm 1), rollback + clipped redo, or
 * the deferred clipped step, predicated on the device. */
zb_status_t zb_post_validate_finish(zb_ctx_t* ctx, const zb_optim_cfg_t* cfg);
/* p contexts of one process (virtual stages): the partial chain 1 -> p, the
 * per-stage predicated steps, then the full state p -> 1 and validation. */
zb_status_t zb_post_validate_local(zb_ctx_t* const* ctxs, int32_t p, const zb_optim_cfg_t* cfg);
/* Report of the last step / validation (syncs). */
zb_status_t zb_ctx_read_pv_report(zb_ctx_t* ctx, zb_pv_report_t* rep);

/* ------------------------------------------------------------------------ */
/* Multi-GPU: one process per GPU, NCCL P2P over NVLink       */
/* ------------------------------------------------------------------------ */

/* 128-byte ncclUniqueId, created on rank 0 and broadcast by the caller
 * (torch.distributed).  ZB_ENCCL if libnccl.so.2 cannot be loaded. */
zb_status_t zb_nccl_unique_id(void* id128);
/* Attach the P2P communicators of this stage (rank = stage, world = p).
 * ids: 2*(world-1) unique ids of 128 bytes (identical on every rank): ids[k]
 * for the activation channel of the pair (k, k+1), ids[world-1+k] for its
 * gradient channel.  Each channel is a 2-rank communicator driven by its own
 * stream.  zb_run_iteration then exchanges activations after F and
 * gradients after B; zb_post_validate_step sends the partial
 * state down the activation channel; in ZB_OPT_PV mode the validation of
 * the step happens inside the NEXT zb_run_iteration (after the stage's
 * speculative warm-up Fs, which are replayed if the weights change — plan.h)
 * or in zb_post_validate_finish when no iteration follows. */
zb_status_t zb_ctx_attach_nccl(zb_ctx_t* ctx, const void* ids, int32_t rank, int32_t world);

/* T_comm of P:127 / P:169 ("T_comm ... collected" during profiling): the median
 * round trip, in ns, of one `bytes` message from this stage to stage+1 (activation
 * channel) and back (gradient channel) over the attached transport, `iters` timed
 * round trips after 2 warm-ups.  Collective: EVERY stage of the pipeline must call
 * it with the same bytes / iters (each answers its upstream neighbour, then pings
 * downstream).  roundtrip_ns = 0 on the last stage; T_comm = max over stages / 2.
 * Blocks the host until the probe finished.  ZB_EINVAL without a transport. */
zb_status_t zb_ctx_comm_probe(zb_ctx_t* ctx, size_t bytes, int32_t iters, int64_t* roundtrip_ns);

/* Attach the k chunk contexts of worker `worker` of a chunked schedule (ZB-V,
 * 1F1B-I; contexts created as virtual stages v of nv): links to chunks on
 * other workers become 2-rank NCCL communicators, ids as for
 * zb_ctx_attach_nccl with world = nv (ids[k] activations of link (k, k+1),
 * ids[nv-1+k] its gradients; identical on every rank), links between two
 * chunks of this worker (ZB-V's v = p-1 -> p turn) an in-process loopback
 * channel.  worker_of[nv]: the worker of every virtual stage.  Then drive the
 * worker with zb_run_iteration_worker.  ZB_ENCCL if libnccl is unavailable. */
zb_status_t zb_ctx_attach_nccl_chunks(zb_ctx_t* const* chunks, int32_t k, const void* ids, int32_t nv,
                                      const int32_t* worker_of, int32_t worker);

/* Data parallelism (App. A): D replicas of the
 * pipeline, each fed its own microbatches; stage s of replica r is one process
 * (GPU).  Attach the replicas of one stage to a D-rank NCCL communicator (id128:
 * one ncclUniqueId per stage, identical on its D ranks; dp_rank in [0, D)).  For
 * p > 1 attach the P2P transport (zb_ctx_attach_nccl) FIRST.  zb_run_iteration then
 * sums the stage's gradients over the replicas with in-place f32 all-reduces, one
 * per W unit (the LM head; per layer fc2, fc1, proj, qkv; the embedding — each
 * issued on a side stream right after the computation that completes it) plus one
 * for the vector region (LayerNorm gammas / betas, biases), before the iteration
 * returns to the post-validation step; ZB_RUN_DP_REORDER reorders the tail Ws per
 * parameter (App. A).  The cross-entropy mean runs over all T m D tokens, so
 * zb_ctx_read_loss returns this replica's share of the global loss.  dp_world = 1
 * is allowed (no communicator; the plan runner with the reordered tail).
 * ZB_ENCCL if libnccl is missing or lacks ncclAllReduce. */
zb_status_t zb_ctx_attach_dp(zb_ctx_t* ctx, const void* id128, int32_t dp_rank, int32_t dp_world);

/* In-process loopback group (test transport for one GPU): world stage
 * contexts of ONE process attach to the same group and are then driven
 * exactly like NCCL-attached contexts, each by its own host thread
 * (zb_run_iteration, zb_post_validate_step / _finish; the calls block only
 * while waiting for a message from a neighbour, up to 300 s, or
 * $ZB_LOOPBACK_TIMEOUT_S, -> ZB_ETIMEOUT).
 * Messages move through device staging buffers owned by the group.  The
 * group is reference counted: zb_loopback_destroy releases the caller's
 * reference; attached contexts keep it alive. */
typedef struct zb_loopback zb_loopback_t;
zb_status_t zb_loopback_create(int32_t world, zb_loopback_t** out);
zb_status_t zb_loopback_destroy(zb_loopback_t* group);
/* rank = the context's stage; world = its p. */
zb_status_t zb_ctx_attach_loopback(zb_ctx_t* ctx, zb_loopback_t* group, int32_t rank);

const char* zb_last_error(void);
const char* zb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ZB_H */
