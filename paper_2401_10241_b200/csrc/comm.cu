// Transports (NCCL, in-process loopback) and the multi-stage iteration runner
// (see comm.h, plan.h).
//
// libnccl.so.2 is dlopen'ed on first use (torch's bundled NCCL is normally
// already loaded, so the same library is shared).  Every adjacent pair has two
// 2-rank communicators (ACT s->s+1, GRAD s+1->s), each driven by its own
// stream on each side; cross-stream ordering uses CUDA events recorded on the
// compute stream.  The loopback transport keeps the same channels and streams.  The runner executes plan::stage_plan op by op:
//   RECV_ACT   act-recv stream waits for "compute reached here" (the slot's previous
//              user W is enqueued before), receives into the slot input buffer;
//              the compute stream waits for the receive
//   F / REPLAY_F  forward into the activation send ring
//   SEND_ACT   act-send stream waits for F, sends the ring buffer; the next F that
//              reuses the buffer waits for the send
//   RECV_GRAD  into the slot's gradient buffer;  B writes dX in the slot input buffer
//   SEND_GRAD  grad-send stream waits for B (or W, 1F1B) and sends from the slot; the
//              next writer of that slot input waits for the send
//   VALIDATE   full state: receive from stage+1 (last stage: its own partial),
//              forward to stage-1, predicated rollback / redo / deferred step, then
//              the host reads the state (tiny D2H) to decide whether to replay.
#include "comm.h"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>

#include "abi_util.h"
#include "gemm.h"
#include "ops.h"
#include "plan.h"
#include "stage.h"

namespace zb {

namespace {
typedef struct {
  char internal[128];
} ncclUniqueId_t;
typedef int (*PGetId)(ncclUniqueId_t*);
typedef int (*PInit)(void**, int, ncclUniqueId_t, int);
typedef int (*PSendRecv)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*PRecv)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*PDestroy)(void*);
typedef int (*PAllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef const char* (*PErr)(int);
constexpr int kNcclUint8 = 1, kNcclFloat32 = 7, kNcclSum = 0;

struct Nccl {
  void* h = nullptr;
  PGetId get_id = nullptr;
  PInit init = nullptr;
  PSendRecv send = nullptr;
  PRecv recv = nullptr;
  PDestroy destroy = nullptr;
  PErr err = nullptr;
  PAllReduce all_reduce = nullptr;  // data parallelism only (checked by attach_dp)
};

Nccl& nccl() {
  static Nccl n;
  if (n.h) return n;
  // ZB_NCCL_LIB: an explicit library path (tests: the 2-process / 1-GPU shim,
  // tests/shim/nccl_ipc.cu); otherwise the already-loaded / system libnccl.so.2.
  const char* env = std::getenv("ZB_NCCL_LIB");
  if (env && *env) {
    n.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!n.h) throw Error(ZB_ENCCL, std::string("cannot load ZB_NCCL_LIB: ") + dlerror());
  }
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (n.h) break;
    n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!n.h) throw Error(ZB_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
  n.get_id = reinterpret_cast<PGetId>(dlsym(n.h, "ncclGetUniqueId"));
  n.init = reinterpret_cast<PInit>(dlsym(n.h, "ncclCommInitRank"));
  n.send = reinterpret_cast<PSendRecv>(dlsym(n.h, "ncclSend"));
  n.recv = reinterpret_cast<PRecv>(dlsym(n.h, "ncclRecv"));
  n.destroy = reinterpret_cast<PDestroy>(dlsym(n.h, "ncclCommDestroy"));
  n.err = reinterpret_cast<PErr>(dlsym(n.h, "ncclGetErrorString"));
  n.all_reduce = reinterpret_cast<PAllReduce>(dlsym(n.h, "ncclAllReduce"));
  if (!n.get_id || !n.init || !n.send || !n.recv || !n.destroy || !n.err) {
    n.h = nullptr;
    throw Error(ZB_ENCCL, "libnccl.so.2 lacks ncclSend / ncclRecv");
  }
  return n;
}

void nck(int r, const char* what) {
  if (r != 0) throw Error(ZB_ENCCL, std::string(what) + ": " + nccl().err(r));
}

enum { C_ACT_TO = 0, C_ACT_FROM = 1, C_GRAD_TO = 2, C_GRAD_FROM = 3 };

// peer index inside a 2-rank pair communicator: the lower stage is rank 0
int peer_of(int which) { return (which == C_ACT_TO || which == C_GRAD_FROM) ? 1 : 0; }

struct NcclTransport : Transport {
  void* comm[4] = {nullptr, nullptr, nullptr, nullptr};
  ~NcclTransport() override {
    for (auto cm : comm)
      if (cm) nccl().destroy(cm);
  }
  void send(int which, const void* buf, size_t bytes, cudaStream_t st) override {
    nck(nccl().send(buf, bytes, kNcclUint8, peer_of(which), comm[which], st), "ncclSend");
  }
  void recv(int which, void* buf, size_t bytes, cudaStream_t st) override {
    nck(nccl().recv(buf, bytes, kNcclUint8, peer_of(which), comm[which], st), "ncclRecv");
  }
};

void sendb(Comm& cm, int which, const void* buf, size_t bytes) { cm.tx->send(which, buf, bytes, cm.stream[which]); }
void recvb(Comm& cm, int which, void* buf, size_t bytes) { cm.tx->recv(which, buf, bytes, cm.stream[which]); }

// stream `a` waits for everything enqueued so far on stream `b`
void order(Comm& cm, cudaStream_t a, cudaStream_t b) {
  cudaEvent_t e = cm.event();
  ZB_CUDA(cudaEventRecord(e, b));
  ZB_CUDA(cudaStreamWaitEvent(a, e, 0));
}
}  // namespace

Comm::~Comm() {
  for (int i = 0; i < 4; ++i)
    if (stream[i]) cudaStreamSynchronize(stream[i]);
  tx.reset();
  for (int i = 0; i < 4; ++i)
    if (stream[i]) cudaStreamDestroy(stream[i]);
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (auto e : act_buf_free) cudaEventDestroy(e);
  for (auto b : act_buf) cudaFree(b);
  for (auto e : grad_buf_free) cudaEventDestroy(e);
  for (auto b : grad_buf) cudaFree(b);
  if (scalars) cudaFree(scalars);
}

cudaEvent_t Comm::event() {
  // a ring of reusable events; 4096 outstanding is far beyond any dependency distance
  if (ev_pool.size() < 4096) {
    cudaEvent_t e;
    ZB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev_pool.push_back(e);
    return e;
  }
  cudaEvent_t e = ev_pool[ev_next];
  ev_next = (ev_next + 1) % static_cast<int>(ev_pool.size());
  return e;
}

void nccl_unique_id(void* id128) {
  ncclUniqueId_t id;
  nck(nccl().get_id(&id), "ncclGetUniqueId");
  std::memcpy(id128, &id, 128);
}

namespace {
// channel streams and the send staging rings of one stage (both transports)
void setup_comm(Ctx& c, Comm& cm) {
  const int rank = cm.rank, world = cm.world;
  const int chans[4] = {rank < world - 1, rank > 0, rank > 0, rank < world - 1};
  for (int w = 0; w < 4; ++w)
    if (chans[w] && !cm.stream[w]) ZB_CUDA(cudaStreamCreateWithFlags(&cm.stream[w], cudaStreamNonBlocking));
  if (rank < world - 1) {
    for (int i = 0; i < 2; ++i) {
      void* b = nullptr;
      ZB_CUDA(cudaMalloc(&b, c.esz * static_cast<size_t>(c.T) * c.h));
      cm.act_buf.push_back(b);
      cudaEvent_t e;
      ZB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ZB_CUDA(cudaEventRecord(e, c.stream));
      cm.act_buf_free.push_back(e);
    }
  }
  if (rank > 0) {
    for (int i = 0; i < 2; ++i) {
      float* b = nullptr;
      ZB_CUDA(cudaMalloc(&b, sizeof(float) * static_cast<size_t>(c.T) * c.h));
      cm.grad_buf.push_back(b);
      cudaEvent_t e;
      ZB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ZB_CUDA(cudaEventRecord(e, c.stream));
      cm.grad_buf_free.push_back(e);
    }
  }
  ZB_CUDA(cudaMalloc(&cm.scalars, 64 + c.esz * static_cast<size_t>(c.T) * c.h));  // 4 PV messages + discard buffer
}
}  // namespace

// T_comm probe: round trips of one `bytes` message per adjacent pair,
// stage s -> s+1 on the activation channel and back on the gradient channel, timed on
// the lower stage's channel streams.  Every stage first answers its upstream neighbour
// (pong), then pings downstream, so the host-side enqueue order is deadlock-free for
// both transports.  Returns the median round trip in ns (0 on the last stage).
int64_t comm_probe(Ctx& c, size_t bytes, int iters) {
  if (!c.comm) throw Error(ZB_EINVAL, "comm probe needs an attached transport");
  Comm& cm = *c.comm;
  const bool up = cm.rank > 0, down = cm.rank < cm.world - 1;
  void *pong = nullptr, *ping = nullptr, *back = nullptr;
  ZB_CUDA(cudaMalloc(&pong, bytes));
  ZB_CUDA(cudaMalloc(&ping, bytes));
  ZB_CUDA(cudaMalloc(&back, bytes));
  ZB_CUDA(cudaMemset(ping, 0, bytes));
  const int warm = 2;
  std::vector<cudaEvent_t> t0(iters + warm), t1(iters + warm);
  for (int i = 0; i < iters + warm; ++i) {
    ZB_CUDA(cudaEventCreate(&t0[i]));
    ZB_CUDA(cudaEventCreate(&t1[i]));
  }
  for (int i = 0; i < iters + warm; ++i) {
    if (up) {
      recvb(cm, C_ACT_FROM, pong, bytes);
      order(cm, cm.stream[C_GRAD_TO], cm.stream[C_ACT_FROM]);
      sendb(cm, C_GRAD_TO, pong, bytes);
    }
    if (down) {
      ZB_CUDA(cudaEventRecord(t0[i], cm.stream[C_ACT_TO]));
      sendb(cm, C_ACT_TO, ping, bytes);
      order(cm, cm.stream[C_GRAD_FROM], cm.stream[C_ACT_TO]);
      recvb(cm, C_GRAD_FROM, back, bytes);
      ZB_CUDA(cudaEventRecord(t1[i], cm.stream[C_GRAD_FROM]));
    }
  }
  for (int w = 0; w < 4; ++w)
    if (cm.stream[w]) ZB_CUDA(cudaStreamSynchronize(cm.stream[w]));
  std::vector<int64_t> rt;
  if (down)
    for (int i = warm; i < iters + warm; ++i) {
      float ms = 0.f;
      ZB_CUDA(cudaEventElapsedTime(&ms, t0[i], t1[i]));
      rt.push_back(static_cast<int64_t>(static_cast<double>(ms) * 1e6 + 0.5));
    }
  for (int i = 0; i < iters + warm; ++i) {
    cudaEventDestroy(t0[i]);
    cudaEventDestroy(t1[i]);
  }
  cudaFree(pong);
  cudaFree(ping);
  cudaFree(back);
  if (rt.empty()) return 0;
  std::sort(rt.begin(), rt.end());
  return rt[rt.size() / 2];
}

void attach_nccl(Ctx& c, const void* ids, int rank, int world) {
  auto cm = std::make_unique<Comm>();
  cm->rank = rank;
  cm->world = world;
  auto tx = std::make_unique<NcclTransport>();
  const char* id = static_cast<const char*>(ids);
  auto init = [&](int which, int pair, bool grad) {
    ncclUniqueId_t u;
    std::memcpy(&u, id + 128 * (grad ? (world - 1 + pair) : pair), 128);
    const int r = (which == C_ACT_TO || which == C_GRAD_FROM) ? 0 : 1;
    nck(nccl().init(&tx->comm[which], 2, u, r), "ncclCommInitRank");
  };
  // increasing pair order on every rank: (s-1, s) before (s, s+1) -> no init deadlock
  if (rank > 0) {
    init(C_ACT_FROM, rank - 1, false);
    init(C_GRAD_TO, rank - 1, true);
  }
  if (rank < world - 1) {
    init(C_ACT_TO, rank, false);
    init(C_GRAD_FROM, rank, true);
  }
  cm->tx = std::move(tx);
  setup_comm(c, *cm);
  c.comm = std::move(cm);
}

// ---------------------------------------------------------------- data parallelism
// The D replicas of one stage share a D-rank communicator; gradient all-reduces (f32 sum, in
// place) run on its own stream, ordered after the W unit that completes them by an event, so
// they overlap the stage's remaining W work (App. A).  The compute stream waits for the last
// all-reduce at the end of the iteration (before the post-validation norm and the step).
DpComm::~DpComm() {
  if (stream) cudaStreamSynchronize(stream);
  if (comm) nccl().destroy(comm);
  if (stream) cudaStreamDestroy(stream);
  for (auto e : ev) cudaEventDestroy(e);
}

cudaEvent_t DpComm::event() {
  if (ev.size() < 256) {
    cudaEvent_t e;
    ZB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
    return e;
  }
  cudaEvent_t e = ev[ev_next];
  ev_next = (ev_next + 1) % static_cast<int>(ev.size());
  return e;
}

void attach_dp(Ctx& c, const void* id128, int dp_rank, int dp_world) {
  if (dp_world < 1 || dp_rank < 0 || dp_rank >= dp_world) throw Error(ZB_EINVAL, "bad data-parallel rank / world");
  auto d = std::make_unique<DpComm>();
  d->rank = dp_rank;
  d->world = dp_world;
  if (dp_world > 1) {
    if (!nccl().all_reduce) throw Error(ZB_ENCCL, "libnccl lacks ncclAllReduce");
    ncclUniqueId_t u;
    std::memcpy(&u, id128, 128);
    nck(nccl().init(&d->comm, dp_world, u, dp_rank), "ncclCommInitRank (data parallel)");
  }
  ZB_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  if (!c.comm) {  // p = 1: the plan runner needs a (transport-less) stage communicator
    if (c.cfg.p != 1) throw Error(ZB_EINVAL, "attach the P2P transport (zb_ctx_attach_nccl) before data parallelism");
    auto cm = std::make_unique<Comm>();
    cm->rank = 0;
    cm->world = 1;
    setup_comm(c, *cm);
    c.comm = std::move(cm);
  }
  c.dp = std::move(d);
  c.dp_world = dp_world;
}

// all-reduce of W unit u's gradient (u = -1: the vector region) after everything enqueued so
// far on the compute stream
void dp_all_reduce(Ctx& c, int u) {
  DpComm& d = *c.dp;
  int64_t off = 0, cnt = 0;
  c.unit_grad_range(u, &off, &cnt);
  cudaEvent_t e = d.event();
  ZB_CUDA(cudaEventRecord(e, c.stream));
  ZB_CUDA(cudaStreamWaitEvent(d.stream, e, 0));
  if (d.world > 1 && cnt > 0)
    nck(nccl().all_reduce(c.grad + off, c.grad + off, static_cast<size_t>(cnt), kNcclFloat32, kNcclSum, d.comm,
                          d.stream),
        "ncclAllReduce");
  ++d.reduces;
}

// the compute stream waits for every all-reduce issued so far
void dp_join(Ctx& c) {
  DpComm& d = *c.dp;
  cudaEvent_t e = d.event();
  ZB_CUDA(cudaEventRecord(e, d.stream));
  ZB_CUDA(cudaStreamWaitEvent(c.stream, e, 0));
}

int64_t dp_reduce_count(const Ctx& c) { return c.dp ? c.dp->reduces : 0; }

// ---------------------------------------------------------------- in-process loopback transport
namespace {
struct LbBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaEvent_t ready = nullptr, freed = nullptr;
};
struct LbMsg {
  int buf;
  size_t bytes;
};
struct LbChannel {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<LbMsg> queue;
  std::deque<LbBuf> bufs;  // deque: stable references while the channel grows
  std::vector<int> free_list;
  ~LbChannel() {
    for (auto& b : bufs) {
      if (b.p) cudaFree(b.p);
      if (b.ready) cudaEventDestroy(b.ready);
      if (b.freed) cudaEventDestroy(b.freed);
    }
  }
};
}  // namespace

struct LoopbackGroup {
  int world = 1;
  std::vector<std::unique_ptr<LbChannel>> act, grad;  // [k]: pair (k, k+1)
};

std::shared_ptr<LoopbackGroup> loopback_create(int world) {
  auto g = std::make_shared<LoopbackGroup>();
  g->world = world;
  for (int k = 0; k + 1 < world; ++k) {
    g->act.push_back(std::make_unique<LbChannel>());
    g->grad.push_back(std::make_unique<LbChannel>());
  }
  return g;
}

namespace {
int loopback_timeout_s() {  // ZB_LOOPBACK_TIMEOUT_S overrides the default 300 s
  static const int t = [] {
    const char* e = std::getenv("ZB_LOOPBACK_TIMEOUT_S");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 300;
  }();
  return t;
}

struct LoopbackTransport : Transport {
  std::shared_ptr<LoopbackGroup> g;
  int rank = 0;
  LbChannel& chan(int which) {
    switch (which) {
      case C_ACT_TO: return *g->act.at(rank);
      case C_ACT_FROM: return *g->act.at(rank - 1);
      case C_GRAD_TO: return *g->grad.at(rank - 1);
      default: return *g->grad.at(rank);
    }
  }
  void send(int which, const void* buf, size_t bytes, cudaStream_t st) override {
    LbChannel& ch = chan(which);
    LbBuf* b = nullptr;
    int idx = -1;
    {
      std::lock_guard<std::mutex> lk(ch.mu);
      for (size_t i = 0; i < ch.free_list.size(); ++i) {
        if (ch.bufs[ch.free_list[i]].cap >= bytes) {
          idx = ch.free_list[i];
          ch.free_list.erase(ch.free_list.begin() + static_cast<long>(i));
          break;
        }
      }
      if (idx < 0) {
        ch.bufs.emplace_back();
        idx = static_cast<int>(ch.bufs.size()) - 1;
        LbBuf& nb = ch.bufs.back();
        nb.cap = bytes < 64 ? 64 : bytes;
        ZB_CUDA(cudaMalloc(&nb.p, nb.cap));
        ZB_CUDA(cudaEventCreateWithFlags(&nb.ready, cudaEventDisableTiming));
        ZB_CUDA(cudaEventCreateWithFlags(&nb.freed, cudaEventDisableTiming));
      }
      b = &ch.bufs[idx];
    }
    ZB_CUDA(cudaStreamWaitEvent(st, b->freed, 0));  // the previous receiver has copied it out
    ZB_CUDA(cudaMemcpyAsync(b->p, buf, bytes, cudaMemcpyDeviceToDevice, st));
    ZB_CUDA(cudaEventRecord(b->ready, st));
    {
      std::lock_guard<std::mutex> lk(ch.mu);
      ch.queue.push_back({idx, bytes});
    }
    ch.cv.notify_all();
  }
  void recv(int which, void* buf, size_t bytes, cudaStream_t st) override {
    LbChannel& ch = chan(which);
    LbMsg msg;
    LbBuf* b = nullptr;
    {
      std::unique_lock<std::mutex> lk(ch.mu);
      if (!ch.cv.wait_for(lk, std::chrono::seconds(loopback_timeout_s()), [&] { return !ch.queue.empty(); }))
        throw Error(ZB_ETIMEOUT, "loopback receive timed out (rank " + std::to_string(rank) + ", channel " +
                                     std::to_string(which) + ")");
      msg = ch.queue.front();
      ch.queue.pop_front();
      b = &ch.bufs[msg.buf];
    }
    if (msg.bytes != bytes)
      throw Error(ZB_EINVAL, "loopback message size mismatch: sent " + std::to_string(msg.bytes) + ", expected " +
                                 std::to_string(bytes));
    ZB_CUDA(cudaStreamWaitEvent(st, b->ready, 0));
    ZB_CUDA(cudaMemcpyAsync(buf, b->p, bytes, cudaMemcpyDeviceToDevice, st));
    ZB_CUDA(cudaEventRecord(b->freed, st));
    {
      std::lock_guard<std::mutex> lk(ch.mu);
      ch.free_list.push_back(msg.buf);
    }
  }
};
}  // namespace

void attach_loopback(Ctx& c, const std::shared_ptr<LoopbackGroup>& g, int rank) {
  if (g->world != c.cfg.p) throw Error(ZB_EINVAL, "loopback group size must equal the context's p");
  auto cm = std::make_unique<Comm>();
  cm->rank = rank;
  cm->world = g->world;
  auto tx = std::make_unique<LoopbackTransport>();
  tx->g = g;
  tx->rank = rank;
  cm->tx = std::move(tx);
  setup_comm(c, *cm);
  c.comm = std::move(cm);
}

// ---------------------------------------------------------------- chunk contexts of one worker
namespace {
// per-channel composition: links to chunks on other workers ride NCCL, links between two
// chunks of this worker (ZB-V's V turn v = p-1 -> p) ride an in-process loopback channel
struct HybridTransport : Transport {
  std::unique_ptr<NcclTransport> nccl;
  std::unique_ptr<LoopbackTransport> local;
  Transport* sub[4] = {nullptr, nullptr, nullptr, nullptr};
  void send(int which, const void* buf, size_t bytes, cudaStream_t st) override {
    if (!sub[which]) throw Error(ZB_EINVAL, "hybrid transport: channel not attached");
    sub[which]->send(which, buf, bytes, st);
  }
  void recv(int which, void* buf, size_t bytes, cudaStream_t st) override {
    if (!sub[which]) throw Error(ZB_EINVAL, "hybrid transport: channel not attached");
    sub[which]->recv(which, buf, bytes, st);
  }
};
}  // namespace

void attach_nccl_chunks(const std::vector<Ctx*>& chunks, const void* ids, int nv, const std::vector<int>& worker_of,
                        int me) {
  if (static_cast<int>(worker_of.size()) != nv) throw Error(ZB_EINVAL, "worker_of must have nv entries");
  std::vector<Ctx*> byv(nv, nullptr);
  for (Ctx* c : chunks) {
    if (c->cfg.p != nv || worker_of.at(c->cfg.stage) != me) throw Error(ZB_EINVAL, "chunk context / worker mismatch");
    byv[c->cfg.stage] = c;
  }
  auto group = loopback_create(nv);
  std::vector<std::unique_ptr<HybridTransport>> tx(nv);
  for (Ctx* c : chunks) {
    const int v = c->cfg.stage;
    tx[v] = std::make_unique<HybridTransport>();
    tx[v]->nccl = std::make_unique<NcclTransport>();
    tx[v]->local = std::make_unique<LoopbackTransport>();
    tx[v]->local->g = group;
    tx[v]->local->rank = v;
  }
  const char* id = static_cast<const char*>(ids);
  auto nccl_init = [&](int v, int which, int link, bool grad, int r) {
    ncclUniqueId_t u;
    std::memcpy(&u, id + 128 * (grad ? (nv - 1 + link) : link), 128);
    nck(nccl().init(&tx[v]->nccl->comm[which], 2, u, r), "ncclCommInitRank");
    tx[v]->sub[which] = tx[v]->nccl.get();
  };
  // every process walks the links in increasing order and joins the remote ones it is on:
  // the lowest pending link always has both participants waiting on it -> no init deadlock
  for (int k = 0; k + 1 < nv; ++k) {
    const int a = k, b = k + 1;
    const bool ha = worker_of[a] == me, hb = worker_of[b] == me;
    if (ha && hb) {
      tx[a]->sub[C_ACT_TO] = tx[a]->local.get();
      tx[a]->sub[C_GRAD_FROM] = tx[a]->local.get();
      tx[b]->sub[C_ACT_FROM] = tx[b]->local.get();
      tx[b]->sub[C_GRAD_TO] = tx[b]->local.get();
    } else if (ha) {
      nccl_init(a, C_ACT_TO, k, false, 0);
      nccl_init(a, C_GRAD_FROM, k, true, 0);
    } else if (hb) {
      nccl_init(b, C_ACT_FROM, k, false, 1);
      nccl_init(b, C_GRAD_TO, k, true, 1);
    }
  }
  for (Ctx* c : chunks) {
    const int v = c->cfg.stage;
    auto cm = std::make_unique<Comm>();
    cm->rank = v;
    cm->world = nv;
    cm->tx = std::move(tx[v]);
    setup_comm(*c, *cm);
    c->comm = std::move(cm);
  }
}

// ---------------------------------------------------------------- post-validation messages
// message layout: double sumsq, int32 nonfinite, pad (16 bytes)
void pv_recv_partial(Ctx& c) {
  Comm& cm = *c.comm;
  if (c.cfg.stage == 0) {
    ZB_CUDA(cudaMemsetAsync(&c.pv->partial_in_sumsq, 0, sizeof(double), c.stream));
    ZB_CUDA(cudaMemsetAsync(&c.pv->partial_in_nf, 0, sizeof(int32_t), c.stream));
    return;
  }
  char* msg = static_cast<char*>(cm.scalars);
  order(cm, cm.stream[C_ACT_FROM], c.stream);
  recvb(cm, C_ACT_FROM, msg, 16);
  order(cm, c.stream, cm.stream[C_ACT_FROM]);
  ZB_CUDA(cudaMemcpyAsync(&c.pv->partial_in_sumsq, msg, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ZB_CUDA(cudaMemcpyAsync(&c.pv->partial_in_nf, msg + 8, sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
}

void pv_send_partial(Ctx& c) {
  Comm& cm = *c.comm;
  if (c.cfg.stage == c.cfg.p - 1) return;
  char* msg = static_cast<char*>(cm.scalars) + 16;
  ZB_CUDA(cudaMemcpyAsync(msg, &c.pv->partial_sumsq, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ZB_CUDA(cudaMemcpyAsync(msg + 8, &c.pv->partial_nf, sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
  order(cm, cm.stream[C_ACT_TO], c.stream);
  sendb(cm, C_ACT_TO, msg, 16);
}

void pv_recv_full(Ctx& c) {
  Comm& cm = *c.comm;
  if (c.cfg.stage == c.cfg.p - 1) {  // the last stage's partial state is the full state
    ZB_CUDA(cudaMemcpyAsync(&c.pv->full_sumsq, &c.pv->partial_sumsq, sizeof(double), cudaMemcpyDeviceToDevice,
                            c.stream));
    ZB_CUDA(cudaMemcpyAsync(&c.pv->full_nf, &c.pv->partial_nf, sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  char* msg = static_cast<char*>(cm.scalars) + 32;
  order(cm, cm.stream[C_GRAD_FROM], c.stream);
  recvb(cm, C_GRAD_FROM, msg, 16);
  order(cm, c.stream, cm.stream[C_GRAD_FROM]);
  ZB_CUDA(cudaMemcpyAsync(&c.pv->full_sumsq, msg, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ZB_CUDA(cudaMemcpyAsync(&c.pv->full_nf, msg + 8, sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
}

void pv_send_full(Ctx& c) {
  Comm& cm = *c.comm;
  if (c.cfg.stage == 0) return;
  char* msg = static_cast<char*>(cm.scalars) + 48;
  ZB_CUDA(cudaMemcpyAsync(msg, &c.pv->full_sumsq, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  ZB_CUDA(cudaMemcpyAsync(msg + 8, &c.pv->full_nf, sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
  order(cm, cm.stream[C_GRAD_TO], c.stream);
  sendb(cm, C_GRAD_TO, msg, 16);
}

// ---------------------------------------------------------------- runner
// Executes plan ops of ONE stage context (its send rings and input pointers).
struct StageExec {
  Ctx& c;
  Comm& cm;
  const int32_t* tokens;
  const int32_t* labels;
  int flags;
  size_t act_bytes, grad_bytes;
  int act_ring = 0, grad_ring = 0, last_act_buf = -1, last_grad_buf = -1;

  StageExec(Ctx& c_, const int32_t* tok, const int32_t* lab, int fl)
      : c(c_), cm(*c_.comm), tokens(tok), labels(lab), flags(fl) {
    act_bytes = c.esz * static_cast<size_t>(c.T) * c.h;
    grad_bytes = sizeof(float) * static_cast<size_t>(c.T) * c.h;  // f32 gradient stream (R-grad32)
  }

  // H2D of host inputs, input checks, per-iteration resets (as the single-stage runner)
  void begin() {
    const size_t nt = static_cast<size_t>(c.cfg.m) * c.T;
    if (flags & ZB_RUN_HOST_INPUTS) {
      if (c.first && tokens) {
        ZB_CUDA(cudaMemcpyAsync(c.tok_stage, tokens, nt * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
        tokens = c.tok_stage;
      }
      if (c.last && labels) {
        ZB_CUDA(cudaMemcpyAsync(c.lab_stage, labels, nt * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
        labels = c.lab_stage;
      }
    }
    if (c.first && !tokens) throw Error(ZB_EINVAL, "tokens required on stage 0");
    if (c.last && !labels) throw Error(ZB_EINVAL, "labels required on the last stage");
    c.first_b_done = c.first_w_done = false;
    c.unit_w_done.assign(c.n_w_units(), 0);
    ZB_CUDA(cudaMemsetAsync(c.loss_acc, 0, sizeof(double), c.stream));
    c.n_timed = 0;
  }

  void exec(const plan::Op& op) {
    const int T = c.T;
    Slot* sl = op.slot >= 0 ? &c.slots.at(op.slot) : nullptr;
    switch (op.type) {
      case plan::OP_RECV_ACT: {
        order(cm, cm.stream[C_ACT_FROM], c.stream);  // the slot's previous user has finished
        recvb(cm, C_ACT_FROM, sl->L[0].x, act_bytes);
        order(cm, c.stream, cm.stream[C_ACT_FROM]);
        break;
      }
      case plan::OP_DISCARD_ACT: {
        recvb(cm, C_ACT_FROM, static_cast<char*>(cm.scalars) + 64, act_bytes);
        break;
      }
      case plan::OP_F:
      case plan::OP_REPLAY_F: {
        void* out = nullptr;
        if (!c.last) {
          last_act_buf = act_ring;
          ZB_CUDA(cudaStreamWaitEvent(c.stream, cm.act_buf_free[act_ring], 0));
          out = cm.act_buf[act_ring];
          act_ring = (act_ring + 1) % static_cast<int>(cm.act_buf.size());
        }
        if (flags & ZB_RUN_TIMING) c.timing_begin(c.n_timed, ZB_F);  // after the waits: pass time only
        const void* in = c.first ? static_cast<const void*>(tokens + static_cast<int64_t>(op.mb) * T) : sl->L[0].x;
        c.forward(op.mb, op.slot, in, out, c.last ? labels + static_cast<int64_t>(op.mb) * T : nullptr);
        if (flags & ZB_RUN_TIMING) c.timing_end(c.n_timed++);
        break;
      }
      case plan::OP_SEND_ACT: {
        order(cm, cm.stream[C_ACT_TO], c.stream);
        sendb(cm, C_ACT_TO, cm.act_buf[last_act_buf], act_bytes);
        ZB_CUDA(cudaEventRecord(cm.act_buf_free[last_act_buf], cm.stream[C_ACT_TO]));
        break;
      }
      case plan::OP_RECV_GRAD: {
        order(cm, cm.stream[C_GRAD_FROM], c.stream);
        recvb(cm, C_GRAD_FROM, sl->dy32, grad_bytes);
        order(cm, c.stream, cm.stream[C_GRAD_FROM]);
        break;
      }
      case plan::OP_B: {
        float* dx = nullptr;
        if (!c.first) {
          last_grad_buf = grad_ring;
          ZB_CUDA(cudaStreamWaitEvent(c.stream, cm.grad_buf_free[grad_ring], 0));
          dx = cm.grad_buf[grad_ring];
          grad_ring = (grad_ring + 1) % static_cast<int>(cm.grad_buf.size());
        }
        if (flags & ZB_RUN_TIMING) c.timing_begin(c.n_timed, ZB_B);
        c.backward_input(op.mb, op.slot, c.last ? nullptr : sl->dy32, dx);
        if (flags & ZB_RUN_TIMING) c.timing_end(c.n_timed++);
        break;
      }
      case plan::OP_SEND_GRAD: {
        order(cm, cm.stream[C_GRAD_TO], c.stream);
        sendb(cm, C_GRAD_TO, cm.grad_buf[last_grad_buf], grad_bytes);  // f32 dX of the stage input
        ZB_CUDA(cudaEventRecord(cm.grad_buf_free[last_grad_buf], cm.stream[C_GRAD_TO]));
        break;
      }
      case plan::OP_W: {
        if (flags & ZB_RUN_TIMING) c.timing_begin(c.n_timed, ZB_W);
        c.backward_weight(op.mb, op.slot);
        if (flags & ZB_RUN_TIMING) c.timing_end(c.n_timed++);
        break;
      }
      case plan::OP_WP: {  // one W unit of one tail microbatch (data parallelism)
        const int sl1[1] = {op.slot};
        c.weight_unit(op.msg, sl1, 1);
        break;
      }
      case plan::OP_ALLREDUCE: {
        dp_all_reduce(c, op.msg);
        break;
      }
      default:
        throw Error(ZB_EINVAL, "StageExec: unexpected op");
    }
  }
  // k adjacent OP_WP of the same unit as one contraction (ZB_RUN_GROUP_W)
  void exec_wp_group(const plan::Op* ops, int k) {
    int sls[kMaxSeg];
    for (int i = 0; i < k; ++i) sls[i] = ops[i].slot;
    c.weight_unit(ops[0].msg, sls, k);
  }
  // W-grouping (ZB_RUN_GROUP_W): k adjacent W ops as one contraction per linear
  void exec_w_group(const plan::Op* ops, int k) {
    int mbs[kMaxSeg], sls[kMaxSeg];
    for (int i = 0; i < k; ++i) {
      mbs[i] = ops[i].mb;
      sls[i] = ops[i].slot;
    }
    if (flags & ZB_RUN_TIMING) c.timing_begin(c.n_timed, ZB_W, k);
    c.backward_weight_group(mbs, sls, k);
    if (flags & ZB_RUN_TIMING) c.timing_end(c.n_timed++);
  }
};

void run_iteration_nccl(Ctx& c, const zb_pass_t* passes, int n, const int32_t* tokens, const int32_t* labels,
                        int flags) {
  const int p = c.cfg.p, m = c.cfg.m, s = c.cfg.stage;
  const bool fused = (flags & ZB_RUN_FUSED_BW) != 0;
  StageExec ex(c, tokens, labels, flags);
  ex.begin();
  const bool pending = c.pv_pending;
  std::vector<plan::Op> ops = plan::stage_plan(passes, n, p, m, s, pending, false, fused);
  std::vector<plan::Op> ops_amend;
  if (pending) ops_amend = plan::stage_plan(passes, n, p, m, s, true, true, fused);
  if (c.dp) {  // the tail Ws as per-unit sub-computations + all-reduces (plan.h dp_tail)
    const bool reorder = (flags & ZB_RUN_DP_REORDER) != 0;
    ops = plan::dp_tail(ops, c.n_w_units(), reorder);
    if (pending) ops_amend = plan::dp_tail(ops_amend, c.n_w_units(), reorder);
  }
  bool switched = false;
  for (size_t k = 0; k < ops.size(); ++k) {
    const plan::Op op = ops[k];
    if (op.type == plan::OP_WP && (flags & ZB_RUN_GROUP_W)) {
      int g = 1;
      while (g < kMaxSeg && k + g < ops.size() && ops[k + g].type == plan::OP_WP && ops[k + g].msg == op.msg) ++g;
      ex.exec_wp_group(&ops[k], g);
      k += g - 1;
      continue;
    }
    if (op.type == plan::OP_W && (flags & ZB_RUN_GROUP_W)) {
      int g = 1;
      while (g < kMaxSeg && k + g < ops.size() && ops[k + g].type == plan::OP_W) ++g;
      ex.exec_w_group(&ops[k], g);
      k += g - 1;
      continue;
    }
    if (op.type != plan::OP_VALIDATE) {
      ex.exec(op);
      continue;
    }
    pv_recv_full(c);
    pv_send_full(c);
    pv_decide_final(c.pv, c.pv_clip, c.stream);
    adamw_apply(c.theta, c.m, c.v, c.grad, c.shadow, c.n_total, c.n_wd, c.shadow ? c.n_shadow : 0, c.pv_opt[0],
                c.pv_opt[1], c.pv_opt[2], c.pv_opt[3], c.pv_opt[4], c.pv, true, c.stream);
    pv_finish_apply(c.pv, c.stream);
    c.pv_pending = false;
    // the host needs the outcome to know whether the speculative Fs must be replayed
    PvState hst;
    ZB_CUDA(cudaMemcpyAsync(&hst, c.pv, sizeof(PvState), cudaMemcpyDeviceToHost, c.stream));
    ZB_CUDA(cudaStreamSynchronize(c.stream));
    const double coef = c.pv_clip / (std::sqrt(hst.full_sumsq) + 1e-6);
    const bool amend = hst.full_nf != 0 || coef < 1.0;  // identical on every stage
    if (amend && !switched) {
      ops = ops_amend;  // same prefix up to and including this VALIDATE
      switched = true;
    }
  }
  if (c.dp) dp_join(c);
}

void run_iteration_worker(const std::vector<Ctx*>& chunks, const zb_pass_t* passes, int n, const int32_t* tokens,
                          const int32_t* labels, int flags) {
  if (chunks.empty()) throw Error(ZB_EINVAL, "no chunk contexts");
  const int nv = chunks[0]->cfg.p, m = chunks[0]->cfg.m;
  std::vector<int> worker_of(nv, -1);
  std::vector<StageExec*> ex(nv, nullptr);
  std::vector<std::unique_ptr<StageExec>> own;
  // passes come grouped by worker (zb_schedule_chunked), chunks x 3m passes per worker
  const int per_worker = 3 * m * static_cast<int>(chunks.size());
  if (per_worker <= 0 || n % per_worker) throw Error(ZB_EINVAL, "pass count is not workers x chunks x 3m");
  for (int i = 0; i < n; ++i) {
    const int v = passes[i].stage, w = i / per_worker;
    if (worker_of[v] >= 0 && worker_of[v] != w) throw Error(ZB_EINVAL, "a virtual stage spans two workers");
    worker_of[v] = w;
  }
  int me = -1;
  for (Ctx* c : chunks) {
    if (c->cfg.p != nv || c->cfg.m != m || !c->comm) throw Error(ZB_EINVAL, "chunk contexts must share p, m and a transport");
    const int v = c->cfg.stage;
    if (me >= 0 && worker_of[v] != me) throw Error(ZB_EINVAL, "chunk contexts belong to different workers");
    me = worker_of[v];
    if (c->pv_pending) throw Error(ZB_ESTATE, "chunked schedules: call zb_post_validate_finish before the next iteration");
    own.emplace_back(new StageExec(*c, c->first ? tokens : nullptr, c->last ? labels : nullptr, flags));
    ex[v] = own.back().get();
    ex[v]->begin();
  }
  for (const plan::WOp& w : plan::worker_plan(passes, n, nv, m, me, worker_of.data(), (flags & ZB_RUN_FUSED_BW) != 0)) {
    if (!ex[w.chunk]) throw Error(ZB_EINVAL, "worker plan references a chunk without a context");
    ex[w.chunk]->exec(w.op);
  }
}

}  // namespace zb
