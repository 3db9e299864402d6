#include "ktimer.h"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace zb {

namespace {
std::atomic<int64_t> g_launches{0};
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count(bool reset) { return reset ? g_launches.exchange(0) : g_launches.load(); }
bool pdl_enabled(int cls) {
  static const int mask = [] {
    const char* e = std::getenv("ZB_PDL");
    return e ? std::atoi(e) : 3;  // default: PDL_GEMM | PDL_ATTN, the TMEM kernels (common.cuh)
  }();
  return (mask & cls) != 0;
}

namespace {
void CUDART_CB print_name(void* name) { std::fprintf(stderr, "[zb] done-> %s\n", static_cast<const char*>(name)); }
}  // namespace

void trace_launch(const void* kern, cudaStream_t st) {
  static const bool on = std::getenv("ZB_TRACE_LAUNCH") != nullptr;
  if (!on) return;
  const char* name = nullptr;
  if (cudaFuncGetName(&name, kern) != cudaSuccess || !name) name = "?";
  std::fprintf(stderr, "[zb] launch %s\n", name);
  cudaLaunchHostFunc(st, print_name, const_cast<char*>(name));
}
namespace ktimer {

namespace {
struct Rec {
  cudaEvent_t a, b;
  int cls;
  double flops;
};
std::mutex mu;
bool on = false;
std::vector<Rec> pending;
std::vector<cudaEvent_t> pool;
double tot_ms[N_CLASSES], tot_flops[N_CLASSES];
int64_t tot_n[N_CLASSES];

cudaEvent_t get_event() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void drain_locked() {
  for (auto& r : pending) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    tot_ms[r.cls] += ms;
    tot_flops[r.cls] += r.flops;
    tot_n[r.cls] += 1;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  pending.clear();
}
}  // namespace

bool enabled() { return on; }

void set_enabled(bool e) {
  std::lock_guard<std::mutex> g(mu);
  on = e;
}

int start(int cls, double flops, cudaStream_t s) {
  if (!on) return -1;
  std::lock_guard<std::mutex> g(mu);
  if (pending.size() > 8192) drain_locked();
  Rec r{get_event(), get_event(), cls, flops};
  cudaEventRecord(r.a, s);
  pending.push_back(r);
  return static_cast<int>(pending.size()) - 1;
}

void stop(int idx, cudaStream_t s) {
  if (idx < 0) return;
  std::lock_guard<std::mutex> g(mu);
  if (idx < static_cast<int>(pending.size())) cudaEventRecord(pending[idx].b, s);
}

void read(int cls, double* ms, double* flops, int64_t* n) {
  std::lock_guard<std::mutex> g(mu);
  drain_locked();
  *ms = tot_ms[cls];
  *flops = tot_flops[cls];
  *n = tot_n[cls];
}

void reset() {
  std::lock_guard<std::mutex> g(mu);
  drain_locked();
  for (int i = 0; i < N_CLASSES; ++i) tot_ms[i] = tot_flops[i] = 0, tot_n[i] = 0;
}

}  // namespace ktimer
}  // namespace zb
