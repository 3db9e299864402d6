// Host scheduler internals behind zb_schedule / zb_simulate (sched.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace zb {
namespace sched {

enum { KIND_F = 0, KIND_B = 1, KIND_W = 2 };

struct Pass {
  int kind;
  int j;
};
typedef std::vector<std::vector<Pass>> Lists;

struct SimResult {
  std::vector<std::vector<int64_t>> start, end;  // per stage, per position
  int64_t cost = 0, work = 0;
  double bubble_rate = 0.0;
};

Lists build_1f1b(int p, int m);
Lists build_zbh1(int p, int m);
Lists build_zbh2(int p, int m);
// per-stage times TF[p], TB[p], TW[p] (each stage's profiled times feed the scheduler)
Lists heuristic(int p, int m, const std::vector<int64_t>& TF, const std::vector<int64_t>& TB,
                const std::vector<int64_t>& TW, int64_t Tc, int64_t MB, int64_t MW, int64_t Mlimit, bool fill_warmup,
                bool skip_lead);
Lists auto_schedule(int p, int m, const std::vector<int64_t>& TF, const std::vector<int64_t>& TB,
                    const std::vector<int64_t>& TW, int64_t Tc, int64_t MB, int64_t MW, int64_t Mlimit, int* chosen);
SimResult simulate(const Lists& lists, const std::vector<int64_t>& TF, const std::vector<int64_t>& TB,
                   const std::vector<int64_t>& TW, int64_t Tcomm, bool fused);
std::vector<int64_t> memory_peaks(const Lists& lists, int64_t MB, int64_t MW);
std::vector<std::vector<int>> assign_slots(const Lists& lists, std::vector<int>* counts);

// ---- several model chunks per worker (sched_v.cpp): ZB-V, 1F1B-I
struct VPass {
  int kind;
  int v;  // virtual stage (model chunk) in [0, chunks * p)
  int j;
};
typedef std::vector<std::vector<VPass>> VLists;  // per worker, in execution order

struct VSimResult {
  std::vector<std::vector<int64_t>> start, end;  // per worker, per position
  int64_t cost = 0, work = 0;
  double bubble_rate = 0.0;
};

int zbv_worker(int p, int v);  // V placement: v < p on worker v, else 2p-1-v
VLists build_zbv(int p, int m);
VLists build_1f1b_interleaved(int p, int m, int chunks);
VSimResult simulate_v(const VLists& lists, int nv, const std::vector<int>& place, const std::vector<int64_t>& TF,
                      const std::vector<int64_t>& TB, const std::vector<int64_t>& TW, int64_t Tcomm, bool fused);
std::vector<int64_t> memory_peaks_v(const VLists& lists, int64_t MB, int64_t MW);
std::vector<std::vector<int>> assign_slots_v(const VLists& lists, int nv, std::vector<int>* counts);
VLists zbv_shift_w(const VLists& lists, int p, int64_t TF, int64_t TB, int64_t TW, int64_t Tc, int64_t MB, int64_t MW,
                   int64_t Mlimit, bool fill);
VLists zbv_schedule(int p, int m, int64_t TF, int64_t TB, int64_t TW, int64_t Tc, int64_t MB, int64_t MW,
                    int64_t Mlimit, int* chosen);

}  // namespace sched
}  // namespace zb
