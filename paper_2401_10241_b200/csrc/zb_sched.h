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
Lists heuristic(int p, int m, int64_t TF, int64_t TB, int64_t TW, int64_t Tc, int64_t MB, int64_t MW, int64_t Mlimit,
                bool fill_warmup, bool skip_lead);
Lists auto_schedule(int p, int m, int64_t TF, int64_t TB, int64_t TW, int64_t Tc, int64_t MB, int64_t MW,
                    int64_t Mlimit, int* chosen);
SimResult simulate(const Lists& lists, const std::vector<int64_t>& TF, const std::vector<int64_t>& TB,
                   const std::vector<int64_t>& TW, int64_t Tcomm, bool fused);
std::vector<int64_t> memory_peaks(const Lists& lists, int64_t MB, int64_t MW);
std::vector<std::vector<int>> assign_slots(const Lists& lists, std::vector<int>* counts);

}  // namespace sched
}  // namespace zb
