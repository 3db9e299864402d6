// Host-side schedule construction and simulation (zb_schedule, zb_simulate).
//
// PAPER.md §2: 1F1B, ZB-H1, ZB-H2 as warm-up / W-deferral / steady
// order parameters (SURVEY.md Appendix A reading, DESIGN.md R-sched);
// §3.1: the AUTO heuristic with its two binary hyper-parameters
// and grid search (SURVEY.md Appendix B reading); App. F: passes
// (i, j, c), Delta-M memory and the dependency constraints (4)-(6) used as
// ASAP execution semantics; §5.3: bubble rate.
// All times and bytes are int64 so the C++ and oracle schedules compare exactly.
#include <algorithm>
#include <cstdint>
#include <deque>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "zb_sched.h"

namespace zb {
namespace sched {

namespace {

Lists generic_builder(int p, int m, const std::vector<int>& warm, const std::vector<int>& defer, bool bf_order) {
  Lists out(p);
  for (int s = 0; s < p; ++s) {
    auto& o = out[s];
    int w = std::min(warm[s], m);
    for (int j = 0; j < w; ++j) o.push_back({KIND_F, j});
    int nf = w, nb = 0, nw = 0;
    while (nb < m) {
      if (!bf_order) {
        if (nf < m) o.push_back({KIND_F, nf++});
        o.push_back({KIND_B, nb++});
        if (nb - nw > defer[s]) o.push_back({KIND_W, nw++});
      } else {
        o.push_back({KIND_B, nb++});
        if (nb - nw > defer[s]) o.push_back({KIND_W, nw++});
        if (nf < m) o.push_back({KIND_F, nf++});
      }
    }
    while (nw < m) o.push_back({KIND_W, nw++});
  }
  return out;
}

}  // namespace

Lists build_1f1b(int p, int m) {
  std::vector<int> w(p), d(p, 0);
  for (int s = 0; s < p; ++s) w[s] = p - 1 - s;
  return generic_builder(p, m, w, d, false);
}

Lists build_zbh1(int p, int m) {
  std::vector<int> w(p), d(p);
  for (int s = 0; s < p; ++s) {
    w[s] = p - 1 - s;
    d[s] = s;
  }
  return generic_builder(p, m, w, d, false);
}

Lists build_zbh2(int p, int m) {
  std::vector<int> w(p), d(p);
  for (int s = 0; s < p; ++s) {
    w[s] = 2 * (p - s) - 1;
    d[s] = 2 * s;
  }
  return generic_builder(p, m, w, d, true);
}

SimResult simulate(const Lists& lists, const std::vector<int64_t>& TF, const std::vector<int64_t>& TB,
                   const std::vector<int64_t>& TW, int64_t Tcomm, bool fused) {
  const int p = static_cast<int>(lists.size());
  int m = 0;
  for (auto& ps : lists[0]) m = std::max(m, ps.j + 1);
  SimResult r;
  r.start.assign(p, {});
  r.end.assign(p, {});
  // end time per (kind, stage, j); -1 = not yet executed
  std::vector<std::vector<int64_t>> endk[3];
  for (int k = 0; k < 3; ++k) endk[k].assign(p, std::vector<int64_t>(m, -1));
  std::vector<size_t> pos(p, 0);
  std::vector<int64_t> free_at(p, 0);
  size_t total = 0, done = 0;
  for (auto& o : lists) total += o.size();
  for (int s = 0; s < p; ++s) {
    r.start[s].assign(lists[s].size(), 0);
    r.end[s].assign(lists[s].size(), 0);
  }
  while (done < total) {
    bool progressed = false;
    for (int s = 0; s < p; ++s) {
      while (pos[s] < lists[s].size()) {
        const Pass& ps = lists[s][pos[s]];
        int64_t t0 = free_at[s];
        bool ready = true;
        auto dep = [&](int kind, int stage, bool comm) {
          int64_t e = endk[kind][stage][ps.j];
          if (e < 0) {
            ready = false;
            return;
          }
          t0 = std::max(t0, e + (comm ? Tcomm : 0));
        };
        if (ps.kind == KIND_F) {
          if (s > 0) dep(KIND_F, s - 1, true);
        } else if (ps.kind == KIND_B) {
          dep(KIND_F, s, false);
          if (s < p - 1) dep(fused ? KIND_W : KIND_B, s + 1, true);
        } else {
          dep(KIND_B, s, false);
        }
        if (!ready) break;
        const int64_t dur = ps.kind == KIND_F ? TF[s] : (ps.kind == KIND_B ? TB[s] : TW[s]);
        r.start[s][pos[s]] = t0;
        r.end[s][pos[s]] = t0 + dur;
        endk[ps.kind][s][ps.j] = t0 + dur;
        free_at[s] = t0 + dur;
        ++pos[s];
        ++done;
        progressed = true;
      }
    }
    if (!progressed) throw std::runtime_error("schedule deadlocks: a dependency can never be met");
  }
  r.cost = 0;
  r.work = 0;
  for (int s = 0; s < p; ++s) {
    if (lists[s].empty()) continue;
    r.cost = std::max(r.cost, r.end[s].back() - r.start[s].front());
    r.work = std::max(r.work, static_cast<int64_t>(m) * (TF[s] + TB[s] + TW[s]));
  }
  r.bubble_rate = r.cost > 0 ? static_cast<double>(r.cost - r.work) / static_cast<double>(r.cost) : 0.0;
  return r;
}

std::vector<int64_t> memory_peaks(const Lists& lists, int64_t MB, int64_t MW) {
  std::vector<int64_t> out;
  for (auto& o : lists) {
    int64_t cur = 0, peak = 0;
    for (auto& ps : o) {
      cur += ps.kind == KIND_F ? MB : (ps.kind == KIND_B ? MW - MB : -MW);
      peak = std::max(peak, cur);
    }
    out.push_back(peak);
  }
  return out;
}

std::vector<std::vector<int>> assign_slots(const Lists& lists, std::vector<int>* counts) {
  std::vector<std::vector<int>> slots(lists.size());
  if (counts) counts->assign(lists.size(), 0);
  for (size_t s = 0; s < lists.size(); ++s) {
    int m = 0;
    for (auto& ps : lists[s]) m = std::max(m, ps.j + 1);
    std::vector<int> of_mb(m, -1);
    std::vector<int> free_list;
    int next = 0;
    for (auto& ps : lists[s]) {
      int sl = -1;
      if (ps.kind == KIND_F) {
        if (!free_list.empty()) {
          auto it = std::min_element(free_list.begin(), free_list.end());
          sl = *it;
          free_list.erase(it);
        } else {
          sl = next++;
        }
        of_mb[ps.j] = sl;
      } else {
        sl = of_mb[ps.j];
        if (ps.kind == KIND_W) free_list.push_back(sl);
      }
      slots[s].push_back(sl);
    }
    if (counts) (*counts)[s] = next;
  }
  return slots;
}

// AUTO heuristic, one reading of §3.1; see DESIGN.md R-auto.
Lists heuristic(int p, int m, const std::vector<int64_t>& TF, const std::vector<int64_t>& TB,
                const std::vector<int64_t>& TW, int64_t Tc, int64_t MB, int64_t MW, int64_t Mlimit, bool fill_warmup,
                bool skip_lead) {
  if (Mlimit < MB) throw std::invalid_argument("M_limit below M_B");
  const int64_t UNKNOWN = -1, NA = -2;  // arrival states; >= 0 means known time
  std::vector<int> nF(p, 0), nB(p, 0), nW(p, 0);
  std::vector<std::deque<int>> pend(p);
  std::vector<int64_t> mem(p, 0), bub(p, 0), busy(p, 0);
  std::vector<bool> started(p, false);
  std::vector<int> last(p, -1);
  std::vector<std::vector<int64_t>> endF(p, std::vector<int64_t>(m, -1)), endB(p, std::vector<int64_t>(m, -1));
  Lists lists(p);

  auto arrivals = [&](int s, int64_t& aF, int64_t& aB) {
    if (nF[s] >= m) aF = NA;
    else if (s == 0) aF = 0;
    else if (endF[s - 1][nF[s]] >= 0) aF = endF[s - 1][nF[s]] + Tc;
    else aF = UNKNOWN;
    if (nB[s] >= nF[s]) aB = NA;
    else if (s == p - 1) aB = endF[s][nB[s]];
    else if (endB[s + 1][nB[s]] >= 0) aB = endB[s + 1][nB[s]] + Tc;
    else aB = UNKNOWN;
  };
  auto known = [](int64_t a) { return a >= 0; };
  auto unfinished = [&]() {
    for (int s = 0; s < p; ++s)
      if (nW[s] < m) return true;
    return false;
  };

  int64_t t = 0;
  long guard = 0;
  while (unfinished()) {
    if (++guard > 100L * p * m + 1000) throw std::runtime_error("heuristic did not terminate");
    for (int s = 0; s < p; ++s) {
      if (nW[s] >= m || busy[s] > t) continue;
      int64_t aF, aB;
      arrivals(s, aF, aB);
      bool memOK = nF[s] < m && mem[s] + MB <= Mlimit;
      if (skip_lead && s < p - 1 && nF[s] < m && nF[s] - nF[s + 1] > 1 && nB[s] > 0 && known(aB) && aB <= t)
        memOK = false;
      const bool Fready = memOK && known(aF) && aF <= t;
      const bool Bready = known(aB) && aB <= t;
      int pick = -1;
      if (nB[s] == 0) {
        if (Bready) {
          pick = KIND_B;
        } else if (Fready) {
          bool delays = (known(aB) && aB < t + TF[s]) || (aB == UNKNOWN && TB[s] + Tc < TF[s]);
          if (!delays || fill_warmup) pick = KIND_F;
        }
      } else {
        if (Bready && Fready) pick = (last[s] == KIND_B) ? KIND_F : KIND_B;
        else if (Bready) pick = KIND_B;
        else if (Fready) pick = KIND_F;
      }
      if (pick < 0 && !pend[s].empty()) {
        // r: next known arrival of F (if memory allows one) or B; "infinite" if none
        bool have_r = false;
        int64_t r = 0;
        if (nF[s] < m && mem[s] + MB <= Mlimit && known(aF)) {
          r = aF;
          have_r = true;
        }
        if (known(aB)) {
          r = have_r ? std::min(r, aB) : aB;
          have_r = true;
        }
        int64_t others = 0;
        bool any_other = false;
        for (int x = 0; x < p; ++x)
          if (x != s) {
            others = any_other ? std::max(others, bub[x]) : bub[x];
            any_other = true;
          }
        if (!any_other) others = 0;
        const bool gap_ok = !have_r || (r - t >= TW[s]);
        if ((nF[s] < m && mem[s] + MB > Mlimit && !Bready) || gap_ok || (nF[s] == m && nB[s] == m)) {
          pick = KIND_W;
        } else if (have_r && r > t && bub[s] + (r - t) > others) {
          pick = KIND_W;
        }
      }
      if (pick < 0) continue;
      if (started[s]) bub[s] += t - busy[s];
      started[s] = true;
      int j;
      if (pick == KIND_F) {
        j = nF[s]++;
        endF[s][j] = t + TF[s];
        mem[s] += MB;
        busy[s] = t + TF[s];
      } else if (pick == KIND_B) {
        j = nB[s]++;
        endB[s][j] = t + TB[s];
        mem[s] += MW - MB;
        pend[s].push_back(j);
        busy[s] = t + TB[s];
      } else {
        j = pend[s].front();
        pend[s].pop_front();
        ++nW[s];
        mem[s] -= MW;
        busy[s] = t + TW[s];
      }
      last[s] = pick;
      lists[s].push_back({pick, j});
    }
    bool have = false;
    int64_t nxt = 0;
    for (int s = 0; s < p; ++s) {
      if (nW[s] >= m) continue;
      auto consider = [&](int64_t v) {
        if (v > t) {
          nxt = have ? std::min(nxt, v) : v;
          have = true;
        }
      };
      if (busy[s] > t) consider(busy[s]);
      int64_t aF, aB;
      arrivals(s, aF, aB);
      if (known(aF)) consider(aF);
      if (known(aB)) consider(aB);
    }
    if (!have) {
      if (unfinished()) throw std::runtime_error("heuristic stalled");
      break;
    }
    t = nxt;
  }
  return lists;
}

Lists auto_schedule(int p, int m, const std::vector<int64_t>& tf, const std::vector<int64_t>& tb,
                    const std::vector<int64_t>& tw, int64_t Tc, int64_t MB, int64_t MW, int64_t Mlimit, int* chosen) {
  struct Cand {
    int idx;
    Lists l;
  };
  std::vector<Cand> cands;
  for (int fill = 0; fill < 2; ++fill)
    for (int skip = 0; skip < 2; ++skip)
      cands.push_back({2 * fill + skip, heuristic(p, m, tf, tb, tw, Tc, MB, MW, Mlimit, fill, skip)});
  {
    Lists h1 = build_zbh1(p, m);
    auto pk = memory_peaks(h1, MB, MW);
    if (*std::max_element(pk.begin(), pk.end()) <= Mlimit) cands.push_back({4, h1});
    Lists h2 = build_zbh2(p, m);
    pk = memory_peaks(h2, MB, MW);
    if (*std::max_element(pk.begin(), pk.end()) <= Mlimit) cands.push_back({5, h2});
  }
  int best = -1;
  int64_t bc = 0, bp = 0;
  int bi = 0;
  for (size_t i = 0; i < cands.size(); ++i) {
    SimResult r = simulate(cands[i].l, tf, tb, tw, Tc, false);
    auto pk = memory_peaks(cands[i].l, MB, MW);
    int64_t peak = *std::max_element(pk.begin(), pk.end());
    bool better = best < 0 || r.cost < bc || (r.cost == bc && (peak < bp || (peak == bp && cands[i].idx < bi)));
    if (better) {
      best = static_cast<int>(i);
      bc = r.cost;
      bp = peak;
      bi = cands[i].idx;
    }
  }
  *chosen = cands[best].idx;
  return cands[best].l;
}

}  // namespace sched
}  // namespace zb
