// Host schedules with several model chunks ("virtual stages") per worker:
// ZB-V (§6) and interleaved 1F1B (1F1B-I), plus
// the virtual-stage simulator (App. F (4)-(6) with a placement), per-worker
// Delta-M memory and the ZB-V W right-shift under M_limit.
// Readings: DESIGN.md R-zbv / R-1f1bi (identical to oracle/zbv.py, which the
// tests compare pass for pass).
#include <algorithm>
#include <cstdint>
#include <deque>
#include <stdexcept>
#include <vector>

#include "zb_sched.h"

namespace zb {
namespace sched {

int zbv_worker(int p, int v) { return v < p ? v : 2 * p - 1 - v; }

namespace {
constexpr int64_t NONE = -1;  // "not executed yet" for end times

struct EndTable {
  int nv, m;
  std::vector<int64_t> e;
  EndTable(int nv_, int m_) : nv(nv_), m(m_), e(static_cast<size_t>(nv_) * m_, NONE) {}
  int64_t& at(int v, int j) { return e[static_cast<size_t>(v) * m + j]; }
};
}  // namespace

// ---------------------------------------------------------------- ZB-V construction (unit times)
VLists build_zbv(int p, int m) {
  if (p < 1 || m < 1) throw std::invalid_argument("p, m >= 1");
  const int V = 2 * p;
  EndTable endF(V, m), endB(V, m);
  std::vector<int> nF(2 * p, 0), nB(2 * p, 0), nW(2 * p, 0);  // [w*2 + c]
  std::vector<int> gchunk(p, -1), gstep(p, 0), ngroups(p, 0);
  VLists lists(p);
  auto cv = [&](int w, int c) { return c == 0 ? w : 2 * p - 1 - w; };
  auto readyF = [&](int w, int c, int64_t t) {
    const int j = nF[2 * w + c];
    if (j >= m) return false;
    const int v = cv(w, c);
    if (v == 0) return true;
    const int64_t e = endF.at(v - 1, j);
    return e != NONE && e <= t;
  };
  auto readyB = [&](int w, int c, int64_t t) {
    const int j = nB[2 * w + c];
    if (j >= nF[2 * w + c]) return false;
    const int v = cv(w, c);
    const int64_t ef = endF.at(v, j);
    if (ef == NONE || ef > t) return false;
    if (v == V - 1) return true;
    const int64_t eb = endB.at(v + 1, j);
    return eb != NONE && eb <= t;
  };
  auto run = [&](int w, int kind, int c, int64_t t) {
    const int v = cv(w, c);
    int j;
    if (kind == KIND_F) {
      j = nF[2 * w + c]++;
      endF.at(v, j) = t + 1;
    } else if (kind == KIND_B) {
      j = nB[2 * w + c]++;
      endB.at(v, j) = t + 1;
    } else {
      j = nW[2 * w + c]++;
    }
    lists[w].push_back({kind, v, j});
  };
  auto unfinished = [&]() {
    for (int i = 0; i < 2 * p; ++i)
      if (nW[i] < m) return true;
    return false;
  };
  int64_t t = 0;
  while (unfinished()) {
    for (int w = 0; w < p; ++w) {
      const int q0 = std::min(2 * p - 1 - w, m), q1 = std::min(w, m);
      if (nF[2 * w] + nF[2 * w + 1] < q0 + q1 && nB[2 * w] == 0 && nB[2 * w + 1] == 0) {  // warm-up
        if (nF[2 * w + 1] < q1 && readyF(w, 1, t)) run(w, KIND_F, 1, t);
        else if (nF[2 * w] < q0 && readyF(w, 0, t)) run(w, KIND_F, 0, t);
        continue;
      }
      if (nF[2 * w] < m || nF[2 * w + 1] < m || gchunk[w] >= 0) {  // steady 1F-1B-1W groups
        if (gchunk[w] < 0) {
          const int g = ngroups[w], lead = p - 1 - w;
          const int c = (g < lead || (g - lead) % 2 == 0) ? 1 : 0;
          gchunk[w] = c;
          gstep[w] = nF[2 * w + c] < m ? 0 : 1;
        }
        const int c = gchunk[w];
        if (gstep[w] == 0) {
          if (readyF(w, c, t)) {
            run(w, KIND_F, c, t);
            gstep[w] = 1;
          }
        } else if (gstep[w] == 1) {
          if (readyB(w, c, t)) {
            run(w, KIND_B, c, t);
            gstep[w] = 2;
          }
        } else {
          run(w, KIND_W, c, t);
          gchunk[w] = -1;
          ++ngroups[w];
        }
        continue;
      }
      bool did = false;  // drain: B first (first chunk first), W fills (second chunk first)
      for (int c = 0; c < 2 && !did; ++c)
        if (readyB(w, c, t)) {
          run(w, KIND_B, c, t);
          did = true;
        }
      for (int c = 1; c >= 0 && !did; --c)
        if (nW[2 * w + c] < nB[2 * w + c]) {
          run(w, KIND_W, c, t);
          did = true;
        }
    }
    ++t;
    if (t > 64LL * p * m + 64) throw std::runtime_error("ZB-V construction did not terminate");
  }
  return lists;
}

// ---------------------------------------------------------------- 1F1B-I
VLists build_1f1b_interleaved(int p, int m, int chunks) {
  if (p < 1 || m < 1 || chunks < 1) throw std::invalid_argument("p, m, chunks >= 1");
  if (m % p) throw std::invalid_argument("1F1B-I needs m divisible by p");
  const int total = m * chunks, cp = chunks * p;
  VLists lists(p);
  for (int w = 0; w < p; ++w) {
    int warm;
    if (chunks == 1) warm = std::min(p - 1 - w, total);
    else warm = m == p ? total : std::min(2 * (p - 1 - w) + (chunks - 1) * p, total);
    auto mb = [&](int k) { return (k / cp) * p + k % p; };
    auto& out = lists[w];
    for (int k = 0; k < warm; ++k) out.push_back({KIND_F, ((k % cp) / p) * p + w, mb(k)});
    int nb = 0;
    auto back = [&]() {
      const int v = (chunks - 1 - (nb % cp) / p) * p + w;
      out.push_back({KIND_B, v, mb(nb)});
      out.push_back({KIND_W, v, mb(nb)});
      ++nb;
    };
    for (int k = warm; k < total; ++k) {
      out.push_back({KIND_F, ((k % cp) / p) * p + w, mb(k)});
      back();
    }
    while (nb < total) back();
  }
  return lists;
}

// ---------------------------------------------------------------- simulator over virtual stages
VSimResult simulate_v(const VLists& lists, int nv, const std::vector<int>& place, const std::vector<int64_t>& TF,
                      const std::vector<int64_t>& TB, const std::vector<int64_t>& TW, int64_t Tcomm, bool fused) {
  const int nw = static_cast<int>(lists.size());
  int m = 0;
  for (auto& l : lists)
    for (auto& q : l) m = std::max(m, q.j + 1);
  EndTable end[3] = {EndTable(nv, m), EndTable(nv, m), EndTable(nv, m)};
  VSimResult r;
  r.start.assign(nw, {});
  r.end.assign(nw, {});
  for (int w = 0; w < nw; ++w) {
    r.start[w].assign(lists[w].size(), 0);
    r.end[w].assign(lists[w].size(), 0);
  }
  std::vector<size_t> pos(nw, 0);
  std::vector<int64_t> free_at(nw, 0);
  size_t total = 0, done = 0;
  for (auto& l : lists) total += l.size();
  while (done < total) {
    bool progressed = false;
    for (int w = 0; w < nw; ++w) {
      while (pos[w] < lists[w].size()) {
        const VPass& q = lists[w][pos[w]];
        int64_t t0 = free_at[w];
        bool ready = true;
        auto dep = [&](int kind, int v) {
          const int64_t e = end[kind].at(v, q.j);
          if (e == NONE) {
            ready = false;
            return;
          }
          t0 = std::max(t0, e + (place[v] != w ? Tcomm : 0));
        };
        if (q.kind == KIND_F) {
          if (q.v > 0) dep(KIND_F, q.v - 1);
        } else if (q.kind == KIND_B) {
          dep(KIND_F, q.v);
          if (q.v < nv - 1) dep(fused ? KIND_W : KIND_B, q.v + 1);
        } else {
          dep(KIND_B, q.v);
        }
        if (!ready) break;
        const int64_t d = q.kind == KIND_F ? TF[q.v] : (q.kind == KIND_B ? TB[q.v] : TW[q.v]);
        r.start[w][pos[w]] = t0;
        r.end[w][pos[w]] = t0 + d;
        end[q.kind].at(q.v, q.j) = t0 + d;
        free_at[w] = t0 + d;
        ++pos[w];
        ++done;
        progressed = true;
      }
    }
    if (!progressed) throw std::runtime_error("schedule deadlocks: a dependency can never be met");
  }
  r.cost = r.work = 0;
  for (int w = 0; w < nw; ++w) {
    if (lists[w].empty()) continue;
    r.cost = std::max(r.cost, r.end[w].back() - r.start[w].front());
    int64_t busy = 0;
    for (auto& q : lists[w]) busy += q.kind == KIND_F ? TF[q.v] : (q.kind == KIND_B ? TB[q.v] : TW[q.v]);
    r.work = std::max(r.work, busy);
  }
  r.bubble_rate = r.cost > 0 ? static_cast<double>(r.cost - r.work) / static_cast<double>(r.cost) : 0.0;
  return r;
}

std::vector<int64_t> memory_peaks_v(const VLists& lists, int64_t MB, int64_t MW) {
  std::vector<int64_t> out;
  for (auto& l : lists) {
    int64_t cur = 0, pk = 0;
    for (auto& q : l) {
      cur += q.kind == KIND_F ? MB : (q.kind == KIND_B ? MW - MB : -MW);
      pk = std::max(pk, cur);
    }
    out.push_back(pk);
  }
  return out;
}

std::vector<std::vector<int>> assign_slots_v(const VLists& lists, int nv, std::vector<int>* counts) {
  int m = 0;
  for (auto& l : lists)
    for (auto& q : l) m = std::max(m, q.j + 1);
  std::vector<std::vector<int>> freel(nv);
  std::vector<int> next(nv, 0);
  std::vector<int> of(static_cast<size_t>(nv) * m, -1);
  std::vector<std::vector<int>> slots(lists.size());
  for (size_t w = 0; w < lists.size(); ++w)
    for (auto& q : lists[w]) {
      int& s = of[static_cast<size_t>(q.v) * m + q.j];
      if (q.kind == KIND_F) {
        auto& fl = freel[q.v];
        if (!fl.empty()) {
          auto it = std::min_element(fl.begin(), fl.end());
          s = *it;
          fl.erase(it);
        } else {
          s = next[q.v]++;
        }
      } else if (q.kind == KIND_W) {
        freel[q.v].push_back(s);
      }
      slots[w].push_back(s);
    }
  if (counts) *counts = next;
  return slots;
}

// ---------------------------------------------------------------- ZB-V W right-shift
VLists zbv_shift_w(const VLists& lists, int p, int64_t TF, int64_t TB, int64_t TW, int64_t Tc, int64_t MB, int64_t MW,
                   int64_t Mlimit, bool fill) {
  const int nv = 2 * p;
  int m = 0;
  for (auto& l : lists)
    for (auto& q : l) m = std::max(m, q.j + 1);
  VLists skel(p), out(p);
  size_t nW = 0, doneW = 0;
  for (int w = 0; w < p; ++w)
    for (auto& q : lists[w]) {
      if (q.kind != KIND_W) skel[w].push_back(q);
      else ++nW;
    }
  EndTable endF(nv, m), endB(nv, m);
  std::vector<size_t> pos(p, 0);
  std::vector<int64_t> busy(p, 0), mem(p, 0);
  std::vector<std::deque<std::pair<int, int>>> pend(p);
  auto ready_at = [&](int w) -> int64_t {  // NONE = unknown
    const VPass& q = skel[w][pos[w]];
    if (q.kind == KIND_F) {
      if (q.v == 0) return 0;
      const int64_t e = endF.at(q.v - 1, q.j);
      return e == NONE ? NONE : e + (zbv_worker(p, q.v - 1) != w ? Tc : 0);
    }
    const int64_t e0 = endF.at(q.v, q.j);
    if (e0 == NONE) return NONE;
    if (q.v == nv - 1) return e0;
    const int64_t e = endB.at(q.v + 1, q.j);
    return e == NONE ? NONE : std::max(e0, e + (zbv_worker(p, q.v + 1) != w ? Tc : 0));
  };
  auto more = [&]() {
    for (int w = 0; w < p; ++w)
      if (pos[w] < skel[w].size()) return true;
    return doneW < nW;
  };
  int64_t t = 0;
  long guard = 0;
  while (more()) {
    if (++guard > 1000L * p * static_cast<long>(std::max<size_t>(1, skel[0].size())) + 1000)
      throw std::runtime_error("shift_w did not terminate");
    for (int w = 0; w < p; ++w) {
      if (busy[w] > t) continue;
      int pick = -1;  // 0 = next skeleton pass, 1 = W
      if (pos[w] < skel[w].size()) {
        const VPass& q = skel[w][pos[w]];
        const int64_t r = ready_at(w);
        if (q.kind == KIND_F && mem[w] + MB > Mlimit) {
          if (pend[w].empty()) throw std::invalid_argument("memory limit blocks F with no pending W");
          pick = 1;
        } else if (r != NONE && r <= t) {
          pick = 0;
        } else if (!pend[w].empty() && (fill || r == NONE || r - t >= TW)) {
          pick = 1;
        }
      } else if (!pend[w].empty()) {
        pick = 1;
      }
      if (pick < 0) continue;
      if (pick == 1) {
        auto vj = pend[w].front();
        pend[w].pop_front();
        out[w].push_back({KIND_W, vj.first, vj.second});
        mem[w] -= MW;
        ++doneW;
        busy[w] = t + TW;
      } else {
        const VPass q = skel[w][pos[w]++];
        out[w].push_back(q);
        if (q.kind == KIND_F) {
          mem[w] += MB;
          endF.at(q.v, q.j) = t + TF;
          busy[w] = t + TF;
        } else {
          mem[w] += MW - MB;
          endB.at(q.v, q.j) = t + TB;
          pend[w].push_back({q.v, q.j});
          busy[w] = t + TB;
        }
      }
    }
    bool have = false;
    int64_t nxt = 0;
    for (int w = 0; w < p; ++w) {
      int64_t c = NONE;
      if (busy[w] > t) {
        c = busy[w];
      } else if (pos[w] < skel[w].size()) {
        const int64_t r = ready_at(w);
        if (r != NONE && r > t) c = r;
      }
      if (c != NONE) {
        nxt = have ? std::min(nxt, c) : c;
        have = true;
      }
    }
    if (!have) {
      bool stalled = true;
      for (int w = 0; w < p; ++w)
        if (busy[w] > t || !pend[w].empty()) stalled = false;
      if (more() && stalled) throw std::runtime_error("shift_w stalled");
      nxt = t + 1;
    }
    t = nxt;
  }
  return out;
}

VLists zbv_schedule(int p, int m, int64_t TF, int64_t TB, int64_t TW, int64_t Tc, int64_t MB, int64_t MW,
                    int64_t Mlimit, int* chosen) {
  VLists base = build_zbv(p, m);
  auto pk0 = memory_peaks_v(base, MB, MW);
  const int64_t lim = Mlimit > 0 ? Mlimit : *std::max_element(pk0.begin(), pk0.end());
  struct Cand {
    int idx;
    VLists l;
  };
  std::vector<Cand> cands{{0, base}};
  for (int idx = 1; idx <= 2; ++idx) {
    try {
      cands.push_back({idx, zbv_shift_w(base, p, TF, TB, TW, Tc, MB, MW, lim, idx == 2)});
    } catch (const std::invalid_argument&) {
    }
  }
  std::vector<int> place(2 * p);
  for (int v = 0; v < 2 * p; ++v) place[v] = zbv_worker(p, v);
  std::vector<int64_t> tf(2 * p, TF), tb(2 * p, TB), tw(2 * p, TW);
  int best = -1;
  int64_t bc = 0, bp = 0;
  for (size_t i = 0; i < cands.size(); ++i) {
    auto pk = memory_peaks_v(cands[i].l, MB, MW);
    const int64_t peak = *std::max_element(pk.begin(), pk.end());
    if (cands[i].idx && peak > lim) continue;
    const VSimResult r = simulate_v(cands[i].l, 2 * p, place, tf, tb, tw, Tc, false);
    if (best < 0 || r.cost < bc || (r.cost == bc && peak < bp)) {  // candidates come in index order
      best = static_cast<int>(i);
      bc = r.cost;
      bp = peak;
    }
  }
  *chosen = cands[best].idx;
  return cands[best].l;
}

}  // namespace sched
}  // namespace zb
