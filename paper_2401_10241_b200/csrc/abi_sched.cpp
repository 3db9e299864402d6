// extern "C" entry points: errors, version, zb_schedule, zb_simulate.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "abi_util.h"
#include "zb_sched.h"
#include "zb.h"

namespace zb {
thread_local std::string g_last_error;
}

extern "C" const char* zb_last_error(void) { return zb::g_last_error.c_str(); }
extern "C" const char* zb_version(void) { return "zb-b200 0.1 (sm_100a)"; }

using namespace zb;

static zb_status_t fill(const sched::Lists& lists, const std::vector<int64_t>& tf, const std::vector<int64_t>& tb,
                        const std::vector<int64_t>& tw, int64_t Tcomm, bool fused, int64_t MB, int64_t MW, int chosen,
                        zb_pass_t* out, int32_t out_cap, zb_sim_t* sim) {
  const int p = static_cast<int>(lists.size());
  size_t n = 0;
  for (auto& o : lists) n += o.size();
  if (out != nullptr && static_cast<size_t>(out_cap) < n) return set_error(ZB_ECAP, "out_cap < 3*p*m");
  sched::SimResult r = sched::simulate(lists, tf, tb, tw, Tcomm, fused);
  std::vector<int> counts;
  auto slots = sched::assign_slots(lists, &counts);
  auto peaks = sched::memory_peaks(lists, MB, MW);
  if (out != nullptr) {
    size_t k = 0;
    for (int s = 0; s < p; ++s)
      for (size_t i = 0; i < lists[s].size(); ++i) {
        zb_pass_t& q = out[k++];
        q.stage = s;
        q.microbatch = lists[s][i].j;
        q.kind = lists[s][i].kind;
        q.slot = slots[s][i];
        q.start = r.start[s][i];
        q.end = r.end[s][i];
      }
  }
  if (sim != nullptr) {
    std::memset(sim, 0, sizeof(*sim));
    sim->cost = r.cost;
    sim->work = r.work;
    sim->bubble_rate = r.bubble_rate;
    for (int s = 0; s < p; ++s) {
      sim->peak_bytes[s] = peaks[s];
      sim->n_slots[s] = counts[s];
    }
    sim->chosen = chosen;
    sim->n_passes = static_cast<int32_t>(n);
  }
  return ZB_OK;
}

static zb_status_t schedule_impl(int32_t p, int32_t m, const std::vector<int64_t>& tf,
                                 const std::vector<int64_t>& tb, const std::vector<int64_t>& tw, int64_t T_comm,
                                 int64_t M_limit, int64_t M_B, int64_t M_W, int32_t family, zb_pass_t* out,
                                 int32_t out_cap, zb_sim_t* sim) {
  for (int s = 0; s < p; ++s)
    if (tf[s] < 0 || tb[s] < 0 || tw[s] < 0) return set_error(ZB_EINVAL, "times and memory must be >= 0");
  if (T_comm < 0 || M_B < 0 || M_W < 0) return set_error(ZB_EINVAL, "times and memory must be >= 0");
  if (out != nullptr && static_cast<int64_t>(out_cap) < 3LL * p * m) return set_error(ZB_ECAP, "out_cap < 3*p*m");
  sched::Lists lists;
  int chosen = -1;
  bool fused = false;
  switch (family) {
    case ZB_1F1B: lists = sched::build_1f1b(p, m); fused = true; break;
    case ZB_H1: lists = sched::build_zbh1(p, m); chosen = 4; break;
    case ZB_H2: lists = sched::build_zbh2(p, m); chosen = 5; break;
    case ZB_AUTO:
      if (M_limit < M_B) return set_error(ZB_ELIMIT, "AUTO needs M_limit >= M_B");
      lists = sched::auto_schedule(p, m, tf, tb, tw, T_comm, M_B, M_W, M_limit, &chosen);
      break;
    default: return set_error(ZB_EINVAL, "unknown family");
  }
  if (family != ZB_AUTO && M_limit > 0) {
    auto pk = sched::memory_peaks(lists, M_B, M_W);
    if (*std::max_element(pk.begin(), pk.end()) > M_limit)
      return set_error(ZB_ELIMIT, "family peak memory exceeds M_limit");
  }
  return fill(lists, tf, tb, tw, T_comm, fused, M_B, M_W, chosen, out, out_cap, sim);
}

extern "C" zb_status_t zb_schedule(int32_t p, int32_t m, int64_t T_F, int64_t T_B, int64_t T_W, int64_t T_comm,
                                   int64_t M_limit, int64_t M_B, int64_t M_W, int32_t family, zb_pass_t* out,
                                   int32_t out_cap, zb_sim_t* sim) {
  ZB_TRY {
    if (p < 1 || p > ZB_MAX_STAGES || m < 1) return set_error(ZB_EINVAL, "need 1 <= p <= 64 and m >= 1");
    return schedule_impl(p, m, std::vector<int64_t>(p, T_F), std::vector<int64_t>(p, T_B),
                         std::vector<int64_t>(p, T_W), T_comm, M_limit, M_B, M_W, family, out, out_cap, sim);
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_schedule_per_stage(int32_t p, int32_t m, const int64_t* T_F, const int64_t* T_B,
                                             const int64_t* T_W, int64_t T_comm, int64_t M_limit, int64_t M_B,
                                             int64_t M_W, int32_t family, zb_pass_t* out, int32_t out_cap,
                                             zb_sim_t* sim) {
  ZB_TRY {
    if (p < 1 || p > ZB_MAX_STAGES || m < 1) return set_error(ZB_EINVAL, "need 1 <= p <= 64 and m >= 1");
    if (!T_F || !T_B || !T_W) return set_error(ZB_EINVAL, "null per-stage time array");
    return schedule_impl(p, m, std::vector<int64_t>(T_F, T_F + p), std::vector<int64_t>(T_B, T_B + p),
                         std::vector<int64_t>(T_W, T_W + p), T_comm, M_limit, M_B, M_W, family, out, out_cap, sim);
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_partition(int32_t L, int32_t p, int32_t* layers) {
  ZB_TRY {
    if (p < 1 || p > ZB_MAX_STAGES || L < p || !layers) return set_error(ZB_EINVAL, "need 1 <= p <= min(L, 64)");
    if (p == 1) {
      layers[0] = L;
    } else if ((L + 2) % p == 0 && (L + 2) / p >= 2) {  // first and last stage one layer fewer
      const int mid = (L + 2) / p;
      for (int s = 0; s < p; ++s) layers[s] = (s == 0 || s == p - 1) ? mid - 1 : mid;
    } else {  // even split, remainder to the middle stages first, then stage 0, then p-1
      for (int s = 0; s < p; ++s) layers[s] = L / p;
      std::vector<int> order;
      for (int s = 1; s < p - 1; ++s) order.push_back(s);
      order.push_back(0);
      order.push_back(p - 1);
      for (int i = 0; i < L % p; ++i) layers[order[i % p]] += 1;
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_simulate(int32_t p, int32_t m, zb_pass_t* passes, int32_t n, const int64_t* T_F,
                                   const int64_t* T_B, const int64_t* T_W, int64_t T_comm, int64_t M_B, int64_t M_W,
                                   int32_t fused, zb_sim_t* sim) {
  ZB_TRY {
    if (p < 1 || p > ZB_MAX_STAGES || m < 1 || passes == nullptr || n != 3 * p * m || !T_F || !T_B || !T_W)
      return set_error(ZB_EINVAL, "zb_simulate: bad arguments");
    sched::Lists lists(p);
    for (int i = 0; i < n; ++i) {
      const zb_pass_t& q = passes[i];
      if (q.stage < 0 || q.stage >= p || q.microbatch < 0 || q.microbatch >= m || q.kind < 0 || q.kind > 2)
        return set_error(ZB_EINVAL, "zb_simulate: pass out of range");
      lists[q.stage].push_back({q.kind, q.microbatch});
    }
    for (auto& o : lists)
      if (static_cast<int>(o.size()) != 3 * m) return set_error(ZB_EINVAL, "zb_simulate: each stage needs 3m passes");
    std::vector<int64_t> tf(T_F, T_F + p), tb(T_B, T_B + p), tw(T_W, T_W + p);
    sched::SimResult r;
    try {
      r = sched::simulate(lists, tf, tb, tw, T_comm, fused != 0);
    } catch (const std::runtime_error& e) {
      return set_error(ZB_ESTATE, e.what());
    }
    // write times back in the caller's order
    std::vector<size_t> pos(p, 0);
    for (int i = 0; i < n; ++i) {
      int s = passes[i].stage;
      passes[i].start = r.start[s][pos[s]];
      passes[i].end = r.end[s][pos[s]];
      ++pos[s];
    }
    std::vector<int> counts;
    sched::assign_slots(lists, &counts);
    auto peaks = sched::memory_peaks(lists, M_B, M_W);
    if (sim) {
      std::memset(sim, 0, sizeof(*sim));
      sim->cost = r.cost;
      sim->work = r.work;
      sim->bubble_rate = r.bubble_rate;
      for (int s = 0; s < p; ++s) {
        sim->peak_bytes[s] = peaks[s];
        sim->n_slots[s] = counts[s];
      }
      sim->chosen = -1;
      sim->n_passes = n;
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_schedule_chunked(int32_t p, int32_t m, int32_t chunks, int64_t T_F, int64_t T_B,
                                           int64_t T_W, int64_t T_comm, int64_t M_limit, int64_t M_B, int64_t M_W,
                                           int32_t family, zb_pass_t* out, int32_t out_cap, zb_sim_t* sim) {
  ZB_TRY {
    if (p < 1 || m < 1 || chunks < 1 || static_cast<int64_t>(chunks) * p > ZB_MAX_STAGES)
      return set_error(ZB_EINVAL, "need p >= 1, m >= 1, 1 <= chunks * p <= 64");
    if (T_F < 0 || T_B < 0 || T_W < 0 || T_comm < 0 || M_B < 0 || M_W < 0)
      return set_error(ZB_EINVAL, "times and memory must be >= 0");
    const int64_t n = 3LL * chunks * p * m;
    if (out != nullptr && static_cast<int64_t>(out_cap) < n) return set_error(ZB_ECAP, "out_cap < 3*chunks*p*m");
    const int nv = chunks * p;
    sched::VLists lists;
    std::vector<int> place(nv);
    int chosen = -1;
    bool fused = false;
    if (family == ZB_V) {
      if (chunks != 2) return set_error(ZB_EINVAL, "ZB-V needs chunks == 2");
      lists = sched::zbv_schedule(p, m, T_F, T_B, T_W, T_comm, M_B, M_W, M_limit, &chosen);
      for (int v = 0; v < nv; ++v) place[v] = sched::zbv_worker(p, v);
      if (M_limit > 0) {
        auto pk = sched::memory_peaks_v(lists, M_B, M_W);
        if (*std::max_element(pk.begin(), pk.end()) > M_limit)
          return set_error(ZB_ELIMIT, "ZB-V needs at least its construction's peak (p stage M_B) per worker");
      }
    } else if (family == ZB_1F1B_I) {
      if (m % p) return set_error(ZB_EINVAL, "1F1B-I needs m divisible by p");
      lists = sched::build_1f1b_interleaved(p, m, chunks);
      for (int v = 0; v < nv; ++v) place[v] = v % p;
      fused = true;
    } else {
      return set_error(ZB_EINVAL, "zb_schedule_chunked: family must be ZB_V or ZB_1F1B_I");
    }
    std::vector<int64_t> tf(nv, T_F), tb(nv, T_B), tw(nv, T_W);
    const sched::VSimResult r = sched::simulate_v(lists, nv, place, tf, tb, tw, T_comm, fused);
    std::vector<int> counts;
    auto slots = sched::assign_slots_v(lists, nv, &counts);
    auto peaks = sched::memory_peaks_v(lists, M_B, M_W);
    if (out != nullptr) {
      size_t k = 0;
      for (int w = 0; w < p; ++w)
        for (size_t i = 0; i < lists[w].size(); ++i) {
          zb_pass_t& q = out[k++];
          q.stage = lists[w][i].v;
          q.microbatch = lists[w][i].j;
          q.kind = lists[w][i].kind;
          q.slot = slots[w][i];
          q.start = r.start[w][i];
          q.end = r.end[w][i];
        }
    }
    if (sim != nullptr) {
      std::memset(sim, 0, sizeof(*sim));
      sim->cost = r.cost;
      sim->work = r.work;
      sim->bubble_rate = r.bubble_rate;
      for (int w = 0; w < p; ++w) sim->peak_bytes[w] = peaks[w];
      for (int v = 0; v < nv; ++v) sim->n_slots[v] = counts[v];
      sim->chosen = chosen;
      sim->n_passes = static_cast<int32_t>(n);
    }
    return ZB_OK;
  }
  ZB_CATCH
}

// ---------------------------------------------------------------- P2P plans (host only)
#include "plan.h"
#include "zb_debug.h"

extern "C" zb_status_t zb_dbg_stage_plan(const zb_pass_t* passes, int32_t n, int32_t p, int32_t m, int32_t stage,
                                         int32_t pv_pending, int32_t amend, int32_t fused, int32_t* out_ops,
                                         int32_t cap, int32_t* n_out) {
  ZB_TRY {
    if (!passes || p < 1 || m < 1 || stage < 0 || stage >= p || !out_ops || !n_out)
      return set_error(ZB_EINVAL, "zb_dbg_stage_plan: bad arguments");
    auto ops = plan::stage_plan(passes, n, p, m, stage, pv_pending != 0, amend != 0, fused != 0);
    *n_out = static_cast<int32_t>(ops.size());
    if (static_cast<int32_t>(ops.size()) > cap) return set_error(ZB_ECAP, "plan longer than cap");
    for (size_t i = 0; i < ops.size(); ++i) {
      out_ops[4 * i] = ops[i].type;
      out_ops[4 * i + 1] = ops[i].mb;
      out_ops[4 * i + 2] = ops[i].msg;
      out_ops[4 * i + 3] = ops[i].slot;
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_dp_plan(const zb_pass_t* passes, int32_t n, int32_t p, int32_t m, int32_t stage,
                                      int32_t pv_pending, int32_t amend, int32_t fused, int32_t n_units,
                                      int32_t reorder, int32_t* out_ops, int32_t cap, int32_t* n_out) {
  ZB_TRY {
    if (!passes || p < 1 || m < 1 || stage < 0 || stage >= p || n_units < 1 || !out_ops || !n_out)
      return set_error(ZB_EINVAL, "zb_dbg_dp_plan: bad arguments");
    auto ops = plan::dp_tail(plan::stage_plan(passes, n, p, m, stage, pv_pending != 0, amend != 0, fused != 0),
                             n_units, reorder != 0);
    *n_out = static_cast<int32_t>(ops.size());
    if (static_cast<int32_t>(ops.size()) > cap) return set_error(ZB_ECAP, "plan longer than cap");
    for (size_t i = 0; i < ops.size(); ++i) {
      out_ops[4 * i] = ops[i].type;
      out_ops[4 * i + 1] = ops[i].mb;
      out_ops[4 * i + 2] = ops[i].msg;
      out_ops[4 * i + 3] = ops[i].slot;
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_speculative_counts(const zb_pass_t* passes, int32_t n, int32_t p, int32_t* out) {
  ZB_TRY {
    if (!passes || p < 1 || !out) return set_error(ZB_EINVAL, "bad arguments");
    auto v = plan::speculative_counts(passes, n, p);
    for (int s = 0; s < p; ++s) out[s] = v[s];
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_worker_plan(const zb_pass_t* passes, int32_t n, int32_t nv, int32_t m, int32_t worker,
                                          const int32_t* worker_of, int32_t fused, int32_t* out_ops, int32_t cap,
                                          int32_t* n_out) {
  ZB_TRY {
    if (!passes || nv < 1 || m < 1 || !worker_of || !out_ops || !n_out)
      return set_error(ZB_EINVAL, "zb_dbg_worker_plan: bad arguments");
    auto ops = plan::worker_plan(passes, n, nv, m, worker, worker_of, fused != 0);
    *n_out = static_cast<int32_t>(ops.size());
    if (static_cast<int32_t>(ops.size()) > cap) return set_error(ZB_ECAP, "plan longer than cap");
    for (size_t i = 0; i < ops.size(); ++i) {
      out_ops[5 * i] = ops[i].op.type;
      out_ops[5 * i + 1] = ops[i].op.mb;
      out_ops[5 * i + 2] = ops[i].op.msg;
      out_ops[5 * i + 3] = ops[i].op.slot;
      out_ops[5 * i + 4] = ops[i].chunk;
    }
    return ZB_OK;
  }
  ZB_CATCH
}
