#include "plan.h"

#include <algorithm>
#include <stdexcept>

namespace zb {
namespace plan {

namespace {
std::vector<std::vector<const zb_pass_t*>> by_stage(const zb_pass_t* passes, int n, int p) {
  std::vector<std::vector<const zb_pass_t*>> L(p);
  for (int i = 0; i < n; ++i) {
    if (passes[i].stage < 0 || passes[i].stage >= p) throw std::invalid_argument("pass stage out of range");
    L[passes[i].stage].push_back(&passes[i]);
  }
  return L;
}
int leading_f(const std::vector<const zb_pass_t*>& l) {
  int k = 0;
  while (k < static_cast<int>(l.size()) && l[k]->kind == ZB_F) ++k;
  return k;
}
}  // namespace

std::vector<int> speculative_counts(const zb_pass_t* passes, int n, int p) {
  auto L = by_stage(passes, n, p);
  std::vector<int> out(p);
  for (int s = 0; s < p; ++s) {
    int lead = leading_f(L[s]);
    out[s] = s == 0 ? lead : std::min(lead, out[s - 1]);
  }
  return out;
}

std::vector<Op> stage_plan(const zb_pass_t* passes, int n, int p, int m, int stage, bool pv_pending, bool amend,
                           bool fused) {
  auto L = by_stage(passes, n, p);
  const auto spec = speculative_counts(passes, n, p);
  const int s = stage;
  const int n_self = spec[s];
  const int n_prev = s > 0 ? spec[s - 1] : 0;
  const auto& mine = L[s];
  std::vector<int> slot_of(m, -1);
  for (auto* q : mine)
    if (q->kind == ZB_F) slot_of[q->microbatch] = q->slot;
  std::vector<Op> ops;
  bool amended = false;
  auto recv_msg = [&](int j) { return amended ? n_prev + j : j; };
  auto send_msg = [&](int j) { return amended ? n_self + j : j; };
  for (size_t i = 0; i <= mine.size(); ++i) {
    if (pv_pending && static_cast<int>(i) == n_self) {
      ops.push_back({OP_VALIDATE, -1, -1, -1});
      if (amend) {
        if (s > 0)
          for (int msg = n_self; msg < n_prev; ++msg) ops.push_back({OP_DISCARD_ACT, -1, msg, -1});
        for (int j = 0; j < n_self; ++j) {
          if (s > 0) ops.push_back({OP_RECV_ACT, j, n_prev + j, slot_of[j]});
          ops.push_back({OP_REPLAY_F, j, -1, slot_of[j]});
          if (s < p - 1) ops.push_back({OP_SEND_ACT, j, n_self + j, slot_of[j]});
        }
        amended = true;
      }
    }
    if (i == mine.size()) break;
    const zb_pass_t& q = *mine[i];
    const int j = q.microbatch;
    if (q.kind == ZB_F) {
      if (s > 0) ops.push_back({OP_RECV_ACT, j, recv_msg(j), q.slot});
      ops.push_back({OP_F, j, -1, q.slot});
      if (s < p - 1) ops.push_back({OP_SEND_ACT, j, send_msg(j), q.slot});
    } else if (q.kind == ZB_B) {
      if (s < p - 1) ops.push_back({OP_RECV_GRAD, j, j, q.slot});
      ops.push_back({OP_B, j, -1, q.slot});
      if (s > 0 && !fused) ops.push_back({OP_SEND_GRAD, j, j, q.slot});
    } else {
      ops.push_back({OP_W, j, -1, q.slot});
      if (s > 0 && fused) ops.push_back({OP_SEND_GRAD, j, j, q.slot});
    }
  }
  return ops;
}

std::vector<Op> dp_tail(const std::vector<Op>& ops, int n_units, bool reorder) {
  if (n_units < 1) throw std::invalid_argument("dp_tail: no W units");
  // the tail: W ops after the stage's last other compute / receive (1F1B's fused backward
  // interleaves its gradient sends, each of which follows its microbatch's W)
  size_t t = ops.size();
  while (t > 0 && (ops[t - 1].type == OP_W || (ops[t - 1].type == OP_SEND_GRAD && t > 1 &&
                                                ops[t - 2].type == OP_W && ops[t - 2].mb == ops[t - 1].mb)))
    --t;
  std::vector<Op> out(ops.begin(), ops.begin() + static_cast<long>(t));
  std::vector<Op> tail, sends;
  for (size_t i = t; i < ops.size(); ++i) (ops[i].type == OP_W ? tail : sends).push_back(ops[i]);
  std::vector<std::pair<int, int>> order;  // (unit, tail index) in execution order
  if (reorder)
    for (int u = 0; u < n_units; ++u)
      for (size_t i = 0; i < tail.size(); ++i) order.push_back({u, static_cast<int>(i)});
  else
    for (size_t i = 0; i < tail.size(); ++i)
      for (int u = 0; u < n_units; ++u) order.push_back({u, static_cast<int>(i)});
  std::vector<int> left_u(n_units, static_cast<int>(tail.size())), left_mb(tail.size(), n_units);
  for (const auto& [u, i] : order) {
    out.push_back({OP_WP, tail[i].mb, u, tail[i].slot});
    if (--left_u[u] == 0) out.push_back({OP_ALLREDUCE, -1, u, -1});
    if (--left_mb[i] == 0)
      for (const Op& sg : sends)
        if (sg.mb == tail[i].mb) out.push_back(sg);
  }
  if (tail.empty())  // no W after the last B (cannot happen for complete lists)
    for (int u = 0; u < n_units; ++u) out.push_back({OP_ALLREDUCE, -1, u, -1});
  out.push_back({OP_ALLREDUCE, -1, -1, -1});
  return out;
}

std::vector<WOp> worker_plan(const zb_pass_t* passes, int n, int nv, int m, int worker, const int* worker_of,
                             bool fused) {
  std::vector<std::vector<std::vector<Op>>> groups(nv);  // per virtual stage of this worker: per pass
  for (int v = 0; v < nv; ++v) {
    if (worker_of[v] != worker) continue;
    for (const Op& op : stage_plan(passes, n, nv, m, v, false, false, fused)) {
      const bool compute = op.type == OP_F || op.type == OP_B || op.type == OP_W;
      const bool recv = op.type == OP_RECV_ACT || op.type == OP_RECV_GRAD;
      // a new group starts at a receive or at a compute op unless the group is still waiting for its pass
      bool fresh = groups[v].empty();
      if (!fresh) {
        bool has_compute = false;
        for (const Op& q : groups[v].back())
          if (q.type == OP_F || q.type == OP_B || q.type == OP_W) has_compute = true;
        fresh = has_compute && (recv || compute);
      }
      if (fresh) groups[v].emplace_back();
      groups[v].back().push_back(op);
    }
  }
  std::vector<size_t> next(nv, 0);
  std::vector<WOp> out;
  for (int i = 0; i < n; ++i) {
    const zb_pass_t& q = passes[i];
    if (q.stage < 0 || q.stage >= nv) throw std::invalid_argument("pass stage out of range");
    if (worker_of[q.stage] != worker) continue;
    auto& g = groups[q.stage];
    if (next[q.stage] >= g.size()) throw std::invalid_argument("worker plan: more passes than plan groups");
    bool match = false;
    for (const Op& op : g[next[q.stage]]) {
      if ((op.type == OP_F || op.type == OP_B || op.type == OP_W) && op.type == q.kind && op.mb == q.microbatch)
        match = true;
      out.push_back({q.stage, op});
    }
    if (!match) throw std::logic_error("worker plan: pass order and plan groups disagree");
    ++next[q.stage];
  }
  return out;
}

}  // namespace plan
}  // namespace zb
