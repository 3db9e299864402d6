"""Oracle schedules, simulator and accounting (test infrastructure only).

A schedule is a list, per stage s in [0, p), of passes (kind, j) with kind in
{"F", "B", "W"} and microbatch j in [0, m): "the ordering of the passes"
(App. F).  Times are Python ints (exact), so costs compare
exactly (SPEC S:81 design decision; reading R-int).

Followed passages
  * 1F1B (Fig. 2 text), ZB-H1, ZB-H2: the generic
    builder of SURVEY.md Appendix A (warm-up count w_s, W deferral d_s,
    steady order), which reproduces Table 2 exactly and Table 4's
    handcrafted columns to all printed decimals.
  * Simulator: App. F constraints (4)-(6) as ASAP execution
    semantics; span = E(last) - S(first); cost = max span; bubble rate
    (cost - m(T_F+T_B+T_W)) / cost.  1F1B's backward is fused: the
    upstream B waits for the downstream W.
  * Memory: order-based prefix sums of App. F's Delta-M: F +M_B,
    B +(M_W - M_B), W -M_W (constraint (7)).
  * AUTO: the heuristic of section 3.1 in the reading of SURVEY.md
    Appendix B, grid search over its two binary hyper-parameters (P:136,
    P:139), plus the handcrafted candidates that fit M_limit.
"""
from __future__ import annotations

from collections import deque
from typing import Dict, List, Optional, Sequence, Tuple

Pass = Tuple[str, int]
Lists = List[List[Pass]]
INF = float("inf")

FAMILIES = ("1f1b", "zbh1", "zbh2", "auto")


def _per_stage(x, p: int) -> List[int]:
    if isinstance(x, (list, tuple)):
        assert len(x) == p
        return list(x)
    return [x] * p


# --------------------------------------------------------------------------
# handcrafted builders (SURVEY Appendix A reading of P:57)
# --------------------------------------------------------------------------

def build_generic(p: int, m: int, warmup: Sequence[int], defer: Sequence[int], order: str) -> Lists:
    """Per stage: w_s warm-up Fs, then the steady loop in `order` ("FB": F then
    B, "BF": B then F) with W(nw) emitted once more than d_s Bs are
    outstanding, then the remaining Ws."""
    lists: Lists = []
    for s in range(p):
        out: List[Pass] = []
        w = min(warmup[s], m)
        out += [("F", j) for j in range(w)]
        nf, nb, nw = w, 0, 0
        while nb < m:
            if order == "FB":
                if nf < m:
                    out.append(("F", nf)); nf += 1
                out.append(("B", nb)); nb += 1
                if nb - nw > defer[s]:
                    out.append(("W", nw)); nw += 1
            else:
                out.append(("B", nb)); nb += 1
                if nb - nw > defer[s]:
                    out.append(("W", nw)); nw += 1
                if nf < m:
                    out.append(("F", nf)); nf += 1
        while nw < m:
            out.append(("W", nw)); nw += 1
        lists.append(out)
    return lists


def build_1f1b(p: int, m: int) -> Lists:
    """1F1B: stage s warms up with p-1-s Fs (one more than the next
    stage), then 1F-1B; W immediately follows its B (fused backward)."""
    return build_generic(p, m, [p - 1 - s for s in range(p)], [0] * p, "FB")


def build_zbh1(p: int, m: int) -> Lists:
    """ZB-H1: 1F1B order with stage s delaying its Ws by s, so all
    stages keep the same number of in-flight microbatches."""
    return build_generic(p, m, [p - 1 - s for s in range(p)], list(range(p)), "FB")


def build_zbh2(p: int, m: int) -> Lists:
    """ZB-H2: 2(p-s)-1 warm-up Fs fill the bubble before the first B;
    W reordered (deferred by 2s) so the layout becomes a parallelogram."""
    return build_generic(p, m, [2 * (p - s) - 1 for s in range(p)], [2 * s for s in range(p)], "BF")


# --------------------------------------------------------------------------
# simulator (App. F constraints (4)-(6) as ASAP execution semantics)
# --------------------------------------------------------------------------

def _deps(kind: str, s: int, j: int, p: int, fused: bool):
    if kind == "F":
        return [("F", s - 1, j, True)] if s > 0 else []
    if kind == "B":
        d = [("F", s, j, False)]
        if s < p - 1:
            d.append(("W" if fused else "B", s + 1, j, True))
        return d
    return [("B", s, j, False)]


def simulate(lists: Lists, TF, TB, TW, Tcomm=0, fused: bool = False) -> Dict:
    """ASAP timing of per-stage orders.  A pass starts at the max of the end of
    its stage's previous pass and each dependency's end (+T_comm if the edge
    crosses stages).  Returns start/end per (s, kind, j), per-stage span and
    busy time, cost = max span and the bubble rate of P:286."""
    p = len(lists)
    TF, TB, TW = _per_stage(TF, p), _per_stage(TB, p), _per_stage(TW, p)
    dur = {"F": TF, "B": TB, "W": TW}
    start: Dict[Tuple[str, int, int], int] = {}
    end: Dict[Tuple[str, int, int], int] = {}
    pos = [0] * p
    free = [0] * p
    total = sum(len(x) for x in lists)
    done = 0
    while done < total:
        progressed = False
        for s in range(p):
            while pos[s] < len(lists[s]):
                kind, j = lists[s][pos[s]]
                deps = _deps(kind, s, j, p, fused)
                if any((k, ss, jj) not in end for k, ss, jj, _ in deps):
                    break
                t0 = free[s]
                for k, ss, jj, comm in deps:
                    t0 = max(t0, end[(k, ss, jj)] + (Tcomm if comm else 0))
                start[(kind, s, j)] = t0
                end[(kind, s, j)] = t0 + dur[kind][s]
                free[s] = t0 + dur[kind][s]
                pos[s] += 1
                done += 1
                progressed = True
        if not progressed:
            raise ValueError("schedule deadlocks: a dependency can never be met")
    spans, busy = [], []
    for s in range(p):
        if not lists[s]:
            spans.append(0); busy.append(0); continue
        k0, j0 = lists[s][0]
        k1, j1 = lists[s][-1]
        spans.append(end[(k1, s, j1)] - start[(k0, s, j0)])
        busy.append(sum(dur[k][s] for k, _ in lists[s]))
    cost = max(spans)
    m = max((j for k, j in lists[0]), default=-1) + 1 if lists and lists[0] else 0
    work = max(m * (TF[s] + TB[s] + TW[s]) for s in range(p))
    rate = (cost - work) / cost if cost else 0.0
    return dict(start=start, end=end, spans=spans, busy=busy, cost=cost, bubble_rate=rate, work=work)


def bubble_rate(cost, m: int, TF, TB, TW) -> float:
    """(cost - m(T_F+T_B+T_W)) / cost."""
    return (cost - m * (TF + TB + TW)) / cost


# --------------------------------------------------------------------------
# memory and slots (App. F Delta-M, constraint (7))
# --------------------------------------------------------------------------

def memory_trace(order: Sequence[Pass], MB: int, MW: int) -> List[int]:
    cur, tr = 0, []
    for k, _ in order:
        cur += MB if k == "F" else (MW - MB if k == "B" else -MW)
        tr.append(cur)
    return tr


def memory_peaks(lists: Lists, MB: int, MW: int) -> List[int]:
    return [max([0] + memory_trace(o, MB, MW)) for o in lists]


def assign_slots(lists: Lists) -> Tuple[List[Dict[int, int]], List[int]]:
    """Stash slot per (stage, microbatch): the lowest free index at F, released
    at W.  Returns per-stage {j: slot} and slot counts."""
    maps, counts = [], []
    for o in lists:
        free: List[int] = []
        nxt = 0
        mp: Dict[int, int] = {}
        for k, j in o:
            if k == "F":
                if free:
                    free.sort()
                    sl = free.pop(0)
                else:
                    sl = nxt; nxt += 1
                mp[j] = sl
            elif k == "W":
                free.append(mp[j])
        maps.append(mp)
        counts.append(nxt)
    return maps, counts


def validate_schedule(lists: Lists, m: int) -> List[str]:
    """Violations (data, not errors): completeness, per-stage
    F < B < W order, and deadlock-freedom of the cross-stage dependencies."""
    out: List[str] = []
    for s, o in enumerate(lists):
        seen = {}
        for i, (k, j) in enumerate(o):
            if (k, j) in seen:
                out.append(f"stage {s}: duplicate {k}{j}")
            seen[(k, j)] = i
        for j in range(m):
            for k in "FBW":
                if (k, j) not in seen:
                    out.append(f"stage {s}: missing {k}{j}")
            if all((k, j) in seen for k in "FBW"):
                if not seen[("F", j)] < seen[("B", j)] < seen[("W", j)]:
                    out.append(f"stage {s}: order of F/B/W of microbatch {j}")
    if not out:
        try:
            simulate(lists, 1, 1, 1, 0)
        except ValueError:
            out.append("cross-stage dependency cycle")
    return out


# --------------------------------------------------------------------------
# AUTO: heuristic of section 3.1 (SURVEY Appendix B reading) + grid search
# --------------------------------------------------------------------------

_NA = "na"


def heuristic(p: int, m: int, TF: int, TB: int, TW: int, Tcomm: int, MB: int, MW: int, Mlimit: int,
              fill_warmup: bool, skip_lead: bool) -> Lists:
    """Global-clock list scheduler following P:132-142:
      * warm-up: as many Fs as memory allows; an F that may delay the first B
        is taken only when fill_warmup (first binary hyper-parameter);
      * steady: 1F-1B alternation; a W is inserted when the gap before the
        next F/B input is >= T_W, or when the gap would make this stage's
        cumulative bubble the largest of all stages, or when the memory
        limit blocks F;
      * stage s keeps at least one more F than stage s+1; when the lead
        exceeds one, skip_lead may skip an F (second hyper-parameter);
      * remaining Ws drain at the end.
    Readings (DESIGN.md R-auto): integer time, stages visited in ascending
    index per tick, W in FIFO order, unknown arrivals assumed >= T_B+T_comm
    away.  Returns per-stage pass lists (the order is the product)."""
    if Mlimit < MB:
        raise ValueError("M_limit below M_B: no F can ever run")
    # per-stage times (the profiled T_F / T_B / T_W of each stage are what the
    # scheduler is fed; DESIGN.md R-auto-stage): scalars mean the same time on every stage
    TF, TB, TW = _per_stage(TF, p), _per_stage(TB, p), _per_stage(TW, p)
    nF, nB, nW = [0] * p, [0] * p, [0] * p
    pend = [deque() for _ in range(p)]
    mem, bub, busy = [0] * p, [0] * p, [0] * p
    started, last = [False] * p, [None] * p
    endF: Dict[Tuple[int, int], int] = {}
    endB: Dict[Tuple[int, int], int] = {}
    lists: Lists = [[] for _ in range(p)]

    def arrivals(s):
        if nF[s] >= m:
            aF = _NA
        elif s == 0:
            aF = 0
        elif (s - 1, nF[s]) in endF:
            aF = endF[(s - 1, nF[s])] + Tcomm
        else:
            aF = None
        if nB[s] >= nF[s]:
            aB = _NA
        elif s == p - 1:
            aB = endF[(s, nB[s])]
        elif (s + 1, nB[s]) in endB:
            aB = endB[(s + 1, nB[s])] + Tcomm
        else:
            aB = None
        return aF, aB

    known = lambda x: x is not None and x != _NA
    t = 0
    guard = 0
    while any(nW[s] < m for s in range(p)):
        guard += 1
        if guard > 100 * p * m + 1000:
            raise RuntimeError("heuristic did not terminate")
        for s in range(p):
            if nW[s] >= m or busy[s] > t:
                continue
            aF, aB = arrivals(s)
            memOK = nF[s] < m and mem[s] + MB <= Mlimit
            if (skip_lead and s < p - 1 and nF[s] < m and nF[s] - nF[s + 1] > 1 and nB[s] > 0
                    and known(aB) and aB <= t):
                memOK = False
            Fready = memOK and known(aF) and aF <= t
            Bready = known(aB) and aB <= t
            pick = None
            if nB[s] == 0:
                if Bready:
                    pick = "B"
                elif Fready:
                    delays = (known(aB) and aB < t + TF[s]) or (aB is None and TB[s] + Tcomm < TF[s])
                    if not delays or fill_warmup:
                        pick = "F"
            else:
                if Bready and Fready:
                    pick = "F" if last[s] == "B" else "B"
                elif Bready:
                    pick = "B"
                elif Fready:
                    pick = "F"
            if pick is None and pend[s]:
                cands = []
                if nF[s] < m and mem[s] + MB <= Mlimit and known(aF):
                    cands.append(aF)
                if known(aB):
                    cands.append(aB)
                r = min(cands) if cands else INF
                others = max((bub[x] for x in range(p) if x != s), default=0)
                if (nF[s] < m and mem[s] + MB > Mlimit and not Bready) or r - t >= TW[s] or \
                        (nF[s] == m and nB[s] == m):
                    pick = "W"
                elif r > t and bub[s] + (r - t) > others:
                    pick = "W"
            if pick is None:
                continue
            if started[s]:
                bub[s] += t - busy[s]
            started[s] = True
            if pick == "F":
                j = nF[s]; nF[s] += 1
                endF[(s, j)] = t + TF[s]
                mem[s] += MB
                busy[s] = t + TF[s]
            elif pick == "B":
                j = nB[s]; nB[s] += 1
                endB[(s, j)] = t + TB[s]
                mem[s] += MW - MB
                pend[s].append(j)
                busy[s] = t + TB[s]
            else:
                j = pend[s].popleft(); nW[s] += 1
                mem[s] -= MW
                busy[s] = t + TW[s]
            last[s] = pick
            lists[s].append((pick, j))
        nxt = INF
        for s in range(p):
            if nW[s] >= m:
                continue
            if busy[s] > t:
                nxt = min(nxt, busy[s])
            aF, aB = arrivals(s)
            for a in (aF, aB):
                if known(a) and a > t:
                    nxt = min(nxt, a)
        if nxt == INF:
            if any(nW[s] < m for s in range(p)):
                raise RuntimeError("heuristic stalled")
            break
        t = nxt
    return lists


def auto_schedule(p: int, m: int, TF: int, TB: int, TW: int, Tcomm: int, MB: int, MW: int, Mlimit: int):
    """Grid search over (fill_warmup, skip_lead) in {0,1}^2, plus
    ZB-H1 / ZB-H2 when their peak fits M_limit.  Candidate index
    = 2*fill_warmup + skip_lead for the heuristic, 4 = ZB-H1, 5 = ZB-H2; the
    minimum (cost, max peak, index) is chosen.  Returns (lists, index, sim)."""
    cands = []
    for fill in (0, 1):
        for skip in (0, 1):
            cands.append((2 * fill + skip, heuristic(p, m, TF, TB, TW, Tcomm, MB, MW, Mlimit, bool(fill), bool(skip))))
    for idx, builder in ((4, build_zbh1), (5, build_zbh2)):
        l = builder(p, m)
        if max(memory_peaks(l, MB, MW)) <= Mlimit:
            cands.append((idx, l))
    best = None
    for idx, l in cands:
        sim = simulate(l, TF, TB, TW, Tcomm)
        key = (sim["cost"], max(memory_peaks(l, MB, MW)), idx)
        if best is None or key < best[0]:
            best = (key, idx, l, sim)
    return best[2], best[1], best[3]


def schedule(family: str, p: int, m: int, TF: int, TB: int, TW: int, Tcomm: int = 0,
             MB: int = 1, MW: int = 1, Mlimit: Optional[int] = None):
    """Oracle side of zb_schedule(): (lists, slot maps, slot counts, sim, chosen)."""
    if family == "1f1b":
        lists, chosen, fused = build_1f1b(p, m), -1, True
    elif family == "zbh1":
        lists, chosen, fused = build_zbh1(p, m), 4, False
    elif family == "zbh2":
        lists, chosen, fused = build_zbh2(p, m), 5, False
    elif family == "auto":
        lim = Mlimit if Mlimit is not None else p * MB
        lists, chosen, _ = auto_schedule(p, m, TF, TB, TW, Tcomm, MB, MW, lim)
        fused = False
    else:
        raise ValueError(family)
    if Mlimit is not None and family != "auto" and max(memory_peaks(lists, MB, MW)) > Mlimit:
        raise ValueError("family peak exceeds M_limit")
    sim = simulate(lists, TF, TB, TW, Tcomm, fused=fused)
    maps, counts = assign_slots(lists)
    return lists, maps, counts, sim, chosen


# --------------------------------------------------------------------------
# closed forms
# --------------------------------------------------------------------------

def table2_bubble(family: str, p: int, TF, TB, TW):
    """Table 2 bubble sizes."""
    return {"1f1b": (p - 1) * (TF + TB + TW), "zbh1": (p - 1) * (TF + TB - TW),
            "zbh2": (p - 1) * (TF + TB - 2 * TW)}[family]


def table2_peak(family: str, p: int, MB, MW):
    """Table 2 peak activation memory, valid when M_W <= M_B."""
    return {"1f1b": p * MB, "zbh1": p * MB, "zbh2": (2 * p - 1) * MB}[family]


def stage_peak(family: str, p: int, i: int, MB, MW):
    """Per-worker memory of P:109 (i is 1-indexed): ZB-H1 (p-i+1)M_B+(i-1)M_W,
    ZB-H2 (2p-2i+1)M_B+(2i-2)M_W; 1F1B (p-i+1)M_B."""
    return {"1f1b": (p - i + 1) * MB, "zbh1": (p - i + 1) * MB + (i - 1) * MW,
            "zbh2": (2 * p - 2 * i + 1) * MB + (2 * i - 2) * MW}[family]


def small_m_cost(family: str, p: int, m: int, TF, TB, TW):
    """App. "small m": 1F1B (m+p-1)(T_F+T_B+T_W); ZB (m+p-1)(T_F+T_B)+T_W."""
    if family == "1f1b":
        return (m + p - 1) * (TF + TB + TW)
    return (m + p - 1) * (TF + TB) + TW


def appendix_b(p: int, TF, TB, Tcomm, MB=1):
    """App. B formulas (1)-(2): k* = floor(((p-1)(T_B+2T_comm)+pT_F)/T_F),
    beta(k) = (p-1)(T_B+2T_comm)+(p-k)T_F, plateau k* M_B, zero-bubble memory
    floor(((p-1)(T_B+2T_comm)+(2p-1)T_F)/T_F) M_B."""
    num = (p - 1) * (TB + 2 * Tcomm)
    k_star = (num + p * TF) // TF
    beta = lambda k: num + (p - k) * TF
    return dict(k_star=k_star, beta_min=beta(k_star), m_plateau=k_star * MB,
                m_zero=((num + (2 * p - 1) * TF) // TF) * MB, beta=beta)


def table1_flops(s: int, b: int, h: int, kind: str) -> int:
    """Table 1: F sbh(24h+4s), B sbh(24h+8s), W sbh(24h)."""
    return {"F": s * b * h * (24 * h + 4 * s), "B": s * b * h * (24 * h + 8 * s), "W": s * b * h * 24 * h}[kind]


def table1_memory(s: int, b: int, h: int, a: int, kind: str) -> int:
    """Table 1 activation memory: B sb(34h+5as), W 32sbh (F 0)."""
    return {"F": 0, "B": s * b * (34 * h + 5 * a * s), "W": 32 * s * b * h}[kind]
