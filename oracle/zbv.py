"""Oracle schedules with several model chunks per worker — ZB-V (PAPER.md
section 6) and interleaved 1F1B (1F1B-I) — test
infrastructure only.

ZB-V splits the model into 2p chunks ("virtual stages" v in [0, 2p)) and
places them in a V: worker w holds v = w (its first chunk, c = 0) and
v = 2p-1-w (its second chunk, c = 1), "layers 1-2 and layers 15-16 on worker
1" for 16 layers and 4 stages.  The forward of a microbatch runs
v = 0 .. 2p-1 (down the workers, then back up); its backward runs
v = 2p-1 .. 0.  A pass is (kind, v, j); a schedule is one list per worker in
execution order.  Times and memory are PER CHUNK here: one chunk pass takes
T_F / T_B / T_W, retains M_B / M_W (a chunk holds half a stage's layers, so
these are half the stage figures of section 2).

Followed passages
  * Placement and dependencies: P:318-320 ("sequentially allocating model
    chunks to workers ... then reversing the order"; "both the forward pass
    and backward pass for each microbatch originate from the same worker").
  * Three phases: warm-up of 2p-i Fs of the first chunk and i-1
    of the second on worker i (1-indexed); steady 1F-1B-1W groups, "p-i
    groups for the second chunk" first, then alternating one group of the
    second and one of the first chunk until the worker's Fs are issued;
    drain with "B being prioritized and W filling the bubbles".
  * W right-shift within the memory limit: "we can straightforwardly
    shift all W to the right, within the memory constraint ... to fill the
    bubbles in the schedule's tail".
Readings (DESIGN.md R-zbv; Fig. 6 itself is missing from PAPER.md):
  * the phases are executed as a unit-time (T_F = T_B = T_W = 1, T_comm = 0)
    list construction; each worker waits (idles) until its next pass is
    ready; in warm-up a ready second-chunk F is taken before a first-chunk F;
    the alternation after the p-i leading groups starts with the second
    chunk; a group whose chunk has no F left is [B, W]; in the drain a ready
    first-chunk B goes before a second-chunk B, and Ws drain oldest first,
    second chunk first.  The resulting order lists ARE the schedule; for
    other times they are executed ASAP by `simulate_v`.
  * W right-shift: Ws are removed from each worker's list and re-inserted by
    an ASAP execution with the given times: a pending W (FIFO) runs when the
    worker's next F / B is not ready (rule "fill": always; rule "gap": only
    if the wait is >= T_W) or when the next F would exceed M_limit.  The
    original list is a candidate too, so the simulated cost never increases
    (SPEC S:238); the minimum (cost, peak, index) wins.
"""
from __future__ import annotations

from collections import deque
from typing import Dict, List, Sequence, Tuple

VPass = Tuple[str, int, int]          # (kind, virtual stage v, microbatch j)
VLists = List[List[VPass]]            # per worker
INF = float("inf")


def worker_of(p: int, v: int) -> int:
    """V placement: v < p on worker v, else on worker 2p-1-v."""
    return v if v < p else 2 * p - 1 - v


def chunk_v(p: int, w: int, c: int) -> int:
    """Virtual stage of worker w's chunk c (0 = first, 1 = second)."""
    return w if c == 0 else 2 * p - 1 - w


# --------------------------------------------------------------------------
# construction (P:322 under unit times)
# --------------------------------------------------------------------------

def build_zbv(p: int, m: int) -> VLists:
    if p < 1 or m < 1:
        raise ValueError("p, m >= 1")
    V = 2 * p
    endF: Dict[Tuple[int, int], int] = {}
    endB: Dict[Tuple[int, int], int] = {}
    nF = [[0, 0] for _ in range(p)]
    nB = [[0, 0] for _ in range(p)]
    nW = [[0, 0] for _ in range(p)]
    lists: VLists = [[] for _ in range(p)]
    group: List = [None] * p      # [chunk, step] of the worker's current steady group
    ngroups = [0] * p

    def readyF(w, c, t):
        j = nF[w][c]
        if j >= m:
            return False
        v = chunk_v(p, w, c)
        return v == 0 or endF.get((v - 1, j), INF) <= t

    def readyB(w, c, t):
        j = nB[w][c]
        if j >= nF[w][c]:
            return False
        v = chunk_v(p, w, c)
        if endF.get((v, j), INF) > t:
            return False
        return v == V - 1 or endB.get((v + 1, j), INF) <= t

    def run(w, kind, c, t):
        v = chunk_v(p, w, c)
        if kind == "F":
            j = nF[w][c]; nF[w][c] += 1; endF[(v, j)] = t + 1
        elif kind == "B":
            j = nB[w][c]; nB[w][c] += 1; endB[(v, j)] = t + 1
        else:
            j = nW[w][c]; nW[w][c] += 1
        lists[w].append((kind, v, j))

    t = 0
    while any(nW[w][c] < m for w in range(p) for c in (0, 1)):
        for w in range(p):
            q0, q1 = min(2 * p - 1 - w, m), min(w, m)     # warm-up: 2p-i first-chunk, i-1 second-chunk Fs
            if nF[w][0] + nF[w][1] < q0 + q1 and nB[w] == [0, 0]:
                if nF[w][1] < q1 and readyF(w, 1, t):
                    run(w, "F", 1, t)
                elif nF[w][0] < q0 and readyF(w, 0, t):
                    run(w, "F", 0, t)
                continue
            if nF[w][0] < m or nF[w][1] < m or group[w] is not None:   # steady 1F-1B-1W groups
                if group[w] is None:
                    g, lead = ngroups[w], p - 1 - w
                    c = 1 if g < lead or (g - lead) % 2 == 0 else 0
                    group[w] = [c, 0 if nF[w][c] < m else 1]
                c, step = group[w]
                if step == 0:
                    if readyF(w, c, t):
                        run(w, "F", c, t); group[w][1] = 1
                elif step == 1:
                    if readyB(w, c, t):
                        run(w, "B", c, t); group[w][1] = 2
                else:
                    run(w, "W", c, t); group[w] = None; ngroups[w] += 1
                continue
            for c in (0, 1):                                  # drain: B first, W fills
                if readyB(w, c, t):
                    run(w, "B", c, t)
                    break
            else:
                for c in (1, 0):
                    if nW[w][c] < nB[w][c]:
                        run(w, "W", c, t)
                        break
        t += 1
        if t > 64 * p * m + 64:
            raise RuntimeError("ZB-V construction did not terminate")
    return lists


# --------------------------------------------------------------------------
# interleaved 1F1B (1F1B-I)
# --------------------------------------------------------------------------

def build_1f1b_interleaved(p: int, m: int, chunks: int) -> VLists:
    """1F1B-I, the baseline of Table 4 (Narayanan et al. 2021): the
    model is cut into chunks * p pieces "cyclically taken by each stage"
    (S:163): v on worker v mod p.  Reading (R-1f1bi, the scheme of
    the cited Megatron-LM implementation): microbatches advance in groups of
    p; the k-th forward of a worker runs chunk (k mod chunks*p) // p on
    microbatch (k // (chunks*p)) * p + k mod p; the k-th backward runs chunk
    chunks-1 - (k mod chunks*p) // p on the same microbatch formula; worker w
    warms up with 2(p-1-w) + (chunks-1) p forwards (all of them when m = p;
    p-1-w when chunks = 1, plain 1F1B),
    then alternates 1F-1B, then drains; each W directly follows its B (the
    fused backward of 1F1B, simulated with fused=True).  m must be a
    multiple of p."""
    if p < 1 or m < 1 or chunks < 1:
        raise ValueError("p, m, chunks >= 1")
    if m % p:
        raise ValueError("1F1B-I needs m divisible by p")
    total = m * chunks
    lists: VLists = []
    for w in range(p):
        if chunks == 1:                       # plain 1F1B
            warm = min(p - 1 - w, total)
        else:
            warm = total if m == p else min(2 * (p - 1 - w) + (chunks - 1) * p, total)

        def mb(k):
            return (k // (chunks * p)) * p + k % p

        out: List[VPass] = [("F", ((k % (chunks * p)) // p) * p + w, mb(k)) for k in range(warm)]
        nb = 0

        def back():
            v = (chunks - 1 - (nb % (chunks * p)) // p) * p + w
            return [("B", v, mb(nb)), ("W", v, mb(nb))]

        for k in range(warm, total):
            out.append(("F", ((k % (chunks * p)) // p) * p + w, mb(k)))
            out += back(); nb += 1
        while nb < total:
            out += back(); nb += 1
        lists.append(out)
    return lists


# --------------------------------------------------------------------------
# simulator over virtual stages (App. F (4)-(6) with a placement)
# --------------------------------------------------------------------------

def _vdeps(kind: str, v: int, j: int, nv: int, fused: bool):
    if kind == "F":
        return [("F", v - 1, j)] if v > 0 else []
    if kind == "B":
        d = [("F", v, j)]
        if v < nv - 1:
            d.append(("W" if fused else "B", v + 1, j))
        return d
    return [("B", v, j)]


def simulate_v(lists: VLists, nv: int, place, TF, TB, TW, Tcomm=0, fused: bool = False) -> Dict:
    """ASAP timing of per-worker lists of (kind, v, j): a pass starts at the
    max of its worker's previous end and each dependency's end, + T_comm when
    the dependency ran on another worker.  place(v) -> worker.  Per-chunk
    times (scalars).  cost = max span; work = busy time of the busiest
    worker; bubble rate (cost - work) / cost."""
    dur = {"F": TF, "B": TB, "W": TW}
    start: Dict[Tuple[str, int, int], int] = {}
    end: Dict[Tuple[str, int, int], int] = {}
    nw = len(lists)
    pos, free = [0] * nw, [0] * nw
    total, done = sum(len(x) for x in lists), 0
    while done < total:
        progressed = False
        for w in range(nw):
            while pos[w] < len(lists[w]):
                kind, v, j = lists[w][pos[w]]
                deps = _vdeps(kind, v, j, nv, fused)
                if any(d not in end for d in deps):
                    break
                t0 = free[w]
                for d in deps:
                    t0 = max(t0, end[d] + (Tcomm if place(d[1]) != w else 0))
                start[(kind, v, j)] = t0
                end[(kind, v, j)] = free[w] = t0 + dur[kind]
                pos[w] += 1
                done += 1
                progressed = True
        if not progressed:
            raise ValueError("schedule deadlocks: a dependency can never be met")
    spans = [end[l[-1]] - start[l[0]] if l else 0 for l in lists]
    busy = [sum(dur[k] for k, _, _ in l) for l in lists]
    cost, work = max(spans), max(busy)
    return dict(start=start, end=end, spans=spans, busy=busy, cost=cost, work=work,
                bubble_rate=(cost - work) / cost if cost else 0.0)


def memory_peaks_v(lists: VLists, MB: int, MW: int) -> List[int]:
    """Per-worker order-based Delta-M prefix peak (constraint (7))."""
    out = []
    for l in lists:
        cur = pk = 0
        for k, _, _ in l:
            cur += MB if k == "F" else (MW - MB if k == "B" else -MW)
            pk = max(pk, cur)
        out.append(pk)
    return out


def assign_slots_v(lists: VLists, nv: int) -> Tuple[Dict[Tuple[int, int], int], List[int]]:
    """Stash slot per (v, j): lowest free slot of context v at F, freed at W."""
    free = [[] for _ in range(nv)]
    nxt = [0] * nv
    mp: Dict[Tuple[int, int], int] = {}
    for l in lists:
        for k, v, j in l:
            if k == "F":
                if free[v]:
                    free[v].sort()
                    mp[(v, j)] = free[v].pop(0)
                else:
                    mp[(v, j)] = nxt[v]; nxt[v] += 1
            elif k == "W":
                free[v].append(mp[(v, j)])
    return mp, nxt


def validate_v(lists: VLists, p: int, m: int) -> List[str]:
    """Completeness, placement, per-(v, j) F < B < W, deadlock freedom."""
    out: List[str] = []
    nv = 2 * p
    seen = {}
    for w, l in enumerate(lists):
        for i, (k, v, j) in enumerate(l):
            if worker_of(p, v) != w:
                out.append(f"worker {w}: {k}{j} of chunk v={v} misplaced")
            if (k, v, j) in seen:
                out.append(f"duplicate {k} v={v} j={j}")
            seen[(k, v, j)] = (w, i)
    for v in range(nv):
        for j in range(m):
            if not all((k, v, j) in seen for k in "FBW"):
                out.append(f"missing pass of v={v} j={j}")
            elif not seen[("F", v, j)][1] < seen[("B", v, j)][1] < seen[("W", v, j)][1]:
                out.append(f"order of F/B/W of v={v} j={j}")
    if not out:
        try:
            simulate_v(lists, nv, lambda v: worker_of(p, v), 1, 1, 1, 0)
        except ValueError:
            out.append("cross-worker dependency cycle")
    return out


# --------------------------------------------------------------------------
# W right-shift within the memory limit
# --------------------------------------------------------------------------

def shift_w(lists: VLists, p: int, TF: int, TB: int, TW: int, Tcomm: int, MB: int, MW: int, Mlimit: int,
            rule: str) -> VLists:
    """Re-insert every worker's Ws (FIFO) into its F/B skeleton by an ASAP
    execution with the given integer times: a W runs when the next F/B is
    not ready (rule "fill"; rule "gap": only if it would wait >= T_W) or
    when the next F would exceed M_limit; the rest drain at the end.
    Raises ValueError if the memory limit cannot be met."""
    nv = 2 * p
    skel = [[x for x in l if x[0] != "W"] for l in lists]
    dur = {"F": TF, "B": TB, "W": TW}
    endF: Dict[Tuple[int, int], int] = {}
    endB: Dict[Tuple[int, int], int] = {}
    pos, busy, mem = [0] * p, [0] * p, [0] * p
    pend = [deque() for _ in range(p)]
    out: VLists = [[] for _ in range(p)]
    nW = sum(1 for l in lists for x in l if x[0] == "W")
    doneW = 0

    def ready_at(w):
        k, v, j = skel[w][pos[w]]
        if k == "F":
            if v == 0:
                return 0
            e = endF.get((v - 1, j))
            return None if e is None else e + (Tcomm if worker_of(p, v - 1) != w else 0)
        e0 = endF.get((v, j))
        if e0 is None:
            return None
        if v == nv - 1:
            return e0
        e = endB.get((v + 1, j))
        return None if e is None else max(e0, e + (Tcomm if worker_of(p, v + 1) != w else 0))

    t = 0
    guard = 0
    while any(pos[w] < len(skel[w]) for w in range(p)) or doneW < nW:
        guard += 1
        if guard > 1000 * p * max(1, len(skel[0])) + 1000:
            raise RuntimeError("shift_w did not terminate")
        for w in range(p):
            if busy[w] > t:
                continue
            pick = None
            if pos[w] < len(skel[w]):
                k, v, j = skel[w][pos[w]]
                r = ready_at(w)
                mem_block = k == "F" and mem[w] + MB > Mlimit
                if mem_block:
                    if not pend[w]:
                        raise ValueError("memory limit blocks F with no pending W")
                    pick = "W"
                elif r is not None and r <= t:
                    pick = "X"
                elif pend[w] and (rule == "fill" or r is None or r - t >= TW):
                    pick = "W"
            elif pend[w]:
                pick = "W"
            if pick is None:
                continue
            if pick == "W":
                v, j = pend[w].popleft()
                out[w].append(("W", v, j)); mem[w] -= MW; doneW += 1
                busy[w] = t + TW
            else:
                k, v, j = skel[w][pos[w]]; pos[w] += 1
                out[w].append((k, v, j))
                if k == "F":
                    mem[w] += MB; endF[(v, j)] = t + TF
                else:
                    mem[w] += MW - MB; endB[(v, j)] = t + TB; pend[w].append((v, j))
                busy[w] = t + dur[k]
        nxt = INF
        for w in range(p):
            if busy[w] > t:
                nxt = min(nxt, busy[w])
            elif pos[w] < len(skel[w]):
                r = ready_at(w)
                if r is not None and r > t:
                    nxt = min(nxt, r)
        if nxt == INF:
            if any(pos[w] < len(skel[w]) for w in range(p)) or doneW < nW:
                if all(busy[w] <= t for w in range(p)) and not any(pend[w] for w in range(p)):
                    raise RuntimeError("shift_w stalled")
            nxt = t + 1
        t = nxt
    return out


def zbv_schedule(p: int, m: int, TF: int, TB: int, TW: int, Tcomm: int = 0, MB: int = 1, MW: int = 1,
                 Mlimit=None):
    """ZB-V with the W right-shift: candidates 0 = the construction, 1 = shift
    rule "gap", 2 = shift rule "fill"; those within M_limit (default: the
    construction's own peak) compete on (cost, max peak, index).
    Returns (lists, chosen, sim)."""
    base = build_zbv(p, m)
    place = lambda v: worker_of(p, v)
    lim = Mlimit if Mlimit is not None else max(memory_peaks_v(base, MB, MW))
    if max(memory_peaks_v(base, MB, MW)) > lim:
        raise ValueError("M_limit below the ZB-V construction's peak (p M_B of a stage)")
    cands = [(0, base)]
    for idx, rule in ((1, "gap"), (2, "fill")):
        try:
            cands.append((idx, shift_w(base, p, TF, TB, TW, Tcomm, MB, MW, lim, rule)))
        except ValueError:
            pass
    best = None
    for idx, l in cands:
        pk = max(memory_peaks_v(l, MB, MW))
        if idx and pk > lim:
            continue
        sim = simulate_v(l, 2 * p, place, TF, TB, TW, Tcomm)
        key = (sim["cost"], pk, idx)
        if best is None or key < best[0]:
            best = (key, idx, l, sim)
    return best[2], best[1], best[3]
