"""The C++ scheduler behind zb_schedule / zb_simulate (libzb.so) against the
oracle (oracle/schedule.py): pass lists, slot ids, predicted start / end, cost
and memory peaks must be IDENTICAL (integer time), over a grid of (p, m,
times, limits) that includes every Table 8 row.  CPU only."""
import random

import pytest

from oracle import schedule as osch
from zbtest_util import ms_to_us, read_csv

lib_ok = True
try:
    from paper_2401_10241_b200 import api
except ImportError:       # library not built: the ABI test reports it
    lib_ok = False

pytestmark = pytest.mark.skipif(not lib_ok, reason="libzb.so not built")


def compare(family, p, m, TF, TB, TW, Tc, MB, MW, lim):
    passes, sim = api.schedule(family, p, m, TF, TB, TW, Tc, M_limit=lim, M_B=MB, M_W=MW)
    lists, maps, counts, osim, chosen = osch.schedule(family, p, m, TF, TB, TW, Tc, MB=MB, MW=MW,
                                                      Mlimit=lim if (family == "auto" or lim > 0) else None)
    got = api.stage_lists(passes, p)
    assert got == [list(o) for o in lists], (family, p, m)
    k = 0
    fused = family == "1f1b"
    for s in range(p):
        for kind, j in lists[s]:
            q = passes[k]
            assert q.slot == maps[s][j]
            assert q.start == osim["start"][(kind, s, j)] and q.end == osim["end"][(kind, s, j)]
            k += 1
    assert sim.cost == osim["cost"]
    assert abs(sim.bubble_rate - osim["bubble_rate"]) < 1e-15
    assert list(sim.n_slots[:p]) == counts
    assert list(sim.peak_bytes[:p]) == osch.memory_peaks(lists, MB, MW)
    if family == "auto":
        assert sim.chosen == chosen


@pytest.mark.parametrize("family", ["1f1b", "zbh1", "zbh2", "auto"])
def test_grid_random(family):
    rnd = random.Random(sum(map(ord, family)))
    for p in (1, 2, 3, 4, 8):
        for m in sorted({1, 2, p, max(1, 2 * p - 1), 3 * p}):
            TW = rnd.randint(1, 60)
            TF = rnd.randint(TW, 100)
            TB = rnd.randint(TF - 5, 120)
            Tc = rnd.randint(0, 5)
            MB, MW = rnd.choice([(10, 10), (39, 32), (5, 2)])
            lim = rnd.choice([p * MB, 2 * p * MB]) if family == "auto" else 0
            compare(family, p, m, TF, TB, TW, Tc, MB, MW, lim)


def test_table8_rows_all_families():
    for t in read_csv("table8_profiled_times.csv"):
        p, m = int(t["p"]), int(t["m"])
        if p > 16:
            continue
        TF, TB, TW, Tc = (ms_to_us(t[k]) for k in ("T_F", "T_B", "T_W", "T_comm"))
        b, h, a = {"1.5B": (6, 2304, 24), "6.2B": (3, 4096, 32), "14.6B": (1, 5120, 40)}[t["model"]]
        MB, MW = osch.table1_memory(1024, b, h, a, "B"), osch.table1_memory(1024, b, h, a, "W")
        for fam in ("1f1b", "zbh1", "zbh2"):
            compare(fam, p, m, TF, TB, TW, Tc, MB, MW, 0)
        for lim in (p * MB, 2 * p * MB):
            compare("auto", p, m, TF, TB, TW, Tc, MB, MW, lim)


def test_table4_from_cpp():
    """zb_schedule reproduces Table 4's 1F1B / ZB-H1 / ZB-H2 / ZB-1p columns."""
    t8 = {(r["model"], r["m"]): r for r in read_csv("table8_profiled_times.csv")}
    for r in read_csv("table4_bubble_rates.csv"):
        p, m, b, h, a = (int(r[k]) for k in ("p", "m", "b", "h", "a"))
        if p > 16:
            continue
        t = t8[(r["model"], r["m"])]
        TF, TB, TW, Tc = (ms_to_us(t[k]) for k in ("T_F", "T_B", "T_W", "T_comm"))
        MB, MW = osch.table1_memory(1024, b, h, a, "B"), osch.table1_memory(1024, b, h, a, "W")
        for fam, col, lim in (("1f1b", "1F1B", 0), ("zbh1", "ZB-H1", 0), ("zbh2", "ZB-H2", 0),
                              ("auto", "ZB-1p", p * MB)):
            _, sim = api.schedule(fam, p, m, TF, TB, TW, Tc, M_limit=lim, M_B=MB, M_W=MW)
            assert round(sim.bubble_rate, 4) == float(r[col]), (r["model"], m, col)


def test_simulate_matches_oracle_per_stage_times():
    p, m = 4, 8
    lists = osch.build_zbh2(p, m)
    TF, TB, TW = [10, 12, 11, 13], [11, 12, 10, 14], [6, 7, 5, 8]
    arr, sim = api.simulate(p, m, lists, TF, TB, TW, 2, M_B=3, M_W=3)
    o = osch.simulate(lists, TF, TB, TW, 2)
    assert sim.cost == o["cost"]
    k = 0
    for s in range(p):
        for kind, j in lists[s]:
            assert arr[k].start == o["start"][(kind, s, j)]
            k += 1


def test_errors():
    from paper_2401_10241_b200._lib import ZbError, ZB_ECAP, ZB_ELIMIT, ZB_EINVAL, lib, zb_pass_t
    with pytest.raises(ZbError) as e:
        api.schedule("auto", 4, 8, 1, 1, 1, 0, M_limit=1, M_B=3, M_W=3)
    assert e.value.code == ZB_ELIMIT
    with pytest.raises(ZbError) as e:
        api.schedule("zbh2", 4, 8, 1, 1, 1, 0, M_limit=4 * 3, M_B=3, M_W=3)
    assert e.value.code == ZB_ELIMIT
    out = (zb_pass_t * 5)()
    assert lib.zb_schedule(4, 8, 1, 1, 1, 0, 0, 1, 1, 1, out, 5, None) == ZB_ECAP
    assert lib.zb_schedule(0, 8, 1, 1, 1, 0, 0, 1, 1, 1, out, 5, None) == ZB_EINVAL
    assert lib.zb_schedule(2, 2, 1, 1, 1, 0, 0, 1, 1, 9, out, 12, None) == ZB_EINVAL


# ---------------------------------------------------------------- chunked schedules (ZB-V, 1F1B-I)

def compare_chunked(family, p, m, chunks, TF, TB, TW, Tc, MB, MW, lim):
    from oracle import zbv
    passes, sim = api.schedule_chunked(family, p, m, chunks, TF, TB, TW, Tc, M_limit=lim, M_B=MB, M_W=MW)
    nv = chunks * p
    if family == "zbv":
        lists, chosen, osim = zbv.zbv_schedule(p, m, TF, TB, TW, Tc, MB, MW, lim if lim > 0 else None)
        place = lambda v: zbv.worker_of(p, v)
        assert sim.chosen == chosen
    else:
        lists = zbv.build_1f1b_interleaved(p, m, chunks)
        place = lambda v: v % p
        osim = zbv.simulate_v(lists, nv, place, TF, TB, TW, Tc, fused=True)
    assert api.worker_lists(passes, p, m, chunks) == lists, (family, p, m)
    maps, counts = zbv.assign_slots_v(lists, nv)
    k = 0
    for w in range(p):
        for kind, v, j in lists[w]:
            q = passes[k]
            assert q.slot == maps[(v, j)]
            assert q.start == osim["start"][(kind, v, j)] and q.end == osim["end"][(kind, v, j)]
            k += 1
    assert sim.cost == osim["cost"] and sim.work == osim["work"]
    assert list(sim.n_slots[:nv]) == counts
    assert list(sim.peak_bytes[:p]) == zbv.memory_peaks_v(lists, MB, MW)


@pytest.mark.parametrize("p,m", [(1, 1), (1, 4), (2, 3), (3, 5), (4, 8), (4, 12), (8, 24), (8, 7), (6, 40)])
def test_zbv_unit_and_table8(p, m):
    compare_chunked("zbv", p, m, 2, 1, 1, 1, 0, 1, 1, 0)
    compare_chunked("zbv", p, m, 2, 9261, 9043, 4669, 601, 5, 3, 0)


def test_zbv_random_limits():
    rnd = random.Random(3)
    for _ in range(40):
        p, m = rnd.randint(1, 6), rnd.randint(1, 20)
        TF, TB, TW, Tc = rnd.randint(1, 60), rnd.randint(1, 60), rnd.randint(1, 60), rnd.randint(0, 8)
        MB, MW = rnd.randint(1, 9), rnd.randint(1, 9)
        from oracle import zbv
        pk = max(zbv.memory_peaks_v(zbv.build_zbv(p, m), MB, MW))
        lim = rnd.choice([0, pk, pk + MB, 2 * pk])
        compare_chunked("zbv", p, m, 2, TF, TB, TW, Tc, MB, MW, lim)


@pytest.mark.parametrize("p,m,chunks", [(1, 2, 1), (2, 4, 2), (4, 8, 2), (4, 12, 3), (8, 24, 3), (8, 8, 4)])
def test_interleaved(p, m, chunks):
    compare_chunked("1f1bi", p, m, chunks, 6174, 6029, 3112, 601, 1, 1, 0)


def test_chunked_errors():
    from paper_2401_10241_b200._lib import ZbError
    with pytest.raises(ZbError):
        api.schedule_chunked("1f1bi", 4, 6, 2, 1, 1, 1)        # m % p != 0
    with pytest.raises(ZbError):
        api.schedule_chunked("zbv", 4, 8, 3, 1, 1, 1)          # ZB-V needs 2 chunks
    with pytest.raises(ZbError):
        api.schedule_chunked("zbv", 40, 8, 2, 1, 1, 1)         # 80 virtual stages > 64


def compare_per_stage(family, p, m, TF, TB, TW, Tc, MB, MW, lim):
    passes, sim = api.schedule_per_stage(family, p, m, TF, TB, TW, Tc, M_limit=lim, M_B=MB, M_W=MW)
    lists, maps, counts, osim, chosen = osch.schedule(family, p, m, list(TF), list(TB), list(TW), Tc, MB=MB, MW=MW,
                                                      Mlimit=lim if (family == "auto" or lim > 0) else None)
    assert api.stage_lists(passes, p) == [list(o) for o in lists], (family, p, m)
    k = 0
    for s in range(p):
        for kind, j in lists[s]:
            q = passes[k]
            assert q.slot == maps[s][j]
            assert q.start == osim["start"][(kind, s, j)] and q.end == osim["end"][(kind, s, j)]
            k += 1
    assert sim.cost == osim["cost"]
    assert abs(sim.bubble_rate - osim["bubble_rate"]) < 1e-15
    if family == "auto":
        assert sim.chosen == chosen
        assert max(sim.peak_bytes[:p]) <= lim
    assert not osch.validate_schedule(lists, m)


@pytest.mark.parametrize("family", ["1f1b", "zbh1", "zbh2", "auto"])
def test_per_stage_times_grid(family):
    """zb_schedule_per_stage (each stage's profiled times feed the scheduler):
    heavier first / last stages (embedding, LM head) and random per-stage jitter."""
    rnd = random.Random(7 + sum(map(ord, family)))
    for p in (2, 3, 4, 8):
        for m in sorted({p, 2 * p - 1, 3 * p}):
            base = [rnd.randint(40, 100) for _ in range(3)]
            TF = [base[0] + rnd.randint(0, 10) for _ in range(p)]
            TB = [base[1] + rnd.randint(0, 15) for _ in range(p)]
            TW = [base[2] + rnd.randint(0, 10) for _ in range(p)]
            TB[-1] += rnd.randint(10, 40)            # LM head on the last stage
            TF[0] += rnd.randint(0, 5)               # embedding on stage 0
            Tc = rnd.randint(0, 4)
            MB, MW = rnd.choice([(10, 10), (39, 32)])
            lim = rnd.choice([p * MB, 2 * p * MB, 3 * p * MB]) if family == "auto" else 0
            compare_per_stage(family, p, m, TF, TB, TW, Tc, MB, MW, lim)


def test_per_stage_uniform_equals_scalar():
    for p, m in ((4, 8), (8, 24)):
        for fam in ("1f1b", "zbh1", "zbh2", "auto"):
            a, sa = api.schedule(fam, p, m, 70, 90, 50, 3, M_limit=2 * p * 10, M_B=10, M_W=10)
            b, sb = api.schedule_per_stage(fam, p, m, [70] * p, [90] * p, [50] * p, 3, M_limit=2 * p * 10, M_B=10,
                                           M_W=10)
            assert [(q.stage, q.microbatch, q.kind, q.slot, q.start, q.end) for q in a] == \
                   [(q.stage, q.microbatch, q.kind, q.slot, q.start, q.end) for q in b]
            assert sa.cost == sb.cost and sa.chosen == sb.chosen


def test_partition_rule_in_library_matches_paper_rule():
    """zb_partition == P:169's rule as written in the data module (first / last stage
    one layer fewer when (L+2) % p == 0) for every (L, p) up to 80 x 64."""
    import zb_synth
    for L in range(1, 81):
        for p in range(1, min(L, 64) + 1):
            assert api.partition(L, p) == zb_synth.partition(L, p), (L, p)
    assert api.partition(22, 8) == [2, 3, 3, 3, 3, 3, 3, 2]
    assert api.partition(62, 8) == [7, 8, 8, 8, 8, 8, 8, 7]
