"""Memory-limit sweep properties (§5.4, §6, App. B
P:465-477) of the library's schedulers on Table 8's 1.5B profile with this
build's memory model (flash attention: M_W = M_B):

* AUTO's simulated bubble never grows (beyond a 1e-3 heuristic wiggle) when
  M_limit grows ("close-to-linear decreasing trend");
* with the paper's memory model (Table 1: M_B = sb(34h+5as), M_W = 32sbh) it
  plateaus at App. B's threshold k* M_B ("the curve should plateau
  around ((p-1)(T_B+2T_comm)+pT_F)/T_F M_B"): within 0.003 of its value at
  3p M_B (with M_W = M_B nothing is freed by B and the plateau moves right —
  the B200 shift DESIGN.md records);
* at 1F1B's memory (p M_B) ZB-V beats AUTO ("when the memory limit is
  below 2pM_B, ZB-V demonstrates a significant advantage"), and below p M_B it
  is rejected (ZB_ELIMIT).
"""
import pytest

from oracle import schedule as osch
from zbtest_util import ms_to_us, read_csv

try:
    from paper_2401_10241_b200 import api
    from paper_2401_10241_b200._lib import ZbError
    LIB = True
except ImportError:
    LIB = False

pytestmark = pytest.mark.skipif(not LIB, reason="libzb.so not built")


@pytest.mark.parametrize("model,m,h,a,b", [("1.5B", 24, 2304, 24, 6), ("6.2B", 32, 4096, 32, 3)])
def test_sweep_properties(model, m, h, a, b):
    t = next(r for r in read_csv("table8_profiled_times.csv") if r["model"] == model and int(r["m"]) == m)
    TF, TB, TW, TC = (ms_to_us(t[k]) for k in ("T_F", "T_B", "T_W", "T_comm"))
    p, MB = 8, 1000
    k_star = osch.appendix_b(p, TF, TB, TC, MB)["k_star"]
    for mb, mw in ((MB, MB), (osch.table1_memory(1024, b, h, a, "B"), osch.table1_memory(1024, b, h, a, "W"))):
        rates = []
        for k in range(1, 3 * p + 1):
            _, sim = api.schedule("auto", p, m, TF, TB, TW, TC, M_limit=k * mb, M_B=mb, M_W=mw)
            assert max(sim.peak_bytes[:p]) <= k * mb
            rates.append(sim.bubble_rate)
        assert all(y <= x + 1e-3 for x, y in zip(rates, rates[1:])), rates   # heuristic: +-1e-3 wiggle
        if mw < mb:   # Table 1 model: plateau at k* M_B
            assert rates[k_star - 1] - rates[-1] <= 3e-3, (k_star, rates)
            assert rates[k_star - 5] - rates[-1] > 5e-3
    _, auto_p = api.schedule("auto", p, m, TF, TB, TW, TC, M_limit=p * MB, M_B=MB, M_W=MB)
    _, zbv_p = api.schedule_chunked("zbv", p, m, 2, TF // 2, TB // 2, TW // 2, TC, M_limit=p * MB, M_B=MB // 2,
                                    M_W=MB // 2)
    assert zbv_p.bubble_rate < auto_p.bubble_rate
    with pytest.raises(ZbError):
        api.schedule_chunked("zbv", p, m, 2, TF // 2, TB // 2, TW // 2, TC, M_limit=p * MB - 1, M_B=MB // 2,
                             M_W=MB // 2)
