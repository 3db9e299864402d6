"""One line per kernel launch of an `ncu --set full` report: duration, tensor-pipe
and issue utilisation, DRAM bytes and throughput, occupancy, registers.
usage: python scripts/ncu_full_summary.py report.ncu-rep [regex]"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
hdr = rows[0]
want = [("gpu__time_duration.sum", "us"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("dram__bytes_read.sum", "dramR"), ("dram__bytes_write.sum", "dramW"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
idx = {k: hdr.index(k) for k, _ in want if k in hdr}
units = rows[1]
print("kernel | " + " | ".join(f"{n}[{units[idx[k]]}]" for k, n in want if k in idx))
for r in rows[2:]:
    name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")])
    cells = []
    for k, n in want:
        if k in idx:
            v = r[idx[k]].replace(",", "")
            try:
                f = float(v)
                cells.append(f"{f:.4g}")
            except ValueError:
                cells.append(v)
    print(f"{name[:60]} | " + " | ".join(cells))
