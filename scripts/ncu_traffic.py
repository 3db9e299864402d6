"""Summarise an ncu DRAM capture of the GEMM launches of one microbatch
(scripts/profile_step.py --layers 2 --m 1 under
 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_gemm)
into profiles/gemm_dram_traffic.json: mean DRAM bytes per GEMM launch, weighted
to the bench step's mix (L layers x 12 layer GEMMs + 3 LM-head GEMMs per
microbatch), next to the algorithmic (compulsory) bytes of the same shapes."""
import csv, collections, json, re, sys

src, out = sys.argv[1], sys.argv[2]
model = sys.argv[3] if len(sys.argv) > 3 else "1.5B"
# bench.py steps: c2 (1.5B, b = 6) and c3 (6.2B, b = 3), s = 1024
L, h, T, V = {"1.5B": (22, 2304, 6144, 50304), "6.2B": (30, 4096, 3072, 50304)}[model]
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        per.setdefault(r[ii], {"name": re.sub(r"\(.*", "", r[ki])})[r[mi]] = float(r[vi].replace(",", ""))
launches = list(per.values())
byt = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in launches]
# the LM-head GEMMs are the three launches touching the [T, V] logits (EPI 5 F / B and the head W)
head_idx = sorted(range(len(byt)), key=lambda i: -byt[i])[:3]
layer = [b for i, b in enumerate(byt) if i not in head_idx]
head = [byt[i] for i in head_idx]
n_layer, n_head = 12 * L, 3
mean = (n_layer * (sum(layer) / len(layer)) + n_head * (sum(head) / len(head))) / (n_layer + n_head)
# algorithmic bytes (each operand read once, outputs written once; W's f32 grad read + written)
e = 2
f = [T * h * e + 3 * h * h * e + T * 3 * h * e, T * h * e + h * h * e + 2 * T * h * e,
     T * h * e + 4 * h * h * e + 2 * T * 4 * h * e, T * 4 * h * e + 4 * h * h * e + 2 * T * h * e]
bw = [T * 3 * h * e + 3 * h * h * e + T * h * 4, T * h * e + h * h * e + T * h * 4,
      T * 4 * h * e + 4 * h * h * e + T * h * 4, T * h * e + 4 * h * h * e + T * 4 * h * e * 2]
w = [T * 3 * h * e + T * h * e + 3 * h * h * 8, T * h * e * 2 + h * h * 8, T * 4 * h * e + T * h * e + 4 * h * h * 8,
     T * h * e + T * 4 * h * e + 4 * h * h * 8]
alg_layer = (sum(f) + sum(bw) + sum(w)) / 12
alg_head = (T * h * e + V * h * e + T * V * 4 + T * V * e + V * h * e + T * h * 4 + T * V * e + T * h * e + V * h * 8) / 3
alg = (n_layer * alg_layer + n_head * alg_head) / (n_layer + n_head)
rec = {"model": model, "dram_bytes_per_launch": round(mean), "algorithmic_bytes_per_launch": round(alg),
       "ratio": round(mean / alg, 3), "launches_captured": len(launches),
       "layer_gemm_mean_bytes": round(sum(layer) / len(layer)), "head_gemm_mean_bytes": round(sum(head) / len(head)),
       "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum, one {model} microbatch (2 layers + head), "
                 f"weighted to the bench step ({L} layers x 12 + 3 head GEMMs); " + src.split("/")[-1]}
try:   # one record per model (bench.py gemm_traffic looks its model up)
    allrec = json.load(open(out))
    if "dram_bytes_per_launch" in allrec:
        allrec = {allrec.get("model", "1.5B"): allrec}
except (OSError, ValueError):
    allrec = {}
allrec[model] = rec
json.dump(allrec, open(out, "w"), indent=1)
print(open(out).read())
