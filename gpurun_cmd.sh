cat > /tmp/one_attn.py <<'PY'
import sys, torch; sys.path.insert(0, ".")
from paper_2401_10241_b200 import api
b, s, a, d = 3, 1024, 32, 128
h = a * d
qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16(); o = torch.empty(b * s, h, device="cuda").bfloat16()
lse = torch.empty(b, a, s, device="cuda")
for _ in range(3): api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc -s 2 -c 1 -o gpurun_out/attn_fwd_full2 python /tmp/one_attn.py > gpurun_out/ncu_attn.log 2>&1
ncu -i gpurun_out/attn_fwd_full2.ncu-rep --page source --csv > gpurun_out/attn_fwd_source2.csv 2>/dev/null
ncu -i gpurun_out/attn_fwd_full2.ncu-rep --page details --csv > gpurun_out/attn_fwd_details2.csv 2>/dev/null
