timeout 60 python scripts/attn_fwd_trace.py 2>&1 | tail -10
