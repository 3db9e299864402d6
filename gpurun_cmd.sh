for ps in 2 3 4 6; do echo per_sm=$ps; ZB_COLRED_PER_SM=$ps timeout 100 python scripts/ops_perf.py 2>&1 | grep -E "ln_bwd_total|bias_h|bias_4h"; done
