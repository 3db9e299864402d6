timeout 60 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_delta python scripts/micro/delta_one.py 2>&1 | grep -E "gpu__time" | tail -3
ZB_LIB=libzb_old.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_delta python scripts/micro/delta_one.py 2>&1 | grep -E "gpu__time" | tail -3
