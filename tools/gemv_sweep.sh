timeout 200 python -m pytest tests/test_gpu_linear.py -x -q -k gemv 2>&1 | tail -2
for wl in 0 4 5 6 8; do echo "WL=$wl"; QLRT_GEMV_WL=$wl timeout 100 python -m pytest tests/test_gpu_linear.py -x -q -k gemv 2>&1 | tail -1; QLRT_GEMV_WL=$wl timeout 200 python tools/bench_mem.py gemv 2>&1 | grep -A3 gemv_ | grep -E "gemv_|single_us"; done
