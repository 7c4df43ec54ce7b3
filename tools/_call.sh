SK_FUSED_PRESCAN=1 timeout 600 python -m pytest tests/test_gpu_jagged_paths.py tests/test_gpu_jagged.py tests/test_gpu_jagged_fuzz.py -x -q 2>&1 | tail -2
timeout 300 python tools/time_jagged.py 1000000 10000000
for b in 2 3 4 6 8; do SK_FUSED_PRESCAN=1 SK_PRESCAN_BPC=$b timeout 300 python tools/time_jagged.py 1000000 10000000 | sed "s/^/bpc=$b /"; done
