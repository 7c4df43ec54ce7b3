timeout 900 python -m pytest tests/test_gpu_memctx.py tests/test_gpu_convert.py tests/test_gpu_graphs.py -x -q 2>&1 | tail -2
