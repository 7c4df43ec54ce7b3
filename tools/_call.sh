timeout 900 python -m pytest tests/test_gpu_sensor.py tests/test_gpu_graphs.py tests/test_gpu_convert.py -x -q 2>&1 | tail -3
