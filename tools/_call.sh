timeout 300 python tools/time_k5.py
timeout 600 python -m pytest tests/test_gpu_sensor.py tests/test_gpu_soakit_plugin.py -x -q 2>&1 | tail -2
