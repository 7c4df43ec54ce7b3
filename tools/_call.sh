timeout 600 python -m pytest tests/test_gpu_soakit_plugin.py tests/test_gpu_sensor.py -x -q 2>&1 | grep -v "^\s*$" | grep -E "Error|error|assert|^E |test_|passed|failed" | head -40
