timeout 900 python -m pytest tests/test_gpu_reco.py tests/test_gpu_sensor.py -x -q 2>&1 | tail -2
