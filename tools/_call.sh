timeout 900 python -m pytest tests/test_gpu_reco.py -x -q 2>&1 | tail -2
timeout 300 python tools/time_reco.py
timeout 300 python tools/time_reco.py
