timeout 600 python -m pytest tests/test_gpu_reco.py -x -q 2>&1 | tail -2
timeout 300 python tools/time_reco.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 python tools/time_reco.py 2>&1 | grep -E "^\s+[a-z_:<>0-9, ]+\(|gpu__time" | paste - - | awk '{print $1, $NF}' | head -36
