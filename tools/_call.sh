timeout 600 python -m pytest tests/test_gpu_reco.py -x -q 2>&1 | tail -2
SK_RECO_TRACE=1 timeout 300 python tools/time_reco.py 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 60 -c 30 python tools/time_reco.py 2>&1 | grep -E "^\s+[a-z_:<>0-9, ]+\(|gpu__time" | paste - - | awk '{print $1, $NF}' | sed -n 9,22p
