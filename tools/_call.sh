for b in 1 2 3 4; do SK_FUSED_BPC=$b timeout 300 python tools/time_jagged.py 1000000 10000000 2>&1 | sed "s/^/bpc=$b /" | tail -2; done
timeout 900 python -m pytest tests/test_gpu_jagged_paths.py tests/test_gpu_jagged.py tests/test_gpu_jagged_fuzz.py tests/test_gpu_external.py tests/test_gpu_shard.py tests/test_gpu_reco.py -x -q 2>&1 | tail -5
