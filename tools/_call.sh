timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo rc=$?
