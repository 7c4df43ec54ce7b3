timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_rc.json 2> gpurun_out/bench_rc.err; echo rc=$?; tail -2 gpurun_out/bench_rc.err
