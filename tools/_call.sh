timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_sp.json 2> gpurun_out/bench_sp.err; echo rc=$?; tail -3 gpurun_out/bench_sp.err
