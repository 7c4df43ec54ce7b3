mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo rc=$?
tail -5 gpurun_out/bench_r02a.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r02a.json 2>gpurun_out/bench_ref_r02a.err; echo rc=$?
tail -3 gpurun_out/bench_ref_r02a.err
