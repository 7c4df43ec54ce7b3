timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02_final2.json 2> gpurun_out/bench_r02_final2.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r02_final2.json 2> gpurun_out/bench_ref_r02_final2.err; echo ref rc=$?
