timeout 600 python -m pytest tests/test_gpu_memctx.py -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
SK_BENCH_DEVICE=0 SK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 3 --warmup 3 --objects 200000000 --e2e-objects 8000000 --no-extra > gpurun_out/bench_n4_sim.json 2> gpurun_out/bench_n4_sim.err; echo n4 rc=$?
tail -c 600 gpurun_out/bench_n4_sim.json
