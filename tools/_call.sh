bash tools/ncu_refresh.sh r02 obj8_a2p obj8_1m sensor_fused sensor_calnoise track_aosoa jagged reco
timeout 300 python tools/time_scan.py > gpurun_out/time_scan_r02.txt 2>&1
INORDER=1 timeout 300 python tools/time_scan.py >> gpurun_out/time_scan_r02.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/launches_r02_bench.log 2>&1; echo launches rc=$?
cp build/csrc/*.ptxas.txt gpurun_out/ 2>/dev/null; true
