#!/bin/bash
# per-kernel times + DRAM bytes of the jagged pack (tools/time_pack.py) -> gpurun_out/pack_ncu.csv
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none --csv --log-file gpurun_out/pack_ncu.csv python tools/time_scan.py > gpurun_out/pack_ncu.log 2>&1
