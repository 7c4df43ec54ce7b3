#!/bin/bash
# ncu --set full captures of the HEAD kernels (one GPU), plus ptxas register
# counts of the library they came from, into gpurun_out/ncu_<tag>_*.ncu-rep.
# usage: tools/ncu_refresh.sh TAG [job ...]   (jobs: see tools/profile_one.py)
tag=${1:-head}; shift
jobs=${@:-obj8_a2p sensor_fused sensor_calnoise track_aosoa jagged}
mkdir -p gpurun_out
for j in $jobs; do
  if [ "$j" = reco ]; then  # the reconstruction of 64 events: tile pass, first process, first check (call 4)
    timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:tile_kernel|check_kernel|process_kernel' -s 42 -c 3 \
        -o gpurun_out/ncu_${tag}_reco -f python tools/time_reco.py > gpurun_out/ncu_${tag}_reco.log 2>&1
    echo "reco rc=$?"; continue
  fi
  case $j in
    jagged) k='regex:pack_reg|pack_fused' ;;
    sensor_calnoise) k='regex:calibrate_kernel|noise_kernel' ;;
    *) k='regex:convert_kernel' ;;
  esac
  c=1; [ "$j" = sensor_calnoise ] && c=2
  timeout 600 ncu --set full --clock-control none --import-source on -k "$k" -s 2 -c $c \
      -o gpurun_out/ncu_${tag}_$j -f python tools/profile_one.py $j 4 > gpurun_out/ncu_${tag}_$j.log 2>&1
  echo "$j rc=$?"
done
