for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_paths.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/san_$t.log
done
