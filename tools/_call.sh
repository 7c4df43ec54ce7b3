for t in 65536 81920 98304; do SK_TILE_BYTES=$t timeout 300 python tools/time_sensor.py | head -1; done
for t in 16384 24576 40960; do SK_TILE_BYTES=$t timeout 300 python tools/time_paths.py 2>&1 | grep particle | sed "s/^/tile=$t /"; done
