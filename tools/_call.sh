for c in 2 3 5; do SK_CTAS=$c timeout 300 python tools/time_paths.py 2>&1 | grep particle | sed "s/^/ctas=$c /"; done
for st in 3 4; do SK_STAGES=$st timeout 300 python tools/time_paths.py 2>&1 | grep particle | sed "s/^/stages=$st /"; done
SK_SPECIALIZE=0 timeout 300 python tools/time_paths.py 2>&1 | grep particle | sed "s/^/nospec /"
