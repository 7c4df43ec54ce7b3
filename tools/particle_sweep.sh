for st in 2 3 4 6; do for tb in 24576 32768 49152; do SK_STAGES=$st SK_TILE_BYTES=$tb CASES=particle timeout 120 python tools/time_paths.py; done; done
for c in 2 3; do SK_CTAS=$c CASES=particle timeout 120 python tools/time_paths.py; done
CASES=particle timeout 120 python tools/time_paths.py
