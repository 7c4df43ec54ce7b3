timeout 300 python tools/reco_host.py 2>&1 | head -50
