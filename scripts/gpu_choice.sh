timeout 300 python scripts/graph_time.py 8 16 24 32 40 48 64 96 128 2>&1 | tail -20
