timeout 300 python scripts/f4_time.py 2>&1 | tail -6
timeout 300 python scripts/e2e_breakdown.py 2>&1 | tail -12
