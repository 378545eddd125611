timeout 600 python scripts/grad_breakdown.py 8 2>&1 | tail -8
timeout 600 python scripts/grad_breakdown.py 1 2>&1 | tail -8
