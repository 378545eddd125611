timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -3
timeout 600 python scripts/phase_profile.py 2>&1 | tee gpurun_out/phase.log
timeout 600 python scripts/grad_breakdown.py 8 2>&1 | tail -7
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
