timeout 600 python scripts/phase_profile.py 2>&1 | tee gpurun_out/phase.log
timeout 600 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -3
