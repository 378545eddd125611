timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -3
timeout 600 python scripts/phase_profile.py 2>&1 | grep -v "B=  8\|B= 64" | tee gpurun_out/phase.log
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
