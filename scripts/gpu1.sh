set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python scripts/gpu_debug.py 2>&1 | tee gpurun_out/debug.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30 | tee gpurun_out/pytest.log
