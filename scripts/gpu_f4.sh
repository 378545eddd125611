nvidia-smi --query-gpu=name --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_fdcheck.py -x -q 2>&1 | tail -30
