timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -15
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
