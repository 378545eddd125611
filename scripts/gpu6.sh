timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --scenarios 8 --no-cpu-baseline --no-gradient > gpurun_out/bench_b8.json 2> gpurun_out/bench_b8.err; echo rc=$?
tail -3 gpurun_out/bench.err
