set -x
timeout 600 python bench.py > gpurun_out/bench_b1.json 2> gpurun_out/bench_b1.err; echo rc=$?
timeout 600 python bench.py --scenarios 8 --no-cpu-baseline --no-gradient > gpurun_out/bench_b8.json 2> gpurun_out/bench_b8.err; echo rc=$?
timeout 600 python bench.py --scenarios 64 --no-cpu-baseline --no-gradient > gpurun_out/bench_b64.json 2> gpurun_out/bench_b64.err; echo rc=$?
tail -5 gpurun_out/*.err
