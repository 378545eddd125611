timeout 600 python bench.py > gpurun_out/bench_b1.json 2> gpurun_out/bench_b1.err; echo rc=$?
timeout 600 python bench.py --scenarios 8 --no-cpu-baseline --no-gradient > gpurun_out/bench_b8.json 2> gpurun_out/bench_b8.err; echo rc=$?
timeout 600 python bench.py --scenarios 64 --no-cpu-baseline --no-gradient > gpurun_out/bench_b64.json 2> gpurun_out/bench_b64.err; echo rc=$?
timeout 300 python bench.py --no-cpu-baseline --no-gradient --steps 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1450 -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --no-gradient --steps 3 > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
