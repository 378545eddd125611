timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 300 python bench.py --no-cpu-baseline --no-gradient --steps 3 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_step_(merge|cf|scan|transfer)" -s 40 -c 8 -o gpurun_out/prof_fwd python bench.py --no-cpu-baseline --no-gradient --steps 3 > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
