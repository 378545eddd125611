timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python scripts/phase_profile.py 2>&1 | grep -v "B=  8\|B= 64" | tee gpurun_out/phase.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
