timeout 200 python scripts/graph_time.py 32 64 256 2>&1 | cut -c1-60
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
