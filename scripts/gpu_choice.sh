# Step-graph check: fused vs graph timings per batch size, the graph's GPU
# equality tests, and the B=256 launch list (profiles/r01/graph_b256_summary.md).
timeout 200 python scripts/graph_time.py 32 64 256 2>&1 | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_persistent.py -x -q 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -c 60 --csv --log-file gpurun_out/launches_graph_b256.csv python scripts/fwd_once.py 30 120 256 3 > gpurun_out/ncu_g.log 2>&1; echo ncu rc=$?
