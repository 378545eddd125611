timeout 200 python scripts/graph_time.py 32 64 256 2>&1 | tail -6
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step -c 60 --csv --log-file gpurun_out/launches_graph_b256.csv python scripts/fwd_once.py 30 120 256 3 > gpurun_out/ncu_g.log 2>&1; echo ncu rc=$?
