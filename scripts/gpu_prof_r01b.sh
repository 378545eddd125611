set -x
timeout 600 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 3 --no-gradient --no-throughput --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward_fused -s 1 -c 1 -o gpurun_out/ncu_fused_c3_r01b -f python scripts/fwd_once.py 30 120 1 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
