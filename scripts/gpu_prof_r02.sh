#!/bin/bash
# Round-2 profiles: plain runs first (exit 0), then ncu on the same commands.
set -e
mkdir -p gpurun_out/r02
python scripts/fwd_once.py 30 120 1 > gpurun_out/r02/plain_fwd.log 2>&1
python scripts/bwd_once.py 8 60 > gpurun_out/r02/plain_bwd.log 2>&1
python scripts/fwd_once.py 30 120 256 3 > gpurun_out/r02/plain_graph.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct
ncu --metrics $M --clock-control none -k regex:k_forward_fused -c 2 --csv --log-file gpurun_out/r02/ncu_fwd_metrics.csv python scripts/fwd_once.py 30 120 1 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_backward_persistent -c 2 --csv --log-file gpurun_out/r02/ncu_bwd_metrics.csv python scripts/bwd_once.py 8 60 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step -c 100 --csv --log-file gpurun_out/r02/ncu_graph_metrics.csv python scripts/fwd_once.py 30 120 256 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_forward_fused -s 1 -c 1 -o gpurun_out/r02/ncu_fwd_full python scripts/fwd_once.py 30 120 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_backward_persistent -s 1 -c 1 -o gpurun_out/r02/ncu_bwd_full python scripts/bwd_once.py 8 60 > /dev/null 2>&1
echo done
# late round 2: scenario-resident forward (mode 4, B=256) and the reverse sweep after the R4/R1 merge
python scripts/scn_once.py 256 120 > gpurun_out/r02/plain_scn.log 2>&1
ncu --metrics $M --clock-control none -k regex:k_forward_scn -s 1 -c 1 --csv --log-file gpurun_out/r02/ncu_scn_b256_metrics.csv python scripts/scn_once.py 256 120 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_backward_persistent -c 2 --csv --log-file gpurun_out/r02/ncu_bwd3_metrics.csv python scripts/bwd_once.py 8 60 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_forward_scn -s 1 -c 1 -o gpurun_out/r02/ncu_scn_full python scripts/scn_once.py 256 30 > /dev/null 2>&1
echo done2
