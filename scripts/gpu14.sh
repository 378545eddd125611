timeout 300 python scripts/prof_persistent.py 1 > gpurun_out/pp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward_fused -s 2 -c 1 -o gpurun_out/prof_fused python scripts/prof_persistent.py 1 > gpurun_out/ncu_f.log 2>&1; echo rc=$?
