timeout 300 python scripts/prof_persistent.py 1 > gpurun_out/pp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward_persistent -s 2 -c 1 -o gpurun_out/prof_persist python scripts/prof_persistent.py 1 > gpurun_out/ncu_p.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_p.log
