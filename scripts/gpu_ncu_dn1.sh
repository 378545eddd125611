set -x
timeout 300 python scripts/fwd_once.py 1 300 1 || exit 1
timeout 300 python scripts/fwd_once.py 30 120 64 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward_fused -s 1 -c 1 -o gpurun_out/ncu_dn1 -f python scripts/fwd_once.py 1 300 1 > gpurun_out/ncu_dn1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward_fused -s 1 -c 1 -o gpurun_out/ncu_b64 -f python scripts/fwd_once.py 30 120 64 > gpurun_out/ncu_b64.log 2>&1
ls -la gpurun_out
