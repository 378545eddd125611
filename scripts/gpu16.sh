timeout 600 python scripts/phase_profile.py 2>&1 | grep "opt=" | tee gpurun_out/phase_opt.log
