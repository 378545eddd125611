"""Wall time of run_gradcheck: device (batched probes) vs the reference build."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_25068_b200 import fdcheck as F
F.run_gradcheck(2, 20, 5, 1e-4, 1)
for cfg in [(20, 20, 5, 1e-4, 1), (5, 60, 21, 1e-4, 7)]:
    t = time.perf_counter(); r = F.run_gradcheck(*cfg); dt = time.perf_counter() - t
    print("device", cfg, f"{dt:.3f} s", r.redraws, r.passed, r.max_rel_err)
try:
    from oracle.oracle import RefLib
    R = RefLib()
    for cfg in [(20, 20, 5, 1e-4, 1), (5, 60, 21, 1e-4, 7)]:
        t = time.perf_counter(); r = R.run_gradcheck(*cfg); dt = time.perf_counter() - t
        print("reference", cfg, f"{dt:.3f} s", r["redraws"], r["passed"])
except Exception as e:
    print("no reference:", e)
