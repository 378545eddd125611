"""C3 nowcast time vs CTAs per scenario of the fused grid (dtg_set_flag 7):
cs_sweep.py [B [T [checkpoint]]] (default B=1, T=120)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T = int(sys.argv[2]) if len(sys.argv) > 2 else 120
CK = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b, b)
ref = None
css = (0, 70, 74, 80, 96, 112, 148, 0) if B == 1 else (0, 10, 12, 14, 16, 17, 0)
for cs in css:
    e.set_flag(7, cs)
    for _ in range(3): e.forward(T, 10, checkpoint=bool(CK))
    e.sync(); best = 1e9
    for r in range(3):
        t = time.perf_counter()
        for _ in range(10): e.forward(T, 10, checkpoint=bool(CK))
        e.sync(); best = min(best, (time.perf_counter() - t) / 10 * 1e3)
    cum = e.read_cum_all()
    if ref is None: ref = cum
    ph, g = e.profile_persistent(T, 10)
    print(f"cs={cs:3d} grid={g:3d} ms/run {best:.3f} same={np.array_equal(ref, cum)} " + " ".join(f"{k}={v:.2f}" for k, v in ph.items()), flush=True)
