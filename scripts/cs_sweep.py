"""C3 B=1 nowcast time vs CTAs per scenario (dtg_set_flag 7)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, 1, 120); e.set_params(p); e.set_state(lk, ps); e.set_noise(7, 0, 0)
ref = None
for cs in (0, 70, 74, 80, 96, 112, 148, 0):
    e.set_flag(7, cs)
    for _ in range(3): e.forward(120, 10)
    e.sync(); best = 1e9
    for r in range(3):
        t = time.perf_counter()
        for _ in range(10): e.forward(120, 10)
        e.sync(); best = min(best, (time.perf_counter() - t) / 10 * 1e3)
    cum = e.read_cum_all()
    if ref is None: ref = cum
    ph, g = e.profile_persistent(120, 10)
    print(f"cs={cs:3d} grid={g:3d} ms/run {best:.3f} same={np.array_equal(ref, cum)} " + " ".join(f"{k}={v:.2f}" for k, v in ph.items()), flush=True)
