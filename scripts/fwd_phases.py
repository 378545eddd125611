"""Per-step phase spans of the fused forward (dtg_profile_persistent) for C3
at B = 1 and B = 8 (the C4 gradient forward), with and without checkpoints."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25068_b200 as P
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
for B in (1, 8):
    e = P.Engine(sc, B, 120); e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b + 1, b)
    e.forward(120, 10); e.sync()
    ph, g = e.profile_persistent(120, 10)
    print(f"B={B} grid={g}: " + "  ".join(f"{k} {v:.2f}" for k, v in ph.items()) + " us/step", flush=True)
