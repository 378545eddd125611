"""Reverse-sweep phase times with parts of R1 disabled (timing only)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8; T = 60
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b + 1, b)
for dbg in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,1,2,4,7".split(","))]:
    e.set_flag(2, dbg)
    e.forward(T, sc.steps_per_interval, checkpoint=True)
    ph, g = e.profile_backward()
    print(dbg, g, {k: round(v, 2) for k, v in ph.items()}, flush=True)
e.set_flag(2, 0)
