"""Which schedule the auto mode picks (last_mode = 100*mode + CTAs per scenario)
for C3 dn=1 and C2 at B=1, call by call: mode_probe.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25068_b200 as P

for name, sc in (("c3_dn1", P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 1, 3600, 300)),
                 ("c2", P.Scenario.grid(50, 400.0, 42, 1000.0).configure(100000, 1, 3600, 300))):
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, 1, 3600)
    e.set_params(p)
    e.set_state(lk, ps)
    e.set_noise(7, 0, 0)
    modes = []
    for T in (10, 3600, 3600):
        e.forward(T, sc.steps_per_interval)
        e.sync()
        modes.append(e.last_mode)
    print(name, "N", sc.n_agents, "L", sc.n_links, "last_mode per call", modes, flush=True)
