"""Fused-forward phase times with parts disabled (timing only; flag 3 bits)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25068_b200 as P
dn = int(sys.argv[1]) if len(sys.argv) > 1 else 30
T = 120 if dn == 30 else 300
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, dn, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b, b)
for dbg in [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2", "3"])]:
    e.set_flag(3, dbg)
    e.forward(T, sc.steps_per_interval)
    ph, g = e.profile_persistent(T, sc.steps_per_interval)
    print(dn, B, dbg, g, {k: round(v, 2) for k, v in ph.items()}, round(sum(ph.values()), 2), flush=True)
