"""Run one forward (after a warm-up) for ncu captures: fwd_once.py DN T B [mode]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25068_b200 as P
DN, T, B = (int(a) for a in sys.argv[1:4])
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, DN, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps); e.set_mode(mode)
for b in range(B): e.set_noise(7, b, b)
e.forward(T, sc.steps_per_interval); e.sync()
e.forward(T, sc.steps_per_interval); e.sync()
print("ok", e.last_mode)
