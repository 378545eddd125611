import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25068_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, 120); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b, b)
for _ in range(3): e.forward(120, 10)
e.sync(); print("ok")
