"""Host-side breakdown of one e2e simulate_forward call (C3)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3)
for _ in range(3): P.simulate_forward(sc, p, seed=7)
t = time.perf_counter(); n = 20
for _ in range(n): P.simulate_forward(sc, p, seed=7)
print("simulate_forward e2e ms", (time.perf_counter() - t) / n * 1e3)
e = P.Engine(sc, 1, 120)
acc = {}
def tick(k, t0):
    t1 = time.perf_counter(); acc[k] = acc.get(k, 0) + t1 - t0; return t1
for it in range(n + 3):
    if it == 3: acc.clear()
    t = time.perf_counter()
    lk, ps = sc.seed_agents(); t = tick("seed_agents(py)", t)
    e.set_params(p); t = tick("set_params", t)
    e.set_state(lk, ps); t = tick("set_state", t)
    e.set_noise(7, 0); t = tick("set_noise", t)
    e.forward(120, 10); e.sync(); t = tick("forward+sync", t)
    c = e.read_cum_all(); t = tick("read_cum_all", t)
    s = e.read_state(0, -1); t = tick("read_state", t)
for k, v in acc.items(): print(f"{k:18s} {v / n * 1e3:8.3f} ms")
