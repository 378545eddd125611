"""Where the first simulate_forward of a new scenario spends its time
(Sioux Falls dn=4, horizons 35..90 min): context creation, uploads, the run,
read-back; then the same calls warm."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from golden_cases import load
d = load("sf_dn4")
P.load().dtg_init()
def sc_for(T):
    sc = P.Scenario.from_links(int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"])
    return sc.configure(2000, 4, T, 300, fit_queues=False)
p = P.LinkParams(*d["params"])
for rep in range(2):
    for T in (525, 600, 900, 1350):
        sc = sc_for(T)
        t0 = time.perf_counter()
        e = P.Engine(sc, 1, T)
        t1 = time.perf_counter()
        lk, ps = sc.seed_agents()
        e.set_params(p); e.set_state(lk, ps); e.set_noise(42, 0, 0)
        t2 = time.perf_counter()
        e.forward(T, 75); e.sync()
        t3 = time.perf_counter()
        cum = e.read_cum_all()
        t4 = time.perf_counter()
        tr = P.simulate_forward(sc, p, seed=42)
        t5 = time.perf_counter()
        print(f"rep {rep} T={T}: create {1e3*(t1-t0):.2f} upload {1e3*(t2-t1):.2f} forward {1e3*(t3-t2):.2f} "
              f"read {1e3*(t4-t3):.2f} | level-2 simulate_forward {1e3*(t5-t4):.2f} ms")
