"""Does allocating fresh output arrays cost the e2e call (first-touch page
faults)?  simulate_forward vs the same C-ABI call into reused arrays, C3."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2603_25068_b200 as P
from paper_2603_25068_b200._lib import ptr

sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3)
p2 = P.LinkParams(p.u * 1.001, p.kappa, p.beta, p.alpha, p.cost)
T, L, N = sc.horizon_steps, sc.n_links, sc.n_agents
for _ in range(3):
    P.simulate_forward(sc, p, seed=7)
n = 50
for rep in range(2):
    t = time.perf_counter()
    for i in range(n):
        P.simulate_forward(sc, p if i % 2 else p2, seed=7, noise_iteration=i)
    a = (time.perf_counter() - t) / n * 1e3
    cum = np.empty((1, T, L))
    lk, ps = np.empty((1, N), np.int32), np.empty((1, N))
    wall = np.zeros(1)
    its = np.zeros(1, np.uint64)
    t = time.perf_counter()
    for i in range(n):
        its[0] = i
        q = p if i % 2 else p2
        sc._check(sc._lib.dtg_simulate_forward(sc._h, *q.arrays(), 7, 1, its, ptr(cum), ptr(lk), ptr(ps),
                                               None, None, ptr(wall)))
    b = (time.perf_counter() - t) / n * 1e3
    print(f"fresh arrays {a:.3f} ms   reused arrays {b:.3f} ms", flush=True)
