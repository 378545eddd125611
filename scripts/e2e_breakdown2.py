"""Host-side breakdown of the streamed e2e path (dtg_forward_read), C3."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
from paper_2603_25068_b200._lib import ptr
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3)
p2 = P.LinkParams(p.u * 1.001, p.kappa, p.beta, p.alpha, p.cost)
for _ in range(3): P.simulate_forward(sc, p, seed=7)
n = 30
t = time.perf_counter()
for i in range(n): P.simulate_forward(sc, p if i % 2 else p2, seed=7, noise_iteration=i)
print("simulate_forward e2e ms", (time.perf_counter() - t) / n * 1e3)
e = P.Engine(sc, 1, 120)
lk, ps = sc.seed_agents(); e.set_state(lk, ps)
L, N, T = sc.n_links, sc.n_agents, 120
cum = np.zeros((T, L)); lo = np.zeros(N, np.int32); po = np.zeros(N)
lib = e._lib
acc = {}
def tick(k, t0):
    t1 = time.perf_counter(); acc[k] = acc.get(k, 0) + t1 - t0; return t1
for it in range(n + 3):
    if it == 3: acc.clear()
    t = time.perf_counter()
    e.set_params(p if it % 2 else p2); t = tick("set_params", t)
    e.set_noise(7, it); t = tick("set_noise", t)
    e.forward(T, 10); e.sync(); t = tick("forward+sync (no reads)", t)
    e.set_params(p if it % 2 else p2); e.set_noise(7, it); t = time.perf_counter()
    lib.dtg_forward_read(e._h, T, 10, 0, ptr(cum), ptr(lo), ptr(po)); t = tick("forward_read(cum+state)", t)
    lib.dtg_forward_read(e._h, T, 10, 0, ptr(cum), None, None); t = tick("forward_read(cum)", t)
    lib.dtg_forward_read(e._h, T, 10, 0, None, ptr(lo), ptr(po)); t = tick("forward_read(state)", t)
    lib.dtg_forward_read(e._h, T, 10, 0, None, None, None); t = tick("forward_read(none)", t)
for k, v in acc.items(): print(f"{k:26s} {v / n * 1e3:8.3f} ms")
