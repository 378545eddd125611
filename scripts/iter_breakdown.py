"""Host-side breakdown of one device calibration iteration (C4 shape, B=8)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
B, T = 8, 60
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_state(lk, ps)
ids = np.array([j for j in range(sc.n_links) if j % 5], np.int32)
e.set_loss_mse(ids, np.zeros((T // sc.steps_per_interval, len(ids))))
spi = sc.steps_per_interval
acc = {}
def tick(name, t0):
    t1 = time.perf_counter(); acc[name] = acc.get(name, 0.0) + (t1 - t0); return t1
for it in range(12):
    if it == 2: acc.clear()
    t = time.perf_counter()
    e.set_params(p); t = tick("set_params", t)
    for b in range(B): e.set_noise(7, it * B + b + 1, b)
    t = tick("set_noise", t)
    e.forward(T, spi, checkpoint=True); t = tick("forward(launch)", t)
    e.sync(); t = tick("forward(sync)", t)
    e.gradient_device_loss(); t = tick("grad(launch)", t)
    e.sync(); t = tick("grad(sync)", t)
    r = e.reduce_draw_rows(B); t = tick("reduce+d2h", t)
for k, v in acc.items(): print(f"{k:18s} {v / 10 * 1e3:8.3f} ms")
print("total", sum(acc.values()) / 10 * 1e3)
t = time.perf_counter()
res = P.calibrate(sc, ids, np.zeros((T // spi, len(ids))), 7, cfg=P.OptimizeConfig(max_iterations=12, patience=100, noise_draws=8))
print("calibrate 12 it wall", res.wall_seconds, "per it", res.wall_seconds / 12 * 1e3, "ms")
