"""Timing of the fused forward for batched cases + exactness against the step graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P


def case(name, dn, T, B, ckpt=False, n=23, ln=1609.34, veh=1000020):
    sc = P.Scenario.grid(n, ln, 42, 1000.0).configure(veh, dn, T, 300)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T)
    e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b, b)
    spi = max(1, sc.steps_per_interval)
    for _ in range(3): e.forward(T, spi, checkpoint=ckpt)
    e.sync()
    t = time.perf_counter()
    for _ in range(10): e.forward(T, spi, checkpoint=ckpt)
    e.sync()
    ms = (time.perf_counter() - t) / 10 * 1e3
    cum = e.read_cum_all(); st = e.read_state(B - 1, -1)
    mode = e.last_mode
    ph, g = e.profile_persistent(T, spi)
    e.set_mode(3); e.forward(T, spi, checkpoint=ckpt)
    same = np.array_equal(cum, e.read_cum_all()) and all(np.array_equal(a, b) for a, b in zip(st, e.read_state(B - 1, -1)))
    print(f"{name:24s} B={B:3d} mode={mode} wall/run={ms:8.3f} ms  per-step us: " +
          " ".join(f"{k}={v:6.2f}" for k, v in ph.items()) + f"  same_as_graph={same}", flush=True)


case("C3 dn30 B=1", 30, 120, 1)
case("C4 fwd ckpt B=8", 30, 60, 8, ckpt=True)
case("C3 dn30 B=64", 30, 120, 64)
case("C3 dn1 B=1", 1, 300, 1)
case("C2 50x50 dn1 B=1", 1, 300, 1, n=50, ln=400.0, veh=100000)
