"""A/B of the speculation schedules: off (flag 4 = 0), idle link-phase lanes
(flag 5 = 0) and warps 2.. during barrier 1 (flag 5 = 1, default)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P


def case(name, n, ln, veh, dn, T):
    sc = P.Scenario.grid(n, ln, 42, 1000.0).configure(veh, dn, T, 300)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, 1, T)
    e.set_params(p); e.set_state(lk, ps); e.set_noise(7, 0, 0)
    spi = max(1, sc.steps_per_interval)
    ref = None
    for spec, split in ((0, 0), (1, 0), (1, 1), (1, 0), (1, 1)):
        e.set_flag(4, spec); e.set_flag(5, split)
        for _ in range(3): e.forward(T, spi)
        e.sync()
        t = time.perf_counter()
        for _ in range(20): e.forward(T, spi)
        e.sync()
        ms = (time.perf_counter() - t) / 20 * 1e3
        cum = e.read_cum_all(); st = e.read_state(0, -1)
        if ref is None: ref = (cum, st)
        same = np.array_equal(ref[0], cum) and all(np.array_equal(a, b) for a, b in zip(ref[1], st))
        ph, g = e.profile_persistent(T, spi)
        print(f"{name:12s} spec={spec} split={split} wall/run={ms:7.3f} ms  " +
              " ".join(f"{k}={v:5.2f}" for k, v in ph.items()) + f" same={same}", flush=True)


case("C3 dn30", 23, 1609.34, 1000020, 30, 120)
case("C1 4x4 dn1", 4, 400.0, 1000, 1, 1800)
