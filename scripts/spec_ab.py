"""A/B of the speculative head decisions (dtg_set_flag 4): wall per run, phase
split, and bit-identical counts / final state."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P


def case(name, n, ln, veh, dn, T, B):
    sc = P.Scenario.grid(n, ln, 42, 1000.0).configure(veh, dn, T, 300)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T)
    e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b, b)
    spi = max(1, sc.steps_per_interval)
    res = {}
    for spec in (0, 1, 0, 1):
        e.set_flag(4, spec)
        for _ in range(3): e.forward(T, spi)
        e.sync()
        t = time.perf_counter()
        for _ in range(10): e.forward(T, spi)
        e.sync()
        ms = (time.perf_counter() - t) / 10 * 1e3
        cum = e.read_cum_all(); st = e.read_state(0, -1)
        ph, g = e.profile_persistent(T, spi)
        if spec in res:
            assert np.array_equal(res[spec][0], cum)
        res[spec] = (cum, st)
        print(f"{name:20s} B={B:3d} spec={spec} grid={g:4d} wall/run={ms:7.3f} ms  per-step us: " +
              " ".join(f"{k}={v:6.2f}" for k, v in ph.items()), flush=True)
    assert np.array_equal(res[0][0], res[1][0]), "counts differ"
    assert all(np.array_equal(a, b) for a, b in zip(res[0][1], res[1][1])), "state differs"
    print("  identical")


case("C3 dn30", 23, 1609.34, 1000020, 30, 120, 1)
case("C3 dn30", 23, 1609.34, 1000020, 30, 60, 8)
case("C1 4x4 dn1", 4, 400.0, 1000, 1, 1800, 1)
case("C3 dn1 (1M agents)", 23, 1609.34, 1000020, 1, 300, 1)
