"""Per-phase timing of the persistent forward kernel (globaltimer stamps)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_25068_b200 as P

def case(name, n, ln, veh, dn, T, B, mode=0, flag=1, opt=0):
    sc = P.Scenario.grid(n, ln, 42, 1000.0).configure(veh, dn, T, 300 if dn < 30 else 300)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T)
    e.set_mode(mode)
    e.set_flag(0, flag)
    e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b, b)
    spi = max(1, sc.steps_per_interval)
    for _ in range(3): e.forward(T, spi)
    e.sync()
    t = time.perf_counter()
    for _ in range(10): e.forward(T, spi)
    e.sync()
    ms = (time.perf_counter() - t) / 10 * 1e3
    ph, g = e.profile_persistent(T, spi)
    tot = sum(ph.values())
    print(f"{name:22s} mode={e.last_mode:4d} B={B:3d} grid={g:4d} wall/run={ms:7.3f} ms  per-step us: " +
          " ".join(f"{k}={v:6.2f}" for k, v in ph.items()) + f"  sum={tot:6.2f}", flush=True)

case("C3 dn30", 23, 1609.34, 1000020, 30, 120, 1, 2, 1)
case("C3 dn30", 23, 1609.34, 1000020, 30, 120, 8, 2, 1)
case("C1 4x4 dn1", 4, 400.0, 1000, 1, 1800, 1)
case("C3 dn30", 23, 1609.34, 1000020, 30, 120, 1)
case("C3 dn30", 23, 1609.34, 1000020, 30, 120, 8)
case("C3 dn30", 23, 1609.34, 1000020, 30, 120, 64)
case("C3 dn1 (1M agents)", 23, 1609.34, 1000020, 1, 300, 1)
case("C2 50x50 dn1 (100k)", 50, 400.0, 100000, 1, 300, 1)
