"""Probe: C3 dn=1 (1,000,020 agents) forward parity vs the C port over a few
steps, then device time per step for the full-hour horizon; batched C3 dn=30
at B scenarios.  Exploratory measurement helper (not part of the product)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_25068_b200 as P  # noqa: E402


def scen(dn, T, veh=1000020):
    return P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(veh, dn, T, 300 if dn > 1 else 300)


def timed(eng, T, spi, reps=3):
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    eng.forward(T, spi, checkpoint=False)
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        ev[0].record(st)
        eng.forward(T, spi, checkpoint=False)
        ev[1].record(st)
        torch.cuda.synchronize()
        out.append(ev[0].elapsed_time(ev[1]))
    return min(out), float(np.median(out))


res = {}
mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode in ("all", "parity"):
    from oracle.oracle import Params, PortLib, PortScenario
    T = 12
    sc = scen(1, T)
    p = sc.sample_parameters(3)
    t0 = time.time()
    tr = P.simulate_forward(sc, p, seed=7)
    f, t, ln, k = sc.links()
    lk, ps = sc.seed_agents()
    port = PortScenario(PortLib(), f, t, ln, delta_n=1, link0=lk, pos0=ps, horizon_steps=T, obs_interval_s=300)
    ref = port.forward(Params(*p.arrays()), 7, 0)
    ok = (np.array_equal(tr.cum_per_step, ref["cum_per_step"]) and np.array_equal(tr.link_final, ref["link"])
          and np.array_equal(tr.pos_final, ref["pos"]))
    res["dn1_parity_12_steps"] = bool(ok)
    res["dn1_N"] = int(sc.n_agents)
    res["dn1_port_s"] = time.time() - t0
if mode in ("all", "time"):
    for dn, T in ((1, 600), (30, 120)):
        sc = scen(dn, T)
        p = sc.sample_parameters(3)
        eng = P.Engine(sc, n_scenarios=1, max_steps=T)
        lk, ps = sc.seed_agents()
        eng.set_params(p)
        eng.set_state(lk, ps)
        eng.set_noise(7, 0)
        spi = sc.steps_per_interval
        for m in (0, 3):
            eng.set_mode(m)
            mn, md = timed(eng, T, spi)
            res[f"dn{dn}_T{T}_mode{m}_ms"] = md
            res[f"dn{dn}_T{T}_mode{m}_us_per_step"] = 1000 * md / T
            res[f"dn{dn}_last_mode_{m}"] = eng.last_mode
        if dn == 1:
            eng.set_mode(0)
            eng.forward(T, spi)
            ph, grid = eng.profile_persistent(T, spi)
            res["dn1_phases"] = ph
            res["dn1_grid"] = grid
if mode in ("all", "batch"):
    T = 120
    sc = scen(30, T)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    for B in (64, 256):
        eng = P.Engine(sc, n_scenarios=B, max_steps=T)
        eng.set_params(p)
        eng.set_state(lk, ps)
        for b in range(B):
            eng.set_noise(7, b, b)
        for m in (0, 3):
            eng.set_mode(m)
            mn, md = timed(eng, T, sc.steps_per_interval)
            res[f"B{B}_mode{m}_ms"] = md
            res[f"B{B}_mode{m}_last"] = eng.last_mode
        del eng
print(json.dumps(res, indent=1))
