import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2603_25068_b200 as P
T = 120
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
for B in (64, 96, 128, 148):
    e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b, b)
    st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
    for m in (0, 3):
        e.set_mode(m); e.forward(T, 10); e.sync()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(st); e.forward(T, 10); e.forward(T, 10); ev[1].record(st); torch.cuda.synchronize()
        print(B, m, e.last_mode, ev[0].elapsed_time(ev[1]) / 2, "ms", flush=True)
    del e
