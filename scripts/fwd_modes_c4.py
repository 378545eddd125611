"""C4 forward with checkpoints (60 steps) per schedule at B=1 and B=8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25068_b200 as P
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 60, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
for B in (1, 8):
    for mode in (1, 2, 3):
        e = P.Engine(sc, B, 60); e.set_stream(st.cuda_stream); e.set_mode(mode); e.set_params(p); e.set_state(lk, ps)
        for b in range(B): e.set_noise(7, b + 1, b)
        for _ in range(3): e.forward(60, 10, checkpoint=True)
        e.sync()
        a, c = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st)
        for _ in range(5): e.forward(60, 10, checkpoint=True)
        c.record(st); torch.cuda.synchronize()
        print(f"B={B} mode={mode} -> {e.last_schedule}: {a.elapsed_time(c)/5:.3f} ms", flush=True)
        del e
