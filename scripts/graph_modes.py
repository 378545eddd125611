"""Batched C3 (B=256, step graph): per-nowcast time with graphs / branches on and off."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_25068_b200 as P
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for graphs, branches in ((1, 0), (1, 1), (0, 1), (0, 0)):
    e = P.Engine(sc, B, 120); e.set_stream(st.cuda_stream); e.set_mode(3)
    e.set_graphs(bool(graphs)); e.set_flag(8, branches)
    e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, 1000 + b, b)
    for _ in range(2): e.forward(120, 10)
    e.sync()
    a, c = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(st)
    for _ in range(3): e.forward(120, 10)
    c.record(st); torch.cuda.synchronize()
    print(f"B={B} graphs={graphs} branches={branches or 'auto'}: {a.elapsed_time(c)/3:.2f} ms per nowcast, launches {e._lib.dtg_last_launches(e._h)}")
    del e
