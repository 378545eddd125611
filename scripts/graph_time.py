"""Forward timing on C3 (dn=30, 120 steps) at B scenarios in the auto (0) and
step-graph (3) schedules, plus the graph's per-kernel split:
graph_time.py B [B ...]; DTG_SPLIT=k sets the graph's scenario branches (flag 8)."""
import os
import sys

sys.path.insert(0, os.environ.get("DTG_VARIANT_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_25068_b200 as P

sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3)
lk, ps = sc.seed_agents()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for B, mode in ((int(a), m) for a in sys.argv[1:] for m in (0, 3)):
    e = P.Engine(sc, B, 120)
    e.set_stream(stream.cuda_stream)
    e.set_params(p)
    e.set_state(lk, ps)
    e.set_mode(mode)
    e.set_flag(8, int(os.environ.get("DTG_SPLIT", "0")))
    for b in range(B):
        e.set_noise(7, 1000 + b, b)
    for _ in range(2):
        e.forward(120, 10)
    e.sync()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(3):
        e.forward(120, 10)
    z.record(stream)
    torch.cuda.synchronize()
    ker, n = e.profile_kernels(120, 10) if mode == 3 else ({}, 0)
    print(f"B={B} mode={e.last_mode} ms/nowcast={a.elapsed_time(z) / 3:.3f} kernels(ms)=",
          {k: round(v, 3) for k, v in ker.items()}, flush=True)
    del e
