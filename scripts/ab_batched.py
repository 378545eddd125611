"""A/B of the batched step graph and the C4 reverse sweep between the in-tree
library and another build: ab_batched.py [path/to/libdtg.so]."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_25068_b200 import _lib
if len(sys.argv) > 1:
    _lib.load_other(sys.argv[1])
import paper_2603_25068_b200 as P

S0 = torch.cuda.Stream()
torch.cuda.set_stream(S0)
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
for B, mode in ((64, 0), (256, 0)):
    e = P.Engine(sc, B, 120); e.set_stream(torch.cuda.current_stream().cuda_stream); e.set_mode(mode)
    e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, 1000 + b, b)
    for _ in range(2): e.forward(120, 10)
    e.sync()
    st = torch.cuda.current_stream(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st)
    for _ in range(3): e.forward(120, 10)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    ker, _ = e.profile_kernels(120, 10)
    print(f"B={B} mode={mode}: {ms:.2f} ms/batch  kernels(ms/nowcast): " + " ".join(f"{k}={v:.2f}" for k, v in ker.items()))
    del e
sc4 = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 60, 300)
e = P.Engine(sc4, 8, 60); st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
e.set_params(p); e.set_state(lk, ps)
for b in range(8): e.set_noise(7, b + 1, b)
ids = np.array([j for j in range(sc4.n_links) if j % 5], np.int32)
e.set_loss_mse(ids, np.zeros((6, len(ids))))
ev = [torch.cuda.Event(True) for _ in range(3)]
f, a = [], []
for _ in range(4):
    ev[0].record(st); e.forward(60, 10, checkpoint=True); ev[1].record(st); e.gradient_device_loss(); ev[2].record(st)
    torch.cuda.synchronize(); f.append(ev[0].elapsed_time(ev[1])); a.append(ev[1].elapsed_time(ev[2]))
print(f"C4 B=8: fwd_ckpt {np.median(f[1:]):.3f} ms  adjoint {np.median(a[1:]):.3f} ms  phases {e.profile_backward()[0] if hasattr(e,'profile_backward') else ''}")
