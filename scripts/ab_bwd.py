"""C4 reverse sweep (8 draws, 60 steps) device time and phase split, in-tree
library vs another build: ab_bwd.py [path/to/libdtg.so]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_25068_b200 import _lib
if len(sys.argv) > 1:
    _lib.load_other(sys.argv[1])
import paper_2603_25068_b200 as P

sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 60, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, 8, 60); st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
DBG = int(os.environ.get("BWD_DBG", "0"))  # timing experiments only (skips work; results invalid)
e.set_params(p); e.set_state(lk, ps)
for b in range(8): e.set_noise(7, b + 1, b)
ids = np.array([j for j in range(sc.n_links) if j % 5], np.int32)
e.set_loss_mse(ids, np.zeros((6, len(ids))))
ev = [torch.cuda.Event(True) for _ in range(3)]
f, a = [], []
for _ in range(8):
    ev[0].record(st); e.forward(60, 10, checkpoint=True); ev[1].record(st); e.gradient_device_loss(); ev[2].record(st)
    torch.cuda.synchronize(); f.append(ev[0].elapsed_time(ev[1])); a.append(ev[1].elapsed_time(ev[2]))
e.forward(60, 10, checkpoint=True)
if DBG:
    e.set_flag(2, DBG)
ph = e.profile_backward()[0]
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'in-tree'} dbg={DBG}: fwd_ckpt {np.median(f[2:]):.3f} ms  adjoint {np.median(a[2:]):.3f} ms  "
      + " ".join(f"{k}={v:.2f}" for k, v in ph.items()))
