"""C3 1-h nowcast (B=1) device time and step phases, in-tree library vs
another build: ab_fwd.py [path/to/libdtg.so]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_25068_b200 import _lib
if len(sys.argv) > 1:
    _lib.load_other(sys.argv[1])
import paper_2603_25068_b200 as P

st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, 1, 120); e.set_stream(st.cuda_stream); e.set_params(p); e.set_state(lk, ps); e.set_noise(7, 0, 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5): e.forward(120, 10)
e.sync()
ts = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(st); e.forward(120, 10); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort()
ph, g = e.profile_persistent(120, 10)
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'in-tree'}: median {ts[10]:.4f} ms min {ts[0]:.4f}  "
      + " ".join(f"{k}={v:.2f}" for k, v in ph.items()))
