"""Batched C3 nowcast (dn=30, 120 steps): ms per batch of the step graph
(mode 3) vs scenario-resident CTAs (mode 4) vs the fused grid (mode 2) per B,
and bit-equality of mode 4 against mode 3: scn_time.py [B ...]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_25068_b200 import _lib
if os.environ.get("DTG_LIB"):  # another build (scripts/build_variants.sh)
    _lib.load_other(os.environ["DTG_LIB"])
import paper_2603_25068_b200 as P
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
Bs = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64, 128, 256]
for B in Bs:
    res, cums = {}, {}
    for mode in (2, 3, 4):
        if mode == 2 and B > 148:
            continue
        e = P.Engine(sc, B, 120); e.set_stream(st.cuda_stream); e.set_mode(mode)
        e.set_params(p); e.set_state(lk, ps)
        for b in range(B): e.set_noise(7, 1000 + b, b)
        for _ in range(2): e.forward(120, 10)
        e.sync()
        a, c = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st)
        for _ in range(3): e.forward(120, 10)
        c.record(st); torch.cuda.synchronize()
        res[mode] = a.elapsed_time(c) / 3
        cums[mode] = [e.read_cum(b) for b in (0, B - 1)]
        del e
    same = all(np.array_equal(x, y) for x, y in zip(cums[3], cums[4]))
    print(f"B={B}: " + "  ".join(f"mode{m} {v:.2f} ms" for m, v in res.items()) + f"  mode4==mode3 {same}", flush=True)
for B in (8, 128, 256):
    e = P.Engine(sc, B, 120); e.set_stream(st.cuda_stream)
    e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, 1000 + b, b)
    e.forward(120, 10); e.sync()
    print(f"B={B} mode4 phases (us/step): " + " ".join(f"{k}={v:.1f}" for k, v in e.profile_scn(120, 10).items()), flush=True)
    del e
