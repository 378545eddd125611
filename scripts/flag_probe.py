"""Forward us/step and bit-equality for values of one engine flag: flag_probe.py FLAG v1,v2,..."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25068_b200 as P
flag = int(sys.argv[1]); vals = [int(v) for v in sys.argv[2].split(",")]
for dn, T, B in ((30, 120, 1), (30, 120, 8), (1, 600, 1)):
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, dn, T, 300)
    p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b, b)
    st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
    ref = None
    out = []
    for v in vals:
        e.set_flag(flag, v)
        e.forward(T, sc.steps_per_interval); e.sync()
        cum = e.read_cum_all()
        if ref is None: ref = cum
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(5):
            ev[0].record(st); e.forward(T, sc.steps_per_interval); ev[1].record(st); torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        out.append(f"v={v}: {1000 * float(np.median(ts)) / T:.2f} us/step same={np.array_equal(cum, ref)}")
    print(f"dn{dn} B{B}: " + " | ".join(out), flush=True)
