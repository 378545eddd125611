"""Forward us/step for the fused kernel's slot mappings (flag 1) at dn30/dn1."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25068_b200 as P
res = {}
for dn, T, B in ((30, 120, 1), (1, 600, 1), (30, 120, 8)):
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, dn, T, 300)
    p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
    for b in range(B): e.set_noise(7, b, b)
    st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
    ref = None
    for m in (-1, 0, 1):
        e.set_flag(1, m)
        e.forward(T, sc.steps_per_interval); e.sync()
        cum = e.read_cum_all()
        if ref is None: ref = cum
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(5):
            ev[0].record(st); e.forward(T, sc.steps_per_interval); ev[1].record(st); torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        res[f"dn{dn}_B{B}_map{m}"] = dict(us_per_step=1000 * float(np.median(ts)) / T, same=bool(np.array_equal(cum, ref)))
print(json.dumps(res, indent=1))
