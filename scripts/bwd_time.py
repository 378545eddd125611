"""Event-timed reverse sweep (C4 shape) vs its phase profile."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25068_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8; T = 60
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b + 1, b)
ids = np.array([j for j in range(sc.n_links) if j % 5], np.int32)
e.set_loss_mse(ids, np.zeros((T // sc.steps_per_interval, len(ids))))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(4):
    e.forward(T, sc.steps_per_interval, checkpoint=True)
    torch.cuda.synchronize()
    ev[0].record(st); e.gradient_device_loss(); ev[1].record(st)
    torch.cuda.synchronize()
    print("gradient_device_loss ms", ev[0].elapsed_time(ev[1]))
e.forward(T, sc.steps_per_interval, checkpoint=True)
e.gradient_device_loss(); e.sync()
ph, g = e.profile_backward()
print("phases sum us/step", sum(ph.values()), "x T =", sum(ph.values()) * T / 1e3, "ms", ph)
