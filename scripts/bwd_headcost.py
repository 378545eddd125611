"""Upper bound of removing R1's head replays: reverse sweep with and without
them (dtg_set_flag 2 = 1 skips the replays; results invalid, timing only)."""
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
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for dbg in (0, 1, 0, 1):
    e.set_flag(2, dbg)
    e.forward(T, sc.steps_per_interval, checkpoint=True); e.gradient_device_loss(); torch.cuda.synchronize()
    e.forward(T, sc.steps_per_interval, checkpoint=True)
    torch.cuda.synchronize()
    ev[0].record(st); e.gradient_device_loss(); ev[1].record(st)
    torch.cuda.synchronize()
    e.forward(T, sc.steps_per_interval, checkpoint=True)
    ph, g = e.profile_backward()
    print(f"dbg={dbg} sweep ms {ev[0].elapsed_time(ev[1]):.3f}  phases", {k: round(v, 2) for k, v in ph.items()}, flush=True)
e.set_flag(2, 0)
