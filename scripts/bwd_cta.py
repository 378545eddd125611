"""Per-CTA spans of the reverse-sweep phases (C4, B=8): imbalance analysis."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
B = 8; T = 60
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b + 1, b)
ids = np.array([j for j in range(sc.n_links) if j % 5], np.int32)
e.set_loss_mse(ids, np.zeros((T // sc.steps_per_interval, len(ids))))
e.forward(T, sc.steps_per_interval, checkpoint=True); e.gradient_device_loss(); e.sync()
e.forward(T, sc.steps_per_interval, checkpoint=True)
ph, g = e.profile_backward()
print("phases", {k: round(v, 2) for k, v in ph.items()})
lib = P.load(); G = C.c_int()
lib.dtg_debug_bwd_stamps(e._h, None, C.byref(G))
s = np.zeros((T, G.value, 8), np.uint64)
lib.dtg_debug_bwd_stamps(e._h, s.ctypes.data_as(C.c_void_p), C.byref(G))
s = s.astype(np.int64)[1:T - 1]
names = ["R1", "R2", "R3", "R4"]
for i, nm in enumerate(names):
    d = (s[:, :, 2 * i + 1] - s[:, :, 2 * i]) / 1e3  # per CTA span of phase i
    start_skew = (s[:, :, 2 * i] - s[:, :, 2 * i].min(1, keepdims=True)) / 1e3
    per_cta = d.mean(0)
    sc_mean = per_cta.reshape(B, -1).mean(1)
    print(f"{nm}: per-CTA span mean {d.mean():.2f} max/step {d.max(1).mean():.2f} us; start skew max {start_skew.max(1).mean():.2f}; "
          f"by scenario {np.round(sc_mean, 2)}; slowest CTA ranks {np.argsort(-per_cta)[:6]}")
