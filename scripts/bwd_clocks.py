import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
fn = C.CDLL(P._lib.LIB_PATH).dtg_debug_bwd_clocks
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8; T = 60
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b + 1, b)
ids = np.array([j for j in range(sc.n_links) if j % 5], np.int32)
e.set_loss_mse(ids, np.zeros((T // sc.steps_per_interval, len(ids))))
out = (C.c_ulonglong * 8)()
e.forward(T, sc.steps_per_interval, checkpoint=True); e.gradient_device_loss(); e.sync(); fn(out)
e.forward(T, sc.steps_per_interval, checkpoint=True); e.gradient_device_loss(); e.sync(); fn(out)
n = out[3]
print("warps", n, "cycles/warp: link loop", out[0] / n, "epilogue", out[1] / n, "links/warp", out[2] / n)
