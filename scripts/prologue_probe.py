import os, sys, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2603_25068_b200 as P
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, 1, 120); e.set_params(p); e.set_state(lk, ps); e.set_noise(7, 0)
e.forward(120, 10); e.sync()
lib = P.load(); nw = C.c_int()
lib.dtg_debug_warp_records(e._h, 120, 10, None, C.byref(nw))
out = np.zeros((120, nw.value, 4), np.uint64)
lib.dtg_debug_warp_records(e._h, 120, 10, out.ctypes.data_as(C.c_void_p), C.byref(nw))
o = out[1:].astype(np.int64)
print("loads+compute (start->after sync) us", ((o[:, :, 2] - o[:, :, 0]) / 1e3).mean(), "max-per-step", ((o[:, :, 2] - o[:, :, 0]) / 1e3).max(1).mean())
print("scan us", ((o[:, :, 3] - o[:, :, 2]) / 1e3).mean())
print("after scan -> loop start us", ((o[:, :, 1] - o[:, :, 3]) / 1e3).mean())
