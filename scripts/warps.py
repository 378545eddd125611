import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
DN = int(sys.argv[2]) if len(sys.argv) > 2 else 30
T = int(sys.argv[3]) if len(sys.argv) > 3 else 120
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, DN, T, 300)
SPI = sc.steps_per_interval
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b, b)
e.forward(T, SPI); e.sync()
lib = P.load(); nw = C.c_int()
lib.dtg_debug_warp_records(e._h, T, SPI, None, C.byref(nw))
out = np.zeros((T, nw.value, 4), np.uint64)
rc = lib.dtg_debug_warp_records(e._h, T, SPI, out.ctypes.data_as(C.c_void_p), C.byref(nw)); assert rc == 0, lib.dtg_last_error(e._h)
o = out[1:].astype(np.int64)
start = o[:, :, 0].min(axis=1, keepdims=True)
pro = (o[:, :, 1] - o[:, :, 0]) / 1e3
loop = (o[:, :, 2] - o[:, :, 1]) / 1e3
endrel = (o[:, :, 2] - start) / 1e3
na = o[:, :, 3]
print(f"B={B} warps={nw.value}", flush=True)
print(f"prologue per warp: mean {pro.mean():.2f} max-per-step mean {pro.max(1).mean():.2f} us")
print(f"slot loop per warp: mean {loop.mean():.2f}, max-per-step mean {loop.max(1).mean():.2f} us")
print(f"warp end rel. to earliest start: max-per-step mean {endrel.max(1).mean():.2f} us")
print(f"start skew across warps: mean {((o[:, :, 0] - start) / 1e3).max(1).mean():.2f} us")
for k in range(8):
    m = na == k
    if m.any(): print(f"  warps with {k} arrived: n={m.sum():6d} loop mean {loop[m].mean():.2f} max {loop[m].max():.2f} us")
m = na >= 8
if m.any(): print(f"  warps with >=8 arrived: n={m.sum()} loop mean {loop[m].mean():.2f} max {loop[m].max():.2f}")
