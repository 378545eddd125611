import sys, os, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2603_25068_b200 as P
lib = P.load()
f = lib._lib if hasattr(lib, '_lib') else lib
fn = C.CDLL(P._lib.LIB_PATH).dtg_debug_head_clocks
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, 1, 120); e.set_params(p); e.set_state(lk, ps); e.set_noise(7, 0, 0)
e.forward(120, 10); e.sync()
out = (C.c_ulonglong * 8)()
fn(out)
e.forward(120, 10); e.sync()
fn(out)

n = out[5]; print("heads", n, "cyc/head: loads", out[0] / n, "draws", out[1] / n, "argmax", out[2] / n, "merge draw", out[3] / n, "atomic+store", out[4] / n)
