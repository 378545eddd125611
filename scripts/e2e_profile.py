"""Where the e2e C-ABI call's time goes beyond the kernel (C3, B=1): the
level-2 call, and the level-1 steps it is made of, host-timed."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_25068_b200 import _lib
if len(sys.argv) > 1:  # another build (scripts/build_variants.sh)
    _lib.load_other(sys.argv[1])
import paper_2603_25068_b200 as P
from paper_2603_25068_b200._lib import ptr

sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
p = sc.sample_parameters(3); p2 = P.LinkParams(p.u * 1.001, p.kappa, p.beta, p.alpha, p.cost)
T, L, N = 120, sc.n_links, sc.n_agents
lib = P.load()
for i in range(5): P.simulate_forward(sc, p if i % 2 else p2, seed=7, noise_iterations=[i])
def tm(f, n=40):
    ts = []
    for i in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); f(i); ts.append(time.perf_counter() - t)
    ts.sort(); return ts[n // 2] * 1e3
print(f"level-2 simulate_forward (python API): {tm(lambda i: P.simulate_forward(sc, p if i % 2 else p2, seed=7, noise_iterations=[i])):.3f} ms")
cum = np.empty((1, T, L)); lk = np.empty((1, N), np.int32); ps = np.empty((1, N)); wall = np.zeros(1)
its = np.zeros(1, np.uint64)
def l2(i):
    its[0] = i; q = p if i % 2 else p2
    sc._check(lib.dtg_simulate_forward(sc._h, *q.arrays(), 7, 1, its, ptr(cum), ptr(lk), ptr(ps), None, None, ptr(wall)))
print(f"level-2 C call, reused arrays: {tm(l2):.3f} ms")
outs = (P.pinned_empty((1, T, L)), P.pinned_empty((1, N), np.int32), P.pinned_empty((1, N)))
print(f"level-2 simulate_forward, pinned out=: {tm(lambda i: P.simulate_forward(sc, p if i % 2 else p2, seed=7, noise_iterations=[i], out=outs)):.3f} ms")
def l2p(i):
    its[0] = i; q = p if i % 2 else p2
    sc._check(lib.dtg_simulate_forward(sc._h, *q.arrays(), 7, 1, its, ptr(outs[0]), ptr(outs[1]), ptr(outs[2]), None, None, ptr(wall)))
print(f"level-2 C call, pinned arrays: {tm(l2p):.3f} ms")
ctx = sc.device_context()
pa = [a.copy() for a in p.arrays()]; pb = [a.copy() for a in p2.arrays()]
def l1_params(i):
    q = pa if i % 2 else pb
    lib.dtg_set_params(ctx, -1, *q); lib.dtg_sync(ctx)
print(f"  dtg_set_params: {tm(l1_params):.3f} ms")
def l1_fwd(i):
    lib.dtg_set_noise(ctx, -1, 7, i); lib.dtg_forward(ctx, T, 10, 0); lib.dtg_sync(ctx)
print(f"  dtg_forward + sync (no read-back): {tm(l1_fwd):.3f} ms")
def l1_fwd_read(i):
    lib.dtg_set_noise(ctx, -1, 7, i); lib.dtg_forward_read(ctx, T, 10, 0, ptr(cum), ptr(lk), ptr(ps))
print(f"  dtg_forward_read (cum + final state): {tm(l1_fwd_read):.3f} ms")
def l1_fwd_read_cum(i):
    lib.dtg_set_noise(ctx, -1, 7, i); lib.dtg_forward_read(ctx, T, 10, 0, ptr(cum), None, None)
print(f"  dtg_forward_read (cum only): {tm(l1_fwd_read_cum):.3f} ms")
st = torch.cuda.Stream(); lib.dtg_set_stream(ctx, C.c_void_p(st.cuda_stream))
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
ds = []
for i in range(20):
    lib.dtg_set_noise(ctx, -1, 7, i); e0.record(st); lib.dtg_forward(ctx, T, 10, 0); e1.record(st); torch.cuda.synchronize(); ds.append(e0.elapsed_time(e1))
ds.sort(); print(f"  device (events around dtg_forward, warm L2): {ds[10]:.3f} ms")
lib.dtg_set_stream(ctx, None)
