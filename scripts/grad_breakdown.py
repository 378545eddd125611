import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25068_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = 60
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(0, True); lk, ps = sc.seed_agents()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
e = P.Engine(sc, B, T); e.set_stream(s.cuda_stream); e.set_params(p); e.set_state(lk, ps)
for b in range(B): e.set_noise(7, b + 1, b)
K = T // 10; L = sc.n_links
seeds = torch.randn(B, K, L, dtype=torch.float64, device='cuda')
grads = torch.empty(B, 5, L, dtype=torch.float64, device='cuda')
def fwd(): e.forward(T, 10, checkpoint=True)
def bwd(): e.backward_device(seeds.data_ptr(), 0, 0, grads.data_ptr())
for f in (fwd, bwd, fwd, bwd): f()
torch.cuda.synchronize()
def timeit(f, n=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(s); f(); b.record(s)
    torch.cuda.synchronize()
    return np.mean([a.elapsed_time(b) for a, b in ev])
print(f"B={B} fwd(ckpt) {timeit(fwd):.3f} ms")
fwd()
print(f"B={B} bwd       {timeit(bwd):.3f} ms  (persistent reverse sweep)")
e.set_mode(3); fwd(); print(f"B={B} bwd graph {timeit(bwd):.3f} ms  (8-kernel graph)"); e.set_mode(0)
fwd(); e.sync()
t = time.perf_counter()
for _ in range(10):
    cum = e.read_cum_all()
rc = (time.perf_counter() - t) / 10 * 1e3
print(f"read_cum x{B}: {rc:.3f} ms")
seeds_h = np.random.default_rng(0).normal(size=(B, K, L))
t = time.perf_counter()
for _ in range(5):
    fwd(); e.backward(snap_seeds=seeds_h)
print(f"fwd+bwd host API: {(time.perf_counter() - t) / 5 * 1e3:.3f} ms")
fwd(); e.sync()
ph, g = e.profile_backward()
print("reverse phases per step (us):", {k: round(v, 2) for k, v in ph.items()}, "grid", g, "sum", round(sum(ph.values()), 2))
