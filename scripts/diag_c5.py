"""Diagnose C5 (optimize_control at C3 scale): per-draw cost gradients of
iteration 0, device vs port, and where the Adam steps they produce differ."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_25068_b200 as P
from oracle.oracle import PortLib, PortScenario, Params
from oracle import optim

T = 180
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
cal = sc.sample_parameters(3)
kinds = sc.links()[3]
tr = P.simulate_forward(sc, cal, seed=7)
phys = [j for j in range(sc.n_links) if kinds[j] == 0]
target = max(phys, key=lambda j: tr.cum_final[j])
desired = 0.5 * float(tr.cum_final[target]) * 30
f, t, ln, _ = sc.links()
lk, ps = sc.seed_agents()
pr = PortScenario(PortLib(), f, t, ln, link0=lk, pos0=ps, delta_n=30, horizon_steps=T, obs_interval_s=300)
L, N = sc.n_links, sc.n_agents
its = list(range(1, 9))
eng = P.Engine(sc, 8, T)
st = torch.cuda.Stream(); eng.set_stream(st.cuda_stream)
eng.set_params(cal); eng.set_state(lk, ps)
for b, it in enumerate(its): eng.set_noise(7, it, b)
eng.forward(T, sc.steps_per_interval, checkpoint=True)
eng.set_loss_control(target, desired)
rows = torch.zeros((8, 5 * L + 2), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
eng.gradient_device_loss(rows.data_ptr()); st.synchronize()
r = rows.cpu().numpy()
for b, it in enumerate(its):
    fw = pr.forward(cal, 7, it)
    c = float(fw["cum_per_step"][-1, target])
    dd = c * 30 + (-desired)
    cs = np.zeros(L); cs[target] = ((0.0 + dd) + dd) * 30
    g = pr.gradient_seeds(cal, 7, it, np.zeros((T // 10, L)), cs, np.zeros(N))
    gd = r[b, :5 * L].reshape(5, L)
    for q, nm in enumerate("u kappa beta alpha cost".split()):
        a, e = gd[q], g[q]
        den = np.abs(e).max()
        zd = ((a == 0) != (e == 0)).sum()
        sg = (np.sign(a) != np.sign(e)).sum()
        big = np.abs(e) > 1e-8
        print(f"draw {b} {nm}: max|ref| {den:.3e} normwise {np.abs(a-e).max()/max(den,1e-300):.2e} "
              f"zero-pattern diffs {zd} sign diffs {sg} (|ref|>1e-8: {big.sum()}, sign diffs there {(np.sign(a)!=np.sign(e))[big].sum()}) "
              f"loss dev {r[b,5*L]} port {dd*dd}")
    # where signs differ, magnitudes
    a, e = gd[4], g[4]
    idx = np.nonzero(np.sign(a) != np.sign(e))[0][:10]
    print("  cost sign diffs:", [(int(i), a[i], e[i]) for i in idx])
