"""Developer check: first divergence of the GPU path vs the C oracle, timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
from oracle.oracle import PortLib, PortScenario

port = PortLib()

def port_of(sc):
    f, t, ln, _ = sc.links(); lk, ps = sc.seed_agents()
    return PortScenario(port, f, t, ln, link0=lk, pos0=ps, delta_n=sc.delta_n, horizon_steps=sc.horizon_steps,
                        obs_interval_s=sc.obs_interval_s)

def check(name, n, ln, seed, veh, dn, T, grad=True):
    sc = P.Scenario.grid(n, ln, seed, 1000.0).configure(veh, dn, T, 300)
    p = sc.sample_parameters(3)
    t0 = time.time(); tr = P.simulate_forward(sc, p, seed=7, record_states=True); t1 = time.time()
    pr = port_of(sc); ref = pr.forward(p, 7, 0, record_states=True); t2 = time.time()
    bad = np.where((tr.states_link != ref['states_link']).any(1) | (tr.states_pos != ref['states_pos']).any(1))[0]
    print(f"{name}: gpu {t1-t0:.3f}s port {t2-t1:.3f}s; bad steps {len(bad)} first {bad[:3]}", flush=True)
    if len(bad):
        t = bad[0]
        d = np.where((tr.states_link[t] != ref['states_link'][t]) | (tr.states_pos[t] != ref['states_pos'][t]))[0]
        print('  agents', d[:10], tr.states_link[t][d[:5]], ref['states_link'][t][d[:5]], tr.states_pos[t][d[:5]], ref['states_pos'][t][d[:5]])
    print('  cum equal', np.array_equal(tr.cum_per_step, ref['cum_per_step']))
    if grad:
        rng = np.random.default_rng(5)
        K, L, N = sc.n_snapshots, sc.n_links, sc.n_agents
        ws, qs, wc, wx = rng.normal(size=(K, L)), rng.normal(size=(K, L)), rng.normal(size=L), rng.normal(size=N)
        t0 = time.time(); g = P.simulate_gradient(sc, p, seed=7, ws=ws, qs=qs, wc=wc, wx=wx); t1 = time.time()
        r = pr.gradient(p, 7, 0, ws=ws, qs=qs, wc=wc, wx=wx); t2 = time.time()
        print(f"  grad gpu {t1-t0:.3f}s port {t2-t1:.3f}s loss {g.loss} {r['loss']}")
        for b, nm in enumerate('u kappa beta alpha cost'.split()):
            den = np.abs(r['grads'][b]).max()
            print(f"   {nm}: normwise {np.abs(g.grads[b]-r['grads'][b]).max()/max(den,1e-300):.3e} (|ref|max {den:.3e})")

check('C1', 4, 400.0, 42, 1000, 1, 1800)
check('C3', 23, 1609.34, 42, 1000020, 30, 120)
