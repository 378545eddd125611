"""GPU parity at the BASELINE configurations' full sizes and on the reference's
own Sioux Falls network ("Next round" item 1).

Oracles:
* reference-build fixtures (tests/golden/make_golden_r2.py: c4_draw1,
  c2_dn25_forward, c2_dn25_gradient, sf_dn4, sf_dn1) — the unmodified
  reference's own outputs;
* the C port (oracle/dtsim_port.c), itself pinned bit-exact to the reference,
  where the reference is too slow (all 8 C4 draws, C2 at dn=1) or runs out of
  int indexing (N x L >= 2^31);
* oracle/optim.py (the calibrate / optimize_control loops over the port).

Bars: link ids, positions, counts, snapshots bit-exact;
gradients normwise <= 1e-9 per block; losses 1e-12 relative.
"""
import os

import numpy as np
import pytest

from conftest import normwise
from golden_cases import GOLDEN, load

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-9
LOSS_RTOL = 1e-12


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _need(name):
    if not os.path.exists(os.path.join(GOLDEN, name + ".npz")):
        pytest.skip(f"fixture {name} not generated (tests/golden/make_golden_r2.py)")
    return load(name)


def port_of(port, sc, T=None):
    from oracle.oracle import PortScenario

    f, t, ln, _ = sc.links()
    lk, ps = sc.seed_agents()
    return PortScenario(port, f, t, ln, link0=lk, pos0=ps, delta_n=sc.delta_n, tau=sc.tau,
                        horizon_steps=sc.horizon_steps if T is None else T, obs_interval_s=sc.obs_interval_s,
                        gumbel_tau=getattr(sc, "gumbel_tau", 0.01), tg=getattr(sc, "trajectory_grafting", True))


def events_of(link0, states_link):
    """(step, agent, from, to) of every link change, as make_golden_r2 derives
    them from the reference's record_states."""
    rows = []
    prev = link0
    for t in range(states_link.shape[0]):
        cur = states_link[t]
        (idx,) = np.nonzero(cur != prev)
        rows += [(t, a, prev[a], cur[a]) for a in idx]
        prev = cur
    return np.array(rows, np.int32).reshape(-1, 4)


def grads_close(got, want, tol=GRAD_TOL):
    for b in range(5):
        err = normwise(got[b], want[b])
        assert err <= tol, f"gradient block {b}: normwise {err:.3e}"


# ---- C4: the calibration the bench times ------------------------------------------
C4_T, C4_DRAWS = 60, 8


def _c4():
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, C4_T, 300)
    truth = sc.sample_parameters(42)
    L = sc.n_links
    obs_ids = np.array([j for j in range(L) if j % 5 != 0], np.int32)
    tr = P.simulate_forward(sc, truth, seed=7)
    obs = tr.cum_per_step[9::10][:, obs_ids] * 30.0
    return sc, truth, obs_ids, obs, tr


def _mid(L):
    mid = lambda lo, hi: np.full(L, lo + (hi - lo) * 0.5)  # BoundedTransform::value(0)
    return P.LinkParams(mid(13.9, 22.2), mid(0.18, 0.22), mid(0.0, 5.0), mid(0.01, 5.0), np.ones(L))


def test_c4_observations_and_first_draw_match_reference():
    """bench.py's C4 inputs (truth run -> observations) and the gradient of
    iteration 0, draw 0 (noise_iteration 1) against the reference build."""
    from oracle.oracle import fnv1a64_c

    d = _need("c4_draw1")
    sc, truth, obs_ids, obs, tr = _c4()
    assert np.array_equal(np.stack(truth.arrays()), d["truth"])
    assert fnv1a64_c(tr.cum_per_step) == int(d["truth_fnv_cum"])
    assert np.array_equal(obs_ids, d["obs_ids"]) and np.array_equal(obs, d["obs"])
    p = _mid(sc.n_links)
    assert np.array_equal(np.stack(p.arrays()), d["params"])
    loss, grads = P.simulate_gradient_mse(sc, p, 7, obs_ids, obs, noise_iterations=[1])
    assert loss[0] == pytest.approx(float(d["loss"]), rel=LOSS_RTOL)
    grads_close(grads[0], d["grads"])


def test_c4_all_eight_draws_against_port(port):
    """All 8 draws of a C4 iteration, batched on the device as the bench runs
    them, each against the port's gradient with the same MSE seeds."""
    from oracle.optim import mse_loss

    sc, truth, obs_ids, obs, _ = _c4()
    p = _mid(sc.n_links)
    its = list(range(1, C4_DRAWS + 1))
    loss, grads = P.simulate_gradient_mse(sc, p, 7, obs_ids, obs, noise_iterations=its)
    pr = port_of(port, sc)
    L = sc.n_links
    for b, it in enumerate(its):
        fw = pr.forward(p, 7, it)
        snaps = fw["cum_per_step"][9::10]
        lv, seeds = mse_loss(snaps, obs_ids, obs, 30)
        g = pr.gradient_seeds(p, 7, it, seeds, np.zeros(L), np.zeros(pr.N))
        assert loss[b] == pytest.approx(lv, rel=LOSS_RTOL), b
        grads_close(grads[b], g)


def test_c4_calibrate_three_iterations_against_optim_oracle(port):
    """calibrate() exactly as bench.py runs it (8 draws, MSE, AdamW from the
    range midpoints), 3 iterations, against oracle/optim.py over the port."""
    from oracle import optim
    from oracle.oracle import Params

    sc, truth, obs_ids, obs, _ = _c4()
    cfg = P.OptimizeConfig(max_iterations=3, patience=10 ** 6, noise_draws=C4_DRAWS)
    res = P.calibrate(sc, obs_ids, obs, 7, cfg=cfg)
    ref = optim.calibrate(port_of(port, sc), obs_ids, obs, 7,
                          cfg=dict(max_iterations=3, patience=10 ** 6, noise_draws=C4_DRAWS), params_cls=Params)
    np.testing.assert_allclose(res.loss_curve, ref["loss_curve"], rtol=LOSS_RTOL, atol=0)
    assert res.best_iteration == ref["best_iteration"]
    np.testing.assert_allclose(np.stack(res.best_params.arrays()), np.stack(ref["best"].arrays()), rtol=1e-9, atol=0)


# ---- C5: control at C3 scale ------------------------------------------------------------
def test_c5_control_three_iterations_against_optim_oracle(port):
    """optimize_control on the C3 net, 90-min horizon (180 steps), 8 draws,
    target = busiest physical link of the uncontrolled run, desired = half
    (bench.py run_control), 3 iterations against oracle/optim.py."""
    from oracle import optim
    from oracle.oracle import Params

    T = 180
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
    cal = sc.sample_parameters(3)
    kinds = sc.links()[3]
    tr = P.simulate_forward(sc, cal, seed=7)
    pr = port_of(port, sc)
    ref_tr = pr.forward(cal, 7, 0)
    assert np.array_equal(tr.cum_per_step, ref_tr["cum_per_step"])
    phys = [j for j in range(sc.n_links) if kinds[j] == 0]
    target = max(phys, key=lambda j: tr.cum_final[j])
    desired = 0.5 * float(tr.cum_final[target]) * 30
    cfg = dict(max_iterations=3, patience=10 ** 6, noise_draws=8)
    res = P.optimize_control(sc, cal, target, desired, 7, cfg=P.OptimizeConfig(**cfg))
    ref = optim.optimize_control(pr, Params(*cal.arrays()), target, desired, 7, cfg=cfg, params_cls=Params)
    np.testing.assert_allclose(res.loss_curve, ref["loss_curve"], rtol=LOSS_RTOL, atol=0)
    np.testing.assert_allclose(res.cost, ref["cost"], rtol=1e-9, atol=0)
    assert res.achieved == pytest.approx(ref["achieved"], rel=LOSS_RTOL)


# ---- C2: 50x50 grid, 12,300 links -------------------------------------------------------
def _c2(dn, T):
    return P.Scenario.grid(50, 400.0, 42, 1000.0).configure(100000, dn, T, 300)


def test_c2_dn25_full_horizon_forward_against_reference():
    from oracle.oracle import fnv1a64_c

    d = _need("c2_dn25_forward")
    sc = _c2(25, 144)
    f, t, ln, k = sc.links()
    assert np.array_equal(f, d["frm"]) and np.array_equal(ln, d["length"]) and np.array_equal(k, d["kind"])
    p = sc.sample_parameters(3)
    assert np.array_equal(np.stack(p.arrays()), d["params"])
    tr = P.simulate_forward(sc, p, seed=7)
    assert np.array_equal(tr.cum_per_step[11::12], d["cum_snap"])
    assert np.array_equal(tr.link_final, d["link"]) and np.array_equal(tr.pos_final, d["pos"])
    assert fnv1a64_c(tr.cum_per_step) == int(d["fnv_cum"])
    assert fnv1a64_c(tr.link_final, tr.pos_final) == int(d["fnv_state"])


def test_c2_dn25_full_horizon_gradient_against_reference():
    d = _need("c2_dn25_gradient")
    sc = _c2(25, 144)
    p = sc.sample_parameters(3)
    L = sc.n_links
    k = np.arange(12)[:, None]
    j = np.arange(L)[None, :]
    ws = (((7 * j + 13 * k) % 11) - 5) / 4.0
    g = P.simulate_gradient(sc, p, seed=7, ws=ws, wc=d["loss_wc"], noise_iteration=int(d["noise"]))
    assert g.loss == pytest.approx(float(d["loss"]), rel=LOSS_RTOL)
    assert np.array_equal(g.snapshots, d["snapshots"]) and np.array_equal(g.cum_final, d["cum_final"])
    assert np.array_equal(g.link_final, d["link"]) and np.array_equal(g.pos_final, d["pos"])
    grads_close(g.grads, d["grads"])


def test_c2_dn1_full_hour_forward_against_port(port):
    """C2 as the bench runs it (dn=1: 100,000 agents, 3,600 steps), the whole
    hour against the port: every step's counts and the final state."""
    from oracle.oracle import fnv1a64_c

    sc = _c2(1, 3600)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7)
    ref = port_of(port, sc).forward(p, 7, 0)
    assert fnv1a64_c(tr.cum_per_step) == fnv1a64_c(ref["cum_per_step"])
    assert np.array_equal(tr.cum_per_step[299::300], ref["cum_per_step"][299::300])
    assert np.array_equal(tr.link_final, ref["link"]) and np.array_equal(tr.pos_final, ref["pos"])


def test_c2_dn1_300_step_gradient_against_port(port):
    sc = _c2(1, 300)
    p = sc.sample_parameters(3)
    rng = np.random.default_rng(2)
    L, N = sc.n_links, sc.n_agents
    ws, wc, wx = rng.normal(size=(1, L)), rng.normal(size=L), rng.normal(size=N)
    g = P.simulate_gradient(sc, p, seed=7, ws=ws, wc=wc, wx=wx, noise_iteration=4)
    r = port_of(port, sc).gradient(p, 7, 4, ws=ws, wc=wc, wx=wx)
    assert g.loss == pytest.approx(r["loss"], rel=LOSS_RTOL)
    assert np.array_equal(g.cum_final, r["cum_final"])
    grads_close(g.grads, r["grads"])


# ---- Sioux Falls: the reference's own network ---------------------------------------------
def sf_scenario(d, T):
    dn = int(d["meta"][4])
    sc = P.Scenario.from_links(int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"])
    sc.configure(2000, dn, T, 300, fit_queues=False)
    lk, ps = sc.seed_agents()
    assert np.array_equal(lk, d["link0"]) and np.array_equal(ps, d["pos0"])
    return sc


@pytest.mark.parametrize("dn", [4, 1])
def test_sioux_falls_forward_against_reference(dn):
    """configs/siouxfalls.toml's network and demand, the full 90-min horizon:
    every step's state (hash over all record_states), counts, and every
    agent's link changes (travel-time events) bit-exact."""
    from oracle.oracle import fnv1a64_c

    d = _need(f"sf_dn{dn}")
    T = int(d["meta"][2])
    sc = sf_scenario(d, T)
    p = P.LinkParams(*d["params"])
    tr = P.simulate_forward(sc, p, seed=42, record_states=True)
    spi = 300 // dn
    assert np.array_equal(tr.cum_per_step[spi - 1::spi], d["cum_snap"])
    assert fnv1a64_c(tr.cum_per_step) == int(d["fnv_cum"])
    assert np.array_equal(tr.link_final, d["link"]) and np.array_equal(tr.pos_final, d["pos"])
    assert fnv1a64_c(tr.states_link, tr.states_pos) == int(d["fnv_states"])
    assert np.array_equal(events_of(d["link0"], tr.states_link), d["events"])


@pytest.mark.parametrize("dn", [4, 1])
def test_sioux_falls_scenario_resident_forward_against_reference(dn):
    """The scenario-resident schedule (mode 4, one CTA per scenario) on the
    reference's own irregular network: counts and final state bit-exact."""
    from oracle.oracle import fnv1a64_c

    d = _need(f"sf_dn{dn}")
    T = int(d["meta"][2])
    sc = sf_scenario(d, T)
    p = P.LinkParams(*d["params"])
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, 1, T)
    e.set_mode(4)
    e.set_params(p)
    e.set_state(lk, ps)
    e.set_noise(42, 0, 0)
    e.forward(T, 300 // dn)
    assert e.last_mode // 1000 == 4
    cum = e.read_cum(0)
    assert fnv1a64_c(cum) == int(d["fnv_cum"])
    fl, fp = e.read_state(0, T)
    assert np.array_equal(fl, d["link"]) and np.array_equal(fp, d["pos"])


@pytest.mark.parametrize("dn", [4, 1])
def test_sioux_falls_gradient_against_reference(dn):
    """The calibration loss (mse_loss_builder over the physical links) on
    Sioux Falls over the 30-min observation window."""
    d = _need(f"sf_dn{dn}")
    sc = sf_scenario(d, int(d["T_grad"]))
    p = P.LinkParams(*d["params"])
    loss, grads = P.simulate_gradient_mse(sc, p, 42, d["obs_ids"], d["obs"], noise_iterations=[1])
    assert loss[0] == pytest.approx(float(d["loss"]), rel=LOSS_RTOL)
    grads_close(grads[0], d["grads"])


# ---- travel times: transfer events from the device merge -----------------------------------
def test_c1_transfer_events_against_reference():
    """Every agent's link changes over the C1 half hour, recorded by the
    device merge (record_transfers), against the changes in the reference's
    record_states (tests/golden/c1_travel.npz)."""
    d = _need("c1_travel")
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 1800, 300)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7, record_transfers=True)
    assert np.array_equal(tr.transfers, d["events"])
    lk0, _ = sc.seed_agents()
    assert np.array_equal(lk0, d["link0"])
    visits = P.link_visits(lk0, tr.transfers)
    done = visits[visits[:, 3] >= 0]
    assert len(done) == len(d["events"])  # every transfer closes one visit
    assert (done[:, 3] > done[:, 2]).all()


@pytest.mark.parametrize("dn", [4, 1])
def test_sioux_falls_transfer_events_against_reference(dn):
    d = _need(f"sf_dn{dn}")
    sc = sf_scenario(d, int(d["meta"][2]))
    tr = P.simulate_forward(sc, P.LinkParams(*d["params"]), seed=42, record_transfers=True)
    assert np.array_equal(tr.transfers, d["events"])


@pytest.mark.parametrize("mode", [0, 1, 3, 4])
def test_c3_transfer_events_every_schedule_against_port(port, mode):
    """C3 (1,000,020 vehicles, dn=30, 1 h), 8 draws batched: the recorded
    events equal the link changes of the port's per-step states, on the fused
    grid, the cluster, the step-graph and the scenario-resident schedules."""
    T, B = 120, 8
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
    p = sc.sample_parameters(3)
    lk0, ps0 = sc.seed_agents()
    e = P.Engine(sc, B, T)
    e.set_mode(mode)
    e.set_params(p)
    e.set_state(lk0, ps0)
    for b in range(B):
        e.set_noise(7, b, b)
    P.load().dtg_set_record_transfers(e._h, 1)
    e.forward(T, sc.steps_per_interval)
    pr = port_of(port, sc)
    for b in (0, B - 1):
        ref = pr.forward(p, 7, b, record_states=True)
        assert np.array_equal(P.transfer_events(e._h, b), events_of(lk0, ref["states_link"]))


# ---- C3 at the stress sizes ------------------------------------------------------------------
def test_c3_dn1_300_steps_against_port(port):
    """C3 at dn=1 (1,000,020 agents), 300 steps (5 min) of every step's counts
    and the final state against the port (the reference cannot hold N x L =
    2.55e9 cells)."""
    from oracle.oracle import fnv1a64_c

    T = 300
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 1, T, 300)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7)
    ref = port_of(port, sc).forward(p, 7, 0)
    assert fnv1a64_c(tr.cum_per_step) == fnv1a64_c(ref["cum_per_step"])
    assert np.array_equal(tr.link_final, ref["link"]) and np.array_equal(tr.pos_final, ref["pos"])


@pytest.mark.parametrize("B", [64, 256])
def test_c3_batched_nowcast_draws_against_port(port, B):
    """The batched throughput configuration (B independent C3 nowcasts in one
    pass: the step graph at B=64, scenario-resident CTAs at B=256) — first,
    middle and last draw against the port."""
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
    p = sc.sample_parameters(3)
    its = [1000 + b for b in range(B)]
    trs = P.simulate_forward(sc, p, seed=7, noise_iterations=its)
    pr = port_of(port, sc)
    for b in (0, B // 2, B - 1):
        ref = pr.forward(p, 7, its[b])
        assert np.array_equal(trs[b].cum_per_step, ref["cum_per_step"]), b
        assert np.array_equal(trs[b].link_final, ref["link"]) and np.array_equal(trs[b].pos_final, ref["pos"]), b
