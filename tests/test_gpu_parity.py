"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Forward: bit-exact per-step cumulative counts, link assignments and fp64
positions.  Gradients: normwise per block <= 1e-9.
"""
import numpy as np
import pytest

from conftest import normwise

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-9


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def port_of(port, sc, **kw):
    from oracle.oracle import PortScenario

    f, t, ln, _ = sc.links()
    lk, ps = sc.seed_agents()
    return PortScenario(port, f, t, ln, link0=lk, pos0=ps, delta_n=sc.delta_n, tau=sc.tau,
                        horizon_steps=sc.horizon_steps, obs_interval_s=sc.obs_interval_s,
                        gumbel_tau=getattr(sc, "gumbel_tau", 0.01),
                        tg=getattr(sc, "trajectory_grafting", True), **kw)


def assert_forward_equal(tr, ref, states=False):
    assert np.array_equal(tr.cum_per_step, ref["cum_per_step"])
    assert np.array_equal(tr.link_final, ref["link"])
    assert np.array_equal(tr.pos_final, ref["pos"])
    if states:
        assert np.array_equal(tr.states_link, ref["states_link"])
        assert np.array_equal(tr.states_pos, ref["states_pos"])


def test_c1_forward_every_step_bit_exact(port):
    """C1: 4x4 grid, 1,000 vehicles, 30 min — every step's state bit-exact."""
    from oracle.oracle import fnv1a64

    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 1800, 300)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7, record_states=True)
    ref = port_of(port, sc).forward(p, 7, 0, record_states=True)
    assert_forward_equal(tr, ref, states=True)
    # SURVEY.md §8c C1 trajectory KAT (measured on the reference build)
    assert tr.cum_final.sum() == 10427
    assert fnv1a64(tr.link_final, tr.pos_final) == 0xAD430DFDF1F897B8
    assert fnv1a64(tr.cum_per_step) == 0x1871BDF9FF357BC5


@pytest.mark.parametrize("tg", [True, False])
def test_c1_gradient_all_blocks(port, tg):
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 900, 300, trajectory_grafting=tg)
    p = sc.sample_parameters(3)
    rng = np.random.default_rng(5)
    K, L, N = sc.n_snapshots, sc.n_links, sc.n_agents
    ws, qs, wc, wx = rng.normal(size=(K, L)), rng.normal(size=(K, L)), rng.normal(size=L), rng.normal(size=N)
    g = P.simulate_gradient(sc, p, seed=7, ws=ws, qs=qs, wc=wc, wx=wx, noise_iteration=3)
    r = port_of(port, sc).gradient(p, 7, 3, ws=ws, qs=qs, wc=wc, wx=wx)
    assert g.loss == pytest.approx(r["loss"], rel=1e-12)
    assert np.array_equal(g.snapshots, r["snapshots"])
    assert np.array_equal(g.cum_final, r["cum_final"])
    for b in range(5):
        assert normwise(g.grads[b], r["grads"][b]) <= GRAD_TOL, b


def test_batched_draws_equal_single_runs(port):
    """B scenarios in one device pass == B separate runs (draw independence)."""
    sc = P.Scenario.grid(5, 350.0, 9, 1000.0).configure(2000, 2, 300, 300)
    p = sc.sample_parameters(4)
    its = [1, 2, 3, 4, 5, 6, 7, 8]
    trs = P.simulate_forward(sc, p, seed=11, noise_iterations=its)
    pr = port_of(port, sc)
    for it, tr in zip(its, trs):
        assert_forward_equal(tr, pr.forward(p, 11, it))
    rng = np.random.default_rng(1)
    wc = rng.normal(size=sc.n_links)
    gs = P.simulate_gradient(sc, p, seed=11, wc=wc, noise_iterations=its)
    for it, g in zip(its, gs):
        r = pr.gradient(p, 11, it, wc=wc)
        for b in range(5):
            assert normwise(g.grads[b], r["grads"][b]) <= GRAD_TOL


def test_c3_forward_chicago_scale(port):
    """C3: 23x23 grid (2,553 links), 1,000,020 vehicles, dn=30, 1 h."""
    from oracle.oracle import fnv1a64

    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7)
    ref = port_of(port, sc).forward(p, 7, 0)
    assert_forward_equal(tr, ref)
    # SURVEY.md §8c C3 forward KAT (reference build, 574.9 s on one core)
    assert tr.cum_final.sum() == 38158
    assert fnv1a64(tr.link_final, tr.pos_final) == 0x5573A3F14223BBBA


def test_c3_dn1_million_agents(port):
    """C3 at dn=1: 1,000,020 agents (the stress variant of SURVEY.md §8d), 12
    steps bit-exact against the C oracle; every layout conserves all agents
    (the kernel's conservation check raises otherwise)."""
    T = 12
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 1, T, 300)
    assert sc.n_agents == 1000020
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7)
    ref = port_of(port, sc).forward(p, 7, 0)
    assert_forward_equal(tr, ref)


def test_context_reuse_state_and_param_caching(port):
    """Scenarios sharing a cached device context (same network, agent count and
    config) and alternating parameter sets: every call must see its own
    initial state and parameters (the upload cache keys on both)."""
    seeded = P.Scenario.grid(3, 300.0, 42, 600.0).configure(300, 1, 90, 30, fit_queues=False)
    lk, ps = seeded.seed_agents()
    rng = np.random.default_rng(0)
    ps2 = np.minimum(ps, rng.uniform(0.0, 1.0, size=len(ps)) * 300.0)
    a = P.Scenario.grid(3, 300.0, 42, 600.0).configure(0, 1, 90, 30, fit_queues=False, custom_init=(lk, ps))
    b = P.Scenario.grid(3, 300.0, 42, 600.0).configure(0, 1, 90, 30, fit_queues=False, custom_init=(lk, ps2))
    assert np.array_equal(a.links()[2], b.links()[2])  # same network -> one shared device context
    p1 = a.sample_parameters(3)
    p2 = a.sample_parameters(4)
    ref = {}
    for name, sc in (("a", a), ("b", b)):
        for pn, p in (("1", p1), ("2", p2)):
            ref[name + pn] = port_of(port, sc).forward(p, 7, 0)
    for key in ("a1", "b1", "a2", "b2", "a1", "a2", "b2", "b1"):
        sc = a if key[0] == "a" else b
        p = p1 if key[1] == "1" else p2
        assert_forward_equal(P.simulate_forward(sc, p, seed=7), ref[key])
    assert a.device_context() == b.device_context()  # the cache really was shared
    # reconfiguring a scenario (new initial state) invalidates what the context holds
    a.configure(0, 1, 90, 30, fit_queues=False, custom_init=(lk, ps2))
    assert_forward_equal(P.simulate_forward(a, p1, seed=7), ref["b1"])


def test_c3_dn1_gradient_short(port):
    """Reverse sweep at 1,000,020 agents (dn=1) over 6 steps: the cum_final and
    final-position loss gradients against the C oracle (normwise 1e-9)."""
    T = 6
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 1, T, 300)
    p = sc.sample_parameters(3)
    rng = np.random.default_rng(11)
    wc = rng.normal(size=sc.n_links)
    wx = rng.normal(size=sc.n_agents)
    g = P.simulate_gradient(sc, p, seed=7, wc=wc, wx=wx)
    r = port_of(port, sc).gradient(p, 7, 0, wc=wc, wx=wx)
    assert abs(g.loss - r["loss"]) <= 1e-9 * max(1.0, abs(r["loss"]))
    for blk in range(5):
        assert normwise(g.grads[blk], r["grads"][blk]) <= GRAD_TOL


@pytest.mark.parametrize("n_draws", [3, 160])
def test_streamed_readback_matches_plain_reads(n_draws):
    """dtg_simulate_forward streams count rows back while the kernel runs
    (dtg_forward_read: progress counter in the persistent schedules, a plain
    post-run copy in the step-graph schedule B > resident grid uses); the
    results equal dtg_forward + dtg_read_cum_all / dtg_read_state."""
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 90, 300)
    p = sc.sample_parameters(3)
    its = list(range(10, 10 + n_draws))
    trs = P.simulate_forward(sc, p, seed=7, noise_iterations=its)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, n_draws, 90)
    e.set_params(p)
    e.set_state(lk, ps)
    for b, it in enumerate(its):
        e.set_noise(7, it, b)
    e.forward(90, sc.steps_per_interval)
    cum = e.read_cum_all()
    for b, tr in enumerate(trs):
        assert np.array_equal(tr.cum_per_step, cum[b])
        lk_b, ps_b = e.read_state(b, -1)
        assert np.array_equal(tr.link_final, lk_b) and np.array_equal(tr.pos_final, ps_b)
