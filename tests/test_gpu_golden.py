"""GPU path vs the reference's own recorded outputs (tests/golden, made by the
reference build) and vs the C oracle on cases the fixtures do not cover.
All calls go through the C-ABI (libdtg.so)."""
import numpy as np
import pytest

from conftest import normwise
from golden_cases import TRAJ_CASES, load, loss_kwargs, meta, params_of, product_scenario

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
GRAD_TOL = 1e-9


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", TRAJ_CASES)
def test_forward_matches_reference_fixture(name):
    d = load(name)
    m = meta(d)
    sc = product_scenario(P, d)
    states = "states_link" in d
    tr = P.simulate_forward(sc, params_of(d, P.LinkParams), seed=m["seed"], noise_iteration=m["noise"],
                            record_states=states)
    assert np.array_equal(tr.link_final, d["link"])
    assert np.array_equal(tr.pos_final, d["pos"])
    assert np.array_equal(tr.cum_final, d["cum_final"])
    if "cum_per_step" in d:
        assert np.array_equal(tr.cum_per_step, d["cum_per_step"])
    if states:
        assert np.array_equal(tr.states_link, d["states_link"])
        assert np.array_equal(tr.states_pos, d["states_pos"])


@pytest.mark.parametrize("name", [n for n in TRAJ_CASES if n != "c1_forward"])
def test_gradient_matches_reference_fixture(name):
    d = load(name)
    m = meta(d)
    sc = product_scenario(P, d)
    g = P.simulate_gradient(sc, params_of(d, P.LinkParams), seed=m["seed"], noise_iteration=m["noise"],
                            **loss_kwargs(d))
    assert g.loss == pytest.approx(float(d["loss"]), rel=1e-12, abs=1e-12)
    assert np.array_equal(g.snapshots, d["snapshots"])
    for b in range(5):
        assert normwise(g.grads[b], d["grads"][b]) <= GRAD_TOL, (b, normwise(g.grads[b], d["grads"][b]))


def test_calibration_mse_gradient_matches_reference():
    d = load("c1_mse")
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 600, 300)
    loss, grads = P.simulate_gradient_mse(sc, P.LinkParams(*d["params"]), 7, d["obs_ids"], d["obs"],
                                          noise_iterations=[1])
    assert loss[0] == pytest.approx(float(d["loss"]), rel=1e-13)
    for b in range(5):
        assert normwise(grads[0][b], d["grads"][b]) <= GRAD_TOL


def test_chicago_scale_gradient_matches_reference():
    """C3 two-step gradient: |grad beta/alpha/cost| ~ 1e8-1e9 (SURVEY §7 hard part 1)."""
    d = load("c3_gradient_2step")
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 2, 30)
    p = sc.sample_parameters(3)
    g = P.simulate_gradient(sc, p, seed=7, ws=d["loss_ws"], wx=d["loss_wx"])
    assert np.array_equal(g.link_final, d["link"]) and np.array_equal(g.pos_final, d["pos"])
    assert g.loss == pytest.approx(float(d["loss"]), rel=1e-12)
    for b in range(5):
        assert normwise(g.grads[b], d["grads"][b]) <= GRAD_TOL


def test_device_gumbel_vs_glibc(port):
    """The Gumbel draws are exact integer arithmetic up to two logs, and the
    device's logs are glibc's (csrc/dtg_libm.h): every draw is bit-identical to
    the port's (glibc) -log(-log u) — no tolerance, no mismatch budget."""
    rng = np.random.default_rng(0)
    n = 1 << 20
    rows = rng.integers(0, 2**40, n, dtype=np.uint64)
    cols = rng.integers(0, 2**20, n, dtype=np.uint64)
    out = np.zeros(n)
    assert P.load().dtg_debug_gumbel(12345, 77, n, rows, cols, out) == 0
    ref = np.array([port.lib.port_gumbel(12345, 77, int(r), int(c)) for r, c in zip(rows[:50000], cols[:50000])])
    assert np.array_equal(out[:50000], ref)


def test_forced_exact_path_matches_fast_path():
    """k_adj_a0's exact ordered-sum path (normally only on near ties) gives the
    same gradients as the fast argmax path."""
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 300, 300)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, 2, 300)
    e.set_params(p)
    e.set_state(lk, ps)
    e.set_noise(7, 0, 0)
    e.set_noise(7, 1, 1)
    rng = np.random.default_rng(3)
    seeds = rng.normal(size=(2, 1, sc.n_links))
    e.forward(300, 300, checkpoint=True)
    g_fast = e.backward(snap_seeds=seeds)
    e.force_slow_path(True)
    e.forward(300, 300, checkpoint=True)
    g_slow = e.backward(snap_seeds=seeds)
    assert np.array_equal(g_fast, g_slow)


def test_deterministic_and_graph_independent():
    sc = P.Scenario.grid(5, 350.0, 9, 1000.0).configure(2000, 2, 200, 300)
    p = sc.sample_parameters(4)
    lk, ps = sc.seed_agents()
    outs = []
    for graphs in (True, True, False):
        e = P.Engine(sc, 3, 200)
        e.set_graphs(graphs)
        e.set_params(p)
        e.set_state(lk, ps)
        for b in range(3):
            e.set_noise(11, b, b)
        e.forward(200, 150, checkpoint=True)
        cum = [e.read_cum(b) for b in range(3)]
        g = e.backward(cum_seeds=np.ones((3, sc.n_links)))
        outs.append((cum, g))
    for cum, g in outs[1:]:
        for a, b in zip(cum, outs[0][0]):
            assert np.array_equal(a, b)
        assert np.array_equal(g, outs[0][1])


def test_zero_horizon_and_input_errors():
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 0, 300)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7)
    lk, ps = sc.seed_agents()
    assert tr.steps == 0 and np.array_equal(tr.link_final, lk) and np.array_equal(tr.pos_final, ps)
    g = P.simulate_gradient(sc, p, seed=7, wc=np.ones(sc.n_links))
    assert np.all(g.grads == 0)
    bad = P.Scenario.from_links(2, [0], [1], [100.0], [0]).configure(
        0, 1, 5, 1, fit_queues=False, custom_init=([0], [-0.5]))
    with pytest.raises(P.UnsupportedError):
        P.simulate_forward(bad, P.LinkParams(*[np.ones(1)] * 5), seed=1)
    bad2 = P.Scenario.from_links(2, [0], [1], [100.0], [0]).configure(
        0, 1, 5, 1, fit_queues=False, custom_init=([3], [1.0]))
    with pytest.raises(P.DtgError, match="does not exist"):
        P.simulate_forward(bad2, P.LinkParams(*[np.ones(1)] * 5), seed=1)
    with pytest.raises(P.DtgError, match="multiple of the time step"):
        sc7 = P.Scenario.grid(3, 200.0, 1, 1000.0).configure(30, 1, 10, 0)
        P.simulate_forward(sc7, sc7.sample_parameters(1), seed=1)


@pytest.mark.slow
def test_stress_dn1_million_agents(port):
    """C3 stress variant: dn = 1, 1,000,020 agents, 60 steps (1 simulated
    minute) bit-exact against the oracle, plus size-independent invariants."""
    from oracle.oracle import PortScenario

    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 1, 60, 60)
    p = sc.sample_parameters(3)
    tr = P.simulate_forward(sc, p, seed=7)
    f, t, ln, _ = sc.links()
    lk, ps = sc.seed_agents()
    ref = PortScenario(port, f, t, ln, link0=lk, pos0=ps, horizon_steps=60, obs_interval_s=60).forward(p, 7, 0)
    assert np.array_equal(tr.cum_per_step, ref["cum_per_step"])
    assert np.array_equal(tr.link_final, ref["link"]) and np.array_equal(tr.pos_final, ref["pos"])
    # invariants: conservation, monotone cumulative counts, positions within links
    assert len(tr.link_final) == 1000020
    assert np.all(np.diff(tr.cum_per_step, axis=0) >= 0)
    assert np.all(tr.pos_final >= -0.01) and np.all(tr.pos_final <= ln[tr.link_final])


def test_sharded_gradient_world1_equals_per_draw_sum():
    """dist.ShardedGradient (the multi-GPU calibration path, here one rank)
    == the ordered sum of per-draw simulate_gradient results."""
    from paper_2603_25068_b200.dist import ShardedGradient, calibration_draws

    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 300, 60)
    p = sc.sample_parameters(3)
    L = sc.n_links
    rng = np.random.default_rng(9)
    ws = rng.normal(size=(5, L))

    def seeds_fn(snaps, cum_final):
        loss = (snaps * ws[None]).sum(axis=(1, 2))
        return loss, np.broadcast_to(ws, snaps.shape).copy(), None

    its = calibration_draws(3, 4)
    loss, gsum, rows = ShardedGradient(sc, 4)(p, 7, its, seeds_fn)
    per = P.simulate_gradient(sc, p, seed=7, ws=ws, noise_iterations=its)
    seq = per[0].grads.copy()
    for g in per[1:]:
        seq += g.grads
    assert np.array_equal(gsum, seq)
    assert loss == pytest.approx(sum(g.loss for g in per) / 4, rel=1e-12)


def test_interleaved_log_equals_scalar_log():
    """The interleaved F-operand Gumbel / log of the head draws (log_sl_v,
    gumbel_sl_v) equal the scalar glibc log on every input the path produces
    (16M draws) and on 16M random positive doubles."""
    import ctypes as C
    lib = P.load()
    mism, flagged = C.c_ulonglong(), C.c_ulonglong()
    assert lib.dtg_debug_log_check(12345, 1 << 24, C.byref(mism), C.byref(flagged)) == 0
    assert mism.value == 0
    assert flagged.value == 0


@pytest.mark.parametrize("which,n", [(0, 10**8), (1, 10**8), (2, 10**8), (3, 1 << 24), (4, 1 << 24),
                                     (5, 1 << 24), (6, 1 << 24), (7, 1 << 24)])
def test_device_libm_bit_identical_to_glibc(which, n):
    """The device exp / log against this host's glibc libm (the reference's):
    10^8 Gumbel-path inputs per log kind, 16M per other kind, 0 mismatches."""
    import ctypes as C
    mism = C.c_ulonglong()
    assert P.load().dtg_debug_libm_check(which, 2024 + which, n, 1, C.byref(mism)) == 0
    assert mism.value == 0
