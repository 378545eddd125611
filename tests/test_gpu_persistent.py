"""The cluster-per-scenario kernel, the persistent cooperative grid kernel and
the 5-kernel step graph are three schedules of the same arithmetic: results must be bit-identical, in all
three grid-assignment modes (several CTAs per scenario, capped CTAs per
scenario, several scenarios per CTA)."""
import numpy as np
import pytest

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(sc, p, B, mode, T, spi, ckpt=True):
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T)
    e.set_mode(mode)
    e.set_params(p)
    e.set_state(lk, ps)
    for b in range(B):
        e.set_noise(7, 100 + b, b)
    e.forward(T, spi, checkpoint=ckpt)
    cum = np.stack([e.read_cum(b) for b in range(B)])
    fin = [e.read_state(b, T) for b in range(B)]
    mid = [e.read_state(b, T // 2) for b in range(B)] if ckpt else None
    return cum, fin, mid


@pytest.mark.parametrize("n,length,veh,dn,T,B", [
    (4, 400.0, 1000, 1, 600, 1),
    (6, 300.0, 2400, 2, 300, 5),
    (23, 1609.34, 1000020, 30, 120, 8),
    (4, 400.0, 1000, 1, 200, 300),  # more scenarios than resident CTAs -> scenario loop
    (4, 400.0, 1000, 1, 100, 37),   # step graph in 4 uneven scenario branches (9, 9, 9, 10)
    (50, 400.0, 100000, 1, 60, 1),  # C2: 12,300 links -> lean layout (per-link arrays in global memory)
    (4, 400.0, 1001, 1, 200, 3),    # odd agent count: scalar slot mapping
])
def test_persistent_equals_step_graph(n, length, veh, dn, T, B):
    sc = P.Scenario.grid(n, length, 42, 1000.0).configure(veh, dn, T, 300 if dn <= 2 else 30 * dn * 10)
    p = sc.sample_parameters(3)
    spi = sc.steps_per_interval
    ref = run(sc, p, B, 3, T, spi)  # 5-kernel step graph
    for mode in (1, 2, 4):        # cluster per scenario, persistent grid, scenario-resident CTAs
        a = run(sc, p, B, mode, T, spi)
        assert np.array_equal(a[0], ref[0]), mode
        for x, y in zip(a[1], ref[1]):
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]), mode
        for x, y in zip(a[2], ref[2]):
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]), mode


@pytest.mark.parametrize("n,length,veh,dn,T,B,tg", [
    (4, 400.0, 1000, 1, 600, 2, True),
    (4, 400.0, 1000, 1, 300, 1, False),
    (6, 300.0, 2400, 2, 300, 3, True),
    (23, 1609.34, 1000020, 30, 60, 8, True),
    (4, 400.0, 1000, 1, 100, 300, True),  # scenario loop in the persistent reverse sweep
])
def test_persistent_backward_equals_step_graph(n, length, veh, dn, T, B, tg):
    sc = P.Scenario.grid(n, length, 42, 1000.0).configure(veh, dn, T, 300 if dn <= 2 else 300,
                                                        trajectory_grafting=tg)
    p = sc.sample_parameters(3)
    spi = sc.steps_per_interval
    K = T // spi
    lk, ps = sc.seed_agents()
    rng = np.random.default_rng(4)
    snap = rng.normal(size=(B, K, sc.n_links))
    cum = rng.normal(size=(B, sc.n_links))
    xs = rng.normal(size=(B, sc.n_agents))
    out = []
    for mode in (0, 3):
        e = P.Engine(sc, B, T)
        e.set_mode(mode)
        e.set_params(p)
        e.set_state(lk, ps)
        for b in range(B):
            e.set_noise(7, 50 + b, b)
        e.forward(T, spi, checkpoint=True)
        out.append(e.backward(snap_seeds=snap if K else None, cum_seeds=cum, x_seeds=xs))
    assert np.array_equal(out[0], out[1])


def test_dn1_full_hour_invariants_and_schedules():
    """C3 at dn=1 (1,000,020 agents) for the full hour (3,600 steps) — sizes the
    oracle cannot run: cumulative counts never decrease, every agent ends on a
    valid link inside it, reruns are bit-identical, and the fused grid kernel
    equals the 5-kernel step graph over the first 300 steps."""
    sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 1, 3600, 300)
    p = sc.sample_parameters(3)
    a = P.simulate_forward(sc, p, seed=7)
    b = P.simulate_forward(sc, p, seed=7)
    assert np.array_equal(a.cum_per_step, b.cum_per_step) and np.array_equal(a.pos_final, b.pos_final)
    assert (np.diff(a.cum_per_step, axis=0) >= 0).all() and (a.cum_per_step >= 0).all()
    _, _, length, _ = sc.links()
    assert a.link_final.min() >= 0 and a.link_final.max() < sc.n_links
    assert (a.pos_final >= -1e-2).all() and (a.pos_final <= length[a.link_final]).all()
    assert len(a.link_final) == 1000020
    T = 300
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, 1, T)
    e.set_params(p)
    e.set_state(lk, ps)
    e.set_noise(7, 0)
    out = []
    for mode in (2, 3):
        e.set_mode(mode)
        e.forward(T, 300)
        out.append((e.read_cum_all(), e.read_state(0, -1)))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1][0], out[1][1][0]) and np.array_equal(out[0][1][1], out[1][1][1])


@pytest.mark.parametrize("n,length,veh,dn,T,B,mode", [
    (4, 400.0, 1000, 1, 600, 1, 2),
    (23, 1609.34, 1000020, 30, 120, 1, 2),
    (23, 1609.34, 1000020, 30, 120, 1, 1),
    (23, 1609.34, 1000020, 1, 40, 1, 2),
])
def test_speculative_head_decisions_are_exact(n, length, veh, dn, T, B, mode):
    """Heads whose decision was drawn one step ahead in the link phase
    (dtg_set_flag 4, CView::spec) give the same trajectory bit for bit as
    heads drawing in the slot phase."""
    sc = P.Scenario.grid(n, length, 42, 1000.0).configure(veh, dn, T, 300)
    p = sc.sample_parameters(3)
    lk, ps = sc.seed_agents()
    out = []
    for spec, split in ((1, 1), (1, 0), (0, 0)):  # barrier-1 warps, link-phase lanes, off
        e = P.Engine(sc, B, T)
        e.set_mode(mode)
        e.set_flag(4, spec)
        e.set_flag(5, split)
        e.set_params(p)
        e.set_state(lk, ps)
        e.set_noise(7, 5, 0)
        e.forward(T, sc.steps_per_interval, checkpoint=True)
        out.append((e.read_cum(0), e.read_state(0, T), e.read_state(0, T // 2)))
    for o in out[1:]:
        assert np.array_equal(out[0][0], o[0])
        for a, b in zip(out[0][1:], o[1:]):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_mode_toggles_on_one_engine_keep_backward_exact():
    """One context, reverse sweeps alternating between the step graph (mode 3)
    and the persistent kernel (mode 0, and after a scenario-resident forward,
    mode 4): the persistent sweep grows the shared vbar buffer, which the
    cached step-graph sweep captured, so the graph must be rebuilt (ADVICE r1:
    stale vbar pointer in bwd_exec)."""
    sc = P.Scenario.grid(6, 300.0, 42, 1000.0).configure(2400, 2, 120, 300)
    p = sc.sample_parameters(3)
    spi, T, B = sc.steps_per_interval, 120, 3
    lk, ps = sc.seed_agents()
    rng = np.random.default_rng(11)
    snap = rng.normal(size=(B, T // spi, sc.n_links))
    xs = rng.normal(size=(B, sc.n_agents))
    e = P.Engine(sc, B, T)
    e.set_params(p)
    e.set_state(lk, ps)
    for b in range(B):
        e.set_noise(7, 40 + b, b)
    got = []
    for mode in (3, 0, 3, 4, 0, 3):
        e.set_mode(mode)
        e.forward(T, spi, checkpoint=True)
        got.append(e.backward(snap_seeds=snap, x_seeds=xs))
    for g in got[1:]:
        assert np.array_equal(g, got[0])


@pytest.mark.parametrize("B", [1, 3])
def test_pinned_result_buffers_equal_pageable(B):
    """simulate_forward(out=pinned_empty(...)): results DMA'd straight into
    page-locked buffers equal the pageable (staged) read-back, call after call
    with the buffers reused."""
    sc = P.Scenario.grid(6, 800.0, 42, 1000.0).configure(18000, 30, 60, 300)
    p = sc.sample_parameters(3)
    T, L, N = sc.horizon_steps, sc.n_links, sc.n_agents
    outs = (P.pinned_empty((B, T, L)), P.pinned_empty((B, N), np.int32), P.pinned_empty((B, N)))
    for call in range(3):
        its = [call * 10 + b for b in range(B)]
        want = P.simulate_forward(sc, p, seed=7, noise_iterations=its)
        got = P.simulate_forward(sc, p, seed=7, noise_iterations=its, out=outs)
        for b in range(B):
            assert np.shares_memory(got[b].cum_per_step, outs[0])  # views of the caller's buffers
            assert np.array_equal(got[b].cum_per_step, want[b].cum_per_step)
            assert np.array_equal(got[b].link_final, want[b].link_final)
            assert np.array_equal(got[b].pos_final, want[b].pos_final)
    with pytest.raises(ValueError):
        P.simulate_forward(sc, p, seed=7, noise_iterations=list(range(B + 1)), out=outs)


def test_scenario_resident_falls_back_when_link_state_exceeds_shared_memory():
    """C2's 12,300 links do not fit one CTA's shared memory: an explicit
    mode 4 runs the step graph instead, with the same results."""
    sc = P.Scenario.grid(50, 400.0, 42, 1000.0).configure(100000, 1, 20, 300)
    p = sc.sample_parameters(3)
    out = []
    for mode in (4, 3):
        e = P.Engine(sc, 2, 20)
        e.set_mode(mode)
        e.set_params(p)
        lk, ps = sc.seed_agents()
        e.set_state(lk, ps)
        for b in range(2):
            e.set_noise(7, b, b)
        e.forward(20, 20)
        assert e.last_mode // 1000 == 3
        out.append([e.read_cum(b) for b in range(2)])
    assert all(np.array_equal(x, y) for x, y in zip(*out))
