"""The device path's input contract at its limits: a link with
more than 16 successors is rejected when the context is built; a merge row
with more than 16 candidates in one step is rejected by the persistent
kernels (16 register / shared-memory candidate slots) and handled by the step
graph and the scenario-resident schedule (32), whose results must equal the C
port's."""
import numpy as np
import pytest

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _params(L):
    rng = np.random.default_rng(5)
    return P.LinkParams(rng.uniform(13.9, 22.2, L), rng.uniform(0.18, 0.22, L), rng.uniform(0.0, 5.0, L),
                        rng.uniform(0.01, 5.0, L), np.ones(L))


def test_out_degree_above_16_is_rejected():
    k = 17  # link 0 ends at node 0, which has 17 outgoing links
    frm = [100] + [0] * k + list(range(1, k + 1))
    to = [0] + list(range(1, k + 1)) + [200 + i for i in range(k)]
    kind = [1] + [0] * k + [2] * k
    sc = P.Scenario.from_links(300, frm, to, [400.0] * len(frm), kind)
    sc.configure(0, 1, 5, 5, fit_queues=False, custom_init=([0], [10.0]))
    with pytest.raises(P.UnsupportedError, match="out-degree"):
        P.simulate_forward(sc, _params(len(frm)), seed=3)


def _merge17():
    """17 links into node 0, one agent at the end of each, a single link out."""
    k = 17
    frm = list(range(1, k + 1)) + [0, 50]
    to = [0] * k + [50, 60]
    kind = [0] * k + [0, 2]
    length = [200.0] * k + [300.0, 5000.0]
    link0 = list(range(k))
    pos0 = [200.0] * k  # arrived (x1 >= L - 0.01 after one step)
    return frm, to, length, kind, link0, pos0


def test_merge_with_17_candidates(port):
    from oracle.oracle import PortScenario

    frm, to, length, kind, link0, pos0 = _merge17()
    L = len(frm)
    p = _params(L)
    T = 3
    sc = P.Scenario.from_links(61, frm, to, length, kind)
    sc.configure(0, 1, T, 1, fit_queues=False, custom_init=(link0, pos0))
    lk, ps = sc.seed_agents()
    # persistent kernels (16 candidate slots): refused, not approximated
    e = P.Engine(sc, 1, T)
    e.set_mode(2)
    e.set_params(p)
    e.set_state(lk, ps)
    e.set_noise(7, 0, 0)
    with pytest.raises(P.UnsupportedError, match="candidates"):
        e.forward(T, 1)
        e.sync()
    # step graph and scenario-resident CTAs (32 slots): exact, against the port
    ref = PortScenario(port, frm, to, length, link0=lk, pos0=ps, horizon_steps=T, obs_interval_s=1).forward(p, 7, 0)
    for mode in (3, 4):
        e = P.Engine(sc, 1, T)
        e.set_mode(mode)
        e.set_params(p)
        e.set_state(lk, ps)
        e.set_noise(7, 0, 0)
        e.forward(T, 1, checkpoint=True)
        assert e.last_mode // 1000 == mode
        cum = e.read_cum(0)
        fl, fp = e.read_state(0, T)
        assert np.array_equal(cum, ref["cum_per_step"]), mode
        assert np.array_equal(fl, ref["link"]) and np.array_equal(fp, ref["pos"]), mode
        assert 1 <= (fl == L - 2).sum() <= T  # at most one admission into the merge link per step
