"""FD-validation instrumentation on the device against
the reference's own outputs (tests/golden/f4_*.npz, made by
tests/golden/make_golden_f4.py from the reference build) and the Python
restatement (oracle/fdcheck_oracle.py): BranchTrace hashes, soft choices,
surrogate record / replay, batched probes and run_gradcheck — all through the
C-ABI (libdtg.so, csrc/dtg_probe.cu)."""
import os

import numpy as np
import pytest

from conftest import normwise

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")
from paper_2603_25068_b200 import fdcheck as F  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
# Replayed counts contain the soft sigmoid sums (observation.cpp:17): libdevice
# exp vs glibc exp may differ in the last bit, nothing else does.
COUNT_ATOL = 1e-12


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def lp(a):
    return P.LinkParams(*[np.array(x, np.float64) for x in a])


def trace_scenario(d, T, dn, tg):
    sc = P.Scenario.from_links(int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"])
    return sc.configure(0, dn, T, T * dn, gumbel_tau=float(d["gumbel_tau"]), trajectory_grafting=bool(tg),
                        fit_queues=False, custom_init=(d["link0"], d["pos0"]))


def chain_scenario(d, soft=True):
    agents, steps, _, _, tg = (int(x) for x in d["meta"])
    sc = P.Scenario.from_links(int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"])
    sc.configure(agents, 1, steps, steps, trajectory_grafting=bool(tg), fit_queues=False)
    return F.set_soft_choices(sc, soft)


@pytest.mark.parametrize("name", ["f4_trace_c1", "f4_trace_g3", "f4_trace_ring2"])
def test_branch_hash_matches_reference(name):
    d = load(name)
    seed, noise, T, dn, tg = (int(x) for x in d["meta"])
    sc = trace_scenario(d, T, dn, tg)
    p = lp(d["params"])
    tr = F.simulate_forward_traced(sc, p, seed, noise, trace_branches=True)
    assert tr.branch_hash == int(d["hash"])
    assert np.array_equal(tr.cum_per_step, d["cum_per_step"])
    assert np.array_equal(tr.link_final, d["link"]) and np.array_equal(tr.pos_final, d["pos"])
    # tracing changes nothing: the fast engine gives the same trajectory
    plain = P.simulate_forward(sc, p, seed=seed, noise_iteration=noise)
    assert np.array_equal(plain.cum_per_step, d["cum_per_step"])
    # without tracing the hash is the FNV offset basis (engine.cpp:251)
    assert F.simulate_forward_traced(sc, p, seed, noise, trace_branches=False).branch_hash == F.OFFSET_BASIS


@pytest.mark.parametrize("name", ["f4_chain_a5", "f4_chain_a21", "f4_chain_notg"])
def test_soft_choices_and_surrogate_match_reference(name):
    d = load(name)
    seed = int(d["meta"][2])
    sc = chain_scenario(d)
    p = lp(d["params"])
    soft = F.simulate_forward_traced(sc, p, seed)
    assert soft.branch_hash == int(d["forward_hash_soft"])
    assert np.array_equal(soft.cum_final, d["cum_final"])
    # recording gradient run (run_gradcheck's base run, pipeline.cpp:525-531)
    tr = F.SurrogateTrace()
    F.set_surrogate(sc, tr)
    _, grads, cumf, h = F.simulate_gradient_traced(sc, p, seed, full_tape=True)
    assert h == int(d["base_hash"])
    assert np.array_equal(cumf, d["cum_final"])
    for b in range(5):
        assert normwise(grads[b], d["grads"][b]) <= 1e-9, b
    # every stencil probe replayed in ONE launch
    tr.replay = True
    probes = [lp(q) for q in d["probe_params"]]
    batch = F.probe_forward_batch(sc, probes, seed)
    base = int(d["base_hash"])
    on = d["probe_hash"] == np.uint64(base)
    assert on.sum() >= 0.8 * len(on)
    for k in range(len(probes)):
        if on[k]:
            assert batch.on_path[k] and int(batch.branch_hash[k]) == base, k
            np.testing.assert_allclose(batch.cum_final[k], d["probe_cum"][k][-1], rtol=0, atol=COUNT_ATOL)
            assert abs(batch.cum_sum[k] - d["probe_sum"][k]) <= COUNT_ATOL
        else:
            assert not batch.on_path[k] or int(batch.branch_hash[k]) != base, k
    # the single-probe API path gives the batch's results (final state exact)
    for k in np.flatnonzero(on)[:3]:
        one = F.simulate_forward_traced(sc, probes[k], seed)
        assert one.branch_hash == base
        assert np.array_equal(one.link_final, d["probe_link"][k])
        assert np.array_equal(one.pos_final, d["probe_pos"][k])
        np.testing.assert_allclose(one.cum_per_step, d["probe_cum"][k], rtol=0, atol=COUNT_ATOL)


def test_gradcheck_reports_match_reference():
    d = load("f4_gradcheck")
    for i, c in enumerate(d["cfgs"]):
        draws, steps, agents, tol, seed = int(c[0]), int(c[1]), int(c[2]), float(c[3]), int(c[4])
        rep = F.run_gradcheck(draws, steps, agents, tol, seed)
        max_rel, redraws, passed = d["report"][i]
        assert rep.redraws == int(redraws) and rep.passed == bool(passed), (c, rep)
        assert abs(rep.max_rel_err - max_rel) <= 1e-9
        np.testing.assert_allclose(rep.per_draw_max, d[f"per_draw_{i}"], atol=1e-9)


def test_gradcheck_matches_oracle_restatement(port):
    from oracle import fdcheck_oracle as O

    got = F.run_gradcheck(3, 50, 15, 1e-4, 123)
    ref = O.run_gradcheck(port, 3, 50, 15, 1e-4, 123)
    assert got.redraws == ref["redraws"] and got.passed == ref["passed"]
    np.testing.assert_allclose(got.per_draw_max, ref["per_draw_max"], atol=1e-9)


def test_branch_hash_matches_oracle_restatement_random_ring():
    """A fresh ring+chord case (not in the fixtures) against the restatement."""
    from oracle import fdcheck_oracle as O
    from oracle.oracle import csr_from_links

    d = load("ring_4")
    seed, noise, T, spi, dn, tg = (int(x) for x in d["meta"])
    sc = trace_scenario(d, T, dn, tg)
    rng = np.random.default_rng(5)
    prm = d["params"] * rng.uniform(0.9, 1.1, size=d["params"].shape)
    got = F.simulate_forward_traced(sc, lp(prm), seed + 1, noise + 3)
    so, su = csr_from_links(d["frm"], d["to"])
    ref = O.simulate((so, su, d["length"]), d["link0"], d["pos0"], prm, T, seed + 1, noise + 3, delta_n=dn,
                     tg=bool(tg), gumbel_tau=float(d["gumbel_tau"]))
    assert got.branch_hash == ref["hash"]
    assert np.array_equal(got.cum_per_step, ref["cum_per_step"])


def test_fractional_soft_choices_are_rejected():
    """A grid has multi-successor rows: relaxed choices would make the state
    fractional, which the compact device state does not represent."""
    sc = P.Scenario.grid(3, 250.0, 5, 600.0).configure(400, 1, 60, 60)
    F.set_soft_choices(sc, True)
    p = sc.sample_parameters(11)
    with pytest.raises(P.UnsupportedError):
        F.simulate_forward_traced(sc, p, 3)
    with pytest.raises(P.UnsupportedError):  # the plain entry points refuse soft choices
        P.simulate_forward(sc, p, seed=3)


def test_surrogate_contract_errors():
    d = load("f4_chain_a5")
    seed = int(d["meta"][2])
    p = lp(d["params"])
    sc = chain_scenario(d, soft=False)
    tr = F.SurrogateTrace()
    F.set_surrogate(sc, tr)
    F.simulate_forward_traced(sc, p, seed)  # recording without soft choices is fine
    tr.replay = True
    with pytest.raises(P.UnsupportedError):  # replay needs one-hot relaxed choices
        F.simulate_forward_traced(sc, p, seed)
    F.set_soft_choices(sc, True)
    with pytest.raises(P.UnsupportedError):  # no gradient of a replay
        F.simulate_gradient_traced(sc, p, seed)
    F.set_surrogate(sc, None)
    with pytest.raises(P.DtgError):  # engine.cpp:306-309: soft + Checkpointed
        F.simulate_gradient_traced(sc, p, seed, full_tape=False)
