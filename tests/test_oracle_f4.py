"""The plain-Python restatement of the FD-validation instrumentation
(oracle/fdcheck_oracle.py) against the reference-generated
fixtures tests/golden/f4_*.npz: BranchTrace hashes, surrogate record / replay
values and run_gradcheck reports — bit for bit."""
import os

import numpy as np
import pytest

from oracle import fdcheck_oracle as F
from oracle.oracle import csr_from_links

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


@pytest.mark.parametrize("name", ["f4_trace_c1", "f4_trace_g3", "f4_trace_ring2"])
def test_branch_hash_hard_choices(name):
    d = load(name)
    seed, noise, T, dn, tg = (int(x) for x in d["meta"])
    succ_off, succ = csr_from_links(d["frm"], d["to"])
    r = F.simulate((succ_off, succ, d["length"]), d["link0"], d["pos0"], d["params"], T, seed, noise,
                   delta_n=dn, tg=bool(tg), gumbel_tau=float(d["gumbel_tau"]))
    assert r["flags"] == 0
    assert np.array_equal(r["cum_per_step"], d["cum_per_step"])
    assert np.array_equal(r["link"], d["link"]) and np.array_equal(r["pos"], d["pos"])
    assert r["hash"] == int(d["hash"])


@pytest.mark.parametrize("name", ["f4_chain_a5", "f4_chain_a21", "f4_chain_notg"])
def test_surrogate_record_replay(name):
    d = load(name)
    agents, steps, seed, attempt, tg = (int(x) for x in d["meta"])
    succ_off, succ = csr_from_links(d["frm"], d["to"])
    net = (succ_off, succ, d["length"])
    link0, pos0 = F.chain_seed(d["length"], agents)
    kw = dict(soft=True, tg=bool(tg))
    soft = F.simulate(net, link0, pos0, d["params"], steps, seed, 0, **kw)
    assert soft["hash"] == int(d["forward_hash_soft"])
    assert np.array_equal(soft["cum_per_step"][-1], d["cum_final"])
    tr = F.Trace()
    rec = F.simulate(net, link0, pos0, d["params"], steps, seed, 0, sur=1, trace=tr, **kw)
    assert rec["hash"] == int(d["forward_hash_record"]) == int(d["base_hash"])
    assert np.array_equal(rec["cum_per_step"][-1], d["cum_final"])
    base = int(d["base_hash"])
    n_on = 0
    for k in range(len(d["probe_sum"])):
        r = F.simulate(net, link0, pos0, d["probe_params"][k], steps, seed, 0, sur=2, trace=tr, **kw)
        assert r["flags"] & ~F.OFF_PATH == 0
        if int(d["probe_hash"][k]) == base:
            n_on += 1
            assert r["hash"] == base and not r["flags"]
            assert np.array_equal(r["cum_per_step"], d["probe_cum"][k])
            assert np.array_equal(r["link"], d["probe_link"][k]) and np.array_equal(r["pos"], d["probe_pos"][k])
            s = 0.0
            for v in r["cum_per_step"][-1]:
                s += v
            assert s == d["probe_sum"][k]
        else:  # off the recorded control path: rejected either way
            assert r["hash"] != base or r["flags"] & F.OFF_PATH
    assert n_on >= 0.8 * len(d["probe_sum"])


def test_gradcheck_reports():
    from oracle.oracle import PortLib

    d = load("f4_gradcheck")
    for i, c in enumerate(d["cfgs"][:2]):
        draws, steps, agents, tol, seed = int(c[0]), int(c[1]), int(c[2]), float(c[3]), int(c[4])
        rep = F.run_gradcheck(PortLib(), draws, steps, agents, tol, seed)
        max_rel, redraws, passed = d["report"][i]
        assert rep["redraws"] == int(redraws) and rep["passed"] == bool(passed)
        assert abs(rep["max_rel_err"] - max_rel) <= 1e-9
        np.testing.assert_allclose(rep["per_draw_max"], d[f"per_draw_{i}"], atol=1e-9)
