"""Host layer of the product (C++ behind the C-ABI, no GPU needed): network
construction, CSR adjacency, parameter sampling, seeding, queue fitting, TNTP
parsing, horizon arithmetic, calibration loss — each against the reference
(golden fixtures; live reference where built)."""
import numpy as np
import pytest

P = pytest.importorskip("paper_2603_25068_b200")

from golden_cases import load, meta  # noqa: E402


@pytest.mark.parametrize("name,n,length,net_seed,veh,dn,pseed", [
    ("c1_forward", 4, 400.0, 42, 1000, 1, 3),
    ("grid5_dn4_tau03", 5, 350.0, 9, 2000, 4, 4),
    ("grid6_dn2_tau1", 6, 300.0, 11, 2400, 2, 5),
])
def test_grid_network_params_seeding_match_reference(name, n, length, net_seed, veh, dn, pseed):
    d = load(name)
    m = meta(d)
    sc = P.Scenario.grid(n, length, net_seed, 1000.0).configure(veh, dn, m["T"], m["obs_s"])
    f, t, ln, k = sc.links()
    assert np.array_equal(f, d["frm"]) and np.array_equal(t, d["to"])
    assert np.array_equal(ln, d["length"])  # includes fit_inflow_queues
    assert np.array_equal(k, d["kind"])
    assert sc.n_nodes == int(d["n_nodes"])
    off, succ = sc.csr()
    assert np.array_equal(off, d["succ_off"]) and np.array_equal(succ, d["succ"])
    p = sc.sample_parameters(pseed)
    assert np.array_equal(np.stack(p.arrays()), d["params"])  # bit-exact (no FMA contraction)
    lk, ps = sc.seed_agents()
    assert np.array_equal(lk, d["link0"]) and np.array_equal(ps, d["pos0"])


def test_chicago_scale_network_matches_reference(ref):
    from oracle.oracle import RefScenario

    a = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
    r = RefScenario.grid(ref, 23, 1609.34, 42, 1000.0).configure(1000020, 30, 120, 300)
    assert a.n_links == r.n_links == 2553
    assert a.n_agents == r.n_agents == 33334
    for x, y in zip(a.links(), r.links()):
        assert np.array_equal(x, y)
    off, succ = a.csr()
    adj = r.adjacency()
    rows, cols = np.nonzero(adj)
    assert np.array_equal(np.repeat(np.arange(a.n_links), np.diff(off)), rows)
    assert np.array_equal(succ, cols)
    for x, y in zip(a.sample_parameters(3).arrays(), r.sample_parameters(3).arrays()):
        assert np.array_equal(x, y)
    for x, y in zip(a.sample_parameters(0, True).arrays(), r.sample_parameters(0, True).arrays()):
        assert np.array_equal(x, y)
    for x, y in zip(a.seed_agents(), r.seed_agents()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name", [f"ring_{i}" for i in range(6)] + ["engine_chain_ckpt", "engine_chain_dn2"])
def test_make_network_csr(name):
    d = load(name)
    sc = P.Scenario.from_links(int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"])
    off, succ = sc.csr()
    assert np.array_equal(off, d["succ_off"]) and np.array_equal(succ, d["succ"])


def test_agent_seeding_known_answer():
    """test_engine.cpp:42-75."""
    sc = P.Scenario.from_links(5, [2, 3, 0], [0, 0, 4], [100.0] * 3, [1, 1, 2])
    sc.configure(4, 1, 0, 300, fit_queues=False)
    lk, ps = sc.seed_agents()
    assert lk.tolist() == [0, 1, 0, 1]
    assert ps.tolist() == [100, 100, 95, 95]
    sc.configure(1, 1, 0, 300, fit_queues=False)
    assert sc.seed_agents()[1].tolist() == [100]
    sc.configure(3, 2, 0, 300, fit_queues=False)
    with pytest.raises(Exception):
        sc.seed_agents()
    sc.configure(100, 1, 0, 300, fit_queues=False)
    with pytest.raises(Exception, match="needs length"):
        sc.seed_agents()
    sc.configure(100, 1, 0, 300, fit_queues=True)
    assert len(sc.seed_agents()[1]) == 100
    assert sc.links()[2][0] >= 49 * 5.0


def test_horizon_arithmetic():
    """test_engine.cpp:77-85."""
    assert P.steps_for_minutes(1, 1.0, 90.0) == 5400
    assert P.steps_for_minutes(2, 1.0, 90.0) == 2700
    with pytest.raises(RuntimeError):
        P.steps_for_minutes(7, 1.0, 1.0)


def test_tntp_parse_and_virtual_links(ref):
    """parse_tntp_text + attach_virtual_links on a small TNTP text, against the
    reference (network built from the same links)."""
    text = """<NUMBER OF ZONES> 3
<NUMBER OF NODES> 4
<FIRST THRU NODE> 1
<NUMBER OF LINKS> 6
<END OF METADATA>
~ tail head cap len fft b pow speed toll type ;
1 2 25900.2 6 6 0.15 4 0 0 1 ;
2 1 25900.2 6 6 0.15 4 0 0 1 ;
2 3 4958.2 4 4 0.15 4 0 0 1 ;
3 2 4958.2 4 4 0.15 4 0 0 1 ;
3 4 4958.2 5 4 0.15 4 0 0 1 ;
4 3 4958.2 5 4 0.15 4 0 0 1 ;
"""
    from oracle.oracle import RefScenario

    sc = P.Scenario.tntp(text, 1609.34, 42, 1000.0)
    f, t, ln, k = sc.links()
    assert f[:6].tolist() == [0, 1, 1, 2, 2, 3] and t[:6].tolist() == [1, 0, 2, 1, 3, 2]
    assert ln[0] == 6 * 1609.34
    phys = RefScenario.from_links(ref, 4, f[:6], t[:6], ln[:6], [0] * 6)
    assert phys.n_links == 6
    bad = "<NUMBER OF NODES> 2\n<END OF METADATA>\n1 2 3 4 5\n"
    with pytest.raises(RuntimeError, match="does not end with"):
        P.Scenario.tntp(bad, 1.0, 1, 1.0)


def test_mse_loss_value_and_seeds(port):
    """Host calibration loss (mse_loss_builder) on the reference's snapshots:
    value bit-equal to the reference's own loss (fixture c1_mse)."""
    from oracle.oracle import Params

    from golden_cases import port_scenario

    d = load("c1_mse")
    g1 = load("c1_gradient")
    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 600, 300)
    lk, ps = sc.seed_agents()
    from oracle.oracle import PortScenario

    f, t, ln, _ = sc.links()
    pr = PortScenario(port, f, t, ln, link0=lk, pos0=ps, horizon_steps=600, obs_interval_s=300)
    fw = pr.forward(Params(*d["params"]), 7, 1)
    snaps = np.ascontiguousarray(fw["cum_per_step"][299::300])
    lib = P.load()
    loss = np.zeros(1)
    seeds = np.zeros_like(snaps)
    rc = lib.dtg_mse_loss(snaps.shape[0], snaps.shape[1], snaps, len(d["obs_ids"]), d["obs_ids"],
                          d["obs"].shape[0], np.ascontiguousarray(d["obs"]), 1, loss, seeds)
    assert rc == 0
    assert loss[0] == float(d["loss"])
    del g1, port_scenario


SF_TNTP = "/root/reference/proj/data/siouxfalls_net.tntp"


@pytest.mark.parametrize("dn", [4, 1])
def test_sioux_falls_tntp_network_and_seeding_match_reference(dn):
    """The product's TNTP parser + attach_virtual_links + fit_inflow_queues +
    seeding on the reference's own data/siouxfalls_net.tntp, as
    configs/siouxfalls.toml builds it, against the reference's network
    (tests/golden/sf_dn*.npz)."""
    import os

    if not os.path.exists(SF_TNTP):
        pytest.skip("reference data not present on this host")
    d = load(f"sf_dn{dn}")
    T = int(d["meta"][2])
    sc = P.Scenario.tntp(open(SF_TNTP).read(), 1609.34, 42, 1000.0).configure(2000, dn, T, 300)
    f, t, ln, k = sc.links()
    assert np.array_equal(f, d["frm"]) and np.array_equal(t, d["to"])
    assert np.array_equal(ln, d["length"]) and np.array_equal(k, d["kind"])
    assert sc.n_nodes == int(d["n_nodes"])
    assert np.array_equal(np.stack(sc.sample_parameters(3).arrays()), d["params"])
    assert np.array_equal(np.stack(sc.sample_parameters(42).arrays()), d["truth"])
    lk, ps = sc.seed_agents()
    assert np.array_equal(lk, d["link0"]) and np.array_equal(ps, d["pos0"])
