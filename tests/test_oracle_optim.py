"""Pin the oracle's restatement of the optimisation loops (oracle/optim.py)
against fixtures the reference itself produced (tests/golden/make_golden.py
optim_cases: calibrate / optimize_control, optimization.cpp:122-295), and
against the reference build when it is present.  CPU only."""
import numpy as np
import pytest

from golden_cases import load


def _port_scn(port, d):
    from oracle.oracle import PortScenario

    return PortScenario(port, d["frm"], d["to"], d["length"], delta_n=1, link0=d["link0"], pos0=d["pos0"],
                        horizon_steps=120, obs_interval_s=30)


def _cfg(d):
    it, pat, draws, lr = d["cfg"]
    return dict(max_iterations=int(it), patience=int(pat), noise_draws=int(draws), lr=float(lr))


def test_transforms_match_reference_formulas():
    from oracle.optim import Bounded, LowerBound

    b = Bounded(13.9, 22.2)
    for v in (13.9, 14.0, 18.05, 22.1999):
        assert abs(b.value(b.raw_of(v)) - v) < 1e-6
    assert b.value(0.0) == 13.9 + (22.2 - 13.9) * 0.5
    lb = LowerBound(0.05)
    for v in (0.06, 1.0, 3.0, 40.0):
        assert abs(lb.value(lb.raw_of(v)) - v) < 1e-9


def test_calibrate_oracle_bit_exact(port):
    from oracle.oracle import Params
    from oracle.optim import calibrate

    d = load("calib_grid3")
    res = calibrate(_port_scn(port, d), d["obs_ids"], d["obs"], int(d["meta"][0]), cfg=_cfg(d), params_cls=Params)
    assert res["iterations"] == int(d["iterations"])
    assert res["best_iteration"] == int(d["best_iteration"])
    np.testing.assert_array_equal(res["loss_curve"], d["loss_curve"])
    assert res["best_loss"] == float(d["best_loss"])
    np.testing.assert_array_equal(np.stack(res["best"].arrays()), d["best"])


def test_calibrate_oracle_from_init_bit_exact(port):
    from oracle.oracle import Params
    from oracle.optim import calibrate

    base = load("calib_grid3")
    d = load("calib_grid3_init")
    init = Params(*d["init"])
    res = calibrate(_port_scn(port, base), base["obs_ids"], base["obs"], 9, init=init, params_cls=Params,
                    cfg=dict(max_iterations=4, patience=20, noise_draws=1, resample_noise=False, lr=0.05))
    np.testing.assert_array_equal(res["loss_curve"], d["loss_curve"])
    assert res["best_iteration"] == int(d["best_iteration"])
    np.testing.assert_array_equal(np.stack(res["best"].arrays()), d["best"])


def test_control_oracle_bit_exact(port):
    from oracle.oracle import Params
    from oracle.optim import optimize_control

    base = load("calib_grid3")
    d = load("control_grid3")
    res = optimize_control(_port_scn(port, base), Params(*d["params"]), int(d["target"]), float(d["desired"]), 7,
                           cfg=dict(max_iterations=5, patience=3, noise_draws=2, lr=0.2), params_cls=Params)
    np.testing.assert_array_equal(res["loss_curve"], d["loss_curve"])
    np.testing.assert_array_equal(res["cost"], d["cost"])
    assert res["achieved"] == float(d["achieved"])
    assert res["gap_fraction"] == float(d["gap_fraction"])
    assert res["iterations"] == int(d["iterations"])
    assert res["zero_gradient_stall"] == bool(d["zero_gradient_stall"])


def test_reference_calibrate_reproduces_fixture(ref):
    """The fixture is what the reference build returns (regeneration check)."""
    from oracle.oracle import RefScenario

    d = load("calib_grid3")
    rs = RefScenario.grid(ref, 3, 300.0, 42, 600.0).configure(300, 1, 120, 30)
    res = rs.calibrate(d["obs_ids"], d["obs"], 5, cfg=_cfg(d))
    np.testing.assert_array_equal(res["loss_curve"], d["loss_curve"])
    np.testing.assert_array_equal(res["best"], d["best"])


def test_reference_calibrate_divergence_is_reported(ref):
    from oracle.oracle import RefScenario

    d = load("calib_grid3")
    rs = RefScenario.grid(ref, 3, 300.0, 42, 600.0).configure(300, 1, 120, 30)
    obs = d["obs"].copy()
    obs[0, 0] = np.inf
    with pytest.raises(FloatingPointError):
        rs.calibrate(d["obs_ids"], obs, 5, cfg=dict(max_iterations=2, noise_draws=1))
