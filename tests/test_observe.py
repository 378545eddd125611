"""Observation / output side through libdtg.so's host
C++ (no GPU needed): synthesize_observations, count_metrics and the count CSV
against fixtures produced by the reference (tests/golden/make_golden.py
observe_cases) and, when built, the reference itself."""
import numpy as np
import pytest

from golden_cases import load

P = pytest.importorskip("paper_2603_25068_b200")
from paper_2603_25068_b200 import observe as O  # noqa: E402


@pytest.fixture(scope="module")
def d():
    return load("observe_c1")


def test_synthesize_observations_bit_exact(d):
    truth = O.CountSeries(d["phys"], 300, d["truth_vals"][:2])
    obs, ids = O.synthesize_observations(truth, 0.1, 0.8, 42)
    assert np.array_equal(ids, d["obs_ids"])
    assert np.array_equal(obs.values, d["obs_vals"])
    assert obs.interval_s == 300
    assert len(ids) == int(np.floor(0.8 * len(d["phys"])))


def test_synthesize_edge_cases():
    truth = O.CountSeries(np.arange(5, dtype=np.int32), 60, np.arange(10, dtype=np.float64).reshape(2, 5))
    obs, ids = O.synthesize_observations(truth, 0.0, 1.0, 7)
    assert np.array_equal(ids, np.arange(5)) and np.array_equal(obs.values, truth.values)
    obs, ids = O.synthesize_observations(truth, 0.5, 0.0, 7)
    assert len(ids) == 0 and obs.values.shape == (2, 0)
    neg = O.CountSeries(np.arange(3, dtype=np.int32), 60, -np.ones((1, 3)))
    obs, _ = O.synthesize_observations(neg, 0.2, 1.0, 1)
    assert (obs.values == 0.0).all()  # clamped at zero like the reference


def test_count_metrics_bit_exact(d):
    m = O.count_metrics(O.CountSeries(d["phys"], 300, d["sim_vals"]), O.CountSeries(d["obs_ids"], 300, d["obs_vals"]))
    mae, r, rd, npairs = d["metrics"]
    assert m.mae == mae and m.pearson_r == r and m.r_defined == bool(rd) and m.n_pairs == int(npairs)
    s = O.CountSeries(d["phys"], 300, d["truth_vals"])
    m = O.count_metrics(s, s)
    assert (m.mae, m.pearson_r, m.r_defined, m.n_pairs) == tuple(
        [d["metrics_self"][0], d["metrics_self"][1], bool(d["metrics_self"][2]), int(d["metrics_self"][3])])


def test_count_metrics_disjoint_and_constant():
    a = O.CountSeries(np.array([1, 2], np.int32), 60, np.ones((3, 2)))
    b = O.CountSeries(np.array([5], np.int32), 60, np.ones((3, 1)))
    m = O.count_metrics(a, b)
    assert m.n_pairs == 0 and not m.r_defined and m.mae == 0.0
    c = O.CountSeries(np.array([2], np.int32), 60, np.ones((3, 1)))
    m = O.count_metrics(a, c)  # increments 1, 0, 0 vs 1, 0, 0
    assert m.n_pairs == 3 and m.mae == 0.0 and m.r_defined


def test_series_csv_byte_identical_and_round_trip(d):
    s = O.CountSeries(d["phys"], 300, d["truth_vals"])
    txt = O.series_to_csv(s)
    assert txt.encode() == bytes(d["csv_truth"])
    txt2 = O.series_to_csv(O.CountSeries(d["obs_ids"], 300, d["obs_vals"]))
    assert txt2.encode() == bytes(d["csv_obs"])
    back = O.series_from_csv(txt)
    assert back.interval_s == 300 and np.array_equal(back.link_ids, np.sort(d["phys"]))
    # %.12g round trip: equal to 12 significant digits
    np.testing.assert_allclose(back.values, d["truth_vals"][:, np.argsort(d["phys"])], rtol=1e-11)


@pytest.mark.parametrize("text,msg", [
    ("", "empty file"),
    ("link_id,t_seconds,cumulative_count\n", "no data rows"),
    ("h\n1,300,2\n1,x,3\n", "malformed row"),
    ("h\n1,300,2\n1,900,3\n", "irregular interval grid"),
    ("h\n1,300,2\n2,300,3\n1,600,4\n", "ragged link sets"),
])
def test_series_from_csv_errors(text, msg):
    with pytest.raises(P.DtgError, match=msg):
        O.series_from_csv(text)


def test_against_reference_build(ref, d):
    oid, ov = ref.synthesize_observations(d["phys"], d["truth_vals"][:2], 300, 0.25, 0.55, 99)
    obs, ids = O.synthesize_observations(O.CountSeries(d["phys"], 300, d["truth_vals"][:2]), 0.25, 0.55, 99)
    assert np.array_equal(ids, oid) and np.array_equal(obs.values, ov)
    rng = np.random.default_rng(5)
    vals = np.cumsum(rng.uniform(0, 20, size=(6, len(d["phys"]))), axis=0)
    assert O.series_to_csv(O.CountSeries(d["phys"], 120, vals)) == ref.series_to_csv(d["phys"], vals, 120)
    m = O.count_metrics(O.CountSeries(d["phys"], 120, vals), O.CountSeries(d["phys"][::2], 120, vals[:4, ::2] * 1.1))
    r = ref.count_metrics(d["phys"], vals, d["phys"][::2], vals[:4, ::2] * 1.1)
    assert (m.mae, m.pearson_r, m.r_defined, m.n_pairs) == (r["mae"], r["pearson_r"], r["r_defined"], r["n_pairs"])


def test_series_from_levels():
    cum = np.cumsum(np.ones((12, 4)), axis=0)
    s = O.series_from_levels(cum, [0, 2], 60, 30.0, 2)
    assert s.n_intervals == 6 and np.array_equal(s.values[:, 0], cum[1::2, 0] * 2)
