"""The reference's analytic choice-frequency tests (test_node_model.cpp:105-149,
acceptance criterion 5) on the device, as ONE batched launch of 10,000
independent one-step scenarios (noise iterations 0..9999):

* link choice on a fork: P(link 1) = e^2 / (e^2 + e^1) = 0.7311 (beta = 0, 2, 1);
* merge of two feeders into one link: exactly one admission per step and
  P(feeder 0 wins) = e^3 / (e^3 + e^1) = 0.8808 (alpha = 3, 1, 1).

The reference keys its trials by step with a fixed stream; here the trials
differ by noise_iteration (engine.cpp:49) — same distribution, independent
draws.  Band: +-0.02 as in the reference."""
import math

import numpy as np
import pytest

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
TRIALS = 10000


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(frm, to, link0, pos0, beta, alpha):
    sc = P.Scenario.from_links(4, frm, to, [100.0] * 3, [0, 0, 0])
    sc.configure(0, 1, 1, 1, fit_queues=False, custom_init=(np.array(link0, np.int32), np.array(pos0)))
    p = P.LinkParams(np.full(3, 16.0), np.full(3, 0.2), np.array(beta, float), np.array(alpha, float),
                     np.ones(3))
    trs = P.simulate_forward(sc, p, seed=99, noise_iterations=range(TRIALS))
    return np.stack([t.link_final for t in trs]), np.stack([t.pos_final for t in trs])


def test_link_choice_frequency_matches_softmax():
    # fork: link 0 (node 0 -> 1) feeds links 1 (1 -> 2) and 2 (1 -> 3)
    link, pos = run([0, 1, 1], [1, 2, 3], [0], [100.0], [0.0, 2.0, 1.0], [1.0, 1.0, 1.0])
    assert set(np.unique(link[:, 0])) <= {1, 2}
    assert np.all(pos[:, 0] == 0.0)  # entrants land exactly at 0 (transfer, node_model.cpp:131-148)
    freq = np.mean(link[:, 0] == 1)
    expected = math.exp(2.0) / (math.exp(2.0) + math.exp(1.0))
    assert abs(freq - expected) < 0.02, freq


def test_merge_admits_exactly_one_by_priority():
    # merge: links 0 (0 -> 2) and 1 (1 -> 2) feed link 2 (2 -> 3)
    link, pos = run([0, 1, 2], [2, 2, 3], [0, 1], [100.0, 100.0], [1.0, 1.0, 1.0], [3.0, 1.0, 1.0])
    admitted = (link == 2).sum(axis=1)
    assert np.all(admitted == 1)  # exactly one admission every step
    loser = np.where(link[:, 0] == 2, 1, 0)
    assert np.all(link[np.arange(TRIALS), loser] == loser)  # the other one waits at its link end
    assert np.all(pos[np.arange(TRIALS), loser] == 100.0)
    freq = np.mean(link[:, 0] == 2)
    expected = math.exp(3.0) / (math.exp(3.0) + math.exp(1.0))
    assert abs(freq - expected) < 0.02, freq
