"""Choices bit-exact by construction.

Every exp / log on the device is glibc's (csrc/dtg_libm.h; bit-identical to
the host libm, tests/test_gpu_golden.py), so the Gumbel noise and both softmax
stages are the reference's values.  What remains are the fast decision rules:
the first argmax read off the logits unless two lie within 2^-40
(softmax_first_argmax) and the merge winner from alpha + g unless the top two
lie within the rounding bound (merge_softmax_fast).  With dtg_debug_decisions
(force_exact=1) every decision takes the exact two_softmax evaluation; the
trajectories, counts and gradients must not change, on every schedule.
"""
import ctypes as C

import numpy as np
import pytest

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def decisions(force):
    n = C.c_ulonglong()
    assert P.load().dtg_debug_decisions(force, C.byref(n)) == 0
    return n.value


def run(sc, p, B, mode, T):
    lk, ps = sc.seed_agents()
    e = P.Engine(sc, B, T)
    e.set_mode(mode)
    e.set_params(p)
    e.set_state(lk, ps)
    for b in range(B):
        e.set_noise(7, 30 + b, b)
    e.forward(T, sc.steps_per_interval, checkpoint=True)
    cum = e.read_cum_all()
    fin = [e.read_state(b, T) for b in range(B)]
    rng = np.random.default_rng(2)
    g = e.backward(snap_seeds=rng.normal(size=(B, T // sc.steps_per_interval, sc.n_links)),
                   x_seeds=rng.normal(size=(B, sc.n_agents)))
    return cum, fin, g


@pytest.mark.parametrize("n,length,veh,dn,T,B,mode", [
    (4, 400.0, 1000, 1, 600, 1, 0),        # C1, fused persistent grid
    (23, 1609.34, 1000020, 30, 60, 8, 0),  # C4's batch, fused grid
    (23, 1609.34, 1000020, 30, 30, 32, 3),  # batched C3, 5-kernel step graph
    (6, 300.0, 2400, 2, 200, 3, 1),         # cluster per scenario
])
def test_forced_exact_decisions_reproduce_everything(n, length, veh, dn, T, B, mode):
    sc = P.Scenario.grid(n, length, 42, 1000.0).configure(veh, dn, T, 300)
    p = sc.sample_parameters(3)
    decisions(0)
    fast = run(sc, p, B, mode, T)
    n_exact = decisions(1)
    forced = run(sc, p, B, mode, T)
    decisions(0)
    print(f"decisions handed to the exact evaluation by the fast rules: {n_exact}")
    assert np.array_equal(fast[0], forced[0])
    for a, b in zip(fast[1], forced[1]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(fast[2], forced[2])
