"""Round-2 golden fixtures, produced by the REFERENCE ITSELF (oracle/_ref).

Full-size BASELINE configurations and the reference's own Sioux Falls network
(VERDICT r1 "Next round" item 1), plus per-agent transfer events for travel
times (item 9).  Each case is a separate sub-command so the slow ones can run
as parallel processes (the reference is single-threaded):

    python tests/golden/make_golden_r2.py c2_fwd     # C2 dn=25, 144 steps   (~35 min)
    python tests/golden/make_golden_r2.py c2_grad    # C2 dn=25 gradient     (~2 h)
    python tests/golden/make_golden_r2.py c4_draw    # C4 one MSE draw        (~25 min)
    python tests/golden/make_golden_r2.py sf         # Sioux Falls dn=4/dn=1  (~2 min)
    python tests/golden/make_golden_r2.py c1_travel  # C1 transfer events     (~10 s)

Needs /root/reference (this container only); the .npz files travel.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib, RefScenario, fnv1a64  # noqa: E402

SF_TNTP = "/root/reference/proj/data/siouxfalls_net.tntp"


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


def stack(p):
    return np.stack(p.arrays())


def closed_form_ws(K, L):
    """Deterministic snapshot weights, exact in fp64 (no RNG in the fixture)."""
    k = np.arange(K)[:, None]
    j = np.arange(L)[None, :]
    return (((7 * j + 13 * k) % 11) - 5) / 4.0


def net_arrays(rs):
    f, t, ln, k = rs.links()
    return dict(frm=f, to=t, length=ln, kind=k, n_nodes=np.int32(rs.n_nodes))


def transfer_events(link0, states_link):
    """(step, agent, from, to) for every link change, step-major then agent
    ascending; step t = the engine step after which the agent is on `to`."""
    prev = link0
    rows = []
    for t in range(states_link.shape[0]):
        cur = states_link[t]
        (idx,) = np.nonzero(cur != prev)
        for a in idx:
            rows.append((t, a, prev[a], cur[a]))
        prev = cur
    return np.array(rows, np.int32).reshape(-1, 4)


def c2(R, grad: bool):
    """C2 (BASELINE configs[1]): 50x50 grid, 400 m, 100,000 vehicles; the
    oracle-feasible platoon dn=25 (N = 4,000), full 1-h horizon (144 steps),
    observation interval 300 s (12 steps)."""
    T = 144
    rs = RefScenario.grid(R, 50, 400.0, 42, 1000.0).configure(100000, 25, T, 300)
    p = rs.sample_parameters(3)
    out = dict(params=stack(p), meta=np.array([7, 0, T, 300, 25, 1], np.float64), **net_arrays(rs))
    t0 = time.time()
    if not grad:
        fw = rs.forward(p, 7, 0)
        cum = fw["cum_per_step"]
        out.update(link=fw["link"], pos=fw["pos"], cum_snap=cum[11::12], cum_final=cum[-1],
                   fnv_state=np.uint64(fnv1a64(fw["link"], fw["pos"])), fnv_cum=np.uint64(fnv1a64(cum)),
                   ref_wall_s=np.float64(time.time() - t0))
        save("c2_dn25_forward", **out)
    else:
        L = rs.n_links
        ws = closed_form_ws(T // 12, L)
        wc = np.cos(np.arange(L) * 0.37)
        g = rs.gradient(p, 7, 2, 1, ws=ws, wc=wc)
        out.update(noise=np.int64(2), loss=np.float64(g["loss"]), grads=g["grads"], snapshots=g["snapshots"],
                   cum_final=g["cum_final"], link=g["link"], pos=g["pos"], loss_wc=wc,
                   ref_wall_s=np.float64(time.time() - t0))
        save("c2_dn25_gradient", **out)


def calibrate_start(L):
    """calibrate()'s first iterate: raw 0 through BoundedTransform::value,
    lo + (hi - lo) * sigmoid(0) (optimization.cpp:27-31, 134-160), cost 1."""
    from oracle.oracle import Params

    mid = lambda lo, hi: np.full(L, lo + (hi - lo) * 0.5)
    return Params(mid(13.9, 22.2), mid(0.18, 0.22), mid(0.0, 5.0), mid(0.01, 5.0), np.ones(L))


def c4_draw(R):
    """C4 exactly as bench.py's calibration runs it, one draw: C3 net, 30-min
    window (60 steps), truth = sample_parameters(42), observations = the truth
    run's snapshot counts x dn on links j % 5 != 0, calibration start = range
    midpoints with cost 1, draw k = 0 of iteration 0 -> noise_iteration 1
    (optimization.cpp:175-177), MSE loss (mse_loss_builder)."""
    T = 60
    rs = RefScenario.grid(R, 23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
    L = rs.n_links
    truth = rs.sample_parameters(42)
    t0 = time.time()
    tr = rs.forward(truth, 7, 0)
    obs_ids = np.array([j for j in range(L) if j % 5 != 0], np.int32)
    obs = tr["cum_per_step"][9::10][:, obs_ids] * 30.0
    mid = calibrate_start(L)
    loss, grads = rs.gradient_mse(mid, 7, 1, obs_ids, obs)
    save("c4_draw1", truth=stack(truth), params=stack(mid), obs_ids=obs_ids, obs=obs,
         truth_cum_final=tr["cum_per_step"][-1], truth_fnv_cum=np.uint64(fnv1a64(tr["cum_per_step"])),
         loss=np.float64(loss), grads=grads, ref_wall_s=np.float64(time.time() - t0))


def sioux_falls(R):
    """The reference's own network (data/siouxfalls_net.tntp) as
    configs/siouxfalls.toml builds it: length_unit_scale 1609.34, virtual
    links 1000 m, seed 42, 2,000 vehicles, interval 300 s; forward over the
    90-min horizon and the MSE gradient over the 30-min observation window, at
    the calibration platoon dn=4 and the truth platoon dn=1."""
    text = open(SF_TNTP).read()
    for dn in (4, 1):
        T_fwd, T_grad = 90 * 60 // dn, 30 * 60 // dn
        spi = 300 // dn
        rs = RefScenario.tntp(R, text, 1609.34, 42, 1000.0).configure(2000, dn, T_fwd, 300)
        truth = rs.sample_parameters(42)
        p = rs.sample_parameters(3)
        fw = rs.forward(p, 42, 0, record_states=True)
        cum = fw["cum_per_step"]
        lk0, ps0 = rs.seed_agents()
        out = dict(params=stack(p), truth=stack(truth), link0=lk0, pos0=ps0, **net_arrays(rs),
                   meta=np.array([42, 0, T_fwd, 300, dn, 1], np.float64),
                   link=fw["link"], pos=fw["pos"], cum_snap=cum[spi - 1::spi], cum_final=cum[-1],
                   fnv_state=np.uint64(fnv1a64(fw["link"], fw["pos"])), fnv_cum=np.uint64(fnv1a64(cum)),
                   fnv_states=np.uint64(fnv1a64(fw["states_link"], fw["states_pos"])),
                   events=transfer_events(lk0, fw["states_link"]))
        rg = RefScenario.tntp(R, text, 1609.34, 42, 1000.0).configure(2000, dn, T_grad, 300)
        tt = rg.forward(truth, 42, 0)
        phys = np.array([j for j in range(rg.n_links) if rg.links()[3][j] == 0], np.int32)
        obs = tt["cum_per_step"][spi - 1::spi][:, phys] * float(dn)
        loss, grads = rg.gradient_mse(p, 42, 1, phys, obs)
        out.update(obs_ids=phys, obs=obs, loss=np.float64(loss), grads=grads, T_grad=np.int32(T_grad))
        save(f"sf_dn{dn}", **out)


def c1_travel(R):
    """C1 (4x4 grid, 1,000 vehicles, dn=1, 30 min): every agent's link change
    from the reference's record_states, i.e. its link-entry steps."""
    rs = RefScenario.grid(R, 4, 400.0, 42, 1000.0).configure(1000, 1, 1800, 300)
    p = rs.sample_parameters(3)
    fw = rs.forward(p, 7, 0, record_states=True)
    lk0, _ = rs.seed_agents()
    ev = transfer_events(lk0, fw["states_link"])
    save("c1_travel", events=ev, link0=lk0, fnv_states=np.uint64(fnv1a64(fw["states_link"], fw["states_pos"])))


def main():
    R = RefLib()
    what = sys.argv[1] if len(sys.argv) > 1 else "fast"
    if what in ("c2_fwd",):
        c2(R, grad=False)
    elif what == "c2_grad":
        c2(R, grad=True)
    elif what == "c4_draw":
        c4_draw(R)
    elif what == "sf":
        sioux_falls(R)
    elif what == "c1_travel":
        c1_travel(R)
    elif what == "fast":
        sioux_falls(R)
        c1_travel(R)
    else:
        raise SystemExit(f"unknown case {what}")


if __name__ == "__main__":
    main()
