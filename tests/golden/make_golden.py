"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs the unmodified reference sources (oracle/_ref/libdtsim_ref.so, built by
`make -C oracle ref` from /root/reference/proj/src) and records inputs and
outputs of simulate_forward / simulate_gradient (and the network/parameter/
seeding helpers) for a set of small and full-size cases.  The fixtures pin the
C oracle port (tests/test_oracle_port.py), the product host layer
(tests/test_host.py) and the GPU path (tests/test_gpu_parity.py) on machines
where /root/reference does not exist.

    python tests/golden/make_golden.py            # all cases (~2 min)
"""
from __future__ import annotations

import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib, RefScenario, csr_from_links, fnv1a64  # noqa: E402

R = RefLib()


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def params_arrays(p):
    return np.stack(p.arrays())


def flat_params(L, u=16.0):
    from oracle.oracle import Params

    return Params(np.full(L, u), np.full(L, 0.2), np.full(L, 1.0), np.full(L, 1.0), np.full(L, 1.0))


def record_case(rs, p, seed, noise, T, spi_s, dn, tg, gt, rng, states=True, grad=True, name=None,
                full_cum=True, loss=None):
    f, t, ln, k = rs.links()
    off, succ = csr_from_links(f, t)
    adj = rs.adjacency()
    # cross-check the CSR against the reference's dense adjacency
    dense = np.zeros_like(adj)
    for i in range(len(off) - 1):
        dense[i, succ[off[i]:off[i + 1]]] = 1.0
    assert np.array_equal(dense, adj)
    lk0, ps0 = rs.seed_agents()
    fw = rs.forward(p, seed, noise, record_states=states)
    out = dict(frm=f, to=t, length=ln, kind=k, succ_off=off, succ=succ, n_nodes=np.int32(rs.n_nodes),
               params=params_arrays(p), link0=lk0, pos0=ps0,
               meta=np.array([seed, noise, T, spi_s, dn, int(tg)], np.float64), gumbel_tau=np.float64(gt),
               cum_final=fw["cum_per_step"][-1] if T else np.zeros(rs.n_links),
               link=fw["link"], pos=fw["pos"],
               fnv_state=np.uint64(fnv1a64(fw["link"], fw["pos"])),
               fnv_cum=np.uint64(fnv1a64(fw["cum_per_step"])))
    if full_cum:
        out["cum_per_step"] = fw["cum_per_step"]
    if states:
        out["states_link"], out["states_pos"] = fw["states_link"], fw["states_pos"]
    if grad:
        L, N = rs.n_links, rs.n_agents
        K = T // int(round(spi_s / dn))
        if loss is None:
            loss = dict(ws=rng.normal(size=(K, L)), qs=rng.normal(size=(K, L)) * 0.1, wc=rng.normal(size=L),
                        qc=None, wx=rng.normal(size=N))
        g = rs.gradient(p, seed, noise, 1, **loss)
        for key, v in loss.items():
            if v is not None:
                out["loss_" + key] = np.asarray(v, np.float64)
        out["loss"] = np.float64(g["loss"])
        out["grads"] = g["grads"]
        out["snapshots"] = g["snapshots"]
    save(name, **out)


def grid_case(name, n, length, net_seed, veh, dn, T, obs_s, pseed, seed, noise=0, tg=True, gt=0.01, **kw):
    rs = RefScenario.grid(R, n, length, net_seed, 1000.0).configure(veh, dn, T, obs_s, gumbel_tau=gt, tg=tg)
    p = rs.sample_parameters(pseed)
    record_case(rs, p, seed, noise, T, obs_s, dn, tg, gt, np.random.default_rng(zlib.crc32(name.encode())), name=name, **kw)


def ring_chord_net(rng, n_nodes, n_chords):
    frm, to = [], []
    for i in range(n_nodes):
        frm += [i, (i + 1) % n_nodes]
        to += [(i + 1) % n_nodes, i]
    for _ in range(n_chords):
        a, b = rng.choice(n_nodes, 2, replace=False)
        frm.append(int(a))
        to.append(int(b))
    kind = [0] * len(frm)
    # virtual inflow into node 0 and a sink out of node n/2 (fresh boundary nodes)
    frm += [n_nodes, n_nodes // 2]
    to += [0, n_nodes + 1]
    kind += [1, 2]
    length = list(rng.uniform(60.0, 240.0, size=len(frm) - 2)) + [400.0, 5000.0]
    return np.array(frm, np.int32), np.array(to, np.int32), np.array(length), np.array(kind, np.int32), n_nodes + 2


def custom_case(name, seed, n_nodes, n_chords, n_agents, dn, T, obs_s, tg, gt):
    rng = np.random.default_rng(seed)
    f, t, ln, k, nn = ring_chord_net(rng, n_nodes, n_chords)
    L = len(f)
    link = rng.integers(0, L, size=n_agents).astype(np.int32)
    pos = rng.uniform(0.0, 1.0, size=n_agents) * ln[link]
    # edge cases: exact ties, agents exactly at / within tolerance of the link end,
    # a slightly negative (still valid) position, several arrived agents on one link
    pos[: n_agents // 10] = ln[link[: n_agents // 10]]
    tie = n_agents // 10
    link[tie + 1] = link[tie]
    pos[tie + 1] = pos[tie]
    pos[tie + 2] = ln[link[tie + 2]] - 0.005
    pos[tie + 3] = -0.005
    link[tie + 4] = link[0]
    pos[tie + 4] = ln[link[0]]
    rs = RefScenario.from_links(R, nn, f, t, ln, k).configure(0, dn, T, obs_s, gumbel_tau=gt, tg=tg, fit=False,
                                                              custom_init=(link, pos))
    pr = rng.uniform(0.5, 1.5, size=(5, L))
    from oracle.oracle import Params

    p = Params(13.9 + 8.3 * pr[0] / 1.5, 0.18 + 0.04 * pr[1] / 1.5, 5.0 * pr[2] / 1.5,
               0.01 + 4.99 * pr[3] / 1.5, pr[4])
    record_case(rs, p, 1000 + seed, seed % 5, T, obs_s, dn, tg, gt, rng, name=name)


def chain_net(phys_len=200.0, virt_len=400.0):
    return (np.array([3, 0, 1, 2], np.int32), np.array([0, 1, 2, 4], np.int32),
            np.array([virt_len, phys_len, phys_len, virt_len]), np.array([1, 0, 0, 2], np.int32), 5)


def optim_cases():
    """calibrate / optimize_control (optimization.cpp:122-295) on a 3x3 grid."""
    rs = RefScenario.grid(R, 3, 300.0, 42, 600.0).configure(300, 1, 120, 30)
    truth = rs.sample_parameters(42)
    tr = rs.forward(truth, 7, 0)
    obs_ids = np.array([j for j in range(rs.n_links) if rs.links()[3][j] == 0], np.int32)
    obs = tr["cum_per_step"][29::30][:, obs_ids] * 1.0
    cfg = dict(max_iterations=6, patience=3, noise_draws=3, lr=0.1)
    cal = rs.calibrate(obs_ids, obs, 5, cfg=cfg)
    L = rs.n_links
    f, t, ln, k = rs.links()
    lk0, ps0 = rs.seed_agents()
    net = dict(frm=f, to=t, length=ln, kind=k, n_nodes=np.int32(rs.n_nodes), link0=lk0, pos0=ps0,
               truth=params_arrays(truth))
    cfgv = np.array([cfg["max_iterations"], cfg["patience"], cfg["noise_draws"], cfg["lr"]], np.float64)
    save("calib_grid3", obs_ids=obs_ids, obs=obs, cfg=cfgv, best=cal["best"], best_loss=np.float64(cal["best_loss"]),
         best_iteration=np.int32(cal["best_iteration"]), iterations=np.int32(cal["iterations"]),
         loss_curve=cal["loss_curve"], meta=np.array([5, 0, 120, 30, 1, 1], np.float64), **net)
    # the same from a given init (raw_of path), one draw, fixed noise
    init = rs.sample_parameters(3)
    cfg1 = dict(max_iterations=4, patience=20, noise_draws=1, resample_noise=False, lr=0.05)
    cal1 = rs.calibrate(obs_ids, obs, 9, cfg=cfg1, init=init)
    save("calib_grid3_init", init=params_arrays(init), best=cal1["best"], best_loss=np.float64(cal1["best_loss"]),
         best_iteration=np.int32(cal1["best_iteration"]), iterations=np.int32(cal1["iterations"]),
         loss_curve=cal1["loss_curve"])
    # control toward 1.5x the achieved count on a busy physical link
    cum_final = tr["cum_per_step"][-1]
    target = int(obs_ids[np.argmax(cum_final[obs_ids])])
    desired = float(cum_final[target]) * 1.5
    cfgc = dict(max_iterations=5, patience=3, noise_draws=2, lr=0.2)
    ctl = rs.optimize_control(truth, target, desired, 7, cfg=cfgc)
    save("control_grid3", params=params_arrays(truth), target=np.int32(target), desired=np.float64(desired),
         cost=ctl["cost"], achieved=np.float64(ctl["achieved"]), gap_fraction=np.float64(ctl["gap_fraction"]),
         best_loss=np.float64(ctl["best_loss"]), iterations=np.int32(ctl["iterations"]),
         zero_gradient_stall=np.int32(ctl["zero_gradient_stall"]), loss_curve=ctl["loss_curve"])


def observe_cases():
    """synthesize_observations / count_metrics / series_to_csv on the C1 truth run."""
    rs = RefScenario.grid(R, 4, 400.0, 42, 1000.0).configure(1000, 1, 1800, 300)
    truth = rs.sample_parameters(42)
    tr = rs.forward(truth, 42, 0)
    f, t, ln, k = rs.links()
    phys = np.array([j for j in range(rs.n_links) if k[j] == 0], np.int32)
    vals = tr["cum_per_step"][299::300][:, phys] * 1.0  # series_from_levels, dn = 1
    window = vals[:2]  # observe_window_min = 10 of 5-min intervals
    oid, ov = R.synthesize_observations(phys, window, 300, 0.1, 0.8, 42)
    # a calibrated-like series: the truth rows perturbed deterministically
    rng = np.random.default_rng(3)
    sim = vals * (1.0 + 0.05 * rng.standard_normal(vals.shape))
    met = R.count_metrics(phys, sim, oid, ov)
    met_self = R.count_metrics(phys, vals, phys, vals)
    csv_truth = R.series_to_csv(phys, vals, 300)
    csv_obs = R.series_to_csv(oid, ov, 300)
    save("observe_c1", phys=phys, truth_vals=vals, obs_ids=oid, obs_vals=ov, sim_vals=sim,
         metrics=np.array([met["mae"], met["pearson_r"], met["r_defined"], met["n_pairs"]], np.float64),
         metrics_self=np.array([met_self["mae"], met_self["pearson_r"], met_self["r_defined"],
                                met_self["n_pairs"]], np.float64),
         csv_truth=np.frombuffer(csv_truth.encode(), np.uint8), csv_obs=np.frombuffer(csv_obs.encode(), np.uint8))


def pipeline_case():
    """synthesize -> calibrate -> nowcast -> metrics on a 3x3 grid, the data flow
    of cmd_synthesize / cmd_calibrate / cmd_nowcast (pipeline.cpp:192-331)."""
    rs = RefScenario.grid(R, 3, 300.0, 42, 600.0).configure(300, 1, 240, 60)
    f, t, ln, k = rs.links()
    phys = np.array([j for j in range(rs.n_links) if k[j] == 0], np.int32)
    truth = rs.sample_parameters(42)
    tr = rs.forward(truth, 42, 0)
    truth_vals = tr["cum_per_step"][59::60][:, phys] * 1.0
    oid, ov = R.synthesize_observations(phys, truth_vals[:2], 60, 0.1, 0.8, 42)
    rw = RefScenario.grid(R, 3, 300.0, 42, 600.0).configure(300, 1, 120, 60)
    cal = rw.calibrate(oid, ov, 42, cfg=dict(max_iterations=5, patience=3, noise_draws=2, lr=0.1))
    from oracle.oracle import Params
    best = Params(*cal["best"])
    now = rs.forward(best, 42, 1000000007)
    now_vals = now["cum_per_step"][59::60][:, phys] * 1.0
    met = R.count_metrics(phys, now_vals, phys, truth_vals)
    save("pipeline_grid3", phys=phys, truth_vals=truth_vals, obs_ids=oid, obs_vals=ov,
         loss_curve=cal["loss_curve"], best=cal["best"], now_vals=now_vals,
         metrics=np.array([met["mae"], met["pearson_r"], met["r_defined"], met["n_pairs"]], np.float64),
         csv_now=np.frombuffer(R.series_to_csv(phys, now_vals, 60).encode(), np.uint8))


def main():
    # RNG known-answer values (include/dtsim/rng.hpp, tensor.cpp:682-699)
    seeds = np.array([0, 1, 7, 42, 2**63 + 5, 0xDEADBEEF], np.uint64)
    keys = np.array([[0, 0, 0], [1, 2, 3], [5, 12, 0], [2**40, 7, 2**33], [3, 999999, 17]], np.uint64)
    bits = np.array([[R.lib.ref_rng_bits(int(s), *map(int, k)) for k in keys] for s in seeds], np.uint64)
    unif = np.array([[R.lib.ref_rng_uniform(int(s), *map(int, k)) for k in keys] for s in seeds])
    forks = np.array([[R.lib.ref_rng_fork(int(s), lab) for lab in range(8)] for s in seeds], np.uint64)
    gum = np.array([[R.lib.ref_gumbel(int(s), int(k[0]), int(k[1]) % 2**31, int(k[2]) % 2**31)
                     for k in keys] for s in seeds])
    save("rng_kat", seeds=seeds, keys=keys, bits=bits, uniform=unif, forks=forks, gumbel=gum)

    # test_engine.cpp:147-192 (checkpointed == full tape) and :194-215
    f, t, ln, k, nn = chain_net(150.0, 200.0)
    rs = RefScenario.from_links(R, nn, f, t, ln, k).configure(5, 1, 25, 5)
    L = rs.n_links
    ws = np.zeros((5, L))
    ws[1] = 0.5
    record_case(rs, flat_params(L, 17.0), 11, 0, 25, 5, 1, True, 0.01, None, name="engine_chain_ckpt",
                loss=dict(ws=ws, qs=None, wc=np.ones(L), qc=None, wx=None))
    f, t, ln, k, nn = chain_net()
    rs = RefScenario.from_links(R, nn, f, t, ln, k).configure(8, 2, 20, 10)
    record_case(rs, flat_params(4), 5, 0, 20, 10, 2, True, 0.01, None, name="engine_chain_dn2",
                loss=dict(ws=None, qs=None, wc=np.ones(4), qc=None, wx=None))
    # test_engine.cpp:127-145: one step, two agents -> {5, 25}
    rs = RefScenario.from_links(R, 2, [0], [1], [100.0], [0]).configure(0, 1, 1, 1, fit=False,
                                                                        custom_init=([0, 0], [0.0, 10.0]))
    record_case(rs, flat_params(1, 15.0), 1, 0, 1, 1, 1, True, 0.01, np.random.default_rng(0), name="engine_two_agent")

    # C1: 4x4 grid, 1000 veh, dn=1, 30 min; gradient over 900 steps
    grid_case("c1_forward", 4, 400.0, 42, 1000, 1, 1800, 300, 3, 7, states=False, grad=False, full_cum=False)
    grid_case("c1_gradient", 4, 400.0, 42, 1000, 1, 900, 300, 3, 7, noise=3, states=False)
    grid_case("c1_gradient_notg", 4, 400.0, 42, 1000, 1, 600, 300, 3, 7, noise=5, tg=False, states=False)
    grid_case("grid5_dn4_tau03", 5, 350.0, 9, 2000, 4, 300, 300, 4, 11, noise=2, gt=0.3, states=True)
    grid_case("grid6_dn2_tau1", 6, 300.0, 11, 2400, 2, 240, 120, 5, 13, noise=1, gt=1.0, states=True)
    # calibration loss (mse_loss_builder, optimization.cpp:84-101)
    rs = RefScenario.grid(R, 4, 400.0, 42, 1000.0).configure(1000, 1, 600, 300)
    truth = rs.sample_parameters(42)
    mean = rs.sample_parameters(0, True)
    tr = rs.forward(truth, 7, 0)
    obs_ids = np.array([j for j in range(rs.n_links) if j % 5 != 0], np.int32)
    obs = tr["cum_per_step"][299::300][:, obs_ids] * 1.0
    loss, grads = rs.gradient_mse(mean, 7, 1, obs_ids, obs)
    save("c1_mse", obs_ids=obs_ids, obs=obs, params=params_arrays(mean), loss=np.float64(loss), grads=grads,
         meta=np.array([7, 1, 600, 300, 1, 1], np.float64))
    # random ring+chord networks with custom initial states (ties, arrived heads)
    for i, (dn, tg, gt) in enumerate([(1, True, 0.01), (1, False, 0.01), (3, True, 0.3), (2, True, 1.0),
                                      (1, True, 5.0), (1, True, 0.01)]):
        custom_case(f"ring_{i}", 100 + i, 10 + 2 * i, 6 + i, 60 + 20 * i, dn, 90 if dn == 1 else 60, 30 * dn,
                    tg, gt)
    # C3 (Chicago-scale) gradient over 2 steps: the 10^10-scale beta/alpha/cost blocks
    rs = RefScenario.grid(R, 23, 1609.34, 42, 1000.0).configure(1000020, 30, 2, 30)
    p = rs.sample_parameters(3)
    rng = np.random.default_rng(23)
    L, N = rs.n_links, rs.n_agents
    ws, wx = rng.normal(size=(2, L)), rng.normal(size=N)
    g = rs.gradient(p, 7, 0, 1, ws=ws, wx=wx)
    save("c3_gradient_2step", loss_ws=ws, loss_wx=wx, grads=g["grads"], loss=np.float64(g["loss"]),
         cum_final=g["cum_final"], link=g["link"], pos=g["pos"], meta=np.array([7, 0, 2, 30, 30, 1], np.float64))


if __name__ == "__main__":
    if sys.argv[1:] == ["optim"]:
        optim_cases()
    elif sys.argv[1:] == ["observe"]:
        observe_cases()
        pipeline_case()
    else:
        main()
        optim_cases()
        observe_cases()
        pipeline_case()
