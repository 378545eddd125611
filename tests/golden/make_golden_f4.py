"""Golden fixtures for the FD-validation instrumentation,
generated from the REFERENCE ITSELF (oracle/_ref/libdtsim_ref.so built from
/root/reference/proj/src by `make -C oracle ref`):

* f4_trace_*.npz   simulate_forward with ForwardOptions.trace_branches
                   (branch_trace.hpp) on hard-choice networks: BranchTrace
                   hash, counts, final state.
* f4_chain_*.npz   run_gradcheck's chain (pipeline.cpp:486-496) with
                   soft_choices: the recording gradient run (FullTape grads,
                   hash) and surrogate replays (car_following.cpp:17-94) of
                   central-difference probes, plus off-path probes.
* f4_gradcheck.npz run_gradcheck (pipeline.cpp:499-585) reports.

    python tests/golden/make_golden_f4.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Params, RefLib, RefScenario, RefSurrogate, csr_from_links  # noqa: E402

R = RefLib()
U64 = np.uint64


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def net_arrays(rs):
    f, t, ln, k = rs.links()
    return dict(frm=f, to=t, length=ln, kind=k, n_nodes=np.int32(rs.n_nodes))


def trace_case(name, rs, p, seed, noise, T, dn, tg, gt):
    lk0, ps0 = rs.seed_agents()
    fw = rs.forward_traced(p, seed, noise, None, True)
    plain = rs.forward(p, seed, noise)
    assert np.array_equal(plain["cum_per_step"], fw["cum_per_step"])  # tracing changes nothing
    save(name, **net_arrays(rs), params=np.stack(p.arrays()), link0=lk0, pos0=ps0,
         meta=np.array([seed, noise, T, dn, int(tg)], np.float64), gumbel_tau=np.float64(gt),
         hash=U64(fw["hash"]), cum_per_step=fw["cum_per_step"], link=fw["link"], pos=fw["pos"])


def trace_cases():
    # C1-like 4x4 grid (hard choices, sinks, merges), 300 steps
    rs = RefScenario.grid(R, 4, 400.0, 42, 1000.0).configure(1000, 1, 300, 300)
    trace_case("f4_trace_c1", rs, rs.sample_parameters(3), 7, 0, 300, 1, True, 0.01)
    # 3x3 grid, platoons of 2, TG off, warm temperature (near-tie rich)
    rs = RefScenario.grid(R, 3, 250.0, 5, 600.0).configure(400, 2, 150, 30, gumbel_tau=1.0, tg=False)
    trace_case("f4_trace_g3", rs, rs.sample_parameters(11), 3, 2, 150, 2, False, 1.0)
    # ring + chords with a custom initial state (ties, negative positions, sinks)
    d = np.load(os.path.join(HERE, "ring_2.npz"))
    seed, noise, T, spi, dn, tg = d["meta"]
    rs = RefScenario.from_links(R, int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"]).configure(
        0, int(dn), int(T), int(spi), gumbel_tau=float(d["gumbel_tau"]), tg=bool(tg), fit=False,
        custom_init=(d["link0"], d["pos0"]))
    trace_case("f4_trace_ring2", rs, Params(*d["params"]), int(seed), int(noise), int(T), int(dn), bool(tg),
               float(d["gumbel_tau"]))


def chain(n_phys=3, link_len=300.0, inflow_len=100.0):
    """make_chain_network (pipeline.cpp:486-496)."""
    frm = [n_phys + 1] + list(range(n_phys)) + [n_phys]
    to = [0] + list(range(1, n_phys + 1)) + [n_phys + 2]
    ln = [inflow_len] + [link_len] * n_phys + [inflow_len]
    kind = [1] + [0] * n_phys + [2]
    return np.array(frm, np.int32), np.array(to, np.int32), np.array(ln), np.array(kind, np.int32), n_phys + 3


def gradcheck_params(seed, attempt, L):
    """run_gradcheck's parameter draw (pipeline.cpp:512-520)."""
    lib = R.lib
    pr = lib.ref_rng_fork(seed, 9000 + attempt)
    uni = lambda lo, hi, a, l: lo + (hi - lo) * lib.ref_rng_uniform(pr, a, l, 0)  # noqa: E731
    rng = [(13.9, 22.2), (0.18, 0.22), (0.0, 5.0), (0.01, 5.0), (0.5, 2.0)]
    return Params(*[np.array([uni(lo, hi, b, l) for l in range(L)]) for b, (lo, hi) in enumerate(rng)])


def chain_case(name, agents, steps, seed, attempt, tg=True, hscale=1e-5, extra_h=()):
    f, t, ln, k, nn = chain()
    rs = RefScenario.from_links(R, nn, f, t, ln, k).configure(agents, 1, steps, steps, tg=tg, fit=False)
    rs.set_soft(True)
    L = rs.n_links
    p = gradcheck_params(seed, attempt, L)
    tr = RefSurrogate(R)
    g = rs.gradient_traced(p, seed, 0, 0, tr, True)
    # the recording forward alone (same hash, plain values)
    rec_fw = rs.forward_traced(p, seed, 0, None, True)
    soft_plain_hash = rec_fw["hash"]
    tr2 = RefSurrogate(R)
    fw_rec = rs.forward_traced(p, seed, 0, tr2, True)
    tr.set_replay(True)
    probes, sums, hashes, cums, links, poss = [], [], [], [], [], []
    for h_mult in (1.0,) + tuple(extra_h):
        for b in range(5):
            for l in range(L):
                arr = [a.copy() for a in p.arrays()]
                x0 = arr[b][l]
                h = hscale * h_mult * max(1.0, abs(x0))
                for sgn in (1.0, -1.0):
                    arr2 = [a.copy() for a in arr]
                    arr2[b][l] = x0 + sgn * h
                    tr.rewind()
                    q = Params(*arr2)
                    try:
                        fw = rs.forward_traced(q, seed, 0, tr, True)
                    except RuntimeError:
                        continue  # trace misaligned: not a usable probe
                    probes.append(np.stack(arr2))
                    sums.append(float(sum(fw["cum_per_step"][-1])))
                    hashes.append(fw["hash"])
                    cums.append(fw["cum_per_step"])
                    links.append(fw["link"])
                    poss.append(fw["pos"])
    save(name, frm=f, to=t, length=ln, kind=k, n_nodes=np.int32(nn),
         meta=np.array([agents, steps, seed, attempt, int(tg)], np.float64), params=np.stack(p.arrays()),
         grads=g["grads"], cum_final=g["cum_final"], base_hash=U64(g["hash"]),
         forward_hash_soft=U64(soft_plain_hash), forward_hash_record=U64(fw_rec["hash"]),
         probe_params=np.array(probes), probe_sum=np.array(sums), probe_hash=np.array(hashes, np.uint64),
         probe_cum=np.array(cums), probe_link=np.array(links), probe_pos=np.array(poss))
    n_on = int(np.sum(np.array(hashes, np.uint64) == U64(g["hash"])))
    print(f"  {name}: {len(hashes)} probes, {n_on} on the base control path")


def gradcheck_cases():
    cfgs = [(20, 20, 5, 1e-4, 1), (5, 40, 10, 1e-4, 1), (4, 60, 21, 1e-4, 7), (3, 30, 12, 1e-9, 11)]
    out = dict(cfgs=np.array(cfgs, np.float64))
    rows = []
    for i, c in enumerate(cfgs):
        r = R.run_gradcheck(*c)
        rows.append([r["max_rel_err"], r["redraws"], int(r["passed"])])
        out[f"per_draw_{i}"] = r["per_draw_max"]
    out["report"] = np.array(rows)
    save("f4_gradcheck", **out)


if __name__ == "__main__":
    trace_cases()
    chain_case("f4_chain_a5", 5, 20, 1, 0)
    chain_case("f4_chain_a21", 21, 60, 7, 0, extra_h=(3e3,))
    chain_case("f4_chain_notg", 12, 40, 11, 2, tg=False, extra_h=(1e4,))
    gradcheck_cases()
