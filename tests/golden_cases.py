"""Load the reference-generated fixtures in tests/golden/ (see make_golden.py)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

TRAJ_CASES = ["engine_chain_ckpt", "engine_chain_dn2", "engine_two_agent", "c1_forward", "c1_gradient",
              "c1_gradient_notg", "grid5_dn4_tau03", "grid6_dn2_tau1"] + [f"ring_{i}" for i in range(6)]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def meta(d):
    seed, noise, T, spi_s, dn, tg = d["meta"]
    return dict(seed=int(seed), noise=int(noise), T=int(T), obs_s=int(spi_s), dn=int(dn), tg=bool(tg),
                gt=float(d["gumbel_tau"]))


def params_of(d, cls):
    return cls(*[np.ascontiguousarray(x) for x in d["params"]])


def loss_kwargs(d):
    return {k: d.get("loss_" + k) for k in ("ws", "qs", "wc", "qc", "wx")}


def port_scenario(port, d):
    from oracle.oracle import PortScenario

    m = meta(d)
    return PortScenario(port, d["frm"], d["to"], d["length"], delta_n=m["dn"], gumbel_tau=m["gt"], tg=m["tg"],
                        link0=d["link0"], pos0=d["pos0"], horizon_steps=m["T"], obs_interval_s=m["obs_s"])


def product_scenario(P, d):
    """The same scenario built through the product's C-ABI (make_network +
    custom_init = the fixture's initial state)."""
    m = meta(d)
    sc = P.Scenario.from_links(int(d["n_nodes"]), d["frm"], d["to"], d["length"], d["kind"])
    sc.configure(0, m["dn"], m["T"], m["obs_s"], gumbel_tau=m["gt"], trajectory_grafting=m["tg"], fit_queues=False,
                 custom_init=(d["link0"], d["pos0"]))
    return sc


def all_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
