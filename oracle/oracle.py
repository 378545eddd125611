"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes access to the two CPU oracles built by ``oracle/Makefile``:

* ``RefLib``  -> ``oracle/_ref/libdtsim_ref.so``: the UNMODIFIED reference
  sources (/root/reference/proj/src) behind ``oracle/ref_shim.cpp``.  Present
  only where it was built (this container, and the GPU box when the built .so
  travelled with the snapshot).
* ``PortLib`` -> ``oracle/_ref/libdtsim_port.so``: the plain-C restatement in
  ``oracle/dtsim_port.c`` (always buildable; pinned against RefLib and the
  committed golden fixtures in ``tests/golden``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdtsim_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libdtsim_port.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u64 = C.c_uint64


def fnv1a64(*arrays: np.ndarray) -> int:
    """FNV-1a 64 over the raw bytes of the arrays, in order (SURVEY §8c KATs)."""
    h = 0xCBF29CE484222325
    for a in arrays:
        for byte in np.ascontiguousarray(a).tobytes():
            h ^= byte
            h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv1a64_fast(*arrays: np.ndarray) -> int:
    """Vectorised FNV-1a 64 (same result as fnv1a64, usable on MB-sized arrays)."""
    data = b"".join(np.ascontiguousarray(a).tobytes() for a in arrays)
    h = 0xCBF29CE484222325
    prime = 0x100000001B3
    mask = 0xFFFFFFFFFFFFFFFF
    for byte in data:  # python loop is the only exact way; still fine for <=10 MB
        h = ((h ^ byte) * prime) & mask
    return h


def fnv1a64_c(*arrays: np.ndarray) -> int:
    """fnv1a64 computed by the C port (for arrays of hundreds of MB)."""
    lib = PortLib().lib
    h = 0xCBF29CE484222325
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = lib.port_fnv1a64(a.ctypes.data, a.nbytes, h)
    return int(h)


def grid_links(n: int, length: float):
    """The synthetic grid generator of SURVEY §8d: for each (r, c) in row-major
    order push the east pair then the south pair."""
    frm, to = [], []
    for r in range(n):
        for c in range(n):
            if c + 1 < n:
                frm += [r * n + c, r * n + c + 1]
                to += [r * n + c + 1, r * n + c]
            if r + 1 < n:
                frm += [r * n + c, (r + 1) * n + c]
                to += [(r + 1) * n + c, r * n + c]
    return np.array(frm, np.int32), np.array(to, np.int32), np.full(len(frm), float(length))


@dataclass
class Params:
    u: np.ndarray
    kappa: np.ndarray
    beta: np.ndarray
    alpha: np.ndarray
    cost: np.ndarray

    def arrays(self):
        return [np.ascontiguousarray(x, dtype=np.float64) for x in (self.u, self.kappa, self.beta, self.alpha, self.cost)]


class RefLib:
    """The reference itself (compiled from /root/reference sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_fork.restype = u64
        L.ref_rng_fork.argtypes = [u64, u64]
        L.ref_rng_bits.restype = u64
        L.ref_rng_bits.argtypes = [u64, u64, u64, u64]
        L.ref_rng_uniform.restype = C.c_double
        L.ref_rng_uniform.argtypes = [u64, u64, u64, u64]
        L.ref_gumbel.restype = C.c_double
        L.ref_gumbel.argtypes = [u64, u64, C.c_int, C.c_int]
        L.ref_scenario_links.restype = C.c_void_p
        L.ref_scenario_links.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp, _ip]
        L.ref_scenario_grid.restype = C.c_void_p
        L.ref_scenario_grid.argtypes = [C.c_int, C.c_double, u64, C.c_double]
        L.ref_scenario_tntp.restype = C.c_void_p
        L.ref_scenario_tntp.argtypes = [C.c_char_p, C.c_double, u64, C.c_double]
        L.ref_scenario_attach_virtual.argtypes = [C.c_void_p, u64, C.c_double]
        L.ref_scenario_free.argtypes = [C.c_void_p]
        L.ref_scenario_config.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int]
        L.ref_scenario_custom_init.argtypes = [C.c_void_p, C.c_int, _ip, _dp]
        L.ref_fit_inflow_queues.argtypes = [C.c_void_p]
        for f in ("ref_n_links", "ref_n_nodes", "ref_n_agents"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_links.argtypes = [C.c_void_p, _ip, _ip, _dp, _ip]
        L.ref_adjacency.argtypes = [C.c_void_p, _dp]
        L.ref_sample_parameters.argtypes = [C.c_void_p, u64, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.ref_seed_agents.argtypes = [C.c_void_p, _ip, _dp]
        L.ref_steps_for_minutes.argtypes = [C.c_int, C.c_double, C.c_double]
        vp = C.c_void_p
        L.ref_forward.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, _dp, _ip, _dp, vp, vp, vp]
        L.ref_gradient.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, C.c_int,
                                   vp, vp, vp, vp, vp, vp, _dp, vp, vp, vp, vp, vp, vp]
        L.ref_gradient_mse.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, C.c_int, _ip, C.c_int, _dp, vp, _dp]
        L.ref_synthesize_observations.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_double, C.c_double, u64,
                                                  C.POINTER(C.c_int), _ip, _dp]
        L.ref_count_metrics.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_int, _ip, _dp, _dp,
                                        C.POINTER(C.c_int)]
        L.ref_series_to_csv.restype = C.c_long
        L.ref_series_to_csv.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_char_p, C.c_long]
        L.ref_calibrate.argtypes = [vp, C.c_int, _ip, C.c_int, _dp, _dp, _dp, _ip, u64, vp, vp, vp, vp, vp,
                                    _dp, _dp, _ip, _ip, _dp]
        L.ref_optimize_control.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_double, _dp, _ip,
                                           C.c_double, u64, _dp, _dp, _ip, _ip, _dp]

        # FD-validation instrumentation (row f4)
        L.ref_scenario_set_soft.argtypes = [vp, C.c_int]
        L.ref_surrogate_new.restype = vp
        L.ref_surrogate_free.argtypes = [vp]
        L.ref_surrogate_set_replay.argtypes = [vp, C.c_int]
        L.ref_surrogate_rewind.argtypes = [vp]
        L.ref_surrogate_sizes.argtypes = [vp, C.POINTER(C.c_long)]
        L.ref_forward_traced.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, vp, C.c_int, vp, vp, vp,
                                         C.POINTER(u64)]
        L.ref_gradient_traced.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, C.c_int, vp, C.c_int, vp, _dp,
                                          vp, C.POINTER(u64)]
        L.ref_run_gradcheck.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, u64, _dp, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), _dp]

    def run_gradcheck(self, draws=20, steps=20, agents=5, tol=1e-4, seed=42):
        """run_gradcheck (pipeline.cpp:499-585) of the reference."""
        mx = np.zeros(1)
        red, ps = C.c_int(0), C.c_int(0)
        per = np.zeros(max(draws, 1))
        self.check(self.lib.ref_run_gradcheck(draws, steps, agents, tol, seed, mx, C.byref(red), C.byref(ps), per))
        return dict(max_rel_err=float(mx[0]), redraws=red.value, passed=bool(ps.value), per_draw_max=per[:draws])

    def err(self) -> str:
        return self.lib.ref_last_error().decode()

    # ---- observation / output side (observation.cpp:46-83, optimization.cpp:297-336,
    # pipeline.cpp:113-127) ------------------------------------------------------------
    def synthesize_observations(self, ids, vals, interval_s, noise_frac, coverage, seed):
        ids = np.ascontiguousarray(ids, np.int32)
        vals = np.ascontiguousarray(vals, np.float64)
        k, n = vals.shape
        m = C.c_int()
        oi = np.zeros(max(n, 1), np.int32)
        ov = np.zeros(max(k * n, 1))
        self.check(self.lib.ref_synthesize_observations(k, n, ids, vals.ravel(), interval_s, noise_frac, coverage,
                                                        seed, C.byref(m), oi, ov))
        mm = m.value
        return oi[:mm].copy(), ov[:k * mm].reshape(k, mm).copy()

    def count_metrics(self, sim_ids, sim_vals, truth_ids, truth_vals):
        a = [np.ascontiguousarray(x, t) for x, t in ((sim_ids, np.int32), (sim_vals, np.float64),
                                                     (truth_ids, np.int32), (truth_vals, np.float64))]
        out3 = np.zeros(3)
        npairs = C.c_int()
        self.check(self.lib.ref_count_metrics(a[1].shape[0], len(a[0]), a[0], a[1].ravel(), a[3].shape[0], len(a[2]),
                                              a[2], a[3].ravel(), out3, C.byref(npairs)))
        return dict(mae=float(out3[0]), pearson_r=float(out3[1]), r_defined=bool(out3[2]), n_pairs=npairs.value)

    def series_to_csv(self, ids, vals, interval_s) -> str:
        ids = np.ascontiguousarray(ids, np.int32)
        vals = np.ascontiguousarray(vals, np.float64)
        n = self.lib.ref_series_to_csv(vals.shape[0], len(ids), ids, vals.ravel(), interval_s, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_series_to_csv(vals.shape[0], len(ids), ids, vals.ravel(), interval_s, buf, n + 1)
        return buf.value.decode()

    def check(self, rc: int):
        if rc != 0:
            raise RuntimeError(self.err())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RefScenario:
    """A reference Scenario object (network + SimConfig + demand)."""

    def __init__(self, lib: RefLib, handle):
        if not handle:
            raise RuntimeError(lib.err())
        self.lib, self.h = lib, handle

    def __del__(self):
        try:
            self.lib.lib.ref_scenario_free(self.h)
        except Exception:
            pass

    @classmethod
    def grid(cls, lib: RefLib, n: int, length: float, net_seed: int = 42, virt_len: float = 1000.0):
        return cls(lib, lib.lib.ref_scenario_grid(n, length, net_seed, virt_len))

    @classmethod
    def tntp(cls, lib: RefLib, text: str, unit_scale: float, net_seed: int = 42, virt_len: float = 1000.0):
        """parse_tntp_text + attach_virtual_links (build_network, pipeline.cpp:165-170).

        The reference's parser (its ``istream >> double``) crashes inside a
        process that has numpy's bundled runtime libraries loaded, so the text
        is parsed by the reference in a numpy-free subprocess; its physical
        links are rebuilt here with make_network (network.cpp:238-247 — the
        same Network parse_tntp_text returns) and the virtual links attached
        in-process.
        """
        import json
        import subprocess
        import sys

        # physical links only: parse without attaching (virtual links are appended after them)
        code = ("import ctypes as C, json, sys\n"
                f"L = C.CDLL({lib.path!r})\n"
                "L.ref_tntp_physical.restype = C.c_int\n"
                "L.ref_tntp_physical.argtypes = [C.c_char_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]\n"
                "L.ref_last_error.restype = C.c_char_p\n"
                "txt = sys.stdin.buffer.read()\n"
                "n = L.ref_tntp_physical(txt, float(sys.argv[1]), None, None, None, None)\n"
                "assert n >= 0, L.ref_last_error()\n"
                "f, t = (C.c_int * n)(), (C.c_int * n)()\n"
                "ln = (C.c_double * n)()\n"
                "nn = C.c_int(0)\n"
                "L.ref_tntp_physical(txt, float(sys.argv[1]), f, t, ln, C.byref(nn))\n"
                "print(json.dumps(dict(n_nodes=nn.value, frm=list(f), to=list(t), length=[x.hex() for x in ln])))\n")
        r = subprocess.run([sys.executable, "-c", code, repr(float(unit_scale))], input=text.encode(),
                           capture_output=True, check=True)
        d = json.loads(r.stdout)
        n = len(d["frm"])
        sc = cls.from_links(lib, d["n_nodes"], d["frm"], d["to"], [float.fromhex(x) for x in d["length"]],
                            [0] * n)
        lib.check(lib.lib.ref_scenario_attach_virtual(sc.h, net_seed, virt_len))
        return sc

    @classmethod
    def from_links(cls, lib: RefLib, n_nodes, frm, to, length, kind):
        frm = np.ascontiguousarray(frm, np.int32)
        return cls(lib, lib.lib.ref_scenario_links(n_nodes, len(frm), frm, np.ascontiguousarray(to, np.int32),
                                                   np.ascontiguousarray(length, np.float64),
                                                   np.ascontiguousarray(kind, np.int32)))

    def configure(self, n_vehicles, delta_n=1, horizon_steps=0, obs_interval_s=300, tau=1.0,
                  gumbel_tau=0.01, tg=True, fit=True, custom_init=None):
        L = self.lib.lib
        L.ref_scenario_config(self.h, n_vehicles, delta_n, tau, gumbel_tau, int(tg), horizon_steps, obs_interval_s)
        if custom_init is not None:
            lk, ps = custom_init
            L.ref_scenario_custom_init(self.h, len(lk), np.ascontiguousarray(lk, np.int32),
                                       np.ascontiguousarray(ps, np.float64))
        if fit:
            self.lib.check(L.ref_fit_inflow_queues(self.h))
        self.horizon_steps = horizon_steps
        return self

    @property
    def n_links(self):
        return self.lib.lib.ref_n_links(self.h)

    @property
    def n_nodes(self):
        return self.lib.lib.ref_n_nodes(self.h)

    @property
    def n_agents(self):
        n = self.lib.lib.ref_n_agents(self.h)
        if n < 0:
            raise RuntimeError(self.lib.err())
        return n

    def links(self):
        Ln = self.n_links
        f, t, k = (np.zeros(Ln, np.int32) for _ in range(3))
        ln = np.zeros(Ln)
        self.lib.lib.ref_links(self.h, f, t, ln, k)
        return f, t, ln, k

    def adjacency(self):
        Ln = self.n_links
        a = np.zeros(Ln * Ln)
        self.lib.lib.ref_adjacency(self.h, a)
        return a.reshape(Ln, Ln)

    def sample_parameters(self, seed: int, mean_mode: bool = False) -> Params:
        Ln = self.n_links
        arr = [np.zeros(Ln) for _ in range(5)]
        self.lib.check(self.lib.lib.ref_sample_parameters(self.h, seed, int(mean_mode), *arr))
        return Params(*arr)

    def seed_agents(self):
        N = self.n_agents
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        self.lib.check(self.lib.lib.ref_seed_agents(self.h, lk, ps))
        return lk, ps

    def forward(self, p: Params, seed: int, noise_iteration: int = 0, record_states=False):
        Ln, N, T = self.n_links, self.n_agents, self.horizon_steps
        cum = np.zeros(T * Ln)
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        sl = np.zeros(T * N, np.int32) if record_states else None
        sp = np.zeros(T * N) if record_states else None
        wall = np.zeros(1)
        self.lib.check(self.lib.lib.ref_forward(self.h, *p.arrays(), seed, noise_iteration, cum, lk, ps,
                                                _ptr(sl), _ptr(sp), _ptr(wall)))
        out = dict(cum_per_step=cum.reshape(T, Ln), link=lk, pos=ps, wall=float(wall[0]))
        if record_states:
            out["states_link"], out["states_pos"] = sl.reshape(T, N), sp.reshape(T, N)
        return out

    def gradient(self, p: Params, seed: int, noise_iteration: int = 0, mode: int = 1,
                 ws=None, qs=None, wc=None, qc=None, wx=None):
        Ln, N, T = self.n_links, self.n_agents, self.horizon_steps
        f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64).ravel()
        ws, qs, wc, qc, wx = map(f, (ws, qs, wc, qc, wx))
        loss = np.zeros(1)
        grads = np.zeros(5 * Ln)
        snaps = np.zeros(max(T, 1) * Ln)
        nsn = np.zeros(1, np.int32)
        cumf = np.zeros(Ln)
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        wall = np.zeros(1)
        self.lib.check(self.lib.lib.ref_gradient(self.h, *p.arrays(), seed, noise_iteration, mode,
                                                 _ptr(ws), _ptr(qs), _ptr(wc), _ptr(qc), _ptr(wx),
                                                 _ptr(loss), grads, _ptr(snaps), _ptr(nsn), _ptr(cumf),
                                                 _ptr(lk), _ptr(ps), _ptr(wall)))
        k = int(nsn[0])
        return dict(loss=float(loss[0]), grads=grads.reshape(5, Ln), snapshots=snaps[: k * Ln].reshape(k, Ln),
                    cum_final=cumf, link=lk, pos=ps, wall=float(wall[0]))

    # ---- FD-validation instrumentation (row f4) ------------------------------
    def set_soft(self, soft: bool):
        self.lib.lib.ref_scenario_set_soft(self.h, int(soft))
        return self

    def forward_traced(self, p: Params, seed: int, noise_iteration: int = 0, surrogate=None,
                       trace_branches=True):
        Ln, N, T = self.n_links, self.n_agents, self.horizon_steps
        cum = np.zeros(T * Ln)
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        h = u64(0)
        self.lib.check(self.lib.lib.ref_forward_traced(
            self.h, *p.arrays(), seed, noise_iteration, surrogate.h if surrogate else None, int(trace_branches),
            _ptr(cum), _ptr(lk), _ptr(ps), C.byref(h)))
        return dict(cum_per_step=cum.reshape(T, Ln), link=lk, pos=ps, hash=int(h.value))

    def gradient_traced(self, p: Params, seed: int, noise_iteration: int = 0, mode: int = 0, surrogate=None,
                        trace_branches=True):
        Ln = self.n_links
        loss, grads, cumf = np.zeros(1), np.zeros(5 * Ln), np.zeros(Ln)
        h = u64(0)
        self.lib.check(self.lib.lib.ref_gradient_traced(
            self.h, *p.arrays(), seed, noise_iteration, mode, surrogate.h if surrogate else None,
            int(trace_branches), _ptr(loss), grads, _ptr(cumf), C.byref(h)))
        return dict(loss=float(loss[0]), grads=grads.reshape(5, Ln), cum_final=cumf, hash=int(h.value))

    def gradient_mse(self, p: Params, seed: int, noise_iteration: int, obs_ids, obs_vals):
        Ln = self.n_links
        obs_ids = np.ascontiguousarray(obs_ids, np.int32)
        obs_vals = np.ascontiguousarray(obs_vals, np.float64)
        loss = np.zeros(1)
        grads = np.zeros(5 * Ln)
        self.lib.check(self.lib.lib.ref_gradient_mse(self.h, *p.arrays(), seed, noise_iteration, len(obs_ids),
                                                     obs_ids, obs_vals.shape[0], obs_vals.ravel(),
                                                     _ptr(loss), grads))
        return float(loss[0]), grads.reshape(5, Ln)


    # ---- optimisation loops (src/optimization.cpp:122-295) -----------------
    @staticmethod
    def _opt(cfg: dict):
        d = dict(lr=0.1, weight_decay=1e-5, beta1=0.9, beta2=0.999, eps=1e-8, patience=20,
                 max_iterations=200, resample_noise=True, noise_draws=1)
        d.update(cfg or {})
        opt = np.array([d["lr"], d["weight_decay"], d["beta1"], d["beta2"], d["eps"]])
        iopt = np.array([d["patience"], d["max_iterations"], int(d["resample_noise"]), d["noise_draws"]], np.int32)
        return d, opt, iopt

    def calibrate(self, obs_ids, obs_vals, seed: int, bounds=None, cfg: dict = None, init: "Params" = None):
        """The reference's calibrate(); returns the CalibrationResult fields.
        bounds = (u_lo, u_hi, kappa_lo, kappa_hi, beta_lo, beta_hi, alpha_lo, alpha_hi)."""
        Ln = self.n_links
        d, opt, iopt = self._opt(cfg)
        b = np.ascontiguousarray(bounds if bounds is not None else
                                 (13.9, 22.2, 0.18, 0.22, 0.0, 5.0, 0.01, 5.0), np.float64)
        ids = np.ascontiguousarray(obs_ids, np.int32)
        vals = np.ascontiguousarray(obs_vals, np.float64).reshape(-1, len(ids))
        best = np.zeros(5 * Ln)
        bl = np.zeros(1)
        bi, its = np.zeros(1, np.int32), np.zeros(1, np.int32)
        curve = np.zeros(max(d["max_iterations"], 1))
        ia = init.arrays() if init is not None else [None] * 5
        rc = self.lib.lib.ref_calibrate(self.h, len(ids), ids, vals.shape[0], vals.ravel(), b, opt, iopt, seed,
                                        *(_ptr(a) for a in ia), best, bl, bi, its, curve)
        if rc == 3:
            raise FloatingPointError(self.lib.err())
        self.lib.check(rc)
        n = int(its[0])
        return dict(best=best.reshape(5, Ln), best_loss=float(bl[0]), best_iteration=int(bi[0]),
                    iterations=n, loss_curve=curve[:n].copy())

    def optimize_control(self, p: "Params", target: int, desired: float, seed: int, cfg: dict = None,
                         cost_floor: float = 0.05):
        Ln = self.n_links
        d, opt, iopt = self._opt(cfg)
        cost = np.zeros(Ln)
        out3 = np.zeros(3)
        its, stall = np.zeros(1, np.int32), np.zeros(1, np.int32)
        curve = np.zeros(max(d["max_iterations"], 1))
        rc = self.lib.lib.ref_optimize_control(self.h, *p.arrays(), target, desired, opt, iopt, cost_floor, seed,
                                               cost, out3, its, stall, curve)
        if rc == 3:
            raise FloatingPointError(self.lib.err())
        self.lib.check(rc)
        n = int(its[0])
        return dict(cost=cost, achieved=float(out3[0]), gap_fraction=float(out3[1]), best_loss=float(out3[2]),
                    iterations=n, zero_gradient_stall=bool(stall[0]), loss_curve=curve[:n].copy())


# ---------------------------------------------------------------------------
# The plain-C port (oracle/dtsim_port.c)
# ---------------------------------------------------------------------------
class _PortNet(C.Structure):
    _fields_ = [("n_links", C.c_int), ("succ_off", C.c_void_p), ("succ", C.c_void_p), ("length", C.c_void_p),
                ("delta_n", C.c_int), ("tau", C.c_double), ("sentinel", C.c_double), ("gumbel_tau", C.c_double),
                ("trajectory_grafting", C.c_int)]


class _PortParams(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("u", "kappa", "beta", "alpha", "cost")]


def csr_from_links(frm, to):
    """Successor CSR of the link adjacency (network.cpp:28-35: j follows i iff
    i != j and to_node[i] == from_node[j]), successors ascending by link id."""
    frm = np.asarray(frm)
    to = np.asarray(to)
    L = len(frm)
    by_from = {}
    for j in range(L):
        by_from.setdefault(int(frm[j]), []).append(j)
    off = [0]
    succ = []
    for i in range(L):
        s = [j for j in by_from.get(int(to[i]), []) if j != i]
        succ += sorted(s)
        off.append(len(succ))
    return np.array(off, np.int32), np.array(succ, np.int32)


class PortLib:
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.port_last_error.restype = C.c_char_p
        L.port_rng_fork.restype = u64
        L.port_rng_fork.argtypes = [u64, u64]
        L.port_rng_bits.restype = u64
        L.port_rng_bits.argtypes = [u64, u64, u64, u64]
        L.port_rng_uniform.restype = C.c_double
        L.port_rng_uniform.argtypes = [u64, u64, u64, u64]
        L.port_gumbel.restype = C.c_double
        L.port_gumbel.argtypes = [u64, u64, u64, u64]
        L.port_fnv1a64.restype = u64
        L.port_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, u64]
        vp = C.c_void_p
        L.port_forward.argtypes = [vp, vp, u64, u64, C.c_int, _ip, _dp, C.c_int, _dp, _ip, _dp, vp, vp]
        L.port_gradient.argtypes = [vp, vp, u64, u64, C.c_int, _ip, _dp, C.c_int, C.c_int,
                                    vp, vp, vp, vp, vp, vp, _dp, vp, vp, vp, vp, vp]
        L.port_gradient_seeds.argtypes = [vp, vp, u64, u64, C.c_int, _ip, _dp, C.c_int, C.c_int, _dp, _dp, _dp, _dp]

    def err(self):
        return self.lib.port_last_error().decode()


class PortScenario:
    """A scenario for the C port: links + config + initial compact state."""

    def __init__(self, lib: PortLib, frm, to, length, delta_n=1, tau=1.0, gumbel_tau=0.01, tg=True,
                 sentinel=99999.0, link0=None, pos0=None, horizon_steps=0, obs_interval_s=300):
        self.lib = lib
        self.length = np.ascontiguousarray(length, np.float64)
        self.succ_off, self.succ = csr_from_links(frm, to)
        self.L = len(self.length)
        self.delta_n, self.tau = delta_n, tau
        self._net = _PortNet(self.L, self.succ_off.ctypes.data, self.succ.ctypes.data, self.length.ctypes.data,
                             delta_n, tau, sentinel, gumbel_tau, int(tg))
        self.link0 = np.ascontiguousarray(link0, np.int32)
        self.pos0 = np.ascontiguousarray(pos0, np.float64)
        self.N = len(self.link0)
        self.horizon_steps = horizon_steps
        dt = tau * delta_n
        self.spi = int(round(obs_interval_s / dt))

    @classmethod
    def from_ref(cls, lib: PortLib, rs: "RefScenario", **kw):
        f, t, ln, _ = rs.links()
        lk, ps = rs.seed_agents()
        return cls(lib, f, t, ln, link0=lk, pos0=ps, **kw)

    def _p(self, p: Params):
        arrs = p.arrays()
        self._keep = arrs
        return _PortParams(*[a.ctypes.data for a in arrs])

    def forward(self, p: Params, seed: int, noise_iteration: int = 0, record_states=False):
        T, L, N = self.horizon_steps, self.L, self.N
        cum = np.zeros(T * L)
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        sl = np.zeros(T * N, np.int32) if record_states else None
        sp = np.zeros(T * N) if record_states else None
        pp = self._p(p)
        rc = self.lib.lib.port_forward(C.byref(self._net), C.byref(pp), seed, noise_iteration, N, self.link0,
                                       self.pos0, T, cum, lk, ps, _ptr(sl), _ptr(sp))
        if rc:
            raise RuntimeError(self.lib.err())
        out = dict(cum_per_step=cum.reshape(T, L), link=lk, pos=ps)
        if record_states:
            out["states_link"], out["states_pos"] = sl.reshape(T, N), sp.reshape(T, N)
        return out

    def gradient(self, p: Params, seed: int, noise_iteration: int = 0, ws=None, qs=None, wc=None, qc=None, wx=None):
        T, L, N = self.horizon_steps, self.L, self.N
        f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64).ravel()
        ws, qs, wc, qc, wx = map(f, (ws, qs, wc, qc, wx))
        loss = np.zeros(1)
        grads = np.zeros(5 * L)
        snaps = np.zeros(max(T, 1) * L)
        nsn = np.zeros(1, np.int32)
        cumf = np.zeros(L)
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        pp = self._p(p)
        rc = self.lib.lib.port_gradient(C.byref(self._net), C.byref(pp), seed, noise_iteration, N, self.link0,
                                        self.pos0, T, self.spi, _ptr(ws), _ptr(qs), _ptr(wc), _ptr(qc), _ptr(wx),
                                        _ptr(loss), grads, _ptr(snaps), _ptr(nsn), _ptr(cumf), _ptr(lk), _ptr(ps))
        if rc:
            raise RuntimeError(self.lib.err())
        k = int(nsn[0])
        return dict(loss=float(loss[0]), grads=grads.reshape(5, L), snapshots=snaps[: k * L].reshape(k, L),
                    cum_final=cumf, link=lk, pos=ps)

    def gradient_seeds(self, p: Params, seed: int, noise_iteration: int, snap_seed, cum_seed, x_seed):
        L = self.L
        grads = np.zeros(5 * L)
        pp = self._p(p)
        rc = self.lib.lib.port_gradient_seeds(C.byref(self._net), C.byref(pp), seed, noise_iteration, self.N,
                                              self.link0, self.pos0, self.horizon_steps, self.spi,
                                              np.ascontiguousarray(snap_seed, np.float64).ravel(),
                                              np.ascontiguousarray(cum_seed, np.float64),
                                              np.ascontiguousarray(x_seed, np.float64), grads)
        if rc:
            raise RuntimeError(self.lib.err())
        return grads.reshape(5, L)


class RefSurrogate:
    """The reference's SurrogateTrace (car_following.hpp:23-29)."""

    def __init__(self, lib: RefLib):
        self.lib, self.h = lib, lib.lib.ref_surrogate_new()

    def __del__(self):
        try:
            self.lib.lib.ref_surrogate_free(self.h)
        except Exception:
            pass

    def set_replay(self, on: bool):
        self.lib.lib.ref_surrogate_set_replay(self.h, int(on))

    def rewind(self):
        self.lib.lib.ref_surrogate_rewind(self.h)

    def sizes(self):
        s = (C.c_long * 4)()
        self.lib.lib.ref_surrogate_sizes(self.h, s)
        return list(s)
