"""Python host API over the C-ABI (include/dtg.h).

Mirrors the reference's simulator surface for this path
(/root/reference/proj/include/dtsim/{network,engine}.hpp): build a Scenario
(network + SimConfig + demand), sample LinkParams, then ``simulate_forward`` /
``simulate_gradient``.  Every call goes to libdtg.so — the C++ host layer
builds the CSR network and compact states, the sm_100a kernels run the
T-step loop and its reverse sweep.  ``Engine`` exposes the level-1 device
context directly (device-resident benchmarking, custom losses, multi-GPU).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import NetDesc, OptimizeConfig as _OptC, ParamRangesC, SimConfig, load, ptr, raise_for

PHYSICAL, VIRTUAL_INFLOW, VIRTUAL_OUTFLOW = 0, 1, 2


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class LinkParams:
    """Per-link parameter vectors (network.hpp:22-28)."""

    u: np.ndarray
    kappa: np.ndarray
    beta: np.ndarray
    alpha: np.ndarray
    cost: np.ndarray

    def arrays(self):
        return [np.ascontiguousarray(x, dtype=np.float64) for x in (self.u, self.kappa, self.beta, self.alpha, self.cost)]

    def copy(self) -> "LinkParams":
        return LinkParams(*[a.copy() for a in self.arrays()])


@dataclass
class Trajectory:
    """Trajectory (engine.hpp:61-74) with compact states."""

    cum_per_step: np.ndarray  # [T, L]
    link_final: np.ndarray    # [N]
    pos_final: np.ndarray     # [N]
    wall_seconds: float = 0.0
    states_link: Optional[np.ndarray] = None  # [T, N]
    states_pos: Optional[np.ndarray] = None
    transfers: Optional[np.ndarray] = None  # [E, 4] (step, agent, from, to); record_transfers

    @property
    def steps(self) -> int:
        return self.cum_per_step.shape[0]

    @property
    def cum_final(self) -> np.ndarray:
        return self.cum_per_step[-1] if self.steps else np.zeros(self.cum_per_step.shape[1])


@dataclass
class GradResult:
    """GradResult (engine.hpp:91-99); grads is [5, L] = u, kappa, beta, alpha, cost."""

    loss: float
    grads: np.ndarray
    snapshots: np.ndarray
    cum_final: np.ndarray
    link_final: np.ndarray
    pos_final: np.ndarray
    wall_seconds: float = 0.0

    @property
    def as_params(self) -> LinkParams:
        return LinkParams(*self.grads)


class Scenario:
    """Scenario (engine.hpp:16-34): network, SimConfig and demand."""

    def __init__(self, handle):
        self._lib = load()
        if not handle:
            raise RuntimeError(self._lib.dtg_scenario_last_error(None).decode())
        self._h = handle
        self.horizon_steps = 0
        self.delta_n = 1
        self.tau = 1.0
        self.obs_interval_s = 300

    def __del__(self):
        try:
            self._lib.dtg_scenario_free(self._h)
        except Exception:
            pass

    # ---- construction ----------------------------------------------------------
    @classmethod
    def grid(cls, n: int, length: float, net_seed: int = 42, virtual_length: float = 1000.0) -> "Scenario":
        """Synthetic n x n grid + attach_virtual_links."""
        return cls(load().dtg_scenario_grid(n, float(length), net_seed, float(virtual_length)))

    @classmethod
    def from_links(cls, n_nodes: int, from_node, to_node, length, kind) -> "Scenario":
        """make_network (network.cpp:238-247) over explicit links."""
        f = np.ascontiguousarray(from_node, np.int32)
        return cls(load().dtg_scenario_from_links(n_nodes, len(f), f, np.ascontiguousarray(to_node, np.int32),
                                                  _f64(length), np.ascontiguousarray(kind, np.int32)))

    @classmethod
    def tntp(cls, text: str, length_unit_scale: float, net_seed: int = 42,
             virtual_length: float = 1000.0) -> "Scenario":
        return cls(load().dtg_scenario_tntp(text.encode(), float(length_unit_scale), net_seed,
                                            float(virtual_length)))

    def _check(self, rc):
        raise_for(rc, self._lib.dtg_scenario_last_error(self._h).decode())

    def configure(self, n_vehicles: int = 0, delta_n: int = 1, horizon_steps: int = 0,
                  obs_interval_s: int = 300, tau: float = 1.0, gumbel_tau: float = 0.01,
                  trajectory_grafting: bool = True, fit_queues: bool = True,
                  custom_init=None) -> "Scenario":
        if custom_init is not None:
            lk, ps = custom_init
            self._check(self._lib.dtg_scenario_custom_init(self._h, len(lk), np.ascontiguousarray(lk, np.int32),
                                                           _f64(ps)))
        self._check(self._lib.dtg_scenario_configure(self._h, n_vehicles, delta_n, tau, gumbel_tau,
                                                     int(trajectory_grafting), horizon_steps, obs_interval_s,
                                                     int(fit_queues)))
        self.horizon_steps, self.delta_n, self.tau, self.obs_interval_s = horizon_steps, delta_n, tau, obs_interval_s
        self.gumbel_tau, self.trajectory_grafting = gumbel_tau, trajectory_grafting
        return self

    # ---- queries -----------------------------------------------------------------
    @property
    def n_links(self) -> int:
        return self._lib.dtg_scenario_n_links(self._h)

    @property
    def n_nodes(self) -> int:
        return self._lib.dtg_scenario_n_nodes(self._h)

    @property
    def n_agents(self) -> int:
        n = self._lib.dtg_scenario_n_agents(self._h)
        if n < 0:
            raise RuntimeError(self._lib.dtg_scenario_last_error(self._h).decode())
        return n

    @property
    def steps_per_interval(self) -> int:
        return int(round(self.obs_interval_s / (self.tau * self.delta_n)))

    @property
    def n_snapshots(self) -> int:
        return self.horizon_steps // self.steps_per_interval

    def links(self):
        L = self.n_links
        f, t, k = (np.zeros(L, np.int32) for _ in range(3))
        ln = np.zeros(L)
        self._lib.dtg_scenario_links(self._h, f, t, ln, k)
        return f, t, ln, k

    def csr(self):
        off = np.zeros(self.n_links + 1, np.int32)
        succ = np.zeros(max(1, self._lib.dtg_scenario_n_edges(self._h)), np.int32)
        self._lib.dtg_scenario_csr(self._h, off, succ)
        return off, succ[: off[-1]]

    def sample_parameters(self, seed: int, mean_mode: bool = False) -> LinkParams:
        L = self.n_links
        a = [np.zeros(L) for _ in range(5)]
        self._check(self._lib.dtg_scenario_sample_parameters(self._h, seed, int(mean_mode), *a))
        return LinkParams(*a)

    def seed_agents(self):
        N = self.n_agents
        lk, ps = np.zeros(N, np.int32), np.zeros(N)
        self._check(self._lib.dtg_scenario_seed_agents(self._h, lk, ps))
        return lk, ps

    def device_context(self):
        return self._lib.dtg_scenario_ctx(self._h)


def steps_for_minutes(delta_n: int, tau: float, minutes: float) -> int:
    n = load().dtg_steps_for_minutes(delta_n, tau, minutes)
    if n < 0:
        raise RuntimeError("horizon must be a whole number of time steps")
    return n


def _its(noise_iteration, noise_iterations):
    its = [noise_iteration] if noise_iterations is None else list(noise_iterations)
    return np.ascontiguousarray(its, dtype=np.uint64)


def transfer_events(ctx, scenario: int = 0) -> np.ndarray:
    """(step, agent, from, to) rows of the last recorded forward of a device
    context (dtg_transfer_events)."""
    lib = load()
    n = C.c_size_t()
    raise_for(lib.dtg_transfer_events(ctx, scenario, None, 0, C.byref(n)), lib.dtg_last_error(ctx).decode())
    out = np.zeros((max(n.value, 1), 4), np.int32)
    raise_for(lib.dtg_transfer_events(ctx, scenario, out.ctypes.data, n.value, C.byref(n)),
              lib.dtg_last_error(ctx).decode())
    return out[: n.value]


def link_visits(link0, transfers) -> np.ndarray:
    """Per-agent link visits [V, 4] = (agent, link, entry_step, exit_step) from
    the initial links and the transfer events; entry -1 = the initial link,
    exit -1 = still on the link at the horizon.  A completed visit's travel
    time is (exit_step - entry_step) engine steps of dt = tau * delta_n
    seconds."""
    rows, open_ = [], {}
    for a, l in enumerate(np.asarray(link0)):
        if l >= 0:
            open_[a] = len(rows)
            rows.append([a, int(l), -1, -1])
    for t, a, _frm, to in np.asarray(transfers).reshape(-1, 4):
        if a in open_:
            rows[open_[a]][3] = int(t)
        open_[int(a)] = len(rows)
        rows.append([int(a), int(to), int(t), -1])
    return np.array(rows, np.int32).reshape(-1, 4)


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (dtg_host_alloc), freed with
    the array.  Results written into such arrays (simulate_forward's `out`)
    are DMA'd from the device directly, without staging copies."""
    import weakref

    lib = load()
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    p = lib.dtg_host_alloc(max(n, 1))
    if not p:
        raise MemoryError(f"dtg_host_alloc({n}) failed")
    arr = np.frombuffer((C.c_char * max(n, 1)).from_address(p), dtype=dt, count=int(np.prod(shape))).reshape(shape)
    weakref.finalize(arr, lib.dtg_host_free, p)
    return arr


def simulate_forward(sc: Scenario, params: LinkParams, seed: int, noise_iteration: int = 0,
                     record_states: bool = False, noise_iterations: Optional[Sequence[int]] = None,
                     record_transfers: bool = False, out=None):
    """simulate_forward (engine.cpp:227-254) on the GPU.  With noise_iterations,
    all draws run batched in one device pass and a list is returned.
    record_transfers: every link change of every agent, recorded by the
    device merge (Trajectory.transfers; travel times via link_visits).
    out: optional (cum_per_step [D, T, L] float64, link_final [D, N] int32,
    pos_final [D, N] float64) arrays to write the results into, e.g. reused
    page-locked buffers from pinned_empty (the results then arrive by DMA)."""
    if record_transfers:
        sc._check(sc._lib.dtg_scenario_set_record_transfers(sc._h, 1))
        try:
            out = simulate_forward(sc, params, seed, noise_iteration, record_states, noise_iterations, out=out)
            ctx = sc.device_context()
            for d, tr in enumerate(out if isinstance(out, list) else [out]):
                tr.transfers = transfer_events(ctx, d)
            return out
        finally:
            sc._check(sc._lib.dtg_scenario_set_record_transfers(sc._h, 0))
    its = _its(noise_iteration, noise_iterations)
    D, T, L, N = len(its), sc.horizon_steps, sc.n_links, sc.n_agents
    if out is not None:
        cum, lk, ps = out
        for a, shp, dt in ((cum, (D, T, L), np.float64), (lk, (D, N), np.int32), (ps, (D, N), np.float64)):
            if a.shape != shp or a.dtype != dt or not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"out array must be a C-contiguous {np.dtype(dt).name} array of shape {shp}")
    else:
        cum = np.empty((D, T, L))  # every entry is written by the call
        lk, ps = np.empty((D, N), np.int32), np.empty((D, N))
    sl = np.zeros((D, T, N), np.int32) if record_states else None
    sp = np.zeros((D, T, N)) if record_states else None
    wall = np.zeros(1)
    sc._check(sc._lib.dtg_simulate_forward(sc._h, *params.arrays(), seed, D, its, ptr(cum), ptr(lk), ptr(ps),
                                           ptr(sl), ptr(sp), ptr(wall)))
    out = [Trajectory(cum[d], lk[d], ps[d], float(wall[0]),
                      None if sl is None else sl[d], None if sp is None else sp[d]) for d in range(D)]
    return out if noise_iterations is not None else out[0]


def simulate_gradient(sc: Scenario, params: LinkParams, seed: int, ws=None, qs=None, wc=None, qc=None,
                      wx=None, noise_iteration: int = 0, noise_iterations: Optional[Sequence[int]] = None):
    """simulate_gradient (engine.cpp:303-429, Checkpointed) with the loss
    sum_k <ws_k, s_k> + 1/2 <qs_k, s_k^2> + <wc, c> + 1/2 <qc, c^2> + <wx, x_final>."""
    its = _its(noise_iteration, noise_iterations)
    D, L, N, K = len(its), sc.n_links, sc.n_agents, sc.n_snapshots
    ws, qs, wc, qc, wx = (None if a is None else _f64(a).ravel() for a in (ws, qs, wc, qc, wx))
    loss = np.zeros(D)
    grads = np.zeros((D, 5, L))
    snaps = np.zeros((D, K, L))
    cumf = np.zeros((D, L))
    lk, ps = np.zeros((D, N), np.int32), np.zeros((D, N))
    wall = np.zeros(1)
    sc._check(sc._lib.dtg_simulate_gradient(sc._h, *params.arrays(), seed, D, its, ptr(ws), ptr(qs), ptr(wc),
                                            ptr(qc), ptr(wx), ptr(loss), ptr(grads), ptr(snaps), ptr(cumf),
                                            ptr(lk), ptr(ps), ptr(wall)))
    out = [GradResult(float(loss[d]), grads[d], snaps[d], cumf[d], lk[d], ps[d], float(wall[0])) for d in range(D)]
    return out if noise_iterations is not None else out[0]


def simulate_gradient_mse(sc: Scenario, params: LinkParams, seed: int, obs_ids, obs_values,
                          noise_iterations: Sequence[int] = (0,)):
    """simulate_gradient with mse_loss_builder (optimization.cpp:84-101)."""
    its = _its(0, noise_iterations)
    D, L = len(its), sc.n_links
    obs_ids = np.ascontiguousarray(obs_ids, np.int32)
    obs_values = np.ascontiguousarray(obs_values, np.float64)
    loss = np.zeros(D)
    grads = np.zeros((D, 5, L))
    sc._check(sc._lib.dtg_simulate_gradient_mse(sc._h, *params.arrays(), seed, D, its, len(obs_ids), obs_ids,
                                                obs_values.shape[0], obs_values.ravel(), ptr(loss), ptr(grads)))
    return loss, grads


@dataclass
class ParamRanges:
    """ParamRanges (network.hpp) — sampling and calibration bounds."""

    u_lo: float = 13.9
    u_hi: float = 22.2
    kappa_lo: float = 0.18
    kappa_hi: float = 0.22
    beta_lo: float = 0.0
    beta_hi: float = 5.0
    alpha_lo: float = 0.01
    alpha_hi: float = 5.0

    def c(self) -> ParamRangesC:
        return ParamRangesC(self.u_lo, self.u_hi, self.kappa_lo, self.kappa_hi, self.beta_lo,
                            self.beta_hi, self.alpha_lo, self.alpha_hi)


@dataclass
class OptimizeConfig:
    """AdamWConfig + OptimizeConfig (optimization.hpp:18-24, 72-82)."""

    lr: float = 0.1
    weight_decay: float = 1e-5
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    patience: int = 20
    max_iterations: int = 200
    resample_noise: bool = True
    noise_draws: int = 1

    def c(self) -> _OptC:
        return _OptC(self.lr, self.weight_decay, self.beta1, self.beta2, self.eps, self.patience,
                     self.max_iterations, int(self.resample_noise), self.noise_draws)


@dataclass
class CalibrationResult:
    """CalibrationResult (optimization.hpp:84-91)."""

    best_params: Optional[LinkParams]
    best_loss: float
    best_iteration: int
    iterations: int
    loss_curve: np.ndarray
    wall_seconds: float


@dataclass
class ControlResult:
    """ControlResult (optimization.hpp:106-116)."""

    cost: np.ndarray
    desired: float
    achieved: float
    gap_fraction: float
    best_loss: float
    iterations: int
    loss_curve: np.ndarray
    zero_gradient_stall: bool
    wall_seconds: float


def calibrate(sc: Scenario, obs_ids, obs_values, seed: int, bounds: Optional[ParamRanges] = None,
              cfg: Optional[OptimizeConfig] = None, init: Optional[LinkParams] = None,
              exchange=None) -> CalibrationResult:
    """calibrate (optimization.cpp:122-219): AdamW fit of (u, kappa, beta, alpha)
    to counts obs_values [K_obs, n_obs] on links obs_ids; each iteration is one
    batched device forward + reverse sweep over its noise draws with the MSE loss
    and the draw sum on the device.  Raises DivergenceError on a non-finite loss."""
    bounds = bounds or ParamRanges()
    cfg = cfg or OptimizeConfig()
    L = sc.n_links
    ids = np.ascontiguousarray(obs_ids, np.int32)
    vals = np.ascontiguousarray(obs_values, np.float64).reshape(-1, max(len(ids), 1))
    best = [np.zeros(L) for _ in range(5)]
    bl, bi, its, wall = C.c_double(), C.c_int(), C.c_int(), C.c_double()
    curve = np.zeros(max(cfg.max_iterations, 1))
    ia = init.arrays() if init is not None else [None] * 5
    bc, oc = bounds.c(), cfg.c()
    sc._check(sc._lib.dtg_calibrate(sc._h, len(ids), ids, vals.shape[0] if len(ids) else 0, vals.ravel(),
                                    C.byref(bc), C.byref(oc), seed, *(ptr(a) for a in ia), *best,
                                    C.byref(bl), C.byref(bi), C.byref(its), curve, C.byref(wall),
                                    None if exchange is None else C.byref(exchange)))
    n = its.value
    return CalibrationResult(LinkParams(*best) if bi.value >= 0 else None, bl.value, bi.value, n,
                             curve[:n].copy(), wall.value)


def optimize_control(sc: Scenario, calibrated: LinkParams, target_link: int, desired: float, seed: int,
                     cfg: Optional[OptimizeConfig] = None, cost_floor: float = 0.05,
                     exchange=None) -> ControlResult:
    """optimize_control (optimization.cpp:221-295) with the device iteration."""
    cfg = cfg or OptimizeConfig()
    L = sc.n_links
    cost = np.zeros(L)
    ach, gap, bl, wall = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    its, stall = C.c_int(), C.c_int()
    curve = np.zeros(max(cfg.max_iterations, 1))
    oc = cfg.c()
    sc._check(sc._lib.dtg_optimize_control(sc._h, *calibrated.arrays(), target_link, desired, C.byref(oc),
                                           cost_floor, seed, cost, C.byref(ach), C.byref(gap), C.byref(bl),
                                           C.byref(its), curve, C.byref(stall), C.byref(wall),
                                           None if exchange is None else C.byref(exchange)))
    n = its.value
    return ControlResult(cost, desired, ach.value, gap.value, bl.value, n, curve[:n].copy(),
                         bool(stall.value), wall.value)


class Engine:
    """Level-1 device context: B scenarios of one network on one GPU."""

    def __init__(self, sc: Scenario, n_scenarios: int = 1, max_steps: int = 1):
        self._lib = load()
        off, succ = sc.csr()
        _, _, length, _ = sc.links()
        self._keep = (off, succ, length)
        nd = NetDesc(sc.n_links, off.ctypes.data, succ.ctypes.data, length.ctypes.data)
        cfg = SimConfig(sc.delta_n, sc.tau, 99999.0, getattr(sc, "gumbel_tau", 0.01),
                        int(getattr(sc, "trajectory_grafting", True)))
        h = C.c_void_p()
        rc = self._lib.dtg_create(C.byref(nd), C.byref(cfg), sc.n_agents, n_scenarios, max_steps, C.byref(h))
        raise_for(rc, self._lib.dtg_last_error(None).decode())
        self._h = h
        self.L, self.N, self.B = sc.n_links, sc.n_agents, n_scenarios
        self.T = 0

    def __del__(self):
        try:
            self._lib.dtg_destroy(self._h)
        except Exception:
            pass

    def _check(self, rc):
        raise_for(rc, self._lib.dtg_last_error(self._h).decode())

    def set_stream(self, stream_ptr: int):
        """Run on this cudaStream_t (e.g. torch.cuda.Stream().cuda_stream).  The
        legacy default stream (handle 0) is rejected: the context would keep its
        own stream and events on stream 0 would not time it."""
        if not stream_ptr:
            raise ValueError("pass a real CUDA stream handle (torch.cuda.Stream()), not the legacy default 0")
        self._check(self._lib.dtg_set_stream(self._h, C.c_void_p(stream_ptr)))

    def set_graphs(self, on: bool):
        self._check(self._lib.dtg_set_graphs(self._h, int(on)))

    def set_mode(self, mode: int):
        """0 auto, 1 cluster per scenario, 2 persistent grid, 3 step graph."""
        self._check(self._lib.dtg_set_mode(self._h, mode))

    def set_flag(self, flag: int, value: int):
        self._check(self._lib.dtg_set_flag(self._h, flag, value))

    @property
    def last_mode(self) -> int:
        """1000 * schedule (1 cluster, 2 persistent grid, 3 step graph,
        4 scenario-resident CTAs) + CTAs per scenario of the last forward."""
        return int(self._lib.dtg_last_mode(self._h))

    @property
    def last_schedule(self) -> dict:
        m = self.last_mode
        names = {1: "cluster per scenario", 2: "fused persistent grid", 3: "5-kernel step graph",
                 4: "scenario-resident CTAs"}
        return {"schedule": names.get(m // 1000, str(m)), "ctas_per_scenario": m % 1000 or None}

    def set_persistent(self, on: bool):
        self._check(self._lib.dtg_set_persistent(self._h, int(on)))

    def profile_scn(self, T: int, steps_per_interval: int) -> dict:
        """Mean per-step span (us) of the scenario-resident forward's phases."""
        ph = np.zeros(9)
        self._check(self._lib.dtg_profile_scn(self._h, T, steps_per_interval, ph))
        return dict(zip(("links", "choice", "merge", "scan", "slots", "step", "head_links", "max_heads",
                         "chosen_links"), ph.tolist()))

    def profile_persistent(self, T: int, steps_per_interval: int):
        """Mean per-step span (us) of the persistent kernel's phases."""
        ph = np.zeros(4)
        g = C.c_int()
        self._check(self._lib.dtg_profile_persistent(self._h, T, steps_per_interval, ph, C.byref(g)))
        return dict(zip(["slot_phase", "barrier1", "link_phase", "barrier2"], ph.tolist())), g.value

    def profile_backward(self):
        """Mean per-step span (us) of the persistent reverse sweep's phases."""
        ph = np.zeros(8)
        g = C.c_int()
        self._check(self._lib.dtg_profile_backward(self._h, ph, C.byref(g)))
        names = ["R1", "bar1", "R2", "bar2", "R3", "bar3", "R4", "bar4"]
        return dict(zip(names, ph.tolist())), g.value

    def force_slow_path(self, on: bool):
        self._check(self._lib.dtg_debug_force_slow_path(self._h, int(on)))

    def set_params(self, p: LinkParams, scenario: int = -1):
        self._check(self._lib.dtg_set_params(self._h, scenario, *p.arrays()))

    def set_state(self, link, pos, scenario: int = -1):
        self._check(self._lib.dtg_set_state(self._h, scenario, np.ascontiguousarray(link, np.int32), _f64(pos)))

    def set_noise(self, root_seed: int, noise_iteration: int, scenario: int = -1):
        self._check(self._lib.dtg_set_noise(self._h, scenario, root_seed, noise_iteration))

    def forward(self, T: int, steps_per_interval: int, checkpoint: bool = False):
        self._check(self._lib.dtg_forward(self._h, T, steps_per_interval, int(checkpoint)))
        self.T = T

    def sync(self):
        self._check(self._lib.dtg_sync(self._h))

    def read_cum(self, scenario: int = 0) -> np.ndarray:
        out = np.zeros((self.T, self.L))
        self._check(self._lib.dtg_read_cum(self._h, scenario, out))
        return out

    def read_cum_all(self) -> np.ndarray:
        """[B, T, L] cumulative counts of every scenario (one device copy)."""
        out = np.zeros((self.B, self.T, self.L))
        self._check(self._lib.dtg_read_cum_all(self._h, out))
        return out

    def read_state(self, scenario: int = 0, step: int = -1):
        lk, ps = np.zeros(self.N, np.int32), np.zeros(self.N)
        self._check(self._lib.dtg_read_state(self._h, scenario, step, lk, ps))
        return lk, ps

    @property
    def n_snapshots(self) -> int:
        return self._lib.dtg_n_snapshots(self._h)

    def backward(self, snap_seeds=None, cum_seeds=None, x_seeds=None) -> np.ndarray:
        grads = np.zeros((self.B, 5, self.L))
        a = [None if s is None else _f64(s).ravel() for s in (snap_seeds, cum_seeds, x_seeds)]
        self._check(self._lib.dtg_backward(self._h, ptr(a[0]), ptr(a[1]), ptr(a[2]), grads))
        return grads

    def backward_device(self, d_snap, d_cum, d_x, d_grads):
        """Device pointers (ints, e.g. torch.Tensor.data_ptr()); no host sync."""
        self._check(self._lib.dtg_backward_device(self._h, C.c_void_p(d_snap), C.c_void_p(d_cum),
                                                  C.c_void_p(d_x), C.c_void_p(d_grads)))

    def set_loss_mse(self, obs_ids, obs_values):
        """Device MSE loss (mse_loss_builder): obs_values [K_obs, n_obs] in vehicles."""
        ids = np.ascontiguousarray(obs_ids, np.int32)
        vals = np.ascontiguousarray(obs_values, np.float64).reshape(-1, max(len(ids), 1))
        self._check(self._lib.dtg_set_loss_mse(self._h, vals.shape[0], len(ids), ids, vals.ravel()))

    def set_loss_control(self, target_link: int, desired: float):
        self._check(self._lib.dtg_set_loss_control(self._h, target_link, desired))

    def gradient_device_loss(self, d_rows: int = 0):
        """Loss + seeds + reverse sweep on the device; rows [B, 5L+2] into the
        device pointer d_rows (0 = the context's own buffer).  No host sync."""
        self._check(self._lib.dtg_gradient_device_loss(self._h, C.c_void_p(d_rows or None)))

    def reduce_draw_rows(self, n_draws: int, d_rows: int = 0, mode: int = 0) -> np.ndarray:
        """Draw-ordered sum of n_draws rows -> [5L+2] host array (grads, loss, extra)."""
        out = np.zeros(5 * self.L + 2)
        self._check(self._lib.dtg_reduce_draw_rows(self._h, n_draws, C.c_void_p(d_rows or None), mode, out))
        return out

    def profile_kernels(self, T: int, steps_per_interval: int, backward: bool = False):
        """Per-kernel-kind device time (ms, CUDA events) of one forward (or the
        reverse sweep of the preceding checkpointed forward)."""
        nk = 0
        while self._lib.dtg_kernel_name(int(backward), nk):
            nk += 1
        ms = np.zeros(nk)
        n = C.c_int64()
        self._check(self._lib.dtg_profile_kernels(self._h, T, steps_per_interval, int(backward), ms, C.byref(n)))
        names = [self._lib.dtg_kernel_name(int(backward), w).decode() for w in range(nk)]
        return dict(zip(names, ms.tolist())), int(n.value)

    def device_cum_ptr(self) -> int:
        return self._lib.dtg_device_cum(self._h) or 0

    @property
    def last_launches(self) -> int:
        return int(self._lib.dtg_last_launches(self._h))
