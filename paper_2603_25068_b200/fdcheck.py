"""FD-validation instrumentation on the device.

Python face of the reference's finite-difference validation modes, run by the
device probe engine (``csrc/dtg_probe.cu``) through the C-ABI in
``include/dtg.h``:

* ``SurrogateTrace`` — car_following.hpp:23-29: a recording run keeps the
  graft / carrier values and min / relu picks; a replay run re-evaluates the
  program with those discontinuities frozen.
* ``soft_choices`` — car_following.hpp:37: relaxed choice tensors; on the
  device every choice value must stay 0 or 1 (one-hot rows such as the
  gradient check's chain), anything else raises ``UnsupportedError``.
* ``trace_branches`` — branch_trace.hpp: FNV-1a hash of every discrete
  decision, bit-identical to the reference's ``branch_hash``.
* ``probe_forward_batch`` — many parameter sets in ONE launch (one CTA each).
* ``run_gradcheck`` — pipeline.cpp:499-585 with all stencil probes of a draw
  batched.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from ._lib import load, ptr, raise_for
from .engine import LinkParams, Scenario, _f64

OFFSET_BASIS = 0xCBF29CE484222325  # BranchTrace::h before any note


class SurrogateTrace:
    """SurrogateTrace (car_following.hpp:23-29), device-resident."""

    def __init__(self):
        self._lib = load()
        self._h = self._lib.dtg_surrogate_create()
        if not self._h:
            raise MemoryError("dtg_surrogate_create")
        self._replay = False

    def __del__(self):
        try:
            self._lib.dtg_surrogate_free(self._h)
        except Exception:
            pass

    @property
    def replay(self) -> bool:
        return self._replay

    @replay.setter
    def replay(self, on: bool):
        self._lib.dtg_surrogate_set_replay(self._h, int(bool(on)))
        self._replay = bool(on)

    def rewind(self):
        self._lib.dtg_surrogate_rewind(self._h)


def set_soft_choices(sc: Scenario, soft: bool) -> Scenario:
    """SimConfig::soft_choices."""
    sc._check(sc._lib.dtg_scenario_set_soft_choices(sc._h, int(bool(soft))))
    return sc


def set_surrogate(sc: Scenario, tr: "SurrogateTrace | None") -> Scenario:
    """SimConfig::surrogate (None detaches).  The scenario keeps a reference."""
    sc._check(sc._lib.dtg_scenario_set_surrogate(sc._h, None if tr is None else tr._h))
    sc._surrogate = tr
    return sc


@dataclass
class TracedTrajectory:
    cum_per_step: np.ndarray
    link_final: np.ndarray
    pos_final: np.ndarray
    branch_hash: int
    wall_seconds: float

    @property
    def cum_final(self) -> np.ndarray:
        return self.cum_per_step[-1] if len(self.cum_per_step) else np.zeros(self.cum_per_step.shape[1])


def simulate_forward_traced(sc: Scenario, params: LinkParams, seed: int, noise_iteration: int = 0,
                            trace_branches: bool = True) -> TracedTrajectory:
    """simulate_forward with ForwardOptions.trace_branches and the scenario's
    soft-choice / surrogate settings (engine.cpp:227-254)."""
    T, L, N = sc.horizon_steps, sc.n_links, sc.n_agents
    cum = np.zeros((T, L))
    lk, ps = np.zeros(N, np.int32), np.zeros(N)
    h = np.zeros(1, np.uint64)
    wall = np.zeros(1)
    sc._check(sc._lib.dtg_simulate_forward_traced(sc._h, *params.arrays(), seed, noise_iteration,
                                                  int(trace_branches), ptr(cum), ptr(lk), ptr(ps), h, ptr(wall)))
    return TracedTrajectory(cum, lk, ps, int(h[0]), float(wall[0]))


def simulate_gradient_traced(sc: Scenario, params: LinkParams, seed: int, noise_iteration: int = 0,
                             full_tape: bool = True, trace_branches: bool = True, ws=None, qs=None, wc=None,
                             qc=None, wx=None):
    """simulate_gradient with trace_branches / soft choices / a recording
    surrogate (engine.cpp:303-429).  Default loss: sum(cum_final) — the
    gradient check's loss (pipeline.cpp:522-524).  Returns (loss, grads[5][L],
    cum_final, branch_hash)."""
    L = sc.n_links
    if all(a is None for a in (ws, qs, wc, qc, wx)):
        wc = np.ones(L)
    ws, qs, wc, qc, wx = (None if a is None else _f64(a).ravel() for a in (ws, qs, wc, qc, wx))
    loss = np.zeros(1)
    grads = np.zeros((5, L))
    cumf = np.zeros(L)
    h = np.zeros(1, np.uint64)
    sc._check(sc._lib.dtg_simulate_gradient_traced(sc._h, *params.arrays(), seed, noise_iteration,
                                                   0 if full_tape else 1, int(trace_branches), ptr(ws), ptr(qs),
                                                   ptr(wc), ptr(qc), ptr(wx), ptr(loss), grads, ptr(cumf), h))
    return float(loss[0]), grads, cumf, int(h[0])


@dataclass
class ProbeBatch:
    cum_final: np.ndarray   # [P][L]
    cum_sum: np.ndarray     # [P]
    branch_hash: np.ndarray  # [P] uint64
    on_path: np.ndarray     # [P] bool


def probe_forward_batch(sc: Scenario, params: Sequence[LinkParams], seed: int, noise_iteration: int = 0,
                        trace_branches: bool = True) -> ProbeBatch:
    """Instrumented forwards of len(params) parameter sets in one launch."""
    L, P = sc.n_links, len(params)
    flat = np.ascontiguousarray(np.stack([np.stack(p.arrays()) for p in params]), np.float64)
    cf = np.zeros((P, L))
    cs = np.zeros(P)
    hs = np.zeros(P, np.uint64)
    op = np.zeros(P, np.int32)
    sc._check(sc._lib.dtg_probe_forward_batch(sc._h, P, flat.ravel(), seed, noise_iteration, int(trace_branches),
                                              ptr(cf), ptr(cs), ptr(hs), ptr(op)))
    return ProbeBatch(cf, cs, hs, op.astype(bool))


@dataclass
class GradcheckReport:  # pipeline.hpp:49-55
    max_rel_err: float
    draws: int
    redraws: int
    passed: bool
    per_draw_max: List[float] = field(default_factory=list)


def run_gradcheck(draws: int = 20, steps: int = 20, agents: int = 5, tol: float = 1e-4,
                  seed: int = 1) -> GradcheckReport:
    """run_gradcheck (pipeline.cpp:499-585) on the device (defaults:
    config.hpp:87-91 and RunConfig::seed = 1, config.hpp:58)."""
    lib = load()
    mx = np.zeros(1)
    red, ps = C.c_int(0), C.c_int(0)
    per = np.zeros(max(draws, 1))
    rc = lib.dtg_run_gradcheck(draws, steps, agents, float(tol), seed, mx, C.byref(red), C.byref(ps), per)
    raise_for(rc, lib.dtg_scenario_last_error(None).decode())
    return GradcheckReport(float(mx[0]), draws, red.value, bool(ps.value), list(per[:draws]))
