"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Plain-Python restatement of the reference's optimisation loops over the C port
(oracle/dtsim_port.c), used to check the device calibrate / optimize_control
 where the reference build is absent:

* AdamW.step          src/optimization.cpp:10-25
* BoundedTransform    src/optimization.cpp:27-46
* LowerBoundTransform src/optimization.cpp:48-59
* mse_loss_builder    src/optimization.cpp:83-101 (value and seeds in tape order)
* calibrate           src/optimization.cpp:122-219
* optimize_control    src/optimization.cpp:221-295

Scalar ``math`` functions (the C library's exp/log/pow/sqrt, as the
reference links) keep every value bit-identical to the reference; numpy is
only used as storage.  Pinned against oracle/_ref (the reference itself) in
tests/test_oracle_optim.py.
"""
from __future__ import annotations

import math

import numpy as np


class AdamW:
    def __init__(self, n: int, lr=0.1, weight_decay=1e-5, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.wd, self.b1, self.b2, self.eps = lr, weight_decay, beta1, beta2, eps
        self.m = [0.0] * n
        self.v = [0.0] * n
        self.t = 0

    def step(self, params: list, grads: list):
        self.t += 1
        bc1 = 1.0 - math.pow(self.b1, self.t)
        bc2 = 1.0 - math.pow(self.b2, self.t)
        for i in range(len(params)):
            self.m[i] = self.b1 * self.m[i] + (1.0 - self.b1) * grads[i]
            self.v[i] = self.b2 * self.v[i] + (1.0 - self.b2) * grads[i] * grads[i]
            mhat = self.m[i] / bc1
            vhat = self.v[i] / bc2
            params[i] -= self.lr * (mhat / (math.sqrt(vhat) + self.eps) + self.wd * params[i])


def _sigmoid(raw: float) -> float:
    return 1.0 / (1.0 + math.exp(-raw)) if raw >= 0.0 else math.exp(raw) / (1.0 + math.exp(raw))


class Bounded:
    def __init__(self, lo: float, hi: float):
        self.lo, self.hi = lo, hi

    def value(self, raw: float) -> float:
        return self.lo + (self.hi - self.lo) * _sigmoid(raw)

    def dvalue(self, raw: float) -> float:
        s = _sigmoid(raw)
        return (self.hi - self.lo) * s * (1.0 - s)

    def raw_of(self, value: float) -> float:
        if self.hi == self.lo:
            return 0.0
        f = (value - self.lo) / (self.hi - self.lo)
        f = min(max(f, 1e-9), 1.0 - 1e-9)
        return math.log(f / (1.0 - f))


class LowerBound:
    def __init__(self, floor: float):
        self.floor = floor

    def value(self, raw: float) -> float:
        sp = raw if raw > 30.0 else math.log1p(math.exp(raw))
        return self.floor + sp

    def dvalue(self, raw: float) -> float:
        return _sigmoid(raw)

    def raw_of(self, value: float) -> float:
        y = max(value - self.floor, 1e-12)
        return y if y > 30.0 else math.log(math.expm1(y))


def mse_loss(snapshots: np.ndarray, obs_ids, obs_vals: np.ndarray, delta_n: int):
    """Value and snapshot seeds of mse_loss_builder in the tape's op order."""
    K, n = obs_vals.shape[0], len(obs_ids)
    if snapshots.shape[0] < K:
        raise RuntimeError("loss: fewer snapshots than observations")
    sc = 1.0 / (float(K) * n)
    seeds = np.zeros_like(snapshots)
    acc = 0.0
    dn = float(delta_n)
    for k in range(K):
        r = 0.0
        for q in range(n):
            i = int(obs_ids[q])
            d = float(snapshots[k, i]) * dn - float(obs_vals[k, q])
            r += d * d
            seeds[k, i] += ((0.0 + sc * d) + sc * d) * dn
        acc = acc + r
    return acc * sc, seeds


def _draw_its(resample: bool, it: int, draws: int):
    return [it * draws + k + 1 if resample else 0 for k in range(draws)]


def calibrate(port, obs_ids, obs_vals, seed: int, bounds=(13.9, 22.2, 0.18, 0.22, 0.0, 5.0, 0.01, 5.0),
              cfg: dict = None, init=None, params_cls=None):
    """calibrate() over a PortScenario; returns the CalibrationResult fields."""
    d = dict(lr=0.1, weight_decay=1e-5, beta1=0.9, beta2=0.999, eps=1e-8, patience=20, max_iterations=200,
             resample_noise=True, noise_draws=1)
    d.update(cfg or {})
    L = port.L
    obs_vals = np.asarray(obs_vals, np.float64).reshape(-1, len(obs_ids))
    tr = [Bounded(bounds[2 * q], bounds[2 * q + 1]) for q in range(4)]
    raw = [0.0] * (4 * L)
    if init is not None:
        arrs = init.arrays()
        for q in range(4):
            for l in range(L):
                raw[q * L + l] = tr[q].raw_of(float(arrs[q][l]))
    cost = np.array(init.arrays()[4], np.float64) if init is not None else np.ones(L)
    adam = AdamW(4 * L, d["lr"], d["weight_decay"], d["beta1"], d["beta2"], d["eps"])
    draws = max(1, d["noise_draws"]) if d["resample_noise"] else 1
    best_loss, best, best_it, since = math.inf, None, -1, 0
    curve = []
    iters = 0
    for it in range(d["max_iterations"]):
        pv = [np.array([tr[q].value(raw[q * L + l]) for l in range(L)]) for q in range(4)]
        params = params_cls(*pv, cost.copy())
        loss = 0.0
        grads = None
        for ni in _draw_its(d["resample_noise"], it, draws):
            fw = port.forward(params, seed, ni)
            T = fw["cum_per_step"].shape[0]
            snaps = np.array([fw["cum_per_step"][t] for t in range(T) if (t + 1) % port.spi == 0])
            lv, seeds = mse_loss(snaps.reshape(-1, L), obs_ids, obs_vals, port.delta_n)
            g = port.gradient_seeds(params, seed, ni, seeds, np.zeros(L), np.zeros(port.N))
            loss += lv / draws
            grads = g.copy() if grads is None else grads + g
        curve.append(loss)
        iters = it + 1
        if not math.isfinite(loss):
            raise FloatingPointError(f"calibration diverged at iteration {it}")
        if loss < best_loss:
            best_loss, best, best_it, since = loss, params, it, 0
        else:
            since += 1
            if since >= d["patience"]:
                break
        rg = [float(grads[q, l]) / draws * tr[q].dvalue(raw[q * L + l]) for q in range(4) for l in range(L)]
        adam.step(raw, rg)
    return dict(best=best, best_loss=best_loss, best_iteration=best_it, iterations=iters,
                loss_curve=np.array(curve))


def optimize_control(port, calibrated, target: int, desired: float, seed: int, cfg: dict = None,
                     cost_floor: float = 0.05, params_cls=None):
    """optimize_control() over a PortScenario; returns the ControlResult fields."""
    d = dict(lr=0.1, weight_decay=1e-5, beta1=0.9, beta2=0.999, eps=1e-8, patience=20, max_iterations=200,
             resample_noise=True, noise_draws=1)
    d.update(cfg or {})
    L, dn = port.L, port.delta_n
    tc = LowerBound(cost_floor)
    base = [np.array(a, np.float64) for a in calibrated.arrays()]
    raw = [tc.raw_of(float(base[4][l])) for l in range(L)]
    adam = AdamW(L, d["lr"], d["weight_decay"], d["beta1"], d["beta2"], d["eps"])
    draws = max(1, d["noise_draws"]) if d["resample_noise"] else 1
    best_loss, best_cost, best_ach, since = math.inf, None, 0.0, 0
    curve, iters, any_nz = [], 0, False
    for it in range(d["max_iterations"]):
        cost = np.array([tc.value(raw[l]) for l in range(L)])
        params = params_cls(*base[:4], cost)
        loss, achieved = 0.0, 0.0
        cg = [0.0] * L
        for ni in _draw_its(d["resample_noise"], it, draws):
            fw = port.forward(params, seed, ni)
            T = fw["cum_per_step"].shape[0]
            c = float(fw["cum_per_step"][-1, target]) if T else 0.0
            dd = c * dn + (-desired)
            cs = np.zeros(L)
            cs[target] = ((0.0 + dd) + dd) * dn
            g = port.gradient_seeds(params, seed, ni, np.zeros((max(T // port.spi, 1), L)), cs, np.zeros(port.N))
            loss += dd * dd / draws
            achieved += c * dn / draws
            for l in range(L):
                cg[l] += float(g[4, l]) / draws
        curve.append(loss)
        iters = it + 1
        if not math.isfinite(loss):
            raise FloatingPointError(f"control diverged at iteration {it}")
        if loss < best_loss:
            best_loss, best_cost, best_ach, since = loss, cost, achieved, 0
        else:
            since += 1
            if since >= d["patience"]:
                break
        rg = [cg[l] * tc.dvalue(raw[l]) for l in range(L)]
        any_nz = any_nz or any(x != 0.0 for x in rg)
        adam.step(raw, rg)
    gap = abs(best_ach - desired) / abs(desired) if desired != 0.0 else abs(best_ach - desired)
    return dict(cost=best_cost, achieved=best_ach, gap_fraction=gap, best_loss=best_loss, iterations=iters,
                zero_gradient_stall=not any_nz, loss_curve=np.array(curve))
