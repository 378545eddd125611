"""Observation / output side of the path.

Count series as the reference's ``CountSeries`` (observation.hpp): link ids,
an interval in seconds and cumulative counts per interval.  The functions call
the C++ restatements in libdtg.so (csrc/dtg_observe.cpp):

* ``series_from_levels``       observation.cpp:27-44 (cum_per_step -> series)
* ``synthesize_observations``  observation.cpp:46-83
* ``count_metrics``            optimization.cpp:297-336
* ``series_to_csv`` / ``series_from_csv``  pipeline.cpp:113-160 (byte-identical)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import DtgError, load


@dataclass
class CountSeries:
    link_ids: np.ndarray  # [n] int32
    interval_s: int
    values: np.ndarray    # [k, n] float64

    @property
    def n_intervals(self) -> int:
        return int(self.values.shape[0])


@dataclass
class Metrics:
    mae: float
    pearson_r: float
    r_defined: bool
    n_pairs: int


def _check(lib, rc):
    if rc != 0:
        raise DtgError(rc, lib.dtg_observe_last_error().decode())


def _series_args(s: CountSeries):
    ids = np.ascontiguousarray(s.link_ids, np.int32)
    vals = np.ascontiguousarray(s.values, np.float64).reshape(-1, max(len(ids), 1))
    return vals.shape[0] if len(ids) else 0, len(ids), ids, vals.ravel()


def series_from_levels(cum_per_step, link_ids, interval_s: int, dt: float, delta_n: int) -> CountSeries:
    """Counts in vehicles at every step that closes an interval (observation.cpp:27-44)."""
    cum = np.asarray(cum_per_step, np.float64)
    ids = np.ascontiguousarray(link_ids, np.int32)
    rows = []
    for t in range(cum.shape[0]):
        k = (t + 1) * dt / interval_s
        if abs(k - round(k)) > 1e-9:
            continue
        rows.append(cum[t, ids] * delta_n)
    return CountSeries(ids, interval_s, np.array(rows).reshape(len(rows), len(ids)))


def synthesize_observations(truth: CountSeries, noise_frac: float, coverage: float, seed: int):
    """(observations, observed link ids) — seeded coverage sample + noise."""
    lib = load()
    k, n, ids, vals = _series_args(truth)
    m = C.c_int()
    oids = np.zeros(max(n, 1), np.int32)
    ovals = np.zeros(max(k * n, 1))
    _check(lib, lib.dtg_synthesize_observations(k, n, ids, vals, truth.interval_s, noise_frac, coverage, seed,
                                                C.byref(m), oids, ovals))
    mm = m.value
    obs = CountSeries(oids[:mm].copy(), truth.interval_s, ovals[:k * mm].reshape(k, mm).copy())
    return obs, oids[:mm].copy()


def count_metrics(sim: CountSeries, truth: CountSeries) -> Metrics:
    lib = load()
    ks, ns, si, sv = _series_args(sim)
    kt, nt, ti, tv = _series_args(truth)
    mae, r = C.c_double(), C.c_double()
    rd, npairs = C.c_int(), C.c_int()
    _check(lib, lib.dtg_count_metrics(ks, ns, si, sv, kt, nt, ti, tv, C.byref(mae), C.byref(r), C.byref(rd),
                                      C.byref(npairs)))
    return Metrics(mae.value, r.value, bool(rd.value), npairs.value)


def series_to_csv(s: CountSeries) -> str:
    lib = load()
    k, n, ids, vals = _series_args(s)
    ln = C.c_size_t()
    _check(lib, lib.dtg_series_to_csv(k, n, ids, vals, s.interval_s, None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    _check(lib, lib.dtg_series_to_csv(k, n, ids, vals, s.interval_s, buf, ln.value + 1, C.byref(ln)))
    return buf.value.decode()


def series_from_csv(text: str) -> CountSeries:
    lib = load()
    k, n, iv = C.c_int(), C.c_int(), C.c_int()
    raw = text.encode()
    _check(lib, lib.dtg_series_from_csv(raw, C.byref(k), C.byref(n), C.byref(iv), None, None, 0, 0))
    ids = np.zeros(n.value, np.int32)
    vals = np.zeros(k.value * n.value)
    _check(lib, lib.dtg_series_from_csv(raw, C.byref(k), C.byref(n), C.byref(iv), ids.ctypes.data_as(C.c_void_p),
                                        vals.ctypes.data_as(C.c_void_p), ids.size, vals.size))
    return CountSeries(ids, iv.value, vals.reshape(k.value, n.value))
