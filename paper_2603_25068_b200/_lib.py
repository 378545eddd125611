"""ctypes bindings of the C-ABI in include/dtg.h (libdtg.so, built in-tree).

Loading fails loudly when the native library is missing: there is no CPU
fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdtg.so")

DTG_OK = 0
DTG_ERR_RUNTIME = 1
DTG_ERR_CONFIG = 2
DTG_ERR_DIVERGENCE = 3
DTG_ERR_CUDA = 4
DTG_ERR_UNSUPPORTED = 5


class DtgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[dtg code {code}] {msg}")
        self.code = code


class UnsupportedError(DtgError):
    pass


class ConfigError(DtgError):
    pass


class DivergenceError(DtgError):
    """Non-finite loss in an optimisation loop (DivergenceError, config.hpp)."""


def raise_for(code: int, msg: str):
    if code == DTG_OK:
        return
    cls = {DTG_ERR_UNSUPPORTED: UnsupportedError, DTG_ERR_CONFIG: ConfigError,
           DTG_ERR_DIVERGENCE: DivergenceError}.get(code, DtgError)
    raise cls(code, msg)


class SimConfig(C.Structure):
    _fields_ = [("delta_n", C.c_int), ("tau", C.c_double), ("sentinel", C.c_double),
                ("gumbel_tau", C.c_double), ("trajectory_grafting", C.c_int)]


class NetDesc(C.Structure):
    _fields_ = [("n_links", C.c_int), ("succ_off", C.c_void_p), ("succ", C.c_void_p), ("length", C.c_void_p)]


class OptimizeConfig(C.Structure):
    """AdamWConfig + OptimizeConfig (optimization.hpp:18-24, 72-82)."""
    _fields_ = [("lr", C.c_double), ("weight_decay", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("patience", C.c_int),
                ("max_iterations", C.c_int), ("resample_noise", C.c_int), ("noise_draws", C.c_int)]


class ParamRangesC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("u_lo", "u_hi", "kappa_lo", "kappa_hi", "beta_lo",
                                          "beta_hi", "alpha_lo", "alpha_hi")]


GatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p)


class DrawExchange(C.Structure):
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("d_local", C.c_void_p), ("d_full", C.c_void_p),
                ("stream", C.c_void_p), ("gather", GatherFn), ("user", C.c_void_p)]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
vp = C.c_void_p
u64 = C.c_uint64
i32 = C.c_int

# (name, restype, argtypes) for every symbol declared in include/dtg.h
SIGNATURES = [
    ("dtg_create", i32, [C.POINTER(NetDesc), C.POINTER(SimConfig), i32, i32, i32, C.POINTER(vp)]),
    ("dtg_destroy", None, [vp]),
    ("dtg_init", i32, []),
    ("dtg_host_alloc", vp, [C.c_size_t]),
    ("dtg_host_free", None, [vp]),
    ("dtg_last_error", C.c_char_p, [vp]),
    ("dtg_set_stream", i32, [vp, vp]),
    ("dtg_get_stream", i32, [vp, C.POINTER(vp), C.POINTER(C.c_int)]),
    ("dtg_set_graphs", i32, [vp, i32]),
    ("dtg_set_persistent", i32, [vp, i32]),
    ("dtg_set_mode", i32, [vp, i32]),
    ("dtg_set_flag", i32, [vp, i32, i32]),
    ("dtg_profile_backward", i32, [vp, _dp, C.POINTER(C.c_int)]),
    ("dtg_profile_scn", i32, [vp, i32, i32, _dp]),
    ("dtg_last_mode", i32, [vp]),
    ("dtg_profile_persistent", i32, [vp, i32, i32, _dp, C.POINTER(C.c_int)]),
    ("dtg_set_params", i32, [vp, i32, _dp, _dp, _dp, _dp, _dp]),
    ("dtg_set_state", i32, [vp, i32, _ip, _dp]),
    ("dtg_set_noise", i32, [vp, i32, u64, u64]),
    ("dtg_forward", i32, [vp, i32, i32, i32]),
    ("dtg_sync", i32, [vp]),
    ("dtg_forward_read", i32, [vp, i32, i32, i32, vp, vp, vp]),
    ("dtg_debug_force_slow_path", i32, [vp, i32]),
    ("dtg_read_cum", i32, [vp, i32, _dp]),
    ("dtg_read_cum_all", i32, [vp, _dp]),
    ("dtg_read_state", i32, [vp, i32, i32, _ip, _dp]),
    ("dtg_n_snapshots", i32, [vp]),
    ("dtg_set_record_transfers", i32, [vp, i32]),
    ("dtg_read_transfers", i32, [vp, i32, _ip]),
    ("dtg_transfer_events", i32, [vp, i32, vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("dtg_scenario_set_record_transfers", i32, [vp, i32]),
    ("dtg_backward", i32, [vp, vp, vp, vp, _dp]),
    ("dtg_backward_device", i32, [vp, vp, vp, vp, vp]),
    ("dtg_set_loss_mse", i32, [vp, i32, i32, _ip, _dp]),
    ("dtg_set_loss_control", i32, [vp, i32, C.c_double]),
    ("dtg_gradient_device_loss", i32, [vp, vp]),
    ("dtg_reduce_draw_rows", i32, [vp, i32, vp, i32, _dp]),
    ("dtg_reduce_draw_rows_head", i32, [vp, i32, vp, i32, _dp]),
    ("dtg_read_reduced_row", i32, [vp, _dp]),
    ("dtg_opt_bounded_init", i32, [vp, _dp, _dp, _dp] + [C.c_double] * 5),
    ("dtg_opt_bounded_step", i32, [vp, i32, C.c_double, C.c_double]),
    ("dtg_opt_bounded_mark_best", i32, [vp]),
    ("dtg_opt_bounded_read", i32, [vp, vp, vp]),
    ("dtg_device_cum", vp, [vp]),
    ("dtg_profile_kernels", i32, [vp, i32, i32, i32, _dp, C.POINTER(C.c_int64)]),
    ("dtg_kernel_name", C.c_char_p, [i32, i32]),
    ("dtg_last_launches", C.c_int64, [vp]),
    ("dtg_scenario_from_links", vp, [i32, i32, _ip, _ip, _dp, _ip]),
    ("dtg_scenario_grid", vp, [i32, C.c_double, u64, C.c_double]),
    ("dtg_scenario_tntp", vp, [C.c_char_p, C.c_double, u64, C.c_double]),
    ("dtg_scenario_free", None, [vp]),
    ("dtg_scenario_configure", i32, [vp, i32, i32, C.c_double, C.c_double, i32, i32, i32, i32]),
    ("dtg_scenario_custom_init", i32, [vp, i32, _ip, _dp]),
    ("dtg_scenario_n_links", i32, [vp]),
    ("dtg_scenario_n_nodes", i32, [vp]),
    ("dtg_scenario_n_agents", i32, [vp]),
    ("dtg_scenario_links", i32, [vp, _ip, _ip, _dp, _ip]),
    ("dtg_scenario_n_edges", i32, [vp]),
    ("dtg_scenario_csr", i32, [vp, _ip, _ip]),
    ("dtg_scenario_sample_parameters", i32, [vp, u64, i32, _dp, _dp, _dp, _dp, _dp]),
    ("dtg_scenario_seed_agents", i32, [vp, _ip, _dp]),
    ("dtg_steps_for_minutes", i32, [i32, C.c_double, C.c_double]),
    ("dtg_simulate_forward", i32, [vp, _dp, _dp, _dp, _dp, _dp, u64, i32, _u64p, vp, vp, vp, vp, vp, vp]),
    ("dtg_simulate_gradient", i32, [vp, _dp, _dp, _dp, _dp, _dp, u64, i32, _u64p,
                                    vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    ("dtg_simulate_gradient_mse", i32, [vp, _dp, _dp, _dp, _dp, _dp, u64, i32, _u64p,
                                        i32, _ip, i32, _dp, vp, vp]),
    ("dtg_calibrate", i32, [vp, i32, _ip, i32, _dp, vp, vp, u64, vp, vp, vp, vp, vp,
                            _dp, _dp, _dp, _dp, _dp, vp, vp, vp, _dp, vp, vp]),
    ("dtg_optimize_control", i32, [vp, _dp, _dp, _dp, _dp, _dp, i32, C.c_double, vp,
                                   C.c_double, u64, _dp, vp, vp, vp, vp, _dp, vp, vp, vp]),
    ("dtg_observe_last_error", C.c_char_p, []),
    ("dtg_synthesize_observations", i32, [i32, i32, _ip, _dp, i32, C.c_double, C.c_double, u64,
                                          C.POINTER(C.c_int), _ip, _dp]),
    ("dtg_count_metrics", i32, [i32, i32, _ip, _dp, i32, i32, _ip, _dp, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("dtg_series_to_csv", i32, [i32, i32, _ip, _dp, i32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("dtg_series_from_csv", i32, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  vp, vp, C.c_size_t, C.c_size_t]),
    ("dtg_scenario_ctx", vp, [vp]),
    ("dtg_mse_loss", i32, [i32, i32, _dp, i32, _ip, i32, _dp, i32, _dp, _dp]),
    ("dtg_debug_gumbel", i32, [u64, u64, i32, _u64p, _u64p, _dp]),
    ("dtg_debug_decisions", i32, [i32, C.POINTER(C.c_ulonglong)]),
    ("dtg_debug_microbench", i32, [i32, i32, i32, _dp]),
    ("dtg_debug_l2_bandwidth", i32, [C.c_longlong, i32, C.POINTER(C.c_double)]),
    ("dtg_debug_step_floor", i32, [i32, i32, C.POINTER(C.c_double)]),
    ("dtg_debug_log_check", i32, [u64, C.c_longlong, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    ("dtg_debug_libm_check", i32, [i32, u64, C.c_longlong, i32, C.POINTER(C.c_ulonglong)]),
    ("dtg_debug_warp_records", i32, [vp, i32, i32, vp, C.POINTER(C.c_int)]),
    ("dtg_debug_bwd_stamps", i32, [vp, vp, C.POINTER(C.c_int)]),
    ("dtg_scenario_last_error", C.c_char_p, [vp]),
    # FD-validation instrumentation
    ("dtg_surrogate_create", vp, []),
    ("dtg_surrogate_free", None, [vp]),
    ("dtg_surrogate_set_replay", i32, [vp, i32]),
    ("dtg_surrogate_rewind", i32, [vp]),
    ("dtg_scenario_set_soft_choices", i32, [vp, i32]),
    ("dtg_scenario_set_surrogate", i32, [vp, vp]),
    ("dtg_simulate_forward_traced", i32, [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, i32, vp, vp, vp, _u64p, vp]),
    ("dtg_simulate_gradient_traced", i32, [vp, _dp, _dp, _dp, _dp, _dp, u64, u64, i32, i32,
                                           vp, vp, vp, vp, vp, vp, _dp, vp, _u64p]),
    ("dtg_probe_forward_batch", i32, [vp, i32, _dp, u64, u64, i32, vp, vp, vp, vp]),
    ("dtg_run_gradcheck", i32, [i32, i32, i32, C.c_double, u64, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                _dp]),
]

_lib = None


def load() -> C.CDLL:
    """Load libdtg.so (raises if it was not built: no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"native library {LIB_PATH} is missing; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def load_other(path: str) -> C.CDLL:
    """Measurement only (A/B against another build, scripts/): load `path` in
    place of the in-tree library; symbols it lacks stay unbound."""
    global _lib
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype = res
            fn.argtypes = args
    _lib = lib
    return lib


def ptr(a):
    """ctypes void* of a numpy array (or None)."""
    return None if a is None else a.ctypes.data_as(C.c_void_p)
