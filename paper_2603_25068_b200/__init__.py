"""B200-native hot path of the differentiable mesoscopic traffic simulator
(arXiv 2603.25068; reference implementation dtsim 1.0.0).

The per-tick vehicle update (Newell car-following, Gumbel-softmax link and
merge choice with straight-through gradients and trajectory grafting,
midpoint counting) and its checkpointed reverse-mode adjoint run as
hand-written sm_100a kernels in ``libdtg.so``; the host API mirrors the
reference's ``simulate_forward`` / ``simulate_gradient``.
"""
from ._lib import ConfigError, DivergenceError, DtgError, UnsupportedError, load  # noqa: F401
from .engine import (  # noqa: F401
    PHYSICAL,
    VIRTUAL_INFLOW,
    VIRTUAL_OUTFLOW,
    CalibrationResult,
    ControlResult,
    Engine,
    GradResult,
    LinkParams,
    OptimizeConfig,
    ParamRanges,
    Scenario,
    Trajectory,
    calibrate,
    link_visits,
    optimize_control,
    pinned_empty,
    simulate_forward,
    simulate_gradient,
    simulate_gradient_mse,
    steps_for_minutes,
    transfer_events,
)

__version__ = "0.1.0"
