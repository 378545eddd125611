"""Multi-GPU: independent stochastic draws sharded over ranks.

The path shards only across noise draws: calibrate() and
optimize_control() average `noise_draws` independent simulate_gradient calls
(/root/reference/proj/src/optimization.cpp:168-191, 248-265).  One process per
GPU runs its contiguous block of draws as one batched device pass; the only
collective is a gather of the per-draw gradient blocks (5 x L fp64 each) and
losses over NCCL, after which every rank sums them in draw order — the
reference's sequential `grads += g.grads` order (optimization.cpp:181-190) —
so the result is bit-identical for 1, 2, 4 or 8 GPUs.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np


def shard(n_draws: int, world: int, rank: int) -> range:
    """Contiguous block of draw indices owned by `rank` (rank-major order)."""
    if n_draws % world:
        raise ValueError(f"{n_draws} draws do not divide over {world} ranks")
    per = n_draws // world
    return range(rank * per, (rank + 1) * per)


def gather_ordered_sum(local, world: int, group=None):
    """All-gather the per-draw blocks `local` [d_local, ...] (torch tensor on
    the communicator's device) and return (all_blocks [D, ...], ordered_sum)."""
    import torch

    if world == 1:
        full = local
    else:
        import torch.distributed as dist

        full = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                           device=local.device)
        dist.all_gather_into_tensor(full, local.contiguous(), group=group)
    acc = full[0].clone()
    for k in range(1, full.shape[0]):
        acc += full[k]
    return full, acc


def calibration_draws(it: int, draws: int) -> List[int]:
    """noise_iteration of draw k at iteration it (optimization.cpp:175-177)."""
    return [it * draws + k + 1 for k in range(draws)]


class ShardedGradient:
    """Sum over `n_draws` draws of simulate_gradient, sharded over ranks.

    `seeds_fn(snapshots [d, K, L], cum_final [d, L]) -> (loss [d], snap_seeds
    [d, K, L], cum_seeds [d, L])` is the host loss (the reference's host loss
    tape, engine.cpp:369-385) applied to this rank's draws.  Returns
    (mean loss, ordered sum of the per-draw [5, L] gradients, all gathered
    per-draw rows).
    """

    def __init__(self, scenario, n_draws: int, world: int = 1, rank: int = 0, device=None,
                 stream_ptr: Optional[int] = None):
        from .engine import Engine

        self.sc = scenario
        self.n_draws, self.world, self.rank = n_draws, world, rank
        self.mine = shard(n_draws, world, rank)
        self.engine = Engine(scenario, n_scenarios=len(self.mine), max_steps=max(1, scenario.horizon_steps))
        if stream_ptr:
            self.engine.set_stream(stream_ptr)
        self.link0, self.pos0 = scenario.seed_agents()
        self.engine.set_state(self.link0, self.pos0)
        self.device = device

    def __call__(self, params, root_seed: int, noise_iterations: Sequence[int],
                 seeds_fn: Callable, group=None):
        import torch

        sc, e = self.sc, self.engine
        T, spi = sc.horizon_steps, sc.steps_per_interval
        e.set_params(params)
        for b, k in enumerate(self.mine):
            e.set_noise(root_seed, noise_iterations[k], b)
        e.forward(T, spi, checkpoint=True)
        K = T // spi
        cum = e.read_cum_all() if T else np.zeros((len(self.mine), 0, sc.n_links))
        snaps = cum[:, spi - 1::spi][:, :K]
        cum_final = cum[:, -1] if T else np.zeros((len(self.mine), sc.n_links))
        loss, snap_seeds, cum_seeds = seeds_fn(snaps, cum_final)
        g = e.backward(snap_seeds=snap_seeds, cum_seeds=cum_seeds) if T else \
            np.zeros((len(self.mine), 5, sc.n_links))
        dev = self.device or (torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
        # loss enters as loss_k / draws, summed in draw order (optimization.cpp:180)
        lk = np.asarray(loss, dtype=np.float64).reshape(-1, 1) / self.n_draws
        local = torch.from_numpy(np.concatenate([g.reshape(len(self.mine), -1), lk], axis=1)).to(dev)
        full, total = gather_ordered_sum(local, self.world, group)
        total = total.cpu().numpy()
        return float(total[-1]), total[:-1].reshape(5, sc.n_links), full.cpu().numpy()


class DeviceDrawExchange:
    """NCCL draw exchange for the device-resident optimisation loops
    (include/dtg.h dtg_draw_exchange): this rank's per-draw rows
    [D/world, 5L+2] are all-gathered, rank-major (= draw order), into
    [D, 5L+2] on `stream`, and every rank reduces all D rows in draw order on
    its device, so calibrate / optimize_control return the single-GPU result
    bit for bit for any world size.  Only O(L) bytes per draw cross NVLink per
    iteration; nothing goes through host memory except the reduced row."""

    def __init__(self, n_links: int, n_draws: int, world: int, rank: int, group=None, stream=None,
                 host_staged: bool = False):
        """host_staged: gather through host memory with a CPU backend (gloo)
        instead of NCCL on the device — the same rows in the same order, for
        process groups without NCCL (e.g. several ranks sharing one GPU in a
        test)."""
        import torch
        import torch.distributed as dist

        from ._lib import DrawExchange, GatherFn

        shard(n_draws, world, rank)  # validates divisibility
        R = 5 * n_links + 2
        self.stream = stream or torch.cuda.Stream()
        self.local = torch.zeros((n_draws // world, R), dtype=torch.float64, device="cuda")
        self.full = torch.zeros((n_draws, R), dtype=torch.float64, device="cuda")
        self.group = group
        self.calls = 0
        self.error = None

        def _gather(_user):
            try:
                with torch.cuda.stream(self.stream):
                    if world > 1 and host_staged:
                        self.stream.synchronize()  # the rows are written on this stream
                        h_local = self.local.cpu()
                        h_full = torch.empty(self.full.shape, dtype=self.full.dtype)
                        dist.all_gather_into_tensor(h_full, h_local, group=self.group)
                        self.full.copy_(h_full)
                    elif world > 1:
                        dist.all_gather_into_tensor(self.full, self.local, group=self.group)
                    else:
                        self.full.copy_(self.local)
                self.calls += 1
                return 0
            except Exception as e:  # reported as a runtime error by the C++ loop
                self.error = e
                return 1

        self._cb = GatherFn(_gather)  # keep the trampoline alive
        self.c = DrawExchange(world, rank, self.local.data_ptr(), self.full.data_ptr(),
                              self.stream.cuda_stream, self._cb, None)


def calibrate_sharded(sc, obs_ids, obs_values, seed: int, cfg=None, bounds=None, init=None,
                      world: int = 1, rank: int = 0, group=None, stream=None, host_staged: bool = False):
    """calibrate() with the iteration's noise draws sharded over `world` GPUs."""
    from .engine import OptimizeConfig, calibrate

    cfg = cfg or OptimizeConfig()
    draws = max(1, cfg.noise_draws) if cfg.resample_noise else 1
    ex = DeviceDrawExchange(sc.n_links, draws, world, rank, group, stream, host_staged)
    return calibrate(sc, obs_ids, obs_values, seed, bounds=bounds, cfg=cfg, init=init, exchange=ex.c)


def optimize_control_sharded(sc, calibrated, target_link: int, desired: float, seed: int, cfg=None,
                             cost_floor: float = 0.05, world: int = 1, rank: int = 0, group=None, stream=None,
                             host_staged: bool = False):
    """optimize_control() with the iteration's noise draws sharded over `world` GPUs."""
    from .engine import OptimizeConfig, optimize_control

    cfg = cfg or OptimizeConfig()
    draws = max(1, cfg.noise_draws) if cfg.resample_noise else 1
    ex = DeviceDrawExchange(sc.n_links, draws, world, rank, group, stream, host_staged)
    return optimize_control(sc, calibrated, target_link, desired, seed, cfg=cfg, cost_floor=cost_floor,
                            exchange=ex.c)
