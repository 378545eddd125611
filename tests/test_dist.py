"""N > 1 host path on CPU: world_size-2 gloo process group.  Each rank owns a
contiguous block of noise draws; per-draw gradients are gathered and summed in
draw order, which must be bit-identical to the single-process sequential sum
(the reference's draw loop, optimization.cpp:173-191).  The C oracle stands in
for the device engine on this GPU-less host."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_all_draws():
    from paper_2603_25068_b200.dist import shard

    for world in (1, 2, 4, 8):
        got = [k for r in range(world) for k in shard(8, world, r)]
        assert got == list(range(8))
    with pytest.raises(ValueError):
        shard(8, 3, 0)


def _port_case():
    from oracle.oracle import PortLib, PortScenario
    import paper_2603_25068_b200 as P

    sc = P.Scenario.grid(4, 400.0, 42, 1000.0).configure(1000, 1, 120, 60)
    f, t, ln, _ = sc.links()
    lk, ps = sc.seed_agents()
    port = PortScenario(PortLib(), f, t, ln, link0=lk, pos0=ps, horizon_steps=120, obs_interval_s=60)
    return sc, port, sc.sample_parameters(3)


def _per_draw(port, p, k, L):
    rng = np.random.default_rng(k)
    g = port.gradient(p, 7, k + 1, ws=rng.normal(size=(2, L)))
    return np.concatenate([g["grads"].ravel(), [g["loss"] / 8]])


def _worker(rank, world, port_no, out_dir):
    import torch.distributed as dist

    from paper_2603_25068_b200.dist import gather_ordered_sum, shard

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank, world_size=world)
    sc, port, p = _port_case()
    rows = np.stack([_per_draw(port, p, k, sc.n_links) for k in shard(8, world, rank)])
    full, total = gather_ordered_sum(torch.from_numpy(rows), world)
    np.save(os.path.join(out_dir, f"total_{rank}.npy"), total.numpy())
    np.save(os.path.join(out_dir, f"full_{rank}.npy"), full.numpy())
    dist.destroy_process_group()


def test_gloo_world2_gather_matches_sequential_sum(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sc, port, p = _port_case()
    rows = [_per_draw(port, p, k, sc.n_links) for k in range(8)]
    seq = rows[0].copy()
    for r in rows[1:]:
        seq += r
    for rank in range(world):
        assert np.array_equal(np.load(tmp_path / f"total_{rank}.npy"), seq)
        assert np.array_equal(np.load(tmp_path / f"full_{rank}.npy"), np.stack(rows))
