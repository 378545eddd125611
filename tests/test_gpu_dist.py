"""World-2 run of the PRODUCT draw-exchange path (dtg_draw_exchange ->
DeviceLoop -> dtg_calibrate / dtg_optimize_control), not the C port: two
processes, each with its own device context on the one GPU a test box has,
exchange their per-draw rows with a host-staged gloo all-gather.  Each rank
runs only its half of the draws; after the gather both must return the
world-1 result bit for bit (draw-ordered reduction).  The ranks'
kernels never wait on each other — the only coupling is the host-side gather.
"""
import os
import socket

import numpy as np
import pytest

from golden_cases import load

P = pytest.importorskip("paper_2603_25068_b200")
torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    d = load("calib_grid3")
    sc = P.Scenario.grid(3, 300.0, 42, 600.0).configure(300, 1, 120, 30)
    return d, sc


CAL = dict(max_iterations=4, patience=10, noise_draws=4, lr=0.1)
CTL = dict(max_iterations=4, patience=10, noise_draws=4, lr=0.2)


def _run(world, rank, host_staged):
    from paper_2603_25068_b200.dist import calibrate_sharded, optimize_control_sharded

    d, sc = _case()
    cal = calibrate_sharded(sc, d["obs_ids"], d["obs"], 5, cfg=P.OptimizeConfig(**CAL), world=world, rank=rank,
                            host_staged=host_staged)
    c = load("control_grid3")
    ctl = optimize_control_sharded(sc, P.LinkParams(*c["params"]), int(c["target"]), float(c["desired"]), 7,
                                   cfg=P.OptimizeConfig(**CTL), world=world, rank=rank, host_staged=host_staged)
    return dict(curve=cal.loss_curve, best=np.stack(cal.best_params.arrays()), ccurve=ctl.loss_curve,
                cost=ctl.cost, achieved=np.float64(ctl.achieved))


def _worker(rank, world, port_no, out_dir):
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank, world_size=world)
    out = _run(world, rank, host_staged=True)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    dist.destroy_process_group()


def test_world2_product_exchange_bit_identical_to_world1(tmp_path):
    import torch.multiprocessing as mp

    ref = _run(1, 0, host_staged=False)
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for rank in range(2):
        got = dict(np.load(tmp_path / f"rank{rank}.npz"))
        for k, v in ref.items():
            assert np.array_equal(got[k], v), (rank, k)


def test_world2_without_stream_is_rejected():
    """with world > 1 the gather is ordered after the rows only
    through the exchange's stream, so a NULL stream must be refused."""
    from paper_2603_25068_b200._lib import DrawExchange, GatherFn

    d, sc = _case()
    local = torch.zeros((2, 5 * sc.n_links + 2), dtype=torch.float64, device="cuda")
    full = torch.zeros((4, 5 * sc.n_links + 2), dtype=torch.float64, device="cuda")
    cb = GatherFn(lambda _u: 0)
    ex = DrawExchange(2, 0, local.data_ptr(), full.data_ptr(), None, cb, None)
    with pytest.raises(Exception, match="stream"):
        P.calibrate(sc, d["obs_ids"], d["obs"], 5, cfg=P.OptimizeConfig(**CAL), exchange=ex)


def test_exchange_stream_is_released_after_the_loop():
    """The cached scenario context returns to its own stream when the loop
    that rebound it to the exchange's stream ends."""
    import ctypes as C

    from paper_2603_25068_b200._lib import load as L
    from paper_2603_25068_b200.dist import calibrate_sharded

    d, sc = _case()
    st = torch.cuda.Stream()
    calibrate_sharded(sc, d["obs_ids"], d["obs"], 5, cfg=P.OptimizeConfig(**CAL), stream=st)
    ctx = sc.device_context()
    s, owned = C.c_void_p(), C.c_int()
    assert L().dtg_get_stream(ctx, C.byref(s), C.byref(owned)) == 0
    assert owned.value == 1 and s.value != st.cuda_stream
