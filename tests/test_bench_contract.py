"""bench.py's launch contract on CPU: `--gpus N` without a launcher re-execs
itself under torch.distributed.run with N ranks (a plain
`python bench.py --gpus 8` used to measure one GPU), and a rank count that
disagrees with --gpus is refused."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    import bench

    seen = {}

    def fake_exec(prog, argv, env):
        seen.update(prog=prog, argv=argv, env=env)
        raise SystemExit(0)

    monkeypatch.setattr(os, "execvpe", fake_exec)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    with pytest.raises(SystemExit):
        bench.main()
    argv = seen["argv"]
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_world_size_must_match_gpus(monkeypatch):
    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        bench.dist_setup(4)
