"""bench.py's command-line contract on CPU: --gpus N > 1 outside torchrun relaunches
itself as N ranks through torch.distributed.run on 127.0.0.1 (so a driver call
`python bench.py --gpus 8` measures 8 NCCL ranks, VERDICT r1 missing #2)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    import bench

    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3", "--warmup", "3"])
    assert bench.main() == 0
    (cmd,) = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--warmup", "3"]


def test_reference_arm_other_ranks_exit(monkeypatch):
    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    assert bench.main() == 0


def test_host_facts():
    import bench

    f = bench.host_facts()
    assert f["nproc"] >= 1 and "cpu_model" in f and f["ram_gib"] > 0
