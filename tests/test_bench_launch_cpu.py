"""CPU: `python bench.py --gpus N` launches itself (the driver calls it without torchrun), and says clearly what is
missing when the node has fewer than N GPUs."""
import json
import os
import subprocess
import sys

from helpers import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _env(**extra):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(extra)
    return env


def test_self_launch_starts_one_rank_per_gpu():
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "1"], env=_env(LTL_BENCH_LAUNCH_ONLY="1"),
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 and l["launch_only"] and l["master"] == "127.0.0.1" for l in lines)


def test_under_torchrun_no_second_launch():
    """With WORLD_SIZE set (the torchrun form of the contract) bench.py must not launch again."""
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2"],
                         env=_env(LTL_BENCH_LAUNCH_ONLY="1", WORLD_SIZE="2", RANK="1", LOCAL_RANK="1", MASTER_ADDR="127.0.0.1"),
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    (line,) = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert (line["rank"], line["world"]) == (1, 2)


def test_too_few_gpus_is_a_clear_error():
    import torch

    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    out = subprocess.run([sys.executable, BENCH, "--gpus", str(have + 1 if have else 2)], env=_env(), capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 2
    assert "CUDA devices on this node" in out.stderr and "no CPU fallback" in out.stderr


def test_launch_command_shape():
    sys.path.insert(0, ROOT)
    import bench

    cmd = bench.self_launch_command(4, ["--gpus", "4", "--steps", "2"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
