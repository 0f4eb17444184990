"""bench.py --gpus N launches N ranks itself (torch.distributed.run on
127.0.0.1) when no torchrun environment is present; checked on CPU with the
launcher self-test (gloo, one all-reduce)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_launch_cmd_shape():
    sys.path.insert(0, str(ROOT))
    import bench

    cmd = bench.launch_cmd(["--gpus", "4", "--steps", "3"], 4, 29512)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-port=29512" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:]


def test_bench_self_launches_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "3", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 3 and line["world_env"] == 3 and line["rank_sum"] == 1 + 2 + 3
    assert out.stderr.count("[bench] rank ") == 3  # every rank logs its communicator
