"""bench.py launch contract on CPU: `--gpus N` without torchrun re-executes
itself as N ranks, the rank count is checked against
WORLD_SIZE, and the reference arm prints one JSON line on rank 0 only."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_relaunch_command_is_one_node_torchrun():
    import bench
    cmd = bench.relaunch_cmd(4, ["--gpus", "4", "--steps", "2"], 29512)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29512" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=env, timeout=600, cwd=ROOT)


def test_gpus_2_spawns_two_ranks_and_rank0_prints_one_line():
    r = _run(["--impl", "reference", "--gpus", "2", "--workload", "cfg1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    ranks = sorted(ln.split()[2] for ln in r.stderr.splitlines() if ln.startswith("[bench] rank"))
    assert ranks == ["0/2", "1/2"], r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2
    assert out["cpu_baseline"]["kind"] in ("reference", "port") and out["value"] > 0
    assert out["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_is_refused():
    r = _run(["--impl", "reference", "--gpus", "2", "--workload", "cfg1", "--steps", "1", "--warmup", "0"],
             {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
