"""bench.py launcher contract on CPU: `--gpus N` without torchrun re-executes as N ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, timeout=300, env=env, cwd=ROOT)


def test_gpus_2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["ranks"] == [0, 1]
    assert "torch.distributed.run" in r.stderr and "--nproc-per-node=2" in r.stderr


def test_gpus_mismatch_with_world_size_fails_loudly():
    r = _run(["--gpus", "4", "--launch-check"], {"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in r.stderr


def test_reference_arm_line_is_consistent():
    """--impl reference (the reference arithmetic on the host cores): one JSON line whose value
    equals transforms_per_step / step time, so ms_per_step x steps is the real run time."""
    r = _run(["--impl", "reference", "-B", "8", "--steps", "2", "--warmup", "1", "--cpu-stride", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["unit"] == "transforms/s" and rec["higher_is_better"]
    assert abs(rec["value"] - rec["transforms_per_step"] * 1000.0 / rec["ms_per_step"]) < 1e-9 * rec["value"]
    cpu = rec["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["cores"] >= 1 and cpu["extrapolated"]
    assert 0.0 < rec["transforms_per_step"] < 2.0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0
