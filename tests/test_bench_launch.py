"""bench.py's launch contract on CPU: `--gpus N` without torchrun's
environment re-launches itself as N ranks (gloo here, NCCL on the GPU box),
the max-over-ranks reduction runs, and both arms print the same `config`."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


@pytest.mark.parametrize("config,n,items", [("c3", 2, [0, 32]), ("c5", 2, [0, 128]),
                                            ("c5", 4, [0, 64])])
def test_gpus_flag_spawns_the_ranks(config, n, items):
    res = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--config", config,
                          "--spawn-selftest"], capture_output=True, text=True, timeout=300,
                         env=_env(), cwd=ROOT)
    assert res.returncode == 0, res.stdout + res.stderr
    line = _last_json(res.stdout)
    assert line["n_gpus"] == n and line["max_over_ranks"] == float(n)
    assert line["rank0_items"] == items
    assert line["config"]["global_batch"] == (32 * n if config == "c3" else 256)


def test_world_size_must_match_gpus():
    res = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--spawn-selftest"],
                         capture_output=True, text=True, timeout=120,
                         env=_env(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"), cwd=ROOT)
    assert res.returncode != 0
    assert "WORLD_SIZE=1" in res.stderr


@pytest.mark.slow
def test_reference_arm_prints_the_workload_config():
    """`--impl reference` (the reference engine on the host) carries the same
    workload-only config object as our arm (bench.workload_config)."""
    from oracle import oracle as o

    if not o.Reference.available():
        o.build()
    if not o.Reference.available():
        pytest.skip("reference library not built")
    sys.path.insert(0, ROOT)
    import bench

    res = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--config", "c5",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, env=_env(), cwd=ROOT)
    assert res.returncode == 0, res.stderr
    line = _last_json(res.stdout)
    assert line["impl"] == "reference" and line["config"] == bench.workload_config("c5", 1)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
