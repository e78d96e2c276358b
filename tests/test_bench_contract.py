"""bench.py's driver contract on CPU: the reference arm (the CPU port of the
reference path) prints one JSON line with the required keys, on the same
metric / config as the GPU arm; under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

from conftest import ROOT

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _run(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=300, env=env or dict(os.environ))
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run(["--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "0", "--ref-rows", "256"])
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert REQUIRED <= set(j), REQUIRED - set(j)
    assert j["impl"] == "reference" and j["unit"] == "dist-evals/s" and j["higher_is_better"] is True
    assert j["value"] > 0 and j["cpu_baseline"]["kind"] == "port" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]
    assert "workload" in j["config"]


def test_reference_arm_non_zero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    assert _run(["--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "0", "--ref-rows", "64"],
                env) == []
