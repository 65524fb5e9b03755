"""CPU: bench.py's reference arm runs on the host (no GPU needed) and prints
the driver's JSON line; the algorithmic-byte model follows SURVEY.md §8d."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_algorithmic_bytes():
    b = bench.algorithmic_bytes(n=10, m=20, aot_cost=30, triangles=4)
    assert b["count"] == 8 * 11 + 4 * 20 + 4 * 20 + 4 * 30
    assert b["list"] == b["count"] + 12 * 4


def test_sample_config_bounded():
    cfg, desc = bench.sample_config("c4")
    assert cfg["npairs"] <= 16 << 20 and cfg["kind"] == "rmat"
    cfg, desc = bench.sample_config("c2")
    assert cfg["npairs"] == 16 << 20 and desc.startswith("full")


def test_reference_arm_json_line():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0", "--cpu-threads", "2"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] == 2
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))["c1"]
    assert line["config"]["m"] == golden["m"] and line["config"]["triangles"] == golden["triangles"]


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""
