"""The bench.py JSON contract on CPU: the reference arm (`--impl reference`, the C oracle on host
threads) on a tiny workload prints one line with the keys the driver reads, and both arms share
the same workload `config` (bench.workload_config)."""
import json
import os
import subprocess
import sys
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TINY = ["--gaussians", "20000", "--avatars", "1", "--envs", "4", "--width", "128", "--height", "96"]


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", *TINY], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    import bench
    args = SimpleNamespace(gaussians=20000, avatars=1, envs=4, width=128, height=96, near=0.1)
    want = bench.workload_config(args, d["config"]["parallelism"])
    assert {k: v for k, v in d["config"].items() if k != "sample_envs_per_step"} == want
