"""The bench.py JSON contract on CPU: the reference arm (`--impl reference`, the C oracle on host
threads) on a tiny workload prints one line with the keys the driver reads, both arms share the
same workload `config` (bench.workload_config), `--gpus N` re-launches itself as N torchrun ranks
(rank 0 alone prints) and a mismatched WORLD_SIZE is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TINY = ["--gaussians", "20000", "--avatars", "1", "--envs", "4", "--width", "128", "--height", "96"]


def _run(extra, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                           "--warmup", "0", *TINY, *extra], capture_output=True, text=True, timeout=600, cwd=ROOT,
                          env=e)


def _line(out):
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(_run([]))
    assert d["impl"] == "reference"
    assert d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    import bench
    args = bench.parse(["--config", "2", *TINY])
    assert d["config"] == bench.workload_config(args, 1)  # identical to the GPU arm's config object


def test_gpus_flag_relaunches_as_ranks():
    """--gpus 2 without a torchrun environment: bench.py runs itself as 2 ranks (127.0.0.1);
    the reference arm prints from rank 0 only."""
    d = _line(_run(["--gpus", "2"]))
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["parallelism"] == "env-sharded x2"


def test_mismatched_world_size_is_refused():
    out = _run(["--gpus", "4"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode == 2 and "refusing" in out.stderr


def test_config4_shards_a_fixed_batch():
    import bench
    args = bench.parse(["--config", "4"])
    assert (args.gaussians, args.envs, args.avatars) == (3_000_000, 1024, 4)
    for world in (1, 2, 4, 8):
        spans = [bench.envs_of_rank(args, world, r) for r in range(world)]
        assert sum(n for _, n in spans) == 1024 and spans[0][0] == 0
        assert all(a + n == b for (a, n), (b, _) in zip(spans, spans[1:]))
    cfg = bench.workload_config(args, 8)
    assert cfg["total_envs"] == 1024 and cfg["scaling"] == "strong"
