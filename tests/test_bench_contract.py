"""bench.py's reference arm (the fp64 oracle on the host cores, `--impl reference`) prints the
driver's JSON line; runs on CPU in seconds."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                                   "--warmup", "0"], cwd=ROOT, text=True, timeout=600)
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "images/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]
    assert "workload" in d["config"]


def test_gpus_flag_spawns_ranks():
    """bench.py --gpus 2 run directly (no WORLD_SIZE) re-executes itself under torchrun: each rank sees
    RANK, LOCAL_RANK, WORLD_SIZE = 2 and the group spans both (gloo all-gather; no GPU needed)."""
    import json, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "env"],
                         capture_output=True, text=True, timeout=180, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    recs = sorted((json.loads(l[4:]) for l in out.stdout.splitlines() if l.startswith("ENV ")), key=lambda r: r["rank"])
    assert [r["rank"] for r in recs] == [0, 1]
    assert [r["local_rank"] for r in recs] == [0, 1]
    assert all(r["world_size"] == 2 and r["gathered_ranks"] == [0, 1] for r in recs)
    assert recs[0]["pid"] != recs[1]["pid"]


def test_gpus_must_match_world_size():
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "env"],
                         capture_output=True, text=True, timeout=120, env=env, cwd=root)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
