"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line (bench.py --impl reference: the reference's compiled primitives, or the
C oracle when oracle/_ref is absent, timed on the host cores) and its
behaviour under torchrun (rank 0 alone runs and prints; other ranks exit 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                           "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, cwd=ROOT,
                          timeout=900)


def test_reference_arm_line():
    out = _run({"RANK": "0", "WORLD_SIZE": "2"})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "KS/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("key-switches/s") and d["n_gpus"] == 2 and d["steps"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["N"] == 65536 and d["config"]["chain_primes"] == 24 and d["config"]["special_primes"] == 3
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "KS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    out = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert out.returncode == 0
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
