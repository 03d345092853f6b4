"""bench.py's reference arm (the CPU oracle timed on the host cores) keeps the
driver's JSON-line contract at N = 1 and under torchrun-style N > 1 (rank 0
prints, the other ranks exit 0 without work).  CPU only."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--size-mib", "4",
                        "--steps", "1", "--warmup", "0"] + args, capture_output=True, text=True, env=env,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    return r.stdout.strip().splitlines()


def test_reference_arm_n1():
    (line,) = _run([])
    d = json.loads(line)
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["ranks"] == 8
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_multi_rank0_prints_others_silent():
    (line,) = _run(["--gpus", "4"], {"RANK": "0", "WORLD_SIZE": "4"})
    d = json.loads(line)
    assert d["n_gpus"] == 4 and d["config"]["ranks"] == 4 and d["scaling"] == "weak"
    assert _run(["--gpus", "4"], {"RANK": "2", "WORLD_SIZE": "4"}) == []
