"""bench.py's contract pieces that run on CPU: the reference arm (the oracle timed on a bounded
sample; the driver runs `bench.py --impl reference`) prints one JSON line with the required keys,
and the algorithmic-bytes formula matches SURVEY §8(d)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_algorithmic_bytes():
    sys.path.insert(0, ROOT)
    import bench
    # C2: 257^3 nodes, 256^3 elements: 81 B per node (u, u_prev, u_next, w, mask) + 1 B per element
    nn, ne = 257 ** 3, 256 ** 3
    assert bench._algorithmic_bytes(nn, ne) == 81 * nn + ne
