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
                        "--warmup", "3", "--ref-budget", "4"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == os.cpu_count()
    assert d["cpu_baseline"]["nproc"] == os.cpu_count() and d["cpu_baseline"]["cpu_model"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_algorithmic_bytes():
    sys.path.insert(0, ROOT)
    import bench
    # C2: 257^3 nodes, 256^3 elements: 81 B per node (u, u_prev, u_next, w, mask) + 1 B per element
    nn, ne = 257 ** 3, 256 ** 3
    assert bench._algorithmic_bytes(nn, ne) == 81 * nn + ne


def test_gpus_n_without_torchrun_refuses_when_gpus_are_missing():
    """`python bench.py --gpus N` (no WORLD_SIZE) relaunches itself as N ranks; with fewer than N
    GPUs visible it exits non-zero instead of silently measuring one GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "OVX_BENCH_DEVICE")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 2 and "needs 2 GPUs" in r.stderr and r.stdout.strip() == ""


def test_gpus_n_spawns_n_ranks(monkeypatch):
    """The relaunch command: torch.distributed.run with N processes on 127.0.0.1, same arguments."""
    sys.path.insert(0, ROOT)
    import bench
    seen = {}
    monkeypatch.setenv("OVX_BENCH_DEVICE", "0")        # test hook: do not require N devices
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    assert bench._spawn_ranks(4) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "7"]


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode != 0 and r.stdout.strip() == ""
