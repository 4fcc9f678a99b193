"""bench.py's reference arm (the CPU oracle) prints one JSON
line with the contract's keys; runs on CPU in seconds (K16)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "K16",
                        "--steps", "1", "--warmup", "0", "--ref-seconds", "0.3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "flips/s" and d["value"] > 0
    assert d["config"]["workload"] == "K16"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_flag_launches_n_ranks():
    """`bench.py --gpus N` (no torchrun environment) starts N ranks itself
    through torch.distributed.run on 127.0.0.1 (the driver's scaling runs);
    checked on CPU with the launcher self-test (gloo group of N processes)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    for n in (2, 3):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launcher-selftest"],
                           capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
        assert d["n_ranks"] == n and d["ranks"] == list(range(n)) and d["pids_distinct"]
