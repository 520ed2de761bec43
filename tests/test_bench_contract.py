"""The driver's bench contract on CPU: `bench.py --impl reference` (the oracle arm) prints one JSON line with the
metric, unit, impl, cpu_baseline and e2e keys the driver reads (run here at --log2d 16 so it takes seconds; the
driver's default is the full workload H).  Also the host logic that counts the rounds k_round runs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--log2d", "16"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_kround_round_accounting():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.kround_rounds(1 << 26) == list(range(2, 10))     # 2^26 >> 9 = 2^17: rounds 10.. are chunked
    assert bench.kround_rounds(1 << 18) == []                       # the chunked rounds start at round 2
    assert bench.kround_rounds(1 << 30) == list(range(2, 14))
