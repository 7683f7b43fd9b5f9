"""bench.py --impl reference on the batch config (C4) runs on CPU only: its line carries the
batch metric (problem-iterations/s, the unit of our C4 arm) from a process pool over the
oracle port, as the reference batches (bench.py:96-106 of the reference)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_batch_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c4", "--cpu-budget", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "problem-iterations/s"
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cpu = line["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["cores"] == (os.cpu_count() or 1) and cpu["value"] == line["value"]
    assert line["config"]["problems"] == 4096
