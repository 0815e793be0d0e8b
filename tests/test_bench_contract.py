"""bench.py's reference arm runs on the CPU (the oracle port of the reference kernels)
and prints the driver's JSON contract: one line with impl, metric, unit, cpu_baseline
and e2e keys.  The B200 arm itself needs a GPU (covered by the gpu-marked tests)."""

import json
import os
import subprocess
import sys

from conftest import REPO


def test_reference_arm_prints_contract_line():
    env = dict(os.environ, PYTHONPATH=REPO)
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=REPO, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "images/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("encrypted-CNN images/sec")
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
