"""bench.py's reference arm runs on the CPU (the oracle port of the reference kernels)
and prints the driver's JSON contract: one line with impl, metric, unit, cpu_baseline
and e2e keys.  The B200 arm itself needs a GPU (covered by the gpu-marked tests)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

sys.path.insert(0, REPO)


def test_reference_arm_prints_contract_line():
    env = dict(os.environ, PYTHONPATH=REPO)
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "cfg2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=REPO,
                         env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "images/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("encrypted-CNN images/sec")
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1
    # cfg2: the sample is the whole batch, so ms_per_step is a whole batch's wall time
    assert d["config"]["images_per_step"] == d["config"]["batch_per_gpu"] == 4096
    assert abs(d["value"] - 4096 / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-3
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.parametrize("config,shards", [("cfg2", 1), ("cfg3", 5), ("cfg4", 10)])
def test_reference_sample_is_exactly_proportional(config, shards):
    """Every layer's sampled unit count is exactly 1/S of the layer (no extrapolation)."""
    import bench
    from paper_2102_00319_b200.configs import NETWORKS

    assert bench.CpuSample.SHARDS[config] == shards
    plan = bench.CpuSample.sample_plan(NETWORKS[config](), shards)
    assert all(cnt * shards == tot for _, _, cnt, tot in plan)
    kinds = [k for k, *_ in plan]
    if config == "cfg4":
        assert kinds == ["conv", "square", "conv", "square", "sumpool", "dense"]
        assert [t for *_, t in plan] == [720, 720, 1000, 1000, 250, 10]
    with pytest.raises(ValueError):
        bench.CpuSample.sample_plan(NETWORKS["cfg4"](), 20)  # 250 pool windows, 10 outputs: not divisible
