"""The library's run-time switches must not change a single bit.

libheb200 reads its switches once per process (two-pass ModUp, FP64 engine off, ModUp
target-set size, side streams, conv CTA width, conv split-limb body off), so every setting
runs in its own subprocess: a seeded ct x ct multiply + relinearise + rescale, a rotation and
a batched conv layer at N = 1024, 8192 and 32768 (two levels) are hashed, and every switch must reproduce the default build's digests --
which `test_gpu_parity.py` / `test_gpu_invariants.py` pin to the oracle.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

SCRIPT = r"""
import hashlib, json, sys, warnings
import numpy as np
warnings.simplefilter("ignore")
sys.path.insert(0, %(repo)r)
from paper_2102_00319_b200.backend import B200Backend
from paper_2102_00319_b200.params import derive_params
from paper_2102_00319_b200 import layers
from paper_2102_00319_b200.model import Conv
out = {}
for m in (1 << 11, 1 << 14, 1 << 16):
    dev = B200Backend(derive_params(m, 180, 40, seed=3), 20)
    keys = dev.keygen(galois_steps=(1,))
    dev.set_eval_key(keys)
    rng = np.random.default_rng(m)
    x, y = rng.uniform(-1, 1, (2, dev.slots))
    a, b = dev.encrypt(x, keys, entropy=1), dev.encrypt(y, keys, entropy=2)
    h = hashlib.sha256()
    for ct in (dev.mul_ct_ct(a, b), dev.rotate(a, 1), dev.mul_ct_ct(dev.mul_ct_ct(a, b), dev.mul_ct_ct(b, b))):
        c0, c1 = dev.cipher_rows_host(ct)
        h.update(np.ascontiguousarray(c0).tobytes())
        h.update(np.ascontiguousarray(c1).tobytes())
    # a batched conv layer (2 filters 3x3 over a 4x4 grid): heb_conv_tensor + relinearise + rescale
    imgs = rng.uniform(0, 1, (dev.slots, 4, 4))
    wts = rng.normal(0, 0.3, (2, 1, 3, 3))
    xb = layers.encrypt_images(dev, imgs, keys)
    wb = dev.encrypt_batch(np.repeat(wts.ravel()[:, None], dev.slots, 1), keys, 1000 + np.arange(wts.size))
    yc, _ = layers.LayerEvaluator(dev).conv(xb, (1, 4, 4), Conv(weights=wts, stride=1), wb, None)
    h.update(yc.buf[:, :, : yc.k].cpu().numpy().tobytes())
    out[str(m)] = h.hexdigest()
print("DIGESTS " + json.dumps(out))
"""

SWITCHES = [
    {"HEB_MODUP_SPLIT": "1"},
    {"HEB_DISABLE_FP64_NTT": "1"},
    {"HEB_MODUP_TS": "1"},
    {"HEB_MODUP_TS": "99"},
    {"HEB_MODUP_CONCURRENT": "0", "HEB_MODDOWN_CONCURRENT": "0"},
    {"HEB_CONV_NARROW": "0"},
    {"HEB_CONV_NARROW": "1"},
    {"HEB_CONV_NO_LIMBS": "1"},
]


def digests(env):
    res = subprocess.run([sys.executable, "-c", SCRIPT % {"repo": REPO}], env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=900)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("DIGESTS ")]
    assert res.returncode == 0 and lines, res.stderr[-3000:]
    return json.loads(lines[-1][8:])


@pytest.fixture(scope="module")
def default_digests():
    return digests({})


@pytest.mark.gpu
@pytest.mark.parametrize("switch", SWITCHES, ids=lambda s: ",".join(f"{k}={v}" for k, v in s.items()))
def test_switch_is_bit_identical_to_default(switch, default_digests):
    assert digests(switch) == default_digests
