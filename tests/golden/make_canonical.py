"""Golden vectors from the REFERENCE's own pipeline and from BASELINE-size ops.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_canonical.py

Outputs (committed):
  tests/golden/canonical_tiny.npz   the reference's `run_inference`
      (`/root/reference/pkg/src/hecnn/executor.py:161-279`) on
      `random_model(input_dims=(8, 8), filters=2, kernel=(3, 3), classes=3, seed=5,
      conv_bias=True)` (conv stride 1 + bias -> act_pool (poly activation with the 1/4
      pool divisor folded, `layers.py:207-216`) -> flatten -> dense + bias) over a
      5-image batch at N = 128: every INPUT ciphertext (the packed batch of
      `pack_batch`, the encrypted model of `encrypt_model`, in the reference's own
      encryption order) and the plaintext weights, so the device evaluator can be fed
      the reference's exact inputs; plus the logit ciphertexts `run_inference` returned.
  tests/golden/canonical_tiny.json  levels, exact scales, noise bits and digests of
      the above, the op counters, and `fullsize_ops`: reference keys and op digests at
      the BASELINE ring sizes (cfg2 N = 8192, cfg3 N = 16384, cfg4 N = 32768):
      encrypt, mul_ct_ct (tensor + relinearise + rescale), mul_ct_pt, add_ct_ct and a
      second-level mul_ct_ct, each a SHA-256 digest of the (c0, c1) residues.

Everything comes from the reference's code path (`hecnn.backends.ckks.CkksBackend`,
`hecnn.model.encrypt_model`, `hecnn.packing.pack_batch`, `hecnn.executor.run_inference`).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
import warnings
from fractions import Fraction

import numpy as np

warnings.simplefilter("ignore")
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from hecnn.backends import chain as ref_chain  # noqa: E402
from hecnn.backends.ckks import CkksBackend  # noqa: E402
from hecnn.executor import ThreadPlan, run_inference  # noqa: E402
from hecnn.model import encrypt_model, random_model  # noqa: E402
from hecnn.packing import ImageBatch, pack_batch  # noqa: E402
from hecnn.params import derive_params  # noqa: E402

from paper_2102_00319_b200.configs import CONFIGS  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def ct_digest(ct) -> str:
    return digest(np.concatenate([ct.payload.c0, ct.payload.c1]))


def frac(x: Fraction) -> str:
    return f"{x.numerator}/{x.denominator}"


def make_backend(m, L, r, seed, extra):
    ref_chain.BASE_EXTRA_BITS = extra
    ref_chain._build_chain_cached.cache_clear()
    return CkksBackend(derive_params(m, L, r, seed=seed))


def stack(cts):
    return np.stack([np.stack([c.payload.c0, c.payload.c1]) for c in cts])


def meta(ct):
    return [ct.level, frac(ct.scale), ct.noise_bits]


def canonical_tiny(golden: dict, arrays: dict) -> None:
    be = make_backend(256, 260, 30, 42, 25)
    keys = be.keygen()
    be.set_eval_key(keys)
    model = random_model(input_dims=(8, 8), filters=2, kernel=(3, 3), classes=3, seed=5, conv_bias=True)
    enc = encrypt_model(be, model, keys)
    batch = ImageBatch(np.random.default_rng(1).uniform(0, 1, (5, 8, 8)))
    cm = pack_batch(be, batch, keys)
    be.counters.reset()
    res = run_inference(be, enc, cm, ThreadPlan(1, 1, 1, 1))
    conv, dense = model.layers[0], model.layers[3]
    act = model.layers[1].act
    cells = [c for row in cm.grid for c in row]
    wconv = [enc.conv_kernels[f].grid[p][q] for f in range(conv.filters) for p in range(3) for q in range(3)]
    bconv = [enc.conv_kernels[f].bias for f in range(conv.filters)]
    wdense = [enc.dense_weights[i][r] for i in range(dense.in_dim) for r in range(dense.out_dim)]
    arrays.update({
        "images": batch.images,
        "conv_weights": conv.weights, "conv_bias": conv.bias,
        "dense_weights": dense.weights, "dense_bias": dense.bias,
        "in_cts": stack(cells), "conv_w_cts": stack(wconv), "conv_b_cts": stack(bconv),
        "dense_w_cts": stack(wdense), "dense_b_cts": stack(enc.dense_bias),
        "logits": stack(res.logits),
    })
    golden["canonical_tiny"] = {
        "params": [256, 260, 30, 42, 25],
        "act": [act.a0, act.a1, act.a2, act.input_scale, 4.0],
        "meta": {"in": meta(cells[0]), "conv_w": meta(wconv[0]), "conv_b": meta(bconv[0]),
                 "dense_w": meta(wdense[0]), "dense_b": meta(enc.dense_bias[0]), "logits": meta(res.logits[0])},
        "logit_digests": [ct_digest(c) for c in res.logits],
        "decrypted": [be.decrypt(c, keys).values[:5].tolist() for c in res.logits],
        "counters": be.counters.snapshot().__dict__,
    }


def fullsize_ops(golden: dict) -> None:
    out = {}
    for name in ("cfg2", "cfg3", "cfg4"):
        cfg = CONFIGS[name]
        t0 = time.time()
        be = make_backend(cfg.m, cfg.modulus_bits, cfg.precision_bits, cfg.key_seed, cfg.base_extra_bits)
        keys = be.keygen()
        be.set_eval_key(keys)
        rng = np.random.default_rng(501)
        x, y = rng.uniform(-1, 1, (2, be.slots))
        a = be.encrypt(x, keys, entropy=7)
        b = be.encrypt(y, keys, entropy=8)
        mul = be.mul_ct_ct(a, b)
        rec = {
            "s_eval": digest(keys.secret.s_eval),
            "pk": digest(np.concatenate([keys.public.b, keys.public.a])),
            "evk": digest(np.concatenate([keys.evaluation.b.ravel(), keys.evaluation.a.ravel()])),
            "a": ct_digest(a), "b": ct_digest(b), "mul": ct_digest(mul),
            "ctpt": ct_digest(be.mul_ct_pt(a, be.encode_plain(y, level=a.level))),
            "add": ct_digest(be.add_ct_ct(a, b)),
            "mul2": ct_digest(be.mul_ct_ct(mul, mul)),
            "mul_meta": meta(mul),
            "mul_dec8": be.decrypt(mul, keys).values[:8].tolist(),
        }
        out[name] = rec
        print(name, "done in", round(time.time() - t0, 1), "s")
    golden["fullsize_ops"] = out


def main() -> None:
    golden: dict = {}
    arrays: dict = {}
    canonical_tiny(golden, arrays)
    fullsize_ops(golden)
    np.savez_compressed(os.path.join(OUT, "canonical_tiny.npz"), **arrays)
    with open(os.path.join(OUT, "canonical_tiny.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "canonical_tiny.npz"))


if __name__ == "__main__":
    main()
