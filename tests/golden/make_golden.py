"""Generate golden vectors by running the REFERENCE package (hecnn) here.

Run in the build container only (needs /root/reference, which does not exist
on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/s128.npz   full arrays for the small ring "S128"
                          (m=256 -> N=128, L=260, r=30, BASE_EXTRA_BITS=25)
  tests/golden/golden.json chain constants, SHA-256 digests of ciphertext
                          payloads for the BASELINE configs, decrypted values,
                          level/scale traces, mini-CNN logits.

Everything here is produced by the reference's own code path
(`hecnn.backends.ckks.CkksBackend`, `hecnn.backends.kernels`), driven through
its public API; the mini-CNN op sequences are composed from those API calls by
`paper_2102_00319_b200.percell` (which only calls public HEBackend ops).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import warnings
from fractions import Fraction

import numpy as np

warnings.simplefilter("ignore")
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from hecnn.backends import chain as ref_chain  # noqa: E402
from hecnn.backends import kernels as ref_kernels  # noqa: E402
from hecnn.backends.ckks import CkksBackend  # noqa: E402
from hecnn.backends.encoding import coeffs_from_slots, slots_from_coeffs  # noqa: E402
from hecnn.params import derive_params  # noqa: E402
from hecnn.model import random_model, encrypt_model  # noqa: E402
from hecnn.packing import ImageBatch, pack_batch  # noqa: E402
from hecnn.executor import run_inference  # noqa: E402

from paper_2102_00319_b200 import percell  # noqa: E402
from paper_2102_00319_b200.model import Conv, Dense, Flatten, Network, PolyAct, SumPool, Square  # noqa: E402
from paper_2102_00319_b200.configs import CONFIGS  # noqa: E402
sys.path.insert(0, os.path.join(REPO, "tests"))
from nets import mini_networks  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def ct_digest(ct) -> str:
    return digest(np.concatenate([ct.payload.c0, ct.payload.c1]))


def make_backend(m, L, r, seed, extra):
    ref_chain.BASE_EXTRA_BITS = extra
    ref_chain._build_chain_cached.cache_clear()
    be = CkksBackend(derive_params(m, L, r, seed=seed))
    return be


def ref_rotate(be, ct, steps: int):
    """Rotation built ONLY from the reference's own machinery (SURVEY.md §8c rotation
    oracle): a Galois key generated exactly like keygen's evk loop (ckks.py:151-176)
    with s^2 replaced by s(X^g) and the sampler tagged (seed, 5, g), the automorphism
    applied in the coefficient domain with the reference NTT kernels, and the key
    switch done by relin_accumulate + moddown_special (ckks.py:359-387) without the
    rescale.  Returns (galois key b digest, c0, c1)."""
    ch, n = be.chain, be.n
    g = pow(5, steps % (n // 2), 2 * n)
    s = be._sample_ternary(be._rng(1))  # keygen's secret
    t = np.zeros(n, dtype=np.int64)
    for i in range(n):
        j = (i * g) % (2 * n)
        if j < n:
            t[j] += s[i]
        else:
            t[j - n] -= s[i]
    s_eval = be._coeffs_to_all_rows(s)
    target = be._coeffs_to_all_rows(t)
    rows_all, digits = ch.num_rows, ch.num_rows - 1
    rng = be._rng(5, g)
    gk_a = np.empty((digits, rows_all, n), dtype=np.uint64)
    gk_b = np.empty_like(gk_a)
    for j in range(digits):
        gk_a[j] = be._sample_uniform_rows(rng, rows_all)
        e_j = be._coeffs_to_all_rows(be._sample_gaussian(rng))
        bj = gk_b[j]
        ref_kernels.mul_rows(gk_a[j], s_eval, ch.p, ch.p_inv, bj)
        ref_kernels.neg_rows(bj, ch.p, bj)
        ref_kernels.add_rows(bj, e_j, ch.p, bj)
        q_j = int(ch.p[j])
        factor = (ch.special_prime % q_j) * ((1 << 64) % q_j) % q_j
        term = np.empty((1, n), dtype=np.uint64)
        ref_kernels.scalar_mul_rows(target[j:j + 1], np.array([factor], dtype=np.uint64), ch.p[j:j + 1],
                                    ch.p_inv[j:j + 1], term)
        ref_kernels.add_rows(bj[j:j + 1], term, ch.p[j:j + 1], bj[j:j + 1])
    k = ct.level + 1

    def sigma(rows):
        c = rows.copy()
        ref_kernels.ntt_inv_rows(c, ch.twiddles[:k], ch.n_inv[:k], ch.p[:k], ch.p_inv[:k])
        out = np.zeros_like(c)
        for i in range(n):
            j = (i * g) % (2 * n)
            if j < n:
                out[:, j] = c[:, i]
            else:
                out[:, j - n] = np.where(c[:, i] == 0, 0, ch.p[:k] - c[:, i])
        ref_kernels.ntt_fwd_rows(out, ch.twiddles[:k], ch.p[:k], ch.p_inv[:k])
        return out

    c0r, c1r = sigma(ct.payload.c0), sigma(ct.payload.c1)
    d2_coeff = c1r.copy()
    ref_kernels.ntt_inv_rows(d2_coeff, ch.twiddles[:k], ch.n_inv[:k], ch.p[:k], ch.p_inv[:k])
    ref_kernels.from_mont_rows(d2_coeff, ch.p[:k], ch.p_inv[:k])
    d2_cent = np.empty((k, n), dtype=np.int64)
    ref_kernels.centered_rows(d2_coeff, ch.p[:k], d2_cent)
    acc0 = np.zeros((k + 1, n), dtype=np.uint64)
    acc1 = np.zeros_like(acc0)
    sp = ch.special_row
    ref_kernels.relin_accumulate(c1r, d2_cent, gk_b, gk_a, sp, ch.twiddles, ch.p, ch.p_inv, ch.r2, acc0, acc1)
    rel0 = np.empty((k, n), dtype=np.uint64)
    rel1 = np.empty_like(rel0)
    sp_inv = be._special_inv[ct.level]
    ref_kernels.moddown_special(acc0, sp, ch.twiddles, ch.n_inv, ch.p, ch.p_inv, ch.r2, sp_inv, rel0)
    ref_kernels.moddown_special(acc1, sp, ch.twiddles, ch.n_inv, ch.p, ch.p_inv, ch.r2, sp_inv, rel1)
    ref_kernels.add_rows(rel0, c0r, ch.p[:k], rel0)
    return digest(gk_b), rel0, rel1


def frac(x: Fraction) -> str:
    return f"{x.numerator}/{x.denominator}"


def small_ring(golden: dict) -> dict:
    arrays: dict[str, np.ndarray] = {}
    be = make_backend(256, 260, 30, 42, 25)
    ch = be.chain
    n = be.n
    arrays.update(p=ch.p, p_inv=ch.p_inv, r2=ch.r2, n_inv=ch.n_inv, twiddles=ch.twiddles)

    # kernels: NTT pairs per prime
    rng = np.random.default_rng(5)
    f = np.stack([rng.integers(0, int(q), n, dtype=np.uint64) for q in ch.p])
    g = f.copy()
    ref_kernels.ntt_fwd_rows(g, ch.twiddles, ch.p, ch.p_inv)
    h = f.copy()
    ref_kernels.ntt_inv_rows(h, ch.twiddles, ch.n_inv, ch.p, ch.p_inv)
    arrays.update(ntt_in=f, ntt_fwd=g, ntt_inv=h)

    # encoding
    vals = rng.uniform(-1, 1, be.slots)
    arrays["enc_values"] = vals
    arrays["enc_coeffs"] = be._encode_coeffs(vals, be.canonical_scale, be.fresh_level)
    arrays["dec_slots"] = slots_from_coeffs(arrays["enc_coeffs"].astype(np.float64), float(be.canonical_scale), n)

    # keys
    keys = be.keygen()
    be.set_eval_key(keys)
    arrays.update(s_eval=keys.secret.s_eval, pk_b=keys.public.b, pk_a=keys.public.a,
                  evk_b=keys.evaluation.b, evk_a=keys.evaluation.a)

    va = rng.uniform(-1, 1, be.slots)
    vb = rng.uniform(-1, 1, be.slots)
    arrays.update(va=va, vb=vb)
    a = be.encrypt(va, keys, entropy=1)
    b = be.encrypt(vb, keys, entropy=2)
    put = lambda name, ct: arrays.update({f"{name}_c0": ct.payload.c0, f"{name}_c1": ct.payload.c1})  # noqa: E731
    put("a", a)
    put("b", b)
    raw = be.mul_ct_ct_raw(a, b)
    arrays.update(raw_d0=raw.payload.d0, raw_d1=raw.payload.d1, raw_d2=raw.payload.d2)
    raw2 = be.raw_add(raw, be.mul_ct_ct_raw(a, a))
    fin = be.raw_finalize(raw2)
    put("fin", fin)
    arrays["fin_dec"] = be.decrypt(fin, keys).values
    pt = be.encode_plain(vb, level=a.level)
    arrays["pt_rows"] = pt.payload.rows
    ctpt = be.mul_ct_pt(a, pt)
    put("ctpt", ctpt)
    put("add", be.add_ct_ct(a, b))
    put("addpt", be.add_ct_pt(a, vb))
    # rescale of a random component at every level
    for lvl in range(1, be.fresh_level + 1):
        comp = np.stack([rng.integers(0, int(q), n, dtype=np.uint64) for q in ch.p[: lvl + 1]])
        arrays[f"resc_in_{lvl}"] = comp
        arrays[f"resc_out_{lvl}"] = be._rescale_comp(comp, lvl)
    # squaring chain down to level 0 (depth boundary)
    ct = be.encrypt(np.full(be.slots, 1.01), keys, entropy=3)
    trace = []
    for step in range(be.fresh_level):
        ct = be.mul_ct_ct(ct, ct)
        put(f"sq{step}", ct)
        trace.append({"level": ct.level, "scale": frac(ct.scale), "noise": ct.noise_bits})
    # drop + aligned multiply
    a3 = be.drop_to_level(a, 3)
    put("drop_mul", be.mul_ct_ct(a3, b))
    # serialization: coefficient-form payloads, a full ciphertext envelope, key payloads
    from hecnn import serialization as ref_ser
    for name, ct in (("a", a), ("fin", fin), ("a3", a3)):
        arrays[f"payload_{name}"] = np.frombuffer(be.cipher_payload_bytes(ct), dtype=np.uint8)
    arrays["record_fin"] = np.frombuffer(ref_ser.cipher_record(be, fin), dtype=np.uint8)
    arrays["envelope_fin"] = np.frombuffer(ref_ser.wrap(ref_ser.KIND_CIPHER, be, ref_ser.cipher_record(be, fin)),
                                           dtype=np.uint8)
    # rotation pinned on the reference's own kernels (no reference API exists for it)
    rot_meta = {}
    for steps in (1, 3):
        gdig, r0, r1 = ref_rotate(be, a, steps)
        arrays[f"rot{steps}_c0"], arrays[f"rot{steps}_c1"] = r0, r1
        rot_meta[str(steps)] = {"galois_key_b": gdig, "level": a.level}
    golden_rot = rot_meta
    kp = be.key_payload_bytes(keys)
    key_digests = {role: hashlib.sha256(data).hexdigest() for role, data in kp.items()}
    golden["s128"] = {
        "m": 256, "L": 260, "r": 30, "seed": 42, "extra": 25,
        "square_trace": trace,
        "fin": {"level": fin.level, "scale": frac(fin.scale), "noise": fin.noise_bits},
        "ctpt": {"level": ctpt.level, "scale": frac(ctpt.scale), "noise": ctpt.noise_bits},
        "counters": be.counters.snapshot().__dict__,
        "key_payload_sha256": key_digests,
        "rotation": golden_rot,
        "payload_meta": {"a": [a.level, frac(a.scale), a.noise_bits], "fin": [fin.level, frac(fin.scale), fin.noise_bits],
                         "a3": [a3.level, frac(a3.scale), a3.noise_bits]},
    }

    # mini CNNs composed from reference API calls
    minis = {}
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))
    for name, net in mini_networks().items():
        be.counters.reset()
        enc = percell.encrypt_network(be, net, keys)
        x = imgs[:, : net.input_dims[0], : net.input_dims[1]]
        grid = percell.encrypt_images(be, x, keys)
        logits = percell.run_network(be, enc, grid)
        dec = np.stack([be.decrypt(c, keys).values for c in logits], axis=1)
        minis[name] = {
            "logit_digests": [ct_digest(c) for c in logits],
            "level": logits[0].level,
            "scale": frac(logits[0].scale),
            "decrypted_first8": dec[:8].tolist(),
            "counters": be.counters.snapshot().__dict__,
        }
        arrays[f"{name}_logits_c0"] = np.stack([c.payload.c0 for c in logits])
        arrays[f"{name}_logits_c1"] = np.stack([c.payload.c1 for c in logits])
    golden["minis"] = minis

    # the reference's own canonical pipeline (run_inference) on a tiny model
    be2 = make_backend(256, 260, 30, 42, 25)
    keys2 = be2.keygen()
    be2.set_eval_key(keys2)
    model = random_model(input_dims=(8, 8), filters=2, kernel=(3, 3), classes=3, seed=5, conv_bias=True)
    enc_model = encrypt_model(be2, model, keys2)
    batch = ImageBatch(np.random.default_rng(1).uniform(0, 1, (5, 8, 8)))
    cm = pack_batch(be2, batch, keys2)
    res = run_inference(be2, enc_model, cm)
    golden["canonical_tiny"] = {
        "logit_digests": [ct_digest(c) for c in res.logits],
        "decrypted": [be2.decrypt(c, keys2).values[:5].tolist() for c in res.logits],
        "level": res.logits[0].level,
        "scale": frac(res.logits[0].scale),
    }
    return arrays


def baseline_configs(golden: dict) -> None:
    out = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        cfg = CONFIGS[name]
        ref_chain.BASE_EXTRA_BITS = cfg.base_extra_bits
        ref_chain._build_chain_cached.cache_clear()
        ch = ref_chain.build_chain(cfg.params())
        out[name] = {
            "primes": [int(x) for x in ch.p],
            "p_inv": [int(x) for x in ch.p_inv],
            "r2": [int(x) for x in ch.r2],
            "n_inv": [int(x) for x in ch.n_inv],
            "twiddle_digest": digest(ch.twiddles),
            "num_levels": ch.num_levels,
        }
    golden["chains"] = out

    # config 1 op digests
    cfg = CONFIGS["cfg1"]
    be = make_backend(cfg.m, cfg.modulus_bits, cfg.precision_bits, cfg.key_seed, cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    rng = np.random.default_rng(101)
    xs = rng.uniform(-1, 1, (4, be.slots))
    ys = rng.uniform(-1, 1, (4, be.slots))
    rec = {
        "s_eval": digest(keys.secret.s_eval),
        "pk": digest(np.concatenate([keys.public.b, keys.public.a])),
        "evk": digest(np.concatenate([keys.evaluation.b.ravel(), keys.evaluation.a.ravel()])),
        "ops": [],
    }
    for i in range(2):
        x = be.encrypt(xs[i], keys, entropy=i)
        y = be.encrypt(ys[i], keys, entropy=256 + i)
        mul = be.mul_ct_ct(x, y)
        ctpt = be.mul_ct_pt(x, be.encode_plain(ys[i], level=x.level))
        add = be.add_ct_ct(x, y)
        rec["ops"].append({
            "x": ct_digest(x), "y": ct_digest(y), "mul": ct_digest(mul),
            "ctpt": ct_digest(ctpt), "add": ct_digest(add),
            "mul_payload": hashlib.sha256(be.cipher_payload_bytes(mul)).hexdigest(),
            "mul_dec8": be.decrypt(mul, keys).values[:8].tolist(),
            "mul_scale": frac(mul.scale),
        })
    golden["cfg1_ops"] = rec


def main() -> None:
    golden: dict = {}
    arrays = small_ring(golden)
    baseline_configs(golden)
    np.savez_compressed(os.path.join(OUT, "s128.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "s128.npz"), os.path.getsize(os.path.join(OUT, "s128.npz")))


if __name__ == "__main__":
    main()
