"""The reference's OWN pipeline, reproduced bit for bit.

`tests/golden/make_canonical.py` ran the reference's `run_inference`
(`/root/reference/pkg/src/hecnn/executor.py:161-279`) on its canonical topology --
conv (stride 1, bias) -> act_pool (`layers.py:207-216`: the degree-2 activation with the
1/4 mean-pool divisor folded into its coefficients, then the WINDOW_ORDER sum) ->
flatten -> dense (+bias) -- and stored every input ciphertext it encrypted (`pack_batch`,
`encrypt_model`, in the reference's own encryption order) and the logits it returned.
Here the same inputs go through

* the CPU oracle, in the reference op order (`percell.run_network`)       [CPU]
* the batched device layer evaluator (`LayerEvaluator.run`, heb_conv /
  heb_poly_act / heb_sumpool / heb_fc)                                     [gpu]
* the device per-op backend (`percell.run_network` on `B200Backend`)        [gpu]

and the logit ciphertexts must equal the reference's (SHA-256 of the residues), the
level / exact scale must match, and the op counters must equal `run_inference`'s.

`fullsize_ops` pins single ops at the BASELINE ring sizes (N = 8192, 16384, 32768)
to reference-generated digests: keys, encrypt, mul_ct_ct, mul_ct_pt, add_ct_ct and a
second-level mul_ct_ct.
"""

import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN_DIR


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def frac(s):
    a, b = s.split("/")
    return Fraction(int(a), int(b))


@pytest.fixture(scope="module")
def canon():
    with open(os.path.join(GOLDEN_DIR, "canonical_tiny.json")) as fh:
        g = json.load(fh)
    return g, dict(np.load(os.path.join(GOLDEN_DIR, "canonical_tiny.npz")))


def canonical_net(g, arr):
    """The reference's random_model topology in this package's layer vocabulary."""
    from paper_2102_00319_b200.model import Conv, Dense, Flatten, Network, PolyAct, SumPool

    a0, a1, a2, s, d = g["canonical_tiny"]["act"]
    conv = Conv(weights=arr["conv_weights"][:, None], stride=1, bias=arr["conv_bias"])
    dense = Dense(weights=arr["dense_weights"], bias=arr["dense_bias"])
    return Network((8, 8), (conv, PolyAct(a0=a0, a1=a1, a2=a2, input_scale=s, pool_divisor=d), SumPool(), Flatten(),
                            dense))


def params(g):
    from paper_2102_00319_b200.params import derive_params

    m, L, r, seed, extra = g["canonical_tiny"]["params"]
    return derive_params(m, L, r, seed=seed), extra


def per_ct_inputs(be, g, arr, make):
    """(EncryptedNetwork, input maps) of per-ciphertext objects built by make(c0, c1, meta)."""
    from paper_2102_00319_b200 import percell
    from paper_2102_00319_b200.model import ledger

    net = canonical_net(g, arr)
    meta = g["canonical_tiny"]["meta"]

    def cts(key, m):
        return [make(x[0], x[1], m) for x in arr[key]]

    conv_w = np.array(cts("conv_w_cts", meta["conv_w"]), dtype=object).reshape(2, 1, 3, 3)
    dense_w = np.array(cts("dense_w_cts", meta["dense_w"]), dtype=object).reshape(arr["dense_weights"].shape)
    enc = percell.EncryptedNetwork(net=net, weights=[conv_w, None, None, None, dense_w],
                                   biases=[cts("conv_b_cts", meta["conv_b"]), None, None, None,
                                           cts("dense_b_cts", meta["dense_b"])],
                                   trace=ledger(net, be.chain, be.canonical_scale))
    cells = cts("in_cts", meta["in"])
    grid = [[cells[i * 8 + j] for j in range(8)] for i in range(8)]
    return enc, [grid]


def check_logits(g, arr, rows, level, scale):
    want = g["canonical_tiny"]
    assert [digest(np.concatenate([c0, c1])) for c0, c1 in rows] == want["logit_digests"]
    assert np.array_equal(np.stack([np.stack(r) for r in rows]), arr["logits"])
    lv, sc, _ = want["meta"]["logits"]
    assert level == lv and scale == frac(sc)


def test_oracle_reproduces_reference_run_inference(canon):
    from oracle.ckks_oracle import OracleBackend, _Cipher
    from paper_2102_00319_b200 import percell

    g, arr = canon
    p, extra = params(g)
    be = OracleBackend(p, extra)
    keys = be.keygen()
    be.set_eval_key(keys)
    enc, maps = per_ct_inputs(be, g, arr, lambda c0, c1, m: be._cipher(_Cipher(c0.copy(), c1.copy()), m[0],
                                                                       frac(m[1]), m[2]))
    be.counters.reset()
    logits = percell.run_network(be, enc, maps)
    check_logits(g, arr, [(c.payload.c0, c.payload.c1) for c in logits], logits[0].level, logits[0].scale)
    assert be.counters.snapshot().__dict__ == g["canonical_tiny"]["counters"]
    got = [be.decrypt(c, keys).values[:5] for c in logits]
    assert np.allclose(got, g["canonical_tiny"]["decrypted"], atol=1e-9, rtol=0)


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_oracle_fullsize_ops_match_reference(name):
    """Reference-generated digests at the BASELINE ring sizes pin the oracle at full N."""
    from oracle.ckks_oracle import OracleBackend
    from paper_2102_00319_b200.configs import CONFIGS

    with open(os.path.join(GOLDEN_DIR, "canonical_tiny.json")) as fh:
        want = json.load(fh)["fullsize_ops"][name]
    cfg = CONFIGS[name]
    be = OracleBackend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    assert digest(keys.secret.s_eval) == want["s_eval"]
    assert digest(np.concatenate([keys.public.pk_b, keys.public.pk_a])) == want["pk"]
    assert digest(np.concatenate([keys.evaluation.evk_b.ravel(), keys.evaluation.evk_a.ravel()])) == want["evk"]
    rng = np.random.default_rng(501)
    x, y = rng.uniform(-1, 1, (2, be.slots))
    a, b = be.encrypt(x, keys, entropy=7), be.encrypt(y, keys, entropy=8)

    def d(ct):
        return digest(np.concatenate([ct.payload.c0, ct.payload.c1]))

    mul = be.mul_ct_ct(a, b)
    assert (d(a), d(b), d(mul)) == (want["a"], want["b"], want["mul"])
    assert d(be.mul_ct_pt(a, be.encode_plain(y, level=a.level))) == want["ctpt"]
    assert d(be.add_ct_ct(a, b)) == want["add"]
    assert d(be.mul_ct_ct(mul, mul)) == want["mul2"]


@pytest.mark.gpu
def test_device_layers_reproduce_reference_run_inference(canon):
    """The batched device evaluator fed the reference's exact input ciphertexts."""
    import torch

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend, CipherBatch
    from paper_2102_00319_b200.model import ledger

    g, arr = canon
    p, extra = params(g)
    be = B200Backend(p, extra)
    keys = be.keygen()
    be.set_eval_key(keys)
    meta = g["canonical_tiny"]["meta"]
    net = canonical_net(g, arr)

    def batch(key, m):
        a = arr[key]
        buf = torch.from_numpy(a.view(np.int64).copy()).to(be.dev)
        return CipherBatch(buf, m[0], frac(m[1]), m[2])

    enc = layers.EncryptedNetworkBatch(
        net, [batch("conv_w_cts", meta["conv_w"]), None, None, None, batch("dense_w_cts", meta["dense_w"])],
        [batch("conv_b_cts", meta["conv_b"]), None, None, None, batch("dense_b_cts", meta["dense_b"])],
        ledger(net, be.chain, be.canonical_scale))
    x = batch("in_cts", meta["in"])
    be.counters.reset()
    out = layers.LayerEvaluator(be).run(enc, x)
    rows = out.buf[:, :, : out.k].cpu().numpy().view(np.uint64)
    check_logits(g, arr, [(r[0], r[1]) for r in rows], out.level, out.scale)
    assert be.counters.snapshot().__dict__ == g["canonical_tiny"]["counters"]
    dec = be.decrypt_batch(out, keys)[:, :5]
    assert np.allclose(dec, g["canonical_tiny"]["decrypted"], atol=1e-9, rtol=0)


@pytest.mark.gpu
def test_device_per_op_reproduces_reference_run_inference(canon):
    """The per-op device backend driven in the reference op order (percell)."""
    from paper_2102_00319_b200 import percell
    from paper_2102_00319_b200.backend import B200Backend

    g, arr = canon
    p, extra = params(g)
    be = B200Backend(p, extra)
    keys = be.keygen()
    be.set_eval_key(keys)
    enc, maps = per_ct_inputs(be, g, arr, lambda c0, c1, m: be.cipher_from_host(c0, c1, m[0], frac(m[1]), m[2]))
    logits = percell.run_network(be, enc, maps)
    check_logits(g, arr, [be.cipher_rows_host(c) for c in logits], logits[0].level, logits[0].scale)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_device_fullsize_ops_match_reference(name):
    """Device keys and ops at the BASELINE ring sizes equal the reference's digests."""
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS

    with open(os.path.join(GOLDEN_DIR, "canonical_tiny.json")) as fh:
        want = json.load(fh)["fullsize_ops"][name]
    cfg = CONFIGS[name]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    host = lambda t: t.cpu().numpy().view(np.uint64)  # noqa: E731
    assert digest(host(keys.secret.s_eval)) == want["s_eval"]
    rng = np.random.default_rng(501)
    x, y = rng.uniform(-1, 1, (2, be.slots))
    a, b = be.encrypt(x, keys, entropy=7), be.encrypt(y, keys, entropy=8)

    def d(ct):
        c0, c1 = be.cipher_rows_host(ct)
        return digest(np.concatenate([c0, c1]))

    mul = be.mul_ct_ct(a, b)
    assert (d(a), d(b), d(mul)) == (want["a"], want["b"], want["mul"])
    assert d(be.mul_ct_pt(a, be.encode_plain(y, level=a.level))) == want["ctpt"]
    assert d(be.add_ct_ct(a, b)) == want["add"]
    assert d(be.mul_ct_ct(mul, mul)) == want["mul2"]
    assert np.allclose(be.decrypt(mul, keys).values[:8], want["mul_dec8"], atol=1e-12, rtol=0)
