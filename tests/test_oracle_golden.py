"""Pin the CPU oracle and the product's host logic to the reference's golden vectors.

The fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py).  Nothing here needs a GPU.
"""

import hashlib
from fractions import Fraction

import numpy as np
import pytest

from conftest import S128, s128_params
from oracle import ckks_oracle as oc
from paper_2102_00319_b200 import hostmath as hm
from paper_2102_00319_b200 import percell
from paper_2102_00319_b200.chain import build_chain
from paper_2102_00319_b200.configs import CONFIGS


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def frac(s):
    a, b = s.split("/")
    return Fraction(int(a), int(b))


class TestChain:
    def test_small_ring_tables_match_reference(self, s128):
        ch = build_chain(s128_params(), S128["extra"])
        for name in ("p", "p_inv", "r2", "n_inv", "twiddles"):
            assert np.array_equal(getattr(ch, name), s128[name]), name

    @pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
    def test_baseline_chains_match_reference(self, golden, name):
        cfg = CONFIGS[name]
        ch = build_chain(cfg.params(), cfg.base_extra_bits)
        g = golden["chains"][name]
        assert [int(x) for x in ch.p] == g["primes"]
        assert [int(x) for x in ch.p_inv] == g["p_inv"]
        assert [int(x) for x in ch.r2] == g["r2"]
        assert [int(x) for x in ch.n_inv] == g["n_inv"]
        assert ch.num_levels == g["num_levels"]
        assert digest(ch.twiddles) == g["twiddle_digest"]

    def test_cfg4_primes_match_reference(self, golden):
        cfg = CONFIGS["cfg4"]
        ch = build_chain(cfg.params(), cfg.base_extra_bits)
        assert [int(x) for x in ch.p] == golden["chains"]["cfg4"]["primes"]


class TestKernels:
    def test_ntt_pair_matches_reference(self, s128):
        f = s128["ntt_in"].copy()
        oc.ntt_fwd_rows(f, s128["twiddles"], s128["p"], s128["p_inv"])
        assert np.array_equal(f, s128["ntt_fwd"])
        h = s128["ntt_in"].copy()
        oc.ntt_inv_rows(h, s128["twiddles"], s128["n_inv"], s128["p"], s128["p_inv"])
        assert np.array_equal(h, s128["ntt_inv"])
        oc.ntt_fwd_rows(h, s128["twiddles"], s128["p"], s128["p_inv"])
        assert np.array_equal(h, s128["ntt_in"])

    @pytest.mark.parametrize("lvl", [1, 2, 3, 4, 5, 6])
    def test_rescale_matches_reference(self, s128, lvl):
        o = oc.OracleCkks(build_chain(s128_params(), S128["extra"]), 42)
        assert np.array_equal(o.rescale(s128[f"resc_in_{lvl}"]), s128[f"resc_out_{lvl}"])


class TestEncoding:
    def test_encode_coeffs_bit_exact(self, s128):
        ch = build_chain(s128_params(), S128["extra"])
        got = hm.encode_coeffs(s128["enc_values"], Fraction(2**30), ch.ring_degree, ch.modulus_at_level(ch.num_levels))
        assert np.array_equal(got, s128["enc_coeffs"])

    def test_decode_bit_exact(self, s128):
        got = hm.slots_from_coeffs(s128["enc_coeffs"].astype(np.float64), float(2**30), 128)
        assert np.array_equal(got, s128["dec_slots"])


class TestOracleBackend:
    def test_keys_match_reference(self, s128, oracle_s128):
        _, keys = oracle_s128
        k = keys.secret
        for name, arr in (("s_eval", k.s_eval), ("pk_b", k.pk_b), ("pk_a", k.pk_a), ("evk_b", k.evk_b), ("evk_a", k.evk_a)):
            assert np.array_equal(arr, s128[name]), name

    def test_ops_match_reference(self, s128, oracle_s128, golden):
        be, keys = oracle_s128
        a = be.encrypt(s128["va"], keys, entropy=1)
        b = be.encrypt(s128["vb"], keys, entropy=2)

        def same(name, ct):
            assert np.array_equal(ct.payload.c0, s128[f"{name}_c0"]), name
            assert np.array_equal(ct.payload.c1, s128[f"{name}_c1"]), name

        same("a", a)
        same("b", b)
        raw = be.mul_ct_ct_raw(a, b)
        for i, d in enumerate((raw.payload.d0, raw.payload.d1, raw.payload.d2)):
            assert np.array_equal(d, s128[f"raw_d{i}"])
        fin = be.raw_finalize(be.raw_add(raw, be.mul_ct_ct_raw(a, a)))
        same("fin", fin)
        assert fin.level == golden["s128"]["fin"]["level"]
        assert fin.scale == frac(golden["s128"]["fin"]["scale"])
        assert np.array_equal(be.decrypt(fin, keys).values, s128["fin_dec"])
        pt = be.encode_plain(s128["vb"], level=a.level)
        assert np.array_equal(pt.payload.rows, s128["pt_rows"])
        ctpt = be.mul_ct_pt(a, pt)
        same("ctpt", ctpt)
        assert ctpt.scale == frac(golden["s128"]["ctpt"]["scale"])
        same("add", be.add_ct_ct(a, b))
        same("addpt", be.add_ct_pt(a, s128["vb"]))
        same("drop_mul", be.mul_ct_ct(be.drop_to_level(a, 3), b))

    def test_square_chain_to_depth_boundary(self, s128, oracle_s128, golden):
        be, keys = oracle_s128
        ct = be.encrypt(np.full(be.slots, 1.01), keys, entropy=3)
        for step, rec in enumerate(golden["s128"]["square_trace"]):
            ct = be.mul_ct_ct(ct, ct)
            assert np.array_equal(ct.payload.c0, s128[f"sq{step}_c0"])
            assert np.array_equal(ct.payload.c1, s128[f"sq{step}_c1"])
            assert ct.level == rec["level"] and ct.scale == frac(rec["scale"])
            assert ct.noise_bits == pytest.approx(rec["noise"])
        from paper_2102_00319_b200.errors import DepthExhausted

        with pytest.raises(DepthExhausted):
            be.mul_ct_ct(ct, ct)

    @pytest.mark.parametrize("name", ["mini2", "mini3", "mini4"])
    def test_mini_cnn_logits_match_reference(self, golden, oracle_s128, name):
        from nets import mini_networks

        be, keys = oracle_s128
        net = mini_networks()[name]
        imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
        be.counters.reset()
        enc = percell.encrypt_network(be, net, keys)
        grid = percell.encrypt_images(be, imgs, keys)
        logits = percell.run_network(be, enc, grid)
        g = golden["minis"][name]
        assert [digest(np.concatenate([c.payload.c0, c.payload.c1])) for c in logits] == g["logit_digests"]
        assert logits[0].scale == frac(g["scale"])
        assert be.counters.snapshot().__dict__ == g["counters"]

    def test_rotation_oracle_permutes_slots(self, oracle_s128):
        be, keys = oracle_s128
        v = np.random.default_rng(4).uniform(-1, 1, be.slots)
        ct = be.encrypt(v, keys, entropy=9)
        rot = be.rotate(ct, 1)
        got = be.decrypt(rot, keys).values
        perm = hm.galois_slot_permutation(be.params.ring_degree, be.galois_element(1))
        assert np.max(np.abs(got - v[perm])) < 1e-5
        assert rot.level == ct.level and rot.scale == ct.scale


@pytest.mark.slow
def test_cfg1_ops_match_reference_digests(golden):
    from oracle.ckks_oracle import OracleBackend

    cfg = CONFIGS["cfg1"]
    be = OracleBackend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    g = golden["cfg1_ops"]
    k = keys.secret
    assert digest(k.s_eval) == g["s_eval"]
    assert digest(np.concatenate([k.pk_b, k.pk_a])) == g["pk"]
    assert digest(np.concatenate([k.evk_b.ravel(), k.evk_a.ravel()])) == g["evk"]
    rng = np.random.default_rng(101)
    xs = rng.uniform(-1, 1, (4, be.slots))
    ys = rng.uniform(-1, 1, (4, be.slots))
    cd = lambda ct: digest(np.concatenate([ct.payload.c0, ct.payload.c1]))  # noqa: E731
    for i, rec in enumerate(g["ops"]):
        x = be.encrypt(xs[i], keys, entropy=i)
        y = be.encrypt(ys[i], keys, entropy=256 + i)
        assert cd(x) == rec["x"] and cd(y) == rec["y"]
        mul = be.mul_ct_ct(x, y)
        assert cd(mul) == rec["mul"]
        assert cd(be.mul_ct_pt(x, be.encode_plain(ys[i], level=x.level))) == rec["ctpt"]
        assert cd(be.add_ct_ct(x, y)) == rec["add"]
        assert np.allclose(be.decrypt(mul, keys).values[:8], rec["mul_dec8"], atol=0, rtol=0)


class TestRotationPinned:
    """Rotation has no reference API; tests/golden/make_golden.py builds it from the
    reference's own keygen loop and kernels (relin_accumulate + moddown_special), so
    the oracle's rotation is pinned to reference arithmetic, not only to itself."""

    @pytest.mark.parametrize("steps", [1, 3])
    def test_rotation_matches_reference_kernels(self, s128, golden, steps):
        from oracle.ckks_oracle import OracleBackend, _Cipher

        be = OracleBackend(s128_params(), S128["extra"])
        keys = be.keygen(galois_steps=(steps,))
        be.set_eval_key(keys)
        g = be.galois_element(steps)
        rec = golden["s128"]["rotation"][str(steps)]
        assert digest(keys.galois[g][0]) == rec["galois_key_b"]
        ct = be._cipher(_Cipher(s128["a_c0"], s128["a_c1"]), rec["level"], be.canonical_scale, 0.0)
        rot = be.rotate(ct, steps)
        assert np.array_equal(rot.payload.c0, s128[f"rot{steps}_c0"])
        assert np.array_equal(rot.payload.c1, s128[f"rot{steps}_c1"])
