"""Bit-exact parity of the CUDA product path against the CPU oracle and the
reference's golden vectors.  Needs a B200 (marked gpu)."""

import hashlib
from fractions import Fraction

import numpy as np
import pytest

from conftest import S128, s128_params

pytestmark = pytest.mark.gpu


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def frac(s):
    a, b = s.split("/")
    return Fraction(int(a), int(b))


@pytest.fixture(scope="module")
def dev_s128():
    from paper_2102_00319_b200.backend import B200Backend

    be = B200Backend(s128_params(), S128["extra"])
    keys = be.keygen(galois_steps=(1,))
    be.set_eval_key(keys)
    return be, keys


def host(be, ct):
    c0, c1 = be.cipher_rows_host(ct)
    return c0, c1


def test_ntt_pair_matches_reference(s128):
    import torch
    from paper_2102_00319_b200.backend import DeviceContext, u64_to_dev, dev_to_u64
    from paper_2102_00319_b200.chain import build_chain

    ctx = DeviceContext(build_chain(s128_params(), S128["extra"]))
    rows = s128["ntt_in"].shape[0]
    d = u64_to_dev(s128["ntt_in"], ctx.device)
    ctx.call("heb_ntt_fwd", d.data_ptr(), 1, rows, 0, rows * ctx.n, ctx.stream)
    assert np.array_equal(dev_to_u64(d), s128["ntt_fwd"])
    ctx.call("heb_ntt_inv", d.data_ptr(), 1, rows, 0, rows * ctx.n, ctx.stream)
    assert np.array_equal(dev_to_u64(d), s128["ntt_in"])
    d = u64_to_dev(s128["ntt_in"], ctx.device)
    ctx.call("heb_ntt_inv", d.data_ptr(), 1, rows, 0, rows * ctx.n, ctx.stream)
    assert np.array_equal(dev_to_u64(d), s128["ntt_inv"])
    torch.cuda.synchronize()


@pytest.mark.parametrize("logn", [6, 8, 10, 12, 13, 14])
def test_ntt_matches_oracle_all_sizes(logn):
    from oracle import ckks_oracle as oc
    from paper_2102_00319_b200.backend import DeviceContext, u64_to_dev, dev_to_u64
    from paper_2102_00319_b200.chain import build_chain
    from paper_2102_00319_b200.params import derive_params

    n = 1 << logn
    ch = build_chain(derive_params(2 * n, 200, 40, seed=1), 20)
    ctx = DeviceContext(ch)
    rng = np.random.default_rng(logn)
    rows = ch.num_rows
    x = np.stack([rng.integers(0, int(q), n, dtype=np.uint64) for q in ch.p])
    ref = x.copy()
    oc.ntt_fwd_rows(ref, ch.twiddles, ch.p, ch.p_inv)
    d = u64_to_dev(np.stack([x, x]), ctx.device)
    ctx.call("heb_ntt_fwd", d.data_ptr(), 2, rows, 0, rows * n, ctx.stream)
    got = dev_to_u64(d)
    assert np.array_equal(got[0], ref) and np.array_equal(got[1], ref)
    ctx.call("heb_ntt_inv", d.data_ptr(), 2, rows, 0, rows * n, ctx.stream)
    assert np.array_equal(dev_to_u64(d)[1], x)


class TestS128:
    def test_keys_bit_exact(self, s128, dev_s128):
        from paper_2102_00319_b200.backend import dev_to_u64

        _, keys = dev_s128
        assert np.array_equal(dev_to_u64(keys.secret.s_eval), s128["s_eval"])
        assert np.array_equal(dev_to_u64(keys.public.b), s128["pk_b"])
        assert np.array_equal(dev_to_u64(keys.public.a), s128["pk_a"])
        assert np.array_equal(dev_to_u64(keys.evaluation.b), s128["evk_b"])
        assert np.array_equal(dev_to_u64(keys.evaluation.a), s128["evk_a"])

    def test_ops_bit_exact(self, s128, dev_s128, golden):
        be, keys = dev_s128
        a = be.encrypt(s128["va"], keys, entropy=1)
        b = be.encrypt(s128["vb"], keys, entropy=2)

        def same(name, ct):
            c0, c1 = host(be, ct)
            assert np.array_equal(c0, s128[f"{name}_c0"]), name
            assert np.array_equal(c1, s128[f"{name}_c1"]), name

        same("a", a)
        same("b", b)
        raw = be.mul_ct_ct_raw(a, b)
        from paper_2102_00319_b200.backend import dev_to_u64

        rh = dev_to_u64(raw.payload.buf)
        for i in range(3):
            assert np.array_equal(rh[i], s128[f"raw_d{i}"]), i
        fin = be.raw_finalize(be.raw_add(raw, be.mul_ct_ct_raw(a, a)))
        same("fin", fin)
        assert fin.scale == frac(golden["s128"]["fin"]["scale"])
        assert np.array_equal(be.decrypt(fin, keys).values, s128["fin_dec"])
        pt = be.encode_plain(s128["vb"], level=a.level)
        assert np.array_equal(dev_to_u64(pt.payload.rows), s128["pt_rows"])
        same("ctpt", be.mul_ct_pt(a, pt))
        same("add", be.add_ct_ct(a, b))
        same("addpt", be.add_ct_pt(a, s128["vb"]))
        same("drop_mul", be.mul_ct_ct(be.drop_to_level(a, 3), b))

    def test_rescale_every_level(self, s128, dev_s128):
        from paper_2102_00319_b200.backend import u64_to_dev, dev_to_u64, ct_desc

        be, _ = dev_s128
        for lvl in range(1, be.fresh_level + 1):
            comp = s128[f"resc_in_{lvl}"]
            d = u64_to_dev(comp[None], be.dev)  # (1 comp, k, n)
            out = be.ctx.empty(1, lvl, be.n)
            be.ctx.call("heb_rescale", ct_desc(d), None, 0, ct_desc(out), 1, 1, lvl, be.ctx.stream)
            assert np.array_equal(dev_to_u64(out)[0], s128[f"resc_out_{lvl}"]), lvl

    def test_square_chain(self, s128, dev_s128, golden):
        be, keys = dev_s128
        ct = be.encrypt(np.full(be.slots, 1.01), keys, entropy=3)
        for step, rec in enumerate(golden["s128"]["square_trace"]):
            ct = be.mul_ct_ct(ct, ct)
            c0, c1 = host(be, ct)
            assert np.array_equal(c0, s128[f"sq{step}_c0"]) and np.array_equal(c1, s128[f"sq{step}_c1"]), step
            assert ct.level == rec["level"] and ct.scale == frac(rec["scale"])

    def test_rotation_matches_oracle(self, dev_s128, oracle_s128):
        be, keys = dev_s128
        ob, okeys = oracle_s128
        v = np.random.default_rng(4).uniform(-1, 1, be.slots)
        ct = be.encrypt(v, keys, entropy=9)
        oct_ = ob.encrypt(v, okeys, entropy=9)
        r = be.rotate(ct, 1)
        orr = ob.rotate(oct_, 1)
        c0, c1 = host(be, r)
        assert np.array_equal(c0, orr.payload.c0) and np.array_equal(c1, orr.payload.c1)
        lvl2 = be.rotate(be.drop_to_level(ct, 2), 1)
        olvl2 = ob.rotate(ob.drop_to_level(oct_, 2), 1)
        assert np.array_equal(host(be, lvl2)[0], olvl2.payload.c0)

    @pytest.mark.parametrize("steps", [1, 3])
    def test_rotation_matches_reference_kernels(self, s128, golden, steps):
        """Device rotation against the reference-kernel rotation fixture (make_golden.ref_rotate)."""
        from paper_2102_00319_b200.backend import B200Backend

        be = B200Backend(s128_params(), S128["extra"])
        keys = be.keygen(galois_steps=(steps,))
        be.set_eval_key(keys)
        rec = golden["s128"]["rotation"][str(steps)]
        g = be.galois_element(steps)
        assert digest(keys.galois[g].b.cpu().numpy().view(np.uint64)) == rec["galois_key_b"]
        ct = be.cipher_from_host(s128["a_c0"], s128["a_c1"], rec["level"], be.canonical_scale, 0.0)
        c0, c1 = be.cipher_rows_host(be.rotate(ct, steps))
        assert np.array_equal(c0, s128[f"rot{steps}_c0"]) and np.array_equal(c1, s128[f"rot{steps}_c1"])

    @pytest.mark.parametrize("name", ["mini2", "mini3", "mini4"])
    def test_mini_cnn_percell_matches_reference(self, golden, dev_s128, name):
        from nets import mini_networks
        from paper_2102_00319_b200 import percell

        be, keys = dev_s128
        net = mini_networks()[name]
        imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
        be.counters.reset()
        enc = percell.encrypt_network(be, net, keys)
        grid = percell.encrypt_images(be, imgs, keys)
        logits = percell.run_network(be, enc, grid)
        g = golden["minis"][name]
        assert [digest(np.concatenate(host(be, c))) for c in logits] == g["logit_digests"]
        assert be.counters.snapshot().__dict__ == g["counters"]


def test_cfg1_digests_match_reference(golden):
    from paper_2102_00319_b200.backend import B200Backend, dev_to_u64
    from paper_2102_00319_b200.configs import CONFIGS

    cfg = CONFIGS["cfg1"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    g = golden["cfg1_ops"]
    assert digest(dev_to_u64(keys.secret.s_eval)) == g["s_eval"]
    assert digest(np.concatenate([dev_to_u64(keys.public.b), dev_to_u64(keys.public.a)])) == g["pk"]
    assert digest(np.concatenate([dev_to_u64(keys.evaluation.b).ravel(), dev_to_u64(keys.evaluation.a).ravel()])) == g["evk"]
    rng = np.random.default_rng(101)
    xs = rng.uniform(-1, 1, (4, be.slots))
    ys = rng.uniform(-1, 1, (4, be.slots))
    cd = lambda ct: digest(np.concatenate(be.cipher_rows_host(ct)))  # noqa: E731
    for i, rec in enumerate(g["ops"]):
        x = be.encrypt(xs[i], keys, entropy=i)
        y = be.encrypt(ys[i], keys, entropy=256 + i)
        assert cd(x) == rec["x"] and cd(y) == rec["y"]
        mul = be.mul_ct_ct(x, y)
        assert cd(mul) == rec["mul"]
        assert hashlib.sha256(be.cipher_payload_bytes(mul)).hexdigest() == rec["mul_payload"]
        assert cd(be.mul_ct_pt(x, be.encode_plain(ys[i], level=x.level))) == rec["ctpt"]
        assert cd(be.add_ct_ct(x, y)) == rec["add"]
        assert list(be.decrypt(mul, keys).values[:8]) == rec["mul_dec8"]


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name", ["mini2", "mini3", "mini4"])
def test_batched_layers_match_reference(golden, dev_s128, name, fused):
    """The batched layer evaluator (one launch sequence per layer) reproduces the
    reference op sequence bit for bit, including levels, scales and counters --
    with the fused convolution kernel and with the generic gather-dot path."""
    from nets import mini_networks
    from paper_2102_00319_b200 import layers

    be, keys = dev_s128
    net = mini_networks()[name]
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
    be.counters.reset()
    enc = layers.encrypt_network(be, net, keys)
    be.counters.reset()
    x = layers.encrypt_images(be, imgs, keys)
    out = layers.LayerEvaluator(be, fused_conv=fused).run(enc, x)
    g = golden["minis"][name]
    digests = [digest(np.concatenate(be.cipher_rows_host(be.batch_to_cipher(out, i)))) for i in range(out.count)]
    assert digests == g["logit_digests"]
    assert out.level == g["level"] and out.scale == frac(g["scale"])
    assert be.counters.snapshot().__dict__ == g["counters"]
    dec = be.decrypt_batch(out, keys)
    assert np.allclose(dec[:, :8].T, np.array(g["decrypted_first8"]), atol=0, rtol=0)


@pytest.mark.parametrize("logn", [14, 15])
def test_ntt_split_rows_match_oracle(logn):
    """N = 2^14 / 2^15 rows run on 2- / 4-CTA clusters (cross-part stages through
    distributed shared memory)."""
    from oracle import ckks_oracle as oc
    from paper_2102_00319_b200.backend import DeviceContext, u64_to_dev, dev_to_u64
    from paper_2102_00319_b200.chain import build_chain
    from paper_2102_00319_b200.params import derive_params

    n = 1 << logn
    ch = build_chain(derive_params(2 * n, 200, 40, seed=1), 20)
    ctx = DeviceContext(ch)
    rng = np.random.default_rng(logn)
    rows = ch.num_rows
    x = np.stack([rng.integers(0, int(q), n, dtype=np.uint64) for q in ch.p])
    ref = x.copy()
    oc.ntt_fwd_rows(ref, ch.twiddles, ch.p, ch.p_inv)
    d = u64_to_dev(np.stack([x, x, x]), ctx.device)
    ctx.call("heb_ntt_fwd", d.data_ptr(), 3, rows, 0, rows * n, ctx.stream)
    got = dev_to_u64(d)
    assert all(np.array_equal(got[i], ref) for i in range(3))
    ctx.call("heb_ntt_inv", d.data_ptr(), 3, rows, 0, rows * n, ctx.stream)
    assert np.array_equal(dev_to_u64(d)[2], x)


@pytest.mark.parametrize("m", [2**13, 2**15, 2**16])
def test_ring_sweep_ops_match_oracle(m):
    """Every payload op bit-exact vs the oracle at N = 4096, 16384 and 32768 (split rows)."""
    from oracle.ckks_oracle import OracleBackend
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.params import derive_params

    params = derive_params(m, 220, 40, seed=3)
    dev, ora = B200Backend(params, 20), OracleBackend(params, 20)
    dk, ok = dev.keygen(galois_steps=(1,)), ora.keygen(galois_steps=(1,))
    dev.set_eval_key(dk)
    ora.set_eval_key(ok)
    rng = np.random.default_rng(m)
    x, y = rng.uniform(-1, 1, (2, dev.slots))

    def same(a, b, what):
        c0, c1 = dev.cipher_rows_host(a)
        assert np.array_equal(c0, b.payload.c0) and np.array_equal(c1, b.payload.c1), what

    dx, dy = dev.encrypt(x, dk, entropy=1), dev.encrypt(y, dk, entropy=2)
    ox, oy = ora.encrypt(x, ok, entropy=1), ora.encrypt(y, ok, entropy=2)
    same(dx, ox, "encrypt")
    dm, om = dev.mul_ct_ct(dx, dy), ora.mul_ct_ct(ox, oy)
    same(dm, om, "mul_ct_ct")
    same(dev.mul_ct_pt(dx, y), ora.mul_ct_pt(ox, y), "mul_ct_pt")
    same(dev.rotate(dx, 1), ora.rotate(ox, 1), "rotate")
    same(dev.mul_ct_ct(dm, dm), ora.mul_ct_ct(om, om), "second level")
    assert np.max(np.abs(dev.decrypt(dm, dk).values - x * y)) < 1e-4


@pytest.mark.parametrize("pipelines", [1, 3])
def test_graph_pipelines_match_direct_run(golden, dev_s128, pipelines):
    """run_many / run_stream replay one captured CUDA graph per pipeline; every step's
    logits must equal the host-issued run (and the reference digests), and the op
    counters must advance as if each step had been issued op by op."""
    import torch

    from nets import mini_networks
    from paper_2102_00319_b200 import layers

    be, keys = dev_s128
    net = mini_networks()["mini3"]
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, imgs, keys)
    ev = layers.LayerEvaluator(be)
    be.counters.reset()
    want = ev.run(enc, x)
    per_run = be.counters.snapshot().__dict__
    want_rows = want.buf.clone()
    seen = []
    ev.run_many(enc, x, 5, pipelines=pipelines, on_output=lambda s, o: seen.append(o.buf.clone()))
    torch.cuda.synchronize()
    assert len(seen) == 5 and all(torch.equal(t, want_rows) for t in seen)
    digests = [digest(np.concatenate(be.cipher_rows_host(be.batch_to_cipher(want, i)))) for i in range(want.count)]
    assert digests == golden["minis"]["mini3"]["logit_digests"]
    host_in = [x.buf.cpu().pin_memory() for _ in range(4)]
    host_out = [torch.empty((want.count, 2, want.k, be.n), dtype=torch.int64).pin_memory() for _ in range(4)]
    be.counters.reset()
    ev.run_stream(enc, host_in, x.level, x.scale, x.noise_bits, host_out, pipelines=pipelines)
    torch.cuda.synchronize()
    assert all(torch.equal(h, want_rows[:, :, : want.k].cpu()) for h in host_out)
    assert be.counters.snapshot().__dict__ == {f: 4 * v for f, v in per_run.items()}


def test_conv_beyond_fused_stage_matches_percell(dev_s128):
    """heb_conv with more taps than the fused kernel's shared-memory stage (81 > 64):
    window indices built on the device, index-driven tensor; bit-identical to the
    reference op sequence (percell) and to the host-indexed gather-dot path."""
    from paper_2102_00319_b200 import layers, percell
    from paper_2102_00319_b200.model import Conv, Dense, Flatten, Network, Square, SumPool

    be, keys = dev_s128
    rng = np.random.default_rng(5)
    net = Network((12, 12), (
        Conv(weights=rng.normal(0, 0.1, (2, 1, 9, 9)), stride=1, bias=rng.normal(0, 0.1, 2)),
        Square(), SumPool(), Flatten(),
        Dense(weights=rng.normal(0, 0.3, (8, 3))),
    ))
    imgs = rng.uniform(0, 1, (be.slots, 12, 12))
    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, imgs, keys)
    fused = layers.LayerEvaluator(be, fused_conv=True).run(enc, x)
    generic = layers.LayerEvaluator(be, fused_conv=False).run(enc, x)
    penc = percell.encrypt_network(be, net, keys)
    logits = percell.run_network(be, penc, percell.encrypt_images(be, imgs, keys))
    for i in range(fused.count):
        a = np.concatenate(be.cipher_rows_host(be.batch_to_cipher(fused, i)))
        b = np.concatenate(be.cipher_rows_host(be.batch_to_cipher(generic, i)))
        c = np.concatenate(host(be, logits[i]))
        assert np.array_equal(a, b) and np.array_equal(a, c)


def test_layer_entry_points_edge_cases(dev_s128):
    """Empty batches are no-ops; out-of-range levels and shapes fail loudly (ValueError
    from HEB_EINVAL) instead of touching memory -- reference errors.py taxonomy."""
    from paper_2102_00319_b200 import _lib
    from paper_2102_00319_b200.backend import ct_desc

    be, _ = dev_s128
    ctx = be.ctx
    evk = be._require_eval_key().evaluation.prep.data_ptr()
    top = be.chain.num_rows - 2  # highest ciphertext level
    buf = ctx.empty(2, 3, top + 1, be.n)
    d = ct_desc(buf)
    none = _lib.HebCt(None, 0, 0)
    ctx.call("heb_square", d, d, 0, top, evk, ctx.stream)                      # count 0: no-op
    ctx.call("heb_fc", d, d, buf.data_ptr(), buf.data_ptr(), 1, none, d, 0, top, evk, ctx.stream)
    ctx.call("heb_poly_act", d, buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), d, 0, top, evk, ctx.stream)
    with pytest.raises(ValueError):
        ctx.call("heb_square", d, d, 1, top + 1, evk, ctx.stream)              # no row to drop into
    with pytest.raises(ValueError):
        ctx.call("heb_square", d, d, 1, 0, evk, ctx.stream)                    # depth exhausted
    with pytest.raises(ValueError):
        ctx.call("heb_poly_act", d, buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), d, 1, 1, evk, ctx.stream)
    with pytest.raises(ValueError):
        ctx.call("heb_conv", d, d, none, d, 1, 4, 4, 1, 5, 5, 1, top, evk, ctx.stream)  # kernel larger than map
    with pytest.raises(ValueError):
        ctx.call("heb_sumpool", d, d, 1, 1, 4, 0, ctx.stream)                  # map narrower than a window
    torch_sync()


def torch_sync():
    import torch

    torch.cuda.synchronize()
