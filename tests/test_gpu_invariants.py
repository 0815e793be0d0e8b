"""Reference test invariants on the device, and worst-case operands for the exact FP64 paths.

* thread safety (`/root/reference/pkg/tests/test_backend_contract.py:387-422`): 16
  concurrent mul_ct_ct on shared operands give identical bits and leave the operands
  untouched -- on one shared stream (serialised by the per-stream scratch lock) and on
  one stream per thread (independent scratch arenas);
* decrypt fault injection (`/root/reference/pkg/tests/test_pipeline_invariants.py:62-71`):
  a corrupted residue row trips the device decrypt's cross-residue guard;
* worst-magnitude operands: the FP64 engine keeps values unreduced and signed between
  stages and argues |v| < 2^47 with an at-most-one quotient error (csrc/ntt.cuh); the
  conv kernel sums exact 20-bit-limb products in FP64.  Every residue = p - 1, alternating
  0 / p - 1, and every residue = (p - 1) / 2 drive those bounds through the NTT (every
  ring size, FP64 and integer rows), a relinearisation (ModUp, ModDown tail) and a
  45-tap conv layer -- bit-exact against the oracle.
"""

from concurrent.futures import ThreadPoolExecutor
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def small(m=1 << 10, L=270, r=35, seed=21, extra=25):
    from oracle.ckks_oracle import OracleBackend
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.params import derive_params

    p = derive_params(m, L, r, seed=seed)
    dev, ora = B200Backend(p, extra), OracleBackend(p, extra)
    dk, ok = dev.keygen(), ora.keygen()
    dev.set_eval_key(dk)
    ora.set_eval_key(ok)
    return dev, ora, dk, ok


@pytest.mark.parametrize("per_thread_stream", [False, True])
def test_shared_operands_across_threads_bit_identical(per_thread_stream):
    import torch

    dev, _, dk, _ = small()
    rng = np.random.default_rng(70)
    xa, xb = rng.uniform(-1, 1, (2, dev.slots))
    a, b = dev.encrypt(xa, dk), dev.encrypt(xb, dk)
    ref = dev.cipher_rows_host(dev.mul_ct_ct(a, b))
    dev.counters.reset()

    def work(_):
        if per_thread_stream:
            st = torch.cuda.Stream(dev.dev)
            st.wait_stream(torch.cuda.default_stream(dev.dev))
            with torch.cuda.stream(st):
                ct = dev.mul_ct_ct(a, b)
                rows = dev.cipher_rows_host(ct)
            return rows
        return dev.cipher_rows_host(dev.mul_ct_ct(a, b))

    with ThreadPoolExecutor(max_workers=8) as pool:
        results = list(pool.map(work, range(16)))
    for c0, c1 in results:
        assert np.array_equal(c0, ref[0]) and np.array_equal(c1, ref[1])
    assert dev.counters.snapshot().ctct_mult == 16
    assert np.max(np.abs(dev.decrypt(a, dk).values - xa)) <= 1e-6


def test_decrypt_detects_out_of_range_coefficients():
    from paper_2102_00319_b200.errors import DecryptionOutOfRange

    dev, _, dk, _ = small()
    ct = dev.encrypt(np.full(dev.slots, 0.5), dk)
    c0, c1 = dev.cipher_rows_host(ct)
    c0 = c0.copy()
    c0[1] = (c0[1] + np.uint64(12345)) % dev.chain.p[1]
    bad = dev.cipher_from_host(c0, c1, ct.level, ct.scale, ct.noise_bits)
    with pytest.raises(DecryptionOutOfRange):
        dev.decrypt(bad, dk)
    # the batched decrypt reports the same fault
    from paper_2102_00319_b200.backend import CipherBatch
    import torch

    buf = torch.stack([bad.payload.buf[:, : ct.level + 1]]).contiguous()
    with pytest.raises(DecryptionOutOfRange):
        dev.decrypt_batch(CipherBatch(buf, ct.level, ct.scale, ct.noise_bits), dk)


def extreme_rows(p: np.ndarray, n: int, kind: str) -> np.ndarray:
    p = p.astype(np.uint64)[:, None]
    if kind == "max":
        return np.repeat(p - np.uint64(1), n, axis=1)
    if kind == "alternating":
        a = np.repeat(p - np.uint64(1), n, axis=1)
        a[:, ::2] = 0
        return a
    return np.repeat((p - np.uint64(1)) // np.uint64(2), n, axis=1)  # "half": the centring boundary


KINDS = ["max", "alternating", "half"]


@pytest.mark.parametrize("logn", [6, 9, 12, 13, 14, 15])
@pytest.mark.parametrize("kind", KINDS)
def test_ntt_worst_magnitudes(logn, kind):
    """FP64 (40-bit) and integer (60-bit) rows at every engine shape incl. split rows."""
    from oracle import ckks_oracle as oc
    from paper_2102_00319_b200.backend import DeviceContext, dev_to_u64, u64_to_dev
    from paper_2102_00319_b200.chain import build_chain
    from paper_2102_00319_b200.params import derive_params

    n = 1 << logn
    ch = build_chain(derive_params(2 * n, 200, 40, seed=1), 20)
    ctx = DeviceContext(ch)
    x = extreme_rows(ch.p, n, kind)
    ref = x.copy()
    oc.ntt_fwd_rows(ref, ch.twiddles, ch.p, ch.p_inv)
    d = u64_to_dev(np.stack([x, x]), ctx.device)
    rows = ch.num_rows
    ctx.call("heb_ntt_fwd", d.data_ptr(), 2, rows, 0, rows * n, ctx.stream)
    got = dev_to_u64(d)
    assert np.array_equal(got[0], ref) and np.array_equal(got[1], ref)
    ctx.call("heb_ntt_inv", d.data_ptr(), 2, rows, 0, rows * n, ctx.stream)
    assert np.array_equal(dev_to_u64(d)[1], x)


def cipher_pair(dev, ora, rows0, rows1, level, scale):
    from oracle.ckks_oracle import _Cipher

    d = dev.cipher_from_host(rows0, rows1, level, scale)
    o = ora._cipher(_Cipher(rows0.copy(), rows1.copy()), level, scale, float("-inf"))
    return d, o


@pytest.mark.parametrize("m", [1 << 11, 1 << 14, 1 << 16])
@pytest.mark.parametrize("kind", KINDS)
def test_relinearisation_worst_magnitudes(m, kind):
    """tensor + relinearise + rescale (ModUp key products, ModDown tail) and ct x pt
    (rescale) on extreme residues, N = 1024 / 8192 / 32768 (split rows)."""
    dev, ora, _, _ = small(m=m, L=220, r=40, seed=5, extra=20)
    k = dev.chain.num_levels + 1
    n = dev.n
    lvl = k - 1
    sc = dev.canonical_scale
    p = dev.chain.p[:k]
    a, oa = cipher_pair(dev, ora, extreme_rows(p, n, kind), extreme_rows(p, n, "max"), lvl, sc)
    b, ob = cipher_pair(dev, ora, extreme_rows(p, n, "alternating"), extreme_rows(p, n, kind), lvl, sc)

    def same(x, y, what):
        c0, c1 = dev.cipher_rows_host(x)
        assert np.array_equal(c0, y.payload.c0) and np.array_equal(c1, y.payload.c1), what

    same(dev.mul_ct_ct(a, b), ora.mul_ct_ct(oa, ob), f"mul_ct_ct {kind}")
    same(dev.mul_ct_ct(a, a), ora.mul_ct_ct(oa, oa), f"square {kind}")
    raw_d = dev.raw_add(dev.mul_ct_ct_raw(a, b), dev.mul_ct_ct_raw(b, a))
    raw_o = ora.raw_add(ora.mul_ct_ct_raw(oa, ob), ora.mul_ct_ct_raw(ob, oa))
    same(dev.raw_finalize(raw_d), ora.raw_finalize(raw_o), f"accumulated raw {kind}")


@pytest.mark.parametrize("kind", KINDS)
def test_conv_layer_worst_magnitudes(kind):
    """45-tap conv (5 channels, 3x3) with every input and weight residue extreme: the
    split-limb FP64 accumulation and the integer 128-bit sums at their largest."""
    import torch

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import CipherBatch
    from paper_2102_00319_b200.model import Conv

    dev, ora, _, _ = small(m=1 << 11, L=220, r=40, seed=5, extra=20)
    k = dev.chain.num_levels + 1
    n, lvl, sc = dev.n, k - 1, dev.canonical_scale
    p = dev.chain.p[:k]
    C, M = 5, 4
    x_rows = np.stack([np.stack([extreme_rows(p, n, kind), extreme_rows(p, n, "max")])] * (C * M * M))
    w_rows = np.stack([np.stack([extreme_rows(p, n, "max"), extreme_rows(p, n, kind)])] * (2 * C * 9))
    x = CipherBatch(torch.from_numpy(x_rows.view(np.int64)).to(dev.dev), lvl, sc)
    w = CipherBatch(torch.from_numpy(w_rows.view(np.int64)).to(dev.dev), lvl, sc)
    y, (F, om, on) = layers.LayerEvaluator(dev).conv(x, (C, M, M), Conv(weights=np.zeros((2, C, 3, 3)), stride=1),
                                                     w, None)
    got = y.buf[:, :, : y.k].cpu().numpy().view(np.uint64)
    from oracle.ckks_oracle import _Cipher

    xo = ora._cipher(_Cipher(x_rows[0, 0], x_rows[0, 1]), lvl, sc, float("-inf"))
    wo = ora._cipher(_Cipher(w_rows[0, 0], w_rows[0, 1]), lvl, sc, float("-inf"))
    raw = None
    for _ in range(C * 9):
        t = ora.mul_ct_ct_raw(xo, wo)
        raw = t if raw is None else ora.raw_add(raw, t)
    want = ora.raw_finalize(raw)
    for o in range(F * om * on):  # every cell sees the same 45 extreme taps
        assert np.array_equal(got[o, 0], want.payload.c0) and np.array_equal(got[o, 1], want.payload.c1), o
