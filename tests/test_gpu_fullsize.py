"""Bit-exact parity at the bench's own full size (config 2: N = 8192, 6-row chain,
4096 images per batch): the WHOLE network, every output ciphertext of every layer,
against the CPU oracle.

The batched device layers (heb_conv / heb_square / heb_sumpool / heb_fc) run over the
cfg2 network; the oracle (a restatement of the reference kernels) recomputes each
layer from the SAME device input ciphertexts of that layer with the reference op
sequence (mul_ct_ct_raw + raw_add per tap, raw_finalize, mul_ct_ct, add_ct_ct in
WINDOW_ORDER), and every residue of every output must match."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2_pair():
    from oracle.ckks_oracle import OracleBackend
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images

    cfg = CONFIGS["cfg2"]
    dev = B200Backend(cfg.params(), cfg.base_extra_bits)
    ora = OracleBackend(cfg.params(), cfg.base_extra_bits)
    dk, ok = dev.keygen(), ora.keygen()
    dev.set_eval_key(dk)
    ora.set_eval_key(ok)
    net = NETWORKS["cfg2"]()
    enc = layers.encrypt_network(dev, net, dk)
    x = layers.encrypt_images(dev, cnn_images(dev.slots, IMAGE_SEEDS["cfg2"]), dk)
    return dev, ora, net, enc, x


def host_rows(batch):
    """(count, 2, k, N) uint64 residues of a device batch (one copy)."""
    return batch.buf[:, :, : batch.k].cpu().numpy().view(np.uint64)


def oracle_cts(ora, batch):
    from oracle.ckks_oracle import _Cipher

    rows = host_rows(batch)
    return [ora._cipher(_Cipher(r[0].copy(), r[1].copy()), batch.level, batch.scale, batch.noise_bits) for r in rows]


def assert_batch_equals(batch, cts, what):
    rows = host_rows(batch)
    assert len(cts) == rows.shape[0]
    bad = [i for i, ct in enumerate(cts)
           if not (np.array_equal(rows[i, 0], ct.payload.c0) and np.array_equal(rows[i, 1], ct.payload.c1))]
    assert not bad, f"{what}: {len(bad)} of {len(cts)} ciphertexts differ (first {bad[:5]})"


def test_cfg2_whole_network_bit_exact_vs_oracle(cfg2_pair):
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.model import WINDOW_ORDER

    dev, ora, net, enc, x = cfg2_pair
    ev = layers.LayerEvaluator(dev)
    conv, dense = net.layers[0], net.layers[4]
    y, dims = ev.conv(x, (1, 28, 28), conv, enc.weights[0], enc.biases[0])
    sq = ev.square(y)
    pooled, pdims = ev.sum_pool(sq, dims)
    F, m, n = dims
    _, pm, pn = pdims
    fi, fj, fc = np.meshgrid(np.arange(pm), np.arange(pn), np.arange(F), indexing="ij")
    flat = (fc * (pm * pn) + fi * pn + fj).ravel()
    logits = ev.dense(pooled, flat, dense, enc.weights[4], enc.biases[4])

    # conv: every cell = sum over the 25 taps of raw products, one raw_finalize
    xs, ws = oracle_cts(ora, x), oracle_cts(ora, enc.weights[0])
    s, (P, Q) = conv.stride, conv.kernel
    cells = []
    for f in range(F):
        for i in range(m):
            for j in range(n):
                raw = None
                for p in range(P):
                    for q in range(Q):
                        t = ora.mul_ct_ct_raw(xs[(i * s + p) * 28 + (j * s + q)], ws[(f * P + p) * Q + q])
                        raw = t if raw is None else ora.raw_add(raw, t)
                cells.append(ora.raw_finalize(raw))
    assert_batch_equals(y, cells, "conv layer")

    # x^2 of every device conv output
    ys = oracle_cts(ora, y)
    assert_batch_equals(sq, [ora.mul_ct_ct(c, c) for c in ys], "square layer")

    # 2x2 sum pool in the reference's WINDOW_ORDER
    sqs = oracle_cts(ora, sq)
    pools = []
    for c in range(F):
        for i in range(pm):
            for j in range(pn):
                acc = None
                for di, dj in WINDOW_ORDER:
                    t = sqs[c * m * n + (2 * i + di) * n + (2 * j + dj)]
                    acc = t if acc is None else ora.add_ct_ct(acc, t)
                pools.append(acc)
    assert_batch_equals(pooled, pools, "sum-pool layer")

    # FC: every class over the 180 flattened pooled inputs
    ps, fw = oracle_cts(ora, pooled), oracle_cts(ora, enc.weights[4])
    outs = []
    for cls in range(dense.out_dim):
        raw = None
        for r, src in enumerate(flat):
            t = ora.mul_ct_ct_raw(ps[int(src)], fw[r * dense.out_dim + cls])
            raw = t if raw is None else ora.raw_add(raw, t)
        outs.append(ora.raw_finalize(raw))
    assert_batch_equals(logits, outs, "FC layer")
