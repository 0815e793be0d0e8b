"""Bit-exact parity at full BASELINE sizes -- config 2 (the bench's workload: N = 8192,
4096 images per batch) and config 3 (N = 16384, 8192 images, polynomial activation):
the WHOLE network, every output ciphertext of every layer, against the CPU oracle.

The batched device layers (heb_conv / heb_square / heb_poly_act / heb_sumpool / heb_fc)
run over the network; the oracle (a restatement of the reference kernels) recomputes each
layer from the SAME device input ciphertexts of that layer with the reference op
sequence (mul_ct_ct_raw + raw_add per tap, raw_finalize, mul_ct_ct, add_ct_ct in
WINDOW_ORDER), and every residue of every output must match."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def make_pair(name):
    from oracle.ckks_oracle import OracleBackend
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images

    cfg = CONFIGS[name]
    dev = B200Backend(cfg.params(), cfg.base_extra_bits)
    ora = OracleBackend(cfg.params(), cfg.base_extra_bits)
    dk, ok = dev.keygen(), ora.keygen()
    dev.set_eval_key(dk)
    ora.set_eval_key(ok)
    net = NETWORKS[name]()
    enc = layers.encrypt_network(dev, net, dk)
    x = layers.encrypt_images(dev, cnn_images(dev.slots, IMAGE_SEEDS[name]), dk)
    return dev, ora, net, enc, x


def host_rows(batch):
    """(count, 2, k, N) uint64 residues of a device batch (one copy)."""
    return batch.buf[:, :, : batch.k].cpu().numpy().view(np.uint64)


def oracle_cts(ora, batch):
    from oracle.ckks_oracle import _Cipher

    rows = host_rows(batch)
    return [ora._cipher(_Cipher(r[0].copy(), r[1].copy()), batch.level, batch.scale, batch.noise_bits) for r in rows]


def assert_batch_equals(batch, cts, what, picks=None):
    """cts[t] must equal device item picks[t] (default: every item, in order)."""
    rows = host_rows(batch)
    picks = list(range(rows.shape[0])) if picks is None else picks
    assert len(cts) == len(picks)
    bad = [i for i, ct in zip(picks, cts)
           if not (np.array_equal(rows[i, 0], ct.payload.c0) and np.array_equal(rows[i, 1], ct.payload.c1))]
    assert not bad, f"{what}: {len(bad)} of {len(cts)} ciphertexts differ (first {bad[:5]})"


def pick(count, sample):
    """All outputs, or `sample` evenly spread ones (first and last included)."""
    if sample is None or sample >= count:
        return list(range(count))
    return sorted(set(np.linspace(0, count - 1, sample).round().astype(int).tolist()))


@pytest.mark.parametrize("name,sample", [("cfg2", None), ("cfg3", None), ("cfg4", 6)])
def test_whole_network_bit_exact_vs_oracle(name, sample):
    """cfg2: conv -> x^2 -> sum-pool -> FC at N = 8192; cfg3: conv -> 0.125x^2+0.5x+0.25
    -> sum-pool -> FC at N = 16384 (the extra ct x pt + rescale level): every output.
    cfg4: conv -> x^2 -> conv(5 channels) -> x^2 -> sum-pool -> FC at N = 32768 with 20
    rows (2-CTA cluster transforms): an oracle relinearisation there takes ~1 s, so
    `sample` evenly spread outputs of every layer (each layer fed the device's full
    output of the previous one)."""
    from paper_2102_00319_b200 import layers, percell
    from paper_2102_00319_b200.model import WINDOW_ORDER, Conv, Dense, Flatten, PolyAct, Square, SumPool

    dev, ora, net, enc, x = make_pair(name)
    ev = layers.LayerEvaluator(dev)
    dims = (1, *net.input_dims)
    flat = None
    for li, layer in enumerate(net.layers):
        C, m, n = dims
        if isinstance(layer, Conv):
            y, dims = ev.conv(x, dims, layer, enc.weights[li], enc.biases[li])
            xs, ws = oracle_cts(ora, x), oracle_cts(ora, enc.weights[li])
            s, (P, Q) = layer.stride, layer.kernel
            F, om, on = dims
            cells, picks = [], pick(F * om * on, sample)
            for o in picks:
                f, i, j = o // (om * on), (o // on) % om, o % on
                raw = None
                for c in range(C):
                    for p in range(P):
                        for q in range(Q):
                            t = ora.mul_ct_ct_raw(xs[c * m * n + (i * s + p) * n + (j * s + q)],
                                                  ws[((f * C + c) * P + p) * Q + q])
                            raw = t if raw is None else ora.raw_add(raw, t)
                cells.append(ora.raw_finalize(raw))
            assert_batch_equals(y, cells, f"{name} conv layer {li}", picks)
        elif isinstance(layer, Square):
            y = ev.square(x)
            xs, picks = oracle_cts(ora, x), pick(x.count, sample)
            assert_batch_equals(y, [ora.mul_ct_ct(xs[o], xs[o]) for o in picks], f"{name} square layer {li}", picks)
        elif isinstance(layer, PolyAct):
            y = ev.poly_act(x, layer)
            pts = percell.act_plaintexts(ora, layer, x.level, x.scale)
            xs, picks = oracle_cts(ora, x), pick(x.count, sample)
            assert_batch_equals(y, [percell.poly_act_cell(ora, xs[o], *pts) for o in picks],
                                f"{name} polynomial activation layer {li}", picks)
        elif isinstance(layer, SumPool):
            y, dims = ev.sum_pool(x, dims)
            xs = oracle_cts(ora, x)
            _, pm, pn = dims
            pools = []
            for c in range(C):
                for i in range(pm):
                    for j in range(pn):
                        acc = None
                        for di, dj in WINDOW_ORDER:
                            t = xs[c * m * n + (2 * i + di) * n + (2 * j + dj)]
                            acc = t if acc is None else ora.add_ct_ct(acc, t)
                        pools.append(acc)
            assert_batch_equals(y, pools, f"{name} sum-pool layer {li}")
        elif isinstance(layer, Flatten):
            fi, fj, fc = np.meshgrid(np.arange(m), np.arange(n), np.arange(C), indexing="ij")
            flat = (fc * (m * n) + fi * n + fj).ravel()
            continue
        elif isinstance(layer, Dense):
            y = ev.dense(x, flat, layer, enc.weights[li], enc.biases[li])
            xs, fw = oracle_cts(ora, x), oracle_cts(ora, enc.weights[li])
            outs, picks = [], pick(layer.out_dim, None if sample is None else 2)
            for cls in picks:
                raw = None
                for r, src in enumerate(flat):
                    t = ora.mul_ct_ct_raw(xs[int(src)], fw[r * layer.out_dim + cls])
                    raw = t if raw is None else ora.raw_add(raw, t)
                outs.append(ora.raw_finalize(raw))
            assert_batch_equals(y, outs, f"{name} FC layer {li}", picks)
        x = y
