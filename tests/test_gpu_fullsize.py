"""Bit-exact parity at full BASELINE sizes: the WHOLE network, every output ciphertext
of every layer, against the CPU oracle --

* config 2: N = 8192, 4096 images, conv 5x5x5 stride 2 -> x^2 -> sum-pool -> FC 180->10;
* config 3: N = 16384, 8192 images, the polynomial activation (extra ct x pt level);
* config 4 (the bench headline): N = 32768, 20 rows, 16384 images, conv1 -> x^2 ->
  conv2 (10 filters 3x3 over 5 channels) -> x^2 -> sum-pool -> FC 250->10 -- all 720 +
  720 + 1000 + 1000 + 250 outputs and all 10 classes (~3450 oracle relinearisations,
  spread over the host cores).

The batched device layers (heb_conv / heb_square / heb_poly_act / heb_sumpool / heb_fc)
run over the network; the oracle (a restatement of the reference kernels) recomputes each
layer from the SAME device input ciphertexts of that layer with the reference op
sequence (mul_ct_ct_raw + raw_add per tap, raw_finalize, mul_ct_ct, add_ct_ct in
WINDOW_ORDER), on a thread pool over all host cores (the reference's own parallel
pattern, executor.py:195-203), and every residue of every output must match."""

import os

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


def oracle_cts(ora, batch, rows=None):
    """Oracle ciphertexts viewing one host copy of a device batch (no per-item copies)."""
    from oracle.ckks_oracle import _Cipher

    rows = host_rows(batch) if rows is None else rows
    return [ora._cipher(_Cipher(r[0], r[1]), batch.level, batch.scale, batch.noise_bits) for r in rows]


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


@pytest.mark.parametrize("name,sample", [("cfg2", None), ("cfg3", None), ("cfg4", None)])
def test_whole_network_bit_exact_vs_oracle(name, sample):
    """Every output of every layer (``sample``: evenly spread outputs only, for quick runs)."""
    from oracle.ckks_oracle import threaded_map
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
            picks = pick(F * om * on, sample)

            def cell(o):
                f, i, j = o // (om * on), (o // on) % om, o % on
                raw = None
                for c in range(C):
                    for p in range(P):
                        for q in range(Q):
                            t = ora.mul_ct_ct_raw(xs[c * m * n + (i * s + p) * n + (j * s + q)],
                                                  ws[((f * C + c) * P + p) * Q + q])
                            raw = t if raw is None else ora.raw_add(raw, t)
                return ora.raw_finalize(raw)

            assert_batch_equals(y, threaded_map(cell, picks), f"{name} conv layer {li}", picks)
            del xs, ws
        elif isinstance(layer, Square):
            y = ev.square(x)
            xs, picks = oracle_cts(ora, x), pick(x.count, sample)
            assert_batch_equals(y, threaded_map(lambda o: ora.mul_ct_ct(xs[o], xs[o]), picks),
                                f"{name} square layer {li}", picks)
            del xs
        elif isinstance(layer, PolyAct):
            y = ev.poly_act(x, layer)
            pts = percell.act_plaintexts(ora, layer, x.level, x.scale)
            xs, picks = oracle_cts(ora, x), pick(x.count, sample)
            assert_batch_equals(y, threaded_map(lambda o: percell.poly_act_cell(ora, xs[o], *pts), picks),
                                f"{name} polynomial activation layer {li}", picks)
            del xs
        elif isinstance(layer, SumPool):
            y, dims = ev.sum_pool(x, dims)
            xs = oracle_cts(ora, x)
            _, pm, pn = dims

            def window(cij):
                c, i, j = cij
                acc = None
                for di, dj in WINDOW_ORDER:
                    t = xs[c * m * n + (2 * i + di) * n + (2 * j + dj)]
                    acc = t if acc is None else ora.add_ct_ct(acc, t)
                return acc

            assert_batch_equals(y, threaded_map(window, list(np.ndindex(C, pm, pn))), f"{name} sum-pool layer {li}")
            del xs
        elif isinstance(layer, Flatten):
            fi, fj, fc = np.meshgrid(np.arange(m), np.arange(n), np.arange(C), indexing="ij")
            flat = (fc * (m * n) + fi * n + fj).ravel()
            continue
        elif isinstance(layer, Dense):
            y = ev.dense(x, flat, layer, enc.weights[li], enc.biases[li])
            xs = oracle_cts(ora, x)
            w = enc.weights[li]
            dout, din = layer.out_dim, layer.in_dim
            picks = pick(dout, None if sample is None else 2)
            # one class at a time (its weight column copied once), its terms split over the
            # host cores in contiguous chunks and summed in order (executor.py:241-267)
            J = max(1, min(din, (os.cpu_count() or 1)))
            bounds = [(din * c) // J for c in range(J + 1)]
            outs = []
            for cls in picks:
                wrows = w.buf[cls::dout][:, :, : w.k].cpu().numpy().view(np.uint64)
                fw = oracle_cts(ora, w, wrows)

                def part(c):
                    raw = None
                    for r in range(bounds[c], bounds[c + 1]):
                        t = ora.mul_ct_ct_raw(xs[int(flat[r])], fw[r])
                        raw = t if raw is None else ora.raw_add(raw, t)
                    return raw

                parts = [p for p in threaded_map(part, range(J)) if p is not None]
                raw = parts[0]
                for p in parts[1:]:
                    raw = ora.raw_add(raw, p)
                outs.append(ora.raw_finalize(raw))
            assert_batch_equals(y, outs, f"{name} FC layer {li}", picks)
        x = y
