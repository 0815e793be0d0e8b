"""Per-ciphertext layer evaluator over the *reference* backend API.

Every function here only calls the public ``HEBackend`` ops
(`/root/reference/pkg/src/hecnn/backends/base.py:283-502`): ``encrypt``,
``encode_plain``, ``mul_ct_ct_raw``, ``raw_add``, ``raw_finalize``,
``mul_ct_ct``, ``mul_ct_pt``, ``add_ct_ct``, ``add_ct_pt``,
``drop_to_level``.  It therefore runs unchanged on the reference
``CkksBackend`` (to compose the BASELINE configs' op sequence from reference
calls) and on this package's ``B200Backend``
(one launch per op).  The batched device evaluator in ``layers.py`` must
produce bit-identical ciphertexts to this sequence.

Op order mirrors the reference layers (`layers.py:92-294`): conv taps in
ascending (channel, p, q), one finalize per cell, then the bias add; pool in
``WINDOW_ORDER``; dense terms in ascending input index.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .errors import DepthExhausted
from .model import WINDOW_ORDER, Conv, Dense, Flatten, Network, PolyAct, SumPool, Square, ledger, weight_entropies, BIAS_ENTROPY_BASE


@dataclass
class EncryptedNetwork:
    net: Network
    weights: list          # per layer: nested lists of CipherVec (or None)
    biases: list           # per layer: list of CipherVec (or None)
    trace: list


def encrypt_network(backend, net: Network, key) -> EncryptedNetwork:
    """Model-owner flow (reference `model.py:446-512`, extended topology).

    Weights are broadcast-encrypted with deterministic entropy tags and
    dropped to the level of their use site; biases are encrypted at the exact
    ledger scale of the layer output and dropped to its level.
    """
    trace = ledger(net, backend.chain, backend.canonical_scale)
    tags = weight_entropies(net)
    slots = backend.slots
    weights, biases = [], []
    bias_tag = BIAS_ENTROPY_BASE

    def enc(value, entropy, level, scale=None):
        ct = backend.encrypt(np.full(slots, float(value)), key, scale=scale, entropy=int(entropy))
        return backend.drop_to_level(ct, level)

    for li, layer in enumerate(net.layers):
        in_level = trace[li]["level"]
        out = trace[li + 1]
        if isinstance(layer, (Conv, Dense)):
            w = layer.weights
            flat = [enc(v, t, in_level) for v, t in zip(w.ravel(), tags[li].ravel())]
            weights.append(np.array(flat, dtype=object).reshape(w.shape))
            if layer.bias is not None:
                bl = [enc(b, bias_tag + r, out["level"], out["scale"]) for r, b in enumerate(layer.bias)]
                bias_tag += len(bl)
                biases.append(bl)
            else:
                biases.append(None)
        else:
            weights.append(None)
            biases.append(None)
    return EncryptedNetwork(net=net, weights=weights, biases=biases, trace=trace)


def encrypt_images(backend, images: np.ndarray, key) -> list:
    """Client packing (reference `packing.py:85-113`): one ciphertext per pixel,
    slot b = image b, entropy = row-major cell index.  Returns [1][m][n]."""
    imgs = np.asarray(images, dtype=np.float64)
    _, m, n = imgs.shape
    grid = [[backend.encrypt(imgs[:, i, j], key, entropy=i * n + j) for j in range(n)] for i in range(m)]
    return [grid]


def act_plaintexts(backend, act: PolyAct, level: int, scale: Fraction):
    """Reference `layers.py:139-161`: encode c2, c1, c0 at the scales that land
    both activation paths on the canonical scale exactly."""
    if level < 2:
        raise DepthExhausted(f"activation needs level >= 2, ciphertext at {level}")
    c0, c1, c2 = act.folded()
    canon = backend.canonical_scale
    p1 = backend.chain.level_primes[level - 1]
    p2 = backend.chain.level_primes[level - 2]
    slots = backend.slots
    pt_quad = backend.encode_plain(np.full(slots, c2), scale=canon * p1 * p2 / (scale * scale), level=level - 1)
    pt_lin = backend.encode_plain(np.full(slots, c1), scale=canon * p1 / scale, level=level)
    pt_const = backend.encode_plain(np.full(slots, c0), scale=canon, level=level - 2)
    return pt_quad, pt_lin, pt_const


def poly_act_cell(backend, y, pt_quad, pt_lin, pt_const):
    """Reference `approx_relu_cell` (`layers.py:164-174`)."""
    t = backend.mul_ct_ct(y, y)
    quad = backend.mul_ct_pt(t, pt_quad)
    lin = backend.mul_ct_pt(y, pt_lin)
    return backend.add_ct_pt(backend.add_ct_ct(quad, lin), pt_const)


def run_network(backend, enc: EncryptedNetwork, maps: list, deltas: list | None = None) -> list:
    """Evaluate the encrypted network op by op; returns the logit ciphertexts.
    ``deltas`` (optional) receives (layer kind, counter delta) per layer."""
    net = enc.net
    flat = None
    for li, layer in enumerate(net.layers):
        before = backend.counters.snapshot() if deltas is not None else None
        if isinstance(layer, Conv):
            w = enc.weights[li]
            p, q = layer.kernel
            s = layer.stride
            m, n = len(maps[0]), len(maps[0][0])
            om, on = layer.out_dims(m, n)
            new = []
            for f in range(layer.filters):
                rows = []
                for i in range(om):
                    row = []
                    for j in range(on):
                        acc = None
                        for c in range(layer.channels):
                            for dp in range(p):
                                for dq in range(q):
                                    t = backend.mul_ct_ct_raw(maps[c][i * s + dp][j * s + dq], w[f, c, dp, dq])
                                    acc = t if acc is None else backend.raw_add(acc, t)
                        cell = backend.raw_finalize(acc)
                        if enc.biases[li] is not None:
                            cell = backend.add_ct_ct(cell, enc.biases[li][f])
                        row.append(cell)
                    rows.append(row)
                new.append(rows)
            maps = new
        elif isinstance(layer, Square):
            maps = [[[backend.mul_ct_ct(c, c) for c in row] for row in fm] for fm in maps]
        elif isinstance(layer, PolyAct):
            first = maps[0][0][0]
            pts = act_plaintexts(backend, layer, first.level, first.scale)
            maps = [[[poly_act_cell(backend, c, *pts) for c in row] for row in fm] for fm in maps]
        elif isinstance(layer, SumPool):
            new = []
            for fm in maps:
                m, n = len(fm), len(fm[0])
                rows = []
                for i in range(m // 2):
                    row = []
                    for j in range(n // 2):
                        acc = None
                        for di, dj in WINDOW_ORDER:
                            cell = fm[2 * i + di][2 * j + dj]
                            acc = cell if acc is None else backend.add_ct_ct(acc, cell)
                        row.append(acc)
                    rows.append(row)
                new.append(rows)
            maps = new
        elif isinstance(layer, Flatten):
            nf = len(maps)
            im, jm = len(maps[0]), len(maps[0][0])
            flat = [None] * (im * jm * nf)
            for i in range(im):
                for j in range(jm):
                    for c in range(nf):
                        flat[(i * jm + j) * nf + c] = maps[c][i][j]
        elif isinstance(layer, Dense):
            w = enc.weights[li]
            out = []
            for r in range(layer.out_dim):
                acc = backend.mul_ct_ct_raw(flat[0], w[0, r])
                for i in range(1, layer.in_dim):
                    acc = backend.raw_add(acc, backend.mul_ct_ct_raw(flat[i], w[i, r]))
                cell = backend.raw_finalize(acc)
                if enc.biases[li] is not None:
                    cell = backend.add_ct_ct(cell, enc.biases[li][r])
                out.append(cell)
            flat = out
        if deltas is not None:
            deltas.append((layer.kind, backend.counters.snapshot() - before))
    return flat
