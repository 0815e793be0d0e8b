"""Wire format for host <-> device transport (csrc/packing.cu): bit-exact against a
numpy restatement, lossless round trip, and the packed serving path."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import S128, s128_params


def np_pack(rows: np.ndarray, primes) -> np.ndarray:
    """Reference packer: (blocks, k, N) residues -> (blocks, words) at bitlen(p_r) bits."""
    blocks, k, n = rows.shape
    out = []
    for blk in range(blocks):
        words = []
        for r in range(k):
            b = int(primes[r]).bit_length()
            acc = 0
            for i, v in enumerate(rows[blk, r].tolist()):
                acc |= int(v) << (i * b)
            nw = (n * b + 63) // 64
            words.extend((acc >> (64 * w)) & ((1 << 64) - 1) for w in range(nw))
        out.append(words)
    return np.array(out, dtype=np.uint64)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 3, 6])
def test_pack_matches_numpy_and_round_trips(k):
    import torch

    from paper_2102_00319_b200.backend import B200Backend, CipherBatch
    from paper_2102_00319_b200.params import derive_params

    be = B200Backend(derive_params(512, 300, 40, seed=3), 20)  # N = 256, 60-bit base, 40-bit levels
    ch = be.chain
    k = min(k, ch.num_levels + 1)
    rng = np.random.default_rng(k)
    rows = np.stack([np.stack([rng.integers(0, int(q), be.n, dtype=np.uint64) for q in ch.p[:k]])
                     for _ in range(6)]).reshape(3, 2, k, be.n)
    dev = torch.from_numpy(rows.view(np.int64)).cuda()
    packed = be.pack_batch(CipherBatch(dev, k - 1, 1))
    want = np_pack(rows.reshape(6, k, be.n), ch.p)
    assert packed.numel() == want.size
    assert np.array_equal(packed.cpu().numpy().view(np.uint64), want.ravel())
    back = torch.zeros_like(dev)
    be.unpack_into(packed, back, k)
    assert torch.equal(back, dev)


@pytest.mark.gpu
def test_packed_serving_path_matches(golden):
    import torch

    from nets import mini_networks
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend

    be = B200Backend(s128_params(), S128["extra"])
    keys = be.keygen()
    be.set_eval_key(keys)
    net = mini_networks()["mini2"]
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, imgs, keys)
    ev = layers.LayerEvaluator(be)
    out = ev.run(enc, x)
    want = out.buf[:, :, : out.k].clone()
    host = [be.pack_batch(x).cpu().pin_memory() for _ in range(3)]
    outs = [torch.empty((want.shape[0], 2, out.k, be.n), dtype=torch.int64).pin_memory() for _ in range(3)]
    ev.run_stream(enc, host, x.level, x.scale, x.noise_bits, outs, pipelines=2, unpacked_shape=tuple(x.buf.shape))
    torch.cuda.synchronize()
    assert all(torch.equal(o, want.cpu()) for o in outs)
