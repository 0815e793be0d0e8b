"""Cells-mode sharding on the device: each rank's batched shard evaluation
(LayerEvaluator.run_cells_shard) summed with finish_cells must reproduce the
single-device logits bit for bit.  Ranks are evaluated one after another on the
one GPU available (no kernel waits on another rank, so this is a faithful
stand-in for the multi-GPU run; the collective itself is covered by the gloo test)."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def shard_logits(be, keys, net, imgs, world):
    import torch

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200 import sharding as sh

    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, imgs, keys)
    ev = layers.LayerEvaluator(be)
    lay = sh.CellsLayout.of(net)
    parts, meta = [], None
    for units in sh.plan_units(lay.filters, lay.pool_rows, world):
        raw, lvl, scale, noise = ev.run_cells_shard(enc, x, units)
        parts.append(raw)
        meta = (lvl, scale, noise)
    out = ev.finish_cells(enc, torch.stack(parts), *meta)
    full = ev.run(enc, x)
    return out, full


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["mini2", "mini3"])
def test_cells_shards_match_reference(golden, name, world):
    from conftest import S128, s128_params
    from nets import mini_networks
    from paper_2102_00319_b200.backend import B200Backend

    be = B200Backend(s128_params(), S128["extra"])
    keys = be.keygen()
    be.set_eval_key(keys)
    net = mini_networks()[name]
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
    out, full = shard_logits(be, keys, net, imgs, world)
    digests = [digest(np.concatenate(be.cipher_rows_host(be.batch_to_cipher(out, i)))) for i in range(out.count)]
    assert digests == golden["minis"][name]["logit_digests"]
    assert out.level == full.level and out.scale == full.scale


def test_cfg2_eight_shards_bit_identical_to_one_device():
    import torch

    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS, NETWORKS, cnn_images

    cfg = CONFIGS["cfg2"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    out, full = shard_logits(be, keys, NETWORKS["cfg2"](), cnn_images(256, 201), 8)
    assert torch.equal(out.buf[:, :, : out.k], full.buf[:, :, : full.k])


def band_logits(be, keys, net, imgs, parts):
    import torch

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200 import sharding as sh

    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, imgs, keys)
    ev = layers.LayerEvaluator(be)
    lay = sh.BandLayout.of(net)
    raws, meta = [], None
    for band in sh.plan_bands(lay.rows2, parts):
        raw, lvl, scale, noise = ev.run_band_shard(enc, x, band)
        raws.append(raw)
        meta = (lvl, scale, noise)
    return ev.finish_cells(enc, torch.stack(raws), *meta), ev.run(enc, x)


@pytest.mark.parametrize("parts", [2, 3])
def test_band_shards_two_conv_match_reference(golden, parts):
    """mini4 (conv -> x^2 -> conv over 2 channels -> x^2 -> pool -> FC) split into conv2 row
    bands (3 bands cut pool windows): the reference's own logit digests."""
    from conftest import S128, s128_params
    from nets import mini_networks
    from paper_2102_00319_b200.backend import B200Backend

    be = B200Backend(s128_params(), S128["extra"])
    keys = be.keygen()
    be.set_eval_key(keys)
    imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))
    out, full = band_logits(be, keys, mini_networks()["mini4"], imgs, parts)
    digests = [digest(np.concatenate(be.cipher_rows_host(be.batch_to_cipher(out, i)))) for i in range(out.count)]
    assert digests == golden["minis"]["mini4"]["logit_digests"]
    assert out.level == full.level and out.scale == full.scale


@pytest.mark.parametrize("parts", [2, 3])
def test_cfg4_band_shards_bit_identical_to_one_device(parts):
    """Config 4 (N = 32768, the config-5 network) split into 2 / 3 bands with conv1 / x^2
    halo recompute: the summed partials finalise to the single-device logits bit for bit."""
    import torch

    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS, NETWORKS, cnn_images

    cfg = CONFIGS["cfg4"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    out, full = band_logits(be, keys, NETWORKS["cfg4"](), cnn_images(256, 401), parts)
    assert torch.equal(out.buf[:, :, : out.k], full.buf[:, :, : full.k])
