"""End-to-end encrypted CNN for the BASELINE configs 2-4 on the device.

Bit-exactness of every op is covered by test_gpu_parity.py (including N = 32768 split
rows); here the full networks run through the batched layer evaluator at their
real ring sizes and the decrypted logits are checked against the float64 plaintext
forward pass with the north-star tolerance (1e-3 absolute, identical argmax)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_config(name, images):
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import CONFIGS, NETWORKS, IMAGE_SEEDS, cnn_images
    from paper_2102_00319_b200.model import plaintext_forward

    cfg = CONFIGS[name]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    net = NETWORKS[name]()
    enc = layers.encrypt_network(be, net, keys)
    imgs = cnn_images(images, IMAGE_SEEDS[name])
    x = layers.encrypt_images(be, imgs, keys)
    out = layers.LayerEvaluator(be).run(enc, x)
    dec = be.decrypt_batch(out, keys)[:, :images].T
    ref = plaintext_forward(net, imgs)
    return out, dec, ref, enc


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_config_logits_match_plaintext(name):
    out, dec, ref, enc = run_config(name, 128)
    assert out.level == enc.trace[-1]["level"] and out.scale == enc.trace[-1]["scale"]
    assert np.max(np.abs(dec - ref)) < 1e-3
    assert np.array_equal(np.argmax(dec, 1), np.argmax(ref, 1))


def test_config4_deep_network_logits_match_plaintext():
    """Config 4: N = 32768, 19 levels, two convolutions (5 channels in conv2)."""
    out, dec, ref, enc = run_config("cfg4", 64)
    assert out.level == enc.trace[-1]["level"]
    assert np.max(np.abs(dec - ref)) < 1e-3
    assert np.array_equal(np.argmax(dec, 1), np.argmax(ref, 1))
