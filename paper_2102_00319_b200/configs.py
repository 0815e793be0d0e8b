"""BASELINE.json configurations expressed in the reference's parameters.

SURVEY.md Appendix B / §8d: each config is an (m, L, r) triple, the chain's
``BASE_EXTRA_BITS`` and seeded synthetic inputs (there is no public dataset:
MNIST is named only by the paper and is absent, so uniform [0,1] pixels and
Gaussian weights of the configs' shapes stand in).

* cfg1  N=4096, 50-bit base + 2x40-bit levels, 50-bit special: primitive
        microbench over 256 seeded ciphertext pairs;
* cfg2  N=8192, 60 + 5x40: conv 5x5x5 s2 -> x^2 -> sumpool -> FC 180->10,
        4096 images;
* cfg3  N=16384, 60 + 6x40: same net with the polynomial activation
        0.125x^2 + 0.5x + 0.25, 8192 images;
* cfg4  N=32768, 60 + 19x40 (+60 special): conv1 5x5x5 s2 -> x^2 -> conv2
        10 filters 3x3 over 5 channels -> x^2 -> sumpool -> FC 250->10,
        16384 images.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import Conv, Dense, Flatten, Network, PolyAct, SumPool, Square
from .params import HEParams, derive_params


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    modulus_bits: int
    precision_bits: int
    base_extra_bits: int
    key_seed: int = 1

    def params(self) -> HEParams:
        import warnings
        from .params import NoMultiplicationWarning

        with warnings.catch_warnings():
            warnings.simplefilter("ignore", NoMultiplicationWarning)
            return derive_params(self.m, self.modulus_bits, self.precision_bits, seed=self.key_seed)


CFG1 = Config("cfg1", 8192, 130, 40, 10)
CFG2 = Config("cfg2", 16384, 260, 40, 20)
CFG3 = Config("cfg3", 32768, 300, 40, 20)
CFG4 = Config("cfg4", 65536, 820, 40, 20)
CONFIGS = {c.name: c for c in (CFG1, CFG2, CFG3, CFG4)}


def cfg1_pairs(slots: int, count: int = 256, seed: int = 101):
    """256 seeded pairs x_i, y_i ~ U[-1, 1]^slots; entropies i and 256+i."""
    rng = np.random.default_rng(seed)
    xs = rng.uniform(-1.0, 1.0, (count, slots))
    ys = rng.uniform(-1.0, 1.0, (count, slots))
    return xs, ys


def cnn_small_conv_net(seed: int = 7, sigma: float = 0.1, act: str = "square") -> Network:
    """Config 2 (act='square') / config 3 (act='poly') network on 28x28 inputs."""
    rng = np.random.default_rng(seed)
    conv = Conv(weights=rng.normal(0.0, sigma, (5, 1, 5, 5)), stride=2)
    dense = Dense(weights=rng.normal(0.0, sigma, (180, 10)))
    mid = Square() if act == "square" else PolyAct(a0=0.25, a1=0.5, a2=0.125, input_scale=1.0, pool_divisor=1.0)
    return Network((28, 28), (conv, mid, SumPool(), Flatten(), dense))


def cnn_deep_net(seed: int = 7, sigma: float = 0.05) -> Network:
    """Config 4 network on 28x28 inputs."""
    rng = np.random.default_rng(seed)
    conv1 = Conv(weights=rng.normal(0.0, sigma, (5, 1, 5, 5)), stride=2)
    conv2 = Conv(weights=rng.normal(0.0, sigma, (10, 5, 3, 3)), stride=1)
    dense = Dense(weights=rng.normal(0.0, sigma, (250, 10)))
    return Network((28, 28), (conv1, Square(), conv2, Square(), SumPool(), Flatten(), dense))


def cnn_images(batch: int, seed: int, dims=(28, 28)) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, (batch, *dims))


NETWORKS = {
    "cfg2": lambda: cnn_small_conv_net(7, 0.1, "square"),
    "cfg3": lambda: cnn_small_conv_net(7, 0.1, "poly"),
    "cfg4": lambda: cnn_deep_net(7, 0.05),
}
IMAGE_SEEDS = {"cfg2": 201, "cfg3": 301, "cfg4": 401}
BATCH = {"cfg2": 4096, "cfg3": 8192, "cfg4": 16384}
