"""Probe: throughput of 1 vs 2 vs 3 concurrent inference pipelines (streams) on cfg2."""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_00319_b200 import layers  # noqa: E402
from paper_2102_00319_b200.backend import B200Backend  # noqa: E402
from paper_2102_00319_b200.configs import CONFIGS, NETWORKS, cnn_images  # noqa: E402


def main():
    cfg = CONFIGS["cfg2"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen()
    be.set_eval_key(keys)
    net = NETWORKS["cfg2"]()
    enc = layers.encrypt_network(be, net, keys)
    x = layers.encrypt_images(be, cnn_images(4096, 201), keys)
    ev = layers.LayerEvaluator(be)
    for _ in range(3):
        ev.run(enc, x)
    torch.cuda.synchronize()
    steps = 12
    for nstreams in (1, 2, 3):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(steps):
            with torch.cuda.stream(streams[s % nstreams]):
                ev.run(enc, x)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"streams={nstreams}: {steps * 4096 / dt:,.0f} img/s  ({dt / steps * 1e3:.2f} ms/batch)")


if __name__ == "__main__":
    main()
