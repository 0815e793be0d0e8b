"""Small test networks shared by the golden generator and the parity tests."""

import numpy as np

from paper_2102_00319_b200.model import Conv, Dense, Flatten, Network, PolyAct, SumPool, Square


def mini_networks():
    rng = np.random.default_rng(11)
    mini2 = Network((10, 10), (
        Conv(weights=rng.normal(0, 0.3, (2, 1, 4, 4)), stride=2, bias=rng.normal(0, 0.1, 2)),
        Square(), SumPool(), Flatten(),
        Dense(weights=rng.normal(0, 0.3, (8, 3)), bias=rng.normal(0, 0.1, 3)),
    ))
    mini3 = Network((10, 10), (
        Conv(weights=rng.normal(0, 0.3, (2, 1, 4, 4)), stride=2),
        PolyAct(a0=0.25, a1=0.5, a2=0.125), SumPool(), Flatten(),
        Dense(weights=rng.normal(0, 0.3, (8, 3))),
    ))
    mini4 = Network((12, 12), (
        Conv(weights=rng.normal(0, 0.3, (2, 1, 4, 4)), stride=2),
        Square(),
        Conv(weights=rng.normal(0, 0.3, (3, 2, 2, 2)), stride=1),
        Square(), SumPool(), Flatten(),
        Dense(weights=rng.normal(0, 0.3, (12, 3))),
    ))
    return {"mini2": mini2, "mini3": mini3, "mini4": mini4}
