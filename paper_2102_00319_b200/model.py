"""Encrypted-CNN description, level/scale ledger and plaintext oracle.

Extends the reference model layer set
(`/root/reference/pkg/src/hecnn/model.py:38-157`, `layers.py:31-84`) to the
topologies BASELINE.json configs 2-4 need:

* ``Conv``      valid cross-correlation with stride and input channels; each
  output cell is one fused inner product of raw degree-2 products, finalized
  once (relinearize + rescale), reference `layers.py:92-127`;
* ``Square``    x*x as one ct-ct multiply (config 2/4 activation);
* ``PolyAct``   the reference's degree-2 activation ``approx_relu_cell``
  (`layers.py:139-174`) with its folded coefficients and exact plaintext
  scales, optionally with the 2x2 pool divisor folded in;
* ``SumPool``   2x2 window sums in the reference ``WINDOW_ORDER``
  (`layers.py:26,189-204`);
* ``Flatten``   row-major, channel-last (`layers.py:224-241`);
* ``Dense``     fused inner product per class + optional bias
  (`layers.py:248-294`).

``ledger`` extends ``pipeline_trace`` (`model.py:165-194`) and
``plaintext_forward`` mirrors `model.py:202-277`, both for the extended set.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .errors import HecnnError, ModelValidationError

WINDOW_ORDER: tuple[tuple[int, int], ...] = ((0, 0), (1, 0), (0, 1), (1, 1))
DEFAULT_ACT_COEFFS = (0.47, 0.50, 0.09)


@dataclass(frozen=True)
class Conv:
    weights: np.ndarray            # (filters, in_channels, P, Q)
    stride: int = 1
    bias: np.ndarray | None = None  # (filters,)
    kind: str = field(default="conv", init=False)

    @property
    def filters(self) -> int:
        return self.weights.shape[0]

    @property
    def channels(self) -> int:
        return self.weights.shape[1]

    @property
    def kernel(self) -> tuple[int, int]:
        return self.weights.shape[2], self.weights.shape[3]

    def out_dims(self, m: int, n: int) -> tuple[int, int]:
        p, q = self.kernel
        if p > m or q > n:
            raise ModelValidationError(f"kernel {self.kernel} larger than input {(m, n)}")
        return (m - p) // self.stride + 1, (n - q) // self.stride + 1


@dataclass(frozen=True)
class Square:
    kind: str = field(default="square", init=False)


@dataclass(frozen=True)
class PolyAct:
    """s*g(y/s)/d with g(u) = a0 + a1 u + a2 u^2 (reference `layers.py:45-75`)."""

    a0: float = DEFAULT_ACT_COEFFS[0]
    a1: float = DEFAULT_ACT_COEFFS[1]
    a2: float = DEFAULT_ACT_COEFFS[2]
    input_scale: float = 1.0
    pool_divisor: float = 1.0
    kind: str = field(default="polyact", init=False)

    def folded(self) -> tuple[float, float, float]:
        s, d = self.input_scale, self.pool_divisor
        return (self.a0 * s / d, self.a1 / d, self.a2 / (s * d))

    def apply(self, y):
        c0, c1, c2 = self.folded()
        return ((y * y) * c2 + y * c1) + c0


@dataclass(frozen=True)
class SumPool:
    kind: str = field(default="sumpool", init=False)


@dataclass(frozen=True)
class Flatten:
    kind: str = field(default="flatten", init=False)


@dataclass(frozen=True)
class Dense:
    weights: np.ndarray            # (in_dim, out_dim)
    bias: np.ndarray | None = None
    kind: str = field(default="dense", init=False)

    @property
    def in_dim(self) -> int:
        return self.weights.shape[0]

    @property
    def out_dim(self) -> int:
        return self.weights.shape[1]


Layer = Conv | Square | PolyAct | SumPool | Flatten | Dense

# levels each layer consumes
_LEVEL_COST = {"conv": 1, "square": 1, "polyact": 2, "sumpool": 0, "flatten": 0, "dense": 1}


@dataclass(frozen=True)
class Network:
    """A validated feed-forward encrypted CNN."""

    input_dims: tuple[int, int]
    layers: tuple[Layer, ...]

    def __post_init__(self) -> None:
        object.__setattr__(self, "layers", tuple(self.layers))
        self.shapes()

    def shapes(self) -> list[tuple]:
        """(channels, m, n) after each layer, or (len,) once flattened."""
        c, (m, n) = 1, self.input_dims
        flat = None
        out = []
        for layer in self.layers:
            if isinstance(layer, Conv):
                if flat is not None:
                    raise ModelValidationError("conv after flatten")
                if layer.channels != c:
                    raise ModelValidationError(f"conv expects {layer.channels} channels, got {c}")
                if layer.bias is not None and layer.bias.shape != (layer.filters,):
                    raise ModelValidationError("conv bias shape mismatch")
                m, n = layer.out_dims(m, n)
                c = layer.filters
            elif isinstance(layer, SumPool):
                if m % 2 or n % 2:
                    raise ModelValidationError(f"2x2 pool needs even dims, got {(m, n)}")
                m, n = m // 2, n // 2
            elif isinstance(layer, Flatten):
                flat = c * m * n
            elif isinstance(layer, Dense):
                if flat is None or layer.in_dim != flat:
                    raise ModelValidationError(f"dense in_dim {layer.in_dim} != flattened length {flat}")
                flat = layer.out_dim
            out.append((flat,) if flat is not None else (c, m, n))
        for layer in self.layers:
            for arr in (getattr(layer, "weights", None), getattr(layer, "bias", None)):
                if arr is not None and not np.all(np.isfinite(arr)):
                    raise ModelValidationError(f"{layer.kind} weights contain NaN/inf")
        return out

    def depth(self) -> int:
        return sum(_LEVEL_COST[layer.kind] for layer in self.layers)


def ledger(net: Network, chain, canonical_scale: Fraction, start_level: int | None = None) -> list[dict]:
    """Per-layer (level, exact scale) of the encrypted pipeline.

    Extends the reference ``pipeline_trace`` (`model.py:165-194`): conv and
    dense rescale once (scale * canon / q_top); square rescales once
    (scale^2 / q_top); the polynomial activation consumes two levels and
    lands on the canonical scale by construction; pool/flatten are free.
    """
    level = chain.num_levels if start_level is None else start_level
    scale = canonical_scale
    steps = [{"layer": "input", "level": level, "scale": scale}]
    for layer in net.layers:
        need = _LEVEL_COST[layer.kind]
        if level < need:
            raise HecnnError(f"chain too short for the {layer.kind} layer")
        if layer.kind in ("conv", "dense"):
            scale = scale * canonical_scale / chain.level_primes[level - 1]
        elif layer.kind == "square":
            scale = scale * scale / chain.level_primes[level - 1]
        elif layer.kind == "polyact":
            scale = canonical_scale
        level -= need
        steps.append({"layer": layer.kind, "level": level, "scale": scale})
    return steps


def plaintext_forward(net: Network, images: np.ndarray) -> np.ndarray:
    """float64 oracle with the encrypted path's operation order (model.py:202-277)."""
    x = np.asarray(images, dtype=np.float64)
    if x.ndim == 2:
        x = x[None]
    maps = [x]
    flat = None
    for layer in net.layers:
        if isinstance(layer, Conv):
            p, q = layer.kernel
            s = layer.stride
            b, m, n = maps[0].shape
            om, on = layer.out_dims(m, n)
            new = []
            for f in range(layer.filters):
                fm = np.empty((b, om, on))
                for i in range(om):
                    for j in range(on):
                        acc = None
                        for c in range(layer.channels):
                            for dp in range(p):
                                for dq in range(q):
                                    t = maps[c][:, i * s + dp, j * s + dq] * layer.weights[f, c, dp, dq]
                                    acc = t if acc is None else acc + t
                        if layer.bias is not None:
                            acc = acc + layer.bias[f]
                        fm[:, i, j] = acc
                new.append(fm)
            maps = new
        elif isinstance(layer, Square):
            maps = [fm * fm for fm in maps]
        elif isinstance(layer, PolyAct):
            maps = [layer.apply(fm) for fm in maps]
        elif isinstance(layer, SumPool):
            new = []
            for fm in maps:
                b, m, n = fm.shape
                pooled = np.empty((b, m // 2, n // 2))
                for i in range(m // 2):
                    for j in range(n // 2):
                        acc = None
                        for di, dj in WINDOW_ORDER:
                            v = fm[:, 2 * i + di, 2 * j + dj]
                            acc = v.copy() if acc is None else acc + v
                        pooled[:, i, j] = acc
                new.append(pooled)
            maps = new
        elif isinstance(layer, Flatten):
            b, im, jm = maps[0].shape
            nf = len(maps)
            flat = np.empty((b, im * jm * nf))
            for i in range(im):
                for j in range(jm):
                    for c in range(nf):
                        flat[:, (i * jm + j) * nf + c] = maps[c][:, i, j]
        elif isinstance(layer, Dense):
            out = np.empty((flat.shape[0], layer.out_dim))
            for r in range(layer.out_dim):
                acc = flat[:, 0] * layer.weights[0, r]
                for i in range(1, layer.in_dim):
                    acc = acc + flat[:, i] * layer.weights[i, r]
                if layer.bias is not None:
                    acc = acc + layer.bias[r]
                out[:, r] = acc
            flat = out
    return flat if flat is not None else np.stack(maps, axis=1)


def flat_index(i: int, j: int, c: int, j_dim: int, channels: int) -> int:
    """Reference flatten order: flat[(i*J + j)*F + c] = maps[c][i][j]."""
    return (i * j_dim + j) * channels + c


# ---------------------------------------------------------------------------
# deterministic encryption entropy for model owners (weights) and clients
# ---------------------------------------------------------------------------

WEIGHT_ENTROPY_BASE = 1 << 40
BIAS_ENTROPY_BASE = 1 << 41


def weight_entropies(net: Network) -> list[np.ndarray]:
    """Per-layer entropy tags for broadcast weight encryption.

    The reference model owner encrypts weights with a process-local counter
    (`model.py:464-466`); explicit per-weight tags make every party's
    ciphertexts reproducible regardless of encryption order.
    """
    out = []
    base = WEIGHT_ENTROPY_BASE
    for layer in net.layers:
        if isinstance(layer, (Conv, Dense)):
            size = layer.weights.size
            out.append(base + np.arange(size, dtype=np.int64).reshape(layer.weights.shape))
            base += size
        else:
            out.append(None)
    return out
