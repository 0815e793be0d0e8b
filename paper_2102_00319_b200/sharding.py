"""Multi-GPU sharding of the encrypted-CNN path.

Every ciphertext op of the path is independent, so the work shards without any
data-path exchange except the final logits:

* ``batches`` mode -- each rank evaluates its own seeded image batch with replicated
  keys and weights (weak scaling); only the logit ciphertexts are gathered.  This is
  what ``bench.py`` runs under torchrun.
* ``cells`` mode -- one batch split over ranks by *units* = (filter, pool row) of the
  first conv -> activation -> 2x2 pool block (the reference's filter x band split,
  `executor.py:86-112,212-229`, without halos because pool windows never straddle a
  unit).  Each rank forms the FC layer's degree-2 partial sums over its own pooled
  cells (`dense_column_partial`, `layers.py:248-259`); the partials are gathered and
  added mod p -- exact, so the result is bit-identical to one device
  (`base.py:144-153`) -- and finalised once (`dense_combine`, `layers.py:262-272`).

* ``bands`` mode -- for two-convolution networks (config 4 / config 5: conv1 -> act ->
  conv2 -> act -> pool -> flatten -> dense) one batch is split over ranks by contiguous
  bands of conv2 output rows (the reference's horizontal band split with a (P-1)-row
  overlap, `executor.py:86-112`): each rank recomputes the conv1 / act rows
  its band reads (the halo) and its conv2 / act cells, sums its cells of every pool window
  it touches (a window cut by a band boundary is summed partially on both ranks), and
  forms the FC layer's degree-2 partial sums over those window sums.  Tensor products are
  bilinear and raw additions exact mod p, so the gathered, summed partials equal the
  single-device accumulation bit for bit.

The collectives are plain ``torch.distributed`` calls on int64-typed tensors
(NCCL over NVLink on B200 ranks, gloo in the CPU tests); the modular sum of the
gathered partials runs on the device (``heb_sum_gather``) or through the backend's
``raw_add``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import WINDOW_ORDER, Conv, Dense, Flatten, Network, PolyAct, SumPool, Square


@dataclass(frozen=True)
class CellsLayout:
    """Shape facts of a conv -> act -> pool -> flatten -> dense network."""

    filters: int
    conv_rows: int      # om
    conv_cols: int      # on
    pool_rows: int
    pool_cols: int

    @classmethod
    def of(cls, net: Network) -> "CellsLayout":
        kinds = [l.kind for l in net.layers]
        if kinds[0] != "conv" or kinds[1] not in ("square", "polyact") or kinds[2] != "sumpool" \
                or kinds[3] != "flatten" or kinds[4] != "dense" or len(kinds) != 5:
            raise ValueError("cells sharding needs conv -> act -> sumpool -> flatten -> dense")
        conv: Conv = net.layers[0]
        om, on = conv.out_dims(*net.input_dims)
        return cls(conv.filters, om, on, om // 2, on // 2)


def plan_units(filters: int, pool_rows: int, world: int) -> list[list[tuple[int, int]]]:
    """Split the (filter, pool row) units into ``world`` contiguous, balanced shards."""
    units = [(f, r) for f in range(filters) for r in range(pool_rows)]
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(len(units), world)
    out, start = [], 0
    for rank in range(world):
        size = base + (1 if rank < extra else 0)
        out.append(units[start:start + size])
        start += size
    return out


def conv_cells(lay: CellsLayout, units) -> list[tuple[int, int, int]]:
    """Conv output cells (f, i, j) a shard computes: both conv rows of each pool row."""
    return [(f, 2 * r + di, j) for f, r in units for di in (0, 1) for j in range(lay.conv_cols)]


def pooled_cells(lay: CellsLayout, units) -> list[tuple[int, int, int]]:
    return [(f, r, j) for f, r in units for j in range(lay.pool_cols)]


def flat_of(lay: CellsLayout, f: int, r: int, j: int) -> int:
    """Reference flatten order flat[(i*J + j)*F + c] (`layers.py:224-241`)."""
    return (r * lay.pool_cols + j) * lay.filters + f


# ---------------------------------------------------------------------------
# per-op (reference API) shard evaluation -- runs on any HEBackend
# ---------------------------------------------------------------------------

def percell_fc_partials(backend, enc, grid, units) -> list:
    """This shard's FC raw partial per class, composed from public HEBackend ops only."""
    from .percell import act_plaintexts, poly_act_cell

    net = enc.net
    lay = CellsLayout.of(net)
    conv: Conv = net.layers[0]
    act = net.layers[1]
    dense: Dense = net.layers[4]
    p, q = conv.kernel
    s = conv.stride
    w = enc.weights[0]
    cells = {}
    for f, i, j in conv_cells(lay, units):
        acc = None
        for c in range(conv.channels):
            for dp in range(p):
                for dq in range(q):
                    t = backend.mul_ct_ct_raw(grid[c][i * s + dp][j * s + dq], w[f, c, dp, dq])
                    acc = t if acc is None else backend.raw_add(acc, t)
        y = backend.raw_finalize(acc)
        if enc.biases[0] is not None:
            y = backend.add_ct_ct(y, enc.biases[0][f])
        cells[(f, i, j)] = y
    if isinstance(act, Square):
        cells = {k: backend.mul_ct_ct(v, v) for k, v in cells.items()}
    else:
        first = next(iter(cells.values()))
        pts = act_plaintexts(backend, act, first.level, first.scale)
        cells = {k: poly_act_cell(backend, v, *pts) for k, v in cells.items()}
    pooled = {}
    for f, r, j in pooled_cells(lay, units):
        acc = None
        for di, dj in WINDOW_ORDER:
            v = cells[(f, 2 * r + di, 2 * j + dj)]
            acc = v if acc is None else backend.add_ct_ct(acc, v)
        pooled[(f, r, j)] = acc
    dw = enc.weights[4]
    order = sorted(pooled, key=lambda fr: flat_of(lay, *fr))
    parts = []
    for cls in range(dense.out_dim):
        acc = None
        for key in order:
            t = backend.mul_ct_ct_raw(pooled[key], dw[flat_of(lay, *key), cls])
            acc = t if acc is None else backend.raw_add(acc, t)
        parts.append(acc)
    return parts


@dataclass(frozen=True)
class BandLayout:
    """Shape facts of a conv -> act -> conv -> act -> sumpool -> flatten -> dense network."""

    in_rows: int
    in_cols: int
    s1: int            # conv1 stride
    p1: int            # conv1 kernel rows
    rows1: int         # conv1 output rows
    cols1: int
    p2: int            # conv2 kernel rows (stride 1)
    rows2: int         # conv2 output rows
    cols2: int
    filters2: int
    pool_cols: int

    @classmethod
    def of(cls, net: Network) -> "BandLayout":
        kinds = [l.kind for l in net.layers]
        if len(kinds) != 7 or kinds[0] != "conv" or kinds[2] != "conv" or kinds[4] != "sumpool" \
                or kinds[5] != "flatten" or kinds[6] != "dense" or kinds[1] not in ("square", "polyact") \
                or kinds[3] not in ("square", "polyact"):
            raise ValueError("band sharding needs conv -> act -> conv -> act -> sumpool -> flatten -> dense")
        c1, c2 = net.layers[0], net.layers[2]
        if c2.stride != 1:
            raise ValueError("band sharding needs a stride-1 second convolution")
        m, n = net.input_dims
        r1, k1 = c1.out_dims(m, n)
        r2, k2 = c2.out_dims(r1, k1)
        return cls(m, n, c1.stride, c1.kernel[0], r1, k1, c2.kernel[0], r2, k2, c2.filters, k2 // 2)

    def conv1_rows(self, a: int, b: int) -> tuple[int, int]:
        """conv1 output rows [a, b + p2 - 1) feed conv2 rows [a, b) (the halo)."""
        return a, b + self.p2 - 1

    def input_rows(self, a: int, b: int) -> tuple[int, int]:
        r0, r1 = self.conv1_rows(a, b)
        return r0 * self.s1, (r1 - 1) * self.s1 + self.p1

    def windows(self, a: int, b: int) -> list[tuple[int, int, int, list[tuple[int, int]]]]:
        """Pool windows (f, r, j) touched by conv2 rows [a, b), each with the conv2 cells
        (row, col) of the window this band owns, in WINDOW_ORDER."""
        out = []
        for f in range(self.filters2):
            for r in range(a // 2, (b + 1) // 2):
                for j in range(self.pool_cols):
                    cells = [(2 * r + di, 2 * j + dj) for di, dj in WINDOW_ORDER if a <= 2 * r + di < b]
                    if cells:
                        out.append((f, r, j, cells))
        return out

    def flat_of(self, f: int, r: int, j: int) -> int:
        return (r * self.pool_cols + j) * self.filters2 + f


def plan_bands(rows: int, parts: int) -> list[tuple[int, int]]:
    """``parts`` contiguous, balanced bands of conv2 output rows."""
    if parts < 1 or parts > rows:
        raise ValueError(f"cannot split {rows} rows into {parts} bands")
    return [((rows * i) // parts, (rows * (i + 1)) // parts) for i in range(parts)]


def plan_batches(batches: int, world: int) -> list[list[tuple[int, int]]]:
    """Config 5: ``batches`` independent batches over ``world`` ranks.  Returns per rank a
    list of (batch, band index) work items together with the band count per batch: ranks
    take whole batches while world <= batches, and split each batch into world / batches
    bands beyond that."""
    if world <= batches:
        if batches % world:
            raise ValueError("world must divide the batch count")
        return [[(b, 0) for b in range(r, batches, world)] for r in range(world)]
    if world % batches:
        raise ValueError("batch count must divide the world")
    per = world // batches
    return [[(r // per, r % per)] for r in range(world)]


def percell_band_partials(backend, enc, grid, band: tuple[int, int]) -> list:
    """This band's FC raw partial per class, composed from public HEBackend ops only."""
    from .percell import act_plaintexts, poly_act_cell

    net = enc.net
    lay = BandLayout.of(net)
    a, b = band
    c1, act1, c2, act2, dense = net.layers[0], net.layers[1], net.layers[2], net.layers[3], net.layers[6]

    def act(layer, cells):
        if isinstance(layer, Square):
            return {k: backend.mul_ct_ct(v, v) for k, v in cells.items()}
        first = next(iter(cells.values()))
        pts = act_plaintexts(backend, layer, first.level, first.scale)
        return {k: poly_act_cell(backend, v, *pts) for k, v in cells.items()}

    def conv(layer, w, bias, src, rows, cols):
        p, q = layer.kernel
        s = layer.stride
        out = {}
        for f in range(layer.filters):
            for i in range(*rows):
                for j in range(cols):
                    acc = None
                    for c in range(layer.channels):
                        for dp in range(p):
                            for dq in range(q):
                                t = backend.mul_ct_ct_raw(src(c, i * s + dp, j * s + dq), w[f, c, dp, dq])
                                acc = t if acc is None else backend.raw_add(acc, t)
                    y = backend.raw_finalize(acc)
                    if bias is not None:
                        y = backend.add_ct_ct(y, bias[f])
                    out[(f, i, j)] = y
        return out

    y1 = act(act1, conv(c1, enc.weights[0], enc.biases[0], lambda c, i, j: grid[c][i][j], lay.conv1_rows(a, b),
                        lay.cols1))
    y2 = act(act2, conv(c2, enc.weights[2], enc.biases[2], lambda c, i, j: y1[(c, i, j)], (a, b), lay.cols2))
    sums = {}
    for f, r, j, cells in lay.windows(a, b):
        acc = None
        for i, jj in cells:
            acc = y2[(f, i, jj)] if acc is None else backend.add_ct_ct(acc, y2[(f, i, jj)])
        sums[(f, r, j)] = acc
    order = sorted(sums, key=lambda k: lay.flat_of(*k))
    dw = enc.weights[6]
    parts = []
    for cls in range(dense.out_dim):
        acc = None
        for key in order:
            t = backend.mul_ct_ct_raw(sums[key], dw[lay.flat_of(*key), cls])
            acc = t if acc is None else backend.raw_add(acc, t)
        parts.append(acc)
    return parts


def allgather_int64(tensor, world: int):
    """All-gather an int64 tensor across ranks -> (world, *shape) (NCCL or gloo)."""
    import torch
    import torch.distributed as dist

    out = [torch.empty_like(tensor) for _ in range(world)]
    dist.all_gather(out, tensor.contiguous())
    return torch.stack(out)


def mod_sum_rows(parts: np.ndarray, primes) -> np.ndarray:
    """Exact modular sum over axis 0 of (world, ..., k, N) uint64 residues."""
    acc = parts[0].astype(np.uint64).copy()
    pr = np.asarray(primes, dtype=np.uint64)[: acc.shape[-2]].reshape((1,) * (acc.ndim - 2) + (-1, 1))
    for other in parts[1:]:
        s = acc + other.astype(np.uint64)  # canonical residues < 2^62: no overflow
        acc = np.where(s >= pr, s - pr, s)
    return acc
