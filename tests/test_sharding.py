"""Multi-rank sharding of one encrypted batch (cells mode) -- host logic on CPU.

World-size-2 gloo processes each evaluate their (filter, pool-row) units with the
CPU oracle through the reference API, all-gather their FC raw partials, add them
mod p and finalise: the logits must equal the reference's single-process logits bit
for bit (golden digests).  The device path of the same plan is covered in
tests/test_gpu_sharding.py.
"""

import hashlib
import os
import socket
import warnings

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_00319_b200 import sharding as sh


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).astype("<u8").tobytes()).hexdigest()


def test_plan_units_cover_every_unit_once():
    for filters, rows in ((5, 6), (2, 2), (10, 5)):
        for world in (1, 2, 3, 4, 8, 16):
            plan = sh.plan_units(filters, rows, world)
            flat = [u for shard in plan for u in shard]
            assert sorted(flat) == [(f, r) for f in range(filters) for r in range(rows)]
            sizes = [len(s) for s in plan]
            assert max(sizes) - min(sizes) <= 1 and len(plan) == world


def test_cells_layout_of_baseline_networks():
    from paper_2102_00319_b200.configs import NETWORKS

    lay = sh.CellsLayout.of(NETWORKS["cfg2"]())
    assert (lay.filters, lay.conv_rows, lay.conv_cols, lay.pool_rows, lay.pool_cols) == (5, 12, 12, 6, 6)
    with pytest.raises(ValueError):
        sh.CellsLayout.of(NETWORKS["cfg4"]())  # two convolutions: bands mode
    cells = sh.conv_cells(lay, [(0, 0), (4, 5)])
    assert len(cells) == 2 * 2 * 12 and (4, 11, 11) in cells


def test_mod_sum_rows_is_exact():
    primes = [2**61 - 1, 1099511480321]
    rng = np.random.default_rng(0)
    parts = np.stack([np.stack([rng.integers(0, p, 64, dtype=np.uint64) for p in primes]) for _ in range(5)])
    got = sh.mod_sum_rows(parts, primes)
    for r, p in enumerate(primes):
        expect = [sum(int(parts[w, r, i]) for w in range(5)) % p for i in range(64)]
        assert [int(v) for v in got[r]] == expect


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out_path):
    warnings.simplefilter("ignore")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(__file__))
        from conftest import S128, s128_params
        from nets import mini_networks
        from oracle.ckks_oracle import OracleBackend, _Raw
        from paper_2102_00319_b200 import percell
        from paper_2102_00319_b200.contract import RawProduct

        be = OracleBackend(s128_params(), S128["extra"])
        keys = be.keygen()
        be.set_eval_key(keys)
        net = mini_networks()[name]
        imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))[:, : net.input_dims[0], : net.input_dims[1]]
        enc = percell.encrypt_network(be, net, keys)
        grid = percell.encrypt_images(be, imgs, keys)
        lay = sh.CellsLayout.of(net)
        units = sh.plan_units(lay.filters, lay.pool_rows, world)[rank]
        parts = sh.percell_fc_partials(be, enc, grid, units)
        local = np.stack([np.stack([p.payload.d0, p.payload.d1, p.payload.d2]) for p in parts])
        gathered = sh.allgather_int64(torch.from_numpy(local.view(np.int64)), world).numpy().view(np.uint64)
        total = sh.mod_sum_rows(gathered, be.chain.p)
        logits = []
        for r, part in enumerate(parts):
            raw = RawProduct(_Raw(*[np.ascontiguousarray(total[r, c]) for c in range(3)]), part.level, part.scale,
                             part.slots, part.fingerprint, part.backend_name, part.noise_bits)
            y = be.raw_finalize(raw)
            if enc.biases[4] is not None:
                y = be.add_ct_ct(y, enc.biases[4][r])
            logits.append(digest(np.concatenate([y.payload.c0, y.payload.c1])))
        if rank == 0:
            with open(out_path, "w") as fh:
                fh.write("\n".join(logits))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["mini2", "mini3"])
def test_two_rank_gloo_cells_sharding_matches_reference(tmp_path, golden, name):
    out = tmp_path / "logits.txt"
    mp.spawn(_worker, args=(2, _free_port(), name, str(out)), nprocs=2, join=True)
    assert out.read_text().split("\n") == golden["minis"][name]["logit_digests"]


# ---------------------------------------------------------------------------
# bands mode: two-convolution networks (config 4 / 5 topology)
# ---------------------------------------------------------------------------

def test_band_layout_and_plans():
    from paper_2102_00319_b200.configs import NETWORKS

    lay = sh.BandLayout.of(NETWORKS["cfg4"]())
    assert (lay.rows1, lay.cols1, lay.rows2, lay.cols2, lay.filters2, lay.pool_cols) == (12, 12, 10, 10, 10, 5)
    assert sh.plan_bands(10, 2) == [(0, 5), (5, 10)]
    assert lay.conv1_rows(5, 10) == (5, 12) and lay.input_rows(0, 5) == (0, 17)
    # every conv2 cell of every window is owned by exactly one band, for any split
    for parts in (1, 2, 3, 4, 5, 10):
        owned = [(f, i, j) for a, b in sh.plan_bands(10, parts) for f, r, jj, cells in lay.windows(a, b)
                 for i, j in cells]
        assert sorted(owned) == sorted((f, i, j) for f in range(10) for i in range(10) for j in range(10))
    # config 5: 4 batches over 1/2/4/8 ranks
    assert sh.plan_batches(4, 1) == [[(0, 0), (1, 0), (2, 0), (3, 0)]]
    assert sh.plan_batches(4, 2) == [[(0, 0), (2, 0)], [(1, 0), (3, 0)]]
    assert sh.plan_batches(4, 8)[5] == [(2, 1)]
    with pytest.raises(ValueError):
        sh.CellsLayout.of(NETWORKS["cfg4"]())
    with pytest.raises(ValueError):
        sh.BandLayout.of(NETWORKS["cfg2"]())


def _band_worker(rank, world, port, out_path):
    warnings.simplefilter("ignore")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(__file__))
        from conftest import S128, s128_params
        from nets import mini_networks
        from oracle.ckks_oracle import OracleBackend, _Raw
        from paper_2102_00319_b200 import percell
        from paper_2102_00319_b200.contract import RawProduct

        be = OracleBackend(s128_params(), S128["extra"])
        keys = be.keygen()
        be.set_eval_key(keys)
        net = mini_networks()["mini4"]
        imgs = np.random.default_rng(13).uniform(0, 1, (be.slots, 12, 12))
        enc = percell.encrypt_network(be, net, keys)
        grid = percell.encrypt_images(be, imgs, keys)
        lay = sh.BandLayout.of(net)
        band = sh.plan_bands(lay.rows2, world)[rank]
        parts = sh.percell_band_partials(be, enc, grid, band)
        local = np.stack([np.stack([p.payload.d0, p.payload.d1, p.payload.d2]) for p in parts])
        gathered = sh.allgather_int64(torch.from_numpy(local.view(np.int64)), world).numpy().view(np.uint64)
        total = sh.mod_sum_rows(gathered, be.chain.p)
        logits = []
        for r, part in enumerate(parts):
            raw = RawProduct(_Raw(*[np.ascontiguousarray(total[r, c]) for c in range(3)]), part.level, part.scale,
                             part.slots, part.fingerprint, part.backend_name, part.noise_bits)
            y = be.raw_finalize(raw)
            logits.append(digest(np.concatenate([y.payload.c0, y.payload.c1])))
        if rank == 0:
            with open(out_path, "w") as fh:
                fh.write("\n".join(logits))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_band_sharding_two_conv_matches_reference(tmp_path, golden, world):
    """conv -> x^2 -> conv(2 channels) -> x^2 -> pool -> FC split into conv2 row bands
    (world 3 cuts pool windows between ranks): logits equal the reference's own run."""
    out = tmp_path / "logits.txt"
    mp.spawn(_band_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    assert out.read_text().split("\n") == golden["minis"]["mini4"]["logit_digests"]
