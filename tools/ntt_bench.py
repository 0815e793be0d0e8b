"""Standalone NTT throughput (heb_ntt_fwd / heb_ntt_inv) on the cfg2 chain.

    python tools/ntt_bench.py [--logn 13] [--batch 4096]

Reports G butterflies/s separately for the FP64-engine rows (40-bit level primes)
and the integer-engine rows (60-bit base / special primes).
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_00319_b200 import _lib  # noqa: E402
from paper_2102_00319_b200.backend import DeviceContext  # noqa: E402
from paper_2102_00319_b200.chain import build_chain  # noqa: E402
from paper_2102_00319_b200.params import derive_params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, default=13)
    ap.add_argument("--batch", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n = 1 << args.logn
    ch = build_chain(derive_params(2 * n, 260, 40, seed=1), 20)
    ctx = DeviceContext(ch)
    rows = ch.num_rows
    buf = torch.randint(0, 1 << 39, (args.batch, rows, n), dtype=torch.int64, device="cuda")
    st = ctx.stream
    bfly = args.batch * (n // 2) * args.logn
    for name, row0, nrows in (("fp64 rows (40-bit)", 1, rows - 2), ("int rows (60-bit)", 0, 1)):
        for fn in ("heb_ntt_fwd", "heb_ntt_inv"):
            view = buf[:, row0:row0 + nrows]
            for _ in range(2):
                ctx.call(fn, view.data_ptr(), args.batch, nrows, row0, rows * n, st)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                ctx.call(fn, view.data_ptr(), args.batch, nrows, row0, rows * n, st)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.reps
            print(f"{name:20s} {fn:12s} {ms:8.3f} ms  {bfly * nrows / ms / 1e6:8.1f} G butterflies/s  "
                  f"{2 * 8 * args.batch * nrows * n / ms / 1e6:8.1f} GB/s")


if __name__ == "__main__":
    main()
