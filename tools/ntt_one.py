"""Launch a few plain NTTs on the cfg2-sized chain (for ncu captures of the NTT engine).

    python tools/ntt_one.py [--rows fp|int] [--inv] [--batch 2048]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_00319_b200.backend import DeviceContext  # noqa: E402
from paper_2102_00319_b200.chain import build_chain  # noqa: E402
from paper_2102_00319_b200.params import derive_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--logn", type=int, default=13)
ap.add_argument("--batch", type=int, default=2048)
ap.add_argument("--rows", default="fp")
ap.add_argument("--inv", action="store_true")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = 1 << a.logn
ch = build_chain(derive_params(2 * n, 260, 40, seed=1), 20)
ctx = DeviceContext(ch)
rows = ch.num_rows
buf = torch.randint(0, 1 << 39, (a.batch, rows, n), dtype=torch.int64, device="cuda")
row0, nrows = (1, rows - 2) if a.rows == "fp" else (0, 1)
fn = "heb_ntt_inv" if a.inv else "heb_ntt_fwd"
for _ in range(a.reps):
    ctx.call(fn, buf[:, row0:].data_ptr(), a.batch, nrows, row0, rows * n, ctx.stream)
torch.cuda.synchronize()
print("ok")
