"""Per-row cost of the fused conv tensor (heb_conv_tensor) on cfg2 shapes.

    python tools/conv_probe.py

Times the launch over rows 0..k-1 for k = 1 (the 60-bit base row only, integer body)
and k = 6 (all rows), with and without the split-limb FP64 body."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_00319_b200.backend import DeviceContext, ct_desc  # noqa: E402
from paper_2102_00319_b200.chain import build_chain  # noqa: E402
from paper_2102_00319_b200.params import derive_params  # noqa: E402


def main():
    n = 8192
    ch = build_chain(derive_params(2 * n, 260, 40, seed=1), 20)
    ctx = DeviceContext(ch)
    K = 6
    x = torch.randint(0, 1 << 39, (784, 2, K, n), dtype=torch.int64, device="cuda")
    w = torch.randint(0, 1 << 39, (125, 2, K, n), dtype=torch.int64, device="cuda")
    raw = torch.empty((720, 3, K, n), dtype=torch.int64, device="cuda")
    st = ctx.stream
    for k in (1, 6):
        for _ in range(2):
            ctx.call("heb_conv_tensor", ct_desc(x), ct_desc(w), ct_desc(raw), 1, 28, 28, 5, 5, 5, 2, k, st)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            ctx.call("heb_conv_tensor", ct_desc(x), ct_desc(w), ct_desc(raw), 1, 28, 28, 5, 5, 5, 2, k, st)
        b.record()
        torch.cuda.synchronize()
        print(f"conv_tensor k={k} limbs={'off' if os.environ.get('HEB_CONV_NO_LIMBS') else 'on'}: "
              f"{a.elapsed_time(b) / 10:.3f} ms")


if __name__ == "__main__":
    main()
