"""heb_unpack_rows throughput on the cfg2 input grid shape (784 cts x 2 comps x 6 rows)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_00319_b200.backend import DeviceContext  # noqa: E402
from paper_2102_00319_b200.chain import build_chain  # noqa: E402
from paper_2102_00319_b200.params import derive_params  # noqa: E402

n, K, count = 8192, 6, 784 * 2
ch = build_chain(derive_params(2 * n, 260, 40, seed=1), 20)
ctx = DeviceContext(ch)
words = int(ctx.call.__self__ and __import__("paper_2102_00319_b200._lib", fromlist=["x"]).lib().heb_packed_words(ctx.handle, K))
packed = torch.randint(0, 2**62, (count, words), dtype=torch.int64, device="cuda")
out = torch.empty((count, K, n), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.call("heb_unpack_rows", packed.data_ptr(), count, K, out.data_ptr(), K * n, ctx.stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    ctx.call("heb_unpack_rows", packed.data_ptr(), count, K, out.data_ptr(), K * n, ctx.stream)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
gb = (packed.numel() + out.numel()) * 8 / 1e9
print(f"unpack {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
