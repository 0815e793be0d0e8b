"""Per-kernel device time of the cfg1 secondary ops (CUDA events around every launch).

    python tools/cfg1_prof.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2102_00319_b200 import _lib  # noqa: E402


class A:
    pipelines = 1


bench.CFG1_STREAMS = 1
_lib.prof_enable(True)
out = bench.cfg1_ops(A(), 0)
prof = _lib.prof_summary()
_lib.prof_enable(False)
tot = sum(v[1] for v in prof.values())
for name, (cnt, ms, nbytes) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:32s} launches {cnt:6d}  ms {ms:9.3f}  share {100 * ms / tot:5.1f}%  us/launch {1e3 * ms / cnt:8.2f}  GB/s {nbytes / ms / 1e6:8.1f}")
print(json.dumps(out["ops"]))
