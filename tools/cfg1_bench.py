"""cfg1 mul+relin+rescale ops/s only (bench.py's secondary line), for A/B runs.

    python tools/cfg1_bench.py [STREAMS]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


class A:
    pipelines = int(sys.argv[1]) if len(sys.argv) > 1 else 3


print(json.dumps(bench.cfg1_ops(A(), 0)))
