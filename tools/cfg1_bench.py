"""cfg1 mul+relin+rescale ops/s only (bench.py's secondary line), for A/B runs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


class A:
    pass


print(json.dumps(bench.cfg1_mulrelin(A(), 0)))
