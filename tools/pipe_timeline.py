"""Per-step CUDA-event timeline of the pipelined evaluator (diagnoses throughput variance).

    python tools/pipe_timeline.py [--pipelines 3] [--steps 10] [--reps 6]
"""
import argparse
import os
import sys
import time
import warnings

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.simplefilter("ignore")

from paper_2102_00319_b200 import layers  # noqa: E402
from paper_2102_00319_b200.backend import B200Backend  # noqa: E402
from paper_2102_00319_b200.configs import BATCH, CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pipelines", type=int, default=3)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--reps", type=int, default=6)
a = ap.parse_args()
cfg = CONFIGS["cfg2"]
be = B200Backend(cfg.params(), cfg.base_extra_bits)
keys = be.keygen()
be.set_eval_key(keys)
net = NETWORKS["cfg2"]()
enc = layers.encrypt_network(be, net, keys)
x = layers.encrypt_images(be, cnn_images(BATCH["cfg2"], IMAGE_SEEDS["cfg2"]), keys)
ev = layers.LayerEvaluator(be)
ev.run_many(enc, x, 3, pipelines=a.pipelines)
torch.cuda.synchronize()
caller = torch.cuda.current_stream()
for rep in range(a.reps):
    P = a.pipelines
    comp = ev._pipeline_streams("compute", P)
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(caller)
    for st in comp:
        st.wait_stream(caller)
    evs = []
    h0 = time.perf_counter()
    hs = []
    for s in range(a.steps):
        st = comp[s % P]
        b = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            b.record(st)
            ev.run(enc, x)
            e.record(st)
        hs.append(time.perf_counter() - h0)
        evs.append((s % P, b, e))
    for st in comp:
        caller.wait_stream(st)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record(caller)
    torch.cuda.synchronize()
    tot = t0.elapsed_time(t1)
    print(f"rep {rep}: total {tot:.1f} ms  host enqueue {hs[-1] * 1e3:.1f} ms")
    for s, (p, b, e) in enumerate(evs):
        print(f"   step {s} pipe {p}: start {t0.elapsed_time(b):7.2f}  end {t0.elapsed_time(e):7.2f}  "
              f"dur {b.elapsed_time(e):6.2f}  host_done {hs[s] * 1e3:7.2f}")
