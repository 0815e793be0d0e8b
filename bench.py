#!/usr/bin/env python
"""Benchmark: encrypted-CNN inference throughput on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config cfg2]

A *step* is one full encrypted inference pass of the config-2 network
(conv 5x5x5 stride 2 -> x^2 -> 2x2 sum-pool -> FC 180->10, N = 8192, 4096 images
packed one image per slot, every weight encrypted) over one batch whose input
ciphertexts are resident in HBM.  Under torchrun each rank runs its own
independent seeded batch (weak scaling); rank 0 gathers the logit ciphertexts
over NCCL.  ``value`` = images of all ranks / max-over-ranks device time.
``e2e`` repeats the measurement through the public API with the step's input
ciphertexts copied from pinned host memory and the logits copied back inside
the timed region.

``--impl reference`` times the reference algorithm on the host cores instead
(the C oracle port of the reference kernels, all host threads, bounded sample
extrapolated by exact op counts -- the reference itself is Python/numba and
not present on the GPU box).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BASELINE_METRIC = "encrypted-CNN images/sec and HE mul+relin ops/sec; % of B200 HBM roofline"
UNIT = "images/s"

# algorithmic (compulsory) HBM bytes and 64-bit modmuls per cfg2 batch
CFG2_PATH_BYTES_PER_BATCH = 3.562e9
CFG2_MODMULS_PER_BATCH = 10.36e9
CFG1_MULRELIN_BYTES_PER_OP = 527_360


def load_peaks() -> dict:
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None
        self.offset = 0

    def mark(self):
        """Start of the timed region: only samples written after this count.  The
        sampler itself is started well before (nvidia-smi start-up perturbs the GPU)."""
        time.sleep(0.12)
        self.offset = os.path.getsize(self.path) if self.path else 0

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            fh.seek(self.offset)
            lines = fh.read().splitlines()
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2102_00319_b200 import _lib, layers
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.comm import LogitGather
    from paper_2102_00319_b200.configs import BATCH, CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images
    from paper_2102_00319_b200.model import plaintext_forward

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    be = B200Backend(cfg.params(), cfg.base_extra_bits, device=local)
    keys = be.keygen()
    be.set_eval_key(keys)
    net = NETWORKS[args.config]()
    enc = layers.encrypt_network(be, net, keys)
    batch = min(BATCH[args.config], be.slots)
    images = cnn_images(batch, IMAGE_SEEDS[args.config] + rank)
    x = layers.encrypt_images(be, images, keys)
    ev = layers.LayerEvaluator(be)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # logit ciphertexts of every rank gathered over NCCL by libheb200 (heb_gather_logits)
    gatherer = LogitGather(world, rank, local) if world > 1 else None

    def gather(out):
        if gatherer is not None:
            return gatherer.gather(out.buf)
        return out.buf

    # correctness spot check against the float64 plaintext oracle (tolerance 1e-3, north star)
    out = ev.run(enc, x)
    dec = be.decrypt_batch(out, keys)[:, :batch].T  # (images, classes)
    ref = plaintext_forward(net, images[:256])
    err = float(np.max(np.abs(dec[:256] - ref)))
    argmax_ok = bool(np.array_equal(np.argmax(dec[:256], 1), np.argmax(ref, 1)))
    out_count, out_k = out.count, out.k
    del out
    be.ctx.release_scratch()  # the check ran on the default stream; the pipelines use their own
    torch.cuda.empty_cache()

    clocks = Clocks(local)
    clocks.start()
    ev.run_many(enc, x, max(args.warmup, args.pipelines), pipelines=args.pipelines, on_output=lambda s, o: gather(o))
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------------------
    clocks.mark()
    gc.disable()  # no collector pauses while the host enqueues the timed steps
    barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    marks = [] if os.environ.get("HEB_TIMELINE") else None
    h0 = time.perf_counter()
    t0.record(stream)
    ev.run_many(enc, x, args.steps, pipelines=args.pipelines, on_output=lambda s, o: gather(o), marks=marks)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    gc.enable()
    if marks:
        for s, (p, b, e, h) in enumerate(marks):
            print(f"timeline step {s} pipe {p}: start {t0.elapsed_time(b):8.2f} end {t0.elapsed_time(e):8.2f}"
                  f"  host enqueued {(h - h0) * 1e3:8.2f}", file=sys.stderr)
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = batch * world * args.steps / (ms_max / 1e3)

    # ---- per-kernel pass: the same K steps on one stream with CUDA events around every
    # launch (heb_prof_*), for the roofline's launch durations and the launch count ------
    prof, prof_ms = {}, 0.0
    if not args.no_prof:
        _lib.prof_enable(True)
        torch.cuda.synchronize()
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        pst = ev.pipeline_stream(0)  # pipeline 0's stream: its scratch arena already exists
        with torch.cuda.stream(pst):
            p0.record(pst)
            for _ in range(args.steps):
                gather(ev.run(enc, x))
            p1.record(pst)
        torch.cuda.synchronize()
        prof = _lib.prof_summary()
        _lib.prof_enable(False)
        prof_ms = p0.elapsed_time(p1)
        torch.cuda.empty_cache()
    # kernel launches in the timed region: kernel nodes of the replayed step graph x steps
    launches = ev.graph_kernel_launches(enc, x, 0) * args.steps

    # ---- end-to-end: host buffers through the public API -------------------------------
    # Every step copies its input ciphertexts from pinned host memory and its logits
    # back; LayerEvaluator.run_stream overlaps the copy of batch s+1 with batch s.  The
    # client hands the grid over in the bit-packed wire format (residues at the bit
    # length of their prime, csrc/packing.cu), unpacked on the device inside the step.
    x_packed = be.pack_batch(x)
    x_hosts = [torch.empty(x_packed.shape, dtype=x_packed.dtype, pin_memory=True) for _ in range(2)]
    for h in x_hosts:
        h.copy_(x_packed)
    del x_packed
    logits_hosts = [torch.empty((out_count, 2, out_k, be.n), dtype=torch.int64, pin_memory=True)
                    for _ in range(args.steps)]

    def e2e_run(nsteps):
        ev.run_stream(enc, [x_hosts[s % 2] for s in range(nsteps)], x.level, x.scale, x.noise_bits,
                      logits_hosts[:nsteps], on_output=lambda s, o: gather(o), pipelines=args.pipelines,
                      unpacked_shape=tuple(x.buf.shape))

    e2e_run(min(args.steps, max(2 * args.pipelines, args.warmup)))
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gc.disable()
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    gc.enable()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = batch * world * args.steps / (float(e2e_ms.item()) / 1e3)

    # ---- secondary: cfg1 HE mul+relin ops/s (256 pairs, one batched launch sequence) ----
    sec = cfg1_mulrelin(args, local) if (rank == 0 and not args.skip_cfg1) else None

    # ---- int64 modmul peak (microbenchmark) ---------------------------------------------
    peak_mm = modmul_peak(be) if rank == 0 else None

    if rank == 0:
        peaks = load_peaks()
        top = max(prof.items(), key=lambda kv: kv[1][1]) if prof else ("none", (0, 1e-9, 0.0))
        name, (cnt, tot_ms, tot_bytes) = top
        achieved = tot_bytes / (tot_ms / 1e3) / 1e9
        traffic = ncu_traffic(name)
        cpu = cpu_baseline(args) if (world == 1 and not args.skip_cpu and args.config == "cfg2") else None
        path_rate = CFG2_PATH_BYTES_PER_BATCH * value / batch / 1e9 if args.config == "cfg2" else None
        line = {
            "metric": BASELINE_METRIC,
            "value": round(value, 3),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u64",
            "data": "synthetic (seeded U[0,1] 28x28 pixels, N(0,0.1^2) weights; MNIST absent)",
            "config": {
                "workload": f"{args.config}: encrypted CNN {' -> '.join(l.kind for l in net.layers)}, "
                            f"N={be.n}, {be.chain.num_levels} levels, {batch} images/GPU",
                "batch_per_gpu": batch,
                "ring_degree": be.n,
                "l2_policy": f"inputs larger than L2 ({x.buf.numel() * 8 / 1e6:.0f} MB of input ciphertexts per step)",
                "parallelism": f"dp{world} (independent batches, logits gathered over NCCL)",
                "pipelines_per_gpu": args.pipelines,
            },
            "roofline": {
                "bound": "hbm",
                "kernel": name,
                "achieved": round(achieved, 2),
                "peak": peaks["hbm_gbs"],
                "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": traffic,
                "launches": cnt,
                "share_of_step": round(tot_ms / max(prof_ms, 1e-9), 4),
                "measured": "CUDA events around every launch in a dedicated pass of the same K steps on one stream",
                "peak_source": peaks["source"],
                "note": "kernel is INT64-multiply bound; see int_roofline",
            },
            "path_roofline": None if path_rate is None else {
                "algorithmic_bytes_per_batch": CFG2_PATH_BYTES_PER_BATCH,
                "achieved_gbs": round(path_rate, 2),
                "frac_of_hbm": round(path_rate / peaks["hbm_gbs"], 4),
                "source": "SURVEY.md §8(d) cfg2 layer-wise compulsory bytes",
            },
            "modmul_rate": None if (peak_mm is None or args.config != "cfg2") else {
                "modmuls_per_batch": CFG2_MODMULS_PER_BATCH,
                "achieved_modmul_per_s": CFG2_MODMULS_PER_BATCH * value / batch,
                "shoup_int_peak_per_s": peak_mm,
                "note": "SURVEY 8(d) modmul count; the 40-bit rows run on the FP64 (DFMA) pipe, "
                        "so the integer Shoup peak is not an upper bound for the mix",
            },
            "compute_roofline": ncu_pipes(name),
            "kernels": {k: {"launches": v[0], "ms": round(v[1], 3), "gbs": round(v[2] / max(v[1], 1e-9) / 1e6, 1)}
                        for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "cpu_baseline": cpu,
            "e2e": {
                "value": round(e2e_value, 3),
                "unit": UNIT,
                "h2d_bytes_per_step": int(x_hosts[0].numel() * 8),
                "wire_format": "bit-packed residues (heb_pack_rows), unpacked on the device in the step",
                "d2h_bytes_per_step": int(out_count * 2 * out_k * be.n * 8),
            },
            "gpu_launches": int(launches),
            "clocks": clk,
            "secondary": sec,
            "check": {"max_abs_err_vs_plaintext": err, "argmax_identical": argmax_ok, "images_checked": 256},
        }
        print(json.dumps(line), flush=True)
    if gatherer is not None:
        gatherer.close()
    if world > 1:
        dist.destroy_process_group()


def cfg1_mulrelin(args, device: int) -> dict:
    """HE mul+relin(+rescale) ops/s on config 1: 256 seeded pairs per batched call."""
    import torch

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend, ct_desc
    from paper_2102_00319_b200.configs import CONFIGS, cfg1_pairs

    cfg = CONFIGS["cfg1"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits, device=device)
    keys = be.keygen()
    be.set_eval_key(keys)
    xs, ys = cfg1_pairs(be.slots)
    a = be.encrypt_batch(xs, keys, np.arange(256))
    b = be.encrypt_batch(ys, keys, 256 + np.arange(256))
    ev = layers.LayerEvaluator(be)
    k = a.k
    # independent 256-pair calls on `streams` concurrent streams (each call: tensor +
    # relinearise + rescale into its own buffers), like the CNN's pipelines
    streams = [torch.cuda.Stream(be.dev) for _ in range(max(1, getattr(args, "pipelines", 3)))]
    raws = [be.ctx.empty(256, 3, k, be.n) for _ in streams]
    outs = [None] * len(streams)

    def step(i):
        st = streams[i % len(streams)]
        with torch.cuda.stream(st):
            raw = raws[i % len(streams)]
            be.ctx.call("heb_tensor", a.desc(), b.desc(), ct_desc(raw), 256, k, 0, be.ctx.stream)
            outs[i % len(streams)] = ev.finalize(raw, a.level, a.scale * b.scale, 0.0)
        return outs[i % len(streams)]

    cur = torch.cuda.current_stream(be.dev)
    for st in streams:
        st.wait_stream(cur)
    for i in range(10 * len(streams)):
        step(i)
    reps = 240  # ~0.4 ms per call: enough calls for a stable rate
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(cur)
    for st in streams:
        st.wait_stream(cur)
    for i in range(reps):
        out = step(i)
    for st in streams:
        cur.wait_stream(st)
    s1.record(cur)
    torch.cuda.synchronize()
    ops = 256 * reps / (s0.elapsed_time(s1) / 1e3)
    peaks = load_peaks()
    dec = be.decrypt_batch(out, keys)
    err = float(np.max(np.abs(dec[:8] - xs[:8] * ys[:8])))
    return {
        "metric": "HE mul+relin+rescale ops/sec (cfg1, N=4096, 256 pairs per call, concurrent calls on "
                  f"{len(streams)} streams)",
        "value": round(ops, 1),
        "hbm_frac": round(ops * CFG1_MULRELIN_BYTES_PER_OP / 1e9 / peaks["hbm_gbs"], 4),
        "max_abs_err": err,
    }


def modmul_peak(be) -> float:
    import ctypes

    import torch

    from paper_2102_00319_b200 import _lib

    ms = ctypes.c_double()
    blocks, threads, iters = 148 * 16, 256, 4096
    _lib.call("heb_bench_modmul", blocks, threads, iters, int(be.chain.primes[1]), ctypes.byref(ms),
              torch.cuda.current_stream().cuda_stream)
    return blocks * threads * iters * 8 / (ms.value / 1e3)


def ncu_traffic(kernel: str):
    """dram bytes per launch of the top kernel from the committed ncu capture, if any."""
    path = os.path.join(REPO, "profiles", "ncu_top_kernel.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    rec = d.get(kernel)
    return rec.get("dram_bytes_per_launch") if rec else None


def ncu_pipes(kernel: str):
    """Pipe utilisation of the top kernel from the committed ncu --set full capture."""
    path = os.path.join(REPO, "profiles", "ncu_top_kernel.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        rec = json.load(fh).get(kernel)
    if not rec:
        return None
    keys = ("fp64_pipe_pct", "alu_pipe_pct", "fma_pipe_pct", "issue_active_pct", "traffic_over_algorithmic", "source")
    out = {k: rec[k] for k in keys if k in rec}
    # per device launch (one per NTT engine for the fused ModUp): the pipe that bounds each
    per = [{k: l[k] for k in ("name", "fp64_pipe_pct", "fma_pipe_pct", "alu_pipe_pct", "issue_active_pct") if k in l}
           for l in rec.get("launches", [])]
    if per:
        out["per_launch"] = per
    return out


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------

class CpuSample:
    """Bounded sample of the cfg2 workload on the CPU oracle (reference algorithm).

    Sample = conv output rows 0-1 (all 5 filters, 120 cells: 25 taps each +
    relinearise/rescale), their x^2 (120 mul+relin), the 30 pooled windows they
    feed, plus the complete FC layer (1800 products, 10 finalizes).  conv/x^2/pool
    are 2/12 of their layers, so batch time = 6 * t(conv+sq+pool sample) + t(FC).
    """

    def __init__(self, config: str = "cfg2"):
        import warnings

        warnings.simplefilter("ignore")
        from oracle.ckks_oracle import OracleBackend, threaded_map
        from paper_2102_00319_b200.configs import BATCH, CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images
        from paper_2102_00319_b200.model import ledger, weight_entropies

        self.map = threaded_map
        cfg = CONFIGS[config]
        be = OracleBackend(cfg.params(), cfg.base_extra_bits)
        keys = be.keygen()
        be.set_eval_key(keys)
        self.be, self.keys = be, keys
        net = NETWORKS[config]()
        conv, dense = net.layers[0], net.layers[4]
        trace = ledger(net, be.chain, be.canonical_scale)
        self.batch = min(BATCH[config], be.slots)
        imgs = cnn_images(self.batch, IMAGE_SEEDS[config])
        tags = weight_entropies(net)
        slots = be.slots
        cells = [(i, j) for i in range(7) for j in range(28)]
        self.x = {}
        for (i, j), ct in zip(cells, threaded_map(lambda ij: be.encrypt(imgs[:, ij[0], ij[1]], keys, entropy=ij[0] * 28 + ij[1]), cells)):
            self.x[(i, j)] = ct
        widx = [(f, p, q) for f in range(5) for p in range(5) for q in range(5)]
        self.w = dict(zip(widx, threaded_map(lambda t: be.encrypt(np.full(slots, conv.weights[t[0], 0, t[1], t[2]]), keys, entropy=int(tags[0][t[0], 0, t[1], t[2]])), widx)))
        fc_level = trace[4]["level"]
        fc_scale = trace[4]["scale"]
        self.fc_in = threaded_map(lambda i: be.drop_to_level(be.encrypt(np.full(slots, 0.1 * (i % 7)), keys, scale=fc_scale, entropy=10_000 + i), fc_level), range(180))
        fidx = [(i, r) for i in range(180) for r in range(10)]
        self.fw = dict(zip(fidx, threaded_map(lambda t: be.drop_to_level(be.encrypt(np.full(slots, dense.weights[t]), keys, entropy=int(tags[4][t])), fc_level), fidx)))
        self.cores = os.cpu_count() or 1

    def _conv_cell(self, fij):
        be = self.be
        f, i, j = fij
        acc = None
        for p in range(5):
            for q in range(5):
                t = be.mul_ct_ct_raw(self.x[(2 * i + p, 2 * j + q)], self.w[(f, p, q)])
                acc = t if acc is None else be.raw_add(acc, t)
        y = be.raw_finalize(acc)
        return be.mul_ct_ct(y, y)

    def _fc_out(self, r):
        be = self.be
        acc = be.mul_ct_ct_raw(self.fc_in[0], self.fw[(0, r)])
        for i in range(1, 180):
            acc = be.raw_add(acc, be.mul_ct_ct_raw(self.fc_in[i], self.fw[(i, r)]))
        return be.raw_finalize(acc)

    def step(self) -> float:
        """Run the sample once; returns extrapolated seconds per full batch."""
        be = self.be
        t0 = time.perf_counter()
        cells = [(f, i, j) for f in range(5) for i in range(2) for j in range(12)]
        sq = dict(zip(cells, self.map(self._conv_cell, cells)))
        windows = [(f, j) for f in range(5) for j in range(6)]

        def pool(fj):
            f, j = fj
            acc = sq[(f, 0, 2 * j)]
            for di, dj in ((1, 0), (0, 1), (1, 1)):
                acc = be.add_ct_ct(acc, sq[(f, di, 2 * j + dj)])
            return acc

        self.map(pool, windows)
        t1 = time.perf_counter()
        self.map(self._fc_out, range(10))
        t2 = time.perf_counter()
        return 6.0 * (t1 - t0) + (t2 - t1)


def cpu_baseline(args) -> dict:
    s = CpuSample(args.config)
    sec = s.step()
    return {
        "value": round(s.batch / sec, 3),
        "unit": UNIT,
        "cores": s.cores,
        "kind": "port",
        "sample": "cfg2 conv rows 0-1 (120 cells x 25 taps + relin), their x^2, 30 pool windows, full FC; "
                  "extrapolated x6 for conv/x^2/pool; C oracle of the reference kernels, ThreadPool over all cores",
    }


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    s = CpuSample(args.config)
    for _ in range(args.warmup if args.warmup < 2 else 1):
        s.step()
    secs = [s.step() for _ in range(args.steps)]
    batch_s = sum(secs) / len(secs)
    value = s.batch / batch_s
    line = {
        "metric": BASELINE_METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "impl": "reference",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(batch_s * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: same network/batch as the b200 arm", "batch_per_gpu": s.batch},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": s.cores, "kind": "port",
                         "sample": "per step: cfg2 conv rows 0-1 + x^2 + pool windows + full FC, extrapolated to the batch"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--pipelines", type=int, default=3,
                    help="concurrent inference pipelines (streams) per GPU")
    ap.add_argument("--no-prof", action="store_true", help="no per-kernel events in the timed region")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-cfg1", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
