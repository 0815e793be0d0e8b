#!/usr/bin/env python
"""Benchmark: encrypted-CNN inference throughput on B200 (BASELINE.json configs 2-4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config cfg4]

A *step* is one full encrypted inference pass of the config's network over one batch
whose input ciphertexts are resident in HBM.  The default is config 4, the largest
configuration that fits one GPU (N = 32768, 19 levels, 16384 images packed one image
per slot: conv1 5x5x5 stride 2 -> x^2 -> conv2 10 filters 3x3 over 5 channels -> x^2 ->
2x2 sum-pool -> FC 250->10, every weight encrypted); ``--config cfg2`` / ``cfg3`` give
the smaller networks.  Under torchrun each rank runs its own independent seeded batch
(weak scaling); rank 0 gathers the logit ciphertexts over NCCL.  ``value`` = images of
all ranks / max-over-ranks device time.  ``e2e`` repeats the measurement through the
public API with the step's input ciphertexts copied from pinned host memory (bit-packed
wire format; ``e2e_u64``: the reference's u64 payload words) and the logits copied back
inside the timed region.

``--impl reference`` times the reference algorithm on the host cores instead (the C
oracle port of the reference kernels driven in the reference op order, all host
threads): each step is an exactly proportional 1/S sample of every layer of the same
network (``CpuSample``), timed as it runs -- the reference itself is Python/numba and is
not present on the GPU box.
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

# algorithmic (compulsory) HBM bytes and 64-bit modmuls per batch
PATH_BYTES_PER_BATCH = {"cfg2": 3.562e9, "cfg3": 7.747e9, "cfg4": 102.46e9}
MODMULS_PER_BATCH = {"cfg2": 10.36e9, "cfg3": 29.1e9, "cfg4": 665.6e9}
# algorithmic bytes per op
CFG1_BYTES_PER_OP = {"mul_relin_rescale": 527_360, "add_ct_ct": 589_824, "mul_ct_pt_rescale": 425_984,
                     "rotate_by_1": 396_288}
CFG1_MULRELIN_BYTES_PER_OP = CFG1_BYTES_PER_OP["mul_relin_rescale"]
CFG1_STREAMS = 3
# concurrent inference pipelines per GPU (a second cfg4 pipeline runs out of HBM)
PIPELINES = {"cfg2": 3, "cfg3": 3, "cfg4": 1}


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
    # back; LayerEvaluator.run_stream overlaps the copy of batch s+1 with batch s.
    # Two client formats: (1) the bit-packed wire format (residues at the bit length of
    # their prime, csrc/packing.cu), unpacked on the device inside the step; (2) the
    # reference's own payload words (u64 per residue, CkksCipher layout).
    logits_hosts = [torch.empty((out_count, 2, out_k, be.n), dtype=torch.int64, pin_memory=True)
                    for _ in range(args.steps)]

    def e2e_measure(host, unpacked_shape):
        def e2e_run(nsteps):
            ev.run_stream(enc, [host] * nsteps, x.level, x.scale, x.noise_bits, logits_hosts[:nsteps],
                          on_output=lambda s, o: gather(o), pipelines=args.pipelines, unpacked_shape=unpacked_shape)

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
        e_ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        return batch * world * args.steps / (float(e_ms.item()) / 1e3)

    x_packed = be.pack_batch(x)
    x_host = torch.empty(x_packed.shape, dtype=x_packed.dtype, pin_memory=True)
    x_host.copy_(x_packed)
    del x_packed
    e2e_value = e2e_measure(x_host, tuple(x.buf.shape))
    packed_bytes = int(x_host.numel() * 8)
    del x_host
    ev.drop_input_buffers()
    e2e_u64 = None
    if not args.skip_u64:
        x_host = torch.empty(tuple(x.buf.shape), dtype=torch.int64, pin_memory=True)
        x_host.copy_(x.buf)
        e2e_u64 = {"value": round(e2e_measure(x_host, None), 3), "unit": UNIT,
                   "h2d_bytes_per_step": int(x_host.numel() * 8),
                   "d2h_bytes_per_step": int(out_count * 2 * out_k * be.n * 8),
                   "wire_format": "u64 words per residue (the reference's CkksCipher payload layout), copied into a "
                                  "device staging buffer and moved into the step's input buffer by one device copy"}
        del x_host
        ev.drop_input_buffers()

    # ---- secondary: cfg1 HE mul+relin ops/s (256 pairs, one batched launch sequence) ----
    sec = cfg1_ops(args, local) if (rank == 0 and not args.skip_cfg1) else None

    # ---- int64 modmul peak (microbenchmark) ---------------------------------------------
    peak_mm = modmul_peak(be) if rank == 0 else None
    peak_bf = butterfly_peaks(be) if rank == 0 else None

    if rank == 0:
        peaks = load_peaks()
        top = max(prof.items(), key=lambda kv: kv[1][1]) if prof else ("none", (0, 1e-9, 0.0))
        name, (cnt, tot_ms, tot_bytes) = top
        achieved = tot_bytes / (tot_ms / 1e3) / 1e9
        traffic = ncu_traffic(name, args.config)
        cpu = cpu_baseline(args) if (world == 1 and not args.skip_cpu) else None
        path_bytes = PATH_BYTES_PER_BATCH[args.config]
        path_rate = path_bytes * value / batch / 1e9
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
            "data": f"synthetic (seeded U[0,1] 28x28 pixels, N(0,{net_sigma(args.config)}^2) weights; MNIST absent)",
            "config": {
                "workload": workload_name(args.config, net, be.n, be.chain.num_levels, batch),
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
                "note": "kernel is bound by the FP64 / integer pipes (NTT butterflies), not HBM: see compute_roofline",
            },
            "path_roofline": {
                "algorithmic_bytes_per_batch": path_bytes,
                "achieved_gbs": round(path_rate, 2),
                "frac_of_hbm": round(path_rate / peaks["hbm_gbs"], 4),
                "source": f"SURVEY.md §8(d) {args.config} layer-wise compulsory bytes",
            },
            "modmul_rate": None if peak_mm is None else {
                "modmuls_per_batch": MODMULS_PER_BATCH[args.config],
                "achieved_modmul_per_s": MODMULS_PER_BATCH[args.config] * value / batch,
                "shoup_int_peak_per_s": peak_mm,
                "note": "SURVEY 8(d) modmul count; the 40-bit rows run on the FP64 (DFMA) pipe, "
                        "so the integer Shoup peak is not an upper bound for the mix",
            },
            "compute_roofline": ncu_pipes(name, args.config),
            "butterfly_roofline": butterfly_roofline(net, be, x.level, prof, args.steps, peak_bf),
            "kernels": {k: {"launches": v[0], "ms": round(v[1], 3), "gbs": round(v[2] / max(v[1], 1e-9) / 1e6, 1)}
                        for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "cpu_baseline": cpu,
            "e2e": {
                "value": round(e2e_value, 3),
                "unit": UNIT,
                "h2d_bytes_per_step": packed_bytes,
                "wire_format": "bit-packed residues (heb_pack_rows), unpacked on the device in the step",
                "d2h_bytes_per_step": int(out_count * 2 * out_k * be.n * 8),
            },
            "e2e_u64": e2e_u64,
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


def run_cfg5(args) -> None:
    """BASELINE config 5: the config-4 network on 4 independent seeded 16384-image
    batches (same keys and weights), sharded over WORLD_SIZE GPUs (strong scaling: the
    total work is fixed).  Ranks take whole batches while world <= 4; beyond that each
    batch is split into world / 4 bands of conv2 output rows (conv1 / x^2 halo recomputed,
    sharding.run_band_shard) whose FC raw partials are all-gathered within the batch's
    rank group over NCCL -- the path's one real exchange -- summed mod p and finalised.
    value = 4 batches x 16384 images / max-over-ranks device time per step."""
    import torch
    import torch.distributed as dist

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200 import sharding as sh
    from paper_2102_00319_b200.backend import B200Backend
    from paper_2102_00319_b200.configs import BATCH, CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images
    from paper_2102_00319_b200.model import plaintext_forward

    batches = 4
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS["cfg4"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits, device=local)
    keys = be.keygen()
    be.set_eval_key(keys)
    net = NETWORKS["cfg4"]()
    enc = layers.encrypt_network(be, net, keys)
    batch = min(BATCH["cfg4"], be.slots)
    plan = sh.plan_batches(batches, world)[rank]
    per = max(1, world // batches)
    lay = sh.BandLayout.of(net)
    bands = sh.plan_bands(lay.rows2, per)
    images = {b: cnn_images(batch, IMAGE_SEEDS["cfg4"] + b) for b, _ in plan}
    xs = {b: layers.encrypt_images(be, images[b], keys) for b, _ in plan}
    ev = layers.LayerEvaluator(be)
    stream = torch.cuda.current_stream()
    group = None
    if per > 1:
        groups = [dist.new_group(list(range(g * per, (g + 1) * per))) for g in range(world // per)]
        group = groups[rank // per]

    def step():
        outs = {}
        for b, band in plan:
            if per == 1:
                outs[b] = ev.run(enc, xs[b])
                continue
            raw, lvl, scale, noise = ev.run_band_shard(enc, xs[b], bands[band])
            got = [torch.empty_like(raw) for _ in range(per)]
            dist.all_gather(got, raw, group=group)
            if band == 0:
                outs[b] = ev.finish_cells(enc, torch.stack(got), lvl, scale, noise)
        return outs

    out = step()  # correctness check: decrypted logits vs the float64 plaintext forward pass
    err, argmax_ok = 0.0, True
    for b, y in out.items():
        dec = be.decrypt_batch(y, keys)[:, :batch].T
        ref = plaintext_forward(net, images[b][:64])
        err = max(err, float(np.max(np.abs(dec[:64] - ref))))
        argmax_ok = argmax_ok and bool(np.array_equal(np.argmax(dec[:64], 1), np.argmax(ref, 1)))
    del out
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    clocks.mark()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = torch.tensor([t0.elapsed_time(t1)], device="cuda")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_max = float(ms.item())
    value = batches * batch * args.steps / (ms_max / 1e3)
    if rank == 0:
        peaks = load_peaks()
        path_rate = PATH_BYTES_PER_BATCH["cfg4"] * value / batch / 1e9
        print(json.dumps({
            "metric": BASELINE_METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (4 seeded U[0,1] 28x28 image batches, N(0,0.05^2) weights; MNIST absent)",
            "config": {"workload": f"cfg5: the cfg4 network on {batches} batches of {batch} images, N={be.n}",
                       "batches": batches, "batch": batch, "parallelism": (
                           f"{world} ranks: whole batches" if per == 1 else
                           f"{world} ranks: {per} conv2-row bands per batch (halo recompute), FC partials "
                           f"all-gathered per batch over NCCL"),
                       "l2_policy": "inputs larger than L2"},
            "path_roofline": {"achieved_gbs": round(path_rate, 2), "frac_of_hbm": round(path_rate / peaks["hbm_gbs"], 4),
                              "source": "SURVEY.md §8(d) cfg4 layer-wise compulsory bytes"},
            "clocks": clk,
            "check": {"max_abs_err_vs_plaintext": err, "argmax_identical": argmax_ok, "images_checked": 64},
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cfg1_ops(args, device: int) -> dict:
    """Config 1 primitive ops/s on the device: 256 seeded pairs per batched call, calls
    issued round-robin on the bench's pipeline count of concurrent streams.  Ops (SURVEY
    §8d): mul+relin+rescale, ct+ct, ct*pt+rescale, rotate-by-1 (Galois element 5)."""
    import torch

    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend, ct_desc
    from paper_2102_00319_b200.configs import CONFIGS, cfg1_pairs

    cfg = CONFIGS["cfg1"]
    be = B200Backend(cfg.params(), cfg.base_extra_bits, device=device)
    keys = be.keygen(galois_steps=(1,))
    be.set_eval_key(keys)
    be.set_galois_key(keys)
    P = 256
    xs, ys = cfg1_pairs(be.slots, P)
    a = be.encrypt_batch(xs, keys, np.arange(P))
    b = be.encrypt_batch(ys, keys, P + np.arange(P))
    ev = layers.LayerEvaluator(be)
    k, n, lvl = a.k, be.n, a.level
    pts = torch.stack([be.encode_plain(ys[i]).payload.rows[:k] for i in range(P)]).contiguous()
    g = be.galois_element(1)
    gk = be._galois_keys[g].prep
    # cfg1 calls are small (256 pairs): concurrent calls on CFG1_STREAMS streams fill the SMs
    # (measured in round 1: 679k -> 822k ops/s from 1 to 3 streams), whatever the headline config uses
    streams = [torch.cuda.Stream(be.dev) for _ in range(max(CFG1_STREAMS, args.pipelines))]
    S = len(streams)
    raws = [be.ctx.empty(P, 3, k, n) for _ in streams]
    outs = [be.ctx.empty(P, 2, k, n) for _ in streams]
    last = {}

    def mul(i):
        be.ctx.call("heb_tensor", a.desc(), b.desc(), ct_desc(raws[i % S]), P, k, 0, be.ctx.stream)
        last["mul"] = ev.finalize(raws[i % S], lvl, a.scale * b.scale, 0.0)

    def add(i):
        be.ctx.call("heb_add", a.desc(), b.desc(), ct_desc(outs[i % S]), P, 2, k, be.ctx.stream)

    def ctpt(i):
        be.ctx.call("heb_mul_plain_rescale", a.desc(), pts.data_ptr(), k * n, ct_desc(outs[i % S]), P, lvl,
                    be.ctx.stream)

    def rot(i):
        be.ctx.call("heb_rotate", a.desc(), gk.data_ptr(), ct_desc(outs[i % S]), P, lvl, g, be.ctx.stream)
        last["rot"] = outs[i % S]

    cur = torch.cuda.current_stream(be.dev)

    def timed(fn, reps):
        for st in streams:
            st.wait_stream(cur)
        for i in range(4 * S):
            with torch.cuda.stream(streams[i % S]):
                fn(i)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(cur)
        for st in streams:
            st.wait_stream(cur)
        for i in range(reps):
            with torch.cuda.stream(streams[i % S]):
                fn(i)
        for st in streams:
            cur.wait_stream(st)
        s1.record(cur)
        torch.cuda.synchronize()
        return P * reps / (s0.elapsed_time(s1) / 1e3)

    peaks = load_peaks()
    res = {}
    for name, fn, reps in (("mul_relin_rescale", mul, 240), ("add_ct_ct", add, 2000), ("mul_ct_pt_rescale", ctpt, 600),
                           ("rotate_by_1", rot, 240)):
        ops = timed(fn, reps)
        res[name] = {"value": round(ops, 1), "unit": "ops/s",
                     "hbm_frac": round(ops * CFG1_BYTES_PER_OP[name] / 1e9 / peaks["hbm_gbs"], 4)}
    dec = be.decrypt_batch(last["mul"], keys)
    res["mul_relin_rescale"]["max_abs_err"] = float(np.max(np.abs(dec[:8] - xs[:8] * ys[:8])))
    return {
        "metric": f"HE ops/sec on cfg1 (N=4096, 256 pairs per call, concurrent calls on {S} streams)",
        "l2_note": "every call reads the same 256 input pairs: the pointwise ops' working set is partly L2-resident, "
                   "so their hbm_frac (algorithmic bytes / measured HBM copy bandwidth) can exceed 1",
        "value": res["mul_relin_rescale"]["value"],
        "unit": "ops/s",
        "ops": res,
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


def butterfly_peaks(be) -> dict:
    """Measured register-only butterfly ceilings of the two NTT engines (heb_bench_butterfly)."""
    import ctypes

    import torch

    from paper_2102_00319_b200 import _lib

    primes = [int(q) for q in be.chain.primes]
    small = [q for q in primes if q < (1 << 42)]
    wide = [q for q in primes if q >= (1 << 42)] or primes
    out = {}
    blocks, threads, iters = 148 * 8, 256, 512
    for kind, name, q in ((1, "fp64", small[0] if small else None), (2, "int", wide[0])):
        if q is None:
            continue
        ms = ctypes.c_double()
        _lib.call("heb_bench_butterfly", kind, blocks, threads, iters, q, ctypes.byref(ms),
                  torch.cuda.current_stream().cuda_stream)
        out[name] = blocks * threads * iters * 128 / (ms.value / 1e3)
    return out


def modup_butterflies(net, be, top_level: int) -> dict:
    """Butterflies and key products of the fused ModUp launches of one inference, from the network
    shape: a relinearisation of `items` ciphertexts at k rows runs, for every target row t (the k
    chain rows and the special prime), one N-point transform per digit j != t ((N/2) log N
    butterflies each) and 2 N key products per digit."""
    from paper_2102_00319_b200.analyzer import analyze

    n = be.n
    logn = n.bit_length() - 1
    primes = [int(q) for q in be.chain.primes]  # chain rows, then the special prime
    is_fp = [q < (1 << 42) for q in primes[:-1]]  # engine of each chain row (ntt.cuh: FP64 engine below 2^42)
    special_fp = primes[-1] < (1 << 42)
    rep = analyze(net, be.params)
    level = top_level
    fp = integer = keyprod = 0
    relins = []
    for lc in rep.per_layer:
        if lc.name in ("conv", "square", "polyact", "dense"):
            k = level + 1
            per_t = (n // 2) * logn
            t_fp = sum((k - 1) for t in range(k) if is_fp[t]) + (k if special_fp else 0)
            t_int = sum((k - 1) for t in range(k) if not is_fp[t]) + (0 if special_fp else k)
            fp += lc.out_cts * t_fp * per_t
            integer += lc.out_cts * t_int * per_t
            keyprod += lc.out_cts * (k + 1) * k * 2 * n
            relins.append({"layer": lc.name, "items": lc.out_cts, "rows": k})
        level -= lc.levels
    return {"fp64": fp, "int": integer, "key_products": keyprod, "relinearisations": relins}


def ncu_record_path(config: str) -> str:
    """The committed ncu --set full capture of this config's top kernel."""
    return os.path.join(REPO, "profiles", f"ncu_top_kernel_{config}.json")


def butterfly_roofline(net, be, top_level, prof, steps, peaks):
    """Compute roofline of the fused ModUp: its NTT butterflies per second against the measured
    register-only butterfly ceilings of the two engines, weighted by the row mix.  The two engine
    launches run concurrently (DFMA vs IMAD/ALU pipes), so the ceiling is the slower engine's time
    (`ceiling_overlapped`); `ceiling_serial` adds the two times.  Key products ride on top of the
    butterflies (not counted in `achieved`), so `frac` understates the pipe use."""
    rec = prof.get("k_ks_modup_fused")
    if not rec or not peaks or "int" not in peaks:
        return None
    w = modup_butterflies(net, be, top_level)
    ms = rec[1] / steps
    t_fp = w["fp64"] / peaks["fp64"] if "fp64" in peaks and w["fp64"] else 0.0
    t_int = w["int"] / peaks["int"]
    total = w["fp64"] + w["int"]
    achieved = total / (ms / 1e3)
    over = total / max(t_fp, t_int)
    serial = total / (t_fp + t_int)
    return {
        "kernel": "k_ks_modup_fused",
        "butterflies_per_step": {"fp64_engine": w["fp64"], "int_engine": w["int"]},
        "key_products_per_step": w["key_products"],
        "ms_per_step": round(ms, 3),
        "achieved_gbf_s": round(achieved / 1e9, 1),
        "peak_fp64_gbf_s": round(peaks.get("fp64", 0.0) / 1e9, 1),
        "peak_int_gbf_s": round(peaks["int"] / 1e9, 1),
        "ceiling_overlapped_gbf_s": round(over / 1e9, 1),
        "ceiling_serial_gbf_s": round(serial / 1e9, 1),
        "frac": round(achieved / over, 4),
        "frac_serial": round(achieved / serial, 4),
        "relinearisations": w["relinearisations"],
        "measured": "heb_bench_butterfly (registers only, the engines' own butterfly code) in this run; "
                    "ModUp time from the per-kernel event pass",
    }


def ncu_traffic(kernel: str, config: str):
    """dram bytes per launch of the top kernel from the config's committed ncu capture, if any."""
    path = ncu_record_path(config)
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    rec = d.get(kernel)
    return rec.get("dram_bytes_per_launch") if rec else None


def ncu_pipes(kernel: str, config: str):
    """Pipe utilisation of the top kernel from the config's committed ncu --set full capture."""
    path = ncu_record_path(config)
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
    """Bounded, exactly proportional sample of one batch of the config's network on the
    CPU oracle (the reference algorithm: the C restatement of its kernels driven through
    the reference's per-ciphertext op sequence, ``percell`` order).

    The sample is 1/S of EVERY layer: the first 1/S of the conv cells (position-major,
    filter fastest), of the activations, of the pool windows and of the FC outputs.
    All cells of a layer cost the same ops (same taps, same level), so one sample is
    exactly 1/S of the batch's HE operations and stands for batch/S images -- no
    per-layer extrapolation.  Layer l's sampled cells read real ciphertexts of the right
    level and scale: the first conv reads the encrypted input pixels its cells cover,
    later layers read the previous layer's sampled outputs (wrapped around).
    """

    SHARDS = {"cfg2": 1, "cfg3": 5, "cfg4": 10}

    def __init__(self, config: str = "cfg4", shards: int | None = None):
        import warnings

        warnings.simplefilter("ignore")
        from oracle.ckks_oracle import OracleBackend, threaded_map
        from paper_2102_00319_b200.configs import BATCH, CONFIGS, IMAGE_SEEDS, NETWORKS, cnn_images
        from paper_2102_00319_b200.model import ledger, weight_entropies
        from paper_2102_00319_b200 import percell

        self.map = threaded_map
        self.percell = percell
        self.config = config
        cfg = CONFIGS[config]
        be = OracleBackend(cfg.params(), cfg.base_extra_bits)
        keys = be.keygen()
        be.set_eval_key(keys)
        self.be, self.keys = be, keys
        net = self.net = NETWORKS[config]()
        S = self.shards = shards or self.SHARDS[config]
        trace = ledger(net, be.chain, be.canonical_scale)
        self.batch = min(BATCH[config], be.slots)
        tags = weight_entropies(net)
        slots = be.slots
        shapes = net.shapes()
        self.plan = self.sample_plan(net, S)  # (kind, layer index, units in the sample, units in the layer)
        # first conv: the input pixels its sampled cells cover, encrypted like pack_batch
        conv0 = net.layers[0]
        _, om, on = shapes[0]
        F = conv0.filters
        n0 = self.plan[0][2]
        self.conv0_cells = [(u % F, (u // F) // on, (u // F) % on) for u in range(n0)]
        rows = max(i for _, i, _ in self.conv0_cells) * conv0.stride + conv0.kernel[0]
        m, n = net.input_dims
        imgs = cnn_images(self.batch, IMAGE_SEEDS[config])
        cells = [(i, j) for i in range(rows) for j in range(n)]
        self.x = dict(zip(cells, threaded_map(
            lambda ij: be.encrypt(imgs[:, ij[0], ij[1]], keys, entropy=ij[0] * n + ij[1]), cells)))
        # weights of the sampled cells, encrypted and dropped to their use-site level (encrypt_network)
        self.w = {}
        for kind, li, cnt, _ in self.plan:
            layer = net.layers[li]
            if kind == "conv":
                idx = list(np.ndindex(*layer.weights.shape))
            elif kind == "dense":
                idx = [(i, r) for i in range(layer.in_dim) for r in range(cnt)]
            else:
                continue
            lvl = trace[li]["level"]
            enc = threaded_map(lambda t: be.drop_to_level(
                be.encrypt(np.full(slots, float(layer.weights[t])), keys, entropy=int(tags[li][t])), lvl), idx)
            self.w[li] = dict(zip(idx, enc))
        self.trace = trace
        self.cores = os.cpu_count() or 1

    @staticmethod
    def sample_plan(net, S: int) -> list:
        """Per layer with work: (kind, layer index, units per 1/S sample, units in the layer);
        units are conv cells, activation cells, pool windows and FC outputs."""
        from paper_2102_00319_b200.model import Conv, Dense, PolyAct, Square, SumPool

        shapes = net.shapes()
        plan = []
        dims = (1, *net.input_dims)
        for li, layer in enumerate(net.layers):
            if isinstance(layer, (Conv, SumPool)):
                units = shapes[li][0] * shapes[li][1] * shapes[li][2]
            elif isinstance(layer, (Square, PolyAct)):
                units = dims[0] * dims[1] * dims[2]
            elif isinstance(layer, Dense):
                units = layer.out_dim
            else:
                units = 0
            if units:
                if units % S:
                    raise ValueError(f"layer {li} ({layer.kind}) has {units} units, not divisible by {S}")
                plan.append((layer.kind, li, units // S, units))
            if len(shapes[li]) == 3:
                dims = shapes[li]
        return plan

    def step(self) -> float:
        """Run the sample once; returns its wall-clock seconds."""
        be, net = self.be, self.net
        t0 = time.perf_counter()
        prev = None
        for kind, li, cnt, _ in self.plan:
            layer = net.layers[li]
            if kind == "conv":
                C, (P, Q), s = layer.channels, layer.kernel, layer.stride
                W = self.w[li]
                if prev is None:
                    def cell(u, W=W, C=C, P=P, Q=Q, s=s):
                        f, i, j = self.conv0_cells[u]
                        acc = None
                        for c in range(C):
                            for dp in range(P):
                                for dq in range(Q):
                                    t = be.mul_ct_ct_raw(self.x[(i * s + dp, j * s + dq)], W[(f, c, dp, dq)])
                                    acc = t if acc is None else be.raw_add(acc, t)
                        return be.raw_finalize(acc)
                else:
                    F = layer.filters

                    def cell(u, W=W, C=C, P=P, Q=Q, F=F, src=prev):
                        f = u % F
                        acc = None
                        for tap, (c, dp, dq) in enumerate(np.ndindex(C, P, Q)):
                            t = be.mul_ct_ct_raw(src[(u * C * P * Q + tap) % len(src)], W[(f, c, dp, dq)])
                            acc = t if acc is None else be.raw_add(acc, t)
                        return be.raw_finalize(acc)
                prev = self.map(cell, range(cnt))
            elif kind == "square":
                prev = self.map(lambda y: be.mul_ct_ct(y, y), prev[:cnt])
            elif kind == "polyact":
                pts = self.percell.act_plaintexts(be, layer, prev[0].level, prev[0].scale)
                prev = self.map(lambda y: self.percell.poly_act_cell(be, y, *pts), prev[:cnt])
            elif kind == "sumpool":
                def window(u, src=prev):
                    acc = src[(4 * u) % len(src)]
                    for d in range(1, 4):
                        acc = be.add_ct_ct(acc, src[(4 * u + d) % len(src)])
                    return acc
                prev = self.map(window, range(cnt))
            elif kind == "dense":
                # the reference executor's stage 2 (executor.py:241-267): class x input-chunk
                # tasks of raw partial dot products, combined in fixed order, then finalized
                W, din = self.w[li], layer.in_dim
                J = max(1, min(din, self.cores // cnt))
                bounds = [(din * c) // J for c in range(J + 1)]

                def part(rc, W=W, src=prev):
                    r, c = divmod(rc, J)
                    acc = None
                    for i in range(bounds[c], bounds[c + 1]):
                        t = be.mul_ct_ct_raw(src[i % len(src)], W[(i, r)])
                        acc = t if acc is None else be.raw_add(acc, t)
                    return acc
                parts = self.map(part, range(cnt * J))

                def combine(r):
                    acc = parts[r * J]
                    for c in range(1, J):
                        acc = be.raw_add(acc, parts[r * J + c])
                    return be.raw_finalize(acc)
                prev = self.map(combine, range(cnt))
        return time.perf_counter() - t0

    def describe(self) -> str:
        parts = ", ".join(f"{kind} {cnt}/{tot}" for kind, _, cnt, tot in self.plan)
        return (f"{self.config}: 1/{self.shards} of every layer per step ({parts}) = {self.batch // self.shards} "
                f"images-equivalent; C oracle of the reference kernels in the reference op order, "
                f"ThreadPool over {self.cores} host threads")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(args) -> dict:
    """One bounded sample of the same workload on the CPU oracle (rank 0, N = 1)."""
    s = CpuSample(args.config)
    s.step()  # numpy / thread-pool warm-up
    sec = s.step()
    return {
        "value": round(s.batch / s.shards / sec, 3),
        "unit": UNIT,
        "cores": s.cores,
        "kind": "port",
        "cpu": cpu_model(),
        "sample": s.describe(),
        "sample_seconds": round(sec, 3),
        "cfg1_ops": cfg1_cpu_ops(),
    }


def cfg1_cpu_ops(pairs: int = 256) -> dict:
    """Config 1 primitive ops/s on the CPU oracle over all host threads."""
    import warnings

    warnings.simplefilter("ignore")
    from oracle.ckks_oracle import OracleBackend, threaded_map
    from paper_2102_00319_b200.configs import CONFIGS, cfg1_pairs

    cfg = CONFIGS["cfg1"]
    be = OracleBackend(cfg.params(), cfg.base_extra_bits)
    keys = be.keygen(galois_steps=(1,))
    be.set_eval_key(keys)
    be.set_galois_key(keys)
    xs, ys = cfg1_pairs(be.slots, pairs)
    a = threaded_map(lambda i: be.encrypt(xs[i], keys, entropy=i), range(pairs))
    b = threaded_map(lambda i: be.encrypt(ys[i], keys, entropy=pairs + i), range(pairs))
    pts = threaded_map(lambda i: be.encode_plain(ys[i]), range(pairs))
    ops = {
        "mul_relin_rescale": lambda i: be.mul_ct_ct(a[i], b[i]),
        "add_ct_ct": lambda i: be.add_ct_ct(a[i], b[i]),
        "mul_ct_pt_rescale": lambda i: be.mul_ct_pt(a[i], pts[i]),
        "rotate_by_1": lambda i: be.rotate(a[i], 1),
    }
    out = {}
    for name, fn in ops.items():
        threaded_map(fn, range(16))
        t0 = time.perf_counter()
        threaded_map(fn, range(pairs))
        out[name] = round(pairs / (time.perf_counter() - t0), 1)
    out["unit"] = "ops/s"
    out["threads"] = os.cpu_count() or 1
    return out


def run_reference(args) -> None:
    """The reference algorithm on the host cores: each step runs one proportional sample
    (CpuSample: 1/S of every layer of the same network, batch and level schedule as the
    b200 arm); ms_per_step is that sample's measured wall time and value the images it
    stands for (batch / S) divided by that time."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    s = CpuSample(args.config)
    # CPU steps need no warm-up (no JIT, no caches worth priming at these sizes; the
    # oracle library is loaded and the thread pool exercised while encrypting the
    # sample's inputs): a cfg4 sample step is ~15 s on 16 cores, so W extra steps would
    # only lengthen the run
    secs = [s.step() for _ in range(args.steps)]
    step_s = sum(secs) / len(secs)
    value = s.batch / s.shards / step_s
    line = {
        "metric": BASELINE_METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "impl": "reference",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "warmup_run": 0,
        "ms_per_step": round(step_s * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": workload_name(args.config, s.net, s.be.n, s.be.chain.num_levels, s.batch),
                   "batch_per_gpu": s.batch, "images_per_step": s.batch // s.shards},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": s.cores, "kind": "port",
                         "cpu": cpu_model(), "sample": s.describe()},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def net_sigma(config: str) -> float:
    return 0.05 if config == "cfg4" else 0.1


def workload_name(config: str, net, n: int, levels: int, batch: int) -> str:
    return (f"{config}: encrypted CNN {' -> '.join(l.kind for l in net.layers)}, N={n}, {levels} levels, "
            f"{batch} images/GPU")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg2", "cfg3", "cfg4", "cfg5"],
                    help="BASELINE config; cfg4 (N = 32768, the largest single-GPU config) is the headline; "
                         "cfg5 = the cfg4 network on 4 batches sharded over the ranks (strong scaling)")
    ap.add_argument("--pipelines", type=int, default=None,
                    help="concurrent inference pipelines (streams) per GPU (default: per config)")
    ap.add_argument("--no-prof", action="store_true", help="no per-kernel events in the timed region")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-cfg1", action="store_true")
    ap.add_argument("--skip-u64", action="store_true", help="no e2e run in the reference's u64 payload format")
    args = ap.parse_args()
    if args.pipelines is None:
        args.pipelines = PIPELINES.get(args.config, 1)
    if args.impl == "reference":
        if args.config == "cfg5":
            args.config = "cfg4"  # the reference arm times the same network per batch
        run_reference(args)
    elif args.config == "cfg5":
        run_cfg5(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
