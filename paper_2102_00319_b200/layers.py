"""Batched encrypted-CNN layer evaluator: one launch sequence per layer.

The reference evaluates a layer as nested Python loops of per-ciphertext ops
(`/root/reference/pkg/src/hecnn/layers.py:92-294`, driven by
`executor.py:161-279` on a thread pool).  Here every layer is a handful of
launches over *all* of its independent ciphertexts:

* conv          -> ``heb_conv``: fused tensor over every window (weights staged in
                   shared memory), one batched relinearise + rescale, bias;
* dense         -> ``heb_fc``: index-driven tensor (lazy 128-bit accumulation),
                   relinearise + rescale, bias;
* square        -> ``heb_square`` (tensor + relinearise + rescale);
* poly act      -> ``heb_poly_act`` (reference ``approx_relu_cell``: square, two
                   ct x pt rescales, adds);
* sum pool      -> ``heb_sumpool`` over the 2x2 windows;
* flatten       -> index remapping only (no data movement).

Ciphertext bits, levels, exact scales, noise estimates and op counters are
identical to running ``percell.run_network`` (the reference op sequence) on
the same backend.  Feature maps are ``CipherBatch`` objects whose items are
laid out channel-major: item = c*(m*n) + i*n + j.
"""

from __future__ import annotations

import time

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _lib
from .backend import B200Backend, CipherBatch, ct_desc
from .contract import noise_sum
from .errors import DepthExhausted, ScaleMismatch
from .model import BIAS_ENTROPY_BASE, WINDOW_ORDER, Conv, Dense, Flatten, Network, PolyAct, SumPool, Square, ledger, weight_entropies
from .percell import act_plaintexts


@dataclass
class EncryptedNetworkBatch:
    net: Network
    weights: list   # per layer: CipherBatch of the flattened weight tensor (or None)
    biases: list    # per layer: CipherBatch (or None)
    trace: list


def encrypt_network(backend: B200Backend, net: Network, key) -> EncryptedNetworkBatch:
    """Model-owner encryption with the same entropy tags as ``percell.encrypt_network``."""
    trace = ledger(net, backend.chain, backend.canonical_scale)
    tags = weight_entropies(net)
    slots = backend.slots
    weights, biases = [], []
    bias_tag = BIAS_ENTROPY_BASE
    for li, layer in enumerate(net.layers):
        in_level = trace[li]["level"]
        out = trace[li + 1]
        if isinstance(layer, (Conv, Dense)):
            w = layer.weights.ravel()
            vals = np.repeat(w[:, None], slots, axis=1)
            wb = backend.encrypt_batch(vals, key, tags[li].ravel())
            weights.append(drop_batch(wb, in_level))
            if layer.bias is not None:
                nb = len(layer.bias)
                bvals = np.repeat(np.asarray(layer.bias, dtype=np.float64)[:, None], slots, axis=1)
                bb = backend.encrypt_batch(bvals, key, bias_tag + np.arange(nb), scale=out["scale"])
                bias_tag += nb
                biases.append(drop_batch(bb, out["level"]))
            else:
                biases.append(None)
        else:
            weights.append(None)
            biases.append(None)
    return EncryptedNetworkBatch(net, weights, biases, trace)


def encrypt_images(backend: B200Backend, images: np.ndarray, key) -> CipherBatch:
    """Client packing: cell (i, j) holds pixel (i, j) of every image, entropy = i*n + j."""
    imgs = np.asarray(images, dtype=np.float64)
    _, m, n = imgs.shape
    vals = imgs.reshape(imgs.shape[0], m * n).T  # (cells, batch)
    return backend.encrypt_batch(vals, key, np.arange(m * n))


def drop_batch(b: CipherBatch, level: int) -> CipherBatch:
    if level > b.level:
        raise ValueError("cannot raise a ciphertext's level")
    return CipherBatch(b.buf, level, b.scale, b.noise_bits)


class LayerEvaluator:
    """Runs an ``EncryptedNetworkBatch`` over a packed input batch on one device."""

    def __init__(self, backend: B200Backend, fused_conv: bool = True):
        self.be = backend
        self.ctx = backend.ctx
        self.fused_conv = fused_conv
        self._idx_cache: dict = {}
        self._unique: dict = {}
        self._streams: dict = {}
        self._graphs: dict = {}
        self._pt_cache: dict = {}
        self._inbufs: dict = {}

    # -- primitives -------------------------------------------------------------------
    def _idx(self, key, builder) -> torch.Tensor:
        t = self._idx_cache.get(key)
        if t is None:
            host = np.ascontiguousarray(builder(), dtype=np.int32)
            t = torch.from_numpy(host).to(self.be.dev)
            self._idx_cache[key] = t
            if host.ndim == 3:  # (a_idx, b_idx) pair: remember operand reuse for the roofline
                self._unique[t[0].data_ptr()] = (len(np.unique(host[0])), len(np.unique(host[1])))
        return t

    def _empty(self, count: int, comps: int, k: int) -> torch.Tensor:
        return self.ctx.empty(count, comps, k, self.be.n)

    def dot(self, a: CipherBatch, b: CipherBatch, ia: torch.Tensor, ib: torch.Tensor, taps: int, n_out: int):
        """raw_o = sum_t a[ia] (x) b[ib]; returns (raw buffer, level, scale, noise)."""
        if a.scale * b.scale != a.scale * b.scale:  # pragma: no cover
            raise ScaleMismatch("unreachable")
        lvl = min(a.level, b.level)
        if lvl < 1:
            raise DepthExhausted("ciphertext-ciphertext multiply at level 0")
        k = lvl + 1
        raw = self._empty(n_out, 3, k)
        ua, ub = self._unique.get(ia.data_ptr(), (n_out * taps, n_out * taps))
        _lib.prof_next_bytes(8.0 * self.be.n * k * (2 * ua + 2 * ub + 3 * n_out))
        self.ctx.call("heb_dot_tensor", a.desc(), b.desc(), ia.data_ptr(), ib.data_ptr(), taps, ct_desc(raw), n_out, k,
                      self.ctx.stream)
        term = noise_sum(a.noise_bits, b.noise_bits)
        if term > float("-inf"):
            term += 1.0
        noise = term + math.log2(taps) if term > float("-inf") else term
        self.be.counters.bump(ctct_mult=n_out * taps, ctct_add=n_out * (taps - 1))
        return raw, lvl, a.scale * b.scale, noise

    def conv_layer(self, x: CipherBatch, w: CipherBatch, bias, c_in: int, m: int, n: int, layer: Conv, n_out: int,
                   taps: int) -> CipherBatch:
        """The whole conv layer (tensor over every window, relinearise + rescale, bias) as
        one heb_conv call; weights staged in shared memory by the fused tensor kernel."""
        lvl = min(x.level, w.level)
        if lvl < 1:
            raise DepthExhausted("ciphertext-ciphertext multiply at level 0")
        term = noise_sum(x.noise_bits, w.noise_bits)
        if term > float("-inf"):
            term += 1.0
        noise = term + math.log2(taps) if term > float("-inf") else term
        out_level, scale, noise = self._finalize_meta(lvl, x.scale * w.scale, noise)
        in_c = bias is not None and bias.level >= out_level
        if bias is not None and bias.scale != scale:
            raise ScaleMismatch("batched add requires equal scales")
        out = self._empty(n_out, 2, lvl)
        evk = self.be._require_eval_key().evaluation
        p, q = layer.kernel
        bdesc = bias.desc() if in_c else _lib.HebCt(None, 0, 0)
        self.ctx.call("heb_conv", x.desc(), w.desc(), bdesc, ct_desc(out), c_in, m, n, layer.filters, p, q,
                      layer.stride, lvl, evk.prep.data_ptr(), self.ctx.stream)
        self.be.counters.bump(ctct_mult=n_out * taps, ctct_add=n_out * (taps - 1))
        y = CipherBatch(out, out_level, scale, noise)
        if bias is None:
            return y
        per = n_out // layer.filters
        if not in_c:  # bias below the output level: the sum drops to the bias level
            for f in range(layer.filters):
                self.add(y, bias_item(bias, f), b_broadcast=True, count=per, a_off=f * per, out=y, out_off=f * per)
        else:
            self.be.counters.bump(ctct_add=n_out)
        return CipherBatch(y.buf, min(y.level, bias.level), y.scale, noise_sum(y.noise_bits, bias.noise_bits))

    def finalize(self, raw: torch.Tensor, level: int, scale: Fraction, noise: float) -> CipherBatch:
        evk = self.be._require_eval_key().evaluation
        n_out = raw.shape[0]
        out = self._empty(n_out, 2, level)
        self.ctx.call("heb_relin_rescale", ct_desc(raw), evk.prep.data_ptr(), ct_desc(out), n_out, level,
                      self.ctx.stream)
        return CipherBatch(out, *self._finalize_meta(level, scale, noise))

    def add(self, a: CipherBatch, b: CipherBatch, b_broadcast: bool = False, count: int | None = None,
            a_off: int = 0, out: CipherBatch | None = None, out_off: int = 0) -> CipherBatch:
        if a.scale != b.scale:
            raise ScaleMismatch("batched add requires equal scales")
        lvl = min(a.level, b.level)
        k = lvl + 1
        n = count if count is not None else a.count
        dst = out.buf if out is not None else self._empty(n, 2, k)
        da = ct_desc(a.buf)
        da.data = a.buf[a_off].data_ptr()
        db = ct_desc(b.buf)
        if b_broadcast:
            db.ct_stride = 0
        dd = ct_desc(dst)
        dd.data = dst[out_off].data_ptr()
        self.ctx.call("heb_add", da, db, dd, n, 2, k, self.ctx.stream)
        self.be.counters.bump(ctct_add=n)
        return CipherBatch(dst, lvl, a.scale, noise_sum(a.noise_bits, b.noise_bits))

    # -- ledger (level / exact scale / noise) of each op, shared by the primitive and the
    #    layer entry points so both paths produce identical CipherBatch metadata ----------
    def _finalize_meta(self, level: int, scale: Fraction, noise: float) -> tuple:
        new_scale = self.be._rescale_scale(scale, level)
        return level - 1, new_scale, max(noise, self.be._round_noise_bits(new_scale))

    @staticmethod
    def _square_noise(y: CipherBatch) -> float:
        if y.noise_bits == float("-inf"):
            return y.noise_bits
        return noise_sum(y.noise_bits, y.noise_bits) + 1.0

    def _mul_plain_meta(self, y_level: int, y_scale: Fraction, y_noise: float, pt, values_mag: float) -> tuple:
        if y_level < 1:
            raise DepthExhausted("ciphertext-plaintext multiply at level 0")
        scale = self.be._rescale_scale(y_scale * pt.scale, y_level)
        noise = y_noise + max(0.0, math.log2(max(values_mag, 1e-300))) + 1.0
        return y_level - 1, scale, max(noise, self.be._round_noise_bits(scale))

    def square(self, y: CipherBatch) -> CipherBatch:
        """x^2 activation: heb_square (tensor + relinearise + rescale) in one call."""
        if y.level < 1:
            raise DepthExhausted("ciphertext-ciphertext multiply at level 0")
        lvl, scale, noise = self._finalize_meta(y.level, y.scale * y.scale, self._square_noise(y))
        out = self._empty(y.count, 2, y.level)
        evk = self.be._require_eval_key().evaluation
        self.ctx.call("heb_square", y.desc(), ct_desc(out), y.count, y.level, evk.prep.data_ptr(), self.ctx.stream)
        self.be.counters.bump(ctct_mult=y.count)
        return CipherBatch(out, lvl, scale, noise)

    def mul_plain(self, y: CipherBatch, pt, values_mag: float) -> CipherBatch:
        meta = self._mul_plain_meta(y.level, y.scale, y.noise_bits, pt, values_mag)
        out = self._empty(y.count, 2, y.level)
        self.ctx.call("heb_mul_plain_rescale", y.desc(), pt.payload.rows.data_ptr(), 0, ct_desc(out), y.count,
                      y.level, self.ctx.stream)
        self.be.counters.bump(ctpt_mult=y.count)
        return CipherBatch(out, *meta)

    def add_plain(self, y: CipherBatch, pt) -> CipherBatch:
        if pt.scale != y.scale:
            raise ScaleMismatch("plaintext addend must be encoded at the ciphertext scale")
        out = self._empty(y.count, 2, y.k)
        self.ctx.call("heb_add_plain", y.desc(), pt.payload.rows.data_ptr(), 0, ct_desc(out), y.count, y.k,
                      self.ctx.stream)
        self.be.counters.bump(ctpt_add=y.count)
        return CipherBatch(out, y.level, y.scale, noise_sum(y.noise_bits, self.be._encode_noise_bits()))

    # -- layers --------------------------------------------------------------------------
    def conv(self, x: CipherBatch, dims: tuple[int, int, int], layer: Conv, w: CipherBatch, bias) -> tuple:
        c_in, m, n = dims
        p, q = layer.kernel
        s = layer.stride
        om, on = layer.out_dims(m, n)
        F = layer.filters
        taps = c_in * p * q
        n_out = F * om * on

        def build():
            f, i, j, c, dp, dq = np.meshgrid(np.arange(F), np.arange(om), np.arange(on), np.arange(c_in),
                                             np.arange(p), np.arange(q), indexing="ij")
            ia = c * (m * n) + (i * s + dp) * n + (j * s + dq)
            ib = ((f * c_in + c) * p + dp) * q + dq
            return np.stack([ia.reshape(n_out, taps), ib.reshape(n_out, taps)])

        if self.fused_conv:
            return self.conv_layer(x, w, bias, c_in, m, n, layer, n_out, taps), (F, om, on)
        else:
            idx = self._idx(("conv", dims, layer.kernel, s, F), build)
            raw, lvl, scale, noise = self.dot(x, w, idx[0], idx[1], taps, n_out)
        y = self.finalize(raw, lvl, scale, noise)
        if bias is not None:
            for f in range(F):
                self.add(y, bias_item(bias, f), b_broadcast=True, count=om * on, a_off=f * om * on, out=y,
                         out_off=f * om * on)
            y = CipherBatch(y.buf, min(y.level, bias.level), y.scale, noise_sum(y.noise_bits, bias.noise_bits))
        return y, (F, om, on)

    def poly_act(self, y: CipherBatch, act: PolyAct) -> CipherBatch:
        key = ("act", act.folded(), y.level, y.scale)
        pts = self._pt_cache.get(key)
        if pts is None:  # encoded once per (activation, level, scale); constant plaintexts
            pts = self._pt_cache[key] = act_plaintexts(self.be, act, y.level, y.scale)
        pt_quad, pt_lin, pt_const = pts
        c0, c1, c2 = act.folded()
        # ledger of approx_relu_cell: t = y^2, quad = t (*) pt_quad, lin = y (*) pt_lin,
        # r = quad + lin (at quad's level), r + pt_const
        t_meta = self._finalize_meta(y.level, y.scale * y.scale, self._square_noise(y))
        q_lvl, q_scale, q_noise = self._mul_plain_meta(*t_meta, pt_quad, abs(c2))
        l_lvl, l_scale, l_noise = self._mul_plain_meta(y.level, y.scale, y.noise_bits, pt_lin, abs(c1))
        if q_scale != l_scale:
            raise ScaleMismatch("batched add requires equal scales")
        if pt_const.scale != q_scale:
            raise ScaleMismatch("plaintext addend must be encoded at the ciphertext scale")
        lvl = min(q_lvl, l_lvl)
        noise = noise_sum(noise_sum(q_noise, l_noise), self.be._encode_noise_bits())
        out = self._empty(y.count, 2, lvl + 1)
        evk = self.be._require_eval_key().evaluation
        self.ctx.call("heb_poly_act", y.desc(), pt_quad.payload.rows.data_ptr(), pt_lin.payload.rows.data_ptr(),
                      pt_const.payload.rows.data_ptr(), ct_desc(out), y.count, y.level, evk.prep.data_ptr(),
                      self.ctx.stream)
        self.be.counters.bump(ctct_mult=y.count, ctpt_mult=2 * y.count, ctct_add=y.count, ctpt_add=y.count)
        return CipherBatch(out, lvl, q_scale, noise)

    def sum_pool(self, y: CipherBatch, dims: tuple[int, int, int]) -> tuple:
        c_in, m, n = dims
        om, on = m // 2, n // 2
        n_out = c_in * om * on

        def build():
            c, i, j = np.meshgrid(np.arange(c_in), np.arange(om), np.arange(on), indexing="ij")
            terms = [c * (m * n) + (2 * i + di) * n + (2 * j + dj) for di, dj in WINDOW_ORDER]
            return np.stack([t.ravel() for t in terms], axis=1)

        del build  # the window indices are arithmetic inside heb_sumpool (WINDOW_ORDER sums are exact mod p)
        out = self._empty(n_out, 2, y.k)
        self.ctx.call("heb_sumpool", y.desc(), ct_desc(out), c_in, m, n, y.level, self.ctx.stream)
        self.be.counters.bump(ctct_add=3 * n_out)
        noise = y.noise_bits
        for _ in range(3):
            noise = noise_sum(noise, y.noise_bits)
        return CipherBatch(out, y.level, y.scale, noise), (c_in, om, on)

    def dense(self, x: CipherBatch, flat_map: np.ndarray, layer: Dense, w: CipherBatch, bias) -> CipherBatch:
        din, dout = layer.in_dim, layer.out_dim

        def build():
            ia = np.broadcast_to(flat_map[None, :], (dout, din))
            ib = np.arange(din)[None, :] * dout + np.arange(dout)[:, None]
            return np.stack([ia, ib])

        idx = self._idx(("dense", din, dout, flat_map.tobytes()), build)
        lvl = min(x.level, w.level)
        if lvl < 1:
            raise DepthExhausted("ciphertext-ciphertext multiply at level 0")
        term = noise_sum(x.noise_bits, w.noise_bits)
        if term > float("-inf"):
            term += 1.0
        noise = term + math.log2(din) if term > float("-inf") else term
        out_level, scale, noise = self._finalize_meta(lvl, x.scale * w.scale, noise)
        in_c = bias is not None and bias.level >= out_level
        if bias is not None and bias.scale != scale:
            raise ScaleMismatch("batched add requires equal scales")
        out = self._empty(dout, 2, lvl)
        evk = self.be._require_eval_key().evaluation
        ua, ub = self._unique.get(idx[0].data_ptr(), (dout * din, dout * din))
        _lib.prof_next_bytes(8.0 * self.be.n * (lvl + 1) * (2 * ua + 2 * ub + 3 * dout))
        self.ctx.call("heb_fc", x.desc(), w.desc(), idx[0].data_ptr(), idx[1].data_ptr(), din,
                      bias.desc() if in_c else _lib.HebCt(None, 0, 0), ct_desc(out), dout, lvl, evk.prep.data_ptr(),
                      self.ctx.stream)
        self.be.counters.bump(ctct_mult=dout * din, ctct_add=dout * (din - 1))
        y = CipherBatch(out, out_level, scale, noise)
        if bias is None:
            return y
        if not in_c:
            return self.add(y, bias)
        self.be.counters.bump(ctct_add=dout)
        return CipherBatch(out, min(y.level, bias.level), scale, noise_sum(noise, bias.noise_bits))

    def run(self, enc: EncryptedNetworkBatch, x: CipherBatch, deltas: list | None = None) -> CipherBatch:
        """One inference over the batch; ``deltas`` (optional) receives (layer kind, counter
        delta) per layer, the runtime side of ``analyzer.verify_against_runtime``."""
        net = enc.net
        dims = (1, *net.input_dims)
        flat_map = None
        for li, layer in enumerate(net.layers):
            before = self.be.counters.snapshot() if deltas is not None else None
            if isinstance(layer, Conv):
                x, dims = self.conv(x, dims, layer, enc.weights[li], enc.biases[li])
            elif isinstance(layer, Square):
                x = self.square(x)
            elif isinstance(layer, PolyAct):
                x = self.poly_act(x, layer)
            elif isinstance(layer, SumPool):
                x, dims = self.sum_pool(x, dims)
            elif isinstance(layer, Flatten):
                c_in, m, n = dims
                i, j, c = np.meshgrid(np.arange(m), np.arange(n), np.arange(c_in), indexing="ij")
                flat_map = (c * (m * n) + i * n + j).ravel()  # flat[(i*n+j)*C + c] = map[c][i][j]
            elif isinstance(layer, Dense):
                x = self.dense(x, flat_map, layer, enc.weights[li], enc.biases[li])
            if deltas is not None:
                deltas.append((layer.kind, self.be.counters.snapshot() - before))
        return x


    # -- serving: host batches in, host logits out, copies overlapped with compute -----
    def _pipeline_streams(self, kind: str, count: int) -> list:
        """Persistent per-pipeline streams (the caching allocator keeps per-stream pools,
        so reusing streams keeps steady-state steps free of fresh device allocations)."""
        pool = self._streams.setdefault(kind, [])
        while len(pool) < count:
            pool.append(torch.cuda.Stream(self.be.dev))
        return pool[:count]

    def pipeline_stream(self, pipeline: int) -> torch.cuda.Stream:
        """The persistent compute stream of ``pipeline`` (its scratch arena is reused)."""
        return self._pipeline_streams("compute", pipeline + 1)[pipeline]

    def captured(self, enc: EncryptedNetworkBatch, x: CipherBatch, pipeline: int):
        """(graph, output, counter delta) -- one inference of ``x`` captured as a CUDA graph.

        The graph replays every launch of ``run`` (and the stream-ordered scratch
        allocations, as graph memory nodes) with one host call; each pipeline owns its
        graph and private memory pool, so replays of different pipelines may overlap.
        The output batch is overwritten by the next replay of the same graph."""
        key = (id(enc), x.buf.data_ptr(), tuple(x.buf.shape), x.level, pipeline)
        hit = self._graphs.get(key)
        if hit is None:
            st = self._pipeline_streams("compute", pipeline + 1)[pipeline]
            st.wait_stream(torch.cuda.current_stream(self.be.dev))
            start = self.be.counters.snapshot().__dict__
            with torch.cuda.stream(st):
                self.run(enc, x)  # builds index caches / kernel attributes outside the capture
            st.synchronize()
            graph = torch.cuda.CUDAGraph(keep_graph=True)  # raw graph kept for graph_kernel_launches
            before = self.be.counters.snapshot().__dict__
            with torch.cuda.graph(graph, pool=torch.cuda.graph_pool_handle(), stream=st,
                                  capture_error_mode="thread_local"):
                out = self.run(enc, x)
            after = self.be.counters.snapshot().__dict__
            delta = {f: after[f] - before[f] for f in after}
            # warm-up and capture are not user-visible evaluations: take their tallies back
            self.be.counters.bump(**{f: start[f] - after[f] for f in after})
            graph.instantiate()
            hit = self._graphs[key] = (graph, out, delta, enc, x.buf)  # keep the captured buffers alive
        return hit[:3]

    def drop_graphs(self) -> None:
        """Destroy every captured graph; their streams' scratch may then be released."""
        streams = {self._pipeline_streams("compute", key[-1] + 1)[key[-1]] for key in self._graphs}
        self._graphs.clear()
        torch.cuda.synchronize(self.be.dev)
        for st in streams:
            self.ctx.call("heb_ctx_clear_captured", st.cuda_stream)

    def graph_kernel_launches(self, enc: EncryptedNetworkBatch, x: CipherBatch, pipeline: int = 0) -> int:
        """Kernel nodes of the captured CUDA graph of one inference (= kernel launches per
        replayed step; every kernel in it is launched by libheb200)."""
        from cuda.bindings import runtime as rt

        graph = self.captured(enc, x, pipeline)[0]
        g = graph.raw_cuda_graph()
        err, _, count = rt.cudaGraphGetNodes(g, 0)
        err, nodes, count = rt.cudaGraphGetNodes(g, count)
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"cudaGraphGetNodes: {err}")
        kernels = 0
        for nd in nodes[:count]:
            err, kind = rt.cudaGraphNodeGetType(nd)
            kernels += int(kind == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel)
        return kernels

    def _replay(self, runner) -> CipherBatch:
        graph, out, delta = runner
        graph.replay()
        self.be.counters.bump(**delta)  # the op tallies a host-issued run would have made
        return out

    def run_stream(self, enc: EncryptedNetworkBatch, host_inputs, level: int, scale: Fraction, noise: float,
                   host_outputs, on_output=None, pipelines: int = 2, graphs: bool = True,
                   unpacked_shape: tuple | None = None) -> None:
        """Evaluate a sequence of pinned host input batches ((B, 2, K, N) int64 tensors).

        Batches are dealt round-robin to ``pipelines`` independent pipelines, each with
        its own device input buffer, copy stream and compute stream: the host->device
        copy of one pipeline's next batch overlaps the other pipelines' evaluation, and
        the pipelines' kernels fill each other's tails on the SMs.  The logits of batch
        s are copied back into ``host_outputs[s]`` (pinned, (out, 2, k, N)).  On return
        the caller's current stream is ordered after all the work.  ``graphs``: replay
        one captured CUDA graph per pipeline instead of re-issuing every launch.
        ``unpacked_shape``: the host inputs are in the bit-packed wire format
        (``B200Backend.pack_batch``) of batches of this (B, 2, K, N) shape; they are
        unpacked on the device, and the next copy of a pipeline overlaps its compute.
        Unpacked (u64 payload) inputs also land in a per-pipeline staging buffer and are
        moved into the graph's input buffer by a device copy, so that a pipeline's next
        host->device copy does not wait for its whole evaluation (the captured graph reads
        its input buffer until the first layer is done); without room for the staging
        buffer the copy goes straight into the input buffer as before.
        """
        caller = torch.cuda.current_stream(self.be.dev)
        P = max(1, pipelines)
        comp = self._pipeline_streams("compute", P)
        copy = self._pipeline_streams("copy", P)
        packed = unpacked_shape is not None
        shape = tuple(unpacked_shape) if packed else tuple(host_inputs[0].shape)
        stage = [None] * P
        if packed:
            for p in range(P):
                key = (("packed",) + tuple(host_inputs[0].shape), p)
                if key not in self._inbufs:
                    self._inbufs[key] = torch.empty(tuple(host_inputs[0].shape), dtype=host_inputs[0].dtype,
                                                    device=self.be.dev)
                stage[p] = self._inbufs[key]
        else:
            try:
                for p in range(P):
                    key = (("staged",) + shape, p)
                    if key not in self._inbufs:
                        self._inbufs[key] = torch.empty(shape, dtype=host_inputs[0].dtype, device=self.be.dev)
                    stage[p] = self._inbufs[key]
            except torch.cuda.OutOfMemoryError:
                for p in range(P):
                    self._inbufs.pop((("staged",) + shape, p), None)
                stage = [None] * P
        staged = all(b is not None for b in stage)
        bufs = []
        for p in range(P):  # persistent per-pipeline device inputs (graph-captured addresses)
            b = self._inbufs.get((shape, p))
            if b is None:
                b = self._inbufs[(shape, p)] = torch.empty(shape, dtype=host_inputs[0].dtype, device=self.be.dev)
            bufs.append(b)
        runners = [self.captured(enc, CipherBatch(bufs[p], level, scale, noise), p) if graphs else None
                   for p in range(P)]
        for st in comp + copy:
            st.wait_stream(caller)
        copied = [torch.cuda.Event() for _ in range(P)]
        consumed = [torch.cuda.Event() for _ in range(P)]
        for s in range(len(host_inputs)):
            p = s % P
            with torch.cuda.stream(copy[p]):
                if s >= P:
                    copy[p].wait_event(consumed[p])
                (stage[p] if staged else bufs[p]).copy_(host_inputs[s], non_blocking=True)
                copied[p].record(copy[p])
            with torch.cuda.stream(comp[p]):
                comp[p].wait_event(copied[p])
                if staged:
                    if packed:
                        self.be.unpack_into(stage[p], bufs[p], level + 1)
                    else:
                        bufs[p].copy_(stage[p], non_blocking=True)
                    consumed[p].record(comp[p])  # staging buffer free: next copy may start
                if graphs:
                    out = self._replay(runners[p])
                else:
                    out = self.run(enc, CipherBatch(bufs[p], level, scale, noise))
                if not staged:
                    consumed[p].record(comp[p])
                host_outputs[s].copy_(out.buf[:, :, : out.k], non_blocking=True)
                if on_output is not None:
                    on_output(s, out)
        for st in comp + copy:
            caller.wait_stream(st)

    def drop_input_buffers(self) -> None:
        """Free the device staging buffers of host inputs (``run_stream``); the
        unpacked per-pipeline inputs stay (captured graphs hold their addresses)."""
        for key in [k for k in self._inbufs if isinstance(k[0], tuple) and k[0][:1] in (("packed",), ("staged",))]:
            del self._inbufs[key]

    def run_many(self, enc: EncryptedNetworkBatch, x: CipherBatch, steps: int, pipelines: int = 2,
                 on_output=None, marks: list | None = None, graphs: bool = True) -> None:
        """Evaluate ``steps`` device-resident batches over ``pipelines`` concurrent streams
        (``graphs``: one captured CUDA graph per pipeline, see ``captured``).
        ``marks`` (diagnostics): receives (pipeline, start event, end event, host time) per step."""
        caller = torch.cuda.current_stream(self.be.dev)
        P = max(1, pipelines)
        comp = self._pipeline_streams("compute", P)
        runners = [self.captured(enc, x, p) for p in range(P)] if graphs else None
        for st in comp:
            st.wait_stream(caller)
        for s in range(steps):
            p = s % P
            with torch.cuda.stream(comp[p]):
                if marks is not None:
                    b, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    b.record()
                if graphs:
                    out = self._replay(runners[p])
                else:
                    out = self.run(enc, x)
                if on_output is not None:
                    on_output(s, out)
                if marks is not None:
                    e.record()
                    marks.append((p, b, e, time.perf_counter()))
        for st in comp:
            caller.wait_stream(st)

    # -- cells-mode sharding (sharding.py): one batch split over ranks -----------------
    def run_cells_shard(self, enc: EncryptedNetworkBatch, x: CipherBatch, units) -> tuple:
        """This rank's FC raw partials (out_dim, 3, k, N) over its (filter, pool row) units."""
        from . import sharding as sh

        net = enc.net
        lay = sh.CellsLayout.of(net)
        conv, act, dense = net.layers[0], net.layers[1], net.layers[4]
        m, n = net.input_dims
        C = conv.channels
        p, q = conv.kernel
        s = conv.stride
        cells = sh.conv_cells(lay, units)
        key = tuple(units)
        taps = C * p * q

        def build_conv():
            ia, ib = [], []
            for f, i, j in cells:
                ia.append([c * m * n + (i * s + dp) * n + (j * s + dq) for c in range(C) for dp in range(p) for dq in range(q)])
                ib.append([((f * C + c) * p + dp) * q + dq for c in range(C) for dp in range(p) for dq in range(q)])
            return np.stack([np.array(ia), np.array(ib)])

        idx = self._idx(("shard_conv", key), build_conv)
        raw, lvl, scale, noise = self.dot(x, enc.weights[0], idx[0], idx[1], taps, len(cells))
        y = self.finalize(raw, lvl, scale, noise)
        if enc.biases[0] is not None:
            bsel = self._idx(("shard_bias", key), lambda: np.array([f for f, _, _ in cells]))
            bias = enc.biases[0]
            gathered = self._empty(len(cells), 2, bias.k)
            self.ctx.call("heb_gather", bias.desc(), bsel.data_ptr(), ct_desc(gathered), len(cells), 2, bias.k,
                          self.ctx.stream)
            y = self.add(y, CipherBatch(gathered, bias.level, bias.scale, bias.noise_bits))
        y = self.square(y) if isinstance(act, Square) else self.poly_act(y, act)
        pos = {c: t for t, c in enumerate(cells)}
        pooled = sh.pooled_cells(lay, units)
        pidx = self._idx(("shard_pool", key), lambda: np.array(
            [[pos[(f, 2 * r + di, 2 * j + dj)] for di, dj in WINDOW_ORDER] for f, r, j in pooled]))
        pool = self._empty(len(pooled), 2, y.k)
        self.ctx.call("heb_sum_gather", y.desc(), pidx.data_ptr(), 4, ct_desc(pool), len(pooled), 2, y.k,
                      self.ctx.stream)
        self.be.counters.bump(ctct_add=3 * len(pooled))
        pnoise = y.noise_bits
        for _ in range(3):
            pnoise = noise_sum(pnoise, y.noise_bits)
        pooled_b = CipherBatch(pool, y.level, y.scale, pnoise)
        dout = dense.out_dim

        def build_fc():
            ia = np.broadcast_to(np.arange(len(pooled))[None, :], (dout, len(pooled)))
            flat = np.array([sh.flat_of(lay, f, r, j) for f, r, j in pooled])
            ib = flat[None, :] * dout + np.arange(dout)[:, None]
            return np.stack([ia, ib])

        fidx = self._idx(("shard_fc", key), build_fc)
        return self.dot(pooled_b, enc.weights[4], fidx[0], fidx[1], len(pooled), dout)

    # -- bands-mode sharding (sharding.py): a two-conv network's batch split by conv2 rows --
    def run_band_shard(self, enc: EncryptedNetworkBatch, x: CipherBatch, band: tuple[int, int]) -> tuple:
        """This rank's FC raw partials (out_dim, 3, k, N) over conv2 output rows [a, b):
        conv1 + act over the rows the band reads (halo recomputed), conv2 + act over the
        band, the band's cells of every pool window it touches summed in WINDOW_ORDER
        (a window cut by the band boundary is summed partially), FC partial sums over the
        window sums.  Returns (raw, level, scale, noise) like ``dot``."""
        from . import sharding as sh

        net = enc.net
        lay = sh.BandLayout.of(net)
        a, b = band
        c1, act1, c2, act2, dense = (net.layers[i] for i in (0, 1, 2, 3, 6))
        if c1.channels != 1:
            raise ValueError("band sharding reads input rows of a single-channel image grid")
        i0, i1 = lay.input_rows(a, b)
        n_in = lay.in_cols
        xb = CipherBatch(x.buf[i0 * n_in: i1 * n_in], x.level, x.scale, x.noise_bits)  # a contiguous row band
        y, dims = self.conv(xb, (1, i1 - i0, n_in), c1, enc.weights[0], enc.biases[0])
        y = self.square(y) if isinstance(act1, Square) else self.poly_act(y, act1)
        y, (F2, rb, cols) = self.conv(y, dims, c2, enc.weights[2], enc.biases[2])
        y = self.square(y) if isinstance(act2, Square) else self.poly_act(y, act2)
        # full windows first, then the windows cut by a band boundary (2 of their 4 cells)
        wins = sorted(lay.windows(a, b), key=lambda w: -len(w[3]))
        pooled = self._empty(len(wins), 2, y.k)
        off = 0
        for terms in (4, 2):
            sel = [w for w in wins if len(w[3]) == terms]
            if not sel:
                continue
            pidx = self._idx(("band_pool", band, terms), lambda: np.array(
                [[f * rb * cols + (i - a) * cols + jj for i, jj in cells] for f, _, _, cells in sel]))
            self.ctx.call("heb_sum_gather", y.desc(), pidx.data_ptr(), terms, ct_desc(pooled[off: off + len(sel)]),
                          len(sel), 2, y.k, self.ctx.stream)
            self.be.counters.bump(ctct_add=(terms - 1) * len(sel))
            off += len(sel)
        pnoise = y.noise_bits
        for _ in range(3):
            pnoise = noise_sum(pnoise, y.noise_bits)
        dout = dense.out_dim

        def build_fc():
            ia = np.broadcast_to(np.arange(len(wins))[None, :], (dout, len(wins)))
            flat = np.array([lay.flat_of(f, r, j) for f, r, j, _ in wins])
            return np.stack([ia, flat[None, :] * dout + np.arange(dout)[:, None]])

        fidx = self._idx(("band_fc", band), build_fc)
        return self.dot(CipherBatch(pooled, y.level, y.scale, pnoise), enc.weights[6], fidx[0], fidx[1], len(wins),
                        dout)

    def finish_cells(self, enc: EncryptedNetworkBatch, parts: torch.Tensor, level: int, scale: Fraction,
                     noise: float) -> CipherBatch:
        """Add the gathered partials (world, out, 3, k, N) mod p, relinearise + rescale, bias."""
        world, dout = parts.shape[0], parts.shape[1]
        k = parts.shape[3]
        flat = parts.reshape(world * dout, 3, k, self.be.n)
        idx = self._idx(("combine", world, dout), lambda: np.array([[w * dout + r for w in range(world)] for r in range(dout)]))
        raw = self._empty(dout, 3, k)
        self.ctx.call("heb_sum_gather", ct_desc(flat), idx.data_ptr(), world, ct_desc(raw), dout, 3, k, self.ctx.stream)
        self.be.counters.bump(ctct_add=dout * (world - 1))
        y = self.finalize(raw, level, scale, noise + math.log2(world))
        bias = enc.biases[len(enc.net.layers) - 1]  # the dense layer is last
        return self.add(y, bias) if bias is not None else y


def bias_item(bias: CipherBatch, i: int) -> CipherBatch:
    return CipherBatch(bias.buf[i:i + 1], bias.level, bias.scale, bias.noise_bits)
