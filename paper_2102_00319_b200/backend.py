"""B200Backend: the reference ``HEBackend`` plugin contract on sm_100a kernels.

Drop-in for `/root/reference/pkg/src/hecnn/backends/ckks.py` (``CkksBackend``):
same keys, same encryption randomness, same payload bits, with every ring
operation executed by libheb200.so through the C ABI (include/heb200.h).
Host work is limited to what the reference also keeps on the host and what
must stay bit-exact there: PCG64 sampling and the float64 FFT slot encoding
(`hostmath.py`).  There is no CPU fallback: constructing the backend without a
CUDA device or without the built library raises ``DeviceError``.

Payloads live in device memory as int64-typed torch tensors holding the u64
residues (torch is used for allocation/streams only).  A ciphertext payload is
a ``(2, K, N)`` view with ``k = level + 1`` active rows, so ``drop_to_level`` is
a free prefix view exactly as in the reference (`ckks.py:279-282`).  Batched
entry points (``encrypt_batch``, ``CipherBatch`` ops) drive the layer
evaluator in ``layers.py``.
"""

from __future__ import annotations

import itertools
import struct
import threading
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from . import hostmath as hm
from . import serialization as ser
from .contract import CipherVec, HEBackend, KeyMaterial, PlainVec, RawProduct
from .errors import DecryptionOutOfRange, DeviceError, FingerprintMismatch, HecnnError
from .params import HEParams

try:
    import torch
except Exception as exc:  # pragma: no cover - torch is part of the image
    raise DeviceError(f"torch is required for device memory: {exc}")


def _require_cuda(device: int) -> None:
    if not torch.cuda.is_available():
        raise DeviceError("B200Backend needs a CUDA device (no CPU fallback exists)")
    if device >= torch.cuda.device_count():
        raise DeviceError(f"CUDA device {device} not present")


def u64_to_dev(arr: np.ndarray, device) -> "torch.Tensor":
    a = np.ascontiguousarray(arr, dtype=np.uint64).view(np.int64)
    return torch.from_numpy(a).to(device, non_blocking=False)


def dev_to_u64(t: "torch.Tensor") -> np.ndarray:
    return t.detach().contiguous().cpu().numpy().view(np.uint64)


def ct_desc(buf: "torch.Tensor") -> _lib.HebCt:
    """heb_ct descriptor of a (B, C, K, N) batch or a (C, K, N) single item."""
    if buf.dim() == 4:
        return _lib.HebCt(buf.data_ptr(), buf.stride(0), buf.stride(1))
    return _lib.HebCt(buf.data_ptr(), buf.numel(), buf.stride(0))


class DeviceContext:
    """One heb_ctx (device tables for one chain) plus its stream binding."""

    def __init__(self, chain, device: int = 0):
        _require_cuda(device)
        self.device = torch.device("cuda", device)
        self.chain = chain
        self.n = chain.ring_degree
        self.log_n = self.n.bit_length() - 1
        self.num_rows = chain.num_rows
        primes = np.array(chain.primes, dtype=np.uint64)
        psi = np.array(chain.psi, dtype=np.uint64)
        handle = ctypes_void_p()
        with torch.cuda.device(self.device):
            _lib.call("heb_ctx_create", ctypes_byref(handle), device, self.log_n, self.num_rows,
                      primes.ctypes.data, psi.ctypes.data)
        self.handle = handle.value
        self._primes_keepalive = (primes, psi)

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def empty(self, *shape) -> "torch.Tensor":
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    def call(self, name: str, *args) -> None:
        # every entry point runs on this context's device (scratch allocations, kernel
        # attributes and launches follow the calling thread's current device)
        if torch.cuda.current_device() != self.device.index:
            with torch.cuda.device(self.device):
                _lib.call(name, self.handle, *args)
            return
        _lib.call(name, self.handle, *args)

    def set_chunk(self, items: int) -> None:
        self.call("heb_ctx_set_chunk", items)

    def release_scratch(self, stream=None) -> None:
        """Free the scratch arena of ``stream`` (default: this context's stream).  Refused
        (DeviceError) while CUDA graphs captured on that stream may replay into it."""
        self.call("heb_ctx_release_scratch", self.stream if stream is None else stream)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().heb_ctx_destroy(h)
            except Exception:
                pass


def ctypes_void_p():
    import ctypes

    return ctypes.c_void_p()


def ctypes_byref(x):
    import ctypes

    return ctypes.byref(x)


# ---------------------------------------------------------------------------
# payloads (immutable views of device memory)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class DevCipher:
    buf: "torch.Tensor"  # (2, K, N) view; rows [0, k) active
    k: int

    def rows(self) -> "torch.Tensor":
        return self.buf[:, : self.k]

    # host copies in the reference CkksCipher layout ((k, N) uint64 per component), for
    # callers that inspect payload residues (reference tests, debugging)
    @property
    def c0(self) -> np.ndarray:
        return dev_to_u64(self.buf[0, : self.k])

    @property
    def c1(self) -> np.ndarray:
        return dev_to_u64(self.buf[1, : self.k])


@dataclass(frozen=True)
class DevRaw:
    buf: "torch.Tensor"  # (3, K, N)
    k: int


@dataclass(frozen=True)
class DevPlain:
    rows: "torch.Tensor"  # (K, N), K >= level + 1


@dataclass(frozen=True)
class DevSecret:
    s_eval: "torch.Tensor"  # (all rows, N)


@dataclass(frozen=True)
class DevPublic:
    b: "torch.Tensor"  # (fresh rows, N)
    a: "torch.Tensor"


@dataclass(frozen=True)
class DevSwitchKey:
    b: "torch.Tensor"     # (digits, all rows, N) reference layout (Montgomery residues)
    a: "torch.Tensor"
    prep: "torch.Tensor"  # (digits, all rows, 2, N, 2) Shoup pairs for the device key switch


@dataclass
class CipherBatch:
    """``B`` ciphertexts sharing level/scale in one (B, 2, K, N) device tensor.

    The batched analogue of a list of ``CipherVec``; cells of a packed image
    grid or of a feature map live here so a layer is one launch over all of
    them.  ``k`` active rows (= level + 1).
    """

    buf: "torch.Tensor"
    level: int
    scale: Fraction
    noise_bits: float = float("-inf")

    @property
    def k(self) -> int:
        return self.level + 1

    @property
    def count(self) -> int:
        return self.buf.shape[0]

    def desc(self) -> _lib.HebCt:
        return ct_desc(self.buf)


# ---------------------------------------------------------------------------
# the backend
# ---------------------------------------------------------------------------

class B200Backend(HEBackend):
    """CKKS on B200: reference-compatible payload math executed by libheb200."""

    name = "b200"
    wire_name = "ckks"  # payload format and math are the reference CKKS backend's (serialization.py)

    def __init__(self, params: HEParams, base_extra_bits: int | None = None, device: int = 0):
        super().__init__(params, base_extra_bits)
        self.n = params.ring_degree
        self.ctx = DeviceContext(self.chain, device)
        self.dev = self.ctx.device
        self._enc_counter = itertools.count()
        self._enc_lock = threading.Lock()

    # -- helpers ----------------------------------------------------------------
    def _rng(self, *tag: int) -> np.random.Generator:
        return hm.make_rng(self.params.rng_seed, *tag)

    def _fresh_noise_bits(self) -> float:
        return hm.fresh_noise_bits(self.n, self.params.precision_bits)

    def coeffs_to_rows(self, coeffs: np.ndarray, rows: int) -> "torch.Tensor":
        """(B, N) or (N,) centred int64 coefficients -> (B, rows, N) eval rows (ckks.py:120-126)."""
        c = np.ascontiguousarray(np.atleast_2d(coeffs), dtype=np.int64)
        src = torch.from_numpy(c).to(self.dev)
        out = self.ctx.empty(c.shape[0], rows, self.n)
        self.ctx.call("heb_spread_ntt", src.data_ptr(), c.shape[0], out.data_ptr(), rows, rows * self.n, self.ctx.stream)
        return out

    # -- keys ---------------------------------------------------------------------
    def _switch_key(self, s_eval, target, rng) -> DevSwitchKey:
        ch = self.chain
        digits = ch.num_rows - 1
        a = np.empty((digits, ch.num_rows, self.n), dtype=np.uint64)
        e = np.empty((digits, self.n), dtype=np.int64)
        for j in range(digits):  # same draw order as the reference keygen loop (ckks.py:159-161)
            a[j] = hm.sample_uniform_rows(rng, ch.p, self.n)
            e[j] = hm.sample_gaussian(rng, self.n)
        a_d = u64_to_dev(a, self.dev)
        e_d = torch.from_numpy(e).to(self.dev)
        kb = self.ctx.empty(digits, ch.num_rows, self.n)
        self.ctx.call("heb_make_switch_key", s_eval.data_ptr(), target.data_ptr(), a_d.data_ptr(), e_d.data_ptr(),
                      kb.data_ptr(), digits, self.ctx.stream)
        return self.prepare_switch_key(kb, a_d)

    def prepare_switch_key(self, kb: "torch.Tensor", ka: "torch.Tensor") -> DevSwitchKey:
        """Attach the Shoup-pair form used by the device key switch (heb_prepare_switch_key)."""
        digits = kb.shape[0]
        prep = self.ctx.empty(digits, self.chain.num_rows, 2, self.n, 2)
        self.ctx.call("heb_prepare_switch_key", kb.data_ptr(), ka.data_ptr(), digits, prep.data_ptr(), self.ctx.stream)
        return DevSwitchKey(b=kb, a=ka, prep=prep)

    def galois_key(self, s_eval, galois: int) -> DevSwitchKey:
        target = self.ctx.empty(self.chain.num_rows, self.n)
        self.ctx.call("heb_galois", s_eval.data_ptr(), target.data_ptr(), 1, self.chain.num_rows, 0, galois,
                      self.ctx.stream)
        return self._switch_key(s_eval, target, self._rng(5, galois))

    def keygen(self, galois_steps=()) -> KeyMaterial:
        """Reference keygen (ckks.py:135-184) with device NTTs; optional Galois keys."""
        ch, n = self.chain, self.n
        rows_all, rows_fresh = ch.num_rows, ch.num_levels + 1
        s = hm.sample_ternary(self._rng(1), n)
        s_eval = self.coeffs_to_rows(s, rows_all)[0]
        rng_pk = self._rng(2)
        pk_a = hm.sample_uniform_rows(rng_pk, ch.p[:rows_fresh], n)
        e = hm.sample_gaussian(rng_pk, n)
        pk_a_d = u64_to_dev(pk_a, self.dev)
        pk_b = self.ctx.empty(rows_fresh, n)
        self.ctx.call("heb_make_public_key", s_eval.data_ptr(), pk_a_d.data_ptr(),
                      torch.from_numpy(e).to(self.dev).data_ptr(), pk_b.data_ptr(), rows_fresh, self.ctx.stream)
        s2 = self.ctx.empty(rows_all, n)
        self.ctx.call("heb_mul_rows", s_eval.data_ptr(), s_eval.data_ptr(), s2.data_ptr(), rows_all, self.ctx.stream)
        evk = self._switch_key(s_eval, s2, self._rng(3))
        gal = {}
        for st in galois_steps:
            g = self.galois_element(st)
            gal[g] = self.galois_key(s_eval, g)
        torch.cuda.synchronize(self.dev)
        return KeyMaterial(
            fingerprint=self.params.fingerprint,
            backend_name=self.name,
            secret=DevSecret(s_eval),
            public=DevPublic(b=pk_b, a=pk_a_d),
            evaluation=evk,
            galois=gal or None,
        )

    # -- encode / encrypt / decrypt ---------------------------------------------------
    def _encode_impl(self, values, scale, level) -> DevPlain:
        coeffs = hm.encode_coeffs(values, scale, self.n, self.chain.modulus_at_level(level))
        return DevPlain(self.coeffs_to_rows(coeffs, level + 1)[0])

    def _sample_encryption(self, values: np.ndarray, scale: Fraction, entropy: int | None):
        m = hm.encode_coeffs(values, scale, self.n, self.chain.modulus_at_level(self.fresh_level))
        if entropy is None:
            with self._enc_lock:
                rng = self._rng(4, 0, next(self._enc_counter))
        else:
            rng = self._rng(4, 1, entropy)
        v = hm.sample_ternary(rng, self.n)
        e0 = hm.sample_gaussian(rng, self.n)
        e1 = hm.sample_gaussian(rng, self.n)
        return v, e0 + m, e1

    def _encrypt_rows(self, v, e0m, e1, key: KeyMaterial, out: "torch.Tensor") -> None:
        pk: DevPublic = key.public
        k = self.fresh_level + 1
        dv = torch.from_numpy(np.ascontiguousarray(v)).to(self.dev)
        d0 = torch.from_numpy(np.ascontiguousarray(e0m)).to(self.dev)
        d1 = torch.from_numpy(np.ascontiguousarray(e1)).to(self.dev)
        self.ctx.call("heb_encrypt", dv.data_ptr(), d0.data_ptr(), d1.data_ptr(), pk.b.data_ptr(), pk.a.data_ptr(),
                      ct_desc(out), v.shape[0], k, self.ctx.stream)

    def _encrypt_impl(self, values, scale, key, entropy) -> DevCipher:
        v, e0m, e1 = self._sample_encryption(values, scale, entropy)
        k = self.fresh_level + 1
        out = self.ctx.empty(1, 2, k, self.n)
        self._encrypt_rows(v[None], e0m[None], e1[None], key, out)
        return DevCipher(out[0], k)

    def encrypt_batch(self, values: np.ndarray, key: KeyMaterial, entropies, scale: Fraction | None = None) -> CipherBatch:
        """Encrypt B slot vectors in one launch; entropy tags as in ``encrypt``."""
        self._check_key(key)
        vals = np.atleast_2d(np.asarray(values, dtype=np.float64))
        scale = self.canonical_scale if scale is None else Fraction(scale)
        B = vals.shape[0]
        v = np.empty((B, self.n), dtype=np.int64)
        e0m = np.empty_like(v)
        e1 = np.empty_like(v)
        for i in range(B):
            v[i], e0m[i], e1[i] = self._sample_encryption(self._as_slot_array(vals[i]), scale, int(entropies[i]))
        k = self.fresh_level + 1
        out = self.ctx.empty(B, 2, k, self.n)
        self._encrypt_rows(v, e0m, e1, key, out)
        return CipherBatch(out, self.fresh_level, scale, self._fresh_noise_bits())

    def decrypt_coeffs_batch(self, buf: "torch.Tensor", k: int, key: KeyMaterial) -> np.ndarray:
        sk: DevSecret = key.secret
        B = buf.shape[0]
        coeffs = torch.empty((B, self.n), dtype=torch.int64, device=self.dev)
        bad = torch.zeros(B, dtype=torch.int64, device=self.dev)
        self.ctx.call("heb_decrypt", ct_desc(buf), sk.s_eval.data_ptr(), coeffs.data_ptr(), bad.data_ptr(), B, k,
                      self.ctx.stream)
        bad_h = bad.cpu().numpy()
        if bad_h.any():
            if k >= 2:
                raise DecryptionOutOfRange(f"{int(bad_h.max())} coefficients inconsistent across residues; "
                                           "ciphertext noise or magnitude exceeded the chain capacity")
            raise DecryptionOutOfRange("coefficients too close to the base modulus at level 0")
        return coeffs.cpu().numpy()

    def _decrypt_impl(self, ct: CipherVec, key: KeyMaterial) -> np.ndarray:
        p: DevCipher = ct.payload
        coeffs = self.decrypt_coeffs_batch(p.buf.unsqueeze(0), ct.level + 1, key)[0]
        return hm.slots_from_coeffs(coeffs.astype(np.float64), float(ct.scale), self.n)

    def decrypt_batch(self, batch: CipherBatch, key: KeyMaterial) -> np.ndarray:
        coeffs = self.decrypt_coeffs_batch(batch.buf, batch.k, key)
        return np.stack([hm.slots_from_coeffs(c.astype(np.float64), float(batch.scale), self.n) for c in coeffs])

    # -- payload math (ckks.py:279-387) ------------------------------------------------
    def _drop_impl(self, ct, level) -> DevCipher:
        return DevCipher(ct.payload.buf, level + 1)

    def _add_ct_ct_impl(self, a, b) -> DevCipher:
        k = a.level + 1
        out = self.ctx.empty(2, k, self.n)
        self.ctx.call("heb_add", ct_desc(a.payload.buf), ct_desc(b.payload.buf), ct_desc(out), 1, 2, k, self.ctx.stream)
        return DevCipher(out, k)

    def _add_ct_pt_impl(self, ct, plain) -> DevCipher:
        k = ct.level + 1
        out = self.ctx.empty(2, k, self.n)
        self.ctx.call("heb_add_plain", ct_desc(ct.payload.buf), plain.payload.rows.data_ptr(), 0, ct_desc(out), 1, k,
                      self.ctx.stream)
        return DevCipher(out, k)

    def _mul_ct_pt_impl(self, ct, plain) -> DevCipher:
        k = ct.level + 1
        out = self.ctx.empty(2, k - 1, self.n)
        self.ctx.call("heb_mul_plain_rescale", ct_desc(ct.payload.buf), plain.payload.rows.data_ptr(), 0,
                      ct_desc(out), 1, ct.level, self.ctx.stream)
        return DevCipher(out, k - 1)

    def _mul_raw_impl(self, a, b) -> DevRaw:
        k = a.level + 1
        out = self.ctx.empty(3, k, self.n)
        self.ctx.call("heb_tensor", ct_desc(a.payload.buf), ct_desc(b.payload.buf), ct_desc(out), 1, k, 0,
                      self.ctx.stream)
        return DevRaw(out, k)

    def _raw_add_impl(self, x, y) -> DevRaw:
        k = x.level + 1
        out = self.ctx.empty(3, k, self.n)
        self.ctx.call("heb_add", ct_desc(x.payload.buf), ct_desc(y.payload.buf), ct_desc(out), 1, 3, k, self.ctx.stream)
        return DevRaw(out, k)

    def _raw_finalize_impl(self, x) -> DevCipher:
        evk: DevSwitchKey = self._require_eval_key().evaluation
        k = x.level + 1
        out = self.ctx.empty(2, k - 1, self.n)
        self.ctx.call("heb_relin_rescale", ct_desc(x.payload.buf), evk.prep.data_ptr(), ct_desc(out), 1, x.level,
                      self.ctx.stream)
        return DevCipher(out, k - 1)

    def _rotate_impl(self, ct, galois) -> DevCipher:
        gk: DevSwitchKey = self._galois_keys[galois]
        k = ct.level + 1
        out = self.ctx.empty(2, k, self.n)
        self.ctx.call("heb_rotate", ct_desc(ct.payload.buf), gk.prep.data_ptr(), ct_desc(out), 1, ct.level, galois,
                      self.ctx.stream)
        return DevCipher(out, k)

    # -- host views (tests / serialization) -------------------------------------------------
    def cipher_rows_host(self, ct: CipherVec) -> tuple[np.ndarray, np.ndarray]:
        """(c0, c1) as (k, N) uint64 arrays in the reference's CkksCipher layout."""
        rows = dev_to_u64(ct.payload.rows())
        return rows[0], rows[1]

    def cipher_from_host(self, c0: np.ndarray, c1: np.ndarray, level: int, scale: Fraction,
                         noise_bits: float = float("-inf")) -> CipherVec:
        buf = u64_to_dev(np.stack([c0, c1]), self.dev)
        return self._cipher(DevCipher(buf, level + 1), level, Fraction(scale), noise_bits)

    # -- transport: bit-packed residue rows (csrc/packing.cu) -------------------------------
    def packed_words(self, k: int) -> int:
        """u64 words of one packed component (rows 0..k-1)."""
        w = _lib.lib().heb_packed_words(self.ctx.handle, k)
        if w < 0:
            _lib.check(int(w), "heb_packed_words")
        return int(w)

    def pack_batch(self, batch: CipherBatch) -> "torch.Tensor":
        """(B * 2 * packed_words(k),) int64 device tensor: the batch in wire format."""
        k, B = batch.k, batch.count
        out = torch.empty(B * 2 * self.packed_words(k), dtype=torch.int64, device=self.dev)
        buf = batch.buf
        if buf.stride(1) != buf.shape[2] * self.n or buf.stride(0) != 2 * buf.stride(1):
            buf = buf.contiguous()
        self.ctx.call("heb_pack_rows", buf.data_ptr(), B * 2, k, buf.stride(1), out.data_ptr(), self.ctx.stream)
        return out

    def unpack_into(self, packed: "torch.Tensor", out: "torch.Tensor", k: int) -> None:
        """Wire format -> rows 0..k-1 of a (B, 2, K, N) device tensor."""
        self.ctx.call("heb_unpack_rows", packed.data_ptr(), out.shape[0] * 2, k, out.data_ptr(), out.stride(1),
                      self.ctx.stream)

    # -- serialization hooks (ckks.py:389-483) ----------------------------------------------
    # The payload format is the reference's: "<II" (k, N) then c0 and c1 as k x N
    # little-endian u64 standard-form coefficients.  Conversion runs on the device
    # (heb_eval_to_coeff / heb_coeff_to_eval) over whole batches in one launch.
    def _rows_to_coeffs(self, rows: "torch.Tensor") -> np.ndarray:
        """(..., k, N) Montgomery eval rows -> host (..., k, N) coefficient words."""
        k = rows.shape[-2]
        buf = rows.contiguous().clone() if rows.is_contiguous() else rows.contiguous()
        count = buf.numel() // (k * self.n)
        self.ctx.call("heb_eval_to_coeff", buf.data_ptr(), count, k, k * self.n, self.ctx.stream)
        return dev_to_u64(buf)

    def _coeffs_to_rows_dev(self, coeffs: np.ndarray) -> "torch.Tensor":
        k = coeffs.shape[-2]
        buf = u64_to_dev(coeffs, self.dev)
        count = buf.numel() // (k * self.n)
        self.ctx.call("heb_coeff_to_eval", buf.data_ptr(), count, k, k * self.n, self.ctx.stream)
        return buf

    def _payload_head(self, data: bytes, level: int) -> int:
        k, n = struct.unpack_from("<II", data, 0)
        if n != self.n or k != level + 1:
            raise FingerprintMismatch("ciphertext payload does not match parameters")
        if len(data) < 8 + 2 * k * n * 8:
            raise HecnnError("truncated ciphertext payload")
        return k

    def cipher_payload_bytes(self, ct: CipherVec) -> bytes:
        k = ct.level + 1
        words = self._rows_to_coeffs(ct.payload.rows())
        return struct.pack("<II", k, self.n) + np.ascontiguousarray(words, dtype="<u8").tobytes()

    def cipher_from_payload(self, data: bytes, level: int, scale: Fraction, noise_bits: float) -> CipherVec:
        k = self._payload_head(data, level)
        words = np.frombuffer(data, dtype="<u8", count=2 * k * self.n, offset=8).reshape(2, k, self.n)
        return self._cipher(DevCipher(self._coeffs_to_rows_dev(words), k), level, Fraction(scale), noise_bits)

    def batch_payloads(self, batch: CipherBatch) -> list[bytes]:
        """cipher_payload_bytes of every item of a batch (one device conversion)."""
        k = batch.k
        words = self._rows_to_coeffs(batch.buf[:, :, :k])
        head = struct.pack("<II", k, self.n)
        return [head + np.ascontiguousarray(w, dtype="<u8").tobytes() for w in words]

    def batch_from_payloads(self, payloads, level: int, scale: Fraction,
                            noise_bits: float = float("-inf")) -> CipherBatch:
        """Inverse of ``batch_payloads``: B payloads at one level -> a (B, 2, k, N) batch."""
        payloads = list(payloads)
        k = level + 1
        words = np.empty((len(payloads), 2, k, self.n), dtype=np.uint64)
        for i, data in enumerate(payloads):
            self._payload_head(data, level)
            words[i] = np.frombuffer(data, dtype="<u8", count=2 * k * self.n, offset=8).reshape(2, k, self.n)
        return CipherBatch(self._coeffs_to_rows_dev(words), level, Fraction(scale), noise_bits)

    def key_payload_bytes(self, key: KeyMaterial) -> dict[str, bytes]:
        """Key roles in the reference's array format (ckks.py:456-466): eval-domain
        Montgomery residues exactly as keygen produced them."""
        parts: dict[str, bytes] = {}
        if key.secret is not None:
            parts["secret"] = ser.pack_array(dev_to_u64(key.secret.s_eval))
        if key.public is not None:
            parts["public"] = ser.pack_array(dev_to_u64(key.public.b)) + ser.pack_array(dev_to_u64(key.public.a))
        if key.evaluation is not None:
            ev = key.evaluation
            parts["evaluation"] = ser.pack_array(dev_to_u64(ev.b)) + ser.pack_array(dev_to_u64(ev.a))
        return parts

    def key_from_payload(self, parts: dict[str, bytes]) -> KeyMaterial:
        """ckks.py:468-487; the evaluation key is uploaded and Shoup-prepared on the device."""
        secret = public = evaluation = None
        if "secret" in parts:
            s, _ = ser.unpack_array(parts["secret"])
            secret = DevSecret(u64_to_dev(s, self.dev))
        if "public" in parts:
            b, off = ser.unpack_array(parts["public"])
            a, _ = ser.unpack_array(parts["public"], off)
            public = DevPublic(b=u64_to_dev(b, self.dev), a=u64_to_dev(a, self.dev))
        if "evaluation" in parts:
            b, off = ser.unpack_array(parts["evaluation"])
            a, _ = ser.unpack_array(parts["evaluation"], off)
            if b.shape != (self.chain.num_rows - 1, self.chain.num_rows, self.n) or a.shape != b.shape:
                raise FingerprintMismatch("evaluation key payload does not match parameters")
            evaluation = self.prepare_switch_key(u64_to_dev(b, self.dev), u64_to_dev(a, self.dev))
        torch.cuda.synchronize(self.dev)
        return KeyMaterial(fingerprint=self.fingerprint, backend_name=self.name, secret=secret, public=public,
                           evaluation=evaluation)

    def batch_to_cipher(self, batch: CipherBatch, i: int) -> CipherVec:
        return self._cipher(DevCipher(batch.buf[i], batch.k), batch.level, batch.scale, batch.noise_bits)
