"""HECN envelope and ciphertext records, byte-compatible with the reference.

Restates `/root/reference/pkg/src/hecnn/serialization.py` (envelope :57-97,
ciphertext record :116-131, keys :144-184) on top of the backend serialization
hooks.  The residue conversion inside ``cipher_payload_bytes`` /
``cipher_from_payload`` is the device path (heb_eval_to_coeff /
heb_coeff_to_eval) for ``B200Backend``; this module only frames bytes.

Backend codes: the B200 backend's payload format and math are the reference
CKKS backend's, so it writes and accepts code 0 ("ckks") -- files move between
the reference and this engine in both directions (``wire_name``).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path

import numpy as np

from .contract import CipherVec, HEBackend, KeyMaterial
from .errors import FingerprintMismatch, HecnnError

MAGIC = b"HECN"
VERSION = 1

KIND_CIPHER = 1
KIND_KEY_SECRET = 2
KIND_KEY_PUBLIC = 3
KIND_KEY_EVAL = 4
KIND_CIPHER_MATRIX = 5
KIND_CIPHER_LIST = 6

BACKEND_CODES = {"ckks": 0, "ref": 1}
BACKEND_NAMES = {v: k for k, v in BACKEND_CODES.items()}

_KEY_KINDS = {"secret": KIND_KEY_SECRET, "public": KIND_KEY_PUBLIC, "evaluation": KIND_KEY_EVAL}
_KIND_ROLES = {v: k for k, v in _KEY_KINDS.items()}

_HEADER = struct.Struct("<4sBBBB16sQQQQ")


def wire_name(backend: HEBackend) -> str:
    return getattr(backend, "wire_name", backend.name)


@dataclass(frozen=True)
class Envelope:
    kind: int
    backend_name: str
    fingerprint: bytes
    m: int
    modulus_bits: int
    precision_bits: int
    payload: bytes


def wrap(kind: int, backend: HEBackend, payload: bytes) -> bytes:
    code = BACKEND_CODES[wire_name(backend)]
    p = backend.params
    return _HEADER.pack(MAGIC, VERSION, kind, code, 0, backend.fingerprint, p.m, p.modulus_bits,
                        p.precision_bits, len(payload)) + payload


def unwrap(data: bytes) -> Envelope:
    if len(data) < _HEADER.size or data[:4] != MAGIC:
        raise HecnnError("not a HECN envelope")
    _, version, kind, code, _, fp, m, l_bits, r_bits, plen = _HEADER.unpack_from(data, 0)
    if version != VERSION:
        raise HecnnError(f"unsupported envelope version {version}")
    if code not in BACKEND_NAMES:
        raise HecnnError(f"unknown backend code {code}")
    payload = data[_HEADER.size:_HEADER.size + plen]
    if len(payload) != plen:
        raise HecnnError("truncated envelope payload")
    return Envelope(kind, BACKEND_NAMES[code], fp, m, l_bits, r_bits, payload)


def _pack_fraction(x: Fraction) -> bytes:
    num = x.numerator.to_bytes((x.numerator.bit_length() + 7) // 8 or 1, "little")
    den = x.denominator.to_bytes((x.denominator.bit_length() + 7) // 8 or 1, "little")
    return struct.pack("<II", len(num), len(den)) + num + den


def _unpack_fraction(data: bytes, offset: int) -> tuple[Fraction, int]:
    nlen, dlen = struct.unpack_from("<II", data, offset)
    offset += 8
    num = int.from_bytes(data[offset:offset + nlen], "little")
    den = int.from_bytes(data[offset + nlen:offset + nlen + dlen], "little")
    return Fraction(num, den), offset + nlen + dlen


def pack_array(arr) -> bytes:
    """ndim u32 | shape u32[ndim] | u64 words (ckks.py:438-441, key payloads)."""
    shape = np.asarray(arr.shape, dtype="<u4")
    return struct.pack("<I", arr.ndim) + shape.tobytes() + np.ascontiguousarray(arr, dtype="<u8").tobytes()


def unpack_array(data: bytes, offset: int = 0):
    """Inverse of ``pack_array``; returns (array, offset after it) (ckks.py:443-454)."""
    (ndim,) = struct.unpack_from("<I", data, offset)
    shape = tuple(int(x) for x in np.frombuffer(data, dtype="<u4", count=ndim, offset=offset + 4))
    count = 1
    for d in shape:
        count *= d
    start = offset + 4 + 4 * ndim
    if start + 8 * count > len(data):
        raise HecnnError("truncated key payload")
    arr = np.frombuffer(data, dtype="<u8", count=count, offset=start).reshape(shape).astype(np.uint64)
    return arr, start + 8 * count


def _record(ct: CipherVec, body: bytes) -> bytes:
    rec = struct.pack("<Id", ct.level, ct.noise_bits) + _pack_fraction(ct.scale) + body
    return struct.pack("<Q", len(rec)) + rec


def cipher_record(backend: HEBackend, ct: CipherVec) -> bytes:
    """u64 length | level u32 | noise f64 | scale fraction | payload (serialization.py:116-121)."""
    return _record(ct, backend.cipher_payload_bytes(ct))


def _parse_record(data: bytes, offset: int) -> tuple[int, float, Fraction, bytes, int]:
    (rlen,) = struct.unpack_from("<Q", data, offset)
    offset += 8
    end = offset + rlen
    if end > len(data):
        raise HecnnError("truncated ciphertext record")
    level, noise = struct.unpack_from("<Id", data, offset)
    scale, body_off = _unpack_fraction(data, offset + 12)
    return level, noise, scale, data[body_off:end], end


def cipher_from_record(backend: HEBackend, data: bytes, offset: int = 0) -> tuple[CipherVec, int]:
    level, noise, scale, body, end = _parse_record(data, offset)
    return backend.cipher_from_payload(body, level, scale, noise), end


def cipher_records(backend, batch) -> bytes:
    """Concatenated records of every ciphertext of a ``CipherBatch`` (one device
    conversion for the whole batch; byte-identical to per-item ``cipher_record``)."""
    out = []
    for body in backend.batch_payloads(batch):
        ct = CipherVec(None, batch.level, batch.scale, backend.slots, backend.fingerprint, backend.name,
                       batch.noise_bits)
        out.append(_record(ct, body))
    return b"".join(out)


def batch_from_records(backend, data: bytes, count: int, offset: int = 0):
    """``count`` consecutive records sharing level/scale -> one ``CipherBatch``."""
    bodies, meta = [], None
    for _ in range(count):
        level, noise, scale, body, offset = _parse_record(data, offset)
        if meta is None:
            meta = (level, scale, noise)
        elif (level, scale) != meta[:2]:
            raise HecnnError("records in one batch must share level and scale")
        bodies.append(body)
    level, scale, noise = meta
    return backend.batch_from_payloads(bodies, level, scale, noise), offset


def read_envelope(path: str | Path, expected_kind: int | None = None, backend: HEBackend | None = None) -> Envelope:
    env = unwrap(Path(path).read_bytes())
    if expected_kind is not None and env.kind != expected_kind:
        raise HecnnError(f"{path}: expected envelope kind {expected_kind}, got {env.kind}")
    if backend is not None:
        if env.backend_name != wire_name(backend):
            raise FingerprintMismatch(f"{path}: written by backend {env.backend_name!r}, not {wire_name(backend)!r}")
        if (env.m, env.modulus_bits, env.precision_bits) != backend.params.public_triple():
            raise FingerprintMismatch(f"{path}: parameter triple does not match context")
        if env.fingerprint != backend.fingerprint:
            raise FingerprintMismatch(f"{path}: key family fingerprint mismatch")
    return env


def save_cipher(backend: HEBackend, ct: CipherVec, path: str | Path) -> None:
    Path(path).write_bytes(wrap(KIND_CIPHER, backend, cipher_record(backend, ct)))


def load_cipher(backend: HEBackend, path: str | Path) -> CipherVec:
    env = read_envelope(path, expected_kind=KIND_CIPHER, backend=backend)
    return cipher_from_record(backend, env.payload)[0]


def save_key(backend: HEBackend, key: KeyMaterial, role: str, path: str | Path) -> None:
    parts = backend.key_payload_bytes(key)
    if role not in parts:
        raise HecnnError(f"key material has no {role!r} part")
    Path(path).write_bytes(wrap(_KEY_KINDS[role], backend, parts[role]))


def load_key(backend: HEBackend, path: str | Path) -> tuple[str, KeyMaterial]:
    env = read_envelope(path, backend=backend)
    role = _KIND_ROLES.get(env.kind)
    if role is None:
        raise HecnnError(f"file {path} is not a key envelope")
    key = backend.key_from_payload({role: env.payload})
    return role, KeyMaterial(fingerprint=env.fingerprint, backend_name=key.backend_name, public=key.public,
                             secret=key.secret, evaluation=key.evaluation)
