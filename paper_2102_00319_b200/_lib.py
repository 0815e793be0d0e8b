"""ctypes binding of libheb200.so (the C ABI declared in include/heb200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, ``lib()`` raises ``DeviceError`` immediately.  Status codes map onto
the reference error taxonomy (`hecnn/errors.py`).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigurationError, DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEB_LIB_PATH") or os.path.join(HERE, "libheb200.so")


class HebCt(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("ct_stride", ctypes.c_int64), ("comp_stride", ctypes.c_int64)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_U = ctypes.c_uint64
_CT = HebCt

# name -> argtypes (all return int status unless listed in _RET)
SIGNATURES: dict[str, list] = {
    "heb_version": [],
    "heb_last_error": [],
    "heb_device_count": [ctypes.POINTER(ctypes.c_int)],
    "heb_ctx_create": [ctypes.POINTER(_P), _I, _I, _I, _P, _P],
    "heb_ctx_destroy": [_P],
    "heb_ctx_ring_degree": [_P],
    "heb_ctx_set_chunk": [_P, _I],
    "heb_ctx_release_scratch": [_P, _P],
    "heb_ctx_clear_captured": [_P, _P],
    "heb_alloc": [ctypes.c_size_t, ctypes.POINTER(_P), _P],
    "heb_free": [_P, _P],
    "heb_h2d": [_P, _P, ctypes.c_size_t, _P],
    "heb_d2h": [_P, _P, ctypes.c_size_t, _P],
    "heb_sync": [_P],
    "heb_ntt_fwd": [_P, _P, _L, _I, _I, _L, _P],
    "heb_ntt_inv": [_P, _P, _L, _I, _I, _L, _P],
    "heb_spread_ntt": [_P, _P, _L, _P, _I, _L, _P],
    "heb_eval_to_coeff": [_P, _P, _L, _I, _L, _P],
    "heb_coeff_to_eval": [_P, _P, _L, _I, _L, _P],
    "heb_add": [_P, _CT, _CT, _CT, _L, _I, _I, _P],
    "heb_add_plain": [_P, _CT, _P, _L, _CT, _L, _I, _P],
    "heb_tensor": [_P, _CT, _CT, _CT, _L, _I, _I, _P],
    "heb_rescale": [_P, _CT, _P, _L, _CT, _L, _I, _I, _P],
    "heb_mul_plain_rescale": [_P, _CT, _P, _L, _CT, _L, _I, _P],
    "heb_prepare_switch_key": [_P, _P, _P, _I, _P, _P],
    "heb_relin_rescale": [_P, _CT, _P, _CT, _L, _I, _P],
    "heb_rotate": [_P, _CT, _P, _CT, _L, _I, _U, _P],
    "heb_galois": [_P, _P, _P, _L, _I, _L, _U, _P],
    "heb_mul_rows": [_P, _P, _P, _P, _I, _P],
    "heb_encrypt": [_P, _P, _P, _P, _P, _P, _CT, _L, _I, _P],
    "heb_decrypt": [_P, _CT, _P, _P, _P, _L, _I, _P],
    "heb_make_public_key": [_P, _P, _P, _P, _P, _I, _P],
    "heb_make_switch_key": [_P, _P, _P, _P, _P, _P, _I, _P],
    "heb_dot_tensor": [_P, _CT, _CT, _P, _P, _I, _CT, _L, _I, _P],
    "heb_conv_tensor": [_P, _CT, _CT, _CT, _I, _I, _I, _I, _I, _I, _I, _I, _P],
    "heb_sum_gather": [_P, _CT, _P, _I, _CT, _L, _I, _I, _P],
    "heb_gather": [_P, _CT, _P, _CT, _L, _I, _I, _P],
    "heb_conv": [_P, _CT, _CT, _CT, _CT, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P],
    "heb_square": [_P, _CT, _CT, _L, _I, _P, _P],
    "heb_poly_act": [_P, _CT, _P, _P, _P, _CT, _L, _I, _P, _P],
    "heb_sumpool": [_P, _CT, _CT, _I, _I, _I, _I, _P],
    "heb_fc": [_P, _CT, _CT, _P, _P, _I, _CT, _CT, _L, _I, _P, _P],
    "heb_comm_unique_id": [_P],
    "heb_comm_init": [ctypes.POINTER(_P), _P, _I, _I, _I],
    "heb_comm_destroy": [_P],
    "heb_gather_logits": [_P, _P, _P, _L, _P],
    "heb_packed_words": [_P, _I],
    "heb_pack_rows": [_P, _P, _L, _I, _L, _P, _P],
    "heb_unpack_rows": [_P, _P, _L, _I, _P, _L, _P],
    "heb_prof_enable": [_I],
    "heb_prof_summary": [ctypes.c_char_p, ctypes.c_size_t],
    "heb_prof_next_bytes": [ctypes.c_double],
    "heb_bench_modmul": [_I, _I, _I, _U, ctypes.POINTER(ctypes.c_double), _P],
    "heb_bench_butterfly": [_I, _I, _I, _I, _U, ctypes.POINTER(ctypes.c_double), _P],
}
_RET = {"heb_last_error": ctypes.c_char_p, "heb_version": ctypes.c_int, "heb_ctx_ring_degree": ctypes.c_int,
        "heb_packed_words": ctypes.c_int64}

_lock = threading.Lock()
_LIB: ctypes.CDLL | None = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and declare every exported entry point."""
    if not os.path.exists(path):
        raise DeviceError(f"CUDA library not built: {path} (run paper_2102_00319_b200.build)")
    lib = ctypes.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RET.get(name, ctypes.c_int)
    return lib


def lib() -> ctypes.CDLL:
    global _LIB
    with _lock:
        if _LIB is None:
            _LIB = load()
        return _LIB


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = (lib().heb_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == -1:
        raise ValueError(text)
    if status == -4:
        raise ConfigurationError(text)
    raise DeviceError(text)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


PROF_ON = False


def prof_enable(on: bool) -> None:
    global PROF_ON
    lib().heb_prof_enable(1 if on else 0)
    PROF_ON = bool(on)


def prof_next_bytes(nbytes: float) -> None:
    """Declare the algorithmic bytes of the next launch (only while profiling)."""
    if PROF_ON:
        lib().heb_prof_next_bytes(float(nbytes))


def prof_summary() -> dict[str, tuple[int, float, float]]:
    """{kernel: (launches, total_ms, algorithmic_bytes)} since prof_enable(True)."""
    size = lib().heb_prof_summary(None, 0)
    if size < 0:
        check(size, "heb_prof_summary")
    buf = ctypes.create_string_buffer(size + 1)
    lib().heb_prof_summary(buf, size + 1)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms, nbytes = line.split()
        out[name] = (int(cnt), float(ms), float(nbytes))
    return out
