"""CPU oracle for the CKKS payload math (TEST INFRASTRUCTURE, not product).

Python/ctypes driver over ``oracle/liboracle.so`` (the C restatement of the
reference numba kernels, see heoracle.c).  ``OracleCkks`` restates the payload
math of the reference ``CkksBackend``
(`/root/reference/pkg/src/hecnn/backends/ckks.py`):

* ``coeffs_to_rows``   -> ckks.py:120-126
* ``keygen``           -> ckks.py:135-184
* ``encode``/``encrypt``-> ckks.py:190-229
* ``decrypt_coeffs``   -> ckks.py:237-269
* ``add``/``add_plain``-> ckks.py:284-302
* ``rescale``          -> ckks.py:304-318
* ``mul_plain``        -> ckks.py:320-331
* ``mul_raw``          -> ckks.py:333-344
* ``raw_add``          -> ckks.py:346-357
* ``raw_finalize``     -> ckks.py:359-387
* ``rotate``           -> no reference counterpart (rotation is a non-goal
  there); defined here as the evaluation-domain Galois
  permutation followed by the reference's own key-switch pair
  (relin_accumulate + moddown_special) against a Galois key generated the
  way keygen builds the relinearisation key, with s^2 replaced by
  sigma_g(s).  Parity for rotation is therefore *unpinned* by the reference.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  It uses the product's host-only helpers (chain tables,
samplers, FFT encoding), which are themselves pinned against the reference's
golden vectors in ``tests/test_oracle_golden.py`` (fixtures from
``tests/golden/make_golden.py``) and ``tests/test_canonical.py`` (the reference's
own ``run_inference`` and BASELINE-size op digests, ``tests/golden/make_canonical.py``).
"""

from __future__ import annotations

import ctypes
import itertools
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from paper_2102_00319_b200 import hostmath as hm
from paper_2102_00319_b200.chain import ModulusChain
from paper_2102_00319_b200.errors import DecryptionOutOfRange, FingerprintMismatch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_I = ctypes.c_int

_SIGS = {
    "or_ntt_fwd_rows": [_u64p, _I, _I, _u64p, _I, _u64p, _u64p],
    "or_ntt_inv_rows": [_u64p, _I, _I, _u64p, _I, _u64p, _u64p, _u64p],
    "or_add_rows": [_u64p, _u64p, _I, _I, _u64p, _u64p],
    "or_neg_rows": [_u64p, _I, _I, _u64p, _u64p],
    "or_mul_rows": [_u64p, _u64p, _I, _I, _u64p, _u64p, _u64p],
    "or_scalar_mul_rows": [_u64p, _u64p, _I, _I, _u64p, _u64p, _u64p],
    "or_from_mont_rows": [_u64p, _I, _I, _u64p, _u64p],
    "or_centered_rows": [_u64p, _I, _I, _u64p, _i64p],
    "or_spread_centered": [_i64p, _I, _I, _u64p, _u64p, _u64p, _u64p],
    "or_ctct_products": [_u64p, _u64p, _u64p, _u64p, _I, _I, _u64p, _u64p, _u64p, _u64p, _u64p],
    "or_divide_drop_last": [_u64p, _I, _I, _u64p, _I, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p],
    "or_relin_accumulate": [_u64p, _i64p, _I, _I, _u64p, _u64p, _I, _I, _u64p, _I, _u64p, _u64p, _u64p, _u64p, _u64p],
    "or_moddown_special": [_u64p, _I, _I, _I, _u64p, _I, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p],
    "or_residue_check": [_i64p, _I, ctypes.c_uint64, _u64p],
    "or_galois_eval": [_u64p, _I, _I, ctypes.c_uint64, _u64p],
}


def load_library() -> ctypes.CDLL:
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"oracle library missing: {_LIB_PATH} (run `make -C oracle`)")
    lib = ctypes.CDLL(_LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_long if name == "or_residue_check" else None
    return lib


_LIB: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load_library()
    return _LIB


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a)


# ---------------------------------------------------------------------------
# kernel-level wrappers (names follow kernels.py)
# ---------------------------------------------------------------------------

def ntt_fwd_rows(f: np.ndarray, tw: np.ndarray, p: np.ndarray, p_inv: np.ndarray) -> None:
    rows, n = f.shape
    lib().or_ntt_fwd_rows(f, rows, n, _c(tw), tw.shape[1], _c(p), _c(p_inv))


def ntt_inv_rows(f, tw, n_inv, p, p_inv) -> None:
    rows, n = f.shape
    lib().or_ntt_inv_rows(f, rows, n, _c(tw), tw.shape[1], _c(n_inv), _c(p), _c(p_inv))


def add_rows(a, b, p, out) -> None:
    rows, n = a.shape
    lib().or_add_rows(_c(a), _c(b), rows, n, _c(p), out)


def neg_rows(a, p, out) -> None:
    rows, n = a.shape
    lib().or_neg_rows(_c(a), rows, n, _c(p), out)


def mul_rows(a, b, p, p_inv, out) -> None:
    rows, n = a.shape
    lib().or_mul_rows(_c(a), _c(b), rows, n, _c(p), _c(p_inv), out)


def scalar_mul_rows(a, c, p, p_inv, out) -> None:
    rows, n = a.shape
    lib().or_scalar_mul_rows(_c(a), _c(c), rows, n, _c(p), _c(p_inv), out)


def from_mont_rows(a, p, p_inv) -> None:
    rows, n = a.shape
    lib().or_from_mont_rows(a, rows, n, _c(p), _c(p_inv))


def centered_rows(a, p, out) -> None:
    rows, n = a.shape
    lib().or_centered_rows(_c(a), rows, n, _c(p), out)


def spread_centered(coeffs, p, r2, p_inv, out) -> None:
    lib().or_spread_centered(_c(coeffs), coeffs.shape[0], p.shape[0], _c(p), _c(r2), _c(p_inv), out)


def ctct_products(a0, a1, b0, b1, p, p_inv, d0, d1, d2) -> None:
    rows, n = a0.shape
    lib().or_ctct_products(_c(a0), _c(a1), _c(b0), _c(b1), rows, n, _c(p), _c(p_inv), d0, d1, d2)


def divide_drop_last(comp, tw, n_inv, p, p_inv, r2, drop_inv, out) -> None:
    k, n = comp.shape
    lib().or_divide_drop_last(_c(comp), k, n, _c(tw), tw.shape[1], _c(n_inv), _c(p), _c(p_inv), _c(r2), _c(drop_inv), out)


def relin_accumulate(d2_eval, d2_cent, evk_b, evk_a, sp_row, tw_all, p_all, p_inv_all, r2_all, acc0, acc1) -> None:
    k, n = d2_eval.shape
    lib().or_relin_accumulate(
        _c(d2_eval), _c(d2_cent), k, n, _c(evk_b), _c(evk_a), evk_b.shape[1], sp_row,
        _c(tw_all), tw_all.shape[1], _c(p_all), _c(p_inv_all), _c(r2_all), acc0, acc1,
    )


def moddown_special(acc, sp_row, tw_all, n_inv_all, p_all, p_inv_all, r2_all, sp_inv, out) -> None:
    k = acc.shape[0] - 1
    n = acc.shape[1]
    lib().or_moddown_special(_c(acc), k, n, sp_row, _c(tw_all), tw_all.shape[1], _c(n_inv_all), _c(p_all), _c(p_inv_all), _c(r2_all), _c(sp_inv), out)


def residue_check(coeffs, q, expect) -> int:
    return int(lib().or_residue_check(_c(coeffs), coeffs.shape[0], int(q), _c(expect)))


def galois_eval(rows: np.ndarray, galois: int) -> np.ndarray:
    r, n = rows.shape
    out = np.empty_like(rows)
    lib().or_galois_eval(_c(rows), r, n, int(galois), out)
    return out


# ---------------------------------------------------------------------------
# payload-level oracle (ckks.py restated)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class OKeys:
    s_eval: np.ndarray          # (all rows, n)
    pk_b: np.ndarray            # (fresh rows, n)
    pk_a: np.ndarray
    evk_b: np.ndarray           # (digits, all rows, n)
    evk_a: np.ndarray
    s_coeffs: np.ndarray        # int64 (n,)


class OracleCkks:
    """CPU restatement of CkksBackend's payload math on numpy arrays.

    Ciphertexts are ``(c0, c1)`` tuples of (k, n) uint64 arrays; raw products
    are ``(d0, d1, d2)``.  Levels are implied by the row count (k = level+1).
    """

    def __init__(self, chain: ModulusChain, seed: int):
        self.ch = chain
        self.n = chain.ring_degree
        self.seed = seed
        self.tw = chain.twiddles
        self._counter = itertools.count()

    # -- helpers ------------------------------------------------------------
    def coeffs_to_rows(self, coeffs: np.ndarray, rows: int) -> np.ndarray:
        ch = self.ch
        out = np.empty((rows, self.n), dtype=np.uint64)
        spread_centered(coeffs.astype(np.int64), ch.p[:rows], ch.r2[:rows], ch.p_inv[:rows], out)
        ntt_fwd_rows(out, self.tw[:rows], ch.p[:rows], ch.p_inv[:rows])
        return out

    def _rng(self, *tag):
        return hm.make_rng(self.seed, *tag)

    # -- keys ---------------------------------------------------------------
    def keygen(self) -> OKeys:
        ch, n = self.ch, self.n
        rows_all = ch.num_rows
        rows_fresh = ch.num_levels + 1
        s = hm.sample_ternary(self._rng(1), n)
        s_eval = self.coeffs_to_rows(s, rows_all)
        rng_pk = self._rng(2)
        pk_a = hm.sample_uniform_rows(rng_pk, ch.p[:rows_fresh], n)
        e = self.coeffs_to_rows(hm.sample_gaussian(rng_pk, n), rows_fresh)
        pk_b = np.empty_like(pk_a)
        mul_rows(pk_a, s_eval[:rows_fresh], ch.p[:rows_fresh], ch.p_inv[:rows_fresh], pk_b)
        neg_rows(pk_b, ch.p[:rows_fresh], pk_b)
        add_rows(pk_b, e, ch.p[:rows_fresh], pk_b)
        s2 = np.empty_like(s_eval)
        mul_rows(s_eval, s_eval, ch.p, ch.p_inv, s2)
        evk_b, evk_a = self._switch_key(s_eval, s2, self._rng(3))
        return OKeys(s_eval=s_eval, pk_b=pk_b, pk_a=pk_a, evk_b=evk_b, evk_a=evk_a, s_coeffs=s)

    def _switch_key(self, s_eval, target_eval, rng):
        """Digit j encrypts (P mod q_j) * target on row j only (ckks.py:151-176)."""
        ch, n = self.ch, self.n
        rows_all = ch.num_rows
        digits = rows_all - 1
        ka = np.empty((digits, rows_all, n), dtype=np.uint64)
        kb = np.empty_like(ka)
        for j in range(digits):
            ka[j] = hm.sample_uniform_rows(rng, ch.p, n)
            e_j = self.coeffs_to_rows(hm.sample_gaussian(rng, n), rows_all)
            mul_rows(ka[j], s_eval, ch.p, ch.p_inv, kb[j])
            neg_rows(kb[j], ch.p, kb[j])
            add_rows(kb[j], e_j, ch.p, kb[j])
            q_j = int(ch.p[j])
            factor = (ch.special_prime % q_j) * ((1 << 64) % q_j) % q_j
            term = np.empty((1, n), dtype=np.uint64)
            scalar_mul_rows(target_eval[j:j + 1], np.array([factor], dtype=np.uint64), ch.p[j:j + 1], ch.p_inv[j:j + 1], term)
            row = kb[j][j:j + 1].copy()
            add_rows(row, term, ch.p[j:j + 1], row)
            kb[j][j] = row[0]
        return kb, ka

    def galois_key(self, keys: OKeys, galois: int):
        """Key switching sigma_g(s) -> s; tag (seed, 5, g) (rotation: no reference)."""
        s_rot = galois_eval(keys.s_eval, galois)
        return self._switch_key(keys.s_eval, s_rot, self._rng(5, galois))

    # -- encode / encrypt / decrypt -----------------------------------------
    def encode(self, values: np.ndarray, scale: Fraction, level: int) -> np.ndarray:
        coeffs = hm.encode_coeffs(values, scale, self.n, self.ch.modulus_at_level(level))
        return self.coeffs_to_rows(coeffs, level + 1)

    def encrypt(self, values, scale: Fraction, keys: OKeys, entropy: int | None = None):
        ch = self.ch
        rows = ch.num_levels + 1
        coeffs = hm.encode_coeffs(values, scale, self.n, ch.modulus_at_level(ch.num_levels))
        m_rows = self.coeffs_to_rows(coeffs, rows)
        rng = self._rng(4, 0, next(self._counter)) if entropy is None else self._rng(4, 1, entropy)
        v = self.coeffs_to_rows(hm.sample_ternary(rng, self.n), rows)
        e0 = self.coeffs_to_rows(hm.sample_gaussian(rng, self.n), rows)
        e1 = self.coeffs_to_rows(hm.sample_gaussian(rng, self.n), rows)
        p, pi = ch.p[:rows], ch.p_inv[:rows]
        c0 = np.empty((rows, self.n), dtype=np.uint64)
        c1 = np.empty_like(c0)
        mul_rows(v, keys.pk_b, p, pi, c0)
        add_rows(c0, e0, p, c0)
        add_rows(c0, m_rows, p, c0)
        mul_rows(v, keys.pk_a, p, pi, c1)
        add_rows(c1, e1, p, c1)
        return c0, c1

    def decrypt_coeffs(self, ct, keys: OKeys) -> np.ndarray:
        ch = self.ch
        c0, c1 = ct
        k = c0.shape[0]
        rows = min(k, 2)
        p, pi = ch.p[:rows], ch.p_inv[:rows]
        m = np.empty((rows, self.n), dtype=np.uint64)
        mul_rows(c1[:rows], keys.s_eval[:rows], p, pi, m)
        add_rows(m, c0[:rows], p, m)
        ntt_inv_rows(m, self.tw[:rows], ch.n_inv[:rows], p, pi)
        from_mont_rows(m, p, pi)
        cent = np.empty((rows, self.n), dtype=np.int64)
        centered_rows(m, p, cent)
        if rows >= 2:
            bad = residue_check(cent[0], ch.p[1], m[1])
            if bad:
                raise DecryptionOutOfRange(f"{bad} coefficients inconsistent across residues")
        elif float(np.max(np.abs(cent[0]))) >= float(ch.base_prime) / 4.0:
            raise DecryptionOutOfRange("coefficients too close to the base modulus at level 0")
        return cent[0]

    def decrypt(self, ct, keys: OKeys, scale: Fraction) -> np.ndarray:
        return hm.slots_from_coeffs(self.decrypt_coeffs(ct, keys).astype(np.float64), float(scale), self.n)

    # -- arithmetic ---------------------------------------------------------
    def add(self, a, b):
        k = min(a[0].shape[0], b[0].shape[0])
        p = self.ch.p[:k]
        out = []
        for x, y in zip(a, b):
            o = np.empty((k, self.n), dtype=np.uint64)
            add_rows(x[:k], y[:k], p, o)
            out.append(o)
        return tuple(out)

    def add_plain(self, ct, pt_rows):
        k = ct[0].shape[0]
        c0 = np.empty((k, self.n), dtype=np.uint64)
        add_rows(ct[0], pt_rows[:k], self.ch.p[:k], c0)
        return c0, ct[1]

    def rescale(self, comp: np.ndarray) -> np.ndarray:
        ch = self.ch
        k = comp.shape[0]
        level = k - 1
        out = np.empty((k - 1, self.n), dtype=np.uint64)
        divide_drop_last(comp, self.tw[:k], ch.n_inv[:k], ch.p[:k], ch.p_inv[:k], ch.r2[:k], ch.drop_inv_mont(level), out)
        return out

    def mul_plain(self, ct, pt_rows):
        ch = self.ch
        k = ct[0].shape[0]
        p, pi = ch.p[:k], ch.p_inv[:k]
        outs = []
        for comp in ct:
            o = np.empty((k, self.n), dtype=np.uint64)
            mul_rows(comp, pt_rows[:k], p, pi, o)
            outs.append(self.rescale(o))
        return tuple(outs)

    def mul_raw(self, a, b):
        ch = self.ch
        k = min(a[0].shape[0], b[0].shape[0])
        d = [np.empty((k, self.n), dtype=np.uint64) for _ in range(3)]
        ctct_products(a[0][:k], a[1][:k], b[0][:k], b[1][:k], ch.p[:k], ch.p_inv[:k], *d)
        return tuple(d)

    def raw_add(self, x, y):
        k = x[0].shape[0]
        out = []
        for u, v in zip(x, y):
            o = np.empty((k, self.n), dtype=np.uint64)
            add_rows(u, v, self.ch.p[:k], o)
            out.append(o)
        return tuple(out)

    def key_switch(self, d2: np.ndarray, kb: np.ndarray, ka: np.ndarray):
        """relin_accumulate + moddown_special pair (ckks.py:366-381) for any switching key."""
        ch = self.ch
        k = d2.shape[0]
        sp = ch.special_row
        coef = d2.copy()
        ntt_inv_rows(coef, self.tw[:k], ch.n_inv[:k], ch.p[:k], ch.p_inv[:k])
        from_mont_rows(coef, ch.p[:k], ch.p_inv[:k])
        cent = np.empty((k, self.n), dtype=np.int64)
        centered_rows(coef, ch.p[:k], cent)
        acc0 = np.zeros((k + 1, self.n), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        relin_accumulate(np.ascontiguousarray(d2), cent, kb, ka, sp, self.tw, ch.p, ch.p_inv, ch.r2, acc0, acc1)
        sp_inv = ch.special_inv_mont(k - 1)
        r0 = np.empty((k, self.n), dtype=np.uint64)
        r1 = np.empty_like(r0)
        moddown_special(acc0, sp, self.tw, ch.n_inv, ch.p, ch.p_inv, ch.r2, sp_inv, r0)
        moddown_special(acc1, sp, self.tw, ch.n_inv, ch.p, ch.p_inv, ch.r2, sp_inv, r1)
        return r0, r1

    def raw_finalize(self, raw, keys: OKeys):
        d0, d1, d2 = raw
        k = d0.shape[0]
        r0, r1 = self.key_switch(d2, keys.evk_b, keys.evk_a)
        add_rows(r0, d0, self.ch.p[:k], r0)
        add_rows(r1, d1, self.ch.p[:k], r1)
        return self.rescale(r0), self.rescale(r1)

    def mul(self, a, b, keys: OKeys):
        return self.raw_finalize(self.mul_raw(a, b), keys)

    def rotate(self, ct, gkey, galois: int):
        """sigma_g on both components, then switch sigma_g(s) -> s; level kept."""
        c0, c1 = ct
        k = c0.shape[0]
        r0, r1 = self.key_switch(galois_eval(c1, galois), *gkey)
        out0 = galois_eval(c0, galois)
        add_rows(out0, r0, self.ch.p[:k], out0)
        return out0, r1


def threaded_map(fn, items, workers: int | None = None):
    """The reference's parallel pattern (executor.py:195-203): a thread pool whose
    native calls release the GIL (ctypes does, as numba nogil does)."""
    workers = workers or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(fn, items))


# ---------------------------------------------------------------------------
# the oracle behind the HEBackend contract (so percell / layer code runs on it)
# ---------------------------------------------------------------------------

from paper_2102_00319_b200.contract import HEBackend, KeyMaterial  # noqa: E402


@dataclass(frozen=True)
class _Cipher:
    c0: np.ndarray
    c1: np.ndarray


@dataclass(frozen=True)
class _Raw:
    d0: np.ndarray
    d1: np.ndarray
    d2: np.ndarray


@dataclass(frozen=True)
class _Plain:
    rows: np.ndarray


class OracleBackend(HEBackend):
    """CPU oracle exposed through the same contract as the device backend.

    Its ``name`` is "ckks" so that it cross-checks the reference's traces; key
    and ciphertext payloads are plain numpy (k, n) arrays exactly like the
    reference's ``CkksCipher``.
    """

    name = "ckks"

    def __init__(self, params, base_extra_bits=None):
        super().__init__(params, base_extra_bits)
        self.o = OracleCkks(self.chain, params.rng_seed)
        self.n = params.ring_degree

    def keygen(self, galois_steps=()) -> KeyMaterial:
        k = self.o.keygen()
        gal = {}
        for st in galois_steps:
            g = self.galois_element(st)
            gal[g] = self.o.galois_key(k, g)
        return KeyMaterial(self.params.fingerprint, self.name, public=k, secret=k, evaluation=k, galois=gal or None)

    def _fresh_noise_bits(self) -> float:
        return hm.fresh_noise_bits(self.n, self.params.precision_bits)

    def _encode_impl(self, values, scale, level):
        return _Plain(self.o.encode(values, scale, level))

    def _encrypt_impl(self, values, scale, key, entropy):
        c0, c1 = self.o.encrypt(values, scale, key.public, entropy)
        return _Cipher(c0, c1)

    def _decrypt_impl(self, ct, key):
        return self.o.decrypt((ct.payload.c0, ct.payload.c1), key.secret, ct.scale)

    def _drop_impl(self, ct, level):
        return _Cipher(ct.payload.c0[: level + 1], ct.payload.c1[: level + 1])

    def _add_ct_ct_impl(self, a, b):
        return _Cipher(*self.o.add((a.payload.c0, a.payload.c1), (b.payload.c0, b.payload.c1)))

    def _add_ct_pt_impl(self, ct, plain):
        return _Cipher(*self.o.add_plain((ct.payload.c0, ct.payload.c1), plain.payload.rows))

    def _mul_ct_pt_impl(self, ct, plain):
        return _Cipher(*self.o.mul_plain((ct.payload.c0, ct.payload.c1), plain.payload.rows))

    def _mul_raw_impl(self, a, b):
        return _Raw(*self.o.mul_raw((a.payload.c0, a.payload.c1), (b.payload.c0, b.payload.c1)))

    def _raw_add_impl(self, x, y):
        return _Raw(*self.o.raw_add((x.payload.d0, x.payload.d1, x.payload.d2), (y.payload.d0, y.payload.d1, y.payload.d2)))

    def _raw_finalize_impl(self, x):
        key = self._require_eval_key().evaluation
        return _Cipher(*self.o.raw_finalize((x.payload.d0, x.payload.d1, x.payload.d2), key))

    def _rotate_impl(self, ct, galois):
        return _Cipher(*self.o.rotate((ct.payload.c0, ct.payload.c1), self._galois_keys[galois], galois))

    # serialization hooks (ckks.py:393-436): INTT + from_mont out, to_mont + NTT in
    def cipher_payload_bytes(self, ct) -> bytes:
        ch, k = self.chain, ct.level + 1
        parts = [struct.pack("<II", k, self.n)]
        for comp in (ct.payload.c0, ct.payload.c1):
            buf = np.ascontiguousarray(comp[:k], dtype=np.uint64).copy()
            ntt_inv_rows(buf, ch.twiddles[:k], ch.n_inv[:k], ch.p[:k], ch.p_inv[:k])
            from_mont_rows(buf, ch.p[:k], ch.p_inv[:k])
            parts.append(buf.astype("<u8").tobytes())
        return b"".join(parts)

    def cipher_from_payload(self, data: bytes, level: int, scale, noise_bits: float):
        ch = self.chain
        k, n = struct.unpack_from("<II", data, 0)
        if n != self.n or k != level + 1:
            raise FingerprintMismatch("ciphertext payload does not match parameters")
        comps = []
        for c in range(2):
            buf = np.frombuffer(data, dtype="<u8", count=k * n, offset=8 + c * k * n * 8).reshape(k, n).astype(np.uint64)
            out = np.empty_like(buf)
            scalar_mul_rows(buf, ch.r2[:k], ch.p[:k], ch.p_inv[:k], out)
            ntt_fwd_rows(out, ch.twiddles[:k], ch.p[:k], ch.p_inv[:k])
            comps.append(out)
        return self._cipher(_Cipher(*comps), level, Fraction(scale), noise_bits)

    def key_payload_bytes(self, key) -> dict:
        """ckks.py:456-466 (the three roles share one OKeys bundle here)."""
        from paper_2102_00319_b200.serialization import pack_array

        parts = {}
        if key.secret is not None:
            parts["secret"] = pack_array(key.secret.s_eval)
        if key.public is not None:
            parts["public"] = pack_array(key.public.pk_b) + pack_array(key.public.pk_a)
        if key.evaluation is not None:
            parts["evaluation"] = pack_array(key.evaluation.evk_b) + pack_array(key.evaluation.evk_a)
        return parts
