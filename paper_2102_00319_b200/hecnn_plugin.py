"""The B200 backend plugged into the REFERENCE package itself (``hecnn``).

When ``hecnn`` is importable (``baseline/_ref``, or ``PYTHONPATH`` pointing at its
source), ``HecnnB200Backend`` is a real subclass of the reference's plugin contract
``hecnn.backends.base.HEBackend`` (`/root/reference/pkg/src/hecnn/backends/base.py:190-602`):
the reference keeps every piece of bookkeeping -- level alignment, exact ``Fraction``
scales, noise estimate, ``OpCounters``, ``DepthExhausted`` / ``ScaleMismatch`` /
``MissingEvalKey`` errors, its own ``CipherVec`` / ``RawProduct`` / ``KeyMaterial`` --
and only the payload hooks (`base.py:554-602`) run here, on the device, through
libheb200 (``B200Backend``'s hook implementations, which touch nothing but
``ct.payload`` / ``ct.level`` / ``plain.payload`` / ``key.*``).

It presents itself as ``name = "ckks"``: payload math and wire format are the reference
CKKS backend's (bit-identical ciphertexts, keys and HECN files), so files written by
either load on the other (`serialization.py:36,193-201` check the backend code).

Binding: ``install()`` adds ``get_backend("b200", params)`` to the
reference registry (`backends/__init__.py:8-19`); ``install(replace_ckks=True)`` makes
``get_backend("ckks", ...)`` return the device backend, which is how the reference's own
test suite is run against it (``pytest -p paper_2102_00319_b200.hecnn_plugin`` with
``HECNN_CKKS_IMPL=b200``).
"""

from __future__ import annotations

import os
from fractions import Fraction

_INSTALLED = False


def _hecnn():
    import hecnn.backends as hbk
    import hecnn.backends.base as hb
    import hecnn.backends.chain as hchain

    return hbk, hb, hchain


def make_backend_class():
    """Build ``HecnnB200Backend`` against the importable ``hecnn``."""
    _, hb, hchain = _hecnn()
    from .backend import B200Backend

    class HecnnB200Backend(hb.HEBackend):
        """hecnn's HEBackend with every payload hook executed on a B200."""

        name = "ckks"

        def __init__(self, params, device: int = 0) -> None:
            super().__init__(params)  # the reference's chain, counters, scale, fingerprint
            dev = B200Backend(params, hchain.BASE_EXTRA_BITS, device=device)
            if [int(x) for x in dev.chain.p] != [int(x) for x in self.chain.p]:
                raise RuntimeError("device chain differs from the reference chain")
            self._dev = dev
            self.ctx = dev.ctx

        # -- keys ------------------------------------------------------------------
        # The reference's key payloads are numpy arrays (CkksSecret.s_eval, CkksPublic.b/a);
        # the device keys stay on the device and are exposed through host views of the
        # same names, so callers that inspect key residues see the reference layout.
        def _wrap_key(self, k):
            return hb.KeyMaterial(fingerprint=self.fingerprint, backend_name=self.name,
                                  public=None if k.public is None else _HostPublic(k.public),
                                  secret=None if k.secret is None else _HostSecret(k.secret),
                                  evaluation=k.evaluation)

        @staticmethod
        def _device_key(key):
            return _DevKey(public=getattr(key.public, "dev", key.public), secret=getattr(key.secret, "dev", key.secret),
                           evaluation=key.evaluation)

        def keygen(self):
            return self._wrap_key(self._dev.keygen())

        def _fresh_noise_bits(self) -> float:  # CkksBackend._fresh_noise_bits (ckks.py:231-235)
            return self._dev._fresh_noise_bits()

        def set_eval_key(self, key) -> None:
            super().set_eval_key(key)
            self._dev._eval_key = key  # the device hooks read key.evaluation (prepared switch key)

        # -- payload hooks (reference base.py:554-584) --------------------------------
        def _encode_impl(self, values, scale, level):
            return self._dev._encode_impl(values, scale, level)

        def _encrypt_impl(self, values, scale, key, entropy):
            return self._dev._encrypt_impl(values, scale, self._device_key(key), entropy)

        def _decrypt_impl(self, ct, key):
            return self._dev._decrypt_impl(ct, self._device_key(key))

        def _drop_impl(self, ct, level):
            return self._dev._drop_impl(ct, level)

        def _add_ct_ct_impl(self, a, b):
            return self._dev._add_ct_ct_impl(a, b)

        def _add_ct_pt_impl(self, ct, plain):
            return self._dev._add_ct_pt_impl(ct, plain)

        def _mul_ct_pt_impl(self, ct, plain):
            return self._dev._mul_ct_pt_impl(ct, plain)

        def _mul_raw_impl(self, a, b):
            return self._dev._mul_raw_impl(a, b)

        def _raw_add_impl(self, x, y):
            return self._dev._raw_add_impl(x, y)

        def _raw_finalize_impl(self, x):
            self._dev._eval_key = self._require_eval_key()
            return self._dev._raw_finalize_impl(x)

        # -- serialization hooks (base.py:590-602; ckks.py:389-487 format) ----------------
        def cipher_payload_bytes(self, ct) -> bytes:
            return self._dev.cipher_payload_bytes(ct)

        def cipher_from_payload(self, data: bytes, level: int, scale: Fraction, noise_bits: float):
            ct = self._dev.cipher_from_payload(data, level, scale, noise_bits)
            return hb.CipherVec(payload=ct.payload, level=level, scale=Fraction(scale), slots=self.slots,
                                fingerprint=self.fingerprint, backend_name=self.name, noise_bits=noise_bits)

        def key_payload_bytes(self, key) -> dict[str, bytes]:
            return self._dev.key_payload_bytes(self._device_key(key))

        def key_from_payload(self, parts: dict[str, bytes]):
            return self._wrap_key(self._dev.key_from_payload(parts))

        # -- host views (tests) ---------------------------------------------------------
        def cipher_rows_host(self, ct):
            return self._dev.cipher_rows_host(ct)

    return HecnnB200Backend


class _HostSecret:
    """Device secret key with a host view ``s_eval`` (reference CkksSecret layout)."""

    def __init__(self, dev):
        self.dev = dev

    @property
    def s_eval(self):
        from .backend import dev_to_u64

        return dev_to_u64(self.dev.s_eval)


class _HostPublic:
    """Device public key with host views ``b`` / ``a`` (reference CkksPublic layout)."""

    def __init__(self, dev):
        self.dev = dev

    @property
    def b(self):
        from .backend import dev_to_u64

        return dev_to_u64(self.dev.b)

    @property
    def a(self):
        from .backend import dev_to_u64

        return dev_to_u64(self.dev.a)


class _DevKey:
    """The device parts of a key bundle, for the device hooks."""

    def __init__(self, public, secret, evaluation):
        self.public, self.secret, self.evaluation = public, secret, evaluation


_CLASS = None


def backend_class():
    global _CLASS
    if _CLASS is None:
        _CLASS = make_backend_class()
    return _CLASS


def install(replace_ckks: bool = False) -> None:
    """Register ``"b200"`` in the reference registry (and optionally stand in for ``"ckks"``)."""
    global _INSTALLED
    hbk, _, _ = _hecnn()
    cls = backend_class()
    if not _INSTALLED:
        original = hbk.get_backend

        def get_backend(name, params):
            if name.lower() == "b200":
                return cls(params)
            return original(name, params)

        get_backend.__doc__ = original.__doc__
        hbk.get_backend = get_backend
        _INSTALLED = True
    if replace_ckks:
        import hecnn.backends.ckks as hckks

        hckks.CkksBackend = cls  # get_backend("ckks", ...) imports the class at call time


# -- pytest plugin: run the reference's own tests against the device backend ------------------
def pytest_configure(config):  # pragma: no cover - exercised on the GPU box
    if os.environ.get("HECNN_CKKS_IMPL", "").lower() == "b200":
        install(replace_ckks=True)
