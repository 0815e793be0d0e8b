"""Ciphertext / key serialization (§8f next #1) against the reference's bytes.

tests/golden/s128.npz holds payloads, a ciphertext record and a whole HECN
envelope written by the reference (`ckks.py:389-487`, `serialization.py`),
see tests/golden/make_golden.py.  CPU tests pin the oracle restatement and the
byte framing in ``paper_2102_00319_b200.serialization``; the ``gpu`` tests run
the device conversion (heb_eval_to_coeff / heb_coeff_to_eval) through
``B200Backend`` and must reproduce the same bytes.
"""

from __future__ import annotations

import hashlib
from fractions import Fraction

import numpy as np
import pytest

from conftest import S128, s128_params
from paper_2102_00319_b200 import serialization as ser
from paper_2102_00319_b200.errors import FingerprintMismatch, HecnnError


def frac(s):
    a, b = s.split("/")
    return Fraction(int(a), int(b))


def _meta(golden, name):
    level, scale, noise = golden["s128"]["payload_meta"][name]
    return level, frac(scale), noise


def _golden_ct(be, s128, golden, name):
    from oracle.ckks_oracle import _Cipher

    level, scale, noise = _meta(golden, name)
    k = level + 1
    src = "a" if name == "a3" else name
    return be._cipher(_Cipher(s128[f"{src}_c0"][:k], s128[f"{src}_c1"][:k]), level, scale, noise)


class TestOraclePayloads:
    @pytest.mark.parametrize("name", ["a", "fin", "a3"])
    def test_payload_bytes_match_reference(self, s128, golden, oracle_s128, name):
        be, _ = oracle_s128
        ct = _golden_ct(be, s128, golden, name)
        assert be.cipher_payload_bytes(ct) == s128[f"payload_{name}"].tobytes()

    @pytest.mark.parametrize("name", ["a", "fin", "a3"])
    def test_payload_round_trip(self, s128, golden, oracle_s128, name):
        be, _ = oracle_s128
        level, scale, noise = _meta(golden, name)
        ct = be.cipher_from_payload(s128[f"payload_{name}"].tobytes(), level, scale, noise)
        ref = _golden_ct(be, s128, golden, name)
        assert np.array_equal(ct.payload.c0, ref.payload.c0)
        assert np.array_equal(ct.payload.c1, ref.payload.c1)

    def test_record_and_envelope_match_reference(self, s128, golden, oracle_s128):
        be, _ = oracle_s128
        fin = _golden_ct(be, s128, golden, "fin")
        assert ser.cipher_record(be, fin) == s128["record_fin"].tobytes()
        env = ser.wrap(ser.KIND_CIPHER, be, ser.cipher_record(be, fin))
        assert env == s128["envelope_fin"].tobytes()

    def test_load_reference_envelope(self, s128, golden, oracle_s128, tmp_path):
        be, _ = oracle_s128
        path = tmp_path / "fin.hecn"
        path.write_bytes(s128["envelope_fin"].tobytes())
        ct = ser.load_cipher(be, path)
        level, scale, noise = _meta(golden, "fin")
        assert (ct.level, ct.scale, ct.noise_bits) == (level, scale, noise)
        assert np.array_equal(ct.payload.c0, s128["fin_c0"])
        ser.save_cipher(be, ct, tmp_path / "again.hecn")
        assert (tmp_path / "again.hecn").read_bytes() == s128["envelope_fin"].tobytes()

    def test_key_payloads_match_reference(self, golden, oracle_s128):
        be, keys = oracle_s128
        parts = be.key_payload_bytes(keys)
        want = golden["s128"]["key_payload_sha256"]
        assert set(parts) == set(want)
        for role, data in parts.items():
            assert hashlib.sha256(data).hexdigest() == want[role], role


class TestFraming:
    def test_array_pack_round_trip(self):
        arr = np.arange(2 * 3 * 5, dtype=np.uint64).reshape(2, 3, 5) * np.uint64(0x9E3779B97F4A7C15)
        data = ser.pack_array(arr) + ser.pack_array(arr[0])
        a, off = ser.unpack_array(data)
        b, end = ser.unpack_array(data, off)
        assert np.array_equal(a, arr) and np.array_equal(b, arr[0]) and end == len(data)
        with pytest.raises(HecnnError):
            ser.unpack_array(data[:-1], off)

    def test_envelope_errors(self, s128, oracle_s128, tmp_path):
        be, _ = oracle_s128
        env = s128["envelope_fin"].tobytes()
        with pytest.raises(HecnnError):
            ser.unwrap(b"XXXX" + env[4:])
        with pytest.raises(HecnnError):
            ser.unwrap(env[:-3])
        with pytest.raises(HecnnError):
            ser.unwrap(env[:4] + b"\x02" + env[5:])
        path = tmp_path / "c.hecn"
        path.write_bytes(env)
        with pytest.raises(HecnnError):
            ser.read_envelope(path, expected_kind=ser.KIND_KEY_EVAL)
        bad_fp = env[:8] + bytes(16) + env[24:]
        path.write_bytes(bad_fp)
        with pytest.raises(FingerprintMismatch):
            ser.load_cipher(be, path)

    def test_payload_shape_mismatch(self, s128, golden, oracle_s128):
        be, _ = oracle_s128
        level, scale, noise = _meta(golden, "fin")
        with pytest.raises(FingerprintMismatch):
            be.cipher_from_payload(s128["payload_fin"].tobytes(), level + 1, scale, noise)


# ---------------------------------------------------------------------------------
# device path
# ---------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def dev_s128():
    from paper_2102_00319_b200.backend import B200Backend

    be = B200Backend(s128_params(), S128["extra"])
    keys = be.keygen()
    be.set_eval_key(keys)
    return be, keys


def _dev_ct(be, s128, golden, name):
    level, scale, noise = _meta(golden, name)
    k = level + 1
    src = "a" if name == "a3" else name
    return be.cipher_from_host(s128[f"{src}_c0"][:k], s128[f"{src}_c1"][:k], level, scale, noise)


@pytest.mark.gpu
class TestDevicePayloads:
    @pytest.mark.parametrize("name", ["a", "fin", "a3"])
    def test_payload_bytes_match_reference(self, s128, golden, dev_s128, name):
        be, _ = dev_s128
        assert be.cipher_payload_bytes(_dev_ct(be, s128, golden, name)) == s128[f"payload_{name}"].tobytes()

    @pytest.mark.parametrize("name", ["a", "fin", "a3"])
    def test_payload_load_matches_reference(self, s128, golden, dev_s128, name):
        be, _ = dev_s128
        level, scale, noise = _meta(golden, name)
        ct = be.cipher_from_payload(s128[f"payload_{name}"].tobytes(), level, scale, noise)
        c0, c1 = be.cipher_rows_host(ct)
        src = "a" if name == "a3" else name
        assert np.array_equal(c0, s128[f"{src}_c0"][: level + 1])
        assert np.array_equal(c1, s128[f"{src}_c1"][: level + 1])

    def test_reference_envelope_loads_and_decrypts(self, s128, golden, dev_s128, tmp_path):
        be, keys = dev_s128
        path = tmp_path / "fin.hecn"
        path.write_bytes(s128["envelope_fin"].tobytes())
        ct = ser.load_cipher(be, path)
        assert np.max(np.abs(be.decrypt(ct, keys).values - s128["fin_dec"])) == 0
        ser.save_cipher(be, ct, tmp_path / "out.hecn")
        assert (tmp_path / "out.hecn").read_bytes() == s128["envelope_fin"].tobytes()

    def test_batch_records(self, s128, golden, dev_s128):
        import torch

        from paper_2102_00319_b200.backend import CipherBatch

        be, _ = dev_s128
        a = _dev_ct(be, s128, golden, "a")
        buf = torch.stack([a.payload.buf, a.payload.buf.flip(-1)])
        batch = CipherBatch(buf, a.level, a.scale, a.noise_bits)
        data = ser.cipher_records(be, batch)
        single = ser.cipher_record(be, a)
        assert data[: len(single)] == single
        back, end = ser.batch_from_records(be, data, 2)
        assert end == len(data)
        assert torch.equal(back.buf, buf)

    def test_key_payload_round_trip(self, s128, golden, dev_s128):
        be, keys = dev_s128
        parts = be.key_payload_bytes(keys)
        for role, data in parts.items():
            assert hashlib.sha256(data).hexdigest() == golden["s128"]["key_payload_sha256"][role], role
        k2 = be.key_from_payload(parts)
        a = _dev_ct(be, s128, golden, "a")
        want = be.cipher_rows_host(be.mul_ct_ct(a, a))
        try:
            be.set_eval_key(k2)
            got = be.cipher_rows_host(be.mul_ct_ct(a, a))
        finally:
            be.set_eval_key(keys)
        assert all(np.array_equal(x, y) for x, y in zip(got, want))

    @pytest.mark.parametrize("log_n", [12, 13, 14, 15])
    def test_round_trip_large_rings(self, log_n):
        """eval -> coeff -> eval is the identity at every device NTT size (incl. the
        2-CTA cluster split at N=32768), and matches the oracle."""
        from oracle import ckks_oracle as oc
        from paper_2102_00319_b200.backend import B200Backend
        from paper_2102_00319_b200.params import derive_params

        be = B200Backend(derive_params(2 << log_n, 200, 40, seed=3), 20)
        ch, n = be.chain, be.n
        k = min(4, ch.num_rows)
        rng = np.random.default_rng(log_n)
        rows = np.stack([rng.integers(0, int(q), n, dtype=np.uint64) for q in ch.p[:k]])
        ct = be.cipher_from_host(rows, rows[::-1].copy() % ch.p[:k, None], k - 1, Fraction(1 << 40))
        data = be.cipher_payload_bytes(ct)
        ref = rows.copy()
        oc.ntt_inv_rows(ref, ch.twiddles[:k], ch.n_inv[:k], ch.p[:k], ch.p_inv[:k])
        oc.from_mont_rows(ref, ch.p[:k], ch.p_inv[:k])
        assert data[8: 8 + k * n * 8] == ref.astype("<u8").tobytes()
        back = be.cipher_from_payload(data, k - 1, Fraction(1 << 40), float("-inf"))
        c0, _ = be.cipher_rows_host(back)
        assert np.array_equal(c0, rows)
