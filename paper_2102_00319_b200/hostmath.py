"""Host-side numerics that must stay bit-identical to the reference.

Two groups, both kept on the host on purpose:

* **slot encoding** — the canonical embedding of
  `/root/reference/pkg/src/hecnn/backends/encoding.py:23-37` (slot s at
  exp(i*pi*(2s+1)/n), float64 numpy FFT).  The float operation order is
  kept identical so that ``np.round`` of the scaled coefficients matches
  the reference bit for bit (SURVEY.md §7 hard part 5);
* **randomness** — the PCG64/SeedSequence streams of
  `/root/reference/pkg/src/hecnn/backends/ckks.py:99-118`: sparse ternary
  (Hamming weight 64), rounded Gaussian (sigma 3.2) and uniform residues,
  tagged (seed, 1) secret, (seed, 2) public, (seed, 3) evaluation,
  (seed, 4, 1, entropy) / (seed, 4, 0, counter) encryption.  Galois keys
  (new here; the reference has no rotation) use the tag (seed, 5, g).

Everything downstream of these integer coefficients (reduction into RNS
rows, NTTs, products) runs on the device.
"""

from __future__ import annotations

from fractions import Fraction
from functools import lru_cache

import numpy as np

from .errors import EncodeOverflow

SIGMA = 3.2
SPARSE_WEIGHT = 64
INT64_COEFF_LIMIT = float(2**62)


# ----------------------------------------------------------------------------
# canonical embedding
# ----------------------------------------------------------------------------

@lru_cache(maxsize=8)
def _odd_root_twist(n: int) -> np.ndarray:
    return np.exp(1j * np.pi * np.arange(n) / n)


def coeffs_from_slots(values: np.ndarray, scale: float, n: int) -> np.ndarray:
    """Real (unrounded) coefficients whose slot embedding is ``values * scale``."""
    half = n // 2
    mirrored = np.empty(n, dtype=np.complex128)
    mirrored[:half] = values
    mirrored[half:] = np.conj(values[::-1])
    spectrum = np.fft.fft(mirrored) / n
    return (spectrum * np.conj(_odd_root_twist(n))).real * scale


def slots_from_coeffs(coeffs: np.ndarray, scale: float, n: int) -> np.ndarray:
    """Slot values of a real coefficient vector divided by ``scale``."""
    twisted = coeffs.astype(np.float64) * _odd_root_twist(n)
    z = np.fft.ifft(twisted) * n
    return z[: n // 2].real / scale


def encode_coeffs(values: np.ndarray, scale: Fraction, n: int, modulus: int) -> np.ndarray:
    """Rounded int64 coefficients with the reference overflow guard (`ckks.py:190-199`)."""
    raw = coeffs_from_slots(values, float(scale), n)
    peak = float(np.max(np.abs(raw))) if raw.size else 0.0
    cap = float(modulus) / 2.0
    if peak >= min(cap, INT64_COEFF_LIMIT):
        raise EncodeOverflow(
            f"scaled coefficients reach {peak:.3g}, beyond the modulus capacity {cap:.3g}"
        )
    return np.round(raw).astype(np.int64)


def fresh_noise_bits(n: int, precision_bits: int) -> float:
    """log2 slot error of a fresh encryption (reference `ckks.py:231-235`)."""
    import math

    weight = min(SPARSE_WEIGHT, n // 2)
    coeff_err = SIGMA * math.sqrt(2.0 * weight + 1.0)
    return math.log2(4.0 * coeff_err * math.sqrt(n)) - precision_bits


def galois_slot_permutation(n: int, galois: int) -> np.ndarray:
    """Slot map of X -> X^g: slot s of the result holds slot ``perm[s]`` of the input.

    Slot s lives at exponent e_s = 2s+1 (mod 2n) and its conjugate at
    2n - e_s.  sigma_g(a)(zeta^e) = a(zeta^(e*g)); for real slot data the
    conjugate copy carries the same value, so the map folds back into
    [0, n/2).
    """
    two_n = 2 * n
    e = (2 * np.arange(n // 2, dtype=np.int64) + 1) * galois % two_n
    e = np.where(e > n, two_n - e, e)
    return (e - 1) // 2


# ----------------------------------------------------------------------------
# samplers (PCG64 streams identical to the reference)
# ----------------------------------------------------------------------------

def make_rng(seed: int, *tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed,) + tag)))


def sample_ternary(rng: np.random.Generator, n: int) -> np.ndarray:
    weight = min(SPARSE_WEIGHT, n // 2)
    out = np.zeros(n, dtype=np.int64)
    where = rng.choice(n, size=weight, replace=False)
    out[where] = rng.integers(0, 2, size=weight, dtype=np.int64) * 2 - 1
    return out


def sample_gaussian(rng: np.random.Generator, n: int) -> np.ndarray:
    return np.round(rng.normal(0.0, SIGMA, n)).astype(np.int64)


def sample_uniform_rows(rng: np.random.Generator, primes, n: int) -> np.ndarray:
    rows = np.empty((len(primes), n), dtype=np.uint64)
    for i, q in enumerate(primes):
        rows[i] = rng.integers(0, int(q), size=n, dtype=np.uint64)
    return rows
