"""Deterministic NTT-friendly modulus chain (host, cold path).

Restates the reference chain construction
(`/root/reference/pkg/src/hecnn/backends/chain.py:24-147`) and its prime/root
utilities (`backends/kernels.py:390-475`):

* one base prime of ``r + BASE_EXTRA_BITS`` bits, then
  ``(L - base_bits) // r`` level primes of ``r`` bits, then one special
  key-switching prime of ``base_bits`` bits (the *second* prime found by the
  base-size search);
* every prime is the result of a descending scan from ``2**bits - 1`` over
  ``p = 1 (mod m)`` with deterministic Miller-Rabin, so every party derives
  identical primes;
* psi = the first ``x >= 2`` whose ``x**((p-1)/2n)`` has order ``2n``;
* the stacked tables (``p``, ``p_inv``, ``r2``, ``n_inv``, ``twiddles``) use
  the reference's Montgomery conventions (R = 2**64) so host arrays compare
  bit-for-bit with the reference's ``ModulusChain``.

Row layout (Appendix A of SURVEY.md): row 0 = base, rows 1..L = level primes
in rescale order (top row dropped first), last row = special prime.

``BASE_EXTRA_BITS`` may be overridden per chain (the BASELINE configs use 10
and 20); it is part of the cache key.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .errors import ConfigurationError
from .params import HEParams

BASE_EXTRA_BITS = 25

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 2**64 (first 12 prime bases)."""
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d & 1 == 0:
        d >>= 1
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_primes_below(bits: int, m: int, count: int, exclude: set[int]) -> list[int]:
    """Descending scan for ``count`` primes ``p = 1 (mod m)``, ``p < 2**bits``.

    Same start point, stride and floor as reference `kernels.py:418-436`.
    """
    out: list[int] = []
    c = (1 << bits) - 1
    c -= (c - 1) % m
    floor = 1 << (bits - 1)
    while len(out) < count:
        if c <= floor:
            raise RuntimeError(f"could not find {count} NTT-friendly primes of {bits} bits for m={m}")
        if c not in exclude and is_prime(c):
            out.append(c)
        c -= m
    return out


def find_2n_root(n: int, p: int) -> int:
    """First generator-derived element of order exactly 2n (reference `kernels.py:439-446`)."""
    e = (p - 1) // (2 * n)
    for x in range(2, 1 << 20):
        y = pow(x, e, p)
        if pow(y, n, p) == p - 1:
            return y
    raise RuntimeError(f"no order-{2 * n} generator found mod {p}")


def mont_neg_inv(p: int) -> int:
    """-p^-1 mod 2**64."""
    return (-pow(p, -1, 1 << 64)) % (1 << 64)


def bitrev_perm(n: int) -> np.ndarray:
    logn = n.bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(logn):
        rev |= ((idx >> b) & 1) << (logn - 1 - b)
    return rev


def twiddle_table(n: int, p: int, psi: int | None = None) -> np.ndarray:
    """tw[i] = psi**bitrev(i) * 2**64 mod p (reference `kernels.py:464-475`)."""
    g = find_2n_root(n, p) if psi is None else psi
    powers = np.empty(n, dtype=object)
    acc = (1 << 64) % p
    for i in range(n):
        powers[i] = acc
        acc = acc * g % p
    return powers[bitrev_perm(n)].astype(np.uint64)


@dataclass(frozen=True)
class ModulusChain:
    """Prime ladder plus the stacked per-row host tables."""

    ring_degree: int
    base_prime: int
    level_primes: tuple[int, ...]
    special_prime: int
    p: np.ndarray
    p_inv: np.ndarray
    r2: np.ndarray
    n_inv: np.ndarray
    psi: tuple[int, ...]
    base_extra_bits: int = BASE_EXTRA_BITS
    _tw: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def num_levels(self) -> int:
        return len(self.level_primes)

    @property
    def num_rows(self) -> int:
        return len(self.level_primes) + 2

    @property
    def special_row(self) -> int:
        return self.num_rows - 1

    @property
    def primes(self) -> list[int]:
        return [self.base_prime, *self.level_primes, self.special_prime]

    @property
    def total_bits(self) -> int:
        return self.base_prime.bit_length() + sum(q.bit_length() for q in self.level_primes)

    @property
    def twiddles(self) -> np.ndarray:
        """(rows, n) Montgomery bit-reversed table, built lazily (host oracle use)."""
        if "tw" not in self._tw:
            self._tw["tw"] = np.stack(
                [twiddle_table(self.ring_degree, q, g) for q, g in zip(self.primes, self.psi)]
            )
        return self._tw["tw"]

    def primes_at_level(self, level: int) -> list[int]:
        return [self.base_prime] + list(self.level_primes[:level])

    def active_rows(self, level: int) -> int:
        return level + 1

    def modulus_at_level(self, level: int) -> int:
        q = self.base_prime
        for lp in self.level_primes[:level]:
            q *= lp
        return q

    def drop_inv_mont(self, level: int) -> np.ndarray:
        """q_drop^-1 mod q_i in Montgomery form (reference `chain.py:73-80`)."""
        drop = self.level_primes[level - 1]
        return np.array(
            [pow(drop, -1, q) * ((1 << 64) % q) % q for q in self.primes_at_level(level - 1)],
            dtype=np.uint64,
        )

    def special_inv_mont(self, level: int) -> np.ndarray:
        """P^-1 mod q_i in Montgomery form (reference `chain.py:82-88`)."""
        return np.array(
            [pow(self.special_prime, -1, q) * ((1 << 64) % q) % q for q in self.primes_at_level(level)],
            dtype=np.uint64,
        )


def chain_capacity(params: HEParams, base_extra_bits: int | None = None) -> int:
    extra = BASE_EXTRA_BITS if base_extra_bits is None else base_extra_bits
    return max(0, (params.modulus_bits - (params.precision_bits + extra)) // params.precision_bits)


@lru_cache(maxsize=32)
def _build_chain_cached(m: int, modulus_bits: int, precision_bits: int, extra: int) -> ModulusChain:
    n = m // 2
    r = precision_bits
    base_bits = r + extra
    n_level = (modulus_bits - base_bits) // r
    if n_level < 0:
        raise ConfigurationError(f"L={modulus_bits} cannot fit the {base_bits}-bit base prime for r={r}")
    try:
        base_pair = find_primes_below(base_bits, m, 2, set())
        base, special = base_pair[0], base_pair[1]
        levels = find_primes_below(r, m, n_level, {base, special}) if n_level else []
    except RuntimeError as exc:
        raise ConfigurationError(str(exc)) from exc
    primes = [base, *levels, special]
    chain = ModulusChain(
        ring_degree=n,
        base_prime=base,
        level_primes=tuple(levels),
        special_prime=special,
        p=np.array(primes, dtype=np.uint64),
        p_inv=np.array([mont_neg_inv(q) for q in primes], dtype=np.uint64),
        r2=np.array([pow(1 << 64, 2, q) for q in primes], dtype=np.uint64),
        n_inv=np.array([pow(n, -1, q) * ((1 << 64) % q) % q for q in primes], dtype=np.uint64),
        psi=tuple(find_2n_root(n, q) for q in primes),
        base_extra_bits=extra,
    )
    if chain.total_bits > modulus_bits:
        raise ConfigurationError("chain exceeds its bit budget")
    return chain


def build_chain(params: HEParams, base_extra_bits: int | None = None) -> ModulusChain:
    """Deterministic chain for (m, L, r[, base_extra_bits])."""
    extra = BASE_EXTRA_BITS if base_extra_bits is None else base_extra_bits
    return _build_chain_cached(params.m, params.modulus_bits, params.precision_bits, extra)
