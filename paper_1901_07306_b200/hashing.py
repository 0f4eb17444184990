"""Seeded hash family -- host side.

The per-packet hashing runs on the device (csrc/sspd_common.cuh).  The host
needs the same family for three things: deriving the seed block that is
passed to every kernel, scalar lookups that the drop-in API exposes
(`hash_full`, `hash_range`, `lsb`, `LdcaSketch.row_column`), and the
division magic for the kernels' exact 64-bit modulo.

Semantics follow the reference `sspd/hashing.py`:
  mix64        hashing.py:48-53   SplitMix64 finalizer, mod 2^64
  derive_seed  hashing.py:64-67   mix64(master ^ (tag & 0xFF) * GOLDEN)
  hash_full    hashing.py:111-117 low 32 bits of mix64(key ^ seed)
  hash_range   hashing.py:120-124 FULL 64-bit mix64(key ^ seed) % m
  lsb          hashing.py:133-141 lowest set bit, 32 for zero
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum
from functools import lru_cache

from .errors import ConfigError

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1
DEFAULT_MASTER_SEED = 0x5EED

GOLDEN = 0x9E3779B97F4A7C15
MUL_A = 0xBF58476D1CE4E5B9
MUL_B = 0x94D049BB133111EB


class Tag(IntEnum):
    """Domain tags of the hash roles (hashing.py:37-45)."""

    H1 = 1
    H2 = 2
    H3 = 3
    ROUTE = 4
    TRACE = 5
    LH_BASE = 16


def mix64(x: int) -> int:
    z = (x + GOLDEN) & M64
    z ^= z >> 30
    z = (z * MUL_A) & M64
    z ^= z >> 27
    z = (z * MUL_B) & M64
    return z ^ (z >> 31)


@lru_cache(maxsize=None)
def derive_seed(master_seed: int, domain_tag: int) -> int:
    # the tag product is not masked before the xor; mix64 masks after the
    # add, so only the low 64 bits matter (SURVEY.md §8 note)
    return mix64(((master_seed & M64) ^ ((domain_tag & 0xFF) * GOLDEN)) & M64)


@dataclass(frozen=True)
class HashSeed:
    seed: int
    domain_tag: int

    @property
    def value(self) -> int:
        return derive_seed(self.seed, self.domain_tag)


class SeedFamily:
    """All role seeds of one run, derived from one master seed."""

    def __init__(self, master_seed: int = DEFAULT_MASTER_SEED):
        self.master_seed = master_seed & M64
        self.h1 = HashSeed(self.master_seed, Tag.H1)
        self.h2 = HashSeed(self.master_seed, Tag.H2)
        self.h3 = HashSeed(self.master_seed, Tag.H3)
        self.route = HashSeed(self.master_seed, Tag.ROUTE)

    def lh(self, row: int) -> HashSeed:
        return HashSeed(self.master_seed, Tag.LH_BASE + row)

    def __eq__(self, other) -> bool:
        return isinstance(other, SeedFamily) and other.master_seed == self.master_seed

    def __hash__(self) -> int:
        return hash(self.master_seed)

    def __repr__(self) -> str:
        return f"SeedFamily(0x{self.master_seed:X})"


def hash64(key: int, seed: HashSeed) -> int:
    return mix64((key & M64) ^ seed.value)


def hash_full(key: int, seed: HashSeed) -> int:
    return hash64(key, seed) & M32


def hash_range(key: int, seed: HashSeed, m: int) -> int:
    if m < 1:
        raise ConfigError(f"hash_range modulus must be >= 1, got {m}")
    return hash64(key, seed) % m


def lsb(x: int) -> int:
    if x == 0:
        return 32
    return (x & -x).bit_length() - 1


# --------------------------------------------------------------- divisors
@dataclass(frozen=True)
class Divisor:
    """Exact 64-bit modulo by a runtime constant (round-up multiplier).

    For d not a power of two, with l = ceil(log2 d):
        magic = floor(2^64 * (2^l - d) / d) + 1      (low 64 bits of 2^64+magic)
        t = mulhi(magic, x);  q = (t + ((x - t) >> 1)) >> (l - 1)
    gives q = floor(x / d) for every x < 2^64 (Granlund & Montgomery 1994,
    fig. 4.1).  The device evaluates exactly this (sspd_common.cuh::mod).
    """

    d: int
    magic: int
    sh1: int
    sh2: int
    pow2: int

    @classmethod
    def of(cls, d: int) -> "Divisor":
        if not 1 <= d < (1 << 32):
            raise ConfigError(f"modulus {d} outside the supported range [1, 2^32)")
        if d & (d - 1) == 0:
            return cls(d=d, magic=0, sh1=0, sh2=0, pow2=1)
        ell = (d - 1).bit_length()
        magic = ((1 << 64) * ((1 << ell) - d)) // d + 1
        assert magic < (1 << 64)
        return cls(d=d, magic=magic, sh1=1, sh2=ell - 1, pow2=0)

    def mod(self, x: int) -> int:
        """Python model of the device arithmetic (used by the CPU tests)."""
        x &= M64
        if self.pow2:
            return x & (self.d - 1)
        t = (self.magic * x) >> 64
        q = (t + ((x - t) >> self.sh1)) >> self.sh2
        return x - q * self.d
