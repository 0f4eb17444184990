"""The scans' 32-bit-key hash (mix64_lo_fast, sspd_common.cuh) against the
64-bit SplitMix64 definition (reference hashing.py:48-53), exhaustively over
all 2^32 keys for the seeds the detector derives plus the carry edge cases of
the split evaluation.  Runs through the C ABI (sspd_check_hash32)."""

import ctypes as C

import pytest

from paper_1901_07306_b200.hashing import GOLDEN, M64, Tag, derive_seed

pytestmark = pytest.mark.gpu


def _seeds():
    out = [0, M64, 0x0123456789ABCDEF]
    # high word + golden high word wraps to 0xFFFFFFFF / 0: the carry of the
    # low add then wraps the high word (hg + 1 = 0)
    ghi = GOLDEN >> 32
    out.append(((0xFFFFFFFF - ghi) & 0xFFFFFFFF) << 32 | 0x55AA55AA)
    out.append(((0x100000000 - ghi) & 0xFFFFFFFF) << 32)
    # high words whose (h ^ h >> 30) changes shape at the carry: 0x3FFFFFFF -> 0x40000000
    out.append(((0x3FFFFFFF - ghi) & 0xFFFFFFFF) << 32 | 0xDEADBEEF)
    for master in (0, 2024):
        for tag in (Tag.H1, Tag.H2, Tag.H3, Tag.LH_BASE, Tag.LH_BASE + 7):
            out.append(derive_seed(master, int(tag)))
    return out


@pytest.mark.parametrize("seed", _seeds())
def test_hash32_exhaustive(cuda, seed):
    from paper_1901_07306_b200 import _abi

    lib = _abi.lib()
    bad, first = C.c_uint64(0), C.c_uint64(0)
    _abi.check(lib.sspd_check_hash32(seed, 0, 1 << 32, C.byref(bad), C.byref(first), None), "check_hash32")
    assert bad.value == 0, f"seed {seed:#x}: {bad.value} mismatches, first key {first.value:#x}"
    assert first.value == M64
