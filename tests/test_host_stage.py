"""Host staging of caller key arrays (csrc/host_stage.cu, abi.cu) -- the
native side of DetectorState.process_batch from host memory.  No GPU:
these are host functions of libsspd_b200.so."""

import os
import sys

import numpy as np
import pytest

from paper_1901_07306_b200._abi import lib

ERR_DATA, ERR_CONFIG = 3, 2


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32, np.uint64, np.int8, np.int16, np.int32,
                                   np.int64])
def test_check_and_pack_every_width(dtype):
    L = lib()
    rng = np.random.default_rng(3)
    hi = min(np.iinfo(dtype).max, 2**32 - 1)
    a = rng.integers(0, hi, size=100_003, dtype=np.uint64, endpoint=True).astype(dtype)
    signed = 1 if np.dtype(dtype).kind == "i" else 0
    assert L.sspd_host_check_u32(a.ctypes.data, len(a), a.itemsize, signed) == 0
    out = np.zeros(len(a), dtype=np.uint32)
    assert L.sspd_host_pack_u32(a.ctypes.data, len(a), a.itemsize, signed, out.ctypes.data) == 0
    assert (out == a.astype(np.uint64).astype(np.uint32)).all()
    if signed:
        bad = a.copy()
        bad[77] = -1
        assert L.sspd_host_check_u32(bad.ctypes.data, len(bad), bad.itemsize, 1) == ERR_DATA
    if np.dtype(dtype).itemsize == 8:
        bad = a.astype(np.uint64)
        bad[-1] = 1 << 32
        assert L.sspd_host_check_u32(bad.ctypes.data, len(bad), 8, 0) == ERR_DATA


@pytest.mark.parametrize("n", [1, 1000, (1 << 14) + 7, 1 << 20])
def test_pack_pairs_on_the_pool(n):
    """Both arrays of a batch, split over the worker pool above 2^14 pairs."""
    L = lib()
    rng = np.random.default_rng(n)
    h = rng.integers(0, 2**32, size=n, dtype=np.uint64)            # 8-byte keys (the reference's astype)
    o = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    dh = np.zeros(n, dtype=np.uint32)
    do = np.zeros(n, dtype=np.uint32)
    assert L.sspd_host_pack_pairs(h.ctypes.data, o.ctypes.data, n, 8, 4, dh.ctypes.data, do.ctypes.data) == 0
    assert (dh == h.astype(np.uint32)).all() and (do == o).all()
    assert L.sspd_host_pack_pairs(h.ctypes.data, o.ctypes.data, n, 3, 4, dh.ctypes.data, do.ctypes.data) == ERR_CONFIG
    assert L.sspd_host_copy_threads() >= 1


@pytest.mark.skipif(sys.platform != "linux", reason="fork")
def test_pack_pairs_after_fork():
    """A forked child gets a pool of its own (the parent's workers do not
    exist there) instead of waiting on them."""
    L = lib()
    a = np.arange(1 << 20, dtype=np.uint32)
    d1, d2 = np.empty_like(a), np.empty_like(a)
    assert L.sspd_host_pack_pairs(a.ctypes.data, a.ctypes.data, len(a), 4, 4, d1.ctypes.data, d2.ctypes.data) == 0
    pid = os.fork()
    if pid == 0:  # pragma: no cover - child
        d1[:] = 0
        rc = L.sspd_host_pack_pairs(a.ctypes.data, a.ctypes.data, len(a), 4, 4, d1.ctypes.data, d2.ctypes.data)
        os._exit(0 if rc == 0 and (d1 == a).all() else 3)
    _, status = os.waitpid(pid, 0)
    assert os.WEXITSTATUS(status) == 0


def test_hostfast_binding_stages_plain_u32_and_declines_the_rest():
    """csrc/hostfast.c (the CPython binding of the drop-in staging copy):
    plain 1-D uint32 pairs are copied by the library's pool; anything else
    (other widths, byte order, strides, unequal lengths, no room) returns -1
    so DetectorState.process_batch takes its general path."""
    from paper_1901_07306_b200.window_detector import _hostfast_pack

    pack = _hostfast_pack()
    if pack is None:
        pytest.skip("_hostfast not built")
    rng = np.random.default_rng(5)
    n = 70_001
    h = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    o = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    dh = np.zeros(n + 8, dtype=np.uint32)
    do = np.zeros(n + 8, dtype=np.uint32)
    assert pack(h, o, dh.ctypes.data + 4 * 8, do.ctypes.data + 4 * 8, n) == n
    assert (dh[8:] == h).all() and (do[8:] == o).all() and not dh[:8].any()
    room = n + 8
    assert pack(h.astype(np.int64), o, dh.ctypes.data, do.ctypes.data, room) == -1
    assert pack(h.astype(">u4"), o.astype(">u4"), dh.ctypes.data, do.ctypes.data, room) == -1
    assert pack(h[::2], o[::2], dh.ctypes.data, do.ctypes.data, room) == -1
    assert pack(h[:-1], o, dh.ctypes.data, do.ctypes.data, room) == -1
    assert pack(h, o, dh.ctypes.data, do.ctypes.data, n - 1) == -1
    assert pack(h[:0], o[:0], dh.ctypes.data, do.ctypes.data, room) == -1
    assert pack(h.reshape(1, -1), o.reshape(1, -1), dh.ctypes.data, do.ctypes.data, room) == -1
