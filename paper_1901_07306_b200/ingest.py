"""Trace ingest and device-side frame checksums.

* `unpack_records` / `read_trace_device`: the reference's binary trace
  format -- little-endian 12-byte (slice, hip, oip) records
  (sspd/evaluation.py:21, read_trace :235-254) -- unpacked on the GPU into
  the SoA arrays the scan kernels stream.
* `device_crc32`: zlib.crc32 of a device buffer, computed by the GPU
  (csrc/ingest.cu), used by `serialize` so a frame's payload checksum never
  needs a host pass over the payload (distributed.py:81-101).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from .errors import DataError

RECORD_BYTES = 12
_POLY = 0xEDB88320


def _gf2_mulmod(a: int, b: int) -> int:
    """a * b mod P, reflected CRC-32 representation (bit 31 = x^0)."""
    m, prod = 1 << 31, 0
    for _ in range(32):
        if a & m:
            prod ^= b
        m >>= 1
        b = (b >> 1) ^ _POLY if b & 1 else b >> 1
    return prod


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    """CRC-32 of A||B from crc(A), crc(B) and |B| (GF(2) shift by 8|B| bits)."""
    acc, p, n, k = 1 << 31, 1 << 30, len2, 0
    pow2 = []
    for _ in range(64):
        pow2.append(p)
        p = _gf2_mulmod(p, p)
    k = 3
    while n:
        if n & 1:
            acc = _gf2_mulmod(pow2[k], acc)
        n >>= 1
        k += 1
    return _gf2_mulmod(acc, crc1) ^ crc2


def device_crc32(buf, nbytes: int | None = None) -> int:
    """zlib.crc32 of the first nbytes of a device uint8 tensor (GPU kernel)."""
    import torch

    from ._device import call, stream_ptr

    n = int(buf.numel() if nbytes is None else nbytes)
    need = ctypes.c_uint64(0)
    call("sspd_crc32", buf.data_ptr(), n, None, None, ctypes.byref(need), stream_ptr())
    scratch = torch.empty(max(4, need.value), dtype=torch.uint8, device=buf.device)
    out = torch.empty(1, dtype=torch.int32, device=buf.device)
    call("sspd_crc32", buf.data_ptr(), n, out.data_ptr(), scratch.data_ptr(), ctypes.byref(need), stream_ptr())
    return int(out.item()) & 0xFFFFFFFF


def unpack_records(records):
    """12-byte records (bytes, numpy structured/uint8 array, or a uint8 torch
    tensor on either device) -> device int32 tensors (slices, hips, oips)."""
    import torch

    from ._device import call, device, stream_ptr

    dev = device()
    if isinstance(records, torch.Tensor):
        raw = records.reshape(-1).view(torch.uint8)
    else:
        arr = np.frombuffer(records, dtype=np.uint8) if isinstance(records, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(records).view(np.uint8).reshape(-1)
        raw = torch.from_numpy(arr.copy() if not arr.flags.writeable else arr)
    if raw.numel() % RECORD_BYTES:
        raise DataError(f"trace is not a whole number of {RECORD_BYTES}-byte records")
    if raw.device.type != "cuda":
        raw = raw.pin_memory().to(dev, non_blocking=True)
    n = raw.numel() // RECORD_BYTES
    out = [torch.empty(max(1, n), dtype=torch.int32, device=dev) for _ in range(3)]
    call("sspd_unpack_records", raw.data_ptr(), n, out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
         stream_ptr())
    return tuple(t[:n] for t in out)


def read_trace_device(path) -> tuple:
    """Binary reference trace file -> device (slices, hips, oips)."""
    raw = Path(path).read_bytes()
    if len(raw) % RECORD_BYTES:
        raise DataError(f"{path} is not a whole number of {RECORD_BYTES}-byte records")
    return unpack_records(raw)
