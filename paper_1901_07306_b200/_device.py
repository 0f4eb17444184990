"""Device plumbing: CUDA buffers and streams come from PyTorch, compute from
libsspd_b200.so.  Nothing here computes on the CPU on the data path.
"""

from __future__ import annotations

import numpy as np

from ._abi import check, lib
from .errors import DataError, DeviceError

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise DeviceError("PyTorch is required for device buffers") from exc


_ready = False


def device():
    global _ready
    if not _ready:
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the sspd B200 path has no CPU fallback")
        lib()
        _ready = True
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_cur_dev = getattr(torch._C, "_cuda_getDevice", None)


def stream_ptr() -> int:
    """Raw cudaStream_t of the current torch stream (a per-launch call: the
    direct C accessors instead of building a torch.cuda.Stream object)."""
    if _raw_stream is not None and _cur_dev is not None:
        return _raw_stream(_cur_dev())
    return torch.cuda.current_stream().cuda_stream


_get_cur = getattr(torch._C, "_cuda_getCurrentStream", None)
_set_cur = getattr(torch._C, "_cuda_setStream", None)


def current_stream():
    """torch.cuda.current_stream() without its lazy-init and device-index
    lookups (per-slide host path: ~1 us instead of ~8)."""
    if _get_cur is None or _cur_dev is None:
        return torch.cuda.current_stream()
    sid, di, dt = _get_cur(_cur_dev())
    return torch.cuda.Stream(stream_id=sid, device_index=di, device_type=dt)


class on_stream:
    """`with torch.cuda.stream(s)` for a stream of the current device,
    switching with the direct C accessors (the torch context manager
    re-resolves the device index on entry and exit, ~10 us per use)."""

    __slots__ = ("s", "prev")

    def __init__(self, s):
        self.s = s
        self.prev = None

    def __enter__(self):
        s = self.s
        if _get_cur is None or _set_cur is None:
            self.prev = torch.cuda.current_stream()
            torch.cuda.set_stream(s)
            return
        self.prev = _get_cur(s.device_index)
        _set_cur(stream_id=s.stream_id, device_index=s.device_index, device_type=s.device_type)

    def __exit__(self, *exc):
        prev = self.prev
        if isinstance(prev, tuple):
            _set_cur(stream_id=prev[0], device_index=prev[1], device_type=prev[2])
        else:
            torch.cuda.set_stream(prev)
        return False


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def zeros_bytes(nbytes: int):
    """Zeroed device byte buffer, padded to 16 B for vector access."""
    return torch.zeros(((nbytes + 15) // 16) * 16, dtype=torch.uint8, device=device())


def ips_to_device(a, name: str = "ips"):
    """Accept a numpy array / sequence / torch tensor of IPv4 addresses and
    return a contiguous 32-bit device tensor (bit pattern = uint32).

    The reference casts inputs with astype(uint64) and would hash wider
    keys in full (short_sketch.py:303-304); this build is IPv4-only and
    rejects keys outside [0, 2^32) instead of silently truncating them.
    """
    if isinstance(a, torch.Tensor):
        if a.dtype in (torch.int32, torch.uint32):
            t = a
        else:
            if a.numel() and (int(a.min()) < 0 or int(a.max()) > 0xFFFFFFFF):
                raise DataError(f"{name}: IPv4 keys must lie in [0, 2^32)")
            t64 = a.to(torch.int64)
            t = torch.where(t64 >= 2**31, t64 - 2**32, t64).to(torch.int32)
        if t.device.type != "cuda":
            t = t.to(device(), non_blocking=True)
        return t.contiguous()
    arr = np.asarray(a)
    if arr.dtype.kind not in "ui":
        raise DataError(f"{name}: integer array expected, got {arr.dtype}")
    if arr.dtype != np.uint32:
        if arr.size and (int(arr.min()) < 0 or int(arr.max()) > 0xFFFFFFFF):
            raise DataError(f"{name}: IPv4 keys must lie in [0, 2^32)")
        arr = arr.astype(np.uint32)
    arr = np.ascontiguousarray(arr.reshape(-1))
    return torch.from_numpy(arr.view(np.int32)).to(device(), non_blocking=False)


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


class PreReadHook:
    """Mixin for the device-resident sketches: reading `_buf` (every access
    path to the payload -- device_buffer(), rows/data, payload_bytes, merge,
    restore, finalize, ...) first runs `_pre_read`, a weak reference to the
    owning DetectorState's flush of host batches it has staged but not yet
    scanned, so no reader ever sees a sketch missing staged packets."""

    _pre_read = None

    @property
    def _buf(self):
        hook = self._pre_read
        if hook is not None:
            fn = hook()
            if fn is not None:
                fn()
        return self.__dict__["_buf_t"]

    @_buf.setter
    def _buf(self, value):
        self.__dict__["_buf_t"] = value
