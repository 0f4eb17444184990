"""Short estimator array vector (SEAV): the candidate sketch, device-backed.

Geometry and semantics are those of the reference `sspd/short_sketch.py`:
a host IP splits into RP (low r bits -> one of 2^r register arrays, "SEA")
and LP (the next addr_bits - r bits).  Row i of an array indexes g-bit
registers by the IBN-bit window of LP starting at ISB_i (wrapping), so
consecutive rows overlap in `a` LP bits.  A sampled opposite IP sets one
register bit in every row (short_sketch.py:289-318); at window end the LPs
of heavy hosts are reassembled from consistent hot columns
(short_sketch.py:347-408).

Here the registers live in one flat device buffer (the reference payload
layout: row 0 .. row SR-1, each (2^r, SC_i) registers C-order, registers
little-endian) and every bulk operation is a CUDA kernel from
libsspd_b200.so.  `.rows` is a host snapshot (numpy), as the reference
exposes numpy arrays.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from ._abi import build_params
from ._device import PreReadHook
from .errors import ConfigError, SeaOverflowError
from .hashing import SeedFamily, hash_full, hash_range, lsb

DEFAULT_RESTORE_CAP = 1 << 20

_REG_DTYPES = ((8, np.uint8), (16, np.uint16), (32, np.uint32), (64, np.uint64))


def tau_from_theta(theta: int, g: int) -> int:
    """Smallest t >= 0 with g * 2^t >= theta (short_sketch.py:38-50)."""
    if theta < 1:
        raise ConfigError(f"theta must be >= 1, got {theta}")
    if g < 1:
        raise ConfigError(f"register width g must be >= 1, got {g}")
    need = -(-theta // g)  # ceil(theta / g)
    return max(0, (need - 1).bit_length())


def register_dtype(g: int):
    for bits, dt in _REG_DTYPES:
        if g <= bits:
            return dt
    raise ConfigError(f"register width g must be <= 64, got {g}")


# ------------------------------------------------------------ one register
@dataclass(frozen=True)
class ShortEstimator:
    """A single g-bit register (host value object, short_sketch.py:61-93)."""

    bits: int = 0
    g: int = 8

    def __post_init__(self):
        if not 0 <= self.bits < (1 << self.g):
            raise ConfigError(f"register value {self.bits} out of range for g={self.g}")

    def update(self, oip: int, tau: int, seeds: SeedFamily) -> "ShortEstimator":
        if lsb(hash_full(oip, seeds.h1)) < tau:
            return self
        return ShortEstimator(self.bits | (1 << hash_range(oip, seeds.h2, self.g)), self.g)

    def weight(self) -> int:
        return bin(self.bits).count("1")

    def is_hot(self) -> bool:
        return self.weight() >= 3

    def _same_width(self, other: "ShortEstimator"):
        if other.g != self.g:
            raise ConfigError(f"register width mismatch: {self.g} vs {other.g}")

    def __and__(self, other: "ShortEstimator") -> "ShortEstimator":
        self._same_width(other)
        return ShortEstimator(self.bits & other.bits, self.g)

    def __or__(self, other: "ShortEstimator") -> "ShortEstimator":
        self._same_width(other)
        return ShortEstimator(self.bits | other.bits, self.g)


def se_update(se: ShortEstimator, oip: int, tau: int, seeds: SeedFamily) -> ShortEstimator:
    return se.update(oip, tau, seeds)


def se_weight(se: ShortEstimator) -> int:
    return se.weight()


def se_is_hot(se: ShortEstimator) -> bool:
    return se.is_hot()


def se_and(x: ShortEstimator, y: ShortEstimator) -> ShortEstimator:
    return x & y


def se_or(x: ShortEstimator, y: ShortEstimator) -> ShortEstimator:
    return x | y


# ---------------------------------------------------------------- geometry
def _positions(isb: int, ibn: int, w: int) -> set[int]:
    return {(isb + j) % w for j in range(ibn)}


@dataclass(frozen=True)
class SeavConfig:
    """Resolved SEAV geometry (validation of short_sketch.py:116-181)."""

    r: int = 4
    sr: int = 4
    a: int = 2
    theta: int = 1024
    g: int = 8
    addr_bits: int = 32
    isb: tuple[int, ...] = field(init=False)
    ibn: tuple[int, ...] = field(init=False)
    sc: tuple[int, ...] = field(init=False)
    tau: int = field(init=False)

    def __post_init__(self):
        if not 0 <= self.r <= 16:
            raise ConfigError(f"r must be in [0, 16], got {self.r}")
        if self.sr < 2:
            raise ConfigError(f"SR must be >= 2 (row overlap needs a partner), got {self.sr}")
        if self.a < 1:
            raise ConfigError(f"overlap a must be >= 1, got {self.a}")
        if not 2 <= self.addr_bits <= 32:
            raise ConfigError(f"addr_bits must be in [2, 32], got {self.addr_bits}")
        w = self.addr_bits - self.r
        if w < 1:
            raise ConfigError(f"r={self.r} leaves no left-part bits for addr_bits={self.addr_bits}")
        step = -(-w // self.sr)
        width = step + self.a
        if width > w:
            raise ConfigError(
                f"index width {width} exceeds left-part width {w} (SR too large or a too large)")
        set_ = object.__setattr__
        set_(self, "isb", tuple(step * i for i in range(self.sr)))
        set_(self, "ibn", (width,) * self.sr)
        set_(self, "sc", tuple(1 << n for n in self.ibn))
        set_(self, "tau", tau_from_theta(self.theta, self.g))
        register_dtype(self.g)
        rows = [_positions(self.isb[i], self.ibn[i], w) for i in range(self.sr)]
        covered = set().union(*rows)
        if covered != set(range(w)):
            missing = sorted(set(range(w)) - covered)
            raise ConfigError(f"constraint 1 violated: left-part bits {missing} not covered by any row")
        for i in range(self.sr):
            nxt = (i + 1) % self.sr
            shared = len(rows[i] & rows[nxt])
            if shared != self.a:
                raise ConfigError(
                    f"constraint 2 violated: rows {i} and {nxt} share {shared} bit positions, "
                    f"expected {self.a}")

    @property
    def lp_bits(self) -> int:
        return self.addr_bits - self.r

    @property
    def register_bytes(self) -> int:
        return np.dtype(register_dtype(self.g)).itemsize

    def index_of(self, row: int, lp: int) -> int:
        """Column of `lp` in `row`: bit j <- LP bit (ISB+j) mod w (short_sketch.py:183-193)."""
        if not 0 <= row < self.sr:
            raise ConfigError(f"row {row} out of range [0, {self.sr})")
        w = self.lp_bits
        lp &= (1 << w) - 1
        s = self.isb[row] % w
        rotated = ((lp >> s) | (lp << (w - s))) & ((1 << w) - 1) if s else lp
        return rotated & ((1 << self.ibn[row]) - 1)

    def index_of_array(self, row: int, lp: np.ndarray) -> np.ndarray:
        """index_of over an array (short_sketch.py:196-205), vectorised: the
        same rotate-right of the w-bit LP (w <= 32, so uint64 holds it)."""
        if not 0 <= row < self.sr:
            raise ConfigError(f"row {row} out of range [0, {self.sr})")
        w = self.lp_bits
        wmask = np.uint64((1 << w) - 1)
        x = np.asarray(lp).astype(np.uint64) & wmask
        s = self.isb[row] % w
        if s:
            x = ((x >> np.uint64(s)) | (x << np.uint64(w - s))) & wmask
        return x & np.uint64((1 << self.ibn[row]) - 1)

    def lp_from_indexes(self, indexes) -> int:
        """Inverse of index_of over all rows (short_sketch.py:196-205)."""
        if len(indexes) != self.sr:
            raise ConfigError(f"need {self.sr} indexes, got {len(indexes)}")
        w = self.lp_bits
        lp = 0
        for i, col in enumerate(indexes):
            s = self.isb[i] % w
            v = int(col) & ((1 << self.ibn[i]) - 1)
            lp |= ((v << s) | (v >> (w - s))) & ((1 << w) - 1) if s else v
        return lp

    def memory_bytes(self) -> int:
        return (1 << self.r) * sum(self.sc) * self.register_bytes


def make_config(r: int = 4, sr: int = 4, a: int = 2, theta: int = 1024, g: int = 8,
                addr_bits: int = 32) -> SeavConfig:
    return SeavConfig(r=r, sr=sr, a=a, theta=theta, g=g, addr_bits=addr_bits)


def index_of(config: SeavConfig, row: int, lp: int) -> int:
    return config.index_of(row, lp)


def lp_from_indexes(config: SeavConfig, indexes) -> int:
    return config.lp_from_indexes(indexes)


@dataclass(frozen=True)
class CandidateHost:
    """A reconstructed IP whose row-register AND has weight >= 3."""

    ip: int
    source_sea: int
    union_weight: int


# ------------------------------------------------------------------ sketch
class _RowList(list):
    """`SeavSketch.rows`: a list of host row snapshots whose item assignment
    writes through to the device."""

    def __init__(self, sketch):
        super().__init__()
        self._sketch = sketch

    def __setitem__(self, i, regs):
        if isinstance(i, slice):
            raise TypeError("assign SeavSketch rows one at a time, or the whole list")
        super().__setitem__(i, self._sketch._store_row(i, regs))

    def __reduce__(self):  # copies and pickles are plain lists of the arrays
        return (list, (list(self),))


class SeavSketch(PreReadHook):
    """Device-resident SEAV with the reference's API (short_sketch.py:259-408).

    Updates are monotone bit-sets (device `red.or`), so permutation,
    sharding + OR-merge and replays give bit-identical state.
    """

    def __init__(self, config: SeavConfig, seeds: SeedFamily,
                 restore_cap: int = DEFAULT_RESTORE_CAP, _ldca_config=None):
        from ._device import zeros_bytes
        from .long_sketch import LdcaConfig

        self.config = config
        self.seeds = seeds
        self.restore_cap = restore_cap
        # the parameter block carries both sketches' geometry; a SEAV alone
        # uses a 1x1 placeholder LDCA geometry that no kernel touches
        self._params = build_params(config, _ldca_config or LdcaConfig(lr=1, lc=1, k=8), seeds)
        self._buf = zeros_bytes(config.memory_bytes())
        self._cand_cap = 1 << 14
        self._radix_sort = False  # learned: candidates too skewed for the finalize's bucket sort
        self._scratch_buf = None

    def _scratch(self, nbytes: int):
        """Device work space of the fused finalize, kept across windows
        (stream-ordered reuse); grows on demand."""
        import torch

        if self._scratch_buf is None or self._scratch_buf.numel() < nbytes:
            self._scratch_buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self._buf.device)
        return self._scratch_buf

    # -- state access ------------------------------------------------------
    @property
    def nbytes(self) -> int:
        return self.config.memory_bytes()

    def memory_bytes(self) -> int:
        return self.config.memory_bytes()

    def device_buffer(self):
        """The flat payload on the device (torch uint8, 16-byte padded)."""
        return self._buf

    def _rebind(self, view):
        """Move the payload into `view` (a 16-byte aligned device uint8 view,
        e.g. a slice of a CUDA-IPC block shared with peer ranks)."""
        if view.numel() < self.nbytes:
            raise ValueError("view too small for the sketch payload")
        view[: self.nbytes].copy_(self._buf[: self.nbytes])
        self._buf = view

    @property
    def rows(self) -> list[np.ndarray]:
        """Host snapshot of the registers, one (2^r, SC_i) array per row.

        The arrays are read-only (an in-place write would not reach the
        device, so it fails loudly); assigning a row through the list
        (`sk.rows[i] = regs`, as the reference's sliding.py:202 does) or the
        whole list (`sk.rows = [...]`) uploads it."""
        flat = self._buf[: self.nbytes].cpu().numpy()
        dt = register_dtype(self.config.g)
        out, off = _RowList(self), 0
        for sc in self.config.sc:
            nb = (1 << self.config.r) * sc * self.config.register_bytes
            row = flat[off:off + nb].view(dt).reshape(1 << self.config.r, sc).copy()
            row.setflags(write=False)
            out.append(row)
            off += nb
        return out

    @rows.setter
    def rows(self, rows) -> None:
        self.load_rows(rows)

    def _store_row(self, i: int, regs) -> np.ndarray:
        """Upload one row's (2^r, SC_i) registers; returns the read-only copy."""
        import torch

        c = self.config
        if not -c.sr <= i < c.sr:
            raise IndexError(f"row {i} out of range")
        i %= c.sr
        a = np.ascontiguousarray(regs, dtype=register_dtype(c.g))
        if a.shape != (1 << c.r, c.sc[i]):
            raise ConfigError(f"row {i} shape {a.shape} != {(1 << c.r, c.sc[i])}")
        off = sum((1 << c.r) * sc for sc in c.sc[:i]) * c.register_bytes
        host = torch.from_numpy(a.view(np.uint8).reshape(-1).copy())
        self._buf[off:off + host.numel()].copy_(host)
        a = a.copy()
        a.setflags(write=False)
        return a

    def load_rows(self, rows) -> None:
        """Upload host register arrays (inverse of `.rows`)."""
        dt = register_dtype(self.config.g)
        payload = b"".join(np.ascontiguousarray(r, dtype=dt).tobytes() for r in rows)
        self.load_payload(payload)

    def clear(self):
        self._buf.zero_()

    def se_at(self, rp: int, row: int, col: int) -> ShortEstimator:
        return ShortEstimator(int(self.rows[row][rp, col]), self.config.g)

    def total_set_bits(self) -> int:
        host = self._buf[: self.nbytes].cpu().numpy()
        return int(np.bitwise_count(host).sum())

    def payload_bytes(self) -> bytes:
        return self._buf[: self.nbytes].cpu().numpy().tobytes()

    def load_payload(self, payload: bytes):
        import torch

        if len(payload) != self.nbytes:
            raise ConfigError(f"payload is {len(payload)} bytes, config requires {self.nbytes}")
        host = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
        self._buf[: self.nbytes].copy_(host)

    # -- updates -----------------------------------------------------------
    def update(self, hip: int, oip: int):
        self.update_batch(np.array([hip], dtype=np.uint64), np.array([oip], dtype=np.uint64))

    def update_batch(self, hips, oips):
        from ._device import call, ips_to_device, stream_ptr

        h = ips_to_device(hips, "hips")
        o = ips_to_device(oips, "oips")
        if h.numel() != o.numel():
            raise ConfigError("hips and oips differ in length")
        call("sspd_scan_discrete", h.data_ptr(), o.data_ptr(), h.numel(), self._params,
             self._buf.data_ptr(), None, stream_ptr())

    def merge(self, other: "SeavSketch"):
        if other.config != self.config or other.seeds != self.seeds:
            raise ConfigError("cannot merge register sketches with different config or seeds")
        from .distributed import device_or_into

        device_or_into(self._buf, [self._buf, other._buf], self.nbytes)

    # -- restore -----------------------------------------------------------
    def _restore_device(self, rp_begin: int, rp_count: int):
        """Run K5 + sort on the device; return (ips, aux, overflow) on host."""
        import torch

        from ._device import call, device, stream_ptr

        dev = device()
        overflow = torch.zeros(rp_count, dtype=torch.uint8, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        while True:
            ip = torch.empty(self._cand_cap, dtype=torch.int32, device=dev)
            aux = torch.empty(self._cand_cap, dtype=torch.int32, device=dev)
            call("sspd_restore", self._buf.data_ptr(), self._params, rp_begin, rp_count,
                 self.restore_cap, ip.data_ptr(), aux.data_ptr(), self._cand_cap,
                 count.data_ptr(), overflow.data_ptr(), stream_ptr())
            n = int(count.item())
            if n <= self._cand_cap:
                break
            self._cand_cap = 1 << (n - 1).bit_length()
            count.zero_()
            overflow.zero_()
        sort_candidates(ip, aux, n)
        return ip[:n], aux[:n], overflow

    def restore_sea(self, rp: int) -> list[CandidateHost]:
        if not 0 <= rp < (1 << self.config.r):
            raise ConfigError(f"rp {rp} out of range")
        ip, aux, overflow = self._restore_device(rp, 1)
        if int(overflow[0].item()):
            raise SeaOverflowError(rp, self.restore_cap)
        return _candidates(ip, aux)

    def restore(self, on_overflow: str = "raise") -> list[CandidateHost]:
        ip, aux, overflow = self._restore_device(0, 1 << self.config.r)
        flagged = np.nonzero(overflow.cpu().numpy())[0]
        for rp in flagged.tolist():
            err = SeaOverflowError(rp, self.restore_cap)
            if on_overflow != "warn":
                raise err
            warnings.warn(str(err), RuntimeWarning, stacklevel=2)
        return _candidates(ip, aux)


def sort_candidates(ip, aux, n: int):
    """Device radix sort of (ip, aux) by ip (restore's `sorted(found)`)."""
    import ctypes

    import torch

    from ._device import call, stream_ptr

    if n <= 1:
        return
    need = ctypes.c_size_t(0)
    call("sspd_sort_candidates", ip.data_ptr(), aux.data_ptr(), n, None, ctypes.byref(need), stream_ptr())
    scratch = torch.empty(need.value, dtype=torch.uint8, device=ip.device)
    call("sspd_sort_candidates", ip.data_ptr(), aux.data_ptr(), n, scratch.data_ptr(),
         ctypes.byref(need), stream_ptr())


def _candidates(ip, aux) -> list[CandidateHost]:
    ips = ip.cpu().numpy().view(np.uint32).tolist()
    auxs = aux.cpu().numpy().view(np.uint32).tolist()
    return [CandidateHost(ip=i, source_sea=a >> 8, union_weight=a & 0xFF) for i, a in zip(ips, auxs)]


def seav_update(sketch: SeavSketch, hip: int, oip: int) -> SeavSketch:
    sketch.update(hip, oip)
    return sketch


def seav_restore(sketch: SeavSketch, on_overflow: str = "raise") -> list[CandidateHost]:
    return sketch.restore(on_overflow=on_overflow)
