"""Sliding-window detection over per-bit timestamps, device-backed.

Mirrors `sspd/sliding.py`: every SEAV/LDCA bit becomes a wrapped
last-active-slice stamp in one flat pool (SEAV slots first, then LDCA,
sliding.py:119-146); a slot is live iff ((now - ts) & mask) < w
(sliding.py:96-102); an amortised sweep every modulus - 2w slices clamps
idle slots so wrapped ages never alias (sliding.py:81-94).

The pool is one device buffer of the smallest unsigned stamp type; the
observe path (K2) is a plain-store kernel, and detect materialises the SEAV
view (K4), restores (K5) and filters straight from the pool (K6 sliding).
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .long_sketch import ldc_estimate
from .short_sketch import SeavSketch
from .window_detector import DetectionReport, DetectorParams, DeviceFinalize, PendingReports, ReportList
from .trace import traced

_UNSIGNED = ((1, np.uint8), (2, np.uint16), (4, np.uint32), (8, np.uint64))


def timestamp_dtype(window_slices: int):
    """Smallest unsigned dtype whose modulus is >= 2w + 2 (sliding.py:24-30)."""
    need = 2 * window_slices + 2
    for nbytes, dt in _UNSIGNED:
        if need <= (1 << (8 * nbytes)):
            return dt
    raise ConfigError(f"window of {window_slices} slices is too large to timestamp")


def _signed_torch(nbytes: int):
    import torch

    return {1: torch.int8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[nbytes]


def _as_signed(value: int, nbytes: int) -> int:
    bits = 8 * nbytes
    value &= (1 << bits) - 1
    return value - (1 << bits) if value >= (1 << (bits - 1)) else value


class TimestampPool:
    """Fixed pool of wrapped per-slot stamps with lazy expiry (sliding.py:33-106)."""

    def __init__(self, n_slots: int, window_slices: int, slice_seconds: float = 1.0):
        import torch

        from ._device import device

        if n_slots < 1:
            raise ConfigError(f"slot count must be >= 1, got {n_slots}")
        if window_slices < 1:
            raise ConfigError(f"window must span >= 1 slice, got {window_slices}")
        self.n_slots = n_slots
        self.window_slices = window_slices
        self.slice_seconds = slice_seconds
        self.now = 0
        self.dtype = timestamp_dtype(window_slices)
        self.ts_bytes = np.dtype(self.dtype).itemsize
        self._modulus = 1 << (8 * self.ts_bytes)
        self._mask = self._modulus - 1
        self._sweep_period = self._modulus - 2 * window_slices
        self._since_sweep = 0
        self.sweep_count = 0
        self._version = 0  # bumped by every stamp write that bypasses SlidingDetector
        self._deferred = None  # _DeferredLdca of the owning SlidingDetector (pending LDCA stamps)
        self._pristine = True  # constructor/reset state (no stamp written since)
        init = (-window_slices) & self._mask  # age == window: just expired
        self._buf = torch.full((n_slots,), _as_signed(init, self.ts_bytes),
                               dtype=_signed_torch(self.ts_bytes), device=device())

    # -- state --------------------------------------------------------------
    def device_buffer(self):
        """The stamp array on the device, with any deferred stamps applied."""
        self.flush()
        return self._buf

    def flush(self, ldca_view=None):
        """Apply the LDCA stamps a deferred scan recorded (sspd_ldca_fold /
        sspd_ldca_fold_ring); in single-bitmap mode with `ldca_view` (a device
        byte buffer) also write the packed active-bit LDCA in the same pass.
        Returns True when the view was written."""
        d = self._deferred
        if d is None:
            return False
        return d.flush(self, ldca_view)

    def _drop_deferred(self):
        """Pending deferred stamps are superseded (every stamp is replaced)."""
        d = self._deferred
        if d is not None:
            d.drop()

    def reset(self):
        """Back to the constructor state (slice 0, every slot just expired)."""
        self._drop_deferred()
        self.now = 0
        self._since_sweep = 0
        self.sweep_count = 0
        self._version += 1
        self._pristine = True
        self._buf.fill_(_as_signed((-self.window_slices) & self._mask, self.ts_bytes))
        if self._deferred is not None:
            self._deferred.restart(self, pristine=True)

    @property
    def ts(self) -> np.ndarray:
        """Host snapshot of the stamps (read-only: assign `pool.ts = arr`
        or use touch / touch_batch to write)."""
        out = self.device_buffer().cpu().numpy().view(self.dtype)
        out.setflags(write=False)
        return out

    @ts.setter
    def ts(self, values: np.ndarray):
        import torch

        arr = np.ascontiguousarray(np.asarray(values, dtype=self.dtype))
        if arr.shape != (self.n_slots,):
            raise ConfigError("timestamp array shape mismatch")
        signed = arr.view(_signed_torch_np(self.ts_bytes))
        self._drop_deferred()  # the new array replaces every stamp
        self._version += 1
        self._pristine = False
        self._buf.copy_(torch.from_numpy(signed))

    def memory_bytes(self) -> int:
        return self.n_slots * self.ts_bytes

    def _wrapped_now(self) -> int:
        return self.now & self._mask

    # -- updates ------------------------------------------------------------
    def touch(self, slot_index: int, now: int | None = None):
        """Stamp one slot; an older stamp never overwrites a newer one."""
        if not 0 <= slot_index < self.n_slots:
            raise ConfigError(f"slot {slot_index} out of range [0, {self.n_slots})")
        now = self.now if now is None else now
        candidate_age = self.now - now
        if candidate_age < 0:
            raise ConfigError(f"cannot stamp future slice {now} (pool is at {self.now})")
        current = int(self.device_buffer()[slot_index].item()) & self._mask
        existing_age = (self._wrapped_now() - current) & self._mask
        if candidate_age < existing_age:
            self._version += 1
            self._pristine = False
            self._buf[slot_index] = _as_signed(now & self._mask, self.ts_bytes)

    def touch_batch(self, slot_indexes):
        """ts[slot_indexes] = now (sliding.py:77-79) by `sspd_touch_slots`.
        numpy indexing semantics: a boolean mask selects, negative indexes
        count from the end, any index out of range raises IndexError before
        a slot is stamped."""
        import torch

        from ._device import call, stream_ptr

        a = np.asarray(slot_indexes)
        if a.dtype == np.bool_:
            if a.shape != (self.n_slots,):
                raise IndexError(f"boolean index of shape {a.shape} does not match {self.n_slots} slots")
            a = np.flatnonzero(a)
        elif a.dtype.kind not in "iu":
            raise IndexError("slot indexes must be integers or a boolean mask")
        a = a.reshape(-1)
        if a.size == 0:
            return
        lo, hi = int(a.min()), int(a.max())
        if lo < -self.n_slots or hi >= self.n_slots:
            bad = hi if hi >= self.n_slots else lo
            raise IndexError(f"index {bad} is out of bounds for axis 0 with size {self.n_slots}")
        idx = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(self._buf.device, non_blocking=False)
        self.flush()
        self._version += 1
        self._pristine = False
        call("sspd_touch_slots", self._buf.data_ptr(), self.n_slots, self.ts_bytes, idx.data_ptr(), idx.numel(),
             self._wrapped_now(), None, stream_ptr())

    def advance_slice(self):
        self.flush()  # deferred stamps belong to the slice that ends here
        self._advance()

    def _advance(self):
        self.now += 1
        self._since_sweep += 1
        if self._since_sweep >= self._sweep_period:
            self._sweep()

    def _sweep(self):
        from ._device import call, stream_ptr

        self.flush()
        clamp = (self.now - self.window_slices) & self._mask
        call("sspd_sweep", self._buf.data_ptr(), self.n_slots, self.ts_bytes, self._wrapped_now(),
             self.window_slices, clamp, stream_ptr())
        self._since_sweep = 0
        self.sweep_count += 1

    # -- queries ------------------------------------------------------------
    def ages(self) -> np.ndarray:
        import torch

        from ._device import call, stream_ptr

        out = torch.empty(self.n_slots, dtype=torch.int64, device=self._buf.device)
        call("sspd_pool_ages", self.device_buffer().data_ptr(), self.n_slots, self.ts_bytes, self._wrapped_now(),
             out.data_ptr(), stream_ptr())
        return out.cpu().numpy().view(np.uint64)

    def active(self) -> np.ndarray:
        return self.ages() < self.window_slices

    def is_active(self, slot_index: int) -> bool:
        current = int(self.device_buffer()[slot_index].item()) & self._mask
        return ((self._wrapped_now() - current) & self._mask) < self.window_slices


def _signed_torch_np(nbytes: int):
    return {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}[nbytes]


def touch(pool: TimestampPool, slot_index: int, now: int) -> TimestampPool:
    pool.touch(slot_index, now)
    return pool


def advance_slice(pool: TimestampPool) -> TimestampPool:
    pool.advance_slice()
    return pool


class _DeferredLdca:
    """LDCA stamps recorded as dirty bitmaps instead of stored
    (sspd_scan_sliding_deferred): within one slice every LDCA store of the
    reference's touch_batch (sliding.py:77-79) writes the same `now`, so the
    scan only marks the touched slots (one red.or into an L2-resident
    LDCA-shaped bitmap) and the stamps are written later, exactly.

    Single-bitmap mode: `dirty` holds the current slice; sspd_ldca_fold
    writes it once per slice (fused with the LDCA view at detect) and clears it.

    Ring mode (when w+1 bitmaps fit `SlidingDetector.ldca_ring_max_bytes`):
    the bitmap of every slice of the window is kept, slot = slice % (w+1).  A
    slot is active iff it was stamped in one of the last w slices, so the
    packed LDCA view is the OR of w bitmaps, maintained as a two-stack
    sliding-window OR: `acc` = OR of the current block's bitmaps (blocks of w
    slices starting at `blk0`); at a block end the block's bitmaps are turned
    in place into suffix ORs, so view(now) = suffix[now-w+1] | acc | dirty[now]
    (sspd_ldca_window_or: a few bitmap passes per detect instead of reading
    and rewriting every LDCA stamp).  Stamps are folded lazily
    (sspd_ldca_fold_ring: slices [fold_lo, cur], newest wins) whenever the
    pool is read, before a sweep, and at block ends before the suffix pass
    overwrites the raw bitmaps.  The view is exact from a pristine pool
    (nothing active before blk0) or once a full block has been recorded since
    the last stamp write that bypassed the detector (`prev_ok`); in between,
    detect folds and materializes the view from the stamps."""

    def __init__(self, params, nbytes: int, window_slices: int = 0, ring: bool = False):
        from ._device import zeros_bytes

        self.params = params
        self.nbytes = nbytes
        self.w = window_slices
        self.ring = None
        self.pending = False  # scanned since the last fold
        self.fresh = True  # the current slice's bitmap is all zeros (nothing scanned into it yet)
        if ring:
            import torch

            from ._device import device

            self.slots = window_slices + 1
            self.stride = -(-nbytes // 16) * 16
            self.ring = torch.zeros(self.slots * self.stride, dtype=torch.uint8, device=device())
            self.acc = zeros_bytes(nbytes)
            self.cur = self.blk0 = self.fold_lo = 0
            self.cur_merged = True
            self.next_zeroed = False
            self.prev_ok = False
            self.pristine = True
            self.version = None
        else:
            self.dirty = zeros_bytes(nbytes)

    # -- common ---------------------------------------------------------------
    def dirty_ptr(self) -> int:
        return self.slot_ptr(self.cur) if self.ring is not None else self.dirty.data_ptr()

    def mark_scanned(self):
        self.pending = True
        self.fresh = False
        if self.ring is not None:
            self.cur_merged = False

    def flush(self, pool, ldca_view=None) -> bool:
        if not self.pending:
            return False
        from ._device import call, stream_ptr

        if self.ring is not None:
            call("sspd_ldca_fold_ring", pool._buf.data_ptr(), pool.ts_bytes, self.params, self.ring.data_ptr(),
                 self.stride, self.slots, self.fold_lo, self.cur, stream_ptr())
            self.fold_lo = self.cur  # the current slice may gather more bits: folded again next time
            self.pending = False
            return False
        call("sspd_ldca_fold", pool._buf.data_ptr(), pool.ts_bytes, self.params, self.dirty.data_ptr(),
             pool._wrapped_now(), pool.window_slices, None if ldca_view is None else ldca_view.data_ptr(),
             stream_ptr())
        self.pending = False
        self.fresh = True  # the fold clears the bitmap
        return ldca_view is not None

    def drop(self):
        """Forget the pending stamps (the pool's stamps are all replaced)."""
        if self.ring is not None:
            self._zero_slot(self.cur)
            self.fold_lo = self.cur
        elif self.pending:
            self.dirty.zero_()
        self.pending = False
        self.fresh = True

    # -- ring mode ------------------------------------------------------------
    @property
    def current(self):
        """The current slice's bitmap (a device view)."""
        if self.ring is None:
            return self.dirty
        off = (self.cur % self.slots) * self.stride
        return self.ring[off: off + self.nbytes]

    def slot_ptr(self, e: int) -> int:
        return self.ring.data_ptr() + (e % self.slots) * self.stride

    def _zero_slot(self, e: int):
        off = (e % self.slots) * self.stride
        self.ring[off: off + self.stride].zero_()

    def restart(self, pool, pristine: bool):
        """Start a new block at the pool's slice.  The caller has folded every
        pending stamp (or dropped it); the view is exact from here only if
        `pristine` (no stamp active) -- else after one full block."""
        if self.ring is None:
            self.drop()
            return
        self.cur = self.blk0 = self.fold_lo = pool.now
        self._zero_slot(self.cur)
        self.acc.zero_()
        self.cur_merged = True
        self.next_zeroed = False
        self.prev_ok = False
        self.pristine = pristine
        self.pending = False
        self.fresh = True
        self.version = pool._version

    def sync(self, pool):
        """Stamps written around the detector (touch*, .ts, the pool's own
        advance_slice) restart the block structure (those paths flushed first)."""
        if pool._version != self.version or pool.now != self.cur:
            self.restart(pool, pristine=False)

    def valid(self) -> bool:
        return self.pristine or self.prev_ok

    def view_into(self, lview):
        """view = suffix[now-w+1] | (acc |= dirty[now])."""
        from ._device import call, stream_ptr

        first = self.cur - self.w + 1
        suffix = self.slot_ptr(first) if self.prev_ok and first <= self.blk0 - 1 else None
        # the next slice's slot (= slice cur - w, outside the window) is
        # cleared in the same pass
        call("sspd_ldca_window_or", self.slot_ptr(self.cur), self.acc.data_ptr(), suffix, lview.data_ptr(),
             self.slot_ptr(self.cur + 1), self.nbytes, stream_ptr())
        self.cur_merged = True
        self.next_zeroed = True

    def advance(self, pool):
        """End of slice `cur` (before the pool's slice advances)."""
        from ._device import call, stream_ptr

        if self.cur == self.blk0 + self.w - 1:  # block end: fold, then suffix ORs in place
            self.flush(pool)
            call("sspd_ldca_suffix_or", self.ring.data_ptr(), self.slots, self.stride, self.blk0, self.w, stream_ptr())
            self.prev_ok = True
            self.pristine = False
            self.blk0 = self.cur + 1
            self.acc.zero_()
            if not self.next_zeroed:
                self._zero_slot(self.cur + 1)
        elif not self.cur_merged:  # acc |= dirty[cur], and clear the next slice's slot
            call("sspd_ldca_window_or", self.slot_ptr(self.cur), self.acc.data_ptr(), None, None,
                 self.slot_ptr(self.cur + 1), self.nbytes, stream_ptr())
        elif not self.next_zeroed:
            self._zero_slot(self.cur + 1)
        self.next_zeroed = False
        if not self.pending:
            self.fold_lo = self.cur + 1
        self.cur += 1
        self.cur_merged = True
        self.fresh = True  # slot cur + 1 was cleared above (or by view_into)


@dataclass(frozen=True)
class _SlotLayout:
    seav_row_base: tuple[int, ...]
    ldca_base: int
    total: int


class SlidingDetector:
    """Sliding-window pipeline over one device timestamp pool (sliding.py:128-248)."""

    pipelined_scan_blocks_per_sm = 2  # K2 grid cap while detect_async runs (measured best on B200)
    pipeline_depth = 2  # view sets of detect_async (detects in flight)
    # detect_async replays the fused finalize of each view set as one CUDA
    # graph (captured per capacity) instead of ~12 launches from the host
    finalize_graphs = True
    # keep the SEAV active-bit view up to date (stamp-time set + expiry log)
    # instead of re-reading the whole SEAV stamp region at every detect
    incremental_seav = True
    seav_log_entries = 1 << 25  # ring of logged SEAV stamps (4 B each)
    # record LDCA stamps in a dirty bitmap and write them once per slice
    # (sspd_ldca_fold, fused with the LDCA view at detect)
    defer_ldca_stamps = True
    # ring mode of the deferred stamps: keep the bitmaps of the whole window
    # ((w+1) x LDCA bytes; 2.5 GB at config 4) and build the LDCA view as a
    # sliding-window OR instead of from the stamps
    ldca_ring_max_bytes = 8 << 30
    # slices at least this large record their LDCA half with the partitioned
    # scan K1b (0 = never); see _partitioned_dirty.  Config 4 (1.8 M packets
    # per slice): 66.2 vs 70.0 ms per trace (B200, bit-exact)
    partitioned_dirty_min_packets = 1 << 20

    def __init__(self, params: DetectorParams | None = None, window_slices: int = 300,
                 slice_seconds: float = 1.0):
        from ._abi import build_params
        from .hashing import SeedFamily

        self.params = params or DetectorParams()
        self.seeds = SeedFamily(self.params.master_seed)
        self.seav_config = self.params.seav_config()
        self.ldca_config = self.params.ldca_config()
        self._params = build_params(self.seav_config, self.ldca_config, self.seeds)
        p = self._params
        self.layout = _SlotLayout(tuple(int(p.slot_row_base[i]) for i in range(self.seav_config.sr)),
                                  int(p.slot_ldca_base), int(p.slot_total))
        self.pool = TimestampPool(self.layout.total, window_slices, slice_seconds)
        self.pair_count = 0

    @property
    def now(self) -> int:
        return self.pool.now

    def advance_slice(self):
        iv = self._iv()
        pool = self.pool
        if iv is not None:
            from ._device import call, stream_ptr

            self._iv_check(iv)
            # reads SEAV stamps only (never deferred): no LDCA fold needed
            call("sspd_seav_advance", pool._buf.data_ptr(), pool.ts_bytes, self._params,
                 iv["view"].device_buffer().data_ptr(), iv["log"].data_ptr(), iv["log"].numel(),
                 iv["meta"].data_ptr(), iv["nseg"], pool.now, pool.window_slices, stream_ptr())
            iv["now"] = pool.now + 1
        ring = self._ring()
        if ring is not None:  # bitmaps stay in the ring: no per-slice fold
            ring.advance(pool)
            pool._advance()
        else:
            pool.advance_slice()

    def reset(self):
        self.pool.reset()
        self.pair_count = 0
        iv = getattr(self, "_iv_state", None)
        if iv:
            iv["view"].clear()
            iv["meta"].zero_()
            iv["version"], iv["now"] = self.pool._version, self.pool.now

    # -- incremental SEAV view -------------------------------------------------
    def _iv(self):
        """State of the incrementally maintained SEAV view, or None when the
        stamp width / geometry has no tracked scan (u16 stamps, g = 8 one-byte
        registers, power-of-two k and lc)."""
        st = getattr(self, "_iv_state", False)
        if st is not False:
            return st
        st = None
        p, pool = self._params, self.pool
        ok = (self.incremental_seav and pool.ts_bytes == 2 and p.g == 8 and p.reg_bytes == 1
              and (p.k & (p.k - 1)) == 0 and (p.lc & (p.lc - 1)) == 0 and p.slot_total < (1 << 32)
              and all((int(p.slot_row_base[i]) & 7) == 0 and (int(p.seav_row_off[i]) & 3) == 0
                      and ((int(p.sc[i]) << p.r) & 3) == 0 for i in range(p.sr)))
        if ok:
            import torch

            from ._device import device

            nseg = 1 << (pool.window_slices + 2 - 1).bit_length()
            st = {"view": SeavSketch(self.seav_config, self.seeds, restore_cap=self.params.restore_cap,
                                     _ldca_config=self.ldca_config),
                  "log": torch.empty(self.seav_log_entries, dtype=torch.int32, device=device()),
                  "meta": torch.zeros(4 + nseg, dtype=torch.int64, device=device()),
                  "nseg": nseg, "version": pool._version, "now": pool.now}
            if not pool._pristine or pool.now or self.pair_count:
                st["meta"][1] = 1  # enabled late: the view starts invalid (full materialization)
        self._iv_state = st
        return st

    def _iv_check(self, iv):
        """Stamps written around the detector (TimestampPool.touch*, .ts,
        advance_slice on the pool itself) invalidate the incremental view:
        from then on every detect materializes it in full (exact)."""
        pool = self.pool
        if pool._version != iv["version"] or pool.now != iv["now"]:
            iv["meta"][1] = 1
            iv["version"], iv["now"] = pool._version, pool.now

    def _deferred(self):
        """The pool's deferred-LDCA state (created on first use), or None when
        the stamps are not u16 with an 8-slot aligned LDCA region."""
        pool, p = self.pool, self._params
        d = pool._deferred
        if d is None and self.defer_ldca_stamps and pool.ts_bytes == 2 and (p.slot_ldca_base & 7) == 0 \
                and p.ldca_bytes % 4 == 0 and p.slot_total < (1 << 32):
            ring = (pool.window_slices + 1) * (-(-p.ldca_bytes // 16) * 16) <= self.ldca_ring_max_bytes
            d = pool._deferred = _DeferredLdca(p, p.ldca_bytes, pool.window_slices, ring=ring)
            # nothing is active in a pool no stamp was ever written to
            d.restart(pool, pristine=pool._pristine and self.pair_count == 0)
        return d if self.defer_ldca_stamps else None

    def _ring(self):
        """The deferred-LDCA state when it runs in ring mode (synchronised
        with the pool), else None."""
        d = self._deferred()
        if d is None or d.ring is None:
            return None
        d.sync(self.pool)
        return d

    def _ldca_view_into(self, lview):
        """Packed active-bit LDCA into `lview`: the sliding-window OR of the
        ring bitmaps, or fused with the fold of the deferred stamps when
        some are pending, else K4 over the stamps."""
        pool = self.pool
        ring = self._ring()
        if ring is not None and ring.valid():
            ring.view_into(lview)
            return
        if pool.flush(ldca_view=lview):
            return
        from ._device import call, stream_ptr

        call("sspd_materialize_ldca", pool.device_buffer().data_ptr(), pool.ts_bytes, self._params,
             pool._wrapped_now(), pool.window_slices, lview.data_ptr(), stream_ptr())

    def _seav_view(self):
        """The SEAV active-bit view for the current slice as a SeavSketch
        (device): the incremental one (materialized in full only if it was
        invalidated), else a full K4 materialization."""
        iv = self._iv()
        if iv is None:
            seav = getattr(self, "_view", None)  # reused across slides: K4 overwrites every register
            if seav is None:
                seav = self._view = self.materialize_seav()
            else:
                self._materialize_into(seav)
            return seav
        from ._device import call, stream_ptr

        self._iv_check(iv)
        pool = self.pool
        meta = iv["meta"]  # int64: the kernel takes &meta[1]
        call("sspd_materialize_seav_if", pool._buf.data_ptr(), pool.ts_bytes, self._params,
             pool._wrapped_now(), pool.window_slices, iv["view"].device_buffer().data_ptr(),
             meta.data_ptr() + meta.element_size(), stream_ptr())
        return iv["view"]

    @traced("observe")
    def observe_batch(self, hips, oips):
        """K2: stamp every slot the discrete path would set (sliding.py:156-185)."""
        from ._device import call, ips_to_device, stream_ptr

        h = ips_to_device(hips, "hips")
        o = ips_to_device(oips, "oips")
        if h.numel() != o.numel():
            raise ConfigError("hips and oips differ in length")
        pool = self.pool
        # once detection is pipelined (detect_async), the scan leaves SM room
        # for the finalize kernels running on the side stream
        cap = self.pipelined_scan_blocks_per_sm if getattr(self, "_async", None) else 0
        iv = self._iv()
        dfr = self._deferred()
        if dfr is not None and dfr.ring is not None:
            dfr.sync(pool)
        if dfr is not None and self._partitioned_dirty(h.numel()):
            # large slices: the LDCA half into the slice's dirty bitmap with
            # the shared-memory partitioned scan (K1b), the SEAV half (stamps
            # + tracking) with K2 restricted to the sampled packets
            if iv is not None:
                self._iv_check(iv)
            if not self._scan_slice_fused(h, o, dfr, iv, pool):
                self._scan_dirty_partitioned(h, o, dfr.dirty_ptr(), fresh=dfr.fresh)
                call("sspd_scan_sliding_seav", h.data_ptr(), o.data_ptr(), h.numel(), self._params,
                     pool._buf.data_ptr(), pool.ts_bytes, pool._wrapped_now(), cap,
                     None if iv is None else iv["view"].device_buffer().data_ptr(),
                     None if iv is None else iv["log"].data_ptr(), 0 if iv is None else iv["log"].numel(),
                     None if iv is None else iv["meta"].data_ptr(), stream_ptr())
            dfr.mark_scanned()
        elif iv is not None or dfr is not None:
            if iv is not None:
                self._iv_check(iv)
            # pool._buf: the scan itself needs no flush (pending and new
            # deferred stamps are the same `now`)
            call("sspd_scan_sliding_deferred", h.data_ptr(), o.data_ptr(), h.numel(), self._params,
                 pool._buf.data_ptr(), pool.ts_bytes, pool._wrapped_now(), cap,
                 None if iv is None else iv["view"].device_buffer().data_ptr(),
                 None if iv is None else iv["log"].data_ptr(), 0 if iv is None else iv["log"].numel(),
                 None if iv is None else iv["meta"].data_ptr(),
                 None if dfr is None else dfr.dirty_ptr(), stream_ptr())
            if dfr is not None:
                dfr.mark_scanned()
        else:
            call("sspd_scan_sliding_capped", h.data_ptr(), o.data_ptr(), h.numel(), self._params,
                 pool.device_buffer().data_ptr(), pool.ts_bytes, pool._wrapped_now(), cap, stream_ptr())
        self.pair_count += int(h.numel())

    def _partitioned_dirty(self, n: int) -> bool:
        """Record this slice's LDCA half with K1b? (env SSPD_SLIDE_PARTITIONED
        = 1 / 0 forces it on / off; else `partitioned_dirty_min_packets`)."""
        env = os.environ.get("SSPD_SLIDE_PARTITIONED")
        if env is not None and env != "":
            want = env != "0"
        else:
            want = self.partitioned_dirty_min_packets > 0 and n >= self.partitioned_dirty_min_packets
        if not want:
            return False
        ok = getattr(self, "_k1b_ok", None)
        if ok is None:
            from ._abi import lib

            ok = self._k1b_ok = int(lib().sspd_scan_partitioned_variant(self._params, 0)) > 0
        return ok

    def _part_scratch_for(self, n: int, device):
        import torch

        from ._abi import lib

        chunk = -(-n // 4) * 4
        need = int(lib().sspd_scan_partitioned_scratch(self._params, chunk))
        buf = getattr(self, "_part_scratch", None)
        if buf is None or buf.numel() < need:
            buf = self._part_scratch = torch.empty(need, dtype=torch.uint8, device=device)
        return buf, chunk

    def _scan_slice_fused(self, h, o, dfr, iv, pool) -> bool:
        """Both halves of the slice in one K1b launch (LDCA half -> the
        slice's dirty bitmap, SEAV stamps from the sampled-packet queue);
        False when it does not apply (the caller then runs K1b + K2's SEAV
        half).  env SSPD_SLIDE_FUSED=0 disables it."""
        from ._abi import ERR_CONFIG, check, lib
        from ._device import stream_ptr

        if pool.ts_bytes != 2 or os.environ.get("SSPD_SLIDE_FUSED", "1") == "0":
            return False
        ok = getattr(self, "_k1b_fused_ok", None)
        if ok is None:
            ok = self._k1b_fused_ok = int(lib().sspd_scan_partitioned_variant(self._params, 0)) == 2
        if not ok:
            return False
        n = int(h.numel())
        buf, chunk = self._part_scratch_for(n, h.device)
        rc = lib().sspd_scan_sliding_partitioned(
            h.data_ptr(), o.data_ptr(), n, self._params, pool._buf.data_ptr(), pool.ts_bytes, pool._wrapped_now(),
            None if iv is None else iv["view"].device_buffer().data_ptr(),
            None if iv is None else iv["log"].data_ptr(), 0 if iv is None else iv["log"].numel(),
            None if iv is None else iv["meta"].data_ptr(), dfr.dirty_ptr(), 1 if dfr.fresh else 0,
            buf.data_ptr(), buf.numel(), chunk, stream_ptr())
        if rc == ERR_CONFIG:
            self._k1b_fused_ok = False
            return False
        check(rc, "sspd_scan_sliding_partitioned")
        return True

    def _scan_dirty_partitioned(self, h, o, dirty_ptr: int, fresh: bool = False):
        import torch

        from ._abi import check, lib
        from ._device import stream_ptr

        n = int(h.numel())
        chunk = -(-n // 4) * 4
        need = int(lib().sspd_scan_partitioned_scratch(self._params, chunk))
        buf = getattr(self, "_part_scratch", None)
        if buf is None or buf.numel() < need:
            buf = self._part_scratch = torch.empty(need, dtype=torch.uint8, device=h.device)
        fn = lib().sspd_scan_partitioned_fresh if fresh else lib().sspd_scan_partitioned
        check(fn(h.data_ptr(), o.data_ptr(), n, self._params, None, dirty_ptr, buf.data_ptr(), buf.numel(), chunk,
                 stream_ptr()), "sspd_scan_partitioned")

    def observe(self, hip: int, oip: int):
        self.observe_batch(np.array([hip], dtype=np.uint64), np.array([oip], dtype=np.uint64))

    def _materialize_into(self, sketch: SeavSketch):
        from ._device import call, stream_ptr

        pool = self.pool
        call("sspd_materialize_seav", pool._buf.data_ptr(), pool.ts_bytes, self._params,
             pool._wrapped_now(), pool.window_slices, sketch.device_buffer().data_ptr(), stream_ptr())

    def materialize_seav(self) -> SeavSketch:
        sketch = SeavSketch(self.seav_config, self.seeds, restore_cap=self.params.restore_cap,
                            _ldca_config=self.ldca_config)
        self._materialize_into(sketch)
        return sketch

    def materialize_ldca(self) -> np.ndarray:
        from ._device import zeros_bytes

        lc = self.ldca_config
        nbytes = lc.lr * lc.lc * lc.k // 8
        out = zeros_bytes(nbytes)
        self._ldca_view_into(out)
        return out[:nbytes].cpu().numpy().reshape(lc.lr, lc.lc, lc.k // 8)

    def materialize_ldca_cell(self, row: int, col: int) -> np.ndarray:
        lc = self.ldca_config
        base = self.layout.ldca_base + (row * lc.lc + col) * lc.k
        ts = self.pool.device_buffer()[base:base + lc.k].cpu().numpy().view(self.pool.dtype).astype(np.uint64)
        ages = (np.uint64(self.pool._wrapped_now()) - ts) & np.uint64(self.pool._mask)
        return np.packbits((ages < self.pool.window_slices).astype(np.uint8), bitorder="little")

    def _estimate(self, hip: int) -> tuple[float, bool]:
        import torch

        from ._device import call, ips_to_device, stream_ptr

        h = ips_to_device(np.array([hip], dtype=np.uint64))
        z0 = torch.empty(1, dtype=torch.int32, device=h.device)
        pool = self.pool
        call("sspd_filter_sliding", pool.device_buffer().data_ptr(), pool.ts_bytes, self._params,
             pool._wrapped_now(), pool.window_slices, h.data_ptr(), 1, None, z0.data_ptr(), None,
             stream_ptr())
        return ldc_estimate(int(z0.item()) & 0xFFFFFFFF, self.ldca_config.k)

    def views_into(self, seav_sketch, ldca_view):
        """Write the current active-bit views -- SEAV registers into
        `seav_sketch` (a SeavSketch of this geometry) and the packed LDCA
        into `ldca_view` (device bytes) -- as detect() builds them (the
        multi-GPU SlidingMerger ORs these across ranks)."""
        self._ldca_view_into(ldca_view)
        sv = self._seav_view()
        if sv is not seav_sketch:
            dst = seav_sketch.device_buffer()
            src = sv.device_buffer()
            n = min(dst.numel(), src.numel())
            dst[:n].copy_(src[:n])

    @traced("detect")
    def detect(self, beta: float | None = None) -> list[DetectionReport]:
        """Materialise (K4: SEAV registers + packed LDCA) -> fused finalize
        (K5 restore, sort, K6 filter, compaction; one host round trip)
        (sliding.py:232-248)."""
        from ._device import call, current_stream, stream_ptr, zeros_bytes

        beta = self.params.beta if beta is None else beta
        cutoff = beta * self.params.theta
        lview = getattr(self, "_ldca_view", None)
        if lview is None:
            lview = self._ldca_view = zeros_bytes(self._params.ldca_bytes)
        self._ldca_view_into(lview)  # first: fused with the fold of deferred stamps
        seav = self._seav_view()
        fin = DeviceFinalize(seav, lview, self._params, self.ldca_config.k, cutoff)
        return fin.reports(self.now, "sliding")

    @traced("detect_async")
    def detect_async(self, beta: float | None = None) -> PendingReports:
        """`detect()` pipelined with the caller's next slices.

        The active-bit views (K4: SEAV registers + packed LDCA) are built on
        the caller's stream, so the next `observe_batch` -- which rewrites
        stamps -- is ordered after them; the fused finalize (K5 restore,
        sort, K6 filter on the LDCA view, compaction) is enqueued on a side
        stream, with no host round trip, and overlaps the next slices' scans
        (K2 is bound by random-store traffic, K5 by issue slots).  Two view
        sets alternate; a set is reused only after the finalize that read it
        has been resolved.  The list resolves on first access; same reports
        as `detect()` (window_id = the slice of this call)."""
        import torch

        from ._device import call, current_stream, stream_ptr, zeros_bytes

        beta = self.params.beta if beta is None else beta
        cutoff = beta * self.params.theta
        st = _async_state(self)
        if len(st["sets"]) != self.pipeline_depth:
            for vs in st["sets"]:
                if vs is not None and vs[2] is not None:
                    vs[2].resolve()
            st["sets"] = [None] * max(1, self.pipeline_depth)
        i = st["n"] % len(st["sets"])
        st["n"] += 1
        vset = st["sets"][i]
        if vset is None:
            vset = st["sets"][i] = [self.materialize_seav(), zeros_bytes(self._params.ldca_bytes), None, {}]
        elif vset[2] is not None:
            vset[2].resolve()  # the finalize `pipeline_depth` calls ago is done with this view set
            vset[2].detach()  # its report arrays leave the set's graph buffers
        seav, lview = vset[0], vset[1]
        self._ldca_view_into(lview)  # first: fused with the fold of deferred stamps
        if self._iv() is not None:  # snapshot of the incremental view (16 MiB at r=16)
            src = self._seav_view().device_buffer()
            dst = seav.device_buffer()
            nbytes = src.numel() * src.element_size()
            if nbytes > dst.numel() * dst.element_size():
                raise ValueError("SEAV view snapshot larger than its view set buffer")
            call("sspd_copy_async", dst.data_ptr(), src.data_ptr(), nbytes, stream_ptr())
        else:
            self._materialize_into(seav)
        views_ready = st.get("views_ready")  # re-recorded per call: wait_event binds the current record
        if views_ready is None:
            views_ready = st["views_ready"] = torch.cuda.Event()
        views_ready.record(current_stream())
        side = st["side"]
        side.wait_event(views_ready)
        graphs = vset[3] if self.finalize_graphs else None
        fin = DeviceFinalize(seav, lview, self._params, self.ldca_config.k, cutoff, stream=side, graphs=graphs)
        vset[2] = fin
        now = self.now
        pending = PendingReports(lambda: fin.reports(now, "sliding"))
        if fin.shared:
            import weakref

            fin.owner = weakref.ref(pending)  # a dropped list needs no private copy of its arrays
        return pending


def _async_state(det):
    """Side stream and two view sets (double buffering)."""
    st = getattr(det, "_async", None)
    if st is None:
        import torch

        st = det._async = {"side": torch.cuda.Stream(device=torch.cuda.current_device()), "sets": [None, None],
                           "n": 0}
    return st


def detect_sliding(detector: SlidingDetector, theta: int | None = None, beta: float | None = None):
    if theta is not None and theta != detector.params.theta:
        raise ValueError(f"detector was configured with theta={detector.params.theta}, got {theta}")
    return detector.detect(beta=beta)
