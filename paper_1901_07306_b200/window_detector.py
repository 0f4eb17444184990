"""Discrete-window detector: one SEAV + one LDCA per window, on one GPU.

Mirrors `sspd/window_detector.py` (DetectorParams :39-69, DetectorState
:72-132).  The B200 differences:

* `process_batch` is ONE fused scan kernel (K1) that updates both sketches
  from one pass over the (hip, oip) stream -- the reference makes two
  passes (SEAV then LDCA, window_detector.py:100-103).
* `finalize_window` runs restore (K5), the device sort, the z0 filter (K6)
  with the keep decision as an integer table lookup, and a stable
  compaction on the device; only the kept (ip, z0) pairs come back to the
  host, where the float estimate is formed with the reference formula.
"""

from __future__ import annotations

import ctypes
import warnings
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from .hashing import DEFAULT_MASTER_SEED, SeedFamily
from .long_sketch import (
    DEFAULT_DESIGN_N,
    DEFAULT_V,
    LdcaConfig,
    LdcaSketch,
    check_noise,
    keep_table,
    ldc_estimate,
    plan_rows,
)
from .short_sketch import DEFAULT_RESTORE_CAP, SeavConfig, SeavSketch, sort_candidates
from .trace import traced

DEFAULT_BETA = 0.8


@dataclass(frozen=True)
class DetectionReport:
    ip: int
    estimated_cardinality: float
    saturated: bool
    window_id: int
    source: str = "discrete"


_EST_CACHE: dict = {}


def estimate_table(k: int) -> list:
    """est[z0] for z0 in [0, k] with the reference formula (long_sketch.py:33-44),
    computed once per k with math.log so every float is bit-identical."""
    t = _EST_CACHE.get(k)
    if t is None:
        t = [ldc_estimate(z0, k)[0] for z0 in range(k + 1)]
        _EST_CACHE[k] = t
    return t


class ReportList(Sequence):
    """The kept (ip, z0) pairs of one finalize, as a read-only sequence of
    DetectionReport built on access.

    Behaves like the reference's list[DetectionReport] (len, iteration,
    indexing, ==, `list += reports`); objects are only created when touched,
    so a window with tens of thousands of saturated candidates does not pay
    Python object construction unless the caller asks for them.  A list
    made by the fused device finalize knows its length from the device
    counts and copies the (ip, z0) arrays to the host on first access."""

    __slots__ = ("_ips", "_z0s", "k", "window_id", "source", "_est", "_n", "_fetch", "__weakref__")

    def __init__(self, ips, z0s, k: int, window_id: int, source: str, n: int | None = None, fetch=None):
        self._ips = ips
        self._z0s = z0s
        self._n = n
        self._fetch = fetch
        self.k = k
        self.window_id = window_id
        self.source = source
        self._est = estimate_table(k)

    def _arrays(self):
        if self._ips is None:
            self._ips, self._z0s = self._fetch()
            self._fetch = None
        return self._ips, self._z0s

    @property
    def ips(self) -> np.ndarray:
        return self._arrays()[0]

    @property
    def z0s(self) -> np.ndarray:
        return self._arrays()[1]

    def __len__(self) -> int:
        return self._n if self._n is not None else len(self.ips)

    def _make(self, i: int) -> DetectionReport:
        z0 = int(self.z0s[i])
        return DetectionReport(ip=int(self.ips[i]), estimated_cardinality=self._est[z0], saturated=z0 == 0,
                               window_id=self.window_id, source=self.source)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._make(j) for j in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("report index out of range")
        return self._make(i)

    def __iter__(self):
        est, wid, src = self._est, self.window_id, self.source
        for ip, z0 in zip(self.ips.tolist(), self.z0s.tolist()):
            yield DetectionReport(ip=ip, estimated_cardinality=est[z0], saturated=z0 == 0, window_id=wid,
                                  source=src)

    def __eq__(self, other) -> bool:
        if isinstance(other, ReportList):
            return (self.k == other.k and self.window_id == other.window_id and self.source == other.source
                    and np.array_equal(self.ips, other.ips) and np.array_equal(self.z0s, other.z0s))
        try:
            return list(self) == list(other)
        except TypeError:
            return NotImplemented

    def __ne__(self, other) -> bool:
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    def copy(self) -> list:
        """A plain list[DetectionReport] (for callers that mutate it)."""
        return list(self)

    def __add__(self, other):
        return list(self) + list(other)

    def __radd__(self, other):
        return list(other) + list(self)

    def __repr__(self) -> str:
        return f"ReportList({len(self)} reports, window_id={self.window_id}, source={self.source!r})"


@dataclass
class DetectorParams:
    theta: int = 1024
    r: int = 4
    sr: int = 4
    a: int = 2
    g: int = 8
    k: int = 8192
    lr: int | None = None
    lc: int | None = None
    v: int = DEFAULT_V
    design_n: float = DEFAULT_DESIGN_N
    beta: float = DEFAULT_BETA
    master_seed: int = DEFAULT_MASTER_SEED
    restore_cap: int = DEFAULT_RESTORE_CAP
    addr_bits: int = 32

    def seav_config(self) -> SeavConfig:
        return SeavConfig(r=self.r, sr=self.sr, a=self.a, theta=self.theta, g=self.g,
                          addr_bits=self.addr_bits)

    def ldca_config(self) -> LdcaConfig:
        lr, lc = self.lr, self.lc
        if lr is None:
            lr, lc = plan_rows(self.v, self.design_n, self.k)
        elif lc is None:
            lc = self.v // lr
        check_noise(self.k, self.design_n, lc, lr)
        return LdcaConfig(lr=lr, lc=lc, k=self.k)


_KEEP_CACHE: dict = {}


def device_keep_table(k: int, cutoff: float):
    """Cached device copy of keep_table(k, cutoff)."""
    import torch

    from ._device import device

    key = (k, cutoff, torch.cuda.current_device())
    t = _KEEP_CACHE.get(key)
    if t is None:
        t = torch.from_numpy(keep_table(k, cutoff)).to(device())
        _KEEP_CACHE[key] = t
    return t


_FINALIZE_SCRATCH: dict = {}  # (capacity, LR, LC) -> sspd_finalize work-space bytes
_SM_COUNT: dict = {}  # device -> SMs


def _hostfast_pack():
    """pack_u32 of the CPython staging binding (csrc/hostfast.c) bound to the
    loaded library's copy pool, or None when the module was not built."""
    try:
        from . import _hostfast
    except ImportError:
        return None
    from ._abi import lib

    _hostfast.set_pack(ctypes.cast(lib().sspd_host_pack_pairs, ctypes.c_void_p).value)
    return _hostfast.pack_u32


class DeviceFinalize:
    """One fused finalize (`sspd_finalize`: K5 restore -> sort -> K6 filter ->
    compaction) enqueued on a stream without any host round trip.

    The candidate capacity is the sketch's learned `_cand_cap`; the two
    device counts and the overflow flags are copied asynchronously into
    pinned memory.  `resolve()` waits for them (one synchronisation), re-runs
    with a larger capacity in the rare case the candidates did not fit (the
    inputs must still be intact: callers resolve before reusing them), and
    emits the reference's overflow warnings (short_sketch.py:398-407).
    `reports()` then returns a ReportList whose arrays are copied on first
    access."""

    def __init__(self, seav: SeavSketch, ldca_buf, params_block, k: int, cutoff: float, stream=None,
                 on_overflow: str = "warn", graphs: dict | None = None):
        import torch

        self.seav, self.ldca, self.p, self.k, self.cutoff = seav, ldca_buf, params_block, k, cutoff
        from ._device import current_stream

        self.stream = stream or current_stream()
        self.on_overflow = on_overflow
        self.m = None
        self.graphs = graphs
        self.shared = False  # self.out / self.h_tail belong to a replayed graph
        self.owner = None  # weakref to the PendingReports handed out for this result, if any
        self.list_ref = None  # weakref to the ReportList that still has to fetch its arrays
        self._launch(max(1024, seav._cand_cap))

    def _enqueue(self, cap: int, out, h_tail, table=None):
        """sspd_finalize into `out` + the pinned copy of its counts/flags."""
        from ._device import call, stream_ptr

        seav = self.seav
        if table is None:
            table = device_keep_table(self.k, self.cutoff)
        base = out.data_ptr()
        need = _FINALIZE_SCRATCH.get(self._scratch_key(cap)) or self._scratch_query(cap)
        scratch = seav._scratch(need)
        call("sspd_finalize", seav._buf.data_ptr(), self.ldca.data_ptr(), self.p, seav.restore_cap,
             table.data_ptr(), cap, base, base + 4 * cap, base + 8 * cap, base + 8 * cap + 16,
             scratch.data_ptr(), ctypes.byref(ctypes.c_size_t(need)), 1 if seav._radix_sort else 0, stream_ptr())
        # counts + flags back in ONE pinned copy
        h_tail.copy_(out[2 * cap:], non_blocking=True)

    def _launch(self, cap: int):
        import torch

        from ._device import on_stream

        seav = self.seav
        self.cap = cap
        nflag_words = ((1 << seav.config.r) + 1 + 3) // 4  # + the bucket-sort flag byte
        dev = seav._buf.device
        # one device block: ip[cap] | z0[cap] | counts (2 x u64) | overflow flags (2^r B) | bucket flag (1 B)
        shape = 2 * cap + 4 + nflag_words
        if self.graphs is not None:
            # per view set: the whole finalize (~12 launches, memsets and the
            # D2H copy of the counts) captured once per capacity / sort mode
            # and replayed as ONE graph launch; buffers belong to the graph.
            # Only the newest graph is kept (a new capacity, sort mode or
            # scratch buffer replaces it: the old one may hold freed scratch
            # pointers).  The keep table is a device INPUT of the graph: the
            # view set owns one (k+1)-byte buffer, refreshed on the stream
            # when beta*theta changes, so the cutoff is not part of the key.
            need = _FINALIZE_SCRATCH.get(self._scratch_key(cap)) or self._scratch_query(cap)
            scratch = seav._scratch(need)  # allocated outside the capture
            key = (cap, seav._radix_sort, self.ldca.data_ptr(), seav.restore_cap, scratch.data_ptr(), self.k)
            keep = self.graphs.get("keep")
            if keep is None or keep[0].numel() != self.k + 1:
                keep = self.graphs["keep"] = [torch.empty(self.k + 1, dtype=torch.uint8, device=dev), None]
            g = self.graphs.get("graph")
            if g is None or g[0] != key:
                self.graphs.pop("graph", None)
                out = torch.empty(shape, dtype=torch.int32, device=dev)
                h_tail = torch.empty(4 + nflag_words, dtype=torch.int32, pin_memory=True)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=self.stream, capture_error_mode="thread_local"):
                    self._enqueue(cap, out, h_tail, table=keep[0])
                g = self.graphs["graph"] = (key, graph, out, h_tail)
            _, graph, self.out, self.h_tail = g
            self.shared = True
            # the view set's previous finalize has been resolved before this
            # launch (detect_async), so its completion event is free to reuse
            ev = self.graphs.get("event")
            if ev is None:
                ev = self.graphs["event"] = torch.cuda.Event()
            with on_stream(self.stream):
                if keep[1] != self.cutoff:  # stream-ordered after every earlier replay's reads
                    keep[0].copy_(device_keep_table(self.k, self.cutoff), non_blocking=True)
                    keep[1] = self.cutoff
                graph.replay()
            ev.record(self.stream)
            self.event = ev
            return
        with torch.cuda.stream(self.stream):
            self.out = torch.empty(shape, dtype=torch.int32, device=dev)
            self.h_tail = torch.empty(4 + nflag_words, dtype=torch.int32, pin_memory=True)
            self._enqueue(cap, self.out, self.h_tail)
            self.event = torch.cuda.Event()
            self.event.record(self.stream)

    def _scratch_key(self, cap: int):
        p = self.p.contents if hasattr(self.p, "contents") else self.p
        return (cap, int(p.lr), int(p.lc))

    def _scratch_query(self, cap: int):
        from ._device import call

        nb = ctypes.c_size_t(0)
        call("sspd_finalize", None, None, self.p, 0, None, cap, None, None, None, None, None, ctypes.byref(nb), 0, 0)
        _FINALIZE_SCRATCH[self._scratch_key(cap)] = nb.value
        return nb.value

    def detach(self):
        """Before the graph that produced this result is replayed again:
        give a resolved, not yet fetched report list private copies of its
        device arrays (async, on the finalize's stream)."""
        import torch

        from ._device import call, on_stream

        if not self.shared or self.out is None:
            return
        self.resolve()
        rl = self.list_ref() if self.list_ref is not None else None
        if self.owner is not None and self.owner() is None and rl is None:  # nobody can read the arrays any more
            self.out = None
            self.shared = False
            return
        m, cap = self.m, self.cap
        with on_stream(self.stream):  # allocated and copied on the finalize's stream
            own = torch.empty(2 * cap if m else 0, dtype=torch.int32, device=self.out.device)
            if m:
                src, dst, sp = self.out.data_ptr(), own.data_ptr(), self.stream.cuda_stream
                call("sspd_copy_async", dst, src, 4 * m, sp)
                call("sspd_copy_async", dst + 4 * cap, src + 4 * cap, 4 * m, sp)
        self.out = own
        self.shared = False

    def resolve(self) -> int:
        """Number of reports (waits for the device counts; idempotent)."""
        if self.m is not None:
            return self.m
        from .errors import SeaOverflowError

        self.event.synchronize()
        nsea = 1 << self.seav.config.r
        found, kept = (int(x) for x in self.h_tail[:4].numpy().view(np.int64))
        if found > self.cap:  # candidates did not fit: learn the size, run again
            self.seav._cand_cap = 1 << (found - 1).bit_length()
            self._launch(self.seav._cand_cap)
            self.event.synchronize()
            found, kept = (int(x) for x in self.h_tail[:4].numpy().view(np.int64))
        if self.h_tail[4:].numpy().view(np.uint8)[nsea]:  # a bucket too large to order: radix sort from now on
            self.seav._radix_sort = True
            self._launch(self.cap)
            self.event.synchronize()
            found, kept = (int(x) for x in self.h_tail[:4].numpy().view(np.int64))
        self.found = found  # candidates restored
        flags = self.h_tail[4:].numpy().view(np.uint8)[:nsea]
        for rp in np.nonzero(flags)[0].tolist():
            err = SeaOverflowError(rp, self.seav.restore_cap)
            if self.on_overflow != "warn":
                raise err
            warnings.warn(str(err), RuntimeWarning, stacklevel=4)
        self.m = kept
        return kept

    def _fetch(self):
        import torch

        m, cap = self.m, self.cap
        host = torch.empty(2 * m, dtype=torch.int32, pin_memory=True)
        with torch.cuda.stream(self.stream):
            host[:m].copy_(self.out[:m], non_blocking=True)
            host[m:].copy_(self.out[cap:cap + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        ev.synchronize()
        both = host.numpy().view(np.uint32)
        self.out = None
        return both[:m].copy(), both[m:].copy()

    def reports(self, window_id: int, source: str) -> "ReportList":
        m = self.resolve()
        if m == 0:
            return ReportList(np.zeros(0, dtype=np.uint32), np.zeros(0, dtype=np.uint32), self.k, window_id, source)
        rl = ReportList(None, None, self.k, window_id, source, n=m, fetch=self._fetch)
        if self.shared:
            import weakref

            self.list_ref = weakref.ref(rl)
        return rl


class PendingReports(Sequence):
    """Report list of `SlidingDetector.detect_async` /
    `DetectorState.finalize_window_async`: the device pipeline is enqueued
    without a host round trip; the first access waits for it, then this
    behaves exactly like the ReportList the synchronous call returns."""

    __slots__ = ("_resolve", "_value", "__weakref__")

    def __init__(self, resolve):
        self._resolve = resolve
        self._value = None

    def result(self) -> ReportList:
        if self._value is None:
            self._value = self._resolve()
            self._resolve = None
        return self._value

    def done(self) -> bool:
        return self._value is not None

    def __len__(self) -> int:
        return len(self.result())

    def __getitem__(self, i):
        return self.result()[i]

    def __iter__(self):
        return iter(self.result())

    def __eq__(self, other) -> bool:
        return self.result() == (other.result() if isinstance(other, PendingReports) else other)

    def __repr__(self) -> str:
        return f"PendingReports({self.result()!r})" if self.done() else "PendingReports(<running>)"


@dataclass
class DetectorState:
    seav: SeavSketch
    ldca: LdcaSketch
    window_id: int = 0
    pair_count: int = 0
    params: DetectorParams = field(default_factory=DetectorParams)

    @classmethod
    def create(cls, params: DetectorParams | None = None) -> "DetectorState":
        params = params or DetectorParams()
        seeds = SeedFamily(params.master_seed)
        scfg = params.seav_config()
        lcfg = params.ldca_config()
        seav = SeavSketch(scfg, seeds, restore_cap=params.restore_cap, _ldca_config=lcfg)
        ldca = LdcaSketch(lcfg, seeds, _seav_config=scfg)
        return cls(seav=seav, ldca=ldca, params=params)

    @property
    def theta(self) -> int:
        return self.seav.config.theta

    def memory_bytes(self) -> tuple[int, int]:
        return self.seav.memory_bytes(), self.ldca.memory_bytes()

    def process_pair(self, hip: int, oip: int):
        self.process_batch(np.array([hip], dtype=np.uint64), np.array([oip], dtype=np.uint64))

    @traced("scan")
    def process_batch(self, hips, oips):
        """K1: one fused pass updating both sketches (window_detector.py:100-103).

        Host arrays (the reference's own call pattern: 65,536-pair numpy
        buffers, cli.py:215-217, distributed.py:225-227) are staged in pinned
        memory and scanned in batches of `host_stage_pairs` by the
        partitioned scan (see `_stage_host`); device tensors are scanned at
        once."""
        hs = self.__dict__.get("_hstage")
        if hs is not None and type(hips) is np.ndarray and type(oips) is np.ndarray:
            fast = hs["fast"]
            if (fast is not None and self.coalesce_host_batches and hs["cap"] == self.host_stage_pairs
                    and hs["hooked"] == (id(self.seav), id(self.ldca))):
                # the reference's call pattern through the CPython binding
                # (buffer protocol, no ctypes objects): -1 = not a plain
                # 1-D uint32 pair of equal length that fits -> paths below
                b, fill = hs["b"], hs["fill"]
                n = fast(hips, oips, hs["ph_addr"][b] + 4 * fill, hs["po_addr"][b] + 4 * fill, hs["cap"] - fill)
                if n > 0:
                    hs["fill"] = fill + n
                    self.pair_count += n
                    if hs["fill"] == hs["cap"]:
                        self._flush_host()
                    return
            # fast path of the reference's call pattern (uint32 numpy views
            # appended to live staging buffers): one native copy, no checks
            # beyond what the slow path would conclude for the same call
            n = hips.shape[0]
            if (hips.dtype == _U32 and oips.dtype == _U32 and hips.ndim == 1 and oips.ndim == 1
                    and n == oips.shape[0] and 0 < n <= hs["cap"] - hs["fill"] and self.coalesce_host_batches
                    and hips.flags.c_contiguous and oips.flags.c_contiguous and hs["cap"] == self.host_stage_pairs
                    and hs["hooked"] == (id(self.seav), id(self.ldca))):
                b, off = hs["b"], 4 * hs["fill"]
                rc = hs["pack"](hips.ctypes.data, oips.ctypes.data, n, 4, 4, hs["ph_addr"][b] + off,
                                hs["po_addr"][b] + off)
                if rc:
                    from ._abi import check
                    check(rc, "sspd_host_pack_pairs")
                hs["fill"] += n
                self.pair_count += n
                if hs["fill"] == hs["cap"]:
                    self._flush_host()
                return
        from ._device import ips_to_device
        from .errors import ConfigError

        if self.coalesce_host_batches and (type(hips) is np.ndarray or _is_host(hips)) and \
                (type(oips) is np.ndarray or _is_host(oips)):
            self._stage_host(hips, oips)
            return
        h = ips_to_device(hips, "hips")
        o = ips_to_device(oips, "oips")
        if h.numel() != o.numel():
            raise ConfigError("hips and oips differ in length")
        self._scan(h.data_ptr(), o.data_ptr(), int(h.numel()))
        self.pair_count += int(h.numel())

    # host-array batches are staged in pinned memory and scanned together
    # (class attributes, not dataclass fields)
    coalesce_host_batches = True
    host_stage_pairs = 1 << 23

    def _stage_host(self, hips, oips):
        """Append a host batch to the pinned staging buffer (one narrowing
        copy, keys checked first: nothing is staged from a rejected batch);
        a full buffer is copied to the device on a copy stream and scanned
        there while the host fills the other buffer.  Every read of either
        sketch (PreReadHook), reset and finalize apply or drop what is
        pending first, so the state any reader sees is exactly the
        reference's after the same process_batch calls (OR commutes)."""
        from ._abi import check, lib
        from .errors import ConfigError, DataError

        h, o = _host_array(hips, "hips"), _host_array(oips, "oips")
        n = int(h.shape[0])
        if n != int(o.shape[0]):
            raise ConfigError("hips and oips differ in length")
        L = lib()
        for a, name in ((h, "hips"), (o, "oips")):
            if a.dtype != np.uint32 and L.sspd_host_check_u32(a.ctypes.data, n, a.dtype.itemsize,
                                                               1 if a.dtype.kind == "i" else 0):
                raise DataError(f"{name}: IPv4 keys must lie in [0, 2^32)")
        hs = self._hstage if self._hstage_ok() else self._host_stage_state()
        pos = 0
        while pos < n:
            take = min(hs["cap"] - hs["fill"], n - pos)
            b, off = hs["b"], 4 * hs["fill"]
            hb, ob = h.dtype.itemsize, o.dtype.itemsize
            check(L.sspd_host_pack_pairs(h.ctypes.data + pos * hb, o.ctypes.data + pos * ob, take, hb, ob,
                                         hs["ph_addr"][b] + off, hs["po_addr"][b] + off), "sspd_host_pack_pairs")
            hs["fill"] += take
            pos += take
            if hs["fill"] == hs["cap"]:
                self._flush_host()
        self.pair_count += n

    def _hstage_ok(self) -> bool:
        """The staging buffers exist and both sketches carry this state's hook."""
        hs = getattr(self, "_hstage", None)
        return hs is not None and hs["cap"] == self.host_stage_pairs and \
            hs["hooked"] == (id(self.seav), id(self.ldca))

    def _host_stage_state(self):
        import weakref

        import torch

        from ._device import device

        hs = getattr(self, "_hstage", None)
        if hs is None or hs["cap"] != self.host_stage_pairs:
            if hs is not None:  # resized: scan what is staged, let the old buffers' copies/scans finish
                self._flush_host()
                torch.cuda.synchronize()
            cap, dev = int(self.host_stage_pairs), device()
            pin = lambda: torch.empty(cap, dtype=torch.int32, pin_memory=True)  # noqa: E731
            dbuf = lambda: torch.empty(cap, dtype=torch.int32, device=dev)  # noqa: E731
            hs = self._hstage = {"cap": cap, "fill": 0, "b": 0, "ph": [pin(), pin()], "po": [pin(), pin()],
                                 "dh": [dbuf(), dbuf()], "do": [dbuf(), dbuf()],
                                 "copied": [None, None], "free": [None, None],
                                 "stream": torch.cuda.Stream(device=dev)}
            hs["ph_addr"] = [t.data_ptr() for t in hs["ph"]]
            from ._abi import lib
            hs["pack"] = lib().sspd_host_pack_pairs
            hs["po_addr"] = [t.data_ptr() for t in hs["po"]]
            hs["fast"] = _hostfast_pack()
        hook = weakref.WeakMethod(self._flush_host)
        if self.seav._pre_read is None or self.seav._pre_read() != self._flush_host:
            self.seav._pre_read = hook
        if self.ldca._pre_read is None or self.ldca._pre_read() != self._flush_host:
            self.ldca._pre_read = hook
        hs["hooked"] = (id(self.seav), id(self.ldca))
        return hs

    def _flush_host(self):
        """Scan the staged host pairs (H2D on the copy stream, scan on the
        caller's stream); the host may refill the other buffer meanwhile."""
        import torch

        hs = getattr(self, "_hstage", None)
        if hs is None or hs["fill"] == 0:
            return
        m, b = hs["fill"], hs["b"]
        hs["fill"] = 0  # first: the scan below reads the sketches (re-entrant hook)
        compute = torch.cuda.current_stream()
        cs = hs["stream"]
        if hs["free"][b] is not None:
            cs.wait_event(hs["free"][b])  # the scan that last read device buffer b is done
        with torch.cuda.stream(cs):
            hs["dh"][b][:m].copy_(hs["ph"][b][:m], non_blocking=True)
            hs["do"][b][:m].copy_(hs["po"][b][:m], non_blocking=True)
            ev = hs["copied"][b] = torch.cuda.Event()
            ev.record(cs)
        compute.wait_event(ev)
        self._scan(hs["dh"][b].data_ptr(), hs["do"][b].data_ptr(), m)
        fr = hs["free"][b] = torch.cuda.Event()
        fr.record(compute)
        hs["b"] = b ^ 1
        if hs["copied"][b ^ 1] is not None:
            hs["copied"][b ^ 1].synchronize()  # its pinned buffers are written next

    def _drop_host(self):
        hs = getattr(self, "_hstage", None)
        if hs is not None:
            hs["fill"] = 0

    # "auto": the shared-memory partitioned scan (K1p) for large batches when
    # the LDCA fits in the SMs' shared memory, else the direct L2 scan (K1).
    scan_mode = "auto"  # or "direct" / "partitioned" (class attributes, not dataclass fields)
    partitioned_min_packets = 1 << 22
    partitioned_chunk = 0  # 0: library default (8 whole 4096-packet tiles per SM per chunk)

    @staticmethod
    def _default_chunk() -> int:
        """Packets per chunk of the partitioned scan's default plan (16 tiles
        of 4,096 packets per SM)."""
        import torch

        from ._abi import lib

        dev = torch.cuda.current_device()
        sms = _SM_COUNT.get(dev)
        if sms is None:
            sms = _SM_COUNT[dev] = int(lib().sspd_device_sm_count(dev))
        return 16 * 4096 * (sms if sms > 0 else 148)

    def _scan(self, h_ptr: int, o_ptr: int, n: int):
        from ._abi import ERR_CONFIG, check, lib
        from ._device import call, stream_ptr

        mode = self.scan_mode
        seav_p = self.seav.device_buffer().data_ptr()
        ldca_p = self.ldca.device_buffer().data_ptr()
        if mode == "partitioned" or (mode == "auto" and n >= self.partitioned_min_packets):
            scratch = getattr(self, "_part_scratch", None)
            # a batch smaller than the library's default chunk is ONE chunk of
            # its own size (smaller bucket scratch, same result)
            chunk = self.partitioned_chunk or (-(-n // 4) * 4 if n < self._default_chunk() else 0)
            need = int(lib().sspd_scan_partitioned_scratch(self.seav._params, chunk))
            if scratch is None or scratch.numel() < need:
                import torch

                scratch = torch.empty(need, dtype=torch.uint8, device=self.ldca.device_buffer().device)
                self._part_scratch = scratch
            rc = lib().sspd_scan_partitioned(h_ptr, o_ptr, n, self.seav._params, seav_p, ldca_p,
                                             scratch.data_ptr(), scratch.numel(), chunk, stream_ptr())
            if rc != ERR_CONFIG or mode == "partitioned":
                check(rc, "sspd_scan_partitioned")
                self.last_scan = "partitioned"
                return
        call("sspd_scan_discrete", h_ptr, o_ptr, n, self.seav._params, seav_p, ldca_p, stream_ptr())
        self.last_scan = "direct"

    @traced("host_stream")
    def process_host_stream(self, hips, oips, chunk_pairs: int = 1 << 23):
        """Stream HOST arrays through two device staging buffers: the H2D copy
        of chunk i+1 (copy stream) overlaps the K1 scan of chunk i (compute
        stream) -- the paper's watch-point buffer (
        distributed.py:222-228 is the CPU analogue).  Pinned torch CPU
        tensors give truly asynchronous copies; numpy arrays are accepted
        (pageable copies).  Returns the number of H2D bytes moved."""
        import torch

        from ._device import call, device, stream_ptr
        from .errors import ConfigError, DataError

        dev = device()
        h = _host_u32_tensor(hips, "hips")
        o = _host_u32_tensor(oips, "oips")
        n = int(h.numel())
        if n != int(o.numel()):
            raise ConfigError("hips and oips differ in length")
        if h.device.type != "cpu" or o.device.type != "cpu":
            raise DataError("process_host_stream takes host arrays; use process_batch for device tensors")
        chunk = max(1024, min(chunk_pairs, n))
        stage = getattr(self, "_stage", None)
        if stage is None or stage[0][0].numel() < chunk:
            stage = [(torch.empty(chunk, dtype=torch.int32, device=dev),
                      torch.empty(chunk, dtype=torch.int32, device=dev)) for _ in range(2)]
            self._stage = stage
            self._copy_stream = torch.cuda.Stream(device=dev)
            self._free = [torch.cuda.Event(), torch.cuda.Event()]
            self._ready = [torch.cuda.Event(), torch.cuda.Event()]
        compute = torch.cuda.current_stream(dev)
        cs = self._copy_stream
        for i, lo in enumerate(range(0, n, chunk)):
            b = i & 1
            m = min(chunk, n - lo)
            with torch.cuda.stream(cs):
                cs.wait_event(self._free[b])
                stage[b][0][:m].copy_(h[lo:lo + m], non_blocking=True)
                stage[b][1][:m].copy_(o[lo:lo + m], non_blocking=True)
                self._ready[b].record(cs)
            compute.wait_event(self._ready[b])
            self._scan(stage[b][0].data_ptr(), stage[b][1].data_ptr(), m)
            self._free[b].record(compute)
        self.pair_count += n
        return 8 * n

    @traced("finalize")
    def finalize_window(self, beta: float | None = None, source: str = "discrete") -> "ReportList":
        beta = self.params.beta if beta is None else beta
        cutoff = beta * self.theta
        k = self.ldca.config.k
        fin = DeviceFinalize(self.seav, self.ldca.device_buffer(), self.seav._params, k, cutoff)
        return fin.reports(self.window_id, source)

    def finalize_window_async(self, beta: float | None = None, source: str = "discrete") -> "PendingReports":
        """finalize_window without a host round trip.  The sketches are
        snapshotted on the device (10 MiB at config 2: a few microseconds)
        and the fused finalize runs on the snapshot, so `reset()` and the
        next window's scan are enqueued at once and the GPU never idles
        between windows.  The list resolves on first access (device counts,
        the reference's overflow warnings, a capacity re-run if needed --
        the snapshot is kept until then).  Two snapshots alternate; one is
        reused only after the finalize that read it has been resolved.  Same
        reports as finalize_window()."""
        from ._device import zeros_bytes

        beta = self.params.beta if beta is None else beta
        cutoff = beta * self.theta
        k = self.ldca.config.k
        snaps = getattr(self, "_snaps", None)
        if snaps is None:
            snaps = self._snaps = [None, None]
            self._snap_i = 0
        i = self._snap_i
        self._snap_i ^= 1
        snap = snaps[i]
        if snap is None:
            snap = snaps[i] = [SeavSketch(self.seav.config, self.seav.seeds, restore_cap=self.seav.restore_cap,
                                          _ldca_config=self.ldca.config), zeros_bytes(self.ldca.nbytes), None]
        elif snap[2] is not None:
            snap[2].resolve()  # the finalize two windows ago is done with this snapshot
        sv = snap[0].device_buffer()
        sv.copy_(self.seav.device_buffer()[: sv.numel()])
        snap[1].copy_(self.ldca.device_buffer()[: snap[1].numel()])
        snap[0]._cand_cap = max(snap[0]._cand_cap, self.seav._cand_cap, *(s[0]._cand_cap for s in snaps if s))
        snap[0]._radix_sort = snap[0]._radix_sort or self.seav._radix_sort or any(s[0]._radix_sort for s in snaps if s)
        fin = DeviceFinalize(snap[0], snap[1], self.seav._params, k, cutoff)
        snap[2] = fin
        wid = self.window_id
        return PendingReports(lambda: fin.reports(wid, source))

    def reset(self):
        self._drop_host()  # staged pairs of the window being cleared need no scan
        self.seav.clear()
        self.ldca.clear()
        self.window_id += 1
        self.pair_count = 0


_U32 = np.dtype(np.uint32)


def _is_host(a) -> bool:
    """A host array argument (numpy, a sequence, or a CPU torch tensor)."""
    import torch

    if isinstance(a, torch.Tensor):
        return a.device.type == "cpu"
    return isinstance(a, (np.ndarray, list, tuple))


def _host_array(a, name: str) -> np.ndarray:
    """Contiguous 1-D integer numpy view of a host key array (no copy when
    it already is one)."""
    if type(a) is np.ndarray and a.ndim == 1 and a.dtype.kind in "ui" and a.flags.c_contiguous:
        return a
    import torch

    from .errors import DataError

    if isinstance(a, torch.Tensor):
        a = a.contiguous().numpy()
        if a.dtype == np.int32:  # torch int32 carries the uint32 bit pattern (ips_to_device)
            a = a.view(np.uint32)
    arr = np.ascontiguousarray(np.asarray(a)).reshape(-1)
    if arr.dtype.kind not in "ui":
        raise DataError(f"{name}: integer array expected, got {arr.dtype}")
    return arr


def _host_u32_tensor(a, name: str):
    """Host IPv4 array as an int32 torch CPU tensor (uint32 bit pattern)."""
    import torch

    from .errors import DataError

    if isinstance(a, torch.Tensor):
        if a.dtype in (torch.int32, torch.uint32):
            return a.contiguous()
        a = a.cpu().numpy()
    arr = np.asarray(a)
    if arr.dtype.kind not in "ui":
        raise DataError(f"{name}: integer array expected, got {arr.dtype}")
    if arr.dtype != np.uint32:
        if arr.size and (int(arr.min()) < 0 or int(arr.max()) > 0xFFFFFFFF):
            raise DataError(f"{name}: IPv4 keys must lie in [0, 2^32)")
        arr = arr.astype(np.uint32)
    return torch.from_numpy(np.ascontiguousarray(arr).view(np.int32))


def process_pair(state: DetectorState, hip: int, oip: int) -> DetectorState:
    state.process_pair(hip, oip)
    return state


def finalize_window(state: DetectorState, theta: int | None = None, beta: float = DEFAULT_BETA):
    if theta is not None and theta != state.theta:
        raise ValueError(f"detector was configured with theta={state.theta}, got {theta}")
    return state.finalize_window(beta=beta)


def reset(state: DetectorState) -> DetectorState:
    state.reset()
    return state
