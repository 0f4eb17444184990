"""Multi-GPU watch-point mode: one process per GPU, OR-merge over NVLink.

The reference simulates watch points in one process and merges serialized
frames with a host OR (distributed.py:231-271, merge_frames :145-173).  On
one 8xB200 box every GPU is a border router over its own shard; at window
end the (SEAV || LDCA) blocks of all ranks are OR-reduced and rank 0 (the
global server) runs restore + filter once.

NCCL has no bitwise-OR reduction (ncclRedOp_t is sum/prod/max/min/avg), so
the merge is our own kernel reading PEER memory directly:

  1. every rank's SEAV+LDCA live in ONE cudaMalloc block whose CUDA IPC
     handle is exchanged once (all_gather_object) and opened by all peers;
  2. reduce-scatter: rank r runs sspd_merge_or over stripe r of all G
     blocks (G-1 of them peers, read over NVLink) into its own stripe r;
  3. gather: rank 0 copies stripe r from rank r for every r != 0.

Root ingress is (G-1)/G of one block instead of (G-1) blocks.  Barriers on
the process group order the phases (no kernel ever waits on another rank's
kernel).  If IPC cannot be opened (e.g. no peer access), the fallback is
an NCCL all_gather of the blocks followed by the same OR kernel locally.

Sliding mode (BASELINE configs[3] across routers): every rank keeps its own
timestamp pool over its shard, advancing slices in lockstep.  The
reference merges pools by the per-slot minimum wrapped age
(merge_timestamp_pools, distributed.py:176-192); a slot of the merged pool
is active iff its minimum age is < w, i.e. iff it is active on SOME rank.
So detection needs only the OR of the ranks' active-bit views (SEAV
registers || packed LDCA: 24 MiB at r = 16) -- the same stripe protocol --
instead of the 403 MB pools (SlidingMerger.detect); the full age-min pool
merge is there too for state hand-over and equivalence checks
(SlidingMerger.merge_pools_to_root).

The transport calls go through an `ops` object so the protocol (striping,
phase order, barriers) is exercised by multi-process gloo tests on CPU
(tests/test_multirank_gloo.py) with a shared-memory stand-in for the
device ops.
"""

from __future__ import annotations

import ctypes

from .trace import traced


def stripes(nbytes: int, world: int, align: int = 16) -> list[tuple[int, int]]:
    """[lo, hi) byte stripe per rank, 16-byte aligned, covering [0, nbytes)."""
    per = -(-nbytes // world)
    per = -(-per // align) * align
    out = []
    for r in range(world):
        lo = min(nbytes, r * per)
        hi = min(nbytes, lo + per)
        out.append((lo, hi))
    return out


def shards_for_rank(n_shards: int, rank: int, world: int) -> list[int]:
    """Config-3 folding: GPU g scans shards g, g+G, g+2G, ... (BASELINE configs[2])."""
    return list(range(rank, n_shards, world))


class DeviceOps:
    """The production transport: CUDA IPC blocks + libsspd_b200 kernels."""

    def __init__(self):
        from ._abi import lib

        self.lib = lib()

    def alloc(self, nbytes: int) -> int:
        from ._abi import check

        p = ctypes.c_void_p()
        check(self.lib.sspd_ipc_alloc(nbytes, ctypes.byref(p)), "sspd_ipc_alloc")
        return p.value

    def free(self, ptr: int):
        self.lib.sspd_ipc_free(ptr)

    def handle(self, ptr: int) -> bytes:
        from ._abi import check

        buf = ctypes.create_string_buffer(64)
        check(self.lib.sspd_ipc_get_handle(ptr, buf), "sspd_ipc_get_handle")
        return buf.raw

    def open(self, handle: bytes) -> int | None:
        p = ctypes.c_void_p()
        rc = self.lib.sspd_ipc_open(handle, ctypes.byref(p))
        return p.value if rc == 0 else None

    def close(self, ptr: int):
        self.lib.sspd_ipc_close(ptr)

    def merge_or(self, srcs: list[int], dst: int, nbytes: int):
        from ._abi import check
        from ._device import stream_ptr

        arr = (ctypes.c_void_p * len(srcs))(*srcs)
        check(self.lib.sspd_merge_or(arr, len(srcs), dst, nbytes, stream_ptr()), "sspd_merge_or")

    def merge_age_min(self, srcs: list[int], dst: int, n_slots: int, ts_bytes: int, now_wrapped: int):
        from ._abi import check
        from ._device import stream_ptr

        arr = (ctypes.c_void_p * len(srcs))(*srcs)
        check(self.lib.sspd_merge_age_min(arr, len(srcs), dst, n_slots, ts_bytes, now_wrapped, stream_ptr()),
              "sspd_merge_age_min")

    def copy(self, dst: int, src: int, nbytes: int):
        from ._abi import check
        from ._device import stream_ptr

        check(self.lib.sspd_copy_async(dst, src, nbytes, stream_ptr()), "sspd_copy_async")

    def sync(self):
        import torch

        torch.cuda.synchronize()

    def tensor(self, ptr: int, nbytes: int):
        """Zero-copy torch uint8 view of a device block."""
        import torch

        class _Cai:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

        return torch.as_tensor(_Cai(), device="cuda")


class BlockMerger:
    """One IPC block per rank and the OR reduce-to-root protocol over it."""

    def __init__(self, nbytes: int, dist, group=None, ops=None, allow_fallback: bool = True):
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ops = ops or DeviceOps()
        self.nbytes = nbytes
        self.base = self.ops.alloc(self.nbytes)
        self._block = self.ops.tensor(self.base, self.nbytes) if hasattr(self.ops, "tensor") else None
        self._open_peers(allow_fallback)
        self.stripes = stripes(self.nbytes, self.world)
        self.last_merge_ms = 0.0

    def _open_peers(self, allow_fallback: bool):
        dist, group = self.dist, self.group
        handles = [None] * self.world
        dist.all_gather_object(handles, self.ops.handle(self.base), group=group)
        self.peers: list[int | None] = []
        ok = True
        for r, h in enumerate(handles):
            if r == self.rank:
                self.peers.append(self.base)
                continue
            p = self.ops.open(h)
            ok &= p is not None
            self.peers.append(p)
        flags = [None] * self.world
        dist.all_gather_object(flags, ok, group=group)
        self.transport = "ipc" if all(flags) else "nccl"
        if self.transport == "nccl" and not allow_fallback:
            raise RuntimeError("CUDA IPC peer mapping failed on some rank")

    def traffic(self) -> dict:
        """Bytes one merge moves: each rank reads its stripe of every peer's
        block (reduce-scatter) and the root reads every other stripe back
        (gather)."""
        lo, hi = self.stripes[self.rank]
        peer_reads = (self.world - 1) * (hi - lo) if self.transport == "ipc" else (self.world - 1) * self.nbytes
        root_ingress = sum(h - l for r, (l, h) in enumerate(self.stripes) if r != 0)
        return {"block_bytes": self.nbytes, "peer_read_bytes_this_rank": peer_reads,
                "root_gather_bytes": root_ingress, "transport": self.transport}

    @traced("merge")
    def merge_to_root(self):
        """After every rank finished scanning: rank 0's block = OR of all blocks.

        `last_merge_ms` = host wall time from the barrier that follows this
        rank's scan to the end of the merge (both data phases, their device
        syncs and the two further barriers)."""
        import time

        self._before_merge()
        if self.transport == "nccl":
            self.ops.sync()
            self.dist.barrier(group=self.group)
            t0 = time.perf_counter()
            self._merge_nccl()
            self.last_merge_ms = (time.perf_counter() - t0) * 1e3
            return
        d = self.dist
        self.ops.sync()
        d.barrier(group=self.group)              # all scans complete
        t0 = time.perf_counter()
        lo, hi = self.stripes[self.rank]
        if hi > lo:                               # reduce-scatter: my stripe of every block
            self.ops.merge_or([p + lo for p in self.peers], self.base + lo, hi - lo)
        self.ops.sync()
        d.barrier(group=self.group)              # all stripes reduced
        if self.rank == 0:                        # gather stripes onto the root
            for r in range(1, self.world):
                lo, hi = self.stripes[r]
                if hi > lo:
                    self.ops.copy(self.base + lo, self.peers[r] + lo, hi - lo)
            self.ops.sync()
        d.barrier(group=self.group)              # root done reading peers
        self.last_merge_ms = (time.perf_counter() - t0) * 1e3

    def _before_merge(self):
        """Hook: make the block complete before peers read it."""

    def _merge_nccl(self):
        import torch

        block = self._block
        out = torch.empty(self.world * self.nbytes, dtype=torch.uint8, device=block.device)
        self.dist.all_gather_into_tensor(out, block, group=self.group)
        if self.rank == 0:
            srcs = [out.data_ptr() + r * self.nbytes for r in range(self.world)]
            self.ops.merge_or(srcs, self.base, self.nbytes)
            self.ops.sync()

    def close(self):
        for r, p in enumerate(self.peers):
            if r != self.rank and p is not None:
                self.ops.close(p)
        self.peers = []


def _two_part_layout(a_bytes: int, b_bytes: int) -> tuple[int, int]:
    """(offset of the second part, block bytes): both parts 16-byte padded."""
    off = -(-a_bytes // 16) * 16
    return off, off + -(-b_bytes // 16) * 16


class OrMerger(BlockMerger):
    """OR-merge a DetectorState's sketches from every rank onto rank 0: the
    state's SEAV and LDCA are moved into the rank's IPC block (SEAV || LDCA),
    so the scans write it directly and the merge needs no copy."""

    def __init__(self, state, dist, group=None, ops=None, allow_fallback: bool = True):
        self.seav_off = 0
        self.ldca_off, nbytes = _two_part_layout(state.seav.nbytes, state.ldca.nbytes)
        super().__init__(nbytes, dist, group, ops, allow_fallback)
        self._state = state
        if self._block is not None:
            state.seav._rebind(self._block[: self.ldca_off])
            state.ldca._rebind(self._block[self.ldca_off:])

    def _before_merge(self):
        # host batches the state has staged but not scanned yet (the pre-read
        # hook of its sketches) must reach the block before peers read it
        flush = getattr(self._state, "_flush_host", None)
        if flush is not None:
            flush()


class SlidingMerger(BlockMerger):
    """N routers sharing one sliding window (one SlidingDetector per rank,
    slices advanced in lockstep).  `detect()` -- called on every rank at the
    same slice -- builds each rank's active-bit views (SEAV registers ||
    packed LDCA) in its IPC block, OR-merges them onto rank 0 and finalizes
    there once: the reports equal a single detector's over the union of the
    ranks' packets (the merged pool's slot is active iff it is active on
    some rank).  `merge_pools_to_root()` is the reference's
    merge_timestamp_pools across ranks (per-slot minimum wrapped age, K8 by
    stripes over peer memory) for state hand-over and checks."""

    def __init__(self, det, dist, group=None, ops=None, allow_fallback: bool = True):
        self.det = det
        p = det._params
        self.seav_bytes, self.ldca_bytes = int(p.seav_bytes), int(p.ldca_bytes)
        self.ldca_off, nbytes = _two_part_layout(self.seav_bytes, self.ldca_bytes)
        super().__init__(nbytes, dist, group, ops, allow_fallback)
        self.seav_view = self.ldca_view = None
        if self._block is not None:
            from .short_sketch import SeavSketch

            sk = SeavSketch(det.seav_config, det.seeds, restore_cap=det.params.restore_cap,
                            _ldca_config=det.ldca_config)
            sk._rebind(self._block[: self.ldca_off])
            self.seav_view = sk
            self.ldca_view = self._block[self.ldca_off: self.ldca_off + self.ldca_bytes]
        self._pool_merger = None

    @traced("merge_detect")
    def detect(self, beta: float | None = None):
        """Every rank: its views into the block; rank 0: the merged report
        list (window_id = the slice, source "sliding"); other ranks: []."""
        from .window_detector import DeviceFinalize

        det = self.det
        det.views_into(self.seav_view, self.ldca_view)
        self.merge_to_root()
        if self.rank != 0:
            return []
        beta = det.params.beta if beta is None else beta
        fin = DeviceFinalize(self.seav_view, self.ldca_view, det._params, det.ldca_config.k,
                             beta * det.params.theta)
        return fin.reports(det.now, "sliding")

    def merge_pools_to_root(self):
        """merge_timestamp_pools over the ranks' pools (distributed.py:176-192):
        every rank copies its pool into an IPC block; rank r age-min-merges
        stripe r of all of them (K8 over peer memory) into its scratch; rank 0
        gathers the stripes.  Returns the merged TimestampPool on rank 0
        (None elsewhere).  The pools must agree on geometry, w and `now`."""
        from .errors import MergeError

        det, pool = self.det, self.det.pool
        meta = (pool.n_slots, pool.ts_bytes, pool.window_slices, pool.now)
        metas = [None] * self.world
        self.dist.all_gather_object(metas, meta, group=self.group)
        if any(m != meta for m in metas):
            raise MergeError(f"timestamp pools disagree across ranks: {sorted(set(metas))}")
        n_slots, tb = pool.n_slots, pool.ts_bytes
        nbytes = n_slots * tb
        if self._pool_merger is None or self._pool_merger.nbytes != 2 * nbytes:
            self._pool_merger = BlockMerger(2 * nbytes, self.dist, self.group, self.ops)
        pm = self._pool_merger
        if pm._block is not None:  # [my pool | merged stripes]
            import torch

            pm._block[:nbytes].copy_(pool.device_buffer().view(torch.uint8))
        else:
            self.ops.put_pool(pm.base, pool)  # CPU stand-in (tests)
        slot_stripes = stripes(n_slots, self.world, align=8)
        self.ops.sync()
        self.dist.barrier(group=self.group)
        lo, hi = slot_stripes[self.rank]
        if hi > lo:
            self.ops.merge_age_min([q + lo * tb for q in pm.peers], pm.base + nbytes + lo * tb, hi - lo, tb,
                                   pool._wrapped_now())
        self.ops.sync()
        self.dist.barrier(group=self.group)
        merged = None
        if self.rank == 0:
            for r in range(1, self.world):
                lo, hi = slot_stripes[r]
                if hi > lo:
                    self.ops.copy(pm.base + nbytes + lo * tb, pm.peers[r] + nbytes + lo * tb, (hi - lo) * tb)
            self.ops.sync()
            merged = (_pool_like(pool, pm._block[nbytes:2 * nbytes]) if pm._block is not None
                      else self.ops.pool_from(pm.base + nbytes, pool))
        self.dist.barrier(group=self.group)
        return merged


def _pool_like(pool, data_u8):
    """A TimestampPool with `pool`'s geometry, window and clock whose stamps
    are a copy of `data_u8` (device bytes)."""
    from .sliding import TimestampPool

    merged = TimestampPool.__new__(TimestampPool)
    merged.__dict__.update({k: v for k, v in pool.__dict__.items() if k not in ("_buf", "_deferred")})
    merged._deferred = None
    merged._buf = data_u8.clone().view(pool._buf.dtype)
    return merged
