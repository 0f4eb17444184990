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


class OrMerger:
    """OR-merge a DetectorState's sketches from every rank onto rank 0."""

    def __init__(self, state, dist, group=None, ops=None, allow_fallback: bool = True):
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ops = ops or DeviceOps()
        s_bytes = state.seav.nbytes
        l_bytes = state.ldca.nbytes
        self.seav_off = 0
        self.ldca_off = -(-s_bytes // 16) * 16
        self.nbytes = self.ldca_off + -(-l_bytes // 16) * 16
        self.base = self.ops.alloc(self.nbytes)
        if hasattr(self.ops, "tensor"):
            block = self.ops.tensor(self.base, self.nbytes)
            state.seav._rebind(block[: self.ldca_off])
            state.ldca._rebind(block[self.ldca_off:])
            self._block = block
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
        self.stripes = stripes(self.nbytes, self.world)
        self.last_merge_ms = 0.0

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
