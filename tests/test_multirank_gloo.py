"""Multi-process (gloo, CPU) tests of the multi-GPU merge protocol.

The production transport reads peer GPUs' blocks over NVLink through CUDA
IPC (paper_1901_07306_b200/multigpu.py DeviceOps).  Only one GPU exists in
this run, so the protocol -- handle exchange, stripe reduce-scatter, root
gather, barrier order, shard folding -- is exercised here by real
torch.distributed ranks with a shared-memory stand-in for the device ops.
"""

import os
import socket
import types

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1901_07306_b200.multigpu import OrMerger, shards_for_rank, stripes


class ShmOps:
    """CPU stand-in for DeviceOps: blocks are POSIX shared memory segments;
    a 'pointer' is (local block id << 40) | byte offset."""

    def __init__(self):
        self.blocks = {}
        self.next = 1

    def _reg(self, shm):
        bid = self.next
        self.next += 1
        self.blocks[bid] = shm
        return bid << 40

    def _view(self, ptr, n):
        shm = self.blocks[ptr >> 40]
        off = ptr & ((1 << 40) - 1)
        return np.ndarray((n,), dtype=np.uint8, buffer=shm.buf, offset=off)

    def alloc(self, nbytes):
        from multiprocessing import shared_memory

        shm = shared_memory.SharedMemory(create=True, size=nbytes)
        np.ndarray((nbytes,), dtype=np.uint8, buffer=shm.buf)[:] = 0
        return self._reg(shm)

    def handle(self, ptr):
        return self.blocks[ptr >> 40].name.encode()

    def open(self, handle):
        from multiprocessing import shared_memory

        return self._reg(shared_memory.SharedMemory(name=handle.decode()))

    def merge_or(self, srcs, dst, n):
        acc = np.zeros(n, dtype=np.uint8)
        for s in srcs:
            acc |= self._view(s, n)
        self._view(dst, n)[:] = acc

    def copy(self, dst, src, n):
        self._view(dst, n)[:] = self._view(src, n)

    def merge_age_min(self, srcs, dst, n_slots, ts_bytes, now):
        """K8 restated: per slot the stamp with the smallest wrapped age."""
        dt = np.dtype(f"u{ts_bytes}")
        mask = (1 << (8 * ts_bytes)) - 1
        stamps = [self._view(s, n_slots * ts_bytes).view(dt).astype(np.int64) for s in srcs]
        ages = np.stack([(now - x) & mask for x in stamps])
        best = np.min(ages, axis=0)
        self._view(dst, n_slots * ts_bytes).view(dt)[:] = ((now - best) & mask).astype(dt)

    def put_pool(self, ptr, pool):
        raw = pool.ts.tobytes()
        self._view(ptr, len(raw))[:] = np.frombuffer(raw, dtype=np.uint8)

    def pool_from(self, ptr, pool):
        return self._view(ptr, pool.n_slots * pool.ts_bytes).view(pool.ts.dtype).copy()

    def sync(self):
        pass

    def close(self, ptr):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, seav_bytes, ldca_bytes, results):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ops = ShmOps()
    state = types.SimpleNamespace(seav=types.SimpleNamespace(nbytes=seav_bytes),
                                  ldca=types.SimpleNamespace(nbytes=ldca_bytes))
    m = OrMerger(state, dist, ops=ops)
    assert m.transport == "ipc"
    for window in range(2):  # two windows through the same mapping
        rng = np.random.default_rng(1000 * window + rank)
        mine = (rng.random(m.nbytes) < 0.05).astype(np.uint8) << rng.integers(0, 8, m.nbytes).astype(np.uint8)
        ops._view(m.base, m.nbytes)[:] = mine
        dist.barrier()
        m.merge_to_root()
        if rank == 0:
            want = np.zeros(m.nbytes, dtype=np.uint8)
            for r in range(world):
                rr = np.random.default_rng(1000 * window + r)
                want |= (rr.random(m.nbytes) < 0.05).astype(np.uint8) << rr.integers(0, 8, m.nbytes).astype(np.uint8)
            results[window] = bool((ops._view(m.base, m.nbytes) == want).all())
        dist.barrier()
    dist.destroy_process_group()


class _FakePool:
    """A TimestampPool's protocol surface: u16 stamps, window, clock."""

    def __init__(self, rank, n=4099, w=9, now=37):
        rng = np.random.default_rng(77 + rank)
        self.n_slots, self.ts_bytes, self.window_slices, self.now = n, 2, w, now
        self.ts = ((now - rng.integers(0, 3 * w, n)) & 0xFFFF).astype(np.uint16)

    def _wrapped_now(self):
        return self.now & 0xFFFF


def _pool_worker(rank, world, port, results):
    import torch.distributed as dist

    from paper_1901_07306_b200.multigpu import SlidingMerger

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ops = ShmOps()
    det = types.SimpleNamespace(pool=_FakePool(rank), _params=types.SimpleNamespace(seav_bytes=4096, ldca_bytes=1000))
    m = SlidingMerger(det, dist, ops=ops)
    merged = m.merge_pools_to_root()
    if rank == 0:
        pools = [_FakePool(r).ts.astype(np.int64) for r in range(world)]
        ages = np.stack([(37 - x) & 0xFFFF for x in pools])
        want = ((37 - ages.min(axis=0)) & 0xFFFF).astype(np.uint16)
        results["pool"] = bool((merged == want).all())
    else:
        results[f"none{rank}"] = merged is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sliding_pool_age_min_protocol_gloo(world):
    """SlidingMerger.merge_pools_to_root (merge_timestamp_pools across ranks,
    distributed.py:176-192): each rank age-min-merges one slot stripe of all
    pools over peer memory, rank 0 gathers -- equals the per-slot minimum
    wrapped age over all ranks' pools."""
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    mp.start_processes(_pool_worker, args=(world, _free_port(), results), nprocs=world, join=True,
                       start_method="spawn")
    assert results["pool"] and all(results[f"none{r}"] for r in range(1, world))


@pytest.mark.parametrize("world", [2, 3])
def test_or_merge_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, 32768 + 5, 65536 + 3, results), nprocs=world,
                       join=True, start_method="spawn")
    assert results[0] and results[1]


def test_stripes_cover_block():
    for n in (16, 1000, 65552, 10 * (1 << 20) + 48):
        for w in (1, 2, 3, 8):
            s = stripes(n, w)
            assert s[0][0] == 0 and s[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
            assert all(lo % 16 == 0 for lo, _ in s)


def test_shard_folding_config3():
    for world in (1, 2, 4, 8):
        got = sorted(x for r in range(world) for x in shards_for_rank(8, r, world))
        assert got == list(range(8))
        assert all(len(shards_for_rank(8, r, world)) == 8 // world for r in range(world))
