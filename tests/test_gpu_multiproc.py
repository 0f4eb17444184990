"""The multi-GPU OR-merge transport (CUDA IPC + merge kernel) exercised by
two real processes sharing the single available GPU.

No kernel waits on another process: the processes only meet at host
barriers (gloo), exactly like the production protocol, so running both
ranks on one device is safe.  Each rank scans its shard into an IPC block;
the merged sketches on rank 0 must equal the single-process scan.
"""

import os
import socket
import warnings

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stream(seed=5, n=400_000):
    rng = np.random.default_rng(seed)
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    hips[:20_000] = 0xC0A80001
    return hips, oips


def _params():
    from paper_1901_07306_b200 import DetectorParams

    return DetectorParams(theta=1024, r=8, k=4096, lr=4, lc=512, design_n=4e5)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_1901_07306_b200 import DetectorState
    from paper_1901_07306_b200.multigpu import OrMerger

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(_params())
    merger = OrMerger(st, dist)
    out[f"transport{rank}"] = merger.transport
    hips, oips = _stream()
    for window in range(2):
        st.process_batch(hips[rank::world], oips[rank::world])
        merger.merge_to_root()
        if rank == 0:
            out[f"seav{window}"] = st.seav.payload_bytes()
            out[f"ldca{window}"] = st.ldca.payload_bytes()
            out[f"rep{window}"] = [(r.ip, r.estimated_cardinality, r.saturated) for r in st.finalize_window()]
        dist.barrier()
        st.reset()
        dist.barrier()
    merger.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_or_merge_two_processes_one_gpu(cuda, world):
    from paper_1901_07306_b200 import DetectorState

    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    assert all(out[f"transport{r}"] == "ipc" for r in range(world))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = DetectorState.create(_params())
    hips, oips = _stream()
    ref.process_batch(hips, oips)
    want = [(r.ip, r.estimated_cardinality, r.saturated) for r in ref.finalize_window()]
    for window in range(2):
        assert out[f"seav{window}"] == ref.seav.payload_bytes()
        assert out[f"ldca{window}"] == ref.ldca.payload_bytes()
        assert out[f"rep{window}"] == want and len(want) >= 1


def test_host_stream_ingest_matches_device_batch(cuda):
    """process_host_stream (pinned double-buffered H2D + scan) == process_batch."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, DetectorState

    rng = np.random.default_rng(12)
    n = 5_000_011
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = DetectorState.create(DetectorParams(r=12, design_n=1e6))
        b = DetectorState.create(DetectorParams(r=12, design_n=1e6))
    a.process_batch(hips, oips)
    h = torch.from_numpy(hips.view(np.int32)).pin_memory()
    o = torch.from_numpy(oips.view(np.int32)).pin_memory()
    moved = b.process_host_stream(h, o, chunk_pairs=1 << 20)
    assert moved == 8 * n
    b.process_host_stream(hips[:1000], oips[:1000])  # pageable numpy, idempotent replay
    assert a.seav.payload_bytes() == b.seav.payload_bytes()
    assert a.ldca.payload_bytes() == b.ldca.payload_bytes()
    assert a.finalize_window() == b.finalize_window()


def _sliding_worker(rank, world, port, out):
    """Rank r = one router of a sliding window over the packets whose index
    is r mod world; slices advanced in lockstep; detect via SlidingMerger at
    every slice (views OR-merged onto rank 0) plus one full age-min pool
    merge at the end."""
    import torch
    import torch.distributed as dist

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from paper_1901_07306_b200.multigpu import SlidingMerger

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(DetectorParams(theta=256, r=8, k=4096, lr=4, lc=256, design_n=2e5), window_slices=9)
    m = SlidingMerger(det, dist)
    out[f"transport{rank}"] = m.transport
    for s, (hips, oips) in enumerate(_slides()):
        det.observe_batch(hips[rank::world], oips[rank::world])
        reps = m.detect()
        if rank == 0:
            out[f"rep{s}"] = [(r.ip, r.estimated_cardinality, r.saturated, r.window_id) for r in reps]
        det.advance_slice()
    merged = m.merge_pools_to_root()
    if rank == 0:
        out["pool"] = merged.ts.tobytes()
    dist.barrier()
    m.close()
    dist.destroy_process_group()


def _slides(n_slides=24):
    rng = np.random.default_rng(44)
    heavy = rng.integers(0, 2**32, size=4, dtype=np.uint64)
    out = []
    for s in range(n_slides):
        n = int(rng.integers(10_000, 30_000))
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        if s < 6 or 12 <= s < 15:  # bursts that expire within the run (w = 9)
            hips[: n // 2] = heavy[s % 4]
        out.append((hips.astype(np.uint32), oips.astype(np.uint32)))
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_sliding_merger_two_processes_one_gpu(cuda, world):
    """N routers sharing one sliding window (north_star (4) in sliding mode):
    per-slide reports from the OR of the ranks' active-bit views and the
    age-min merged pool (merge_timestamp_pools across ranks) equal a single
    detector's over all packets."""
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_sliding_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    assert all(out[f"transport{r}"] == "ipc" for r in range(world))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = SlidingDetector(DetectorParams(theta=256, r=8, k=4096, lr=4, lc=256, design_n=2e5), window_slices=9)
    total = 0
    for s, (hips, oips) in enumerate(_slides()):
        ref.observe_batch(hips, oips)
        want = [(r.ip, r.estimated_cardinality, r.saturated, r.window_id) for r in ref.detect()]
        assert out[f"rep{s}"] == want, s
        total += len(want)
        ref.advance_slice()
    assert total > 0
    assert out["pool"] == ref.pool.ts.tobytes()
