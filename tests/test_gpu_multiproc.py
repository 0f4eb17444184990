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
