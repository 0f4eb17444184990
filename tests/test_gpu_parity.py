"""CUDA path vs the reference's golden vectors and the pinned CPU oracle.

Every test here drives the drop-in API (paper_1901_07306_b200) -> ctypes ->
libsspd_b200.so kernels on the GPU.  Bar: bit-exact bytes, identical
candidate lists, identical reports (float estimates compared with ==).
"""

import hashlib
import warnings
import zlib

import numpy as np
import pytest

from conftest import params_block, params_from

pytestmark = pytest.mark.gpu


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def rep_list(reps):
    return [[r.ip, repr(r.estimated_cardinality), r.saturated, r.window_id, r.source] for r in reps]


def make_state(dp):
    from paper_1901_07306_b200 import DetectorState

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return DetectorState.create(dp)


@pytest.mark.parametrize("idx", range(12))
def test_golden_sketch_cases(cuda, golden, garr, idx):
    if idx >= len(golden["sketches"]):
        pytest.skip("no such case")
    case = golden["sketches"][idx]
    dp = params_from(case["params"])
    st = make_state(dp)
    st.process_batch(garr[case["hips"]], garr[case["oips"]])
    assert sha(st.seav.payload_bytes()) == case["seav_sha"], case["name"]
    assert sha(st.ldca.payload_bytes()) == case["ldca_sha"], case["name"]
    with warnings.catch_warnings(record=True) as wl:
        warnings.simplefilter("always")
        cands = st.seav.restore(on_overflow="warn")
    over = sorted(int(str(w.message).split("rp=")[1].split()[0]) for w in wl if "rp=" in str(w.message))
    assert over == case["overflow"]
    assert [[c.ip, c.source_sea, c.union_weight] for c in cands] == case["candidates"]
    for ip, z0 in case["z0"]:
        assert int(st.ldca.zero_counts(np.array([ip]))[0]) == z0
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert rep_list(st.finalize_window()) == [r[:3] + [0, "discrete"] for r in case["reports"]]


def test_config1_end_to_end(cuda, golden):
    from paper_1901_07306_b200 import DetectorParams
    from tools.workloads import CONFIG1, generate

    c = golden["config1"]
    hips, oips, _ = generate(CONFIG1)
    st = make_state(DetectorParams())
    for lo in range(0, len(hips), 1 << 16):  # the CLI's 64 Ki-pair buffers (cli.py:215-217)
        st.process_batch(hips[lo:lo + (1 << 16)], oips[lo:lo + (1 << 16)])
    assert sha(st.seav.payload_bytes()) == c["seav_sha"]
    assert sha(st.ldca.payload_bytes()) == c["ldca_sha"]
    assert [[x.ip, x.source_sea, x.union_weight] for x in st.seav.restore()] == c["candidates"]
    assert rep_list(st.finalize_window()) == c["reports"]
    # one launch over the whole window gives the same state
    st2 = make_state(DetectorParams())
    st2.process_batch(hips, oips)
    assert st2.seav.payload_bytes() == st.seav.payload_bytes()
    assert st2.ldca.payload_bytes() == st.ldca.payload_bytes()


def test_config1_device_generated_stream(cuda, golden):
    """The torch/CUDA generator backend emits the identical stream."""
    import torch

    from tools.workloads import CONFIG1, generate

    h, o, _ = generate(CONFIG1, "torch", cuda)
    hb = h.cpu().numpy().view(np.uint32)
    ob = o.cpu().numpy().view(np.uint32)
    assert sha(hb.tobytes() + ob.tobytes()) == golden["config1"]["stream_sha"]
    del torch


def test_overflow_semantics(cuda, golden, garr):
    from paper_1901_07306_b200 import SeaOverflowError, SeavConfig, SeavSketch, SeedFamily

    g = golden["overflow"]
    sk = SeavSketch(SeavConfig(), SeedFamily(), restore_cap=g["cap"])
    sk.load_payload(garr[g["payload"]].tobytes())
    with pytest.warns(RuntimeWarning, match="rp=3"):
        cands = sk.restore(on_overflow="warn")
    assert [[c.ip, c.source_sea, c.union_weight] for c in cands] == g["candidates"]
    with pytest.raises(SeaOverflowError) as err:
        sk.restore()
    assert err.value.rp == 3
    with pytest.raises(SeaOverflowError):
        sk.restore_sea(7)
    assert sk.restore_sea(1) == [c for c in cands if c.source_sea == 1]
    big = SeavSketch(SeavConfig(), SeedFamily(), restore_cap=10**9)
    big.load_payload(garr[g["payload"]].tobytes())
    # 3.3 M tuples counted exactly, emitted only when weight >= 3
    assert len(big.restore_sea(7)) == g["rp7_uncapped_count"]


@pytest.mark.parametrize("geom", [
    dict(theta=64, r=4, k=1024, lr=3, lc=32),
    dict(theta=32, r=2, sr=5, a=1, k=2048, lr=4, lc=100),
    dict(theta=128, r=8, g=16, k=1000, lr=5, lc=77),
    dict(theta=16, r=2, sr=6, a=1, g=32, k=512, lr=9, lc=64),
    dict(theta=4096, r=8, sr=3, a=4, g=64, k=2048, lr=2, lc=512),
    dict(theta=1024, r=12, k=8192, lr=8, lc=1024),
    dict(theta=256, r=16, k=4096, lr=2, lc=4096),
    dict(theta=8, r=4, addr_bits=16, k=256, lr=2, lc=16),
    dict(theta=1024, r=16, k=8192, lr=8, lc=8192),  # config 5: 64 MiB LDCA
    # the warp restore's hot-mask enumeration beyond SR = 4 / 64-column rows:
    dict(theta=256, r=16, sr=4, a=1, k=4096, lr=4, lc=512),   # SR = 4, 32-column rows
    dict(theta=256, r=12, sr=4, a=1, k=4096, lr=4, lc=512),   # SR = 4, 64-column rows
    dict(theta=256, r=12, sr=5, a=1, k=4096, lr=4, lc=512),   # stack walk, SR = 5
    dict(theta=256, r=8, sr=6, a=1, k=4096, lr=4, lc=512),    # SR = 6
    dict(theta=256, r=11, sr=7, a=2, k=4096, lr=4, lc=512),   # SR = 7
    dict(theta=256, r=16, sr=8, a=1, k=4096, lr=4, lc=512),   # SR = 8, 8-column rows
])
def test_random_streams_vs_oracle(cuda, oracle, geom):
    """Geometries beyond the golden set, checked against the pinned oracle."""
    from paper_1901_07306_b200 import DetectorParams

    dp = DetectorParams(design_n=1e5, **geom)
    _, lcfg, p = params_block(dp)
    rng = np.random.default_rng(zlib.crc32(repr(sorted(geom.items())).encode()))
    n = 300_000
    span = 1 << dp.addr_bits
    hips = rng.integers(0, span, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    heavy = rng.integers(0, span, size=12, dtype=np.uint64)
    for i, h in enumerate(heavy):
        hips[i * 6000:(i + 1) * 6000 - i * 300] = h
    st = make_state(dp)
    st.process_batch(hips, oips)
    seav, ldca = oracle.scan(p, hips, oips, threads=8)
    assert st.seav.payload_bytes() == seav.tobytes()
    assert st.ldca.payload_bytes() == ldca.tobytes()
    ips, rps, ws, over = oracle.restore(p, seav, dp.restore_cap)
    with warnings.catch_warnings(record=True):
        warnings.simplefilter("always")
        got = st.seav.restore(on_overflow="warn")
    assert [(c.ip, c.source_sea, c.union_weight) for c in got] == list(
        zip(ips.tolist(), rps.tolist(), ws.tolist()))
    z0 = oracle.filter_z0(p, ldca, ips)
    assert (st.ldca.zero_counts(ips) == z0).all()


def test_edge_inputs(cuda):
    from paper_1901_07306_b200 import DataError, DetectorParams

    st = make_state(DetectorParams(design_n=2e5))
    st.process_batch(np.array([], dtype=np.uint32), np.array([], dtype=np.uint32))
    assert st.seav.total_set_bits() == 0 and st.finalize_window() == []
    st.process_pair(0xC0A80101, 0xDEADBEEF)
    assert st.pair_count == 1
    assert 1 <= int(np.unpackbits(st.ldca.data).sum()) <= st.ldca.config.lr
    with pytest.raises(DataError):
        st.process_batch(np.array([2**32], dtype=np.uint64), np.array([1], dtype=np.uint64))
    with pytest.raises(DataError):
        st.process_batch(np.array([-1], dtype=np.int64), np.array([1], dtype=np.int64))


def test_unaligned_and_ragged_batches(cuda, oracle):
    """Odd offsets take the scalar kernel; any split gives the same state."""
    import torch

    from paper_1901_07306_b200 import DetectorParams

    dp = DetectorParams(theta=64, design_n=2e5)
    _, _, p = params_block(dp)
    rng = np.random.default_rng(3)
    n = 100_003
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    seav, ldca = oracle.scan(p, hips, oips, threads=8)
    st = make_state(dp)
    h = torch.from_numpy(hips.view(np.int32)).cuda()
    o = torch.from_numpy(oips.view(np.int32)).cuda()
    for lo, hi in [(0, 1), (1, 7), (7, 4099), (4099, 50_000), (50_000, n)]:
        st.process_batch(h[lo:hi], o[lo:hi])  # device views at unaligned offsets
    assert st.seav.payload_bytes() == seav.tobytes()
    assert st.ldca.payload_bytes() == ldca.tobytes()


def test_reset_replay_and_merge(cuda):
    from paper_1901_07306_b200 import DetectorParams

    rng = np.random.default_rng(10)
    hips = rng.integers(0, 2**32, size=50_000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=50_000, dtype=np.uint64)
    dp = DetectorParams(theta=128, design_n=2e5)
    st = make_state(dp)
    st.process_batch(hips, oips)
    a, b = st.seav.payload_bytes(), st.ldca.payload_bytes()
    st.reset()
    assert st.window_id == 1 and st.seav.total_set_bits() == 0 and not st.ldca.data.any()
    st.process_batch(hips, oips)
    st.process_batch(hips, oips)  # idempotent OR
    assert st.seav.payload_bytes() == a and st.ldca.payload_bytes() == b
    shards = [make_state(dp) for _ in range(4)]
    for w in range(4):
        shards[w].process_batch(hips[w::4], oips[w::4])
    for s in shards[1:]:
        shards[0].seav.merge(s.seav)
        shards[0].ldca.merge(s.ldca)
    assert shards[0].seav.payload_bytes() == a and shards[0].ldca.payload_bytes() == b


PART_CASES = {
    # case: (geometry, expected variant: 2 = K1b b-axis partitions, 1 = K1p word ranges)
    "uniform": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    "skewed": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    "skewed_oip": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    "tiny_chunks": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    "k4096_hb0": (dict(theta=1024, r=12, k=4096, lr=8, lc=512), 2),
    "k16384_hb2": (dict(theta=1024, r=12, k=16384, lr=8, lc=512), 2),
    "k32768_hb3": (dict(theta=1024, r=16, k=32768, lr=8, lc=256), 2),
    "nonpow2": (dict(theta=512, r=8, k=1000, lr=7, lc=333), 1),
    "legacy_pow2": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 1),
    "legacy_skewed": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 1),
    # K1b consumer modes other than the default warp-specialised global-load drain
    "cons_inline": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    "cons_tma_skewed_oip": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    "cons_flags_skewed_oip": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    # K1b flush by threads (16-B stores) instead of TMA bulk stores
    "flush_threads_skewed_oip": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
    # K1b with ONE staging buffer (two producer barriers per tile) instead of two
    "single_buffer_skewed_oip": (dict(theta=1024, r=12, k=8192, lr=8, lc=1024), 2),
}


@pytest.mark.parametrize("case", list(PART_CASES))
def test_partitioned_scan_vs_oracle(cuda, oracle, case, monkeypatch):
    """The partitioned scans are bit-identical to the oracle: K1b (LDCA cut
    along b in shared memory, one 16-B entry per packet) and K1p (word-range
    partitions; forced with SSPD_PART_LEGACY for pow2 geometries), including
    the overflow fallbacks a skewed stream triggers -- one host (K1p: its
    8 cells take half of all updates) or one opposite IP (K1b: half of all
    packets go to ONE partition, overflowing its staging row and regions)."""
    from paper_1901_07306_b200 import DetectorParams
    from paper_1901_07306_b200._abi import lib

    geom, variant = PART_CASES[case]
    if case.startswith("legacy"):
        monkeypatch.setenv("SSPD_PART_LEGACY", "1")
    if case.startswith("cons_"):
        monkeypatch.setenv("SSPD_BPART_CONS", {"cons_inline": "0", "cons_flags_skewed_oip": "3"}.get(case, "2"))
    if case.startswith("flush_threads"):
        monkeypatch.setenv("SSPD_BPART_FLUSH_TMA", "0")
    if case.startswith("single_buffer"):
        monkeypatch.setenv("SSPD_BPART_DB", "0")
    dp = DetectorParams(design_n=1e6, **geom)
    _, _, p = params_block(dp)
    rng = np.random.default_rng(77)
    n = 3_000_017
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    if case in ("skewed", "legacy_skewed"):
        hips[: n // 2] = 0xC0A80001  # one host: its 8 cells take half of all updates
        hips[n // 2: n // 2 + 100_000] = 0x0A000001
    if case in ("skewed_oip", "cons_tma_skewed_oip", "flush_threads_skewed_oip", "cons_flags_skewed_oip",
                "single_buffer_skewed_oip"):
        oips[: n // 2] = 0x08080808  # one opposite IP: one b, so one K1b partition
        oips[n // 2: n // 2 + 100_000] = 0x01010101
        perm = rng.permutation(n)
        hips, oips = hips[perm], oips[perm]
    seav, ldca = oracle.scan(p, hips, oips, threads=8)
    st = make_state(dp)
    st.scan_mode = "partitioned"
    assert lib().sspd_scan_partitioned_variant(st.seav._params, 0) == variant
    if case == "tiny_chunks":
        st.partitioned_chunk = 1 << 14
    if case in ("skewed_oip", "cons_tma_skewed_oip", "flush_threads_skewed_oip", "cons_flags_skewed_oip",
                "single_buffer_skewed_oip", "k16384_hb2"):
        st.partitioned_chunk = 1 << 20  # several chunks: the warp-specialised drain overlaps production
    st.process_batch(hips[: n // 3], oips[: n // 3])
    st.process_batch(hips[n // 3:], oips[n // 3:])
    assert st.seav.payload_bytes() == seav.tobytes()
    assert st.ldca.payload_bytes() == ldca.tobytes()


@pytest.mark.parametrize("n", [1, 1000, 8192, 8193, 100_003, 1024 * 1024 + 1, 3_000_017])
def test_compaction_is_stable(cuda, n):
    """sspd_compact_reports (multi-segment and single-CTA forms) keeps order;
    above 1,024 segments the multi-segment form scans the segment counts."""
    import ctypes

    import torch

    from paper_1901_07306_b200._device import call, stream_ptr

    rng = np.random.default_rng(n)
    ip = torch.from_numpy(rng.integers(0, 2**31, n, dtype=np.int64).astype(np.int32)).cuda()
    z0 = torch.from_numpy(rng.integers(0, 8193, n, dtype=np.int64).astype(np.int32)).cuda()
    keep = torch.from_numpy((rng.random(n) < 0.37).astype(np.uint8)).cuda()
    want = keep.cpu().numpy().astype(bool)
    for multi in (True, False):
        ip_o = torch.zeros(n, dtype=torch.int32, device="cuda")
        z0_o = torch.zeros(n, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        need = ctypes.c_size_t(0)
        if multi:
            call("sspd_compact_reports", ip.data_ptr(), z0.data_ptr(), keep.data_ptr(), n, ip_o.data_ptr(),
                 z0_o.data_ptr(), cnt.data_ptr(), None, ctypes.byref(need), stream_ptr())
            scratch = torch.empty(need.value, dtype=torch.uint8, device="cuda")
            call("sspd_compact_reports", ip.data_ptr(), z0.data_ptr(), keep.data_ptr(), n, ip_o.data_ptr(),
                 z0_o.data_ptr(), cnt.data_ptr(), scratch.data_ptr(), ctypes.byref(need), stream_ptr())
        else:
            call("sspd_compact_reports", ip.data_ptr(), z0.data_ptr(), keep.data_ptr(), n, ip_o.data_ptr(),
                 z0_o.data_ptr(), cnt.data_ptr(), None, None, stream_ptr())
        m = int(cnt.item())
        assert m == int(want.sum())
        assert (ip_o[:m].cpu().numpy() == ip.cpu().numpy()[want]).all()
        assert (z0_o[:m].cpu().numpy() == z0.cpu().numpy()[want]).all()


@pytest.mark.slow
def test_config2_full_window_bit_exact_vs_oracle(cuda, oracle):
    """The bench workload itself (BASELINE configs[1]: 268,435,456 packets,
    SEAV r=12, LDCA 8 MiB) through the default scan (K1p) and the fused
    finalize: SEAV/LDCA bytes and the full report list (ips, estimates,
    saturation) equal the CPU oracle's, bit for bit."""
    import hashlib
    import math

    import torch

    from paper_1901_07306_b200 import DetectorParams
    from tools.workloads import CONFIG2, generate

    dp = DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=80.5e6)
    _, _, p = params_block(dp)
    hips, oips, supers = generate(CONFIG2, "torch", cuda)
    st = make_state(dp)
    st.process_batch(hips, oips)
    assert st.last_scan == "partitioned"
    reps = st.finalize_window()
    got = [(r.ip, r.estimated_cardinality, r.saturated) for r in reps]
    h = hips.cpu().numpy().view(np.uint32)
    o = oips.cpu().numpy().view(np.uint32)
    del hips, oips
    torch.cuda.empty_cache()
    seav, ldca = oracle.scan(p, h, o, threads=oracle.cpu_threads())
    sha = lambda b: hashlib.sha256(bytes(b)).hexdigest()  # noqa: E731
    assert sha(st.seav.payload_bytes()) == sha(seav.tobytes())
    assert sha(st.ldca.payload_bytes()) == sha(ldca.tobytes())
    ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
    z0 = oracle.filter_z0(p, ldca, ips)
    k = dp.k
    want = []
    for ip, z in zip(ips.tolist(), z0.tolist()):
        est, sat = (k * math.log(k), True) if z == 0 else (-k * math.log(z / k), False)
        if sat or est >= dp.beta * dp.theta:
            want.append((int(ip), est, sat))
    assert got == want
    assert set(supers.tolist()) <= {r[0] for r in got}


def test_config5_geometry_host_stream_windows_vs_oracle(cuda, oracle):
    """Config-5 geometry (LDCA 64 MiB: LR=8, LC=8192, k=8192 -- too big for
    shared memory, so the L2-red scan K1 runs; SEAV r=16) streamed from
    pinned host memory in 2^22-pair chunks over two windows with a reset
    between: each window's sketches and report list equal the oracle's."""
    import math

    import torch

    from paper_1901_07306_b200 import DetectorParams

    dp = DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=8192, design_n=5e7)
    _, _, p = params_block(dp)
    st = make_state(dp)
    rng = np.random.default_rng(55)
    for window in range(2):
        n = (1 << 23) + 12345
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        heavy = rng.integers(0, 2**32, size=16, dtype=np.uint64).astype(np.uint32)
        for i, h in enumerate(heavy):
            hips[i * 20_000:(i + 1) * 20_000 - i * 700] = h
        h_t = torch.from_numpy(hips.view(np.int32)).pin_memory()
        o_t = torch.from_numpy(oips.view(np.int32)).pin_memory()
        assert st.process_host_stream(h_t, o_t, chunk_pairs=1 << 22) == 8 * n
        reps = st.finalize_window()
        seav, ldca = oracle.scan(p, hips, oips, threads=oracle.cpu_threads())
        assert st.seav.payload_bytes() == seav.tobytes()
        assert st.ldca.payload_bytes() == ldca.tobytes()
        ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
        z0 = oracle.filter_z0(p, ldca, ips)
        k = dp.k
        want = [int(ip) for ip, z in zip(ips.tolist(), z0.tolist())
                if z == 0 or -k * math.log(z / k) >= dp.beta * dp.theta]
        assert [r.ip for r in reps] == want
        assert set(heavy.tolist()) <= set(want)
        assert all(r.window_id == window for r in list(reps)[:3])
        st.reset()


def test_finalize_window_async_equals_sync(cuda):
    """Pipelined windows: finalize_window_async (device snapshot, resolved
    later, two snapshots alternating) gives the same lists as
    finalize_window, including a capacity re-run resolved after later
    windows were already scanned into the live sketches."""
    from paper_1901_07306_b200 import DetectorParams

    dp = DetectorParams(theta=256, r=8, k=4096, lr=4, lc=256, design_n=1e6)
    a, b = make_state(dp), make_state(dp)
    a.seav._cand_cap = b.seav._cand_cap = 8  # force the re-run path
    rng = np.random.default_rng(77)
    pend, want = [], []
    for w in range(5):
        n = 200_000
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        for i in range(6 + w):
            hips[i * 4000:(i + 1) * 4000] = rng.integers(0, 2**32, dtype=np.uint64)
        for st in (a, b):
            st.process_batch(hips, oips)
        pend.append(a.finalize_window_async())
        want.append([(r.ip, r.estimated_cardinality, r.saturated, r.window_id) for r in b.finalize_window()])
        a.reset()
        b.reset()
    got = [[(r.ip, r.estimated_cardinality, r.saturated, r.window_id) for r in p] for p in pend]
    assert got == want and all(len(x) >= 6 for x in want)


@pytest.mark.parametrize("skewed", [False, True])
def test_finalize_bucket_sort_vs_oracle(cuda, oracle, skewed):
    """The fused finalize orders candidates with a bucket sort (buckets of
    the top IP bits, <= 64 keys per warp); a bucket above that (here: 150
    super points inside one /16) raises the kernel's flag and the finalize is
    re-run with the radix sort, learned for the sketch.  Both give the
    oracle's report list."""
    import math

    from paper_1901_07306_b200 import DetectorParams

    dp = DetectorParams(theta=256, r=8, k=4096, lr=4, lc=256, design_n=4e5)
    _, _, p = params_block(dp)
    rng = np.random.default_rng(31 + skewed)
    n = 1_200_000
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    nheavy = 150
    if skewed:
        heavy = (0x0A0B0000 + rng.choice(1 << 16, size=nheavy, replace=False)).astype(np.uint64)
    else:
        heavy = rng.integers(0, 2**32, size=nheavy, dtype=np.uint64)
    per = 1200
    hips[: nheavy * per] = np.repeat(heavy, per)
    perm = rng.permutation(n)
    hips, oips = hips[perm], oips[perm]
    st = make_state(dp)
    st.process_batch(hips, oips)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        reports = st.finalize_window()
    seav, ldca = oracle.scan(p, hips, oips, threads=8)
    ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
    z0 = oracle.filter_z0(p, ldca, ips)
    k = dp.k
    want = [int(ip) for ip, z in zip(ips, z0) if z == 0 or -k * math.log(z / k) >= dp.beta * dp.theta]
    got = [r.ip for r in reports]
    assert got == want
    assert st.seav._radix_sort == skewed
    assert len(set(heavy.tolist()) & set(got)) > nheavy // 2


@pytest.mark.parametrize("lr,lc,k", [(8, 1024, 8192), (4, 256, 4096), (5, 64, 4128), (3, 128, 8200)])
def test_finalize_partly_saturated_ldca_vs_oracle(cuda, oracle, lr, lc, k):
    """The filter's cell summary (cell_zeros_kernel) skips full LDCA cells:
    an LDCA whose cells are a mix of full, nearly full and half-set ones
    drives every branch -- all cells full (z0 = 0 without a read), one cell
    not full (z0 from the summary), several (AND over the non-full cells
    only) -- across the LR = 8 / 16-byte / word / byte filter paths.  The
    report list equals the oracle's on the same bytes."""
    import math

    from paper_1901_07306_b200 import DetectorParams

    dp = DetectorParams(theta=256, r=8, k=k, lr=lr, lc=lc, design_n=4e5)
    _, _, p = params_block(dp)
    rng = np.random.default_rng(lr * 7 + k)
    n = 400_000
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    heavy = rng.integers(0, 2**32, size=300, dtype=np.uint64)
    hips[: 300 * 600] = np.repeat(heavy, 600)
    st = make_state(dp)
    st.process_batch(hips, oips)
    cb = k // 8
    cells = lr * lc
    kind = rng.choice(3, size=cells, p=[0.75, 0.15, 0.10])
    ldca = np.empty((cells, cb), dtype=np.uint8)
    ldca[kind == 0] = 0xFF
    dense = np.packbits(rng.random(((kind == 1).sum(), cb * 8)) < 0.995, axis=1)
    ldca[kind == 1] = dense
    ldca[kind == 2] = rng.integers(0, 256, size=((kind == 2).sum(), cb), dtype=np.uint8)
    st.ldca.load_payload(ldca.tobytes())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        reports = st.finalize_window()
    seav = np.frombuffer(st.seav.payload_bytes(), dtype=np.uint8)
    ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
    z0 = oracle.filter_z0(p, ldca.reshape(-1), ips)
    want = [(int(ip), int(z)) for ip, z in zip(ips.tolist(), z0.tolist())
            if z == 0 or -k * math.log(z / k) >= dp.beta * dp.theta]
    got = [(r.ip, r.estimated_cardinality) for r in reports]
    est = {z: (k * math.log(k) if z == 0 else -k * math.log(z / k)) for _, z in want}
    assert [ip for ip, _ in got] == [ip for ip, _ in want]
    assert [e for _, e in got] == [est[z] for _, z in want]
    zs = [z for _, z in want]
    assert zs.count(0) > 10 and sum(1 for z in zs if z) > 10  # both the shortcut and the read paths ran


@pytest.mark.parametrize("n", [1, 2, 5, 1023, 4097, 100_003, 1_048_579])
def test_candidate_radix_sort_stable(cuda, n):
    """sspd_sort_candidates (csrc/radix.cu, no CUB): keys ascending, values
    carried along, equal keys in their input order (stable), clustered and
    duplicated keys included."""
    import ctypes

    import torch

    from paper_1901_07306_b200._device import call, stream_ptr

    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    keys[: n // 3] = (keys[: n // 3] & 0xFF) | 0xC0A80000  # one /16: deep equal prefixes
    keys[n // 2: n // 2 + n // 5] = keys[n // 2]           # runs of duplicates
    vals = np.arange(n, dtype=np.uint32)
    k = torch.from_numpy(keys.view(np.int32)).cuda()
    v = torch.from_numpy(vals.view(np.int32)).cuda()
    need = ctypes.c_size_t(0)
    call("sspd_sort_candidates", k.data_ptr(), v.data_ptr(), n, None, ctypes.byref(need), stream_ptr())
    scratch = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    call("sspd_sort_candidates", k.data_ptr(), v.data_ptr(), n, scratch.data_ptr(), ctypes.byref(need), stream_ptr())
    order = np.argsort(keys, kind="stable")
    assert (k.cpu().numpy().view(np.uint32) == keys[order]).all()
    assert (v.cpu().numpy().view(np.uint32) == vals[order]).all()
