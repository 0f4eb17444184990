"""Sliding-window pool kernels and the distributed merge on the GPU vs the
reference's golden vectors."""

import hashlib
import warnings

import numpy as np
import pytest

from conftest import params_from

pytestmark = pytest.mark.gpu


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def rep_list(reps):
    return [[r.ip, repr(r.estimated_cardinality), r.saturated, r.window_id, r.source] for r in reps]


def test_sliding_golden_steps(cuda, golden, garr):
    from paper_1901_07306_b200 import SlidingDetector

    g = golden["sliding"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(params_from(g["params"]), window_slices=g["w"])
    hips, oips, slices = garr[g["hips"]], garr[g["oips"]], garr[g["slices"]]
    for step in g["steps"]:
        sel = slices == step["slice"]
        det.observe_batch(hips[sel], oips[sel])
        assert det.now == step["now"]
        assert sha(det.pool.ts.tobytes()) == step["pool_sha"], step["slice"]
        if step["seav_view_sha"]:
            assert sha(det.materialize_seav().payload_bytes()) == step["seav_view_sha"]
            assert sha(det.materialize_ldca().tobytes()) == step["ldca_view_sha"]
        if step["reports"] is not None:
            assert rep_list(det.detect()) == step["reports"], step["slice"]
        det.advance_slice()


def test_wraparound_sweep_golden(cuda, golden):
    from paper_1901_07306_b200 import TimestampPool

    pool = TimestampPool(64, window_slices=100)
    assert pool.ts.dtype == np.uint8
    rng = np.random.default_rng(9)
    snaps = iter(golden["wrap"]["snaps"])
    for now in range(1, 1200):
        pool.advance_slice()
        if now % 7 == 0 and now <= 900:
            pool.touch_batch(rng.integers(0, 64, size=5))
        if now % 50 == 0:
            snap = next(snaps)
            assert pool.sweep_count == snap[1]
            assert sha(pool.ts.tobytes()) == snap[2]
            assert pool.active().astype(np.uint8).tolist() == snap[3]


def test_pool_scalar_api(cuda):
    from paper_1901_07306_b200 import ConfigError, TimestampPool

    pool = TimestampPool(4, window_slices=10)
    for _ in range(6):
        pool.advance_slice()
    pool.touch(1, now=6)
    pool.touch(1, now=3)  # older stamp loses
    for _ in range(9):
        pool.advance_slice()
    assert pool.is_active(1)
    pool.advance_slice()
    assert not pool.is_active(1)
    with pytest.raises(ConfigError):
        pool.touch(0, now=pool.now + 1)
    with pytest.raises(ConfigError):
        pool.touch(4)


def test_merge_pools_golden(cuda, golden, garr):
    from paper_1901_07306_b200 import TimestampPool, merge_timestamp_pools

    g = golden["merge_pools"]
    pools = []
    for name in g["inputs"]:
        p = TimestampPool(len(garr[name]), window_slices=g["w"])
        p.now = g["now"]
        p.ts = garr[name]
        pools.append(p)
    merged = merge_timestamp_pools(pools)
    assert (merged.ts == garr[g["merged"]]).all()


def test_sliding_equals_discrete(cuda):
    """One slide covering the whole stream == the discrete window, bit-exact
    (test_acceptance.py:190-218 criterion 8)."""
    from paper_1901_07306_b200 import DetectorParams, DetectorState, SlidingDetector

    params = DetectorParams(theta=1024, k=8192, lr=2, lc=512, design_n=3e4)
    w = 300
    rng = np.random.default_rng(800)
    n = 300_000
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    hips[:3000] = 0x0A0B0C0D
    hips[3000:4000] = 0x0A0B0C0E
    slices = rng.integers(0, w, size=n)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        disc = DetectorState.create(params)
        det = SlidingDetector(params, window_slices=w)
    disc.process_batch(hips, oips)
    for s in range(w):
        sel = slices == s
        det.observe_batch(hips[sel], oips[sel])
        if s < w - 1:
            det.advance_slice()
    assert det.materialize_seav().payload_bytes() == disc.seav.payload_bytes()
    assert (det.materialize_ldca() == disc.ldca.data).all()
    a = [(r.ip, r.estimated_cardinality, r.saturated) for r in det.detect()]
    b = [(r.ip, r.estimated_cardinality, r.saturated) for r in disc.finalize_window()]
    assert a == b and len(b) >= 1


def test_route_golden(cuda, golden, garr):
    from paper_1901_07306_b200 import SeedFamily, route_pairs

    g = golden["route"]
    for n_wp in (1, 3, 7, 8, 16):
        assert (route_pairs(garr[g["hips"]], garr[g["oips"]], n_wp, "hash", SeedFamily())
                == garr[g[f"hash_{n_wp}"]]).all()
    rr = route_pairs(garr[g["hips"]], garr[g["oips"]], 3, "round-robin", SeedFamily())
    assert (rr == np.arange(len(rr)) % 3).all()


def test_frames_and_merge_golden(cuda, golden, garr):
    from paper_1901_07306_b200 import DetectorState, merge_frames, parse_frame, serialize, simulate_window

    g = golden["frames"]
    params = params_from(g["params"])
    states = []
    for wp in range(3):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            st = DetectorState.create(params)
        st.process_batch(garr[f"frames/h{wp}"], garr[f"frames/o{wp}"])
        states.append(st)
    blobs = [serialize(s.seav, 5) for s in states] + [serialize(s.ldca, 5) for s in states]
    assert [sha(b) for b in blobs] == g["frame_sha"]
    mseav, mldca = merge_frames([parse_frame(b) for b in blobs])
    assert sha(mseav.payload_bytes()) == g["merged_seav_sha"]
    assert sha(mldca.payload_bytes()) == g["merged_ldca_sha"]
    hips = np.concatenate([garr[f"frames/h{i}"] for i in range(3)])
    oips = np.concatenate([garr[f"frames/o{i}"] for i in range(3)])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sim = simulate_window(params, 3, hips, oips, 4)
    assert rep_list(sim.reports) == g["sim_reports"]
    assert sha(sim.global_seav.payload_bytes()) == g["sim_seav_sha"]
    assert sha(sim.global_ldca.payload_bytes()) == g["sim_ldca_sha"]


@pytest.mark.parametrize("route", ["hash", "round-robin"])
@pytest.mark.parametrize("n_wp", [1, 4, 16])
def test_partition_invariance(cuda, route, n_wp):
    from paper_1901_07306_b200 import DetectorParams, simulate_window

    params = DetectorParams(theta=1024, k=4096, lr=2, lc=64, design_n=4e3)
    rng = np.random.default_rng(6)
    hips = rng.integers(0, 2**32, size=12_000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=12_000, dtype=np.uint64)
    hips[:3000] = 0x11223344
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = simulate_window(params, 0, hips, oips, 1)
        res = simulate_window(params, 0, hips, oips, n_wp, route=route, buffer_pairs=37 if n_wp == 4 else 65536)
    assert res.global_seav.payload_bytes() == ref.global_seav.payload_bytes()
    assert res.global_ldca.payload_bytes() == ref.global_ldca.payload_bytes()
    assert res.reports == ref.reports and len(res.reports) >= 1


@pytest.mark.parametrize("off", [0, 1, 2, 3, 7])
def test_sliding_observe_device_slices_vs_oracle(cuda, oracle, off):
    """K2 fast path (u16 stamps, pow2 geometry) on device slices at every
    16-byte misalignment: pool bytes equal the oracle's, slide by slide."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=1024, k=8192, lr=8, lc=256, design_n=1e5)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(params, window_slices=300)
    rng = np.random.default_rng(100 + off)
    n = 60_013
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    hips[:5000] = 0x0A000001
    h = torch.from_numpy(hips.view(np.int32)).cuda()
    o = torch.from_numpy(oips.view(np.int32)).cuda()
    pool = det.pool.ts.copy()
    cuts = [off, off + 1, off + 4098, off + 20_001, n - 3, n]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        det.observe_batch(h[lo:hi], o[lo:hi])
        oracle.observe(det._params, hips[lo:hi], oips[lo:hi], pool, det.pool._wrapped_now())
        assert (det.pool.ts == pool).all(), (lo, hi)
        det.advance_slice()


@pytest.mark.parametrize("r", [4, 8, 16])
def test_views_fast_paths_vs_oracle(cuda, oracle, r):
    """K4 fast paths (4 SEAV registers / 4 LDCA bytes per thread, u16
    stamps) on a random pool whose ages straddle the window edge, at every
    wrapped `now`, vs the oracle's materialize_* (sliding.py:191-220)."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=1024, r=r, k=4096, lr=4, lc=64, design_n=1e5)
    w = 300
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(params, window_slices=w)
    rng = np.random.default_rng(r)
    n = det.pool.n_slots
    for now in (0, 299, 300, 65535, 40000):
        edge = rng.integers(w - 3, w + 3, size=n)          # around the window edge
        ages = np.where(rng.random(n) < 0.5, rng.integers(0, 2 * w + 2, size=n), edge)
        pool = ((now - ages) & 0xFFFF).astype(np.uint16)
        det.pool.ts = pool
        det.pool.now = now
        got_s = det.materialize_seav().payload_bytes()
        got_l = det.materialize_ldca().tobytes()
        want_s = oracle.materialize_seav(det._params, pool, now & 0xFFFF, w)
        want_l = oracle.materialize_ldca(det._params, pool, now & 0xFFFF, w)
        assert got_s == want_s.tobytes(), now
        assert got_l == want_l.tobytes(), now
        torch.cuda.synchronize()


def test_detect_async_equals_detect(cuda):
    """detect_async (views on the caller's stream, K5/K6 on a side stream,
    two alternating view sets) returns exactly detect()'s lists, slide by
    slide, while later slices keep rewriting the pool."""
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=256, r=8, k=4096, lr=4, lc=256, design_n=2e5)
    w = 20
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = SlidingDetector(params, window_slices=w)
        b = SlidingDetector(params, window_slices=w)
    rng = np.random.default_rng(2024)
    heavy = rng.integers(0, 2**32, size=6, dtype=np.uint64)
    pending, sync = [], []
    for s in range(60):
        n = int(rng.integers(1_000, 40_000))
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        hips[: n // 4] = heavy[(s // 10) % len(heavy)]  # heavy hosts come and go
        a.observe_batch(hips, oips)
        b.observe_batch(hips, oips)
        pending.append(a.detect_async())
        sync.append(rep_list(b.detect()))
        a.advance_slice()
        b.advance_slice()
    got = [rep_list(p) for p in pending]
    assert got == sync
    assert sum(len(x) for x in sync) > 0


@pytest.mark.slow
def test_config4_scaled_trace_vs_oracle(cuda, oracle):
    """Config 4 at 1/8 scale (2^26 timestamped packets over ~298 one-second
    slices, w = 300, r = 16, LDCA 8 MiB), driven exactly like the bench
    (observe per slice, pipelined detect_async at EVERY slide): the pool
    bytes at the end and the report lists at sampled slides equal the
    oracle's (observe -> materialize -> restore -> filter), bit for bit."""
    import hashlib
    import math

    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from tools.workloads import CONFIG4, CONFIG4_TIMING, TimingSpec, generate, scaled

    spec = scaled(CONFIG4, 8)
    timing = TimingSpec(rate_pps=spec.n_packets / (CONFIG4.n_packets / CONFIG4_TIMING.rate_pps))
    hips, oips, supers, ts = generate(spec, "torch", cuda, timing=timing)
    slices = (ts // 1000).cpu().numpy()
    n_sl = int(slices[-1]) + 1
    bounds = np.searchsorted(slices, np.arange(n_sl + 1))
    dp = DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.7e7)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(dp, window_slices=300)
    p = det._params
    h_np = hips.cpu().numpy().view(np.uint32)
    o_np = oips.cpu().numpy().view(np.uint32)
    pool = det.pool.ts.copy()
    check = {n_sl // 4, n_sl // 2, n_sl - 1}
    pending, want = {}, {}
    for s in range(n_sl):
        lo, hi = int(bounds[s]), int(bounds[s + 1])
        if hi > lo:
            det.observe_batch(hips[lo:hi], oips[lo:hi])
            oracle.observe(p, h_np[lo:hi], o_np[lo:hi], pool, det.pool._wrapped_now())
        pending[s] = det.detect_async()
        if s in check:
            now, w = det.pool._wrapped_now(), det.pool.window_slices
            seav = oracle.materialize_seav(p, pool, now, w)
            ldca = oracle.materialize_ldca(p, pool, now, w)
            ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
            z0 = oracle.filter_z0(p, ldca, ips)
            k = dp.k
            rows = []
            for ip, z in zip(ips.tolist(), z0.tolist()):
                est, sat = (k * math.log(k), True) if z == 0 else (-k * math.log(z / k), False)
                if sat or est >= dp.beta * dp.theta:
                    rows.append((int(ip), est, sat))
            want[s] = rows
        det.advance_slice()
    torch.cuda.synchronize()
    sha = lambda b: hashlib.sha256(bytes(b)).hexdigest()  # noqa: E731
    assert sha(det.pool.ts.tobytes()) == sha(pool.tobytes())
    for s, rows in want.items():
        got = [(r.ip, r.estimated_cardinality, r.saturated) for r in pending[s]]
        assert got == rows, s
        assert all(r.window_id == s for r in list(pending[s])[:3])
    assert sum(len(pending[s]) for s in pending) > 0


def test_incremental_seav_view_equals_full_materialization(cuda):
    """The incrementally maintained SEAV view (stamp-time set + per-slice
    expiry log) equals a full K4 materialization of the pool at every
    slide: through expiries (400 slides > w = 150), hosts coming and going,
    re-touched slots, empty slices, a pool write that bypasses the detector
    (the view then degrades to full materialization, still exact), and a
    reset; detect() equals a detector without the incremental view."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=512, r=8, k=4096, lr=2, lc=64, design_n=1e5)
    w = 150
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = SlidingDetector(params, window_slices=w)
        b = SlidingDetector(params, window_slices=w)
    b.incremental_seav = False
    assert a.pool.ts_bytes == 2
    rng = np.random.default_rng(31)
    heavy = rng.integers(0, 2**32, size=5, dtype=np.uint64)

    def step(s):
        n = 0 if s % 37 == 5 else int(rng.integers(500, 12_000))
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        if n:
            hips[: n // 3] = heavy[(s // 60) % len(heavy)]
            oips[: n // 6] = oips[0]  # re-touched slots within the slice
        for det in (a, b):
            det.observe_batch(hips, oips)
        inc = a._seav_view().device_buffer()
        full = a.materialize_seav().device_buffer()
        assert torch.equal(inc[: full.numel()], full), s
        if s % 25 == 0:
            assert rep_list(a.detect()) == rep_list(b.detect()), s
        for det in (a, b):
            det.advance_slice()

    for s in range(400):
        step(s)
    assert a._iv() is not None and int(a._iv()["meta"][1].item()) == 0  # stayed incremental
    a.pool.touch_batch(np.arange(0, 64, 3))  # bypasses the detector
    b.pool.touch_batch(np.arange(0, 64, 3))
    for s in range(400, 420):
        step(s)
    assert int(a._iv()["meta"][1].item()) == 1  # invalidated -> full materialization
    for det in (a, b):
        det.reset()
    assert int(a._iv()["meta"][1].item()) == 0
    for s in range(420, 600):
        step(s)


def test_deferred_ldca_stamps_equal_direct_stamps(cuda):
    """Deferred LDCA stamps (dirty bitmap + sspd_ldca_fold, fused with the
    LDCA view at detect) leave exactly the pool the direct u16 stores leave,
    through every way the pool is read or written: several observes per
    slice, reads mid-slice (ts, ages, is_active, materialize_ldca), detect
    and detect_async, touch / touch_batch / ts assignment around the
    detector, a forced anti-alias sweep, pool merge, and reset."""
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector, merge_timestamp_pools

    params = DetectorParams(theta=256, r=8, k=4096, lr=4, lc=256, design_n=2e5)
    w = 130  # u16 stamps (2w + 2 > 255); 170 slices so slots expire
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = SlidingDetector(params, window_slices=w)
        b = SlidingDetector(params, window_slices=w)
    b.defer_ldca_stamps = False
    assert a.pool.ts_bytes == 2 and a._deferred() is not None and b._deferred() is None
    rng = np.random.default_rng(99)
    heavy = rng.integers(0, 2**32, size=4, dtype=np.uint64)
    base = a.layout.ldca_base
    pend = []
    for s in range(170):
        for _ in range(1 + s % 3):  # several batches per slice
            n = int(rng.integers(1, 20_000))
            hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
            oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
            hips[: n // 3] = heavy[(s // 9) % len(heavy)]
            a.observe_batch(hips, oips)
            b.observe_batch(hips, oips)
        if s % 7 == 3:  # reads mid-slice, then more packets in the same slice
            assert np.array_equal(a.pool.ts, b.pool.ts), s
            slot = base + int(rng.integers(0, a.layout.total - base))
            assert a.pool.is_active(slot) == b.pool.is_active(slot)
            assert np.array_equal(a.materialize_ldca(), b.materialize_ldca()), s
            hips = rng.integers(0, 2**32, size=5000, dtype=np.uint64)
            oips = rng.integers(0, 2**32, size=5000, dtype=np.uint64)
            a.observe_batch(hips, oips)
            b.observe_batch(hips, oips)
        if s % 5 == 1 and s % 20 == 1:
            assert rep_list(a.detect()) == rep_list(b.detect()), s
        else:
            pend.append((a.detect_async(), b.detect_async()))
        if s == 20:  # writes around the detector
            idx = np.arange(base, base + 4096, 7)
            for det in (a, b):
                det.pool.touch_batch(idx)
                det.pool.touch(base + 5)
        if s == 30:
            ts = a.pool.ts.copy()
            ts[base: base + 1000] = (a.pool.now - 3) & a.pool._mask
            a.observe_batch(heavy, heavy)  # pending deferred stamps, then replaced
            a.pool.ts = ts
            b.observe_batch(heavy, heavy)
            b.pool.ts = ts
        if s == 150:  # force the anti-alias sweep at the next advance
            for det in (a, b):
                det.pool._since_sweep = det.pool._sweep_period - 1
        a.advance_slice()
        b.advance_slice()
        assert np.array_equal(a.pool.ages(), b.pool.ages()), s
    assert a.pool.sweep_count == b.pool.sweep_count == 1
    for x, y in pend:
        assert rep_list(x) == rep_list(y)
    assert sum(len(x) for x, _ in pend) > 0
    # merge: the deferred pool's pending stamps take part
    hips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
    a.observe_batch(hips, hips)
    b.observe_batch(hips, hips)
    ma = merge_timestamp_pools([a.pool, b.pool])
    assert np.array_equal(ma.ts, b.pool.ts) and ma._deferred is None
    a.observe_batch(hips, hips[::-1].copy())
    a.reset()
    b.reset()
    assert np.array_equal(a.pool.ts, b.pool.ts)
    assert not a.pool._deferred.pending and int(a.pool._deferred.current.count_nonzero()) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("async_detect", [False, True])
@pytest.mark.parametrize("geom", [(4096, 4, 256), (64, 3, 37), (4096, 4, 256, "misaligned"),
                                  (4096, 8, 256, "partitioned"), (4096, 8, 256, "partitioned_unfused")],
                         ids=["ldca16B", "ldca_pad8_nonpow2", "misaligned_inputs", "k1b_dirty_bitmaps",
                              "k1b_dirty_bitmaps_two_launches"])
def test_ldca_ring_window_or_equals_direct_stamps(cuda, async_detect, geom, monkeypatch):
    """Ring mode of the deferred LDCA stamps (the LDCA view as a two-stack
    sliding-window OR of per-slice bitmaps, stamps folded lazily) against
    direct u16 stores over 2.7 windows from a pristine pool: detect at every
    slide across two block ends (suffix passes) with expiring slots, pool
    reads mid-block, a write around the detector (restart: stamps-based view
    for one block, then the ring again), and reset.  `ldca_pad8`: 888 LDCA
    bytes, so the ring pads each slice's bitmap to 896 B (the fold must step
    by the padded stride, not the LDCA size) and lc = 37 (the generic u16
    scan must fill the dirty bitmaps).  `misaligned_inputs`: device hips /
    oips at different 16-B offsets (no fast path either).
    `k1b_dirty_bitmaps`: every slice in ONE launch of the partitioned scan
    K1b (LDCA half into the slice's bitmap, SEAV stamps + view + log from
    its sampled-packet queue, sspd_scan_sliding_partitioned);
    `_two_launches`: K1b for the LDCA half, K2 for the SEAV half."""
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    k, lr, lc = geom[:3]
    misaligned = len(geom) > 3 and geom[3] == "misaligned"
    if len(geom) > 3 and geom[3].startswith("partitioned"):  # the LDCA half of every slice through K1b
        monkeypatch.setenv("SSPD_SLIDE_PARTITIONED", "1")
        monkeypatch.setenv("SSPD_SLIDE_FUSED", "0" if geom[3].endswith("unfused") else "1")
    params = DetectorParams(theta=256, r=8, k=k, lr=lr, lc=lc, design_n=2e5)
    w = 129
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = SlidingDetector(params, window_slices=w)
        b = SlidingDetector(params, window_slices=w)
    b.defer_ldca_stamps = False
    assert a._deferred().ring is not None and a._deferred().valid()
    assert (a._deferred().stride == a._params.ldca_bytes) == (a._params.ldca_bytes % 16 == 0)
    rng = np.random.default_rng(7)
    heavy = rng.integers(0, 2**32, size=3, dtype=np.uint64)
    base = a.layout.ldca_base
    pend = []
    modes = []
    for s in range(350):
        n = int(rng.integers(0, 3000)) if s % 11 else 0  # some empty slices
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        if s < 40 or 150 <= s < 175:  # bursts that expire inside the run
            hips[: n // 2] = heavy[s % 3]
        if misaligned and n:
            hd = torch.from_numpy(hips.astype(np.uint32).view(np.int32)).cuda()
            od = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
            od[1:] = torch.from_numpy(oips.astype(np.uint32).view(np.int32)).cuda()
            a.observe_batch(hd, od[1:])
        elif s % 4 == 1 and n > 1:  # two batches in one slice: the second ORs into a used bitmap
            a.observe_batch(hips[: n // 3], oips[: n // 3])
            a.observe_batch(hips[n // 3:], oips[n // 3:])
        else:
            a.observe_batch(hips, oips)
        b.observe_batch(hips, oips)
        if s == 200:  # a write around the detector: restart, stamps-based view for one block
            for det in (a, b):
                det.pool.touch_batch(np.arange(base, base + 2048, 5))
        if s % 37 == 5:
            assert np.array_equal(a.pool.ts, b.pool.ts), s
            assert np.array_equal(a.materialize_ldca(), b.materialize_ldca()), s
        modes.append(a._ring().valid())
        if async_detect:
            pend.append((s, a.detect_async(), b.detect_async()))
        else:
            assert rep_list(a.detect()) == rep_list(b.detect()), s
        a.advance_slice()
        b.advance_slice()
    for s, x, y in pend:
        assert rep_list(x) == rep_list(y), s
    assert np.array_equal(a.pool.ts, b.pool.ts)
    d = a._ring()
    assert d.prev_ok and d.blk0 == 200 + w  # block ends after 128, 257 (pristine), 328 (restart at 200)
    assert all(modes[:200]) and not any(modes[200:200 + w]) and all(modes[200 + w:])
    a.reset()
    b.reset()
    assert a._ring().valid() and np.array_equal(a.pool.ts, b.pool.ts)


@pytest.mark.gpu
def test_detect_async_lists_outlive_their_view_set(cuda):
    """detect_async replays each view set's finalize graph into the same
    device buffers: a list still held when its set is reused -- as the
    PendingReports or only as the resolved ReportList -- keeps its own copy
    of the arrays; dropped lists cost no copy.  Every held list equals the
    synchronous detect() of a twin detector."""
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=256, r=16, k=4096, lr=4, lc=256, design_n=2e5)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = SlidingDetector(params, window_slices=16)
        b = SlidingDetector(params, window_slices=16)
    rng = np.random.default_rng(5)
    heavy = rng.integers(0, 2**32, size=5, dtype=np.uint64)
    held, want = {}, {}
    for s in range(30):
        n = int(rng.integers(5_000, 40_000))
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        hips[: n // 3] = heavy[s % 5]
        a.observe_batch(hips, oips)
        b.observe_batch(hips, oips)
        p = a.detect_async()
        ref = rep_list(b.detect())
        if s % 3 == 0:
            held[s] = p  # the pending handle
        elif s % 3 == 1:
            held[s] = p.result()  # only the resolved list (its arrays not fetched yet)
        want[s] = ref
        a.advance_slice()
        b.advance_slice()
    assert {s: rep_list(x) for s, x in held.items()} == {s: want[s] for s in held}
    assert sum(len(want[s]) for s in held) > 0


@pytest.mark.gpu
def test_detect_async_graph_cache_varying_beta(cuda):
    """detect_async with beta changing from slide to slide: each view set
    keeps ONE finalize graph (the keep table is a device input refreshed on
    the stream, not part of the graph key), and every list equals the
    synchronous detect(beta) of a twin detector."""
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=256, r=12, k=4096, lr=4, lc=256, design_n=2e5)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = SlidingDetector(params, window_slices=8)
        b = SlidingDetector(params, window_slices=8)
    rng = np.random.default_rng(11)
    heavy = rng.integers(0, 2**32, size=6, dtype=np.uint64)
    betas = [0.8, 0.3, 1.5, 0.8, 0.05]
    pend = []
    for s in range(25):
        n = int(rng.integers(5_000, 30_000))
        hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
        hips[: n // 2] = heavy[rng.integers(0, 6, size=n // 2)]
        a.observe_batch(hips, oips)
        b.observe_batch(hips, oips)
        beta = betas[s % len(betas)]
        pend.append((s, a.detect_async(beta), rep_list(b.detect(beta))))
        a.advance_slice()
        b.advance_slice()
    for s, x, want in pend:
        assert rep_list(x) == want, s
    assert sum(len(w) for _, _, w in pend) > 0
    for vset in a._async["sets"]:
        # one graph (the newest), its keep table and its reused completion event
        assert vset is not None and set(vset[3]) <= {"graph", "keep", "event"}
