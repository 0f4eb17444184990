"""Drop-in behaviour: the reference test-suite's behavioural checks
 re-stated against the B200 package.  Each test names the
reference test it mirrors."""

import math
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fresh(**kw):
    from paper_1901_07306_b200 import DetectorParams, DetectorState

    kw.setdefault("design_n", 2e5)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return DetectorState.create(DetectorParams(**kw))


def heavy_host(state, hip, n_oips, rng):
    oips = np.unique(rng.integers(0, 2**32, size=n_oips + 64, dtype=np.uint64))[:n_oips]
    state.process_batch(np.full(n_oips, hip, dtype=np.uint64), oips)


# --- short sketch (test_short_sketch.py) ----------------------------------------
def test_rp_routing_separates_arrays(cuda):  # :257-263
    from paper_1901_07306_b200 import SeavSketch, SeedFamily, make_config

    sk = SeavSketch(make_config(theta=8), SeedFamily())
    sk.update(0x10, 5)
    sk.update(0x13, 5)
    for row in sk.rows:
        assert {int(rp) for rp in np.nonzero(row)[0]} == {0, 3}


def test_scalar_update_matches_batch_and_is_idempotent(cuda):  # :249-291
    from paper_1901_07306_b200 import SeavSketch, SeedFamily, make_config

    cfg = make_config(theta=64)
    rng = np.random.default_rng(12)
    hips = rng.integers(0, 2**32, size=300, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=300, dtype=np.uint64)
    a, b = SeavSketch(cfg, SeedFamily()), SeavSketch(cfg, SeedFamily())
    a.update_batch(hips, oips)
    for h, o in zip(hips.tolist(), oips.tolist()):
        b.update(h, o)
        b.update(h, o)
    assert a.payload_bytes() == b.payload_bytes()
    assert a.se_at(int(hips[0]) & 15, 0, cfg.index_of(0, int(hips[0]) >> 4)).bits == int(
        a.rows[0][int(hips[0]) & 15, cfg.index_of(0, int(hips[0]) >> 4)])


def test_host_snapshots_read_only_and_row_assignment_uploads(cuda):
    """`.rows` / `.data` are host snapshots: in-place writes fail loudly;
    `sk.rows[i] = regs` (the reference's sliding.py:202 idiom) and
    `ldca.data = arr` upload."""
    from paper_1901_07306_b200 import LdcaConfig, LdcaSketch, SeavSketch, SeedFamily, make_config

    cfg = make_config(theta=64)
    rng = np.random.default_rng(5)
    hips = rng.integers(0, 2**32, size=2000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=2000, dtype=np.uint64)
    a, b = SeavSketch(cfg, SeedFamily()), SeavSketch(cfg, SeedFamily())
    a.update_batch(hips, oips)
    with pytest.raises(ValueError):
        a.rows[0][0, 0] = 1
    rows_b = b.rows
    for i, r in enumerate(a.rows):
        rows_b[i] = r
    assert b.payload_bytes() == a.payload_bytes()
    assert (rows_b[1] == a.rows[1]).all()
    b.clear()
    b.rows = a.rows
    assert b.payload_bytes() == a.payload_bytes()
    with pytest.raises(Exception):
        rows_b[0] = np.zeros((3, 3))

    la, lb = LdcaSketch(LdcaConfig(), SeedFamily()), LdcaSketch(LdcaConfig(), SeedFamily())
    la.update_batch(hips, oips)
    with pytest.raises(ValueError):
        la.data[0, 0, 0] = 1
    lb.data = la.data
    assert lb.payload_bytes() == la.payload_bytes()


def test_restore_single_heavy_host_and_sorted_unique(cuda):  # :342-352, :418-426
    from paper_1901_07306_b200 import SeavSketch, SeedFamily, make_config

    sk = SeavSketch(make_config(theta=1024), SeedFamily())
    rng = np.random.default_rng(21)
    hip = 0xC0A80101
    sk.update_batch(np.full(4096, hip, dtype=np.uint64), rng.integers(0, 2**32, size=4096, dtype=np.uint64))
    found = sk.restore()
    cand = next(c for c in found if c.ip == hip)
    assert cand.source_sea == hip & 0xF and cand.union_weight >= 3
    ips = [c.ip for c in found]
    assert ips == sorted(set(ips))


def test_restore_matches_brute_force_12bit(cuda):  # :355-415
    from paper_1901_07306_b200 import SeavSketch, SeedFamily, make_config

    cfg = make_config(r=4, sr=4, a=2, theta=64, addr_bits=12)
    sk = SeavSketch(cfg, SeedFamily())
    rng = np.random.default_rng(33)
    heavy = rng.integers(0, 1 << 12, size=6, dtype=np.uint64)
    for h in heavy:
        sk.update_batch(np.full(256, h, dtype=np.uint64), rng.integers(0, 2**32, size=256, dtype=np.uint64))
    sk.update_batch(rng.integers(0, 1 << 12, size=3000, dtype=np.uint64),
                    rng.integers(0, 2**32, size=3000, dtype=np.uint64))
    rows = sk.rows
    expected = set()
    for rp in range(1 << cfg.r):
        for lp in range(1 << cfg.lp_bits):
            regs = [int(rows[i][rp, cfg.index_of(i, lp)]) for i in range(cfg.sr)]
            union = (1 << cfg.g) - 1
            for v in regs:
                union &= v
            if all(bin(v).count("1") >= 3 for v in regs) and bin(union).count("1") >= 3:
                expected.add((lp << cfg.r) | rp)
    got = {c.ip for c in sk.restore()}
    assert got == expected and got >= {int(h) for h in heavy}


def test_merge_rejects_mismatched_config(cuda):  # :328-332
    from paper_1901_07306_b200 import ConfigError, SeavSketch, SeedFamily, make_config

    with pytest.raises(ConfigError):
        SeavSketch(make_config(), SeedFamily()).merge(SeavSketch(make_config(r=2, sr=5, a=1), SeedFamily()))


# --- long sketch (test_long_sketch.py) -----------------------------------------
def small_ldca(lr=2, lc=16, k=64):
    from paper_1901_07306_b200 import LdcaConfig, LdcaSketch, SeedFamily

    return LdcaSketch(LdcaConfig(lr=lr, lc=lc, k=k), SeedFamily())


def test_one_pair_sets_at_most_lr_bits_and_untouched_is_zero(cuda):  # :108-160
    sk = small_ldca(lr=3)
    assert sk.estimate(777) == (0.0, False)
    sk.update(42, 4242)
    snap = sk.data.copy()
    assert 1 <= int(np.unpackbits(snap).sum()) <= 3
    sk.update(42, 4242)
    assert (sk.data == snap).all()


def test_union_never_exceeds_rows_and_matches_host_and(cuda):  # :181-193
    rng = np.random.default_rng(15)
    sk = small_ldca(lr=2, lc=4, k=512)
    sk.update_batch(rng.integers(0, 2**32, size=3000, dtype=np.uint64),
                    rng.integers(0, 2**32, size=3000, dtype=np.uint64))
    probe = 0xDDDD1111
    union = sk.union_register(probe)
    data = sk.data
    cells = [data[i, sk.row_column(i, probe)] for i in range(2)]
    assert (union == (cells[0] & cells[1])).all()
    ones = int(np.unpackbits(union).sum())
    assert all(ones <= int(np.unpackbits(c).sum()) for c in cells)
    est, sat = sk.estimate(probe)
    z0 = 512 - ones
    assert (est, sat) == ((512 * math.log(512), True) if z0 == 0 else (-512 * math.log(z0 / 512), False))


def test_single_host_estimate_accuracy(cuda):  # :162-178 (200 trials, <= 5 % mean error)
    from paper_1901_07306_b200 import LdcaConfig, LdcaSketch, SeedFamily

    k, n, trials = 8192, 1024, 200
    rng = np.random.default_rng(99)
    rel, signed = [], []
    for t in range(trials):
        sk = LdcaSketch(LdcaConfig(lr=2, lc=64, k=k), SeedFamily(master_seed=t))
        hip = int(rng.integers(0, 2**32))
        oips = np.unique(rng.integers(0, 2**32, size=n + 40, dtype=np.uint64))[:n]
        sk.update_batch(np.full(n, hip, dtype=np.uint64), oips)
        est, saturated = sk.estimate(hip)
        assert not saturated
        rel.append(abs(est - n) / n)
        signed.append((est - n) / n)
    assert np.mean(rel) <= 0.05 and abs(np.mean(signed)) <= 0.02


# --- window detector (test_window_detector.py) ----------------------------------
def test_detects_heavy_host_and_estimates(cuda):  # :285-295
    st = fresh()
    heavy_host(st, 0x0A000001, 2048, np.random.default_rng(8))
    reports = st.finalize_window()
    assert [r.ip for r in reports] == [0x0A000001]
    rep = reports[0]
    assert rep.source == "discrete" and not rep.saturated
    assert rep.estimated_cardinality == pytest.approx(2048, rel=0.1)


def test_register_sharing_candidate_filtered(cuda):  # :303-331
    st = fresh()
    cfg = st.seav.config
    rng = np.random.default_rng(16)
    rp = 5
    lp_h = int(rng.integers(0, 1 << cfg.lp_bits))
    light = (lp_h << cfg.r) | rp
    heavies = []
    for i in range(cfg.sr):
        lp_s = int(rng.integers(0, 1 << cfg.lp_bits))
        for j in range(cfg.ibn[i]):
            pos = (cfg.isb[i] + j) % cfg.lp_bits
            lp_s = (lp_s & ~(1 << pos)) | (lp_h & (1 << pos))
        heavies.append((lp_s << cfg.r) | rp)
        heavy_host(st, heavies[-1], 4096, rng)
    heavy_host(st, light, st.theta // 16, rng)
    assert light in {c.ip for c in st.seav.restore()}
    reported = {r.ip for r in st.finalize_window()}
    assert light not in reported and set(heavies) <= reported


def test_beta_monotone_and_reports_from_restore(cuda):  # :334-350
    st = fresh()
    rng = np.random.default_rng(30)
    for hip in rng.integers(0, 2**32, size=6, dtype=np.uint64).tolist():
        heavy_host(st, hip, int(rng.integers(700, 3000)), rng)
    strict = {r.ip for r in st.finalize_window(beta=1.0)}
    loose = {r.ip for r in st.finalize_window(beta=0.5)}
    assert strict <= loose <= {c.ip for c in st.seav.restore()}


def test_functional_wrappers(cuda):  # :394-402
    from paper_1901_07306_b200.window_detector import finalize_window, process_pair, reset

    st = fresh()
    process_pair(st, 1, 2)
    assert st.pair_count == 1 and finalize_window(st) == []
    with pytest.raises(ValueError):
        finalize_window(st, theta=999)
    reset(st)
    assert st.window_id == 1


def test_report_list_behaves_like_a_list(cuda):
    st = fresh()
    rng = np.random.default_rng(31)
    for hip in (0x0A000001, 0x0A000002, 0x0B000003):
        heavy_host(st, hip, 2048, rng)
    reps = st.finalize_window()
    lst = list(reps)
    assert len(reps) == len(lst) == 3 and reps == lst and lst == reps
    assert reps[0] == lst[0] and reps[-1] == lst[-1] and reps[1:] == lst[1:]
    acc = []
    acc += reps
    assert acc == lst and reps + [] == lst
    assert [r.window_id for r in reps] == [0, 0, 0]


# --- distributed (test_distributed.py) -------------------------------------------
def test_frame_round_trip_and_size(cuda):  # :45-60
    from paper_1901_07306_b200 import LdcaSketch, SeavSketch, deserialize, parse_frame, serialize

    st = fresh(k=4096, lr=2, lc=64, design_n=4e3)
    rng = np.random.default_rng(1)
    empty_sizes = (len(serialize(st.seav, 0)), len(serialize(st.ldca, 0)))
    st.process_batch(rng.integers(0, 2**32, size=8000, dtype=np.uint64),
                     rng.integers(0, 2**32, size=8000, dtype=np.uint64))
    for sketch in (st.seav, st.ldca):
        blob = serialize(sketch, window_id=7)
        back = deserialize(blob)
        assert back.payload_bytes() == sketch.payload_bytes() and parse_frame(blob).window_id == 7
    assert isinstance(deserialize(serialize(st.seav, 0)), SeavSketch)
    assert isinstance(deserialize(serialize(st.ldca, 0)), LdcaSketch)
    assert (len(serialize(st.seav, 0)), len(serialize(st.ldca, 0))) == empty_sizes


def test_merge_errors(cuda):  # :129-159
    from paper_1901_07306_b200 import DetectorParams, DetectorState, MergeError, merge_frames, parse_frame
    from paper_1901_07306_b200 import SketchFrame, serialize

    st = fresh(k=4096, lr=2, lc=64, design_n=4e3)
    frames = [parse_frame(serialize(st.seav, 0)), parse_frame(serialize(st.ldca, 0))]
    with pytest.raises(MergeError, match="ldca"):
        merge_frames(frames[:1])
    with pytest.raises(MergeError):
        merge_frames([])
    with pytest.raises(MergeError, match="window"):
        merge_frames(frames + [parse_frame(serialize(st.seav, 1)), parse_frame(serialize(st.ldca, 1))])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        other = DetectorState.create(DetectorParams(theta=2048, k=4096, lr=2, lc=64, design_n=4e3))
    with pytest.raises(MergeError, match="config"):
        merge_frames(frames + [parse_frame(serialize(other.seav, 0)), parse_frame(serialize(other.ldca, 0))])
    tweaked = SketchFrame(kind=frames[0].kind, config_block=b"\x00" * len(frames[0].config_block), window_id=0,
                          payload=frames[0].payload)
    with pytest.raises(MergeError):
        merge_frames([tweaked] + frames)


def test_topology_frames_and_windows(cuda, tmp_path):  # :245-266
    from paper_1901_07306_b200 import DetectorParams, parse_frame, simulate_topology

    params = DetectorParams(theta=1024, k=4096, lr=2, lc=64, design_n=4e3)
    rng = np.random.default_rng(11)
    hips = rng.integers(0, 2**32, size=6000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=6000, dtype=np.uint64)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = simulate_topology(params, np.zeros(6000, dtype=np.uint32), hips, oips, n_wp=2, frames_dir=tmp_path)
        assert [r.window_id for r in simulate_topology(params, rng.integers(0, 20, size=6000).astype(np.uint32),
                                                       hips, oips, n_wp=2, window_slices=10)] == [0, 1]
    assert len(res) == 1
    names = sorted(p.name for p in tmp_path.iterdir())
    assert names == ["wp0_win0_ldca.sspd", "wp0_win0_seav.sspd", "wp1_win0_ldca.sspd", "wp1_win0_seav.sspd"]
    for p in tmp_path.iterdir():
        parse_frame(p.read_bytes())


# --- sliding (test_sliding.py) ------------------------------------------------------
def test_expiry_boundary_and_all_expire(cuda):  # :27-69
    from paper_1901_07306_b200 import TimestampPool

    pool = TimestampPool(4, window_slices=5)
    pool.touch(0)
    for _ in range(4):
        pool.advance_slice()
        assert pool.is_active(0)
    pool.advance_slice()
    assert not pool.is_active(0)
    pool = TimestampPool(64, window_slices=3)
    pool.touch_batch(np.arange(64))
    for _ in range(3):
        pool.advance_slice()
    assert not pool.active().any()


def test_touch_batch_numpy_index_semantics(cuda):  # sliding.py:77-79 is `ts[slot_indexes] = now`
    from paper_1901_07306_b200 import TimestampPool

    rng = np.random.default_rng(3)
    for ts_window in (3, 300, 40000):  # u8 / u16 / u32 stamps
        pool = TimestampPool(1000, window_slices=ts_window)
        ref = pool.ts.copy()
        for step in range(4):
            idx = rng.integers(-1000, 1000, size=300)
            pool.touch_batch(idx)
            ref[idx] = pool._wrapped_now()
            mask = rng.random(1000) < 0.1
            pool.touch_batch(mask)
            ref[mask] = pool._wrapped_now()
            pool.touch_batch(np.array([], dtype=np.int64))
            assert (pool.ts == ref).all(), (ts_window, step)
            pool.advance_slice()
            ref = pool.ts.copy()
        before = pool.ts.copy()
        for bad in (np.array([5, 1000]), np.array([-1001, 3]), np.array([2**63], dtype=np.uint64)):
            with pytest.raises(IndexError):
                pool.touch_batch(bad)
        with pytest.raises(IndexError):
            pool.touch_batch(np.ones(7, dtype=bool))
        assert (pool.ts == before).all()


def test_boundary_straddler_found_only_by_sliding(cuda):  # :165-196, acceptance criterion 7
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    params = DetectorParams(theta=1024, k=4096, lr=2, lc=32, design_n=2e3)
    rng = np.random.default_rng(77)
    hip = 0x0B0C0D0E
    first = np.unique(rng.integers(0, 2**32, size=560, dtype=np.uint64))[:512]
    second = np.unique(rng.integers(2**31, 2**32, size=560, dtype=np.uint64))[:512]
    for half in (first, second):
        st = fresh(theta=1024, k=4096, lr=2, lc=32, design_n=2e3)
        st.process_batch(np.full(512, hip, dtype=np.uint64), half)
        assert [r.ip for r in st.finalize_window()] == []
    per_slice = {}
    for j in range(5):
        per_slice[5 + j] = first[j * 103: (j + 1) * 103 + (512 - 5 * 103) * (j == 4)]
        per_slice[10 + j] = second[j * 103: (j + 1) * 103 + (512 - 5 * 103) * (j == 4)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(params, window_slices=10)
    hits = []
    for s in range(16):
        chunk = per_slice.get(s, np.array([], dtype=np.uint64))
        if len(chunk):
            det.observe_batch(np.full(len(chunk), hip, dtype=np.uint64), chunk)
        hits += [(s, r.ip) for r in det.detect()]
        det.advance_slice()
    assert (14, hip) in hits


def test_detect_after_everything_expired_is_empty(cuda):  # :199-207
    from paper_1901_07306_b200 import DetectorParams, SlidingDetector

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(DetectorParams(theta=1024, k=4096, lr=2, lc=32, design_n=2e3), window_slices=4)
    rng = np.random.default_rng(3)
    det.observe_batch(np.full(2048, 0x01010101, dtype=np.uint64), rng.integers(0, 2**32, size=2048, dtype=np.uint64))
    assert det.detect()
    for _ in range(4):
        det.advance_slice()
    assert det.detect() == []


# --- the reference's own call pattern: 65,536-pair host buffers (cli.py:215-217)
@pytest.mark.parametrize("stage", [1 << 23, 100_003])
def test_host_batches_staged_bit_exact_vs_oracle(cuda, oracle, stage):
    """process_batch fed host arrays the way `sspd detect` and
    simulate_window feed it (65,536-pair buffers; uint64 like the
    reference's astype, plus uint32 and CPU-tensor batches) is staged in
    pinned memory and scanned in large batches.  Reads in the middle
    (payload_bytes, rows, finalize), device-tensor batches interleaved, a
    rejected batch (nothing of it staged) and reset (staged pairs dropped)
    all see exactly the reference's state; `stage` = 100,003 forces many
    flushes through both staging buffers."""
    import torch

    from conftest import params_block
    from paper_1901_07306_b200 import DetectorParams
    from paper_1901_07306_b200.errors import DataError

    dp = DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=2e6)
    _, _, p = params_block(dp)
    rng = np.random.default_rng(31)
    n = 1_500_000
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    hips[:300_000] = rng.integers(0, 2**32, size=40, dtype=np.uint64)[rng.integers(0, 40, size=300_000)]
    st = fresh(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=2e6)
    st.host_stage_pairs = stage
    seav = np.zeros(p.seav_bytes, dtype=np.uint8)
    ldca = np.zeros(p.ldca_bytes, dtype=np.uint8)
    B = 65_536
    for i, lo in enumerate(range(0, n, B)):
        h, o = hips[lo:lo + B], oips[lo:lo + B]
        if i % 5 == 1:
            h, o = h.astype(np.uint32), o.astype(np.uint32)
        elif i % 5 == 2:
            h = torch.from_numpy(h.astype(np.uint32).view(np.int32))
            o = torch.from_numpy(o.astype(np.uint32).view(np.int32))
        elif i % 5 == 3:
            h = torch.from_numpy(h.astype(np.uint32).view(np.int32)).cuda()  # device batch, scanned at once
            o = torch.from_numpy(o.astype(np.uint32).view(np.int32)).cuda()
        st.process_batch(h, o)
        oracle.scan(p, hips[lo:lo + B], oips[lo:lo + B], seav, ldca, threads=4)
        if i == 7:  # a read mid-stream sees every staged pair
            assert st.seav.payload_bytes() == seav.tobytes()
            assert st.ldca.payload_bytes() == ldca.tobytes()
        if i == 9:
            bad = hips[lo:lo + B].copy()
            bad[-1] = 1 << 32
            with pytest.raises(DataError):
                st.process_batch(bad, oips[lo:lo + B])
    assert st.pair_count == n
    assert st.seav.payload_bytes() == seav.tobytes()
    assert st.ldca.payload_bytes() == ldca.tobytes()
    reps = st.finalize_window()
    ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
    z0 = oracle.filter_z0(p, ldca, ips)
    k = dp.k
    want = [int(ip) for ip, z in zip(ips, z0) if z == 0 or -k * math.log(z / k) >= dp.beta * dp.theta]
    assert [r.ip for r in reps] == want and len(want) > 0
    st.process_batch(hips[:1000], oips[:1000])  # staged, then dropped by reset
    st.reset()
    assert st.seav.total_set_bits() == 0 and not st.ldca.data.any()
    st.process_pair(int(hips[0]), int(oips[0]))
    s1, l1 = oracle.scan(p, hips[:1], oips[:1])
    assert st.seav.payload_bytes() == s1.tobytes() and st.ldca.payload_bytes() == l1.tobytes()


# --- device plumbing ---------------------------------------------------------------
def test_fast_stream_helpers_match_torch(cuda):
    """_device.current_stream / on_stream (the per-slide host path) select and
    restore exactly what torch.cuda.current_stream / torch.cuda.stream do,
    nested, and on an exception."""
    import torch

    from paper_1901_07306_b200._device import current_stream, on_stream

    base = torch.cuda.current_stream()
    assert current_stream() == base
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with on_stream(s1):
        assert torch.cuda.current_stream() == s1 and current_stream() == s1
        with on_stream(s2):
            assert torch.cuda.current_stream() == s2
        assert torch.cuda.current_stream() == s1
    assert torch.cuda.current_stream() == base
    with pytest.raises(RuntimeError):
        with on_stream(s2):
            raise RuntimeError("inside")
    assert torch.cuda.current_stream() == base
    # work issued inside lands on the selected stream
    x = torch.zeros(1 << 20, device="cuda")
    with on_stream(s1):
        x.add_(1)
        ev = torch.cuda.Event()
        ev.record()
    s1.synchronize()
    assert ev.query() and float(x[0]) == 1.0
