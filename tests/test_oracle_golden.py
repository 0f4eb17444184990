"""Pin the CPU oracle (oracle/sspd_oracle.c) to the reference's own outputs.

The golden vectors were produced by executing the reference package
(tests/golden/make_golden.py).  Every oracle function used as a checker by
the GPU tests is verified here first.
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import params_block, params_from


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def reports_from(ips, z0s, k, cutoff, window_id=0, source="discrete"):
    """finalize_window's float step (window_detector.py:105-125) on oracle z0."""
    out = []
    for ip, z0 in zip(ips, z0s):
        if z0 == 0:
            est, sat = k * math.log(k), True
        else:
            est, sat = -k * math.log(z0 / k), False
        if sat or est >= cutoff:
            out.append([int(ip), repr(est), sat, window_id, source])
    return out


def test_hash_kats(oracle, golden):
    h = golden["hash"]
    for k, v in h["mix64"]:
        assert oracle.mix64(k) == v
    for m, t, v in h["derive_seed"]:
        assert oracle.derive_seed(m, t) == v
    from paper_1901_07306_b200.hashing import SeedFamily

    s = SeedFamily()
    for k, m, v in h["hash_range"]:
        assert oracle.hash_range(k, s.h3.value, m) == v
    for k, m, v in h["hash_range_random"]:
        assert oracle.hash_range(k, s.lh(3).value, m) == v
    for k, v in h["hash_full_h1"]:
        assert oracle.mix64(k ^ s.h1.value) & 0xFFFFFFFF == v


@pytest.mark.parametrize("idx", range(12))
def test_sketch_case(oracle, golden, garr, idx):
    if idx >= len(golden["sketches"]):
        pytest.skip("no such case")
    case = golden["sketches"][idx]
    dp = params_from(case["params"])
    scfg, lcfg, p = params_block(dp)
    hips, oips = garr[case["hips"]], garr[case["oips"]]
    seav, ldca = oracle.scan(p, hips, oips)
    assert sha(seav) == case["seav_sha"], case["name"]
    assert sha(ldca) == case["ldca_sha"], case["name"]
    ips, rps, ws, over = oracle.restore(p, seav, dp.restore_cap)
    assert [[int(a), int(b), int(c)] for a, b, c in zip(ips, rps, ws)] == case["candidates"]
    assert np.nonzero(over)[0].tolist() == case["overflow"]
    z0 = oracle.filter_z0(p, ldca, ips)
    assert [[int(a), int(b)] for a, b in zip(ips[:64], z0[:64])] == case["z0"]
    assert reports_from(ips, z0, lcfg.k, dp.beta * dp.theta) == case["reports"]


def test_multithreaded_scan_equals_single(oracle, golden, garr):
    case = next(c for c in golden["sketches"] if c["name"] == "r12")
    _, _, p = params_block(params_from(case["params"]))
    hips, oips = garr[case["hips"]], garr[case["oips"]]
    seav, ldca = oracle.scan(p, hips, oips, threads=4)
    assert sha(seav) == case["seav_sha"] and sha(ldca) == case["ldca_sha"]


def test_overflow_case(oracle, golden, garr):
    from paper_1901_07306_b200.window_detector import DetectorParams

    g = golden["overflow"]
    _, _, p = params_block(DetectorParams(design_n=2e5))
    seav = garr[g["payload"]]
    ips, rps, ws, over = oracle.restore(p, seav, g["cap"])
    assert np.nonzero(over)[0].tolist() == g["overflow"]
    assert [[int(a), int(b), int(c)] for a, b, c in zip(ips, rps, ws)] == g["candidates"]


def test_config1_stream_and_sketches(oracle, golden):
    from paper_1901_07306_b200.window_detector import DetectorParams
    from tools.workloads import CONFIG1, generate

    c = golden["config1"]
    hips, oips, supers = generate(CONFIG1)
    assert sha(hips.tobytes() + oips.tobytes()) == c["stream_sha"]
    assert supers.tolist() == c["supers"]
    dp = DetectorParams()
    _, lcfg, p = params_block(dp)
    seav, ldca = oracle.scan(p, hips, oips, threads=4)
    assert sha(seav) == c["seav_sha"] and sha(ldca) == c["ldca_sha"]
    ips, rps, ws, over = oracle.restore(p, seav, dp.restore_cap)
    assert [[int(a), int(b), int(x)] for a, b, x in zip(ips, rps, ws)] == c["candidates"]
    z0 = oracle.filter_z0(p, ldca, ips)
    assert reports_from(ips, z0, lcfg.k, dp.beta * dp.theta) == c["reports"]


def test_sliding_steps(oracle, golden, garr):
    """Pool snapshots, views and reports of a 29-slice run (sliding.py:33-248)."""
    g = golden["sliding"]
    dp = params_from(g["params"])
    _, lcfg, p = params_block(dp)
    w = g["w"]
    hips, oips, slices = garr[g["hips"]], garr[g["oips"]], garr[g["slices"]]
    from paper_1901_07306_b200.sliding import timestamp_dtype

    dt = timestamp_dtype(w)
    mask = np.iinfo(dt).max
    pool = np.full(p.slot_total, (-w) & mask, dtype=dt)
    now = 0
    for step in g["steps"]:
        sel = slices == step["slice"]
        oracle.observe(p, hips[sel], oips[sel], pool, now & mask)
        assert sha(pool.tobytes()) == step["pool_sha"], step["slice"]
        seav = oracle.materialize_seav(p, pool, now & mask, w)
        if step["seav_view_sha"]:
            assert sha(seav) == step["seav_view_sha"]
            assert sha(oracle.materialize_ldca(p, pool, now & mask, w)) == step["ldca_view_sha"]
        if step["reports"] is not None:
            ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
            ldca = oracle.materialize_ldca(p, pool, now & mask, w)
            z0 = oracle.filter_z0(p, ldca, ips)
            assert reports_from(ips, z0, lcfg.k, dp.beta * dp.theta, now, "sliding") == step["reports"]
        now += 1  # no sweep within 29 slices (period 256 - 2w)


def test_wraparound_sweep(oracle, golden):
    """uint8 stamps, w=100: sweep every 56 slices keeps ages from aliasing."""
    rng = np.random.default_rng(9)
    w, mask = 100, 0xFF
    pool = np.full(64, (-w) & mask, dtype=np.uint8)
    now, since, sweeps = 0, 0, 0
    snaps = iter(golden["wrap"]["snaps"])
    for t in range(1, 1200):
        now += 1
        since += 1
        if since >= 256 - 2 * w:
            oracle.sweep(pool, now & mask, w, (now - w) & mask)
            since, sweeps = 0, sweeps + 1
        if t % 7 == 0 and t <= 900:
            pool[rng.integers(0, 64, size=5)] = now & mask
        if t % 50 == 0:
            snap = next(snaps)
            assert snap[0] == t and snap[1] == sweeps
            assert sha(pool.tobytes()) == snap[2]
            ages = (np.uint64(now & mask) - pool.astype(np.uint64)) & np.uint64(mask)
            assert (ages < w).astype(np.uint8).tolist() == snap[3]


def test_merge_pools(oracle, golden, garr):
    g = golden["merge_pools"]
    pools = [garr[n] for n in g["inputs"]]
    out = oracle.merge_age_min(pools, g["now"] & 0xFFFF)
    assert (out == garr[g["merged"]]).all()


def test_route_hash(oracle, golden, garr):
    from paper_1901_07306_b200.hashing import SeedFamily

    g = golden["route"]
    for n_wp in (1, 3, 7, 8, 16):
        lanes = oracle.route_hash(garr[g["hips"]], garr[g["oips"]], SeedFamily().route.value, n_wp)
        assert (lanes == garr[g[f"hash_{n_wp}"]]).all()


def test_exact_cardinalities_oracle(oracle, golden, garr):
    """Numpy ExactOracle restatement vs the reference's (evaluation.py:32-58)."""
    from tools.workloads import CONFIG1, generate

    g = golden["exact"]
    hosts, counts = oracle.exact_cardinalities(garr["exact/hips"], garr["exact/oips"])
    assert (hosts == garr["exact/hosts"]).all() and (counts == garr["exact/counts"]).all()
    assert [int(h) for h in hosts[counts >= 64]] == g["small"]["super_64"]
    hips, oips, _ = generate(CONFIG1)
    hosts, counts = oracle.exact_cardinalities(hips, oips)
    c = g["config1"]
    assert len(hosts) == c["n_hosts"] and sha(hosts.tobytes()) == c["hosts_sha"]
    assert sha(counts.astype(np.int64).tobytes()) == c["counts_sha"]
    assert [int(h) for h in hosts[counts >= 1024]] == c["truth_1024"]


def test_metrics_host_logic(golden):
    """FPR/FNR/FTR normalised by |truth| (evaluation.py:73-97): the host
    arithmetic of the drop-in module against the reference's values."""
    from paper_1901_07306_b200 import UndefinedMetricError, metrics, metrics_report

    for det, truth, want in golden["exact"]["metric_kats"]:
        got = metrics_report(det, truth)
        assert {k: repr(v) for k, v in got.items()} == want
        assert metrics(det, truth) == (got["fpr"], got["fnr"], got["ftr"])
    with pytest.raises(UndefinedMetricError):
        metrics([1, 2], [])


def test_metric_rates_reference_cases():
    """test_evaluation.py:65-100 re-stated on the drop-in metric functions."""
    from paper_1901_07306_b200 import metrics, metrics_report

    truth = list(range(50))
    assert metrics(truth, truth) == (0.0, 0.0, 0.0)
    fpr, fnr, ftr = metrics(truth + [999], truth)
    assert fpr == pytest.approx(0.02) and fnr == 0.0 and ftr == pytest.approx(0.02)
    fpr, fnr, _ = metrics(truth[:-2], truth)
    assert fnr == pytest.approx(0.04) and fpr == 0.0
    assert metrics(list(range(100, 110)), list(range(5)))[0] == pytest.approx(2.0)
    rep = metrics_report([1, 2, 3, 99], [1, 2, 3, 4])
    assert rep["precision_nonpaper"] == pytest.approx(3 / 4) and rep["detected"] == 4 and rep["truth"] == 4
