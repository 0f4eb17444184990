"""Generate the golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
It writes tests/golden/golden.json (+ golden.npz for raw arrays).  Nothing
at test time reads /root/reference: the tests compare the CPU oracle and
the CUDA path against these committed fixtures.

Each case stores its own inputs (so numpy RNG stream changes can never
silently change a fixture) and the reference's outputs: SEAV/LDCA payload
bytes (raw when small, SHA-256 always), restore candidates, detection
reports (float estimates as repr strings, compared exactly), sliding pool
snapshots, merged pools, routing lanes and frame bytes.
"""

from __future__ import annotations

import hashlib
import json
import sys
import warnings
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import sspd  # noqa: E402
from sspd import distributed as ref_dist  # noqa: E402
from sspd.hashing import SeedFamily, derive_seed, hash_full, hash_range, mix64  # noqa: E402
from sspd.long_sketch import LdcaConfig, plan_rows  # noqa: E402
from sspd.short_sketch import SeavConfig, SeavSketch, tau_from_theta  # noqa: E402
from sspd.sliding import SlidingDetector, TimestampPool, timestamp_dtype  # noqa: E402
from sspd.window_detector import DetectorParams, DetectorState  # noqa: E402

from tools.workloads import CONFIG1, generate  # noqa: E402

ARR: dict[str, np.ndarray] = {}


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def put(name: str, a: np.ndarray) -> str:
    ARR[name] = np.ascontiguousarray(a)
    return name


def reports_list(reps):
    return [[r.ip, repr(r.estimated_cardinality), bool(r.saturated), r.window_id, r.source] for r in reps]


def params_dict(p: DetectorParams) -> dict:
    return {k: getattr(p, k) for k in ("theta", "r", "sr", "a", "g", "k", "lr", "lc", "v", "design_n",
                                       "beta", "master_seed", "restore_cap", "addr_bits")}


def hash_kats():
    keys = [0, 1, 2, 0xDEADBEEF, 0xFFFFFFFF, 0x7FFFFFFF, 0xC0A80101, 123456789]
    masters = [0x5EED, 0, 1, 0xDEADBEEF, (1 << 64) - 1]
    tags = [1, 2, 3, 4, 5] + list(range(16, 16 + 64))
    moduli = [1, 2, 7, 8, 16, 100, 174, 1000, 1024, 8192, 12345, 65535, 1 << 20, (1 << 31) - 1, (1 << 32) - 5]
    seeds = SeedFamily()
    out = {
        "mix64": [[k, mix64(k)] for k in keys + [(1 << 64) - 1, 1 << 63]],
        "derive_seed": [[m, t, derive_seed(m, t)] for m in masters for t in tags],
        "hash_full_h1": [[k, hash_full(k, seeds.h1)] for k in keys],
        "hash_range": [[k, m, hash_range(k, seeds.h3, m)] for k in keys for m in moduli],
    }
    rng = np.random.default_rng(5)
    big = rng.integers(0, 2**64, size=2000, dtype=np.uint64).tolist()
    out["hash_range_random"] = [[k, m, hash_range(k, seeds.lh(3), m)] for k in big for m in moduli[:8]]
    return out


def geometry_kats():
    cases = []
    for r in (0, 2, 4, 8, 12, 16):
        for sr in (2, 3, 4, 5, 6, 8):
            for a in (1, 2, 3):
                for g in (8, 16):
                    for ab in (12, 32):
                        item = {"r": r, "sr": sr, "a": a, "g": g, "addr_bits": ab, "theta": 1024}
                        try:
                            c = SeavConfig(r=r, sr=sr, a=a, theta=1024, g=g, addr_bits=ab)
                            item.update(isb=list(c.isb), ibn=list(c.ibn), sc=list(c.sc), tau=c.tau,
                                        memory_bytes=c.memory_bytes())
                        except sspd.ConfigError as e:
                            item["error"] = str(e)
                        cases.append(item)
    taus = [[t, g, tau_from_theta(t, g)] for t in (1, 7, 8, 9, 64, 1000, 1024, 1025, 10**6) for g in (1, 8, 16, 64)]
    plans = []
    for v, n, k, mr in [(8192, 1e6, 8192, None), (8192, 1e6, 8192, 8), (64, 1e9, 8192, 8), (1024, 1e5, 1024, None),
                        (2048, 3e5, 1024, None), (65536, 8e7, 8192, 8), (8192, 2e3, 4096, 8)]:
        plans.append([v, n, k, mr, list(plan_rows(v, n, k, max_rows=mr))])
    dts = [[w, np.dtype(timestamp_dtype(w)).name] for w in (1, 100, 127, 128, 300, 32767, 40000)]
    return {"seav": cases, "tau": taus, "plan_rows": plans, "timestamp_dtype": dts}


def sketch_case(name, params: DetectorParams, hips, oips, raw_ldca_limit=1 << 17, batches=None, inputs=None):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(params)
        if batches:
            for lo in range(0, len(hips), batches):
                st.process_batch(hips[lo:lo + batches], oips[lo:lo + batches])
        else:
            st.process_batch(hips, oips)
        seav_b = st.seav.payload_bytes()
        ldca_b = st.ldca.payload_bytes()
        with warnings.catch_warnings(record=True) as wl:
            warnings.simplefilter("always")
            cands = st.seav.restore(on_overflow="warn")
        overflow = sorted(int(str(w.message).split("rp=")[1].split()[0]) for w in wl
                          if "rp=" in str(w.message))
        reps = st.finalize_window()
    item = {
        "name": name,
        "params": params_dict(params),
        "lr": st.ldca.config.lr, "lc": st.ldca.config.lc,
        "hips": put(f"{inputs or name}/hips", np.asarray(hips, dtype=np.uint32)),
        "oips": put(f"{inputs or name}/oips", np.asarray(oips, dtype=np.uint32)),
        "seav_sha": sha(seav_b), "ldca_sha": sha(ldca_b),
        "seav_bytes": len(seav_b), "ldca_bytes": len(ldca_b),
        "candidates": [[c.ip, c.source_sea, c.union_weight] for c in cands],
        "overflow": overflow,
        "reports": reports_list(reps),
        "z0": [[c.ip, int(st.ldca.config.k - np.unpackbits(st.ldca.union_register(c.ip)).sum())]
               for c in cands[:64]],
    }
    if len(seav_b) <= (1 << 17):
        item["seav_raw"] = put(f"{name}/seav", np.frombuffer(seav_b, dtype=np.uint8))
    if len(ldca_b) <= raw_ldca_limit:
        item["ldca_raw"] = put(f"{name}/ldca", np.frombuffer(ldca_b, dtype=np.uint8))
    return item


def sketch_cases():
    out = []
    rng = np.random.default_rng(1)
    n = 8000
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    hips[: n // 4] = 0x11223344
    out.append(sketch_case("small_k4096", DetectorParams(theta=1024, k=4096, lr=2, lc=64, design_n=4e3), hips, oips))

    rng = np.random.default_rng(12)
    hips = rng.integers(0, 2**32, size=20_000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=20_000, dtype=np.uint64)
    hips[:4096] = 0x7F000001
    out.append(sketch_case("default_20k", DetectorParams(design_n=2e5), hips, oips))

    rng = np.random.default_rng(11)
    hips = rng.integers(0, 2**32, size=5000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=5000, dtype=np.uint64)
    out.append(sketch_case("theta64", DetectorParams(theta=64, k=1024, lr=3, lc=32, design_n=5e3), hips, oips))

    # 12-bit address space, planted supers among light hosts
    rng = np.random.default_rng(52)
    hosts = rng.permutation(1 << 12)[: 20 + 1500].astype(np.uint64)
    sup, bg = hosts[:20], hosts[20:]
    hl, ol = [], []
    for h in sup:
        hl.append(np.full(128, h, dtype=np.uint64))
        ol.append(rng.integers(0, 2**32, size=128, dtype=np.uint64))
    counts = rng.integers(1, 9, size=len(bg))
    hl.append(np.repeat(bg, counts))
    ol.append(rng.integers(0, 2**32, size=int(counts.sum()), dtype=np.uint64))
    out.append(sketch_case("addr12", DetectorParams(theta=64, r=4, sr=4, a=2, addr_bits=12, k=512, lr=2, lc=16,
                                                    design_n=1e3), np.concatenate(hl), np.concatenate(ol)))

    rng = np.random.default_rng(61)
    oips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
    hips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
    hips[:256] = 0x0A0A0A0A
    out.append(sketch_case("g16", DetectorParams(theta=16, g=16, k=2048, lr=2, lc=64, design_n=3e3), hips, oips))

    rng = np.random.default_rng(71)
    hips = rng.integers(0, 2**32, size=6000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=6000, dtype=np.uint64)
    hips[:2000] = 0x01020304
    out.append(sketch_case("nonpow2", DetectorParams(theta=512, k=1000, lr=5, lc=100, design_n=6e3), hips, oips))
    out.append(sketch_case("planned47", DetectorParams(theta=1024, lr=47, lc=174, design_n=1e6), hips, oips,
                           raw_ldca_limit=0, inputs="nonpow2"))
    out.append(sketch_case("g32_sr5", DetectorParams(theta=128, r=2, sr=5, a=1, g=32, k=512, lr=2, lc=32,
                                                     design_n=6e3), hips, oips, inputs="nonpow2"))
    out.append(sketch_case("g64_r0", DetectorParams(theta=256, r=0, sr=4, a=2, g=64, k=256, lr=1, lc=16,
                                                    design_n=6e3), hips, oips, inputs="nonpow2"))

    rng = np.random.default_rng(81)
    hips = rng.integers(0, 2**32, size=200_000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=200_000, dtype=np.uint64)
    hips[:30_000] = 0xC0A80001
    hips[30_000:33_000] = 0xC0A80002
    out.append(sketch_case("r12", DetectorParams(theta=1024, r=12, design_n=2e5), hips, oips, raw_ldca_limit=0))
    out.append(sketch_case("r16", DetectorParams(theta=1024, r=16, k=4096, lr=4, lc=512, design_n=2e5), hips, oips,
                           raw_ldca_limit=0, inputs="r12"))
    out.append(sketch_case("r8_theta128", DetectorParams(theta=128, r=8, k=2048, lr=4, lc=256, design_n=2e5),
                           hips, oips, raw_ldca_limit=0, inputs="r12"))
    return out


def overflow_case():
    """Flooded array rp=3 with a small cap (test_short_sketch.py:429-449)."""
    cfg = SeavConfig()
    sk = SeavSketch(cfg, SeedFamily(), restore_cap=64)
    for row in sk.rows:
        row[3, :] = 0xFF
        row[7, ::3] = 0x0F
    rng = np.random.default_rng(5)
    hip = 0xC0A80000 | 0x1
    oips = rng.integers(0, 2**32, size=4096, dtype=np.uint64)
    sk.update_batch(np.full(4096, hip, dtype=np.uint64), oips)
    payload = sk.payload_bytes()
    with warnings.catch_warnings(record=True) as wl:
        warnings.simplefilter("always")
        cands = sk.restore(on_overflow="warn")
    sk2 = SeavSketch(cfg, SeedFamily(), restore_cap=10**9)
    sk2.load_payload(payload)
    try:
        big = sk2.restore_sea(7)
        big_n = len(big)
    except sspd.SeaOverflowError:
        big_n = -1
    return {
        "payload": put("overflow/seav", np.frombuffer(payload, dtype=np.uint8)),
        "cap": 64,
        "overflow": sorted(int(str(w.message).split("rp=")[1].split()[0]) for w in wl),
        "candidates": [[c.ip, c.source_sea, c.union_weight] for c in cands],
        "rp7_uncapped_count": big_n,
    }


def config1_case():
    hips, oips, supers = generate(CONFIG1)
    params = DetectorParams()
    st = DetectorState.create(params)
    for lo in range(0, len(hips), 1 << 16):
        st.process_batch(hips[lo:lo + (1 << 16)], oips[lo:lo + (1 << 16)])
    seav_b, ldca_b = st.seav.payload_bytes(), st.ldca.payload_bytes()
    cands = st.seav.restore(on_overflow="warn")
    reps = st.finalize_window()
    return {
        "stream_sha": sha(hips.tobytes() + oips.tobytes()),
        "n": len(hips),
        "supers": supers.tolist(),
        "seav_sha": sha(seav_b), "ldca_sha": sha(ldca_b),
        "seav_raw": put("config1/seav", np.frombuffer(seav_b, dtype=np.uint8)),
        "candidates": [[c.ip, c.source_sea, c.union_weight] for c in cands],
        "reports": reports_list(reps),
    }


def sliding_case():
    params = DetectorParams(theta=1024, k=4096, lr=2, lc=32, design_n=2e3)
    w = 12
    rng = np.random.default_rng(6)
    n = 20_000
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    hips[:2048] = 0x0A0A0A0A
    slices = rng.integers(0, 2 * w + 5, size=n).astype(np.uint8)
    det = SlidingDetector(params, window_slices=w)
    steps = []
    for s in range(2 * w + 5):
        sel = slices == s
        det.observe_batch(hips[sel], oips[sel])
        rep = det.detect() if s % 3 == 0 or s == w - 1 else None
        steps.append({
            "slice": s, "now": det.now,
            "pool_sha": sha(det.pool.ts.tobytes()),
            "seav_view_sha": sha(det.materialize_seav().payload_bytes()) if s % 4 == 0 else None,
            "ldca_view_sha": sha(det.materialize_ldca().tobytes()) if s % 4 == 0 else None,
            "reports": reports_list(rep) if rep is not None else None,
        })
        det.advance_slice()
    return {"params": params_dict(params), "w": w, "hips": put("sliding/hips", hips.astype(np.uint32)),
            "oips": put("sliding/oips", oips.astype(np.uint32)), "slices": put("sliding/slices", slices),
            "steps": steps}


def wrap_case():
    """uint8 stamps over 1200 slices with sweeps (test_sliding.py:80-93)."""
    pool = TimestampPool(64, window_slices=100)
    rng = np.random.default_rng(9)
    snaps = []
    for now in range(1, 1200):
        pool.advance_slice()
        if now % 7 == 0 and now <= 900:
            pool.touch_batch(rng.integers(0, 64, size=5))
        if now % 50 == 0:
            snaps.append([now, pool.sweep_count, sha(pool.ts.tobytes()), pool.active().astype(np.uint8).tolist()])
    return {"snaps": snaps}


def merge_pools_case():
    pools = [TimestampPool(4096, window_slices=30) for _ in range(3)]
    rng = np.random.default_rng(13)
    for s in range(50):
        for p in pools:
            p.touch_batch(rng.integers(0, 4096, size=40))
            p.advance_slice()
    ins = [put(f"mergepools/in{i}", p.ts.copy()) for i, p in enumerate(pools)]
    merged = ref_dist.merge_timestamp_pools(pools)
    return {"inputs": ins, "now": pools[0].now, "w": 30, "merged": put("mergepools/out", merged.ts.copy())}


def route_case():
    rng = np.random.default_rng(4)
    hips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
    out = {"hips": put("route/hips", hips.astype(np.uint32)), "oips": put("route/oips", oips.astype(np.uint32))}
    for n_wp in (1, 3, 7, 8, 16):
        out[f"hash_{n_wp}"] = put(f"route/hash_{n_wp}", ref_dist.route_pairs(hips, oips, n_wp, "hash", SeedFamily()))
    return out


def frames_case():
    rng = np.random.default_rng(1)
    params = DetectorParams(theta=1024, k=4096, lr=2, lc=64, design_n=4e3)
    states = []
    for wp in range(3):
        hips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
        oips = rng.integers(0, 2**32, size=3000, dtype=np.uint64)
        hips[:700] = 0x11223344
        st = DetectorState.create(params)
        st.process_batch(hips, oips)
        put(f"frames/h{wp}", hips.astype(np.uint32))
        put(f"frames/o{wp}", oips.astype(np.uint32))
        states.append(st)
    blobs = [ref_dist.serialize(s.seav, 5) for s in states] + [ref_dist.serialize(s.ldca, 5) for s in states]
    frames = [ref_dist.parse_frame(b) for b in blobs]
    mseav, mldca = ref_dist.merge_frames(frames)
    sim = ref_dist.simulate_window(params, 3, np.concatenate([ARR[f"frames/h{i}"] for i in range(3)]),
                                   np.concatenate([ARR[f"frames/o{i}"] for i in range(3)]), 4)
    return {"params": params_dict(params), "frame_sha": [sha(b) for b in blobs], "frame_len": [len(b) for b in blobs],
            "merged_seav_sha": sha(mseav.payload_bytes()), "merged_ldca_sha": sha(mldca.payload_bytes()),
            "sim_reports": reports_list(sim.reports), "sim_seav_sha": sha(sim.global_seav.payload_bytes()),
            "sim_ldca_sha": sha(sim.global_ldca.payload_bytes())}


def exact_case():
    """ExactOracle / metrics (evaluation.py:32-97) on a small skewed stream
    (raw arrays) and on the config-1 stream (hashes + truth + metrics)."""
    from sspd.evaluation import ExactOracle, metrics_report

    rng = np.random.default_rng(9)
    pool_h = rng.integers(0, 2**32, size=300, dtype=np.uint64)
    hips = pool_h[rng.integers(0, 300, size=20000)]
    oips = rng.integers(0, 5000, size=20000, dtype=np.uint64) * np.uint64(7919)
    hips[:4000] = pool_h[0]                      # one heavy host
    hips[4000:4100] = 0xFFFFFFFF                 # extreme keys
    oips[4000:4100] = np.arange(100) % 37
    hips[4100:4150] = 0
    oips[4100:4150] = 0xFFFFFFFF
    ex = ExactOracle(hips, oips)
    small = {"hips": put("exact/hips", hips.astype(np.uint32)), "oips": put("exact/oips", oips.astype(np.uint32)),
             "hosts": put("exact/hosts", ex.hosts), "counts": put("exact/counts", ex.counts),
             "super_64": ex.superpoints(64)}
    c_hips, c_oips, supers = generate(CONFIG1)
    ex1 = ExactOracle(c_hips, c_oips)
    st = DetectorState.create(DetectorParams())
    for lo in range(0, len(c_hips), 1 << 16):
        st.process_batch(c_hips[lo:lo + (1 << 16)], c_oips[lo:lo + (1 << 16)])
    det = [r.ip for r in st.finalize_window()]
    truth = ex1.superpoints(1024)
    cfg1 = {"n_hosts": int(len(ex1.hosts)), "hosts_sha": sha(ex1.hosts.astype(np.uint32).tobytes()),
            "counts_sha": sha(ex1.counts.astype(np.int64).tobytes()), "truth_1024": truth,
            "max_count": int(ex1.counts.max()), "total_distinct": int(ex1.counts.sum()),
            "metrics": {k: repr(v) for k, v in metrics_report(det, truth).items()}}
    kats = []
    for det_k, truth_k in (([1, 2, 3], [2, 3, 4, 5]), ([], [7]), ([9, 9, 8], [8]), ([1], [1])):
        kats.append([det_k, truth_k, {k: repr(v) for k, v in metrics_report(det_k, truth_k).items()}])
    return {"small": small, "config1": cfg1, "metric_kats": kats}


def update(keys):
    """Recompute only the named cases into the existing fixtures."""
    golden = json.loads((HERE / "golden.json").read_text())
    ARR.update(dict(np.load(HERE / "golden.npz")))
    for key in keys:
        golden[key] = CASES[key]()
    (HERE / "golden.json").write_text(json.dumps(golden, indent=None, separators=(",", ":")))
    np.savez_compressed(HERE / "golden.npz", **ARR)
    print("updated", keys)


CASES = {}


def main():
    golden = {
        "generator": "tests/golden/make_golden.py (reference sspd 0.1.0 from /root/reference/pkg/src)",
        "hash": hash_kats(),
        "geometry": geometry_kats(),
        "sketches": sketch_cases(),
        "overflow": overflow_case(),
        "config1": config1_case(),
        "sliding": sliding_case(),
        "wrap": wrap_case(),
        "merge_pools": merge_pools_case(),
        "route": route_case(),
        "frames": frames_case(),
        "exact": exact_case(),
    }
    (HERE / "golden.json").write_text(json.dumps(golden, indent=None, separators=(",", ":")))
    np.savez_compressed(HERE / "golden.npz", **ARR)
    print("wrote", HERE / "golden.json", (HERE / "golden.json").stat().st_size, "bytes;",
          HERE / "golden.npz", (HERE / "golden.npz").stat().st_size, "bytes")


CASES.update(exact=exact_case, frames=frames_case, route=route_case)

if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--update":
        update(sys.argv[2:])
    else:
        main()
