"""GPU ExactOracle (csrc/exact.cu) against the reference's golden truth
sets and the numpy restatement; full-size properties at 2^28 keys."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def test_exact_golden_small_and_config1(cuda, golden, garr):
    from paper_1901_07306_b200 import DetectorParams, DetectorState, ExactOracle, metrics_report
    from tools.workloads import CONFIG1, generate

    g = golden["exact"]
    ex = ExactOracle(garr["exact/hips"], garr["exact/oips"])
    assert ex.hosts.dtype == np.uint32 and ex.counts.dtype == np.int64
    assert (ex.hosts == garr["exact/hosts"]).all() and (ex.counts == garr["exact/counts"]).all()
    assert ex.superpoints(64) == g["small"]["super_64"]
    assert ex.cardinality(0xFFFFFFFF) == 37 and ex.cardinality(0) >= 1 and ex.cardinality(12345) == 0

    hips, oips, _ = generate(CONFIG1)
    ex1 = ExactOracle(hips, oips)
    c = g["config1"]
    assert len(ex1.hosts) == c["n_hosts"] and sha(ex1.hosts.tobytes()) == c["hosts_sha"]
    assert sha(ex1.counts.tobytes()) == c["counts_sha"]
    truth = ex1.superpoints(1024)
    assert truth == c["truth_1024"]
    st = DetectorState.create(DetectorParams())
    st.process_batch(hips, oips)
    det = [r.ip for r in st.finalize_window()]
    assert {k: repr(v) for k, v in metrics_report(det, truth).items()} == c["metrics"]


@pytest.mark.parametrize("case", ["empty", "one", "same_key", "one_host", "all_distinct_hosts", "random"])
def test_exact_edge_cases_vs_oracle(cuda, oracle, case):
    from paper_1901_07306_b200 import ExactOracle

    rng = np.random.default_rng(len(case))
    n = {"empty": 0, "one": 1, "same_key": 5000, "one_host": 70001, "all_distinct_hosts": 100_000,
         "random": 3_000_017}[case]
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    if case == "same_key":
        hips[:], oips[:] = 0xFFFFFFFF, 0xFFFFFFFF
    elif case == "one_host":
        hips[:] = 0x0A000001
        oips = (oips % 40000).astype(np.uint32)
    elif case == "random":
        hips = (hips % 200_000).astype(np.uint32)
        oips = (oips % 3_000).astype(np.uint32)
    ex = ExactOracle(hips, oips)
    want_h, want_c = oracle.exact_cardinalities(hips, oips)
    assert (ex.hosts == want_h).all() and (ex.counts == want_c).all()
    assert ex.superpoints(2) == [int(h) for h in want_h[want_c >= 2]]


def test_exact_full_size_config2_properties(cuda):
    """2^28-packet config-2 window (device-resident input): planted super
    points carry their exact planted cardinality, counts sum to the number
    of distinct pairs, hosts strictly ascending."""
    import torch

    from paper_1901_07306_b200 import ExactOracle
    from tools.workloads import CONFIG2, cardinalities, generate

    hips, oips, supers = generate(CONFIG2, "torch", cuda)
    ex = ExactOracle(hips, oips)
    assert (np.diff(ex.hosts.astype(np.int64)) > 0).all()
    keys = (hips.to(torch.int64) & 0xFFFFFFFF) << 32 | (oips.to(torch.int64) & 0xFFFFFFFF)
    n_distinct = int(torch.unique(keys).numel())
    del keys
    assert int(ex.counts.sum()) == n_distinct
    planted = cardinalities(CONFIG2)[:CONFIG2.n_super]  # distinct by construction
    assert sorted(ex.cardinality(int(s)) for s in supers) == sorted(planted.tolist())
    assert len(ex.hosts) == CONFIG2.n_sources


# --- the reference's oracle tests (test_evaluation.py:27-60) re-stated -------

def test_empty_trace_oracle(cuda):  # :27-29
    from paper_1901_07306_b200 import ExactOracle

    oracle = ExactOracle(np.array([], dtype=np.uint64), np.array([], dtype=np.uint64))
    assert oracle.superpoints(1) == []


def test_oracle_counts_distinct_only(cuda):  # :32-40
    from paper_1901_07306_b200 import ExactOracle

    oracle = ExactOracle(np.array([1, 1, 1, 2, 2], dtype=np.uint64), np.array([9, 9, 8, 7, 7], dtype=np.uint64))
    assert oracle.cardinality(1) == 2 and oracle.cardinality(2) == 1 and oracle.cardinality(3) == 0
    assert oracle.superpoints(2) == [1]
    assert oracle.superpoints(1) == [1, 2]


def test_boundary_inclusion(cuda):  # :43-47
    from paper_1901_07306_b200 import ExactOracle, oracle_superpoints

    oracle = ExactOracle(np.repeat(np.uint64(5), 10), np.arange(10, dtype=np.uint64))
    assert oracle_superpoints(oracle, 10) == [5]
    assert oracle_superpoints(oracle, 11) == []


def test_oracle_implementations_agree(cuda):  # :50-60 (seeded instead of hypothesis)
    from paper_1901_07306_b200 import ExactOracle

    rng = np.random.default_rng(60)
    for _ in range(50):
        m = int(rng.integers(0, 301))
        pairs = rng.integers(0, 51, size=(m, 2))
        fast = ExactOracle(pairs[:, 0].astype(np.uint64), pairs[:, 1].astype(np.uint64))
        slow: dict[int, set] = {}
        for h, o in pairs.tolist():
            slow.setdefault(h, set()).add(o)
        slow_c = {h: len(v) for h, v in slow.items()}
        assert {int(h): int(c) for h, c in zip(fast.hosts, fast.counts)} == slow_c
        for theta in (1, 2, 5):
            assert fast.superpoints(theta) == sorted(h for h, c in slow_c.items() if c >= theta)
