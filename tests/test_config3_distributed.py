"""Config 3 (BASELINE configs[2]) at 1/256 scale: 8 routers, every planted
super split over 2-8 routers so that NO router sees it above threshold; only
the OR-merged sketches reveal it.  Shards are folded onto G = 1, 2, 4, 8
"GPUs" (GPU g scans shards g, g+G, ...) and every fold must give the same
merged bytes and the same report list."""

import warnings

import numpy as np
import pytest

from conftest import params_block

SCALE = 256


def _params():
    from paper_1901_07306_b200 import DetectorParams

    # config-3 geometry at this scale: SEAV r=16, LDCA 8 MiB
    return DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=1e7)


@pytest.fixture(scope="module")
def shards():
    from tools.workloads import CONFIG3, generate_shard, sharded_scaled

    spec = sharded_scaled(CONFIG3, SCALE)
    return spec, [generate_shard(spec, r) for r in range(spec.n_shards)]


def _reports(oracle, p, dp, seav, ldca):
    import math

    ips, _, _, _ = oracle.restore(p, seav, dp.restore_cap)
    z0 = oracle.filter_z0(p, ldca, ips)
    k = dp.k
    return [int(ip) for ip, z in zip(ips, z0) if z == 0 or -k * math.log(z / k) >= dp.beta * dp.theta]


def test_supers_only_visible_after_merge_oracle(oracle, shards):
    spec, data = shards
    dp = _params()
    _, _, p = params_block(dp)
    supers = set(data[0][2].tolist())
    merged_s = np.zeros(p.seav_bytes, dtype=np.uint8)
    merged_l = np.zeros(p.ldca_bytes, dtype=np.uint8)
    for h, o, _ in data:
        s, l = oracle.scan(p, h, o, threads=4)
        assert not supers & set(_reports(oracle, p, dp, s, l)), "a super was visible on one router"
        merged_s |= s
        merged_l |= l
    assert supers <= set(_reports(oracle, p, dp, merged_s, merged_l))


@pytest.mark.gpu
@pytest.mark.parametrize("gpus", [1, 2, 4, 8])
def test_shard_folding_and_device_merge(cuda, oracle, shards, gpus):
    from paper_1901_07306_b200 import DetectorState
    from paper_1901_07306_b200.distributed import device_or_into
    from paper_1901_07306_b200.multigpu import shards_for_rank

    spec, data = shards
    dp = _params()
    _, _, p = params_block(dp)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ranks = [DetectorState.create(dp) for _ in range(gpus)]
    for g, st in enumerate(ranks):
        for r in shards_for_rank(spec.n_shards, g, gpus):
            st.process_batch(data[r][0], data[r][1])
    root = ranks[0]
    device_or_into(root.seav.device_buffer(), [s.seav.device_buffer() for s in ranks], root.seav.nbytes)
    device_or_into(root.ldca.device_buffer(), [s.ldca.device_buffer() for s in ranks], root.ldca.nbytes)
    h = np.concatenate([d[0] for d in data])
    o = np.concatenate([d[1] for d in data])
    seav, ldca = oracle.scan(p, h, o, threads=8)
    assert root.seav.payload_bytes() == seav.tobytes()
    assert root.ldca.payload_bytes() == ldca.tobytes()
    got = [r.ip for r in root.finalize_window()]
    assert got == _reports(oracle, p, dp, seav, ldca)
    assert set(data[0][2].tolist()) <= set(got)
