import sys; sys.path.insert(0, ".")
import warnings
import numpy as np
from paper_1901_07306_b200 import DetectorParams, SlidingDetector
params = DetectorParams(theta=256, r=8, k=64, lr=3, lc=37, design_n=2e5)
w = 129
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    a = SlidingDetector(params, window_slices=w)
    b = SlidingDetector(params, window_slices=w)
    c = SlidingDetector(params, window_slices=w)
b.defer_ldca_stamps = False
c.ldca_ring_max_bytes = 0
print("deferred a", a._deferred().ring is not None, "c", c._deferred().ring)
rng = np.random.default_rng(7)
heavy = rng.integers(0, 2**32, size=3, dtype=np.uint64)
for s in range(4):
    n = int(rng.integers(0, 3000)) if s % 11 else 0
    hips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    oips = rng.integers(0, 2**32, size=n, dtype=np.uint64)
    hips[: n // 2] = heavy[s % 3]
    for d in (a, b, c):
        d.observe_batch(hips, oips)
    la, lb, lc_ = a.materialize_ldca(), b.materialize_ldca(), c.materialize_ldca()
    print(s, n, "ldca views a==b", np.array_equal(la, lb), "c==b", np.array_equal(lc_, lb), la.sum(), lb.sum(), lc_.sum())
    print("   seav a==b", a.materialize_seav().payload_bytes() == b.materialize_seav().payload_bytes())
    ra, rb, rc = a.detect(), b.detect(), c.detect()
    print("   reports", len(ra), len(rb), len(rc))
    print("   ts equal", np.array_equal(a.pool.ts, b.pool.ts), np.array_equal(c.pool.ts, b.pool.ts))
    for d in (a, b, c):
        d.advance_slice()
