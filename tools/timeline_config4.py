"""Two-stream timeline of the config-4 sliding loop (diagnostic).

    python tools/timeline_config4.py

CUDA events on the caller's stream (slice start, after the scan, after the
views of detect_async) and on detect_async's side stream (after the fused
finalize) for every slide; prints the device timestamps of a few early and
late slides, to see how the scan/view work and the finalize overlap.
"""
import sys, time, warnings, torch, numpy as np
sys.path.insert(0, '.')
from paper_1901_07306_b200 import DetectorParams, SlidingDetector
from tools.workloads import CONFIG4, CONFIG4_TIMING, generate
dev = torch.device('cuda', 0)
hips, oips, supers, ts = generate(CONFIG4, "torch", dev, timing=CONFIG4_TIMING)
slices = ts // 1000
n_sl = int(slices[-1].item()) + 1
bounds = torch.searchsorted(slices, torch.arange(n_sl + 1, device=dev, dtype=slices.dtype)).cpu().tolist()
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8), window_slices=300)
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(2):
    det.reset(); pend = []; ev = []
    main = torch.cuda.current_stream()
    t0 = E(); t0.record(main)
    for s in range(n_sl):
        lo, hi = bounds[s], bounds[s + 1]
        a = E(); a.record(main)
        det.observe_batch(hips[lo:hi], oips[lo:hi])
        b = E(); b.record(main)
        pend.append(det.detect_async())
        c = E(); c.record(main)
        side = det._async["side"]
        d = E(); d.record(side)
        det.advance_slice()
        ev.append((a, b, c, d))
    tot = sum(len(p) for p in pend)
    torch.cuda.synchronize()
    if rep == 1:
        for s in list(range(100, 112)) + list(range(280, 290)):
            a, b, c, d = ev[s]
            f = lambda e: t0.elapsed_time(e) * 1000
            print(f"slide {s}: main start {f(a):9.1f} scan_end {f(b):9.1f} views_end {f(c):9.1f} | side fin_end {f(d):9.1f} | scan {f(b)-f(a):6.1f} views {f(c)-f(b):6.1f}")
