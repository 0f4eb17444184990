"""Pure host cost of the config-4 per-slide loop (diagnostic, not a bench).

    python tools/host_overhead_config4.py

Same detector and loop as the bench's config 4, but every slice carries only
1,024 packets, so the device work per slide is small and the loop time is
the host's own cost (Python, ctypes, launch calls) per observe / detect_async
/ advance_slice."""
import sys, time, warnings, torch
sys.path.insert(0, '.')
from paper_1901_07306_b200 import DetectorParams, SlidingDetector
dev = torch.device('cuda', 0)
g = torch.Generator(device=dev); g.manual_seed(1)
n_sl, per = 299, 1024
hips = torch.randint(0, 2**31, (n_sl * per,), device=dev, dtype=torch.int32, generator=g)
oips = torch.randint(0, 2**31, (n_sl * per,), device=dev, dtype=torch.int32, generator=g)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8), window_slices=300)
for rep in range(3):
    det.reset(); pend = []
    t = [0.0, 0.0, 0.0]
    torch.cuda.synchronize(); T0 = time.perf_counter()
    for s in range(n_sl):
        a = time.perf_counter()
        det.observe_batch(hips[s * per:(s + 1) * per], oips[s * per:(s + 1) * per])
        b = time.perf_counter()
        pend.append(det.detect_async())
        c = time.perf_counter()
        det.advance_slice()
        d = time.perf_counter()
        while len(pend) > det.pipeline_depth:
            len(pend.pop(0))
        t[0] += b - a; t[1] += c - b; t[2] += d - c
    T1 = time.perf_counter()
    print("loop %.1f ms (%.0f us/slide): observe %.1f, detect_async %.1f, advance %.1f us/slide"
          % ((T1 - T0) * 1e3, (T1 - T0) / n_sl * 1e6, *(x / n_sl * 1e6 for x in t)))
