"""Host-side cost of the config-4 sliding loop (diagnostic, not a bench).

    python tools/host_profile_config4.py

Runs the bench's per-slide loop (observe_batch -> detect_async ->
advance_slice) twice and prints the host time per call and per slide, then a
cProfile of one more pass: separates Python/launch overhead from waiting on
the device (Event.synchronize).
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
for rep in range(2):
    det.reset()
    t = np.zeros(3); pend = []
    torch.cuda.synchronize(); T0 = time.perf_counter()
    for s in range(n_sl):
        lo, hi = bounds[s], bounds[s + 1]
        a = time.perf_counter(); det.observe_batch(hips[lo:hi], oips[lo:hi]); b = time.perf_counter()
        pend.append(det.detect_async()); c = time.perf_counter()
        det.advance_slice(); d = time.perf_counter()
        t += [b - a, c - b, d - c]
    T1 = time.perf_counter()
    tot = sum(len(p) for p in pend)
    torch.cuda.synchronize(); T2 = time.perf_counter()
    print("per slide us: observe %.1f detect_async %.1f advance %.1f | loop %.1f ms, drain %.1f ms" % (*(t / n_sl * 1e6), (T1 - T0) * 1e3, (T2 - T1) * 1e3))
import cProfile, pstats
det.reset(); pend = []
pr = cProfile.Profile(); pr.enable()
for s in range(n_sl):
    lo, hi = bounds[s], bounds[s + 1]
    det.observe_batch(hips[lo:hi], oips[lo:hi]); pend.append(det.detect_async()); det.advance_slice()
tot = sum(len(p) for p in pend)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
