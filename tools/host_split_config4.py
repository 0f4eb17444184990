"""Host time of the config-4 sliding loop split into Python work and
waiting on the device (diagnostic, not a bench).

    python tools/host_split_config4.py

Wraps torch.cuda.Event.synchronize (the only blocking call of the loop) to
accumulate the time the host spends waiting; the rest of the loop is host
work (Python + launches).  If waiting is small, the host is the bound."""
import sys, time, warnings, torch
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
wait = [0.0]
orig = torch.cuda.Event.synchronize
def timed_sync(self):
    a = time.perf_counter(); orig(self); wait[0] += time.perf_counter() - a
torch.cuda.Event.synchronize = timed_sync
for rep in range(3):
    det.reset(); pend = []; wait[0] = 0.0
    torch.cuda.synchronize(); T0 = time.perf_counter()
    for s in range(n_sl):
        lo, hi = bounds[s], bounds[s + 1]
        det.observe_batch(hips[lo:hi], oips[lo:hi])
        pend.append(det.detect_async())
        det.advance_slice()
        while len(pend) > det.pipeline_depth:
            len(pend.pop(0))
    T1 = time.perf_counter()
    for p in pend:
        len(p)
    torch.cuda.synchronize(); T2 = time.perf_counter()
    print("loop %.1f ms: host work %.1f ms, waiting %.1f ms (%.0f us/slide work); drain %.1f ms"
          % ((T1 - T0) * 1e3, (T1 - T0 - wait[0]) * 1e3, wait[0] * 1e3, (T1 - T0 - wait[0]) / n_sl * 1e6,
             (T2 - T1) * 1e3))
