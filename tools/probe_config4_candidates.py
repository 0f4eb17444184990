"""Config-4 probe: candidates restored / kept per slide (DeviceFinalize.resolve)."""
import sys, time, warnings
sys.path.insert(0, ".")
import torch
from paper_1901_07306_b200 import DetectorParams, SlidingDetector
from paper_1901_07306_b200 import window_detector as wd
from tools.workloads import CONFIG4, CONFIG4_TIMING, generate

rec = []
orig = wd.DeviceFinalize.resolve
def resolve(self):
    first = self.m is None
    m = orig(self)
    if first:
        rec.append((self.found, m, self.cap))
    return m
wd.DeviceFinalize.resolve = resolve
dev = torch.device("cuda", 0)
hips, oips, supers, ts = generate(CONFIG4, "torch", dev, timing=CONFIG4_TIMING)
slices = ts // 1000
n_sl = int(slices[-1].item()) + 1
bounds = torch.searchsorted(slices, torch.arange(n_sl + 1, device=dev, dtype=slices.dtype)).cpu().tolist()
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8), window_slices=300)
for s in range(n_sl):
    det.observe_batch(hips[bounds[s]:bounds[s + 1]], oips[bounds[s]:bounds[s + 1]])
    r = det.detect()
    det.advance_slice()
for s in (0, 1, 5, 10, 30, 60, 100, 150, 200, 250, 298):
    if s < len(rec):
        print("slide", s, "found", rec[s][0], "kept", rec[s][1], "cap", rec[s][2])
ld = det.ldca_view() if hasattr(det, "ldca_view") else None
lv = torch.zeros(8 << 20, dtype=torch.uint8, device=dev)
det._ldca_view_into(lv)
bits = torch.bitwise_count(lv).sum().item() if hasattr(torch, "bitwise_count") else None
import numpy as np
b = int(np.unpackbits(lv.cpu().numpy()).sum())
print("ldca view density", b / (8 * lv.numel()))
sv = det._seav_view().device_buffer()
print("seav nonzero bytes frac", (sv != 0).float().mean().item(), "popcnt/8", float(np.unpackbits(sv.cpu().numpy()).mean()))
