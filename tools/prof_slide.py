"""Host-side cost per slide of the config-4 loop (diagnostic).

Times, with time.perf_counter and no extra synchronisation, how long the
host spends issuing observe_batch / detect / advance per slide, and the
GPU time of the whole trace (CUDA events), to tell host-bound from
device-bound.  python tools/prof_slide.py [--packets N] [--async]"""

import argparse
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from tools.workloads import CONFIG4, CONFIG4_TIMING, TimingSpec, generate, scaled

    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=0)
    ap.add_argument("--async", dest="asyn", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    spec, timing = CONFIG4, CONFIG4_TIMING
    if args.packets:
        spec = scaled(CONFIG4, max(1, CONFIG4.n_packets // args.packets))
        timing = TimingSpec(rate_pps=spec.n_packets / (CONFIG4.n_packets / CONFIG4_TIMING.rate_pps))
    hips, oips, supers, ts = generate(spec, "torch", dev, timing=timing)
    slices = ts // 1000
    n_sl = int(slices[-1].item()) + 1
    bounds = torch.searchsorted(slices, torch.arange(n_sl + 1, device=dev, dtype=slices.dtype)).cpu().tolist()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8),
                              window_slices=300)
    for rep in range(2):
        det.reset()
        torch.cuda.synchronize()
        t_obs = t_det = t_adv = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        w0 = time.perf_counter()
        pend = []
        for s in range(n_sl):
            lo, hi = bounds[s], bounds[s + 1]
            a = time.perf_counter()
            det.observe_batch(hips[lo:hi], oips[lo:hi])
            b = time.perf_counter()
            pend.append(det.detect_async() if args.asyn else det.detect())
            c = time.perf_counter()
            det.advance_slice()
            d = time.perf_counter()
            t_obs += b - a
            t_det += c - b
            t_adv += d - c
        total = sum(len(p) for p in pend)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        print(f"rep {rep}: wall {wall*1e3:.1f} ms, gpu-events {e0.elapsed_time(e1):.1f} ms, per slide host: "
              f"observe {t_obs/n_sl*1e6:.0f} us, detect {t_det/n_sl*1e6:.0f} us, advance {t_adv/n_sl*1e6:.0f} us; "
              f"reports {total}")


if __name__ == "__main__":
    main()
