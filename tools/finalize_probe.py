"""GPU time of one slide's fused finalize (the CUDA-graph replay of
`sspd_finalize` that `SlidingDetector.detect_async` launches), alone on its
stream, against the sum of its kernels' durations (tuning probe, not a bench).

    python tools/finalize_probe.py [--packets N] [--slides S] [--reps R]

Scans the first S slices of the config-4 trace, builds the slide's views
once, then replays the finalize R times between CUDA events on the side
stream (each replay resolved before the next) and prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import sys
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from paper_1901_07306_b200._device import zeros_bytes
    from paper_1901_07306_b200.window_detector import DeviceFinalize
    from tools.workloads import CONFIG4, CONFIG4_TIMING, TimingSpec, generate, scaled

    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=0)
    ap.add_argument("--slides", type=int, default=150)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    spec, timing = CONFIG4, CONFIG4_TIMING
    if args.packets:
        spec = scaled(CONFIG4, max(1, CONFIG4.n_packets // args.packets))
        timing = TimingSpec(rate_pps=spec.n_packets / (CONFIG4.n_packets / CONFIG4_TIMING.rate_pps))
    hips, oips, _, ts = generate(spec, "torch", dev, timing=timing)
    slices = ts // 1000
    n_sl = int(slices[-1].item()) + 1
    bounds = torch.searchsorted(slices, torch.arange(n_sl + 1, device=dev, dtype=slices.dtype)).cpu().tolist()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        det = SlidingDetector(DetectorParams(theta=1024, r=16, k=8192, lr=8, lc=1024, design_n=2.15e8),
                              window_slices=300)
    for s in range(min(args.slides, n_sl)):
        lo, hi = bounds[s], bounds[s + 1]
        if hi > lo:
            det.observe_batch(hips[lo:hi], oips[lo:hi])
        det.advance_slice()
    seav = det.materialize_seav()
    lview = zeros_bytes(det._params.ldca_bytes)
    det._ldca_view_into(lview)
    if det._iv() is not None:
        src = det._seav_view().device_buffer()
        seav.device_buffer()[: src.numel()].copy_(src)
    else:
        det._materialize_into(seav)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    graphs: dict = {}
    cutoff = det.params.beta * det.params.theta
    fin = DeviceFinalize(seav, lview, det._params, det.ldca_config.k, cutoff, stream=side, graphs=graphs)
    m = fin.resolve()
    fin = DeviceFinalize(seav, lview, det._params, det.ldca_config.k, cutoff, stream=side, graphs=graphs)
    fin.resolve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(args.reps):
        e0.record(side)
        fin = DeviceFinalize(seav, lview, det._params, det.ldca_config.k, cutoff, stream=side, graphs=graphs)
        e1.record(side)
        fin.resolve()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    print(json.dumps({"slides_scanned": min(args.slides, n_sl), "reports": m, "candidates": fin.found,
                      "finalize_us_median": round(times[len(times) // 2], 2), "finalize_us_min": round(times[0], 2)}))


if __name__ == "__main__":
    main()
