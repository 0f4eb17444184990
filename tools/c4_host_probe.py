"""Where a config-4 slide's time goes on the host (tuning probe, not a bench).

    python tools/c4_host_probe.py [--packets N] [--depth D]

Runs the bench's config-4 step (observe + detect_async + advance per slice,
lists consumed at the pipeline depth) once to warm up, then once more with
perf_counter around each host call, and prints one JSON line: the GPU time
of the step (CUDA events), the host wall time, and the host time per slide
of each call
(`finalize_wait`: inside DeviceFinalize.resolve, i.e. waiting for the GPU).  When the host's per-slide sum is close to the GPU's per-slide
time, the trace is launch/host bound rather than kernel bound.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_1901_07306_b200 import DetectorParams, SlidingDetector
    from tools.workloads import CONFIG4, CONFIG4_TIMING, TimingSpec, generate, scaled

    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=0)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--no-detect", action="store_true")
    ap.add_argument("--fine", action="store_true", help="time the sections of detect_async")
    ap.add_argument("--profile", default="", help="write cProfile stats of the timed step (top 60 by tottime)")
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
    if args.depth:
        det.pipeline_depth = args.depth
    acc = {"observe": 0.0, "detect_async": 0.0, "advance": 0.0, "resolve": 0.0, "finalize_wait": 0.0}
    from paper_1901_07306_b200 import window_detector as wd

    orig = wd.DeviceFinalize.resolve
    timing_on = [False]

    def timed_resolve(self):
        t0 = time.perf_counter()
        try:
            return orig(self)
        finally:
            if timing_on[0]:
                acc["finalize_wait"] += time.perf_counter() - t0

    wd.DeviceFinalize.resolve = timed_resolve
    fine = {}
    if args.fine:
        install_fine(det, fine, timing_on)

    def step(timed):
        det.reset()
        pending = []
        pc = time.perf_counter
        for s in range(n_sl):
            lo, hi = bounds[s], bounds[s + 1]
            t0 = pc()
            if hi > lo:
                det.observe_batch(hips[lo:hi], oips[lo:hi])
            t1 = pc()
            if not args.no_detect:
                pending.append(det.detect_async())
            t2 = pc()
            det.advance_slice()
            t3 = pc()
            while len(pending) > det.pipeline_depth:
                len(pending.pop(0))
            t4 = pc()
            if timed:
                acc["observe"] += t1 - t0
                acc["detect_async"] += t2 - t1
                acc["advance"] += t3 - t2
                acc["resolve"] += t4 - t3
        for r in pending:
            len(r)

    step(False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    timing_on[0] = True
    if args.profile:
        import cProfile
        import pstats

        prof = cProfile.Profile()
        prof.enable()
        step(True)
        prof.disable()
        with open(args.profile, "w") as f:
            pstats.Stats(prof, stream=f).sort_stats("tottime").print_stats(60)
            pstats.Stats(prof, stream=f).sort_stats("cumulative").print_stats(60)
    else:
        step(True)
    timing_on[0] = False
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    gpu_ms = e0.elapsed_time(e1)
    out = {"slides": n_sl, "packets": int(hips.numel()), "depth": det.pipeline_depth, "gpu_ms": round(gpu_ms, 3),
           "wall_ms": round(wall * 1e3, 3), "gpu_us_per_slide": round(gpu_ms * 1e3 / n_sl, 2),
           "host_us_per_slide": {k: round(v * 1e6 / n_sl, 2) for k, v in acc.items()},
           "host_busy_us_per_slide": round((acc["observe"] + acc["detect_async"] + acc["advance"] + acc["resolve"]
                                            - acc["finalize_wait"]) * 1e6 / n_sl, 2)}
    if fine:
        out["detect_async_sections_us"] = {k: round(v * 1e6 / n_sl, 2) for k, v in fine.items()}
    print(json.dumps(out))


def install_fine(det, fine, timing_on):
    """A copy of sliding.py's detect_async with perf_counter between its
    sections (keep in step with the library's)."""
    import types

    import torch

    from paper_1901_07306_b200 import sliding as sl
    from paper_1901_07306_b200._device import call, current_stream, stream_ptr, zeros_bytes
    from paper_1901_07306_b200.window_detector import DeviceFinalize, PendingReports

    def tick(name, t0):
        t1 = time.perf_counter()
        if timing_on[0]:
            fine[name] = fine.get(name, 0.0) + t1 - t0
        return t1

    def detect_async(self, beta=None):
        t = time.perf_counter()
        beta = self.params.beta if beta is None else beta
        cutoff = beta * self.params.theta
        st = sl._async_state(self)
        i = st["n"] % len(st["sets"])
        st["n"] += 1
        vset = st["sets"][i]
        if vset is None:
            vset = st["sets"][i] = [self.materialize_seav(), zeros_bytes(self._params.ldca_bytes), None, {}]
        elif vset[2] is not None:
            vset[2].resolve()
            t = tick("a_resolve", t)
            vset[2].detach()
        t = tick("b_detach", t)
        seav, lview = vset[0], vset[1]
        self._ldca_view_into(lview)
        t = tick("c_ldca_view", t)
        if self._iv() is not None:
            src = self._seav_view().device_buffer()
            t = tick("d_seav_view", t)
            dst = seav.device_buffer()
            call("sspd_copy_async", dst.data_ptr(), src.data_ptr(), src.numel() * src.element_size(), stream_ptr())
            t = tick("e_seav_copy", t)
        else:
            self._materialize_into(seav)
        views_ready = st.get("views_ready")
        if views_ready is None:
            views_ready = st["views_ready"] = torch.cuda.Event()
        views_ready.record(current_stream())
        side = st["side"]
        side.wait_event(views_ready)
        t = tick("f_events", t)
        graphs = vset[3] if self.finalize_graphs else None
        fin = DeviceFinalize(seav, lview, self._params, self.ldca_config.k, cutoff, stream=side, graphs=graphs)
        t = tick("g_finalize_launch", t)
        vset[2] = fin
        now = self.now
        pending = PendingReports(lambda: fin.reports(now, "sliding"))
        if fin.shared:
            import weakref

            fin.owner = weakref.ref(pending)
        tick("h_pending", t)
        return pending

    det.detect_async = types.MethodType(detect_async, det)


if __name__ == "__main__":
    main()
