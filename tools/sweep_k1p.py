"""Tuning sweep of the partitioned scan (K1p) knobs on one config-2 window.

    python tools/sweep_k1p.py [--packets N] [--reps R] KEY=V[,KEY=V...] ...

Each argument is one setting ("direct" = the L2-red kernel K1, a
reference for the bytes) of SSPD_PART_* environment knobs (read by the
library at launch); the stream is generated once on the GPU.  For every
setting the scan is timed with CUDA events (mean of R launches after one
warm-up) and its LDCA/SEAV bytes are compared with the first setting's, so a
knob can never trade correctness for speed.  Prints one JSON line per
setting.  Not a bench number (no finalize, no clocks check): tuning only.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_1901_07306_b200 import DetectorParams, DetectorState
    from tools.workloads import CONFIG2, generate, scaled

    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("settings", nargs="*", default=[""])
    args = ap.parse_args()
    spec = CONFIG2 if not args.packets else scaled(CONFIG2, max(1, CONFIG2.n_packets // args.packets))
    dev = torch.device("cuda", 0)
    hips, oips, _ = generate(spec, "torch", dev)
    n = int(hips.numel())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=80.5e6))
    st.scan_mode = "partitioned"
    ref = None
    for setting in args.settings:
        st.scan_mode = "direct" if setting == "direct" else "partitioned"
        env = {} if setting == "direct" else dict(kv.split("=", 1) for kv in setting.split(",") if kv)
        st.partitioned_chunk = int(env.pop("chunk", 0))  # packets per chunk (0 = library default)
        for k in [k for k in os.environ if k.startswith(("SSPD_PART_", "SSPD_BPART_"))]:
            del os.environ[k]
        os.environ.update(env)
        st.reset()
        st.process_batch(hips, oips)  # warm-up (and correctness sample)
        torch.cuda.synchronize()
        digest = hashlib.sha256(st.ldca.payload_bytes() + st.seav.payload_bytes()).hexdigest()
        ref = ref or digest
        times = []
        for _ in range(args.reps):
            st.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            st.process_batch(hips, oips)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = sum(times) / len(times)
        print(json.dumps({"setting": env, "scan_ms": round(ms, 4), "min_ms": round(min(times), 4),
                          "gpps": round(n / ms / 1e6, 3), "bit_exact_vs_first": digest == ref,
                          "last_scan": st.last_scan}), flush=True)


if __name__ == "__main__":
    main()
