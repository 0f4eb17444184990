"""A/B of library builds on the config-2 window (tuning only, not a bench).

    SSPD_B200_LIB=path/to/lib.so python tools/ab_scan.py [--reps R] [--tag T]

Prints one JSON line: the hash floor (sspd_microbench_hash at 1 and 2 CTAs
per SM), the default scan's mean time over R launches (CUDA events, after a
warm-up) and the SHA-256 of the resulting SEAV + LDCA bytes, so two builds
can be compared for speed and checked for identical sketches.
"""
from __future__ import annotations

import argparse
import ctypes
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

    from paper_1901_07306_b200 import _abi
    if os.environ.get("AB_DROP_SYMS"):  # an older build without newer entry points
        for name in os.environ["AB_DROP_SYMS"].split(","):
            _abi._SIGS.pop(name, None)
    from paper_1901_07306_b200 import DetectorParams, DetectorState
    from paper_1901_07306_b200._abi import lib
    from tools.workloads import CONFIG2, generate

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--tag", default=os.environ.get("SSPD_B200_LIB", "default"))
    ap.add_argument("--packets", type=int, default=0, help="scan only the first N pairs (e.g. a config-4 slice)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    hips, oips, _ = generate(CONFIG2, "torch", dev)
    if args.packets:
        hips, oips = hips[:args.packets].contiguous(), oips[:args.packets].contiguous()
    n = int(hips.numel())
    dp = DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=80.5e6)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(dp)
    st.partitioned_min_packets = 1  # the partitioned scan at any size
    sink = torch.empty(4096 * 148, dtype=torch.int32, device=dev)
    floor = {}
    for bps in (1, 2):
        v = ctypes.c_double(0.0)
        rc = lib().sspd_microbench_hash(hips.data_ptr(), oips.data_ptr(), n, st.seav._params, bps, sink.data_ptr(),
                                        ctypes.byref(v), torch.cuda.current_stream().cuda_stream)
        floor[bps] = round(v.value / 1e9, 3) if rc == 0 else None
    st.process_batch(hips, oips)
    torch.cuda.synchronize()
    digest = hashlib.sha256(st.ldca.payload_bytes() + st.seav.payload_bytes()).hexdigest()[:16]
    times = []
    for _ in range(args.reps):
        st.reset()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.process_batch(hips, oips)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
    ms = sum(times) / len(times)
    print(json.dumps({"tag": args.tag, "scan": getattr(st, "last_scan", None), "scan_ms": round(ms, 4),
                      "scan_gpps": round(n / ms / 1e6, 3), "min_ms": round(min(times), 4),
                      "hash_floor_gpps": floor, "digest": digest}), flush=True)


if __name__ == "__main__":
    main()
