"""Per-launch time of the partitioned scan on ONE small batch (a config-4
slice is ~1.8 M pairs), launches back to back (tuning probe, not a bench).

    [SSPD_B200_LIB=lib.so] python tools/slice_probe.py [--packets N] [--reps R] [--tag T] SETTING ...

A SETTING is `chunk=C` (packets per chunk; 0 = the whole batch as one chunk),
`fresh=1` (sspd_scan_partitioned_fresh: the fold stores into a zeroed
buffer, as a sliding slice's dirty bitmap) plus SSPD_* environment knobs, comma separated.  R launches of
sspd_scan_partitioned are issued on one stream between two CUDA events, so
the mean excludes host launch gaps; the LDCA/SEAV bytes of every setting are
compared with the first setting's.  Also prints the hash floor
(sspd_microbench_hash) at the same size.
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

    from paper_1901_07306_b200 import DetectorParams, DetectorState
    from paper_1901_07306_b200._abi import lib
    from tools.workloads import CONFIG2, generate

    ap = argparse.ArgumentParser()
    ap.add_argument("--packets", type=int, default=1_800_000)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--tag", default=os.environ.get("SSPD_B200_LIB", "default"))
    ap.add_argument("settings", nargs="*", default=["chunk=0"])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    hips, oips, _ = generate(CONFIG2, "torch", dev)
    n = args.packets
    hips, oips = hips[:n].contiguous(), oips[:n].contiguous()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=80.5e6))
    p = st.seav._params
    stream = torch.cuda.current_stream().cuda_stream
    sink = torch.empty(4096 * 148, dtype=torch.int32, device=dev)
    v = ctypes.c_double(0.0)
    lib().sspd_microbench_hash(hips.data_ptr(), oips.data_ptr(), n, p, 1, sink.data_ptr(), ctypes.byref(v), stream)
    floor_us = n / v.value * 1e6 if v.value else None
    seav = st.seav.device_buffer()
    ldca = st.ldca.device_buffer()
    ref = None
    for setting in args.settings:
        kv = dict(x.split("=", 1) for x in setting.split(",") if x)
        chunk = int(kv.pop("chunk", "0")) or (-(-n // 4) * 4)
        fresh = kv.pop("fresh", "0") == "1"  # sspd_scan_partitioned_fresh (a zeroed sliding dirty bitmap)
        old = {k: os.environ.get(k) for k in kv}
        os.environ.update(kv)
        try:
            need = int(lib().sspd_scan_partitioned_scratch(p, chunk))
            scratch = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)

            def launch():
                fn = lib().sspd_scan_partitioned_fresh if fresh else lib().sspd_scan_partitioned
                rc = fn(hips.data_ptr(), oips.data_ptr(), n, p, seav.data_ptr(), ldca.data_ptr(), scratch.data_ptr(),
                        need, chunk, stream)
                assert rc == 0, rc

            seav.zero_()
            ldca.zero_()
            launch()
            torch.cuda.synchronize()
            digest = hashlib.sha256(ldca.cpu().numpy().tobytes() + seav.cpu().numpy().tobytes()).hexdigest()[:16]
            ref = ref or digest
            for _ in range(3):
                launch()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                launch()
            b.record()
            b.synchronize()
            us = a.elapsed_time(b) * 1e3 / args.reps
        finally:
            for k, o in old.items():
                if o is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = o
        print(json.dumps({"tag": args.tag, "setting": setting, "packets": n, "chunk": chunk, "us_per_launch": round(us, 2),
                          "gpps": round(n / us / 1e3, 2), "hash_floor_us": round(floor_us, 2) if floor_us else None,
                          "bit_exact_vs_first": digest == ref}), flush=True)


if __name__ == "__main__":
    main()
