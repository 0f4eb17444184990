"""Drop-in call pattern probe (tuning only): one config-2-sized window fed as
65,536-pair numpy process_batch calls, as the reference CLI does
(cli.py:215-217).  Prints the staging copy's own rate (pack only) and the
whole pattern (process_batch x calls + finalize_window + reset), for the
host-copy knobs in the environment (SSPD_HOST_COPY_THREADS, SSPD_HOST_COPY_NT).
"""
import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.getcwd())


def main():
    import numpy as np
    import torch

    from paper_1901_07306_b200 import DetectorParams, DetectorState
    from paper_1901_07306_b200._abi import lib

    n, B = 1 << 28, 65536
    rng = np.random.default_rng(1)
    h = rng.integers(0, 2**32, size=n, dtype=np.uint32)
    o = rng.integers(0, 2**32, size=n, dtype=np.uint32)
    L = lib()
    cap = 1 << 23
    ph = torch.empty(cap, dtype=torch.int32, pin_memory=True)
    po = torch.empty(cap, dtype=torch.int32, pin_memory=True)
    pa, pb = ph.data_ptr(), po.data_ptr()
    L.sspd_host_pack_pairs(h.ctypes.data, o.ctypes.data, B, 4, 4, pa, pb)
    t = time.perf_counter()
    for lo in range(0, n, B):
        off = 4 * (lo % cap)
        L.sspd_host_pack_pairs(h.ctypes.data + 4 * lo, o.ctypes.data + 4 * lo, B, 4, 4, pa + off, pb + off)
    pack_s = time.perf_counter() - t
    if os.environ.get("SSPD_PROBE_STAGE_PAIRS"):  # pinned staging size (pairs) per buffer
        DetectorState.host_stage_pairs = int(os.environ["SSPD_PROBE_STAGE_PAIRS"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(DetectorParams(theta=1024, r=12, k=8192, lr=8, lc=1024, design_n=80.5e6))

    def step():
        for lo in range(0, n, B):
            st.process_batch(h[lo:lo + B], o[lo:lo + B])
        st.finalize_window()
        st.reset()

    step()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        step()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    # python-side cost of one call alone (staging disabled: no copy, no scan)
    print(json.dumps({"threads": L.sspd_host_copy_threads(), "nt": os.environ.get("SSPD_HOST_COPY_NT", "default"),
                      "stage_pairs": DetectorState.host_stage_pairs,
                      "pack_gbs": round(8 * n / pack_s / 1e9, 2), "pack_us_per_call": round(pack_s / (n // B) * 1e6, 2),
                      "dropin_gpps": round(n / best / 1e9, 3), "dropin_ms": round(best * 1e3, 2),
                      "cpus": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    main()
