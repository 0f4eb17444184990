import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
n = 1 << 28
B = 65536
rng = np.random.default_rng(1)
h = rng.integers(0, 2**32, size=n, dtype=np.uint32)
o = rng.integers(0, 2**32, size=n, dtype=np.uint32)
from paper_1901_07306_b200._abi import lib
import torch
L = lib()
ph = torch.empty(1 << 23, dtype=torch.int32, pin_memory=True)
po = torch.empty(1 << 23, dtype=torch.int32, pin_memory=True)
pa, pb = ph.data_ptr(), po.data_ptr()
L.sspd_host_pack_pairs(h.ctypes.data, o.ctypes.data, B, 4, 4, pa, pb)
t = time.perf_counter()
for lo in range(0, n, B):
    off = 4 * (lo % (1 << 23))
    L.sspd_host_pack_pairs(h.ctypes.data + 4 * lo, o.ctypes.data + 4 * lo, B, 4, 4, pa + off, pb + off)
dt = time.perf_counter() - t
print(json.dumps({"threads": L.sspd_host_copy_threads(), "us_per_call": dt / (n // B) * 1e6,
                  "GBps": 8 * n / dt / 1e9, "cpus": os.cpu_count()}))
