"""ctypes front-end of the CPU oracle (oracle/sspd_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs as the checker / CPU baseline; never by the product
package.  Functions mirror the reference (file:line in sspd_oracle.c) and
take numpy arrays plus the product's POD parameter block (pure data).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_lib = None


def build():
    src = HERE / "sspd_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        from paper_1901_07306_b200._abi import Params_t

        L = C.CDLL(str(LIB))
        P = C.POINTER(Params_t)
        vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
        sigs = {
            "or_mix64": (u64, [u64]),
            "or_derive_seed": (u64, [u64, u32]),
            "or_hash_range": (u64, [u64, u64, u64]),
            "or_seav_update": (None, [P, vp, vp, u64, vp]),
            "or_ldca_update": (None, [P, vp, vp, u64, vp]),
            "or_scan": (C.c_int, [P, vp, vp, u64, vp, vp, C.c_int]),
            "or_restore": (C.c_int64, [P, vp, u32, u32, u64, vp, vp, u64, vp]),
            "or_filter": (None, [P, vp, vp, u64, vp]),
            "or_restore_mt": (C.c_int64, [P, vp, u32, u32, u64, vp, vp, u64, vp, C.c_int]),
            "or_filter_mt": (None, [P, vp, vp, u64, vp, C.c_int]),
            "or_observe": (None, [P, vp, vp, u64, vp, u32, u64]),
            "or_sweep": (None, [vp, u64, u32, u64, u64, u64]),
            "or_materialize_seav": (None, [P, vp, u32, u64, u64, vp]),
            "or_materialize_ldca": (None, [P, vp, u32, u64, u64, vp]),
            "or_merge_age_min": (None, [C.POINTER(vp), C.c_int, vp, u64, u32, u64]),
            "or_route_hash": (None, [vp, vp, u64, u64, u64, vp]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _u32(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.uint32:
        a = a.astype(np.uint32)
    return np.ascontiguousarray(a)


def _p(a) -> int:
    return a.ctypes.data


def mix64(x: int) -> int:
    return lib().or_mix64(x)


def derive_seed(master: int, tag: int) -> int:
    return lib().or_derive_seed(master, tag)


def hash_range(key: int, seed: int, m: int) -> int:
    return lib().or_hash_range(key, seed, m)


def scan(params, hips, oips, seav: np.ndarray | None = None, ldca: np.ndarray | None = None,
         threads: int = 1):
    """SEAV/LDCA bytes after process_batch(hips, oips) (window_detector.py:100-103)."""
    h, o = _u32(hips), _u32(oips)
    if seav is None:
        seav = np.zeros(params.seav_bytes, dtype=np.uint8)
    if ldca is None:
        ldca = np.zeros(params.ldca_bytes, dtype=np.uint8)
    lib().or_scan(params, _p(h), _p(o), len(h), _p(seav), _p(ldca), threads)
    return seav, ldca


def restore(params, seav: np.ndarray, cap: int, rp_begin: int = 0, rp_count: int | None = None,
            threads: int = 1):
    """(ips, rps, weights, overflow[rp]) sorted by ip (short_sketch.py:347-408);
    `threads` > 1 restores ranges of SEAs concurrently (same result)."""
    if rp_count is None:
        rp_count = 1 << params.r
    seav = np.ascontiguousarray(seav, dtype=np.uint8)
    over = np.zeros(max(1, rp_count), dtype=np.uint8)
    capacity = 1 << 12
    while True:
        ips = np.zeros(capacity, dtype=np.uint32)
        aux = np.zeros(capacity, dtype=np.uint32)
        n = lib().or_restore_mt(params, _p(seav), rp_begin, rp_count, cap, _p(ips), _p(aux), capacity, _p(over),
                                threads)
        if n <= capacity:
            break
        capacity = n
    return ips[:n], aux[:n] >> 8, aux[:n] & 0xFF, over[:rp_count]


def filter_z0(params, ldca: np.ndarray, ips, threads: int = 1) -> np.ndarray:
    ips = _u32(ips)
    z0 = np.zeros(max(1, len(ips)), dtype=np.uint32)
    lib().or_filter_mt(params, _p(np.ascontiguousarray(ldca, dtype=np.uint8)), _p(ips), len(ips), _p(z0), threads)
    return z0[: len(ips)]


def observe(params, hips, oips, pool: np.ndarray, now_wrapped: int):
    h, o = _u32(hips), _u32(oips)
    lib().or_observe(params, _p(h), _p(o), len(h), _p(pool), pool.dtype.itemsize, now_wrapped)


def sweep(pool: np.ndarray, now_wrapped: int, window: int, clamp: int):
    lib().or_sweep(_p(pool), len(pool), pool.dtype.itemsize, now_wrapped, window, clamp)


def materialize_seav(params, pool: np.ndarray, now_wrapped: int, window: int) -> np.ndarray:
    out = np.zeros(params.seav_bytes, dtype=np.uint8)
    lib().or_materialize_seav(params, _p(pool), pool.dtype.itemsize, now_wrapped, window, _p(out))
    return out


def materialize_ldca(params, pool: np.ndarray, now_wrapped: int, window: int) -> np.ndarray:
    out = np.zeros(params.ldca_bytes, dtype=np.uint8)
    lib().or_materialize_ldca(params, _p(pool), pool.dtype.itemsize, now_wrapped, window, _p(out))
    return out


def merge_age_min(pools: list[np.ndarray], now_wrapped: int) -> np.ndarray:
    out = np.empty_like(pools[0])
    arr = (C.c_void_p * len(pools))(*[_p(p) for p in pools])
    lib().or_merge_age_min(arr, len(pools), _p(out), len(out), out.dtype.itemsize, now_wrapped)
    return out


def route_hash(hips, oips, seed_route: int, n_wp: int) -> np.ndarray:
    h, o = _u32(hips), _u32(oips)
    lanes = np.zeros(max(1, len(h)), dtype=np.int64)
    lib().or_route_hash(_p(h), _p(o), len(h), seed_route, n_wp, _p(lanes))
    return lanes[: len(h)]


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def exact_cardinalities(hips, oips) -> tuple[np.ndarray, np.ndarray]:
    """ExactOracle.__init__ (evaluation.py:35-40) restated with numpy:
    sort-unique of (hip << 32 | oip), then distinct keys per host.
    Returns (hosts uint32 ascending, counts int64)."""
    key = (_u32(hips).astype(np.uint64) << np.uint64(32)) | _u32(oips).astype(np.uint64)
    distinct = np.unique(key)
    hosts, counts = np.unique(distinct >> np.uint64(32), return_counts=True)
    return hosts.astype(np.uint32), counts.astype(np.int64)
