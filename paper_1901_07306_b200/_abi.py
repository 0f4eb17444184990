"""ctypes mirror of include/sspd_b200.h and the library loader.

The product path calls the CUDA library ONLY through these bindings.  If the
shared library is missing or cannot be loaded the import of the
device-backed classes fails loudly (DeviceError) -- there is no CPU
fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, DataError, DeviceError, SspdError

MAX_SR = 16
MAX_LR = 64
LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsspd_b200.so"

OK, ERR_CONFIG, ERR_DATA, ERR_CUDA, ERR_CAPACITY = 0, 2, 3, 4, 5


class Divisor_t(C.Structure):
    _fields_ = [("d", C.c_uint64), ("magic", C.c_uint64), ("sh1", C.c_uint32),
                ("sh2", C.c_uint32), ("pow2", C.c_uint32), ("pad_", C.c_uint32)]


class Params_t(C.Structure):
    _fields_ = [
        ("seed_h1", C.c_uint64), ("seed_h2", C.c_uint64), ("seed_h3", C.c_uint64),
        ("seed_route", C.c_uint64), ("seed_lh", C.c_uint64 * MAX_LR),
        ("r", C.c_uint32), ("sr", C.c_uint32), ("a", C.c_uint32), ("g", C.c_uint32),
        ("addr_bits", C.c_uint32), ("lp_bits", C.c_uint32), ("tau", C.c_uint32),
        ("reg_bytes", C.c_uint32),
        ("isb", C.c_uint32 * MAX_SR), ("ibn", C.c_uint32 * MAX_SR), ("sc", C.c_uint32 * MAX_SR),
        ("seav_row_off", C.c_uint64 * MAX_SR), ("seav_bytes", C.c_uint64),
        ("lr", C.c_uint32), ("lc", C.c_uint32), ("k", C.c_uint32), ("pad0_", C.c_uint32),
        ("ldca_bytes", C.c_uint64),
        ("div_g", Divisor_t), ("div_k", Divisor_t), ("div_lc", Divisor_t),
        ("slot_row_base", C.c_uint64 * MAX_SR), ("slot_ldca_base", C.c_uint64),
        ("slot_total", C.c_uint64),
    ]


def divisor_t(div) -> Divisor_t:
    return Divisor_t(div.d, div.magic, div.sh1, div.sh2, div.pow2, 0)


def build_params(seav_cfg, ldca_cfg, seeds) -> Params_t:
    """Resolve the POD parameter block from the drop-in config objects."""
    from .hashing import Divisor

    if seav_cfg.sr > MAX_SR:
        raise ConfigError(f"SR={seav_cfg.sr} exceeds the {MAX_SR} rows the kernels implement")
    if ldca_cfg.lr > MAX_LR:
        raise ConfigError(f"LR={ldca_cfg.lr} exceeds the {MAX_LR} rows the kernels implement")
    if max(seav_cfg.ibn) > 16:
        raise ConfigError("SEAV index width above 16 bits is not implemented on the device")
    p = Params_t()
    p.seed_h1 = seeds.h1.value
    p.seed_h2 = seeds.h2.value
    p.seed_h3 = seeds.h3.value
    p.seed_route = seeds.route.value
    for i in range(ldca_cfg.lr):
        p.seed_lh[i] = seeds.lh(i).value
    w = seav_cfg.lp_bits
    p.r, p.sr, p.a, p.g = seav_cfg.r, seav_cfg.sr, seav_cfg.a, seav_cfg.g
    p.addr_bits, p.lp_bits, p.tau = seav_cfg.addr_bits, w, seav_cfg.tau
    p.reg_bytes = seav_cfg.register_bytes
    off = 0
    slot = 0
    for i in range(seav_cfg.sr):
        p.isb[i] = seav_cfg.isb[i] % w
        p.ibn[i] = seav_cfg.ibn[i]
        p.sc[i] = seav_cfg.sc[i]
        p.seav_row_off[i] = off
        p.slot_row_base[i] = slot
        off += (1 << seav_cfg.r) * seav_cfg.sc[i] * p.reg_bytes
        slot += (1 << seav_cfg.r) * seav_cfg.sc[i] * seav_cfg.g
    p.seav_bytes = off
    p.lr, p.lc, p.k = ldca_cfg.lr, ldca_cfg.lc, ldca_cfg.k
    p.ldca_bytes = ldca_cfg.lr * ldca_cfg.lc * ldca_cfg.k // 8
    p.div_g = divisor_t(Divisor.of(seav_cfg.g))
    p.div_k = divisor_t(Divisor.of(ldca_cfg.k))
    p.div_lc = divisor_t(Divisor.of(ldca_cfg.lc))
    p.slot_ldca_base = slot
    p.slot_total = slot + ldca_cfg.lr * ldca_cfg.lc * ldca_cfg.k
    return p


_VP = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32
_PP = C.POINTER(Params_t)
_SIGS = {
    "sspd_abi_version": (C.c_int, []),
    "sspd_params_size": (C.c_size_t, []),
    "sspd_device_sm_count": (C.c_int, [C.c_int]),
    "sspd_hash_range_host": (_U64, [_U64, _U64, C.POINTER(Divisor_t)]),
    "sspd_mix64_host": (_U64, [_U64]),
    "sspd_scan_discrete": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _VP, _VP]),
    "sspd_scan_partitioned": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "sspd_scan_partitioned_fresh": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "sspd_scan_partitioned_scratch": (_U64, [_PP, _U64]),
    "sspd_scan_partitioned_variant": (C.c_int, [_PP, _U64]),
    "sspd_host_check_u32": (C.c_int, [_VP, _U64, _U32, C.c_int]),
    "sspd_host_pack_u32": (C.c_int, [_VP, _U64, _U32, C.c_int, _VP]),
    "sspd_host_pack_pairs": (C.c_int, [_VP, _VP, _U64, _U32, _U32, _VP, _VP]),
    "sspd_host_copy_threads": (C.c_int, []),
    "sspd_scan_sliding": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _U32, _U64, _VP]),
    "sspd_scan_sliding_capped": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _U32, _U64, _U32, _VP]),
    "sspd_scan_sliding_tracked": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _U32, _U64, _U32, _VP, _VP, _U64, _VP, _VP]),
    "sspd_seav_advance": (C.c_int, [_VP, _U32, _PP, _VP, _VP, _U64, _VP, _U32, _U64, _U64, _VP]),
    "sspd_materialize_seav_if": (C.c_int, [_VP, _U32, _PP, _U64, _U64, _VP, _VP, _VP]),
    "sspd_sweep": (C.c_int, [_VP, _U64, _U32, _U64, _U64, _U64, _VP]),
    "sspd_touch_slots": (C.c_int, [_VP, _U64, _U32, _VP, _U64, _U64, _VP, _VP]),
    "sspd_materialize_seav": (C.c_int, [_VP, _U32, _PP, _U64, _U64, _VP, _VP]),
    "sspd_materialize_ldca": (C.c_int, [_VP, _U32, _PP, _U64, _U64, _VP, _VP]),
    "sspd_scan_sliding_deferred": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _U32, _U64, _U32, _VP, _VP, _U64, _VP, _VP,
                                             _VP]),
    "sspd_scan_sliding_seav": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _U32, _U64, _U32, _VP, _VP, _U64, _VP, _VP]),
    "sspd_scan_sliding_partitioned": (C.c_int, [_VP, _VP, _U64, _PP, _VP, _U32, _U64, _VP, _VP, _U64, _VP, _VP,
                                                C.c_int, _VP, _U64, _U64, _VP]),
    "sspd_ldca_fold": (C.c_int, [_VP, _U32, _PP, _VP, _U64, _U64, _VP, _VP]),
    "sspd_ldca_window_or": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _VP]),
    "sspd_ldca_fold_ring": (C.c_int, [_VP, _U32, _PP, _VP, _U64, _U32, _U64, _U64, _VP]),
    "sspd_ldca_suffix_or": (C.c_int, [_VP, _U32, _U64, _U64, _U64, _VP]),
    "sspd_pool_ages": (C.c_int, [_VP, _U64, _U32, _U64, _VP, _VP]),
    "sspd_restore": (C.c_int, [_VP, _PP, _U32, _U32, _U64, _VP, _VP, _U64, _VP, _VP, _VP]),
    "sspd_sort_candidates": (C.c_int, [_VP, _VP, _U64, _VP, C.POINTER(C.c_size_t), _VP]),
    "sspd_filter": (C.c_int, [_VP, _PP, _VP, _U64, _VP, _VP, _VP, _VP]),
    "sspd_filter_sliding": (C.c_int, [_VP, _U32, _PP, _U64, _U64, _VP, _U64, _VP, _VP, _VP, _VP]),
    "sspd_compact_reports": (C.c_int, [_VP, _VP, _VP, _U64, _VP, _VP, _VP, _VP, C.POINTER(C.c_size_t), _VP]),
    "sspd_merge_or": (C.c_int, [C.POINTER(_VP), C.c_int, _VP, _U64, _VP]),
    "sspd_merge_age_min": (C.c_int, [C.POINTER(_VP), C.c_int, _VP, _U64, _U32, _U64, _VP]),
    "sspd_route_pairs": (C.c_int, [_VP, _VP, _U64, _PP, C.POINTER(Divisor_t), C.c_int, _U64, _VP, _VP]),
    "sspd_microbench_red": (C.c_int, [_VP, _U64, C.c_int, C.c_int, C.POINTER(C.c_double), _VP]),
    "sspd_microbench_hash": (C.c_int, [_VP, _VP, _U64, _PP, C.c_int, _VP, C.POINTER(C.c_double), _VP]),
    "sspd_check_hash32": (C.c_int, [_U64, _U64, _U64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _VP]),
    "sspd_microbench_store16": (C.c_int, [_VP, _U64, C.c_int, C.c_int, C.POINTER(C.c_double), _VP]),
    "sspd_ipc_alloc": (C.c_int, [_U64, C.POINTER(_VP)]),
    "sspd_ipc_free": (C.c_int, [_VP]),
    "sspd_ipc_get_handle": (C.c_int, [_VP, C.c_char_p]),
    "sspd_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(_VP)]),
    "sspd_ipc_close": (C.c_int, [_VP]),
    "sspd_copy_async": (C.c_int, [_VP, _VP, _U64, _VP]),
    "sspd_unpack_records": (C.c_int, [_VP, _U64, _VP, _VP, _VP, _VP]),
    "sspd_crc32": (C.c_int, [_VP, _U64, _VP, _VP, C.POINTER(_U64), _VP]),
    "sspd_finalize": (C.c_int, [_VP, _VP, _PP, _U64, _VP, _U64, _VP, _VP, _VP, _VP, _VP, C.POINTER(C.c_size_t),
                                _U32, _VP]),
    "sspd_exact_cardinalities": (C.c_int, [_VP, _VP, _U64, _VP, _VP, _VP, _VP, C.POINTER(C.c_size_t), _VP]),
}

_lib = None


def lib():
    """Load libsspd_b200.so once; raise DeviceError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("SSPD_B200_LIB", LIB_PATH))
    if not path.exists():
        raise DeviceError(
            f"{path} is missing: build it with `python -m paper_1901_07306_b200.build` "
            "(there is no CPU fallback)")
    handle = C.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.sspd_abi_version() != 1:
        raise DeviceError("libsspd_b200.so ABI version mismatch")
    if handle.sspd_params_size() != C.sizeof(Params_t):
        raise DeviceError(
            f"sspd_params layout mismatch: C {handle.sspd_params_size()} vs ctypes {C.sizeof(Params_t)}")
    _lib = handle
    return _lib


def check(rc: int, what: str):
    """Map a C-ABI status onto the reference exception classes."""
    if rc == OK:
        return
    if rc == ERR_CONFIG:
        raise ConfigError(f"{what}: configuration rejected by the device library")
    if rc == ERR_DATA:
        raise DataError(f"{what}: invalid data/buffer")
    if rc == ERR_CUDA:
        raise DeviceError(f"{what}: CUDA launch failed")
    raise SspdError(f"{what}: status {rc}")
