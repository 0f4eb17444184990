"""CPU-only checks: the C-ABI library loads and exports what the header
declares, the host-side logic (configs, planner, hashing, divisors,
frames) matches the reference's golden vectors.  No kernel launches."""

import re
import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "sspd_b200.h").read_text()
    return sorted(set(re.findall(r"SSPD_API\s+[\w\s\*]+?\b(sspd_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1901_07306_b200 import _abi

    lib = _abi.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(_abi._SIGS) == set(names)
    assert lib.sspd_abi_version() == 1
    assert lib.sspd_params_size() == __import__("ctypes").sizeof(_abi.Params_t)


def test_device_modulo_matches_reference_hash_range(golden):
    """sspd_hash_range_host runs the kernels' fast-modulo code on the host."""
    import ctypes

    from paper_1901_07306_b200 import _abi
    from paper_1901_07306_b200.hashing import Divisor, SeedFamily

    lib = _abi.lib()
    s = SeedFamily()
    for k, m, v in golden["hash"]["hash_range"]:
        d = _abi.divisor_t(Divisor.of(m))
        assert lib.sspd_hash_range_host(k, s.h3.value, ctypes.byref(d)) == v
    for k, m, v in golden["hash"]["hash_range_random"]:
        d = _abi.divisor_t(Divisor.of(m))
        assert lib.sspd_hash_range_host(k, s.lh(3).value, ctypes.byref(d)) == v
    for k, v in golden["hash"]["mix64"]:
        assert lib.sspd_mix64_host(k) == v


def test_divisor_exhaustive_edges():
    from paper_1901_07306_b200.hashing import Divisor

    rng = np.random.default_rng(0)
    xs = [0, 1, 2**32 - 1, 2**32, 2**63, 2**64 - 1, 2**64 - 2] + rng.integers(0, 2**64, 400, dtype=np.uint64).tolist()
    ds = list(range(1, 300)) + [2**31 - 1, 2**31 + 1, 2**32 - 1, 2**32 - 5, 3 * 2**30, 1000, 8191, 174]
    for d in ds:
        dv = Divisor.of(d)
        for x in xs:
            assert dv.mod(int(x)) == int(x) % d, (x, d)


def test_hash_family_golden(golden):
    from paper_1901_07306_b200.hashing import SeedFamily, derive_seed, hash_full, hash_range, lsb, mix64

    h = golden["hash"]
    for k, v in h["mix64"]:
        assert mix64(k) == v
    for m, t, v in h["derive_seed"]:
        assert derive_seed(m, t) == v
    s = SeedFamily()
    for k, m, v in h["hash_range"]:
        assert hash_range(k, s.h3, m) == v
    for k, v in h["hash_full_h1"]:
        assert hash_full(k, s.h1) == v
    assert [lsb(x) for x in (0, 1, 2, 8, 0x80000000, 12)] == [32, 0, 1, 3, 31, 2]


def test_geometry_golden(golden):
    from paper_1901_07306_b200 import ConfigError, SeavConfig, plan_rows, tau_from_theta
    from paper_1901_07306_b200.sliding import timestamp_dtype

    g = golden["geometry"]
    for c in g["seav"]:
        kw = {k: c[k] for k in ("r", "sr", "a", "g", "addr_bits", "theta")}
        if "error" in c:
            with pytest.raises(ConfigError) as e:
                SeavConfig(**kw)
            assert str(e.value) == c["error"]
        else:
            cfg = SeavConfig(**kw)
            assert (list(cfg.isb), list(cfg.ibn), list(cfg.sc), cfg.tau, cfg.memory_bytes()) == (
                c["isb"], c["ibn"], c["sc"], c["tau"], c["memory_bytes"])
    for t, gg, v in g["tau"]:
        assert tau_from_theta(t, gg) == v
    for v, n, k, mr, out in g["plan_rows"]:
        assert list(plan_rows(v, n, k, max_rows=mr)) == out
    for w, name in g["timestamp_dtype"]:
        assert np.dtype(timestamp_dtype(w)).name == name


def test_index_round_trip():
    from paper_1901_07306_b200 import make_config

    for cfg in (make_config(), make_config(r=2, sr=5, a=1), make_config(r=12), make_config(r=16)):
        rng = np.random.default_rng(101)
        for lp in rng.integers(0, 1 << cfg.lp_bits, size=2000, dtype=np.uint64).tolist():
            idx = [cfg.index_of(i, lp) for i in range(cfg.sr)]
            assert cfg.lp_from_indexes(idx) == lp
            for i in range(cfg.sr):  # bit j of col = LP bit (isb+j) % w (short_sketch.py:183-193)
                ref = sum(((lp >> ((cfg.isb[i] + j) % cfg.lp_bits)) & 1) << j for j in range(cfg.ibn[i]))
                assert idx[i] == ref


def test_index_of_array_vectorised_matches_scalar():
    """index_of_array (short_sketch.py:196-205) is the scalar map over an
    array, any integer dtype and shape; out-of-range LP bits are masked."""
    from paper_1901_07306_b200 import make_config

    for cfg in (make_config(), make_config(r=2, sr=5, a=1), make_config(r=12), make_config(r=16)):
        rng = np.random.default_rng(7)
        lp = rng.integers(0, 1 << 40, size=(40, 25), dtype=np.uint64)
        for i in range(cfg.sr):
            got = cfg.index_of_array(i, lp)
            assert got.shape == lp.shape and got.dtype == np.uint64
            assert got.reshape(-1).tolist() == [cfg.index_of(i, int(x)) for x in lp.reshape(-1).tolist()]
            assert cfg.index_of_array(i, lp.astype(np.int64)).tolist() == got.tolist()
        with pytest.raises(Exception):
            cfg.index_of_array(cfg.sr, lp)


def test_ldc_estimate_and_keep_table():
    import math

    from paper_1901_07306_b200 import ConfigError, ldc_estimate
    from paper_1901_07306_b200.long_sketch import keep_table

    assert ldc_estimate(1024, 1024) == (0.0, False) or ldc_estimate(1024, 1024)[0] == 0.0
    assert ldc_estimate(512, 1024)[0] == pytest.approx(709.78, abs=0.01)
    assert ldc_estimate(0, 8192) == (8192 * math.log(8192), True)
    with pytest.raises(ConfigError):
        ldc_estimate(1025, 1024)
    t = keep_table(8192, 0.8 * 1024)
    # the reference's float cut falls between z0=7412 and 7413
    assert t[0] == 1 and t[1:7413].all() and not t[7413:].any()


def test_frame_parse_errors_host_only():
    from paper_1901_07306_b200 import (FrameChecksumError, FrameMagicError, FrameTruncatedError,
                                       FrameVersionError, parse_frame)

    payload = bytes(range(256)) * 4
    cfg = struct.pack("<BBBBIIHIQ", 0, 0, 0, 0, 0, 4096, 2, 64, 0x5EED)
    body = struct.pack("<4sBB", b"SSPD", 1, 1) + cfg + struct.pack("<II", 7, len(payload)) + payload
    blob = body + struct.pack("<I", zlib.crc32(body))
    f = parse_frame(blob)
    assert (f.kind, f.window_id, f.payload, f.kind_name) == (1, 7, payload, "ldca")
    with pytest.raises(FrameMagicError):
        parse_frame(b"NOPE" + blob[4:])
    with pytest.raises(FrameVersionError):
        parse_frame(blob[:4] + b"\x09" + blob[5:])
    with pytest.raises(FrameTruncatedError):
        parse_frame(blob[: len(blob) // 2])
    with pytest.raises(FrameTruncatedError):
        parse_frame(blob + b"\x00")
    with pytest.raises(FrameTruncatedError):
        parse_frame(blob[:10])
    bad = bytearray(blob)
    bad[100] ^= 0x40
    with pytest.raises(FrameChecksumError):
        parse_frame(bytes(bad))


def test_workload_generator_backends_agree():
    import torch

    from tools.workloads import CONFIG2, generate, scaled

    spec = scaled(CONFIG2, 256)
    h, o, s = generate(spec)
    h2, o2, s2 = generate(spec, "torch", "cpu")
    assert (h2.numpy().view(np.uint32) == h).all() and (o2.numpy().view(np.uint32) == o).all()
    assert len(h) == spec.n_packets and (s == s2).all()
    key = np.unique((h.astype(np.uint64) << np.uint64(32)) | o)
    hosts, counts = np.unique(key >> np.uint64(32), return_counts=True)
    assert len(hosts) == spec.n_sources
    assert set(s.tolist()) <= set(hosts[counts >= 1500].tolist())
    del torch
