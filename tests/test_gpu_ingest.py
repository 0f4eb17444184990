"""Device trace ingest (12-byte reference records) and the device CRC-32
used to seal frames, against numpy / zlib."""

import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 7, 4095, 4096, 4097, 8191, 65536 * 3 + 5, 8 * (1 << 20), 8 * (1 << 20) + 13])
def test_device_crc32_matches_zlib(cuda, n):
    import torch

    from paper_1901_07306_b200.ingest import device_crc32

    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, size=n, dtype=np.uint8)
    buf = torch.from_numpy(data).cuda()
    assert device_crc32(buf) == zlib.crc32(data.tobytes())
    if n > 3:  # unaligned start
        assert device_crc32(buf[3:]) == zlib.crc32(data[3:].tobytes())


def test_crc32_combine_host():
    from paper_1901_07306_b200.ingest import crc32_combine

    rng = np.random.default_rng(1)
    for la, lb in [(0, 0), (1, 0), (0, 5), (40, 32768), (7, 1 << 20)]:
        a = rng.integers(0, 256, size=la, dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, size=lb, dtype=np.uint8).tobytes()
        assert crc32_combine(zlib.crc32(a), zlib.crc32(b), lb) == zlib.crc32(a + b)


def test_unpack_records_and_trace_file(cuda, tmp_path):
    from paper_1901_07306_b200.ingest import read_trace_device, unpack_records

    rng = np.random.default_rng(2)
    n = 100_003
    rec = np.empty(n, dtype=[("slice", "<u4"), ("hip", "<u4"), ("oip", "<u4")])
    rec["slice"] = rng.integers(0, 300, n)
    rec["hip"] = rng.integers(0, 2**32, n, dtype=np.uint64)
    rec["oip"] = rng.integers(0, 2**32, n, dtype=np.uint64)
    for got in (unpack_records(rec), unpack_records(rec.tobytes())):
        s, h, o = (t.cpu().numpy().view(np.uint32) for t in got)
        assert (s == rec["slice"]).all() and (h == rec["hip"]).all() and (o == rec["oip"]).all()
    path = tmp_path / "t.bin"
    path.write_bytes(rec.tobytes())
    s, h, o = (t.cpu().numpy().view(np.uint32) for t in read_trace_device(path))
    assert (h == rec["hip"]).all()
    path.write_bytes(rec.tobytes()[:-1])
    from paper_1901_07306_b200 import DataError

    with pytest.raises(DataError):
        read_trace_device(path)
