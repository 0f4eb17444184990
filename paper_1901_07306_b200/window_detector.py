"""Discrete-window detector: one SEAV + one LDCA per window, on one GPU.

Mirrors `sspd/window_detector.py` (DetectorParams :39-69, DetectorState
:72-132).  The B200 differences:

* `process_batch` is ONE fused scan kernel (K1) that updates both sketches
  from one pass over the (hip, oip) stream -- the reference makes two
  passes (SEAV then LDCA, window_detector.py:100-103).
* `finalize_window` runs restore (K5), the device sort, the z0 filter (K6)
  with the keep decision as an integer table lookup, and a stable
  compaction on the device; only the kept (ip, z0) pairs come back to the
  host, where the float estimate is formed with the reference formula.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from .hashing import DEFAULT_MASTER_SEED, SeedFamily
from .long_sketch import (
    DEFAULT_DESIGN_N,
    DEFAULT_V,
    LdcaConfig,
    LdcaSketch,
    check_noise,
    keep_table,
    ldc_estimate,
    plan_rows,
)
from .short_sketch import DEFAULT_RESTORE_CAP, SeavConfig, SeavSketch, sort_candidates

DEFAULT_BETA = 0.8


@dataclass(frozen=True)
class DetectionReport:
    ip: int
    estimated_cardinality: float
    saturated: bool
    window_id: int
    source: str = "discrete"


@dataclass
class DetectorParams:
    theta: int = 1024
    r: int = 4
    sr: int = 4
    a: int = 2
    g: int = 8
    k: int = 8192
    lr: int | None = None
    lc: int | None = None
    v: int = DEFAULT_V
    design_n: float = DEFAULT_DESIGN_N
    beta: float = DEFAULT_BETA
    master_seed: int = DEFAULT_MASTER_SEED
    restore_cap: int = DEFAULT_RESTORE_CAP
    addr_bits: int = 32

    def seav_config(self) -> SeavConfig:
        return SeavConfig(r=self.r, sr=self.sr, a=self.a, theta=self.theta, g=self.g,
                          addr_bits=self.addr_bits)

    def ldca_config(self) -> LdcaConfig:
        lr, lc = self.lr, self.lc
        if lr is None:
            lr, lc = plan_rows(self.v, self.design_n, self.k)
        elif lc is None:
            lc = self.v // lr
        check_noise(self.k, self.design_n, lc, lr)
        return LdcaConfig(lr=lr, lc=lc, k=self.k)


_KEEP_CACHE: dict = {}


def device_keep_table(k: int, cutoff: float):
    """Cached device copy of keep_table(k, cutoff)."""
    import torch

    from ._device import device

    key = (k, cutoff, torch.cuda.current_device())
    t = _KEEP_CACHE.get(key)
    if t is None:
        t = torch.from_numpy(keep_table(k, cutoff)).to(device())
        _KEEP_CACHE[key] = t
    return t


def filter_candidates(seav: SeavSketch, ldca_buf, params_block, k: int, cutoff: float,
                      on_overflow: str = "warn", sliding=None):
    """Device restore -> sort -> z0 filter -> stable compaction.

    Returns host lists (ips, z0s) of the kept candidates, sorted by ip, and
    warns (or raises) once per overflowed register array like
    SeavSketch.restore(on_overflow) (short_sketch.py:392-408).
    `sliding` = (pool, ts_bytes, now_wrapped, window) to read the LDCA from
    a timestamp pool instead of a packed buffer.
    """
    import torch

    from ._device import call, stream_ptr
    from .errors import SeaOverflowError

    ip, aux, overflow = seav._restore_device(0, 1 << seav.config.r)
    n = ip.numel()
    flagged = np.nonzero(overflow.cpu().numpy())[0].tolist()
    for rp in flagged:
        err = SeaOverflowError(rp, seav.restore_cap)
        if on_overflow != "warn":
            raise err
        warnings.warn(str(err), RuntimeWarning, stacklevel=3)
    if n == 0:
        return [], []
    dev = ip.device
    table = device_keep_table(k, cutoff)
    z0 = torch.empty(n, dtype=torch.int32, device=dev)
    keep = torch.empty(n, dtype=torch.uint8, device=dev)
    if sliding is None:
        call("sspd_filter", ldca_buf.data_ptr(), params_block, ip.data_ptr(), n, table.data_ptr(),
             z0.data_ptr(), keep.data_ptr(), stream_ptr())
    else:
        pool, ts_bytes, now_w, window = sliding
        call("sspd_filter_sliding", pool.data_ptr(), ts_bytes, params_block, now_w, window,
             ip.data_ptr(), n, table.data_ptr(), z0.data_ptr(), keep.data_ptr(), stream_ptr())
    ip_out = torch.empty(n, dtype=torch.int32, device=dev)
    z0_out = torch.empty(n, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    call("sspd_compact_reports", ip.data_ptr(), z0.data_ptr(), keep.data_ptr(), n, ip_out.data_ptr(),
         z0_out.data_ptr(), cnt.data_ptr(), None, None, stream_ptr())
    m = int(cnt.item())
    ips = ip_out[:m].cpu().numpy().view(np.uint32).tolist()
    z0s = z0_out[:m].cpu().numpy().view(np.uint32).tolist()
    return ips, z0s


@dataclass
class DetectorState:
    seav: SeavSketch
    ldca: LdcaSketch
    window_id: int = 0
    pair_count: int = 0
    params: DetectorParams = field(default_factory=DetectorParams)

    @classmethod
    def create(cls, params: DetectorParams | None = None) -> "DetectorState":
        params = params or DetectorParams()
        seeds = SeedFamily(params.master_seed)
        scfg = params.seav_config()
        lcfg = params.ldca_config()
        seav = SeavSketch(scfg, seeds, restore_cap=params.restore_cap, _ldca_config=lcfg)
        ldca = LdcaSketch(lcfg, seeds, _seav_config=scfg)
        return cls(seav=seav, ldca=ldca, params=params)

    @property
    def theta(self) -> int:
        return self.seav.config.theta

    def memory_bytes(self) -> tuple[int, int]:
        return self.seav.memory_bytes(), self.ldca.memory_bytes()

    def process_pair(self, hip: int, oip: int):
        self.process_batch(np.array([hip], dtype=np.uint64), np.array([oip], dtype=np.uint64))

    def process_batch(self, hips, oips):
        """K1: one fused pass updating both sketches (window_detector.py:100-103)."""
        from ._device import call, ips_to_device, stream_ptr
        from .errors import ConfigError

        h = ips_to_device(hips, "hips")
        o = ips_to_device(oips, "oips")
        if h.numel() != o.numel():
            raise ConfigError("hips and oips differ in length")
        call("sspd_scan_discrete", h.data_ptr(), o.data_ptr(), h.numel(), self.seav._params,
             self.seav.device_buffer().data_ptr(), self.ldca.device_buffer().data_ptr(), stream_ptr())
        self.pair_count += int(h.numel())

    def finalize_window(self, beta: float | None = None, source: str = "discrete") -> list[DetectionReport]:
        beta = self.params.beta if beta is None else beta
        cutoff = beta * self.theta
        k = self.ldca.config.k
        ips, z0s = filter_candidates(self.seav, self.ldca.device_buffer(), self.seav._params, k, cutoff)
        reports = []
        for ip, z0 in zip(ips, z0s):
            est, saturated = ldc_estimate(z0, k)
            reports.append(DetectionReport(ip=ip, estimated_cardinality=est, saturated=saturated,
                                           window_id=self.window_id, source=source))
        return reports

    def reset(self):
        self.seav.clear()
        self.ldca.clear()
        self.window_id += 1
        self.pair_count = 0


def process_pair(state: DetectorState, hip: int, oip: int) -> DetectorState:
    state.process_pair(hip, oip)
    return state


def finalize_window(state: DetectorState, theta: int | None = None, beta: float = DEFAULT_BETA):
    if theta is not None and theta != state.theta:
        raise ValueError(f"detector was configured with theta={state.theta}, got {theta}")
    return state.finalize_window(beta=beta)


def reset(state: DetectorState) -> DetectorState:
    state.reset()
    return state
