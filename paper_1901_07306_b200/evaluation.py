"""Ground truth and accuracy metrics at GPU scale.

Drop-in for the reference's `ExactOracle` and metric helpers
(sspd/evaluation.py:32-97).  The sort-unique of the (hip << 32 | oip) keys
runs on the GPU (csrc/exact.cu, `sspd_exact_cardinalities`), so configs
2-5 (2^28+ packets) get their truth set in milliseconds instead of a
host-side np.unique; `hosts`/`counts` are then host arrays exactly as the
reference holds them (hosts ascending uint32, counts int64).  The metric
functions are the reference's host set arithmetic (FPR, FNR and their sum
FTR, all normalised by the TRUE super-point count, evaluation.py:73-97).
"""

from __future__ import annotations

import ctypes

import numpy as np

from .errors import UndefinedMetricError


class ExactOracle:
    """Exact per-host distinct opposite-IP counts (evaluation.py:32-58).

    `hips`/`oips` may be numpy arrays or device tensors (no host copy is
    made of device inputs).  Computed on the GPU; raises DeviceError when
    no GPU / library is present (there is no CPU fallback)."""

    def __init__(self, hips, oips):
        import torch

        from ._device import call, ips_to_device, stream_ptr

        h = ips_to_device(hips, "hips")
        o = ips_to_device(oips, "oips")
        if h.numel() != o.numel():
            raise ValueError("hips and oips must have the same length")
        n = int(h.numel())
        need = ctypes.c_size_t(0)
        call("sspd_exact_cardinalities", h.data_ptr(), o.data_ptr(), n, None, None, None, None,
             ctypes.byref(need), stream_ptr())
        scratch = torch.empty(max(256, need.value), dtype=torch.uint8, device=h.device)
        hosts = torch.empty(max(1, n), dtype=torch.int32, device=h.device)
        counts = torch.empty(max(1, n), dtype=torch.int32, device=h.device)
        n_hosts = torch.zeros(1, dtype=torch.int64, device=h.device)
        call("sspd_exact_cardinalities", h.data_ptr(), o.data_ptr(), n, hosts.data_ptr(), counts.data_ptr(),
             n_hosts.data_ptr(), scratch.data_ptr(), ctypes.byref(need), stream_ptr())
        m = int(n_hosts.item())
        del scratch
        self.hosts = hosts[:m].cpu().numpy().view(np.uint32).copy()
        self.counts = counts[:m].cpu().numpy().view(np.uint32).astype(np.int64)

    @classmethod
    def from_mapping(cls, cardinalities: dict[int, int]) -> "ExactOracle":
        oracle = cls.__new__(cls)
        items = sorted(cardinalities.items())
        oracle.hosts = np.array([ip for ip, _ in items], dtype=np.uint32)
        oracle.counts = np.array([c for _, c in items], dtype=np.int64)
        return oracle

    def cardinality(self, hip: int) -> int:
        i = np.searchsorted(self.hosts, hip)
        if i < len(self.hosts) and self.hosts[i] == hip:
            return int(self.counts[i])
        return 0

    def superpoints(self, theta: int) -> list[int]:
        """Hosts with at least theta distinct opposite IPs, sorted."""
        return [int(ip) for ip in self.hosts[self.counts >= theta]]


def oracle_superpoints(oracle: ExactOracle, theta: int) -> list[int]:
    return oracle.superpoints(theta)


def metrics(detected: list[int], truth: list[int]) -> tuple[float, float, float]:
    """(FPR, FNR, FTR), all normalised by the true super-point count
    (evaluation.py:73-81)."""
    truth_set = set(truth)
    if not truth_set:
        raise UndefinedMetricError("metrics are undefined for an empty truth set")
    detected_set = set(detected)
    fpr = len(detected_set - truth_set) / len(truth_set)
    fnr = len(truth_set - detected_set) / len(truth_set)
    return fpr, fnr, fpr + fnr


def metrics_report(detected: list[int], truth: list[int]) -> dict[str, float]:
    """Metrics plus a conventional precision figure (evaluation.py:84-97)."""
    fpr, fnr, ftr = metrics(detected, truth)
    detected_set, truth_set = set(detected), set(truth)
    precision = (len(detected_set & truth_set) / len(detected_set)) if detected_set else 1.0
    return {
        "fpr": fpr,
        "fnr": fnr,
        "ftr": ftr,
        "precision_nonpaper": precision,
        "detected": float(len(detected_set)),
        "truth": float(len(truth_set)),
    }
