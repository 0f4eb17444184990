"""Opt-in tracing of the device path (SURVEY.md §5 "tracing/profiling").

With `SSPD_NVTX=1` in the environment every window-level operation pushes an
NVTX range ("sspd.scan", "sspd.finalize", "sspd.observe", "sspd.detect",
"sspd.merge", ...), so `ncu --nvtx --nvtx-include "sspd.finalize/"` (or any
NVTX-aware timeline tool) can select the kernels of one stage.  Off by
default: the ranges cost ~1 µs of host time each.
"""

from __future__ import annotations

import contextlib
import os

_ENABLED = os.environ.get("SSPD_NVTX", "") not in ("", "0")


def enabled() -> bool:
    return _ENABLED


@contextlib.contextmanager
def nvtx(name: str):
    """NVTX range `sspd.<name>` around the enclosed host code (no-op unless enabled)."""
    if not _ENABLED:
        yield
        return
    import torch

    torch.cuda.nvtx.range_push(f"sspd.{name}")
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()


def traced(name: str):
    """Method decorator: run the call inside `nvtx(name)` when enabled."""

    def wrap(fn):
        if not _ENABLED:
            return fn
        import functools

        @functools.wraps(fn)
        def inner(*args, **kwargs):
            with nvtx(name):
                return fn(*args, **kwargs)

        return inner

    return wrap
