"""Reference-side binding: run the reference package's own call sites on the
B200 path.

The reference (`sspd`, pure Python + numpy) has no FFI; its Python API is
the plug-in surface.  `install()` rebinds the module globals
through which the reference's callers reach that API -- the CLI
(`cli.py:206-300`: `_detect_windows`, `cmd_slide`, `cmd_distsim`), the
topology simulation (`distributed.py:231-292`) and the evaluation oracle --
to this package's device classes, so an unmodified `sspd` program runs its
scans, restores, filters and merges on the GPU.  This is the shim
INTEGRATION.md §1 documents; tests/test_gpu_refshim.py runs the reference
CLI with and without it and compares the output files byte for byte.
"""

from __future__ import annotations

_SAVED: dict = {}


def install() -> None:
    """Point the imported reference package at the B200 implementation
    (idempotent).  Import the reference first (e.g. with baseline/_ref on
    sys.path)."""
    import sspd.cli as cli
    import sspd.distributed as di
    import sspd.evaluation as ev
    import sspd.sliding as sl
    import sspd.window_detector as wd

    import paper_1901_07306_b200 as b200

    binds = [
        (wd, "DetectorState", b200.DetectorState), (wd, "DetectorParams", b200.DetectorParams),
        (di, "DetectorState", b200.DetectorState), (di, "DetectorParams", b200.DetectorParams),
        (cli, "DetectorState", b200.DetectorState), (cli, "DetectorParams", b200.DetectorParams),
        (sl, "SlidingDetector", b200.SlidingDetector), (cli, "SlidingDetector", b200.SlidingDetector),
        (sl, "TimestampPool", b200.TimestampPool),
        (di, "merge_frames", b200.merge_frames), (di, "merge_timestamp_pools", b200.merge_timestamp_pools),
        (di, "simulate_window", b200.simulate_window), (di, "simulate_topology", b200.simulate_topology),
        (cli, "simulate_topology", b200.simulate_topology),
        (ev, "ExactOracle", b200.ExactOracle), (cli, "ExactOracle", b200.ExactOracle),
    ]
    for mod, name, obj in binds:
        key = (mod.__name__, name)
        if key not in _SAVED:
            _SAVED[key] = getattr(mod, name, None)
        setattr(mod, name, obj)


def uninstall() -> None:
    """Restore the reference's own bindings."""
    import importlib

    for (modname, name), obj in _SAVED.items():
        setattr(importlib.import_module(modname), name, obj)
    _SAVED.clear()
