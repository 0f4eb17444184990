"""Time the REFERENCE implementation itself (the installed pure-Python
`sspd` package in baseline/_ref) on the host CPU -- bench.py's
`cpu_baseline.reference_python` (SURVEY.md §8(d) CPU baseline items 1-2).

  * single process: DetectorState.process_batch in 65,536-pair buffers (the
    `sspd detect` default, cli.py:215-217) over a prefix of the workload,
    then finalize_window (window_detector.py:100-125);
  * P processes: every process is one watch point scanning its own
    prefix-sized slice, serialize()s both sketches; the parent parses the
    frames, merge_frames()s them and finalizes once (distributed.py:81-173).

This is a measurement tool for the baseline only: it never touches the
CUDA product, and it reads the reference from baseline/_ref (installed with
pip from the reference source), never from /root/reference.
"""

from __future__ import annotations

import multiprocessing as mp
import sys
import time
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
BUFFER_PAIRS = 65_536  # cli.py default buffer (RunConfig.buffer_pairs)


def available() -> bool:
    return (REF / "sspd" / "__init__.py").exists()


def _import_ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import sspd  # noqa: F401  (the reference package)
    from sspd.distributed import merge_frames, parse_frame, serialize
    from sspd.window_detector import DetectorParams, DetectorState

    return DetectorParams, DetectorState, serialize, parse_frame, merge_frames


def _params(geom: dict):
    DetectorParams = _import_ref()[0]
    return DetectorParams(**geom)


def _scan(state, hips, oips):
    for lo in range(0, len(hips), BUFFER_PAIRS):
        state.process_batch(hips[lo:lo + BUFFER_PAIRS], oips[lo:lo + BUFFER_PAIRS])


def _worker(args):
    geom, hips, oips = args
    DetectorParams, DetectorState, serialize, _, _ = _import_ref()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(DetectorParams(**geom))
    _scan(st, hips, oips)
    return serialize(st.seav, 0), serialize(st.ldca, 0)


def time_single(geom: dict, hips, oips) -> dict:
    """Mpps of the reference's process_batch + finalize_window, one process."""
    _, DetectorState, _, _, _ = _import_ref()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        st = DetectorState.create(_params(geom))
        t0 = time.perf_counter()
        _scan(st, hips, oips)
        reps = st.finalize_window()
        dt = time.perf_counter() - t0
    return {"value": round(len(hips) / dt / 1e6, 4), "unit": "Mpps", "cores": 1, "packets": len(hips),
            "seconds": round(dt, 3), "reports": len(reps)}


def time_multi(geom: dict, slices: list, procs: int) -> dict:
    """P watch-point processes (one slice each) + serialize -> merge_frames ->
    finalize on the parent.  The pool is started (and the reference imported
    in every worker) before the clock starts."""
    _, DetectorState, _, parse_frame, merge_frames = _import_ref()
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_import_ref_noop, range(procs))
        t0 = time.perf_counter()
        frames = pool.map(_worker, [(geom, h, o) for h, o in slices])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            seav, ldca = merge_frames([parse_frame(f) for pair in frames for f in pair])
            st = DetectorState(seav=seav, ldca=ldca, params=_params(geom))
            reps = st.finalize_window()
        dt = time.perf_counter() - t0
    n = sum(len(h) for h, _ in slices)
    return {"value": round(n / dt / 1e6, 4), "unit": "Mpps", "cores": procs, "packets": n,
            "seconds": round(dt, 3), "reports": len(reps)}


def _import_ref_noop(_):
    _import_ref()
    return 0
