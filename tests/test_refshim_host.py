"""The reference-side binding (paper_1901_07306_b200.refshim) rebinds the
reference package's call sites without touching the GPU."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.skipif(not (REF / "sspd" / "cli.py").exists(),
                                reason="reference package not installed in baseline/_ref")


def test_refshim_rebinds_reference_globals():
    """install() points the reference's call sites at the B200 classes and
    uninstall() restores them (no GPU work)."""
    sys.path.insert(0, str(REF))
    try:
        import sspd.cli as cli
        import sspd.window_detector as wd

        import paper_1901_07306_b200 as b200
        from paper_1901_07306_b200 import refshim

        orig = wd.DetectorState
        refshim.install()
        assert wd.DetectorState is b200.DetectorState and cli.SlidingDetector is b200.SlidingDetector
        assert cli.simulate_topology is b200.simulate_topology
        refshim.uninstall()
        assert wd.DetectorState is orig
    finally:
        sys.path.remove(str(REF))
        for m in [m for m in sys.modules if m == "sspd" or m.startswith("sspd.")]:
            del sys.modules[m]
