"""Run the REFERENCE command line (`sspd`, from baseline/_ref) -- unmodified,
or with the B200 binding installed first (`--b200`: refshim.install()).

    python tools/run_ref_cli.py [--b200] <sspd arguments...>

Used by tests/test_gpu_refshim.py to compare the reference CLI's output
files with and without the GPU path behind its own call sites."""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(1, str(ROOT))

if __name__ == "__main__":
    argv = sys.argv[1:]
    if argv and argv[0] == "--b200":
        argv = argv[1:]
        import sspd  # noqa: F401  (the reference package must be imported first)

        from paper_1901_07306_b200 import refshim

        refshim.install()
    from sspd.cli import main

    sys.exit(main(argv))
