"""Reference-side integration: the reference's OWN command line (`sspd`,
pip-installed from its source into baseline/_ref) run unmodified on the
CPU and with the B200 binding installed (paper_1901_07306_b200.refshim,
the shim INTEGRATION.md §1 documents), on the same trace files.  The
report CSVs of `detect` (cli.py:206-233), `slide` (cli.py:236-257) and
`distsim` (cli.py:260-300, hash and round-robin routing) and the distsim
merge-equivalence log must be byte-identical.

The config-1 stream (BASELINE configs[0]) is written as a 600-slice
reference trace file (two 300-slice windows)."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "sspd" / "cli.py").exists(),
                                 reason="reference package not installed in baseline/_ref")]


def _cli(args, b200: bool):
    cmd = [sys.executable, str(ROOT / "tools" / "run_ref_cli.py")] + (["--b200"] if b200 else []) + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (b200, r.stdout[-2000:], r.stderr[-4000:])
    return r.stdout


@pytest.fixture(scope="module")
def traces(tmp_path_factory):
    d = tmp_path_factory.mktemp("traces")
    code = f"""
import sys
import numpy as np
sys.path.insert(0, {str(REF)!r}); sys.path.insert(1, {str(ROOT)!r})
from sspd.evaluation import Trace, write_trace
from tools.workloads import CONFIG1, generate
h, o, _ = generate(CONFIG1)
n = len(h)
write_trace(Trace(slices=(np.arange(n, dtype=np.uint64) * 600 // n).astype(np.uint32), hips=h, oips=o,
                  truth={{}}), {str(d / "c1.bin")!r})
m = 200_000
write_trace(Trace(slices=(np.arange(m, dtype=np.uint64) * 60 // m).astype(np.uint32), hips=h[:m], oips=o[:m],
                  truth={{}}), {str(d / "slide.bin")!r})
"""
    subprocess.run([sys.executable, "-c", code], check=True, timeout=600)
    return d


@pytest.mark.parametrize("cmd", ["detect", "distsim-hash", "distsim-rr", "slide"])
def test_reference_cli_output_bytes_equal_with_b200_binding(cuda, traces, tmp_path, cmd):
    outs = {}
    for b200 in (False, True):
        tag = "gpu" if b200 else "cpu"
        out = tmp_path / f"{cmd}_{tag}.csv"
        if cmd == "detect":
            args = ["detect", "--trace", str(traces / "c1.bin"), "--out", str(out)]
        elif cmd.startswith("distsim"):
            log = tmp_path / f"{cmd}_{tag}_merge.txt"
            args = ["distsim", "--trace", str(traces / "c1.bin"), "--out", str(out), "--merge-log", str(log),
                    "--n-wp", "4", "--route", "hash" if cmd.endswith("hash") else "round-robin",
                    "--frames-dir", str(tmp_path / f"frames_{tag}")]
        else:
            args = ["slide", "--trace", str(traces / "slide.bin"), "--out", str(out), "--window-slices", "10",
                    "--detect-every", "3", "--r", "8", "--k", "1024", "--lr", "4", "--lc", "128", "--theta", "64"]
        stdout = _cli(args, b200).replace(str(out), "<out>")
        outs[tag] = (out.read_bytes(), stdout)
        if cmd.startswith("distsim"):
            outs[tag] += (log.read_bytes(),)
    assert outs["gpu"][0] == outs["cpu"][0]  # report CSV bytes
    assert outs["gpu"][1] == outs["cpu"][1]  # the CLI's own summary line
    assert outs["cpu"][0].count(b"\n") > 10
    if cmd.startswith("distsim"):
        assert outs["gpu"][2] == outs["cpu"][2]  # merge-equivalence log (bit-identity vs single scanner)
        frames = sorted(p.name for p in (tmp_path / "frames_gpu").iterdir())
        assert frames == sorted(p.name for p in (tmp_path / "frames_cpu").iterdir())
        for name in frames:  # the watch points' serialized frames (CRC-32 from the device)
            assert (tmp_path / "frames_gpu" / name).read_bytes() == (tmp_path / "frames_cpu" / name).read_bytes()
