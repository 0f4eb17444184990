"""Summarise ncu CSV metric dumps of the scan kernels into
profiles/scan_ncu_summary.json (read by bench.py for the `traffic` and
issue-roofline fields).

    python tools/ncu_summary.py <kernel-key> <packets> <ncu --csv metrics file> [...]

kernel-key: "partitioned" or "direct".
"""

import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles" / "scan_ncu_summary.json"
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "": 1, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "request": 1}


def parse(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, ni, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    out: dict = {}
    for r in rows[hi + 1:]:
        if "scan_" not in r[ki]:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        out.setdefault(r[ni], []).append(v)
    return {k: sum(v) / len(v) for k, v in out.items()}


def main():
    key, packets, path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    m = parse(path)
    summary = json.loads(OUT.read_text()) if OUT.exists() else {}
    summary[key] = {
        "packets_per_launch": packets,
        "duration_s": m.get("gpu__time_duration.sum"),
        "dram_bytes_per_packet": (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / packets,
        "dram_read_bytes_per_packet": m.get("dram__bytes_read.sum", 0) / packets,
        "dram_write_bytes_per_packet": m.get("dram__bytes_write.sum", 0) / packets,
        "warp_inst_per_packet": m.get("smsp__inst_executed.sum", 0) / packets,
        "l2_red_requests_per_packet": m.get("lts__t_requests_srcunit_tex_op_red.sum", 0) / packets,
        "issue_active_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "shared_atom_bank_conflict_frac": (m["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"] /
                                           m["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"])
        if m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum") else None,
        "source": f"ncu --metrics (profiles/{Path(path).name}), config-2 stream",
    }
    OUT.write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary[key], indent=1))


if __name__ == "__main__":
    main()
