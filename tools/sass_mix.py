"""Opcode mix of a SASS span (ALU vs FMA pipe issue balance).

usage: python tools/sass_mix.py CUBIN FUNCTION [MARKER]
Counts the instructions of FUNCTION between the first and last line holding
MARKER (default: the SplitMix64 multiplier 0x1ce4e5b9, i.e. the hashing
region) and groups them by the pipe they issue to (B300_MICROARCH.md: IMAD on
the fma pipe, IADD3/LOP3/SHF on the alu pipe; both take 2 cycles per warp
instruction per SMSP, so a span needs max(N, 2*alu, 2*fma) issue cycles).
"""
import re
import subprocess
import sys
from collections import Counter

ALU = {"IADD3", "LOP3", "SHF", "ISETP", "SEL", "LEA", "PRMT", "IABS", "IMNMX", "VIMNMX", "FMNMX", "SHL", "SHR", "PLOP3",
       "MOV", "FLO", "POPC", "BREV", "LEA.HI"}
FMA = {"IMAD", "FFMA", "FMUL", "FADD", "HFMA2", "IMUL", "IDP"}


def main():
    cubin, fn = sys.argv[1], sys.argv[2]
    marker = sys.argv[3] if len(sys.argv) > 3 else "0x1ce4e5b9"
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, cubin], capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
    idx = [i for i, l in enumerate(lines) if marker in l]
    span = lines[idx[0]:idx[-1] + 1] if idx else lines
    c = Counter()
    for l in span:
        body = re.sub(r"^\s+/\*[0-9a-f]+\*/\s+", "", l)
        body = re.sub(r"^@!?U?P\w+\s+", "", body)
        op = body.split()[0].rstrip(";").split(".")[0]
        c[op] += 1
    alu = sum(v for k, v in c.items() if k in ALU)
    fma = sum(v for k, v in c.items() if k in FMA)
    n = sum(c.values())
    print(f"span {len(span)} instr: alu {alu} fma {fma} other {n - alu - fma} -> issue-cycle bound "
          f"{max(n, 2 * alu, 2 * fma)} (N {n}, 2*alu {2 * alu}, 2*fma {2 * fma}); hashes (marker) {len(idx)}")
    print(" ".join(f"{k}:{v}" for k, v in c.most_common(16)))


if __name__ == "__main__":
    main()
