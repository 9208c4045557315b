"""Per-source-line instruction / stall breakdown of one kernel in an ncu report.

    python profiles/ncu_lines.py <report.ncu-rep> [top_n] [--ops] [--kernel REGEX]

Reads `ncu -i ... --page source --csv --print-source cuda,sass` (SASS rows
interleaved under their CUDA source line) and prints, per file:line, the share
of warp instructions executed and of stall samples, plus (--ops) the SASS
opcode mix. Used to attribute the search kernel's instructions per hop.
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict


def load(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
    kernel = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
    rows = load(rep, kernel)
    fname, hdr, cur = "?", None, None
    inst = defaultdict(float)
    samp = defaultdict(float)
    src = {}
    ops = defaultdict(float)
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:  # a CUDA source line
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()
            continue
        if cur is None or len(r) < len(hdr):
            continue
        try:
            n = float(r[hdr.index("Instructions Executed")] or 0)
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        inst[cur] += n
        samp[cur] += s
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        ops[op.split(".")[0]] += n
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
    print(f"{'file:line':24s} {'inst%':>6s} {'stall%':>6s}  source")
    for k in sorted(inst, key=lambda k: -inst[k])[:top]:
        print(f"{k[0][:14]:>14s}:{k[1]:<5d}   {100 * inst[k] / ti:5.1f}  {100 * samp[k] / ts:5.1f}   {src.get(k, '')[:90]}")
    if "--ops" in sys.argv:
        print("\nSASS opcode mix (share of warp instructions):")
        for op in sorted(ops, key=lambda o: -ops[o])[:30]:
            print(f"  {op:12s} {100 * ops[op] / ti:5.1f}%")


if __name__ == "__main__":
    main()
