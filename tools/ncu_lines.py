"""Per-source-line instruction and stall shares from an ncu report (dev tool).

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 45
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hd = None
out = []
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hd = r
        continue
    if hd and len(r) == len(hd) and r[0]:
        try:
            out.append((cur, int(r[0]), r[1].strip(), float(r[4] or 0), float(r[7] or 0)))
        except ValueError:
            pass
ti = sum(o[4] for o in out) or 1
ts = sum(o[3] for o in out) or 1
print(f"total warp instructions {ti:.3e}")
for o in sorted(out, key=lambda o: -o[4])[:n]:
    print(f"{o[0][:12]:12s}:{o[1]:4d} ins {100 * o[4] / ti:5.1f}% smp {100 * o[3] / ts:5.1f}%  {o[2][:90]}")
