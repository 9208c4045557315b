"""Summarize an ncu report (.ncu-rep) into a committed text file.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep profiles/<tag>.txt [launches.csv]
"""

import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active", "sm__maximum_warps_per_active_cycle_pct",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    lines = [f"# ncu summary of {rep}", ""]
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"## kernel: {name}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"{m:70s} {row[i]:>22s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    stalls.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in stalls) or 1
        lines.append("")
        lines.append("warp stall samples (share):")
        for v, h in sorted(stalls, reverse=True)[:12]:
            lines.append(f"  {h:32s} {100 * v / tot:5.1f}%")
        lines.append("")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    cur, hd, rows = None, None, []
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) == 2:
            continue
        if r and r[0] == "Line No":
            hd = r
            continue
        if hd and len(r) == len(hd) and r[0]:
            try:
                rows.append((cur, r[0], r[1].strip(), float(r[4] or 0), float(r[7] or 0)))
            except ValueError:
                pass
    ts = sum(r[3] for r in rows) or 1
    ti = sum(r[4] for r in rows) or 1
    lines.append("top source lines by stall samples (file:line samples% instructions% source):")
    for f, ln, s, smp, ins in sorted(rows, key=lambda r: -r[3])[:30]:
        lines.append(f"  {f[:14]:14s}:{ln:>4s} {100 * smp / ts:5.1f}% {100 * ins / ti:5.1f}%  {s[:90]}")
    if len(sys.argv) > 3:
        lines.append("")
        lines.append(f"launch list ({sys.argv[3]}): kernel, gpu__time_duration.sum")
        rr = list(csv.reader(open(sys.argv[3])))
        h = None
        for r in rr:
            if "Kernel Name" in r:
                h = r
                continue
            if h and len(r) == len(h):
                d = dict(zip(h, r))
                lines.append(f"  {d['Kernel Name'][:70]:70s} {d.get('Metric Value', '')} {d.get('Metric Unit', '')}")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
