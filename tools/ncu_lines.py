"""Per-source-line summary of an ncu --import-source report: warp-stall samples and executed
warp instructions of one kernel, top lines first.  Usage: ncu_lines.py REPORT KERNEL [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
isamp, iins = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) == len(hdr) and r[0] not in ("", "Line No"):
        try:
            lines.append((int(r[isamp]), int(r[iins]), r[0], r[1][:110]))
        except ValueError:
            pass
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"{kern}: {ts} stall samples, {ti / 1e9:.3f} G warp instructions")
for s, i, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins  L{ln:>5} {src}")
