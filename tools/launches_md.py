"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as a markdown table.

usage: python tools/launches_md.py profiles/r1_launches_config2.csv STEPS "COMMAND" > profiles/r1_launches_config2.md
STEPS = bench steps inside the capture (timed + warm-up), used for the per-step column.
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    path, steps, cmd = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = [ln for ln in open(path) if ln.startswith('"')]
    data = list(csv.DictReader(rows))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in data:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"^bb::(<unnamed>::)?", "", name)
        name = name.split("(")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}[r["Metric Unit"]]
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
    total = sum(tot.values())
    print(f"# ncu launch list: `{cmd}` ({steps} steps incl. warm-up)")
    print("# `ncu --metrics gpu__time_duration.sum --clock-control none -c 600`; cold-cache and serialised by ncu:")
    print(f"# compare SHARES with the live bench stage timing, not absolutes.  Raw csv: {path.split('/')[-1]}")
    print(f"# total {total:.1f} ms over {steps} steps\n")
    print("| kernel | total ms | launches | ms / step | share |")
    print("|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k[:60]} | {tot[k]:.3f} | {cnt[k]} | {tot[k] / steps:.3f} | {100 * tot[k] / total:.1f}% |")


if __name__ == "__main__":
    main()
