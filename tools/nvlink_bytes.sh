#!/bin/bash
# NVLink bytes moved by a command (nvidia-smi nvlink throughput counters, data payload, all links of
# every GPU), read before and after it: evidence of what the multi-GPU hand-off puts on NVLink.
#   tools/nvlink_bytes.sh OUT.txt -- <command...>
out=$1; shift; [ "$1" = "--" ] && shift
nvidia-smi nvlink -gt d > "$out.before" 2>&1
"$@"
rc=$?
nvidia-smi nvlink -gt d > "$out.after" 2>&1
python3 - "$out.before" "$out.after" > "$out" <<'PY'
import re, sys
def parse(p):
    cur, d = None, {}
    for ln in open(p):
        m = re.match(r"GPU (\d+):", ln)
        if m: cur = int(m.group(1)); continue
        m = re.search(r"Link (\d+): Data (Tx|Rx): (\d+) KiB", ln)
        if m and cur is not None:
            d[(cur, m.group(2))] = d.get((cur, m.group(2)), 0) + int(m.group(3))
    return d
a, b = parse(sys.argv[1]), parse(sys.argv[2])
for k in sorted(b):
    print(f"GPU {k[0]} {k[1]}: {(b[k] - a.get(k, 0)) / 1024**2:.3f} GiB")
PY
exit $rc
