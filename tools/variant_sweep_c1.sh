#!/bin/bash
# variant_sweep.sh for the config1 workload (1 MiB, latency bound)
cp paper_2604_21072_b200/libbbcodec.so /tmp/libbbcodec.orig.so
mkdir -p gpurun_out
for v in "$@"; do
  cp _variants/$v.so paper_2604_21072_b200/libbbcodec.so
  timeout 300 python bench.py --workload config1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/swc1_$v.json 2>gpurun_out/swc1_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/swc1_$v.json').read().strip().splitlines()[-1]); s=d['stages_ms_per_step']
print('$v', round(d['value'],3), round(d['ms_per_step'],3), {k:round(v,3) for k,v in s.items() if v > 0.05}, d['lossless'], d['bit_exact_timed_step'])" \
    || echo "$v failed"
done
cp /tmp/libbbcodec.orig.so paper_2604_21072_b200/libbbcodec.so
