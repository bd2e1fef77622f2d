#!/bin/bash
# On the GPU box: bench each _variants/NAME.so in place of the product library (restored after).
#   gpurun -- 'bash tools/variant_sweep.sh NAME1 NAME2 ...'
cp paper_2604_21072_b200/libbbcodec.so /tmp/libbbcodec.orig.so
mkdir -p gpurun_out
for v in "$@"; do
  cp _variants/$v.so paper_2604_21072_b200/libbbcodec.so
  timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw_$v.json 2>gpurun_out/sw_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/sw_$v.json')); s=d['stages_ms_per_step']
print('$v', round(d['value'],3), round(d['ms_per_step'],2),
      {k.replace('deflate.','d.').replace('inflate.','i.'):round(v,2) for k,v in s.items() if v > 0.9}, d['lossless'])" \
    || echo "$v failed"
done
cp /tmp/libbbcodec.orig.so paper_2604_21072_b200/libbbcodec.so
