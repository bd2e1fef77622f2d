#!/bin/bash
# variant_sweep.sh for any workload: WORKLOAD=config3 bash tools/variant_sweep_w.sh NAME...
w=${WORKLOAD:-config2}
cp paper_2604_21072_b200/libbbcodec.so /tmp/libbbcodec.orig.so
mkdir -p gpurun_out
for v in "$@"; do
  cp _variants/$v.so paper_2604_21072_b200/libbbcodec.so
  timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/sw_$v.json 2>gpurun_out/sw_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/sw_$v.json').read().strip().splitlines()[-1]); s=d['stages_ms_per_step']
print('$w $v', round(d['value'],3), round(d['ms_per_step'],2),
      {k.replace('deflate.','d.').replace('inflate.','i.'):round(v,2) for k,v in s.items() if k.startswith(__import__('os').environ.get('STAGES','inflate')) and v > 0.2}, d['lossless'])" \
    || echo "$v failed"
done
cp /tmp/libbbcodec.orig.so paper_2604_21072_b200/libbbcodec.so
