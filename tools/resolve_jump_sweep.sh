#!/bin/bash
# On the GPU box: parity tests with the default jump-round cap, then config2/config3 benches
# for several caps on the pointer-doubling rounds (BB_RESOLVE_JUMPS) of the inflate resolve,
# with the sampled mean chain length printed (BB_RESOLVE_DEBUG).
#   gpurun -- 'bash tools/resolve_jump_sweep.sh 0 4 6'
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_deflate.py tests/test_gpu_specdec.py tests/test_gpu_kvchunk.py -x -q \
  > gpurun_out/jump_tests.log 2>&1; echo tests=$?
for w in config3 config2; do
  BB_RESOLVE_DEBUG=1 timeout 300 python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline --no-e2e 2>&1 \
    | grep "resolve:" | tail -n 2
done
for r in "$@"; do
  for w in config3 config2; do
    BB_RESOLVE_JUMPS=$r timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/jump_${w}_$r.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/jump_${w}_$r.json').read().strip().splitlines()[-1]); s=d['stages_ms_per_step']
print('$w r=$r', round(d['value'],3), round(d['ms_per_step'],2), 'resolve', round(s['inflate.resolve'],2), d['lossless'])" \
      || echo "$w $r failed"
  done
done
