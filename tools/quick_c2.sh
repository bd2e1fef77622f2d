# parity tests of the encoder + one config2 bench line (K4 stages); args: extra pytest files
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_deflate.py tests/test_gpu_fullsize.py $@ -x -q -m gpu > gpurun_out/t_q.log 2>&1; tail -2 gpurun_out/t_q.log
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_q.log 2>&1
tail -1 gpurun_out/b_q.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(round(d['ms_per_step'],2), round(d['value'],3), d['bit_exact_timed_step']['match'], {k:round(v,2) for k,v in d['stages_ms_per_step'].items() if v>0.5})"
