# A/B of decoder stage times: bench.py configs under env switches (stage ms per step)
# usage: bash tools/stage_ab.sh "" "BB_X=1" "BB_Y=1"   (each argument one variant; "" = defaults)
mkdir -p gpurun_out
show() { python -c "
import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);st=d['stages_ms_per_step']
print(sys.argv[2], round(d['ms_per_step'],3), {k[8:]:round(v,3) for k,v in st.items() if k.startswith(__import__('os').environ.get('STAGES','inflate'))})" $1 "$2"; }
for w in ${WORKLOADS:-config1 config2}; do
  for v in "$@"; do
    env $v python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; show gpurun_out/ab.json "$w [$v]"
  done
done
