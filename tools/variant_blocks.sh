# On the GPU box: K6 (blocks_trees) per library variant on config2 and config1
cp paper_2604_21072_b200/libbbcodec.so /tmp/libbbcodec.orig.so
for v in "$@"; do
  [ "$v" = cur ] && cp /tmp/libbbcodec.orig.so paper_2604_21072_b200/libbbcodec.so || cp _variants/$v.so paper_2604_21072_b200/libbbcodec.so
  for w in config2 config1; do
    timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms_per_step']
print('$v', '$w', round(d['ms_per_step'],3), 'blocks', round(s['deflate.blocks_trees'],3), d['lossless'], d['bit_exact_timed_step']['match'])"
  done
done
cp /tmp/libbbcodec.orig.so paper_2604_21072_b200/libbbcodec.so
