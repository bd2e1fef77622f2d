# K4G vs the classic K4 walk on every workload: ms/step, value, the K4 stages, parity flags
for w in ${WORKLOADS:-config1 config2 config3 config4 config5}; do
  for v in ${VARIANTS:-"" BB_K4_CLASSIC=1}; do
    env $v timeout 600 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$w" "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
st = d.get("stages_ms_per_step") or {}
k4 = {k[8:]: round(v, 3) for k, v in st.items() if k.startswith(("deflate.gram", "deflate.profile", "deflate.k4"))}
print(sys.argv[1], f"[{sys.argv[2]}]", round(d["ms_per_step"], 3), round(d["value"], 3), d.get("unit"), k4,
      d.get("lossless"), (d.get("bit_exact_timed_step") or {}).get("match"))
PY
  done
done
