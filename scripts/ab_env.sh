# A/B of environment switches on bench configs (CONFIGS entries "name" or "name:points") -> stdout
for c in ${CONFIGS:-cluster2B scene500M}; do
 name=${c%%:*}; pts=""; [ "$name" != "$c" ] && pts="--points ${c##*:}"
 for v in ${VARIANTS:-"X=0"}; do
  env $v timeout 600 python bench.py --config $name $pts --steps 5 --warmup 3 --stages --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  LABEL="$c $v" python - <<'PY'
import json, os
d = json.loads(open("gpurun_out/ab.json").read())
print(os.environ["LABEL"], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 3), [round(x, 2) for x in d["stages_ms"].values()])
PY
 done
done
