# A/B of prebuilt library variants (_variants/<name>.so) on bench configs ("name" or "name:points") -> stdout
for c in ${CONFIGS:-cluster2B scene500M}; do
 name=${c%%:*}; pts=""; [ "$name" != "$c" ] && pts="--points ${c##*:}"
 for lib in ${LIBS:-base match}; do
  cp _variants/$lib.so paper_2302_14801_b200/_lib/liblodb200.so
  timeout 600 python bench.py --config $name $pts --steps 5 --warmup 3 --stages --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  LABEL="$c $lib" python - <<'PY'
import json, os
d = json.loads(open("gpurun_out/ab.json").read())
print(os.environ["LABEL"], round(d["value"] / 1e9, 3), round(d["ms_per_step"], 3), [round(x, 2) for x in d["stages_ms"].values()],
      "scatter", round(d["roofline"]["ms_per_build"], 2))
PY
 done
done
cp _variants/base.so paper_2302_14801_b200/_lib/liblodb200.so
